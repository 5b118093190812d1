// Top-k selection and cross-shard merge (a9).
//
// Order: distance ascending, ties by ascending global entity id (Q13).
// Distances map to order-preserving uint32 keys (NaN -> max, -0 -> +0), so (key, id) packed
// in a uint64 sorts exactly in that order.
//
// k_topk: one CTA per query row (or per 16k-entry chunk of a long row, the chunks then merged
// by k_merge); warp select with per-warp thresholds (see the kernel).
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "kgq_internal.cuh"

namespace kgq {

__device__ __forceinline__ uint32_t fkey(float f) {
  if (f != f) return 0xFFFFFFFFu;
  if (f == 0.0f) f = 0.0f;
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// In-place ascending bitonic sort of P (power of two) uint64 values in shared memory.
__device__ void bitonic_sort_u64(unsigned long long* v, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const unsigned long long a = v[lo], b = v[hi];
        if ((a > b) == up) {
          v[lo] = b;
          v[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

constexpr int kTopkThreads = 256;
constexpr int64_t kTopkStage = 16384;  // entries per CTA when a row is split

// Warp-cooperative ascending bitonic sort of P (power of two, >= 64) uint64 in shared memory.
__device__ __forceinline__ void warp_bitonic_sort(unsigned long long* v, int P) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < P / 2; i += 32) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const unsigned long long a = v[lo], b = v[hi];
        if ((a > b) == up) {
          v[lo] = b;
          v[hi] = a;
        }
      }
      __syncwarp();
    }
  }
}

// k_topk: CTA (b, c) selects the k best (distance, index) of row b restricted to
// [c*chunk, min(n, (c+1)*chunk)) and writes them at [(c*B + b)*k, ...).  With one chunk that is
// the final [B, k] answer; with several it is the candidate list k_merge reduces.
// Warp select: each warp streams a contiguous slice of the chunk with coalesced loads, keeps
// its k best packed keys (key << 32 | index: a strict total order = distance, then id) in
// shared memory, and only elements below its current k-th best go to a 32-entry buffer; a
// full buffer is merged by a warp bitonic sort.  In random order that is ~k ln(n/k) buffer
// entries per warp, so almost every element costs one load and one compare.  The warps' lists
// are then merged by one block-wide bitonic sort.
__global__ void __launch_bounds__(kTopkThreads)
    k_topk(const float* __restrict__ dist, int64_t ldd, int64_t n_total, int64_t chunk, int k,
           int64_t id_base, const int32_t* __restrict__ invalid, float* __restrict__ od,
           int32_t* __restrict__ oi, int B, int P) {
  extern __shared__ unsigned long long wl[];  // [warps][P] lists, then the block merge area
  const int b = blockIdx.x;
  const int64_t c0 = (int64_t)blockIdx.y * chunk;
  const int64_t n = (n_total - c0 < chunk ? n_total - c0 : chunk);
  const float* row = dist + (int64_t)b * ldd + c0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int W = kTopkThreads / 32;
  od += ((int64_t)blockIdx.y * B + b) * k;
  oi += ((int64_t)blockIdx.y * B + b) * k;
  if (invalid && invalid[b]) {
    for (int j = tid; j < k; j += blockDim.x) {
      od[j] = __uint_as_float(0x7FFFFFFFu);
      oi[j] = -1;
    }
    return;
  }
  unsigned long long* lst = wl + wid * P;  // [0, k) sorted best, [k, k+32) buffer, rest max
  for (int j = lane; j < P; j += 32) lst[j] = ~0ull;
  __syncwarp();
  unsigned long long tau = ~0ull;  // current k-th best of this warp (packed key)
  float tau_f = __uint_as_float(0x7F800000u);  // its distance (+inf while the list is short)
  int cnt = 0;
  auto merge = [&]() {
    warp_bitonic_sort(lst, P);
    for (int j = k + lane; j < P; j += 32) lst[j] = ~0ull;
    __syncwarp();
    tau = lst[k - 1];
    tau_f = tau == ~0ull ? __uint_as_float(0x7F800000u) : fkey_inv((uint32_t)(tau >> 32));
    cnt = 0;
  };
  constexpr int U = 8;  // loads in flight per lane (the loop is latency-bound otherwise)
  const int64_t per = ((n + W - 1) / W + 32 * U - 1) / (32 * U) * (32 * U);
  const int64_t w0 = (int64_t)wid * per, w1 = (w0 + per < n ? w0 + per : n);
  // seed the list with the warp's first 32 elements, sorted in registers, so the threshold
  // starts at their k-th best instead of +inf (saves the merges of the first pass)
  int64_t start = w0;
  if (k <= 32 && w0 < w1) {
    const int64_t i = w0 + lane;
    unsigned long long v = i < w1 ? (((unsigned long long)fkey(row[i]) << 32) | (uint32_t)i) : ~0ull;
    for (int size = 2; size <= 32; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, stride);
        const bool up = ((lane & size) == 0);
        const bool lower = (lane & stride) == 0;
        v = (lower == up) ? (v < o ? v : o) : (v > o ? v : o);
      }
    }
    if (lane < k) lst[lane] = v;
    __syncwarp();
    tau = lst[k - 1];
    tau_f = tau == ~0ull ? __uint_as_float(0x7F800000u) : fkey_inv((uint32_t)(tau >> 32));
    start = w0 + 32;
  }
  for (int64_t base = start; base < w1; base += 32 * U) {
    float x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      x[u] = i < w1 ? row[i] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      // a warp scans its slice in increasing index order, so an element equal to the current
      // k-th best distance has a larger id than it and cannot displace it: strict < on the
      // float is exact; keys are packed only for the rare candidates
      const bool q = i < w1 && x[u] < tau_f;
      const unsigned m = __ballot_sync(0xffffffffu, q);
      if (m) {
        const int add = __popc(m);
        if (cnt + add > 32) merge();
        if (q) lst[k + cnt + __popc(m & ((1u << lane) - 1u))] = ((unsigned long long)fkey(x[u]) << 32) | (uint32_t)i;
        __syncwarp();
        cnt += add;
        if (cnt == 32) merge();
      }
    }
  }
  if (cnt) merge();
  __syncthreads();
  // block merge of the W warp lists (k each)
  unsigned long long* all = wl + W * P;
  int Q = 1;
  while (Q < W * k) Q <<= 1;
  for (int j = tid; j < Q; j += blockDim.x) all[j] = j < W * k ? wl[(j / k) * P + (j % k)] : ~0ull;
  __syncthreads();
  bitonic_sort_u64(all, Q);
  for (int j = tid; j < k; j += blockDim.x) {
    const unsigned long long v = all[j];
    const uint32_t key = (uint32_t)(v >> 32);
    if (v == ~0ull) {  // fewer than k entries in a short chunk: padding sorts last in k_merge
      od[j] = __uint_as_float(0x7FFFFFFFu);
      oi[j] = -1;
    } else {
      od[j] = fkey_inv(key);
      oi[j] = (int32_t)(id_base + c0 + (int64_t)(uint32_t)(v & 0xFFFFFFFFu));
    }
  }
}

// k_topk_reg (k <= 32): the same selection with each warp's k best held in REGISTERS, one
// packed key per lane, sorted across lanes 0..k-1.  A candidate (distance <= the warp's k-th
// best distance, then exact packed-key comparison, so the scan order does not matter for ties)
// is inserted with one ballot + one shuffle: no shared memory and no sorting passes.  WPR warps
// share one (row, chunk) task; their lists are merged by insertion at the end.  Rows are read
// as float4 (4 entries per lane, 512 contiguous bytes per warp instruction), U loads in flight.
// Out-of-range entries read as NaN, which never pass the filter (NaN distances sort last).
constexpr int kRegThreads = 128;

__device__ __forceinline__ void reg_insert(unsigned long long& lk, unsigned long long cand, int k,
                                           int lane, unsigned long long& tk, float& tf) {
  const unsigned long long up = __shfl_up_sync(0xffffffffu, lk, 1);
  const unsigned gt = __ballot_sync(0xffffffffu, lk > cand);  // lanes >= k hold ~0 > cand
  const int p = __ffs(gt) - 1;
  if (lane > p) lk = up;
  else if (lane == p) lk = cand;
  if (lane >= k) lk = ~0ull;
  tk = __shfl_sync(0xffffffffu, lk, k - 1);
  tf = tk == ~0ull ? __uint_as_float(0x7F800000u) : fkey_inv((uint32_t)(tk >> 32));
}

template <int WPR>
__global__ void __launch_bounds__(kRegThreads, 4)
    k_topk_reg(const float* __restrict__ dist, int64_t ldd, int64_t n_total, int64_t chunk, int k,
               int64_t id_base, const int32_t* __restrict__ invalid, float* __restrict__ od,
               int32_t* __restrict__ oi, int B, int tasks) {
  constexpr int TPB = kRegThreads / 32 / WPR;  // tasks per block
#ifndef KGQ_TOPK_U
#define KGQ_TOPK_U 8
#endif
  constexpr int U = KGQ_TOPK_U;  // float4 loads in flight per lane (16 x 128 B lines per warp at 8)
  __shared__ unsigned long long part[kRegThreads / 32][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int t = blockIdx.x * TPB + wid / WPR, sub = wid % WPR;
  const bool live = t < tasks;
  const int b = live ? t % B : 0, c = live ? t / B : 0;
  const bool dead = !live || (invalid && invalid[b]);
  const int64_t c0 = (int64_t)c * chunk;
  const int64_t n = dead ? 0 : (n_total - c0 < chunk ? n_total - c0 : chunk);
  const float* row = dist + (int64_t)b * ldd + c0;
  unsigned long long lk = ~0ull, tk = ~0ull;
  float tf = __uint_as_float(0x7F800000u);
  const float kNaN = __uint_as_float(0x7FFFFFFFu);
  const int64_t per = ((n + WPR - 1) / WPR + 127) / 128 * 128;
  const int64_t w0 = (int64_t)sub * per, w1 = (w0 + per < n ? w0 + per : n);
  const bool vec = (((uintptr_t)row) & 15) == 0;
  for (int64_t base = w0; base < w1; base += 128 * U) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 128 + lane * 4;
      if (vec && i + 4 <= w1) {
        x[u] = __ldg(reinterpret_cast<const float4*>(row + i));
      } else {
        x[u].x = i < w1 ? row[i] : kNaN;
        x[u].y = i + 1 < w1 ? row[i + 1] : kNaN;
        x[u].z = i + 2 < w1 ? row[i + 2] : kNaN;
        x[u].w = i + 3 < w1 ? row[i + 3] : kNaN;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float mn = fminf(fminf(x[u].x, x[u].y), fminf(x[u].z, x[u].w));
      if (!__any_sync(0xffffffffu, mn <= tf)) continue;
      const int64_t i0 = base + u * 128 + lane * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float xv = j == 0 ? x[u].x : j == 1 ? x[u].y : j == 2 ? x[u].z : x[u].w;
        const unsigned long long key = ((unsigned long long)fkey(xv) << 32) | (uint32_t)(i0 + j);
        unsigned m = __ballot_sync(0xffffffffu, xv <= tf);
        while (m) {
          const int src = __ffs(m) - 1;
          const unsigned long long cand = __shfl_sync(0xffffffffu, key, src);
          if (cand < tk) reg_insert(lk, cand, k, lane, tk, tf);
          m &= m - 1;
          m &= __ballot_sync(0xffffffffu, xv <= tf);
        }
      }
    }
  }
  if (WPR > 1) {
    part[wid][lane] = lk;
    __syncthreads();
    if (sub == 0) {
      for (int w = 1; w < WPR; ++w) {
        const unsigned long long mine = part[wid + w][lane];
        unsigned m = __ballot_sync(0xffffffffu, lane < k && mine < tk);
        while (m) {
          const int src = __ffs(m) - 1;
          const unsigned long long cand = __shfl_sync(0xffffffffu, mine, src);
          if (cand < tk) reg_insert(lk, cand, k, lane, tk, tf);
          m &= m - 1;
        }
      }
    }
  }
  if (!live || sub != 0 || lane >= k) return;
  const int64_t o = ((int64_t)c * B + b) * k + lane;
  if (lk == ~0ull) {  // fewer than k entries (short chunk, NaN row, invalid query)
    od[o] = kNaN;
    oi[o] = -1;
  } else {
    od[o] = fkey_inv((uint32_t)(lk >> 32));
    oi[o] = (int32_t)(id_base + c0 + (int64_t)(uint32_t)(lk & 0xFFFFFFFFu));
  }
}

// k_topk_cmin (k <= 32): one CTA of four warps per query row, using the score epilogue's
// minima of 32-entity blocks.  Warp w owns a quarter of the blocks.  Pass 1: each lane takes
// the minimum over its blocks; the k-th smallest of a warp's 32 lane minima comes from k
// distinct blocks, each holding an entry <= it, so it bounds the row's k-th best distance from
// above, and tau = the smallest of the four warps' bounds is one too (for i.i.d. block minima it
// selects ~1.1 k blocks).  Pass 2: the warps load only the blocks whose minimum is <= tau (one
// coalesced 128-byte load each, eight in flight) and append every entry <= tau -- a superset of
// the k best, ties included -- to a shared list (ballot compaction, typically 10-30 entries);
// one block-wide bitonic sort of the packed (distance, id) keys gives the exact top-k.  If more
// than kCandCap entries tie below tau (adversarial ties), warp 0 falls back to a register-list
// scan of the same blocks.  Reads ~n/32 + ~k x 32 values per row instead of n.
constexpr int kCminWarps = 4;
constexpr int kCandCap = 256;

__global__ void __launch_bounds__(32 * kCminWarps)
    k_topk_cmin(const float* __restrict__ dist, int64_t ldd, const float* __restrict__ cmin, int64_t ldc,
                int64_t n, int k, int64_t id_base, const int32_t* __restrict__ invalid,
                const int32_t* __restrict__ out_row, float* __restrict__ od, int32_t* __restrict__ oi, int B,
                const PeerPush pp) {
  pdl_grid_sync();
  __shared__ float wtau[kCminWarps];
  __shared__ unsigned long long cand[kCandCap];
  __shared__ int blist[kCminWarps][kCandCap];  // per warp: qualifying block ids
  __shared__ int ncand;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int b = blockIdx.x;
  const int ob = out_row ? out_row[b] : b;  // output / invalid-flag row (mixed batches)
  const float kNaN = __uint_as_float(0x7FFFFFFFu), kInf = __uint_as_float(0x7F800000u);
  od += (int64_t)ob * k;
  oi += (int64_t)ob * k;
  if (invalid && invalid[ob]) {
    if (wid == 0 && lane < k) {
      od[lane] = kNaN;
      oi[lane] = -1;
    }
    if (wid == 0 && pp.on()) peer_push_warp(pp, ob, k, ~0ull, lane);  // N2: fused all-gather
    return;
  }
  if (threadIdx.x == 0) ncand = 0;
  const int64_t nblk = (n + 31) / 32;
  const int64_t per = (nblk + kCminWarps - 1) / kCminWarps;
  const int64_t j0w = (int64_t)wid * per, j1w = j0w + per < nblk ? j0w + per : nblk;
  const float* cm = cmin + (int64_t)b * ldc;
  const float* row = dist + (int64_t)b * ldd;
  // ---- pass 1: warp bound = k-th smallest lane minimum over this warp's blocks ----
  float lmin = kInf;
  for (int64_t g0 = j0w; g0 < j1w; g0 += 32 * 8) {
    float xs[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t j = g0 + u * 32 + lane;
      xs[u] = j < j1w ? cm[j] : kInf;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) lmin = fminf(lmin, xs[u]);
  }
  float v = lmin;  // ascending bitonic sort across the warp
  for (int size = 2; size <= 32; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const float o = __shfl_xor_sync(0xffffffffu, v, stride);
      const bool up = (lane & size) == 0, lower = (lane & stride) == 0;
      v = (lower == up) ? fminf(v, o) : fmaxf(v, o);
    }
  if (lane == k - 1) wtau[wid] = v;  // +inf if fewer than k lanes hold blocks
  __syncthreads();
  float tau = wtau[0];
#pragma unroll
  for (int w = 1; w < kCminWarps; ++w) tau = fminf(tau, wtau[w]);
  // ---- pass 2: every entry <= tau of the blocks whose minimum is <= tau -> shared list ----
  // first compact this warp's qualifying block ids (ballot + prefix count), then load them
  // eight at a time: no load slots are spent on unselected blocks
  const unsigned lt = (1u << lane) - 1u;
  int* bl = blist[wid];
  int nsel = 0;
  for (int64_t g0 = j0w; g0 < j1w; g0 += 32) {
    const float x = g0 + lane < j1w ? cm[g0 + lane] : kNaN;
    const unsigned m = __ballot_sync(0xffffffffu, x <= tau);
    const int p = nsel + __popc(m & lt);
    if (x <= tau && p < kCandCap) bl[p] = (int)(g0 + lane);
    nsel += __popc(m);
  }
  if (nsel > kCandCap) {  // >= kCandCap + 1 candidates: force the register-scan path
    if (lane == 0) atomicAdd(&ncand, kCandCap + 1);
    nsel = 0;
  }
  __syncwarp();
  for (int i0 = 0; i0 < nsel; i0 += 8) {
    int blk[8];
    float vv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // up to eight blocks' loads in flight
      blk[u] = i0 + u < nsel ? bl[i0 + u] : -1;
      const int e = blk[u] * 32 + lane;
      vv[u] = blk[u] >= 0 && e < n ? row[e] : kNaN;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (blk[u] < 0) break;
      const bool pass = vv[u] <= tau;
      const unsigned m = __ballot_sync(0xffffffffu, pass);
      if (!m) continue;
      int base = 0;
      if (lane == 0) base = atomicAdd(&ncand, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      const int slot = base + __popc(m & lt);
      if (pass && slot < kCandCap)
        cand[slot] = ((unsigned long long)fkey(vv[u]) << 32) | (uint32_t)(blk[u] * 32 + lane);
    }
  }
  __syncthreads();
  const int nc = ncand;
  if (nc <= kCandCap) {
    // k smallest of <= 256 distinct (key, id) candidates by warp 0: each lane keeps up to 8 in
    // registers; k rounds of warp arg-min, the owner drops its winner (no block-wide sort)
    if (wid != 0) return;
    unsigned long long v[kCandCap / 32];
#pragma unroll
    for (int m = 0; m < kCandCap / 32; ++m) v[m] = lane + 32 * m < nc ? cand[lane + 32 * m] : ~0ull;
    unsigned long long mine = ~0ull;
#pragma unroll
    for (int m = 0; m < kCandCap / 32; ++m) mine = v[m] < mine ? v[m] : mine;
    unsigned long long key = ~0ull;  // output j = lane
    for (int j = 0; j < k; ++j) {
      unsigned long long w = mine;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, w, o);
        w = t < w ? t : w;
      }
      if (lane == j) key = w;
      if (w == ~0ull) break;  // fewer than k candidates: the rest stay empty
      if (mine == w) {        // keys are unique (ids): exactly one lane owns w
        mine = ~0ull;
#pragma unroll
        for (int m = 0; m < kCandCap / 32; ++m) {
          if (v[m] == w) v[m] = ~0ull;
          mine = v[m] < mine ? v[m] : mine;
        }
      }
    }
    unsigned long long gk = ~0ull;  // (key, global id) of output j = lane
    if (lane < k) {
      if (key == ~0ull) {  // fewer than k entries
        od[lane] = kNaN;
        oi[lane] = -1;
      } else {
        const uint32_t gid = (uint32_t)(id_base + (int64_t)(uint32_t)(key & 0xFFFFFFFFu));
        od[lane] = fkey_inv((uint32_t)(key >> 32));
        oi[lane] = (int32_t)gid;
        gk = (key & 0xFFFFFFFF00000000ull) | gid;
      }
    }
    if (pp.on()) peer_push_warp(pp, ob, k, gk, lane);  // N2: fused all-gather
    return;
  }
  // ---- overflow (more than kCandCap entries <= tau): register-list scan by warp 0 ----
  if (wid != 0) return;
  unsigned long long lk = ~0ull, tk = ~0ull;
  float tf = kInf;
  for (int64_t g0 = 0; g0 < nblk; g0 += 32) {
    const float x = g0 + lane < nblk ? cm[g0 + lane] : kNaN;
    unsigned sel = __ballot_sync(0xffffffffu, x <= tau);
    while (sel) {
      const int o = __ffs(sel) - 1;
      sel &= sel - 1;
      if (__shfl_sync(0xffffffffu, x, o) > fminf(tf, tau)) continue;
      const int64_t i = (g0 + o) * 32 + lane;
      const float vi = i < n ? row[i] : kNaN;
      const unsigned long long key = ((unsigned long long)fkey(vi) << 32) | (uint32_t)i;
      unsigned m = __ballot_sync(0xffffffffu, vi <= fminf(tf, tau));
      while (m) {
        const int src = __ffs(m) - 1;
        const unsigned long long c = __shfl_sync(0xffffffffu, key, src);
        if (c < tk) reg_insert(lk, c, k, lane, tk, tf);
        m &= m - 1;
        m &= __ballot_sync(0xffffffffu, vi <= fminf(tf, tau));
      }
    }
  }
  unsigned long long gk = ~0ull;
  if (lane < k) {
    if (lk == ~0ull) {
      od[lane] = kNaN;
      oi[lane] = -1;
    } else {
      const uint32_t gid = (uint32_t)(id_base + (int64_t)(uint32_t)(lk & 0xFFFFFFFFu));
      od[lane] = fkey_inv((uint32_t)(lk >> 32));
      oi[lane] = (int32_t)gid;
      gk = (lk & 0xFFFFFFFF00000000ull) | gid;
    }
  }
  if (pp.on()) peer_push_warp(pp, ob, k, gk, lane);  // N2: fused all-gather
}

int launch_topk_cmin(const float* dist, int64_t ldd, const float* cmin, int64_t ldc, int B, int64_t n,
                     int k, int64_t id_base, const int32_t* invalid, float* out_d, int32_t* out_i,
                     cudaStream_t st, const PeerPush& pp) {
  launch_pdl(k_topk_cmin, dim3(B), dim3(32 * kCminWarps), 0, st, dist, ldd, cmin, ldc, n, k, id_base, invalid,
             (const int32_t*)nullptr, out_d, out_i, B, pp);
  return 1;
}

// ---- merge of the fused scorer's lists (score_tc.cu EpiBetaScore<NB, true>) -----------------
// Output row b has nl (<= 128) sorted lists of k (order key << 32 | shard column) keys, ~0-padded
// -- one per (N stripe, column half) of the tensor-core scorer -- at cand[b * ldcand + l * k].  One
// warp per row: lane l holds the heads of lists l + 32 j, k rounds of warp arg-min, the winner
// advances its list.  The
// columns of different lists are disjoint, so keys are unique and the result is exactly the first
// k of the row in (distance, id) order.  Rows [0, rows1) have nl1 lists, the rest nl2 (mixed
// batches: non-union then union scorer launch).
// lane j < k writes output j of the row from its merged key (fewer than k entities: NaN / -1)
__device__ __forceinline__ void topk_lists_out(unsigned long long key, int lane, int k, int ob, int64_t id_base,
                                               float* od, int32_t* oi, const PeerPush& pp) {
  unsigned long long gk = ~0ull;
  if (lane < k) {
    if (key == ~0ull) {
      od[lane] = __uint_as_float(0x7FFFFFFFu);
      oi[lane] = -1;
    } else {
      const uint32_t gid = (uint32_t)(id_base + (int64_t)(uint32_t)(key & 0xFFFFFFFFu));
      od[lane] = fkey_inv((uint32_t)(key >> 32));
      oi[lane] = (int32_t)gid;
      gk = (key & 0xFFFFFFFF00000000ull) | gid;
    }
  }
  if (pp.on()) peer_push_warp(pp, ob, k, gk, lane);  // N2: fused all-gather
}

__global__ void __launch_bounds__(128)  // (a register cap for 12 / 16 blocks per SM spills: slower)
    k_topk_lists(const unsigned long long* __restrict__ cand, int64_t ldcand, int k, int rows1, int nl1, int nl2,
                 int64_t id_base, const int32_t* __restrict__ invalid, const int32_t* __restrict__ out_row,
                 float* __restrict__ od, int32_t* __restrict__ oi, int B, const PeerPush pp) {
  pdl_grid_sync();
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const int ob = out_row ? out_row[b] : b;
  od += (int64_t)ob * k;
  oi += (int64_t)ob * k;
  if (invalid && invalid[ob]) {
    if (lane < k) {
      od[lane] = __uint_as_float(0x7FFFFFFFu);
      oi[lane] = -1;
    }
    if (pp.on()) peer_push_warp(pp, ob, k, ~0ull, lane);
    return;
  }
  const int nl = b < rows1 ? nl1 : nl2;
  const unsigned long long* row = cand + (int64_t)b * ldcand;
  if (nl <= 32 && k <= 16) {
    // <= 32 lists: lane l loads its whole list up front (independent loads, no load per round)
    // and shifts it down as its head is consumed
    unsigned long long lst[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) lst[j] = (lane < nl && j < k) ? row[(int64_t)lane * k + j] : ~0ull;
    unsigned long long key = ~0ull;  // output j = lane
    for (int j = 0; j < k; ++j) {
      unsigned long long w = lst[0];
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, w, o);
        w = t < w ? t : w;
      }
      if (lane == j) key = w;
      if (w == ~0ull) break;  // fewer than k entities
      if (lst[0] == w) {      // unique keys: exactly one lane's head
#pragma unroll
        for (int q = 0; q < 15; ++q) lst[q] = lst[q + 1];
        lst[15] = ~0ull;
      }
    }
    topk_lists_out(key, lane, k, ob, id_base, od, oi, pp);
    return;
  }
  // lane l holds the heads of lists l, l + 32, l + 64, l + 96 (<= 128 lists)
  int pos[4];
  unsigned long long head[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    pos[j] = 0;
    head[j] = lane + 32 * j < nl ? row[(int64_t)(lane + 32 * j) * k] : ~0ull;
  }
  unsigned long long key = ~0ull;  // output j = lane
  for (int j = 0; j < k; ++j) {
    unsigned long long mine = head[0];
#pragma unroll
    for (int q = 1; q < 4; ++q) mine = head[q] < mine ? head[q] : mine;
    unsigned long long w = mine;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, w, o);
      w = t < w ? t : w;
    }
    if (lane == j) key = w;
    if (w == ~0ull) break;  // fewer than k entities
    if (mine == w) {        // unique keys: exactly one head of one lane
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (head[q] == w) {
          ++pos[q];
          head[q] = pos[q] < k ? row[(int64_t)(lane + 32 * q) * k + pos[q]] : ~0ull;
        }
    }
  }
  topk_lists_out(key, lane, k, ob, id_base, od, oi, pp);
}

// <= 8 lists per row, k <= 16, no peer push (the mixed step's fused rows: 3 stripes x 2 column
// halves): eight lanes per row, four rows per warp -- three shuffle levels per round instead of
// five and a quarter of the warps (the one-row-per-warp merge is latency-bound: 21 us for the C2
// step's 12,288 rows).  Same keys, same order as k_topk_lists: bit-identical outputs.
__global__ void __launch_bounds__(128)
    k_topk_lists8(const unsigned long long* __restrict__ cand, int64_t ldcand, int k, int rows1, int nl1, int nl2,
                  int64_t id_base, const int32_t* __restrict__ invalid, const int32_t* __restrict__ out_row,
                  float* __restrict__ od, int32_t* __restrict__ oi, int B) {
  pdl_grid_sync();
  const int lane = threadIdx.x & 31, gl = lane & 7;
  const int b = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4 + (lane >> 3);
  const bool live = b < B;
  const int ob = live ? (out_row ? out_row[b] : b) : 0;
  const bool bad = live && invalid && invalid[ob];
  const int nl = b < rows1 ? nl1 : nl2;
  const unsigned long long* row = cand + (int64_t)(live ? b : 0) * ldcand;
  unsigned long long lst[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) lst[j] = (live && !bad && gl < nl && j < k) ? row[(int64_t)gl * k + j] : ~0ull;
  unsigned long long o0 = ~0ull, o1 = ~0ull;  // outputs gl and gl + 8 of this lane's row
  for (int j = 0; j < k; ++j) {               // k is warp-uniform: the shuffles stay converged
    unsigned long long w = lst[0];
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, w, o);
      w = t < w ? t : w;
    }
    if (j == gl) o0 = w;
    if (j == gl + 8) o1 = w;
    if (w != ~0ull && lst[0] == w) {  // unique keys: exactly one lane's head
#pragma unroll
      for (int q = 0; q < 15; ++q) lst[q] = lst[q + 1];
      lst[15] = ~0ull;
    }
  }
  if (!live) return;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int jj = gl + 8 * h;
    if (jj >= k) continue;
    const unsigned long long key = h ? o1 : o0;
    float* d = od + (int64_t)ob * k + jj;
    int32_t* i = oi + (int64_t)ob * k + jj;
    if (bad || key == ~0ull) {
      *d = __uint_as_float(0x7FFFFFFFu);
      *i = -1;
    } else {
      *d = fkey_inv((uint32_t)(key >> 32));
      *i = (int32_t)(uint32_t)(id_base + (int64_t)(uint32_t)(key & 0xFFFFFFFFu));
    }
  }
}

int launch_topk_lists(const unsigned long long* cand, int64_t ldcand, int k, int B, int rows1, int nl1, int nl2,
                      int64_t id_base, const int32_t* invalid, const int32_t* out_row, float* out_d, int32_t* out_i,
                      cudaStream_t st, const PeerPush& pp) {
  if (B <= 0) return 0;
  if (nl1 <= 8 && nl2 <= 8 && k <= 16 && !pp.on()) {
    launch_pdl(k_topk_lists8, dim3((B + 15) / 16), dim3(128), 0, st, cand, ldcand, k, rows1, nl1, nl2, id_base,
               invalid, out_row, out_d, out_i, B);
    return 1;
  }
  launch_pdl(k_topk_lists, dim3((B + 3) / 4), dim3(128), 0, st, cand, ldcand, k, rows1, nl1, nl2, id_base, invalid,
             out_row, out_d, out_i, B, pp);
  return 1;
}

int launch_topk_cmin_map(const float* dist, int64_t ldd, const float* cmin, int64_t ldc, int B, int64_t n,
                         int k, int64_t id_base, const int32_t* invalid, const int32_t* out_row, float* out_d,
                         int32_t* out_i, cudaStream_t st, const PeerPush& pp) {
  if (B <= 0) return 0;
  launch_pdl(k_topk_cmin, dim3(B), dim3(32 * kCminWarps), 0, st, dist, ldd, cmin, ldc, n, k, id_base, invalid,
             out_row, out_d, out_i, B, pp);
  return 1;
}

int64_t topk_chunk(int64_t n, int k) {
  // long rows are split so that many CTAs share a query; chunks * k must fit k_merge (4096)
  if (n <= kTopkStage * 2) return n;
  int64_t c = kTopkStage;
  while ((n + c - 1) / c * k > 4096) c *= 2;
  return c;
}

void launch_topk_kernel(dim3 grid, const float* dist, int64_t ldd, int64_t n, int64_t chunk, int k,
                        int64_t id_base, const int32_t* invalid, float* od, int32_t* oi, int B,
                        cudaStream_t st) {
  if (k <= 32) {
    const int tasks = (int)(grid.x * grid.y);
    // enough warps in flight to cover memory latency: ~16 per SM
    const int wpr = tasks >= 2048 ? 1 : tasks >= 768 ? 2 : 4;
    const int tpb = kRegThreads / 32 / wpr;
    const int blocks = (tasks + tpb - 1) / tpb;
    if (wpr == 1)
      k_topk_reg<1><<<blocks, kRegThreads, 0, st>>>(dist, ldd, n, chunk, k, id_base, invalid, od, oi, B, tasks);
    else if (wpr == 2)
      k_topk_reg<2><<<blocks, kRegThreads, 0, st>>>(dist, ldd, n, chunk, k, id_base, invalid, od, oi, B, tasks);
    else
      k_topk_reg<4><<<blocks, kRegThreads, 0, st>>>(dist, ldd, n, chunk, k, id_base, invalid, od, oi, B, tasks);
    return;
  }
  int P = 64;
  while (P < k + 32) P <<= 1;
  int Q = 1;
  while (Q < (kTopkThreads / 32) * k) Q <<= 1;
  const int smem = (int)(((kTopkThreads / 32) * P + Q) * sizeof(unsigned long long));
  static SmemAttr attr;
  smem_attr_once(k_topk, 64 * 1024, attr);
  k_topk<<<grid, kTopkThreads, smem, st>>>(dist, ldd, n, chunk, k, id_base, invalid, od, oi, B, P);
}

int launch_topk(const float* dist, int64_t ldd, int B, int64_t n, int k, int64_t id_base,
                const int32_t* invalid, float* out_d, int32_t* out_i, float* tmp_d, int32_t* tmp_i,
                cudaStream_t st) {
  const int64_t chunk = topk_chunk(n, k);
  const int nch = (int)((n + chunk - 1) / chunk);
  if (nch == 1) {
    launch_topk_kernel(dim3(B, 1), dist, ldd, n, n, k, id_base, invalid, out_d, out_i, B, st);
    return 1;
  }
  launch_topk_kernel(dim3(B, nch), dist, ldd, n, chunk, k, id_base, invalid, tmp_d, tmp_i, B, st);
  return 1 + launch_merge(nch, B, k, tmp_d, tmp_i, out_d, out_i, st);
}

// Merge parts x [B, k] candidate lists into [B, k] (a9).  ids are global; NaN rows sort last.
__global__ void k_merge(int parts, int B, int k, const float* __restrict__ in_d,
                        const int32_t* __restrict__ in_i, float* __restrict__ od,
                        int32_t* __restrict__ oi) {
  extern __shared__ unsigned long long v[];
  const int b = blockIdx.x;
  const int m = parts * k;
  int P = 1;
  while (P < m) P <<= 1;
  for (int j = threadIdx.x; j < P; j += blockDim.x) {
    if (j < m) {
      const int p = j / k, c = j % k;
      const int64_t o = ((int64_t)p * B + b) * k + c;
      const uint32_t key = fkey(in_d[o]);
      const uint32_t id = key == 0xFFFFFFFFu ? 0xFFFFFFFFu : (uint32_t)in_i[o];
      v[j] = ((unsigned long long)key << 32) | id;
    } else {
      v[j] = ~0ull;
    }
  }
  __syncthreads();
  bitonic_sort_u64(v, P);
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const unsigned long long x = v[j];
    const uint32_t key = (uint32_t)(x >> 32);
    od[(int64_t)b * k + j] = fkey_inv(key);
    oi[(int64_t)b * k + j] = key == 0xFFFFFFFFu ? -1 : (int32_t)(uint32_t)(x & 0xFFFFFFFFu);
  }
}

int launch_merge(int parts, int B, int k, const float* in_d, const int32_t* in_i, float* out_d,
                 int32_t* out_i, cudaStream_t st) {
  int P = 1;
  while (P < parts * k) P <<= 1;
  k_merge<<<B, 256, (size_t)P * sizeof(unsigned long long), st>>>(parts, B, k, in_d, in_i, out_d,
                                                                   out_i);
  return 1;
}

}  // namespace kgq
