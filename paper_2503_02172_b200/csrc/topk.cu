// Top-k selection and cross-shard merge (a9).
//
// Order: distance ascending, ties by ascending global entity id (Q13).
// Distances map to order-preserving uint32 keys (NaN -> max, -0 -> +0), so (key, id) packed
// in a uint64 sorts exactly in that order.
//
// k_topk: one CTA per query row.  Radix select (4 passes of 8-bit digits over the row) finds
// the k-th smallest key T and how many of the T-ties to keep; a compaction pass collects the
// keys < T (any order) and the first ties by ascending index (block-wide ordered scan); a
// bitonic sort of the <= 256 survivors gives the final order.
#include <stdint.h>

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
constexpr int64_t kTopkChunkMin = 16384;  // entries per CTA when a row is split

__global__ void __launch_bounds__(kTopkThreads)
    k_topk(const float* __restrict__ dist, int64_t ldd, int64_t n_total, int64_t chunk, int k,
           int64_t id_base, const int32_t* __restrict__ invalid, float* __restrict__ od,
           int32_t* __restrict__ oi, int B) {
  // CTA (b, c) selects the k best of row b restricted to [c*chunk, min(n, (c+1)*chunk)) and
  // writes them at [(c*B + b)*k, ...): with one chunk that is the final [B, k] answer, with
  // several it is the candidate list k_merge reduces (multi-CTA top-k for long rows).
  const int b = blockIdx.x;
  const int64_t c0 = (int64_t)blockIdx.y * chunk;
  const int64_t n = (n_total - c0 < chunk ? n_total - c0 : chunk);
  const float* row = dist + (int64_t)b * ldd + c0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  od += ((int64_t)blockIdx.y * B + b) * k;
  oi += ((int64_t)blockIdx.y * B + b) * k;
  const int kout = k;
  k = (int)(n < k ? n : k);  // a short last chunk contributes all of its entries
  if (invalid && invalid[b]) {
    for (int j = tid; j < kout; j += blockDim.x) {
      od[j] = __uint_as_float(0x7FFFFFFFu);
      oi[j] = -1;
    }
    return;
  }
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_prefix, s_kk;
  __shared__ unsigned long long sel[kMaxK];
  __shared__ int s_less;
  __shared__ int s_wsum[kTopkThreads / 32];

  uint32_t prefix = 0, mask = 0, kk = (uint32_t)k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    hist[tid] = 0;
    __syncthreads();
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const uint32_t key = fkey(row[i]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (wid == 0) {
      // lane owns bins [8*lane, 8*lane+8)
      uint32_t c[8], s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[lane * 8 + j];
        s += c[j];
      }
      uint32_t incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      uint32_t before = incl - s;
      // the lane whose range contains the kk-th element
      const bool mine = before < kk && kk <= incl;
      if (mine) {
        uint32_t cum = before;
        for (int j = 0; j < 8; ++j) {
          if (cum + c[j] >= kk) {
            s_prefix = prefix | ((uint32_t)(lane * 8 + j) << shift);
            s_kk = kk - cum;
            break;
          }
          cum += c[j];
        }
      }
    }
    __syncthreads();
    prefix = s_prefix;
    kk = s_kk;
    mask |= 255u << shift;
    __syncthreads();
  }
  const uint32_t T = prefix;  // key of the k-th smallest; keep kk of its ties
  const int n_less = k - (int)kk;
  if (tid == 0) s_less = 0;
  __syncthreads();
  uint32_t eq_before = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + tid;
    const uint32_t key = i < n ? fkey(row[i]) : 0xFFFFFFFFu;
    if (i < n && key < T) {
      const int pos = atomicAdd(&s_less, 1);
      sel[pos] = ((unsigned long long)key << 32) | (uint32_t)i;
    }
    const bool eq = i < n && key == T;
    const uint32_t bal = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) s_wsum[wid] = __popc(bal);
    __syncthreads();
    uint32_t off = 0, tot = 0;
    for (int w = 0; w < kTopkThreads / 32; ++w) {
      if (w < wid) off += s_wsum[w];
      tot += s_wsum[w];
    }
    const uint32_t rank = eq_before + off + __popc(bal & ((1u << lane) - 1u));
    if (eq && rank < kk) sel[n_less + rank] = ((unsigned long long)key << 32) | (uint32_t)i;
    eq_before += tot;
    __syncthreads();
  }
  int P = 1;
  while (P < k) P <<= 1;
  for (int j = k + tid; j < P; j += blockDim.x) sel[j] = ~0ull;
  __syncthreads();
  bitonic_sort_u64(sel, P);
  for (int j = tid; j < kout; j += blockDim.x) {
    if (j < k) {
      const unsigned long long v = sel[j];
      od[j] = fkey_inv((uint32_t)(v >> 32));
      oi[j] = (int32_t)(id_base + c0 + (int64_t)(uint32_t)(v & 0xFFFFFFFFu));
    } else {  // padding of a short chunk: sorts last in k_merge
      od[j] = __uint_as_float(0x7FFFFFFFu);
      oi[j] = -1;
    }
  }
}

int64_t topk_chunk(int64_t n, int k) {
  // long rows are split so that many CTAs share a query; chunks * k must fit k_merge (4096)
  if (n <= kTopkChunkMin * 2) return n;
  int64_t c = kTopkChunkMin;
  while ((n + c - 1) / c * k > 4096) c *= 2;
  return c;
}

int launch_topk(const float* dist, int64_t ldd, int B, int64_t n, int k, int64_t id_base,
                const int32_t* invalid, float* out_d, int32_t* out_i, float* tmp_d, int32_t* tmp_i,
                cudaStream_t st) {
  const int64_t chunk = topk_chunk(n, k);
  const int nch = (int)((n + chunk - 1) / chunk);
  if (nch == 1) {
    k_topk<<<dim3(B, 1), kTopkThreads, 0, st>>>(dist, ldd, n, n, k, id_base, invalid, out_d, out_i, B);
    return 1;
  }
  k_topk<<<dim3(B, nch), kTopkThreads, 0, st>>>(dist, ldd, n, chunk, k, id_base, invalid, tmp_d, tmp_i, B);
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
