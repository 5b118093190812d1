// N2: fused cross-shard all-gather of the top-k over peer memory (peer.cuh has
// the buffer layout and the ordering argument).  The common path pushes from inside the
// pruned top-k kernel (topk.cu k_topk_cmin); k_peer_push covers the other top-k paths by
// pushing finished output rows; k_peer_merge is the receiving side.
#include <stdint.h>

#include "common.cuh"
#include "kgq_internal.cuh"

namespace kgq {

namespace {

__device__ __forceinline__ uint32_t order_key(float f) {  // = topk.cu fkey: NaN -> max, -0 -> +0
  if (f != f) return 0xFFFFFFFFu;
  if (f == 0.0f) f = 0.0f;
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float order_key_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
  for (int o = 16; o; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}


// One warp per output row: keys of the row's k outputs (ids -1 -> the empty key ~0).
__global__ void k_peer_push(const PeerPush pp, int B, int k, const float* __restrict__ od,
                            const int32_t* __restrict__ oi) {
  pdl_grid_sync();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= B) return;
  const uint32_t ep = *pp.epoch;
  const size_t s = pp.slot(ep, pp.rank, pp.row0 + row);
  for (int j = lane; j < k; j += 32) {
    const int32_t id = oi[(int64_t)row * k + j];
    const unsigned long long key =
        id < 0 ? ~0ull : ((unsigned long long)order_key(od[(int64_t)row * k + j]) << 32) | (uint32_t)id;
    for (int p = 0; p < pp.world; ++p) pp.key[p][s * pp.max_k + j] = key;
  }
  __syncwarp();  // see peer_push_warp
  if (lane < pp.world) st_release_sys(pp.flag[lane] + s, ep);
}

// One warp per row: wait until every rank published this row for the current epoch (system-
// scope acquire on this rank's own flags), then a world-way merge of the sorted key lists.  A
// rank that does not deliver within timeout_ns is reported through err (kind 3: row, rank), the
// row is output as NaN / -1 and the session is poisoned on every rank (peer.cuh; later merges
// report kind 4), so a missing peer can neither hang the GPU nor pair lists of different submits.  The CTA that finishes
// last advances the epoch for the next submit (done: a zeroed counter, reset by that CTA).
constexpr int kMergeWarps = 4;
__global__ void __launch_bounds__(32 * kMergeWarps)
    k_peer_merge(const PeerPush pp, int B, int k, float* __restrict__ od, int32_t* __restrict__ oi,
                 int32_t* err, long long timeout_ns, uint32_t* epoch, uint32_t* done) {
  pdl_grid_sync();
  extern __shared__ unsigned long long sk[];  // [kMergeWarps][world * k]
  __shared__ uint32_t s_ep;
  if (threadIdx.x == 0) s_ep = *epoch;
  __syncthreads();
  const uint32_t ep = s_ep;
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(done, 1u) == gridDim.x - 1) {  // every CTA has read ep
    *done = 0;
    *epoch = ep + 1u;
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * kMergeWarps + wid;
  if (row >= B) return;
  const int W = pp.world;
  unsigned long long* s = sk + (size_t)wid * W * k;
  bool ok = true;
  if (ld_acquire_sys(pp.hdr[pp.rank]) != 0u) {  // poisoned session: no list can be trusted
    ok = false;
    if (lane == 0 && atomicCAS(err, 0, 4) == 0) {
      err[1] = row;
      err[2] = 0;
      err[3] = 0;
    }
  } else if (lane < W) {
    const uint32_t* f = pp.flag[pp.rank] + pp.slot(ep, lane, row);
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned ns = 32;
    while (ld_acquire_sys(f) != ep) {
      __nanosleep(ns);
      ns = ns < 1024 ? 2 * ns : ns;
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if ((long long)(t - t0) > timeout_ns) {
        ok = false;
        if (atomicCAS(err, 0, 3) == 0) {
          err[1] = row;
          err[2] = lane;
          err[3] = 0;
        }
        for (int p = 0; p < W; ++p) st_release_sys(pp.hdr[p], 1u);  // poison every rank's session
        break;
      }
    }
  }
  unsigned okm = __ballot_sync(0xffffffffu, ok);
  if (okm != 0xffffffffu) okm = 0u;  // a missing rank or a poisoned session: the row is NaN / -1
  const unsigned long long* keys = pp.key[pp.rank];
  for (int i = lane; i < W * k; i += 32) {
    const int src = i / k, j = i - src * k;
    s[i] = (okm >> src) & 1u ? __ldcg(keys + pp.slot(ep, src, row) * pp.max_k + j) : ~0ull;
  }
  __syncwarp();
  int pos = 0;  // lane r < W: head of rank r's list
  for (int j = 0; j < k; ++j) {
    const unsigned long long h = lane < W && pos < k ? s[lane * k + pos] : ~0ull;
    const unsigned long long m = warp_min_u64(h);
    const unsigned win = __ballot_sync(0xffffffffu, lane < W && h == m);
    if (m != ~0ull && lane == __ffs(win) - 1) ++pos;  // distinct ids: one list holds m
    if (lane == 0) {  // as k_merge (a9): NaN keys sort last and carry id -1
      const int64_t o = (int64_t)row * k + j;
      const uint32_t key = (uint32_t)(m >> 32);
      od[o] = order_key_inv(key);
      oi[o] = key == 0xFFFFFFFFu ? -1 : (int32_t)(uint32_t)(m & 0xFFFFFFFFu);
    }
  }
}

}  // namespace

int launch_peer_push(const PeerPush& pp, int B, int k, const float* out_d, const int32_t* out_i, cudaStream_t st) {
  if (B <= 0) return 0;
  launch_pdl(k_peer_push, dim3((B + 3) / 4), dim3(128), 0, st, pp, B, k, out_d, out_i);
  return 1;
}

int launch_peer_merge(const PeerPush& pp, int B, int k, float* out_d, int32_t* out_i, int32_t* err,
                      long long timeout_ns, cudaStream_t st) {
  if (B <= 0) return 0;
  const size_t smem = (size_t)kMergeWarps * pp.world * k * sizeof(unsigned long long);
  static SmemAttr attr;
  smem_attr_once(k_peer_merge, 200 * 1024, attr);
  launch_pdl(k_peer_merge, dim3((B + kMergeWarps - 1) / kMergeWarps), dim3(32 * kMergeWarps), smem, st, pp, B, k,
             out_d, out_i, err, timeout_ns, const_cast<uint32_t*>(pp.epoch), const_cast<uint32_t*>(pp.epoch) + 1);
  return 1;
}

}  // namespace kgq
