// N2: the cross-shard all-gather of the per-shard top-k fused into the top-k
// kernel, over peer memory (NVLink P2P / NVSwitch on a multi-GPU node; plain device memory for
// the virtual shards of one GPU).  Replaces a9's NCCL all-gather + k_merge round trip.
//
// Every rank owns one "peer buffer" of identical layout (symmetric allocation; the pointers of
// all ranks' buffers are registered with kgq_set_peers):
//   hdr  [64]                          uint32   hdr[0] = session broken (a rank timed out)
//   flag [2][world][max_rows]          uint32   epoch of the last push of (parity, source, row)
//   key  [2][world][max_rows][max_k]   uint64   (order key of dist << 32) | global id, ascending
// The context's device epoch starts at 1 (kgq_set_peers) and kgq_merge_peers advances it once
// all its rows are merged (the last CTA to finish); a submit's top-k writes row r's k keys into
// slot (epoch & 1, rank, r) of EVERY rank's buffer (its own included) and then publishes
// flag = epoch there with a system-scope release.  kgq_merge_peers waits (acquire) for the
// world flags of each row and merges the world sorted lists.  Parity double-buffering makes
// back-to-back submits safe: rank p can only push epoch e + 2 after its merge of e + 1, which
// waited for this rank's push of e + 1, which this rank issued after its merge of e finished
// reading the parity-(e & 1) slots.  The host side keeps pushes and merges paired: a submit on a
// peered context is rejected while its previous push has not been merged, and a merge without
// a push is rejected (kgq_api.cu push_outstanding), so a push can never overwrite a slot that
// a peer's merge of the same epoch is reading.  A merge that times out on a missing rank
// poisons the session: it sets hdr[0] in EVERY rank's buffer, and from then on every merge on
// every rank returns NaN / -1 rows and reports KGQ_ESTATE until all ranks call kgq_set_peers
// again -- the epochs of the ranks may have diverged, and pairing lists of different submits
// silently is what the poison prevents.
#pragma once
#include <stdint.h>

namespace kgq {

constexpr int kMaxPeers = 8;

struct PeerPush {
  unsigned long long* key[kMaxPeers] = {};  // rank p's key array
  uint32_t* flag[kMaxPeers] = {};           // rank p's flag array
  uint32_t* hdr[kMaxPeers] = {};            // rank p's header (hdr[0]: session broken)
  const uint32_t* epoch = nullptr;          // this context's device epoch (bumped per submit)
  int world = 0, rank = 0, max_rows = 0, max_k = 0;
  int row0 = 0;                             // output row offset of this launch's rows
  __host__ __device__ bool on() const { return world > 0; }
  __device__ size_t slot(uint32_t ep, int src, int row) const {
    return ((size_t)(ep & 1u) * world + src) * max_rows + row;
  }
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Called by all 32 lanes of one warp after it wrote output row `row` (launch-local): lane j < k
// holds the row's j-th key.  Writes the keys to every rank's buffer, then lane p publishes the
// row's flag on rank p.
__device__ __forceinline__ void peer_push_warp(const PeerPush& pp, int row, int k, unsigned long long key, int lane) {
  const uint32_t ep = *pp.epoch;
  const size_t s = pp.slot(ep, pp.rank, pp.row0 + row);
  if (lane < k)
    for (int p = 0; p < pp.world; ++p) pp.key[p][s * pp.max_k + lane] = key;
  // the warp barrier orders every lane's key stores before lane p's flag store, and a release
  // at system scope is cumulative: a peer that acquires the flag sees all k keys
  __syncwarp();
  if (lane < pp.world) st_release_sys(pp.flag[lane] + s, ep);
}

}  // namespace kgq
