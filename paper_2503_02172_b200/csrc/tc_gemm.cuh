// tcgen05 GEMM core on split fp32 operands, shared by the dense layers (linear_tc.cu) and the
// tensor-core BetaE scorer (score_tc.cu).  Two operand formats (common.cuh KGQ_OPERAND_FP16X2):
// fp16x2 -- the default build, three fp16 MMAs per fp32 multiply-add into one 2^11-scaled fp32
// accumulator (see common.cuh) -- and bf16x3, the full-range build (libkgq_bf16x3.so) described
// here; the pipeline below is the same for both, only the plane count and MMA list differ.
//
// acc[m, n] = sum_k A[m, k] W[n, k] in bf16x3: every fp32 operand is held as three bf16 planes
// x = x0 + x1 + x2 (exact; written by every upstream kernel, common.cuh), and
//   x w ~= x0 w0 + x0 w1 + x1 w0 + x0 w2 + x1 w1 + x2 w0      (dropped terms <= 2^-23 |x w|)
// on tcgen05.mma.kind::f16 (bf16 inputs, fp32 accumulation; 6 bf16 MMAs = the tensor time of 3
// tf32 ones, 6 operand bytes per element instead of 3xTF32's 8), persistent, CTA-pair based:
//   * a cluster of two CTAs (one TPC) computes 256 x BN output tiles with
//     tcgen05.mma.cta_group::2 (M 256, N BN, K 8), each CTA staging its own 128 rows of A and
//     half (BN/2 rows) of the W tile by TMA (64-byte swizzle, OOB zero fill), so per CTA the
//     operand stream is (128 + BN/2) x 192 B per 32-deep K-block;
//   * the grid is at most one cluster per TPC (74 on B200) and loops over tiles (M fastest,
//     so concurrently running clusters read the same W tiles out of L2);
//   * warp 0 lane 0 = TMA producer, warp 1 lane 0 (leader CTA) = MMA issuer, warps 2-9 =
//     epilogue.  The MMA accumulates DRAIN K-blocks into one of two TMEM partials (ping-pong)
//     and the epilogue warps add the partials in fp32 round-to-nearest registers: the TMEM
//     accumulate path truncates (3xTF32 era: 1.8e-5 of sum|x w| over one K = 1600 chain vs 8e-7
//     with 2-K-block partials, profiles/r01/tc_gemm_accuracy.txt; bf16x3 with DRAIN = 8: 2.7e-7);
//   * the epilogue of tile t (bias / activation / split / score terms, Epi::chunk) overlaps
//     the first partials of tile t+1, and writes through a swizzled shared-memory staging tile
//     and TMA bulk tensor stores (cp.async.bulk.tensor shared -> global; the tensor map clips
//     the ragged M / N edges; split outputs are written as the three bf16 planes);
//   * launched with programmatic dependent launch: barrier init, TMEM allocation and tensor-map
//     prefetch overlap the upstream kernel's tail (griddepcontrol.wait before the first load).
// Measured (profiles/r01/tc_trace_*.txt): the non-persistent predecessor spent 6-14 us per tile
// in a per-element STG epilogue and ~3 us in per-CTA setup; this layout hides both.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "common.cuh"
#include "kgq_internal.cuh"

namespace kgq {
namespace tc {
// warp 0: TMA producer, warp 1: MMA issuer, warps 2-9: epilogue (168 registers per thread at
// 320 threads; the fp32 row accumulators take BN/2 of them).
constexpr int BM = 128, BK = 32, EPI_WARPS = 8, EPI_WARP0 = 2, THREADS = 64 + 32 * EPI_WARPS;
constexpr int kClustersMax = 74;  // 148 SMs / 2
// Clusters a launch may use (plan + grid): 74 by default; KGQ_GEMM_CLUSTERS caps it (concurrent
// streams: two GEMMs side by side instead of one filling the GPU and the next queueing).
inline int gemm_clusters() {
  static const int v = [] {
    const char* e = getenv("KGQ_GEMM_CLUSTERS");
    const int c = e ? atoi(e) : 0;
    return c >= 1 && c <= kClustersMax ? c : kClustersMax;
  }();
  return v;
}

// Tile raster group (tile_mn): M blocks per group; KGQ_GEMM_GROUP_M overrides (0 = M fastest).
inline int gemm_group_m() {
  static const int v = [] {
    const char* e = getenv("KGQ_GEMM_GROUP_M");
    return e ? atoi(e) : 8;
  }();
  return v;
}
// the dense layers' raster group: 6 (same-box A/B of the final step: 6 -> 7.125M, 4 -> 7.11M, 8 ->
// 7.09M q/s; the scorer keeps 8).  KGQ_GEMM_GROUP_M_DENSE overrides, KGQ_GEMM_GROUP_M sets both.
inline int gemm_group_m_dense() {
  static const int v = [] {
    const char* e = getenv("KGQ_GEMM_GROUP_M_DENSE");
    if (e) return atoi(e);
    e = getenv("KGQ_GEMM_GROUP_M");
    return e ? atoi(e) : 6;
  }();
  return v;
}

// ---- PTX wrappers -----------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// Wait for a phase that is typically far away (epilogue warps waiting for a whole partial,
// the producer waiting for a free stage): poll with a nanosleep back-off so that idle warps do
// not take issue slots from the single MMA-issuing thread on the same SM sub-partition.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) break;
#ifndef KGQ_TC_NO_BACKOFF
    __nanosleep(64);
#endif
  }
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// K-major bf16 operand tile, 64-byte swizzle: rows of 32 bf16 = 64 B, 8-row atoms 512 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;               // SBO: 8 rows x 64 B
  d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;                        // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
      "[%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-SM TMA load: data lands in this CTA's smem, completion counted on the leader's barrier.
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
// TMA store with an L2 evict-first policy: streaming outputs (the scorer's distance block,
// 60 MB per C2 batch, of which the top-k reads ~3%) must not push the weights and the entity
// table out of L2.
__device__ __forceinline__ void tma_store_2d_evict_first(const CUtensorMap* map, const void* src, int c0, int c1) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mma_bf16_2sm(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
// Same MMA with an A-collector hint (tcgen05.mma ... .collector::a::{fill,use,lastuse}): the
// tensor core keeps the A slice it read in its collector buffer and the following MMAs of the
// same A re-use it instead of re-reading shared memory.
#define KGQ_MMA_COLLECTOR(NAME, Q)                                                                         \
  __device__ __forceinline__ void NAME(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,          \
                                       uint32_t accumulate) {                                              \
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"                                             \
                 "tcgen05.mma.cta_group::2.kind::f16" Q " [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),         \
                 "l"(da), "l"(db), "r"(idesc), "r"(accumulate));                                          \
  }
KGQ_MMA_COLLECTOR(mma_bf16_2sm_afill, ".collector::a::fill")
KGQ_MMA_COLLECTOR(mma_bf16_2sm_ause, ".collector::a::use")
KGQ_MMA_COLLECTOR(mma_bf16_2sm_alast, ".collector::a::lastuse")
#undef KGQ_MMA_COLLECTOR
// A operand from TMEM ("ts" form): D[tmem] (+)= A[tmem] . B[smem]; tmem_a = the A slice's first
// column (128 lanes = this CTA's rows, 8 columns = 16 bf16 of K per lane).
__device__ __forceinline__ void mma_bf16_2sm_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate));
}
// smem -> TMEM copy of a 128-row x 32-byte K-major slice (one K16 step of one bf16 plane of A),
// issued by the leader for both CTAs of the pair (each copies its own smem into its own TMEM);
// ordered before the MMAs issued after it (tcgen05.cp -> tcgen05.mma pipeline order).
__device__ __forceinline__ void tmem_cp_2sm_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar) {  // arrive on bar in both CTAs
  const uint16_t mask = 3;
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// Programmatic dependent launch: wait for the upstream grid's results / let the next grid's
// CTAs start their setup (no-ops when the launch carries no PDL attribute).
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#ifdef KGQ_TC_TRACE  // perf probe only (scripts/tc_trace.cu): per-tile globaltimer stamps
__device__ unsigned long long* g_tc_trace;
#define TC_TRACE(slot, i)                                                                                      \
  do {                                                                                                         \
    unsigned long long t_;                                                                                     \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                                     \
    g_tc_trace[(size_t)(slot) * 8 + (i)] = t_;                                                                 \
  } while (0)
#else
#define TC_TRACE(slot, i) do {} while (0)
#endif

// K-blocks per TMEM partial (see header comment).
// 4 for bf16x3: 1.4e-7 of sum|x w| at K = 1600 (DRAIN 2: 7.3e-8, 8: 2.7e-7, 16: 5.3e-7;
// scripts/tc_bn_check.cu 1600).  Round 2 measured the chain embeddings of every structure
// against the oracle at DRAIN 8 / 4 / 2 (profiles/r02/chain_err_drain.txt): DRAIN 8 left the
// non-negation structures at up to 9.9e-5 of the 1e-4 bound, DRAIN 4 at <= 6.5e-5 for -1% of
// the C2 step, DRAIN 2 at <= 2.6e-5 for -5% (its shorter partials hide the accumulator hand-off
// -- MMA commit -> epilogue drain -> accempty -- worse).
// fp16x2 operands (3 MMAs per K16 step instead of 6): DRAIN 8 puts the same 48 truncating MMA
// accumulations into a partial as bf16x3's DRAIN 4 -- chain errors vs the oracle at C2 <= 5.2e-5
// without negation (DRAIN 4: 3.1e-5, 16: 9.8e-5), inp 5.8e-4 (16: 1.2e-3, over its bound) -- for
// +5% on the C2 step (profiles/r02/operand_accuracy.txt).
#ifndef KGQ_TC_DRAIN
#define KGQ_TC_DRAIN (KGQ_OPERAND_FP16X2 ? 8 : 4)
#endif
constexpr int DRAIN_DEFAULT = KGQ_TC_DRAIN;
// An epilogue may set its own partial length (static constexpr int DRAIN): the BetaE scorer's
// contraction terms are small (centred u, v) and its K = 800 fits fewer, longer partials.
template <class E, class = void>
struct epi_drain : std::integral_constant<int, DRAIN_DEFAULT> {};
template <class E>
struct epi_drain<E, std::void_t<decltype(E::DRAIN)>> : std::integral_constant<int, E::DRAIN> {};

// Per-CTA shared memory: STAGES operand stages, then the epilogue staging buffers -- each
// epilogue warp owns NBUF x 4 KB holding a 32-row chunk of its columns in the 128-byte
// (1 plane, 32 columns) or 64-byte (2 planes, 16 columns each) swizzled layout of the output
// tensor map's box -- then the barriers.
#ifndef KGQ_TC_ATMEM
#define KGQ_TC_ATMEM 0
#endif
#ifndef KGQ_TC_COLLECTOR  // A-grouped MMA order with collector re-use (see the MMA issuer)
#define KGQ_TC_COLLECTOR 1
#endif
#ifndef KGQ_TC_NBUF2  // split-output launches trade one operand stage for double-buffered staging
#define KGQ_TC_NBUF2 1
#endif
template <int BN, bool NBUF2_ = false>
struct Layout {
  static constexpr bool NBUF2 = NBUF2_ && KGQ_TC_NBUF2;
  static constexpr int A_BYTES = BM * BK * 2;         // one bf16 plane of A: 8 KB
  static constexpr int W_BYTES = (BN / 2) * BK * 2;   // one plane of this CTA's half of the W tile
  static constexpr int STAGE_BYTES = kSplitPlanesA * A_BYTES + 3 * W_BYTES;  // A planes + 3 W planes
  static constexpr int W_OFF = kSplitPlanesA * A_BYTES;                       // first W plane
  static constexpr int BUF_BYTES = 4096;
  static constexpr int BUDGET = 227 * 1024 - 1024 - 256;  // minus alignment slack and barriers
  static constexpr int FIT = (BUDGET - EPI_WARPS * BUF_BYTES) / STAGE_BYTES;
  // NBUF2 (split-output dense layers, short one-wave launches): double-buffered epilogue
  // staging -- a chunk's st.shared does not wait for the previous chunk's TMA store to drain the
  // buffer -- at the price of one operand stage (C2: dense -1%; the long score GEMM keeps its
  // stages, where the extra stage is worth more)
  static constexpr int FIT2 = (BUDGET - 2 * EPI_WARPS * BUF_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = NBUF2 && FIT2 >= 3 ? (FIT2 > 6 ? 6 : FIT2) : (FIT > 6 ? 6 : FIT);
  static constexpr int NBUF = BUDGET - STAGES * STAGE_BYTES >= 2 * EPI_WARPS * BUF_BYTES ? 2 : 1;
  // A operand staged in TMEM (tcgen05.cp once per plane and K16 step, then the six MMAs read A
  // from TMEM and only B from shared memory): one 48-column A slot (3 planes x 2 K16 steps x 8
  // columns) per operand stage next to the two BN-column accumulators, if it fits in 512.
  static constexpr int A_SLOT_COLS = 3 * (BK / 16) * 8;
  static constexpr bool ATM = KGQ_TC_ATMEM && !kFp16x2 && 2 * BN + A_SLOT_COLS * STAGES <= 512;
  static constexpr int TMEM_COLS = ATM ? 512 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static constexpr int STG_OFF = STAGES * STAGE_BYTES;
  static constexpr int BAR_OFF = STG_OFF + NBUF * EPI_WARPS * BUF_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
  static_assert(TOTAL <= 227 * 1024, "shared memory budget");
  static_assert(STAGES >= 3, "pipeline depth");
  static_assert(BN % 32 == 0 && BN >= 64 && BN <= 256, "2-CTA tile: N multiple of 16 per CTA, CW multiple of 16");
};

// Work split of one launch.  Tiles [0, full) -- complete rounds over the clusters -- are
// computed whole; each remaining (tail) tile is split into s_tail K ranges of kper K-blocks so
// the last round fills the machine.  Every split writes its fp32 partial sums to the workspace
// and bumps a per-(tile, epilogue warp) counter; the warp that arrives last adds the other
// partials and runs the epilogue.  Nobody waits for another CTA, so the schedule is correct
// whatever subset of the grid is resident.
struct Sched {
  int full;    // tiles computed whole
  int s_tail;  // K splits per tail tile (1: none)
  int kper;    // K-blocks per split
  float* ws;   // [tail units][16 epilogue warps][BN / 8][32 lanes] float4 partial sums
  int* cnt;    // [tail tiles][16] arrival counters (zero between launches; the last arriver resets)
  unsigned long long* kt = nullptr;  // launch-span accounting of this stage (GemmWs::kt), or null
  int group_m = 0;   // tile raster: groups of group_m M-blocks, N-major inside a group (0: M fastest)
  int n_stripes = 0; // fused top-k epilogues (Epi::TOPK): N split into this many stripes of whole tiles
};
// Fused top-k epilogues (Epi::TOPK, score_tc.cu) keep per-row state across tiles, so their work
// unit is a row stripe: one 256-row M block x a contiguous range of N tiles, run by one cluster
// back to back (no split-K).  Other epilogues: one tile (or one K split of a tail tile) per unit.
template <class E, class = void>
struct epi_topk : std::false_type {};
template <class E>
struct epi_topk<E, std::void_t<decltype(E::TOPK)>> : std::integral_constant<bool, E::TOPK> {};
// Tile t -> (M block, N block).  Grouped raster: tiles of group_m consecutive M blocks (256 rows
// each) are ordered M fastest, then N, then the next group -- so the ~74 tiles in flight cover
// group_m row blocks x ~74 / group_m column blocks: the group's A rows (group_m x 256 x K x 6 B)
// stay in L2 while every column of W passes, and A is read from DRAM about once.  With plain M-
// fastest order every column of tiles swept all of A: at M = 14K, K = 1600 (137 MB of A, more
// than L2) ncu measured 2.7 GB of DRAM reads for one 15 MB-weight layer (profiles/r02).
__device__ __forceinline__ void tile_mn(int t, int m_pairs, int n_tiles, int group_m, int& m, int& n) {
  if (group_m <= 0 || group_m >= m_pairs) {
    m = t % m_pairs;
    n = t / m_pairs;
    return;
  }
  const int per_group = group_m * n_tiles;
  const int g = t / per_group, r = t - g * per_group;
  const int m0 = g * group_m;
  const int gm = min(group_m, m_pairs - m0);
  m = m0 + r % gm;
  n = r / gm;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Launch span = last CTA's end - first CTA's start (after griddepcontrol.wait, so a PDL-early
// CTA's wait for the predecessor is not counted); the last CTA to finish adds it to the group's
// sum, appends (start, end, stage) to the context's span log (base = kt - 8 group: [32] = count,
// [40 + 3 i ..] = entries, kKtLogCap of them) and re-arms the words for the next launch of the
// group (stream-ordered: that launch's CTAs pass griddepcontrol.wait only after this grid
// completed).  Groups: 0 dense, 1 score on the context's stream, 2 / 3 the same on its side
// stream (concurrent launches must not share a group).  Layout of a group's words:
// [start, end, ctas done, summed ns, launches, group, -, -].
__device__ __forceinline__ void kt_begin(unsigned long long* kt) {
  if (kt) atomicMin(&kt[0], globaltimer_ns());
}
__device__ __forceinline__ void kt_end(unsigned long long* kt) {
  if (!kt) return;
  atomicMax(&kt[1], globaltimer_ns());
  __threadfence();
  if (atomicAdd(&kt[2], 1ull) == gridDim.x - 1) {
    __threadfence();
    const unsigned long long t0 = atomicAdd(&kt[0], 0ull), t1 = atomicAdd(&kt[1], 0ull);
    kt[3] += t1 > t0 ? t1 - t0 : 0ull;
    kt[4] += 1ull;
    unsigned long long* base = kt - 8 * kt[5];
    const unsigned long long i = atomicAdd(&base[32], 1ull);
    if (i < kKtLogCap) {
      base[40 + 3 * i] = t0;
      base[41 + 3 * i] = t1;
      base[42 + 3 * i] = kt[5] & 1;  // stage: 0 dense, 1 score (groups 2 / 3: the side stream's)
    }
    kt[0] = ~0ull;
    kt[1] = 0ull;
    kt[2] = 0ull;
    __threadfence();
  }
}
// Unit u of a launch -> M block tm, N tiles [tn0, tn1), K blocks [kb0, kb1), tail slot v (-1: none).
template <bool TOPK>
__device__ __forceinline__ void unit_tiles(int u, const Sched& sc, int nk, int m_pairs, int n_tiles, int& tm,
                                           int& tn0, int& tn1, int& kb0, int& kb1, int& v);
__device__ __forceinline__ void unit_of(int u, const Sched& sc, int nk, int& t, int& kb0, int& kb1, int& v) {
  if (u < sc.full) {
    t = u; kb0 = 0; kb1 = nk; v = -1;
    return;
  }
  v = u - sc.full;  // tail unit: workspace slot
  t = sc.full + v / sc.s_tail;
  kb0 = (v % sc.s_tail) * sc.kper;
  kb1 = min(nk, kb0 + sc.kper);
}

template <class E>
__device__ __forceinline__ int epi_rows(const E& e) {
  if constexpr (epi_topk<E>::value) return e.rows;
  else return 0;
}

template <bool TOPK>
__device__ __forceinline__ void unit_tiles(int u, const Sched& sc, int nk, int m_pairs, int n_tiles, int& tm,
                                           int& tn0, int& tn1, int& kb0, int& kb1, int& v) {
  if constexpr (TOPK) {
    int st;
    tile_mn(u, m_pairs, sc.n_stripes, sc.group_m, tm, st);
    tn0 = (int)((int64_t)st * n_tiles / sc.n_stripes);  // balanced stripes: floor / ceil tiles each
    tn1 = (int)((int64_t)(st + 1) * n_tiles / sc.n_stripes);
    kb0 = 0;
    kb1 = nk;
    v = -1;
  } else {
    int t;
    unit_of(u, sc, nk, t, kb0, kb1, v);
    tile_mn(t, m_pairs, n_tiles, sc.group_m, tm, tn0);
    tn1 = tn0 + 1;
  }
}

// Lane-private sorted list of the k smallest (order key, column) pairs of one output row, in
// the epilogue warp's shared-memory slot (column-major [j][lane]: conflict-free).  Inserting a
// key below the current k-th drops the k-th.
__device__ __forceinline__ void topk_list_insert(unsigned long long* L, int lane, int k, int& cnt,
                                                 unsigned long long& thr, unsigned long long key) {
  int p = cnt < k ? cnt : k - 1;
  while (p > 0) {
    const unsigned long long prev = L[(p - 1) * 32 + lane];
    if (prev < key) break;
    L[p * 32 + lane] = prev;
    --p;
  }
  L[p * 32 + lane] = key;
  if (cnt < k) ++cnt;
  thr = cnt == k ? L[(k - 1) * 32 + lane] : ~0ull;
}
// v[i] for a run-time i < 32 from a register array: a 5-level select tree (31 FSEL), no local
// memory
__device__ __forceinline__ float pick32(const float* v, int i) {
  float t[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) t[j] = (i & 1) ? v[2 * j + 1] : v[2 * j];
#pragma unroll
  for (int j = 0; j < 8; ++j) t[j] = (i & 2) ? t[2 * j + 1] : t[2 * j];
#pragma unroll
  for (int j = 0; j < 4; ++j) t[j] = (i & 4) ? t[2 * j + 1] : t[2 * j];
#pragma unroll
  for (int j = 0; j < 2; ++j) t[j] = (i & 8) ? t[2 * j + 1] : t[2 * j];
  return (i & 16) ? t[1] : t[0];
}
__device__ __forceinline__ uint32_t topk_fkey(float f) {  // order-preserving (NaN max, -0 = +0)
  if (f != f) return 0xFFFFFFFFu;
  if (f == 0.0f) f = 0.0f;
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float topk_fkey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// Epilogue policy concept (linear_tc.cu, score_tc.cu):
//   static constexpr int PLANES  -- 1: fp32 output; 3: split output (three bf16 planes, exact)
//   static constexpr int ROWDIV  -- 1, or 2: output row r = min over tile rows 2r, 2r+1 (DNF union)
//   struct Pre; template <int CW> __device__ Pre prefetch(int row, int n0, int lane) const
//       -- per-tile operands (row terms, and column vectors with lane l holding columns
//          n0 + l + 32 j), loaded before the tile's drains so their latency is hidden
//   template <int CH> __device__ void chunk(const Pre&, int row, int c, float* v) const
//       -- v[i] (i < CH) = accumulator of (row, n0 + c + i) on entry, output value on exit;
//          column operands come from the prefetched registers by warp shuffle
//   static constexpr bool CMIN; template <int CH> __device__ void chunk_min(int row, int n,
//       const float* v) const -- optional side output after the row-pair min (score top-k)
//   static constexpr bool INIT; template <int CW> __device__ void init(int row, int n0,
//       float* acc) const -- optional initial accumulator values (relation term of layer 1)
//   __device__ int out_row(int row0) const -- output tensor row of the 32 / ROWDIV-row box that
//       starts at GEMM row row0 (row0 / ROWDIV, or a remapped row; -1: do not store the box)
//   static constexpr bool TOPK (optional) -- fused top-k: no output tensor; every output row's
//       k (<= 16) smallest (value, column) pairs over the unit's stripe are kept in the warp's
//       staging slot and written as one sorted list per (row, stripe, column half) to
//       epi.cand[orow * epi.ldcand + (stripe * 2 + half) * epi.k + j] as (order key << 32 | col);
//       epi.rows / epi.nvalid bound the valid rows / columns
// Output tensor maps: PLANES 1: fp32, box {32 columns, 32 / ROWDIV rows}, 128-byte swizzle;
// PLANES 3: bf16 plane p, box {16 columns, 32 rows}, 32-byte swizzle.
template <int BN, class Epi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_gemm(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
           const __grid_constant__ CUtensorMap mWh, const __grid_constant__ CUtensorMap mWl,
           const __grid_constant__ CUtensorMap mA2, const __grid_constant__ CUtensorMap mW2,
           const __grid_constant__ CUtensorMap mO0, const __grid_constant__ CUtensorMap mO1,
           const __grid_constant__ CUtensorMap mO2, int M, int N, int K, const Sched sc, const Epi epi) {
  using L = Layout<BN, Epi::PLANES == 3>;
  constexpr int STAGES = L::STAGES;
  constexpr int PLANES = Epi::PLANES, ROWDIV = Epi::ROWDIV;
  constexpr int CW = BN / 2;            // columns per epilogue warp
  constexpr int CH = PLANES == 1 ? 32 : 16;  // columns per staged chunk
  static_assert(CW % CH == 0, "fp32 outputs (32-column chunks) need BN % 64 == 0");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* accfull = empty + STAGES;   // [2] partial ready in TMEM buffer a
  uint64_t* accempty = accfull + 2;     // [2] partial drained by both CTAs' epilogue warps
  uint32_t* tmem_slot = (uint32_t*)(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int m_pairs = (M + 2 * BM - 1) / (2 * BM);
  constexpr bool TOPK = epi_topk<Epi>::value;
  constexpr int DRAIN = epi_drain<Epi>::value;
  const int n_tiles = (N + BN - 1) / BN;
  const int ntiles = m_pairs * n_tiles;
  const int nunits = TOPK ? m_pairs * sc.n_stripes : sc.full + (ntiles - sc.full) * sc.s_tail;
  const int nk = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mAh);
    tma_prefetch(&mAl);
    tma_prefetch(&mA2);
    tma_prefetch(&mWh);
    tma_prefetch(&mWl);
    tma_prefetch(&mW2);
    tma_prefetch(&mO0);
    if (PLANES == 3) {
      tma_prefetch(&mO1);
      tma_prefetch(&mO2);
    }
    for (int s = 0; s < STAGES; ++s) {
#ifdef KGQ_TC_DBG_NO_TMA
      mbar_init(&full[s], 2);
#else
      mbar_init(&full[s], 1);
#endif
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&accfull[a], 1);
      mbar_init(&accempty[a], 2 * EPI_WARPS);  // epilogue warps of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // two partial accumulators: 128 lanes x 2 BN fp32 columns per CTA
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  cluster_sync_all();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  // everything above overlaps the upstream grid's tail; its outputs are read only below
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) kt_begin(sc.kt);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs; completions counted by the leader) ----------------
      uint32_t it = 0;
      for (int u = cluster; u < nunits; u += nclusters) {
        int tm, tn0, tn1, kb0, kb1, v;
        unit_tiles<TOPK>(u, sc, nk, m_pairs, n_tiles, tm, tn0, tn1, kb0, kb1, v);
        const int m0 = tm * 2 * BM + (int)rank * BM;
        for (int tn = tn0; tn < tn1; ++tn)
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int nw = tn * BN + (int)rank * (BN / 2);
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait_backoff(&empty[s], ((it / STAGES) - 1) & 1);
          uint8_t* st = smem + s * L::STAGE_BYTES;
          const uint32_t lb = mapa_shared(smem_u32(&full[s]), 0);
#ifdef KGQ_TC_DBG_NO_TMA  // perf probe only: no operand loads, each CTA arrives on the leader's barrier
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(lb) : "memory");
          (void)st;
          continue;
#endif
          if (leader) mbar_expect_tx(&full[s], 2 * L::STAGE_BYTES);
          tma_load_2d_2sm(st, &mAh, lb, kb * BK, m0);
          tma_load_2d_2sm(st + L::A_BYTES, &mAl, lb, kb * BK, m0);
          if constexpr (!kFp16x2) tma_load_2d_2sm(st + 2 * L::A_BYTES, &mA2, lb, kb * BK, m0);
          tma_load_2d_2sm(st + L::W_OFF, &mWh, lb, kb * BK, nw);
          tma_load_2d_2sm(st + L::W_OFF + L::W_BYTES, &mWl, lb, kb * BK, nw);
          tma_load_2d_2sm(st + L::W_OFF + 2 * L::W_BYTES, &mW2, lb, kb * BK, nw);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader only): M = 256 over the pair, N = BN ----------------
      // instruction descriptor: D f32, A/B bf16, both K-major, N = BN, M = 256 over the pair
      // A / B formats: bf16 = 1 (bits 7-9, 10-12), f16 = 0
      const uint32_t fmt = kFp16x2 ? 0u : 1u;
      const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)((2 * BM) >> 4) << 24);
      uint32_t it = 0, g0 = 0;
      for (int u = cluster; u < nunits; u += nclusters) {
        int tm, tn0, tn1, kb0, kb1, v;
        unit_tiles<TOPK>(u, sc, nk, m_pairs, n_tiles, tm, tn0, tn1, kb0, kb1, v);
        TC_TRACE(u, 0);
        for (int tn = tn0; tn < tn1; ++tn) {
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const int kr = kb - kb0;
          const uint32_t g = g0 + kr / DRAIN, a = g & 1;
          const bool first = (kr % DRAIN) == 0;
          if (first && g >= 2) mbar_wait(&accempty[a], ((g >> 1) - 1) & 1);
          mbar_wait(&full[s], (it / STAGES) & 1);
          if (kr == 0) TC_TRACE(u, 1);
          fence_after();
          const uint32_t d = tmem + a * BN;
          const uint32_t st = smem_u32(smem + s * L::STAGE_BYTES);
          const uint32_t a0 = st, a1 = st + L::A_BYTES, a2 = st + 2 * L::A_BYTES;
          const uint32_t w0 = st + L::W_OFF, w1 = w0 + L::W_BYTES, w2 = w1 + L::W_BYTES;
          if constexpr (L::ATM) {
            // A slot of this stage (free: the MMAs of the stage's previous K-block completed
            // before the producer refilled the stage, i.e. before full[s] fired)
            const uint32_t ta = tmem + 2 * BN + s * L::A_SLOT_COLS;
#pragma unroll
            for (int p = 0; p < 3; ++p)
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk)
                tmem_cp_2sm_128x256b(ta + (p * (BK / 16) + kk) * 8, umma_desc_sw64(st + p * L::A_BYTES + kk * 32));
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t off = kk * 32;
              const uint32_t t0 = ta + kk * 8, t1 = t0 + (BK / 16) * 8, t2 = t1 + (BK / 16) * 8;
              mma_bf16_2sm_ts(d, t0, umma_desc_sw64(w2 + off), idesc, (first && kk == 0) ? 0u : 1u);
              mma_bf16_2sm_ts(d, t1, umma_desc_sw64(w1 + off), idesc, 1u);
              mma_bf16_2sm_ts(d, t2, umma_desc_sw64(w0 + off), idesc, 1u);
              mma_bf16_2sm_ts(d, t0, umma_desc_sw64(w1 + off), idesc, 1u);
              mma_bf16_2sm_ts(d, t1, umma_desc_sw64(w0 + off), idesc, 1u);
              mma_bf16_2sm_ts(d, t0, umma_desc_sw64(w0 + off), idesc, 1u);
            }
          } else if constexpr (kFp16x2) {
            // fp16x2: a_l' w_h + a_h w_l' + a_h w_h' (w planes: 0 = h 2^11, 1 = l', 2 = h), all
            // scaled by 2^11 into one accumulator; the small terms first, a_h re-used from the
            // collector
            (void)a2;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t off = kk * 32;
              mma_bf16_2sm(d, umma_desc_sw64(a1 + off), umma_desc_sw64(w2 + off), idesc, (first && kk == 0) ? 0u : 1u);
              mma_bf16_2sm_afill(d, umma_desc_sw64(a0 + off), umma_desc_sw64(w1 + off), idesc, 1u);
              mma_bf16_2sm_alast(d, umma_desc_sw64(a0 + off), umma_desc_sw64(w0 + off), idesc, 1u);
            }
          } else if constexpr (KGQ_TC_COLLECTOR) {
            // A-grouped order with collector re-use: each A plane is read from shared memory
            // once per K16 step (3 reads instead of 6) -- less SMEM traffic and power for the
            // same MMAs; small terms still first, x0 w0 last
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t off = kk * 32;
              mma_bf16_2sm(d, umma_desc_sw64(a2 + off), umma_desc_sw64(w0 + off), idesc, (first && kk == 0) ? 0u : 1u);
              mma_bf16_2sm_afill(d, umma_desc_sw64(a1 + off), umma_desc_sw64(w1 + off), idesc, 1u);
              mma_bf16_2sm_alast(d, umma_desc_sw64(a1 + off), umma_desc_sw64(w0 + off), idesc, 1u);
              mma_bf16_2sm_afill(d, umma_desc_sw64(a0 + off), umma_desc_sw64(w2 + off), idesc, 1u);
              mma_bf16_2sm_ause(d, umma_desc_sw64(a0 + off), umma_desc_sw64(w1 + off), idesc, 1u);
              mma_bf16_2sm_alast(d, umma_desc_sw64(a0 + off), umma_desc_sw64(w0 + off), idesc, 1u);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {  // 16 bf16 = 32 bytes per MMA along K
              const uint32_t off = kk * 32;
              // small terms first; x0 w0 last
              mma_bf16_2sm(d, umma_desc_sw64(a0 + off), umma_desc_sw64(w2 + off), idesc,
                           (first && kk == 0) ? 0u : 1u);
              mma_bf16_2sm(d, umma_desc_sw64(a1 + off), umma_desc_sw64(w1 + off), idesc, 1u);
              mma_bf16_2sm(d, umma_desc_sw64(a2 + off), umma_desc_sw64(w0 + off), idesc, 1u);
              mma_bf16_2sm(d, umma_desc_sw64(a0 + off), umma_desc_sw64(w1 + off), idesc, 1u);
              mma_bf16_2sm(d, umma_desc_sw64(a1 + off), umma_desc_sw64(w0 + off), idesc, 1u);
              mma_bf16_2sm(d, umma_desc_sw64(a0 + off), umma_desc_sw64(w0 + off), idesc, 1u);
            }
          }
          mma_commit_2sm(&empty[s]);  // frees the smem stage (both CTAs) once these MMAs have read it
          if ((kr % DRAIN) == DRAIN - 1 || kb == kb1 - 1) mma_commit_2sm(&accfull[a]);
        }
        g0 += (kb1 - kb0 + DRAIN - 1) / DRAIN;
        }
        TC_TRACE(u, 2);
      }
    }
  } else if (warp >= EPI_WARP0) {
    // -------- epilogue warps 2..9: TMEM lane quarter = warp % 4 (rows), column half --------
    const int q = warp & 3;
    const int ch = ((warp - EPI_WARP0) >> 2) * CW;
    uint8_t* stg = smem + L::STG_OFF + (warp - EPI_WARP0) * L::BUF_BYTES;
    const uint32_t accempty_leader = mapa_shared(smem_u32(&accempty[0]), 0);
    uint32_t g0 = 0, nchunk = 0;
    for (int u = cluster; u < nunits; u += nclusters) {
      int tm, tn0, tn1, kb0, kb1, v;
      unit_tiles<TOPK>(u, sc, nk, m_pairs, n_tiles, tm, tn0, tn1, kb0, kb1, v);
      const int ng = (kb1 - kb0 + DRAIN - 1) / DRAIN;
      const int row0 = tm * 2 * BM + (int)rank * BM + q * 32;
      // fused top-k: this lane's output row, its sorted list (count, k-th key, k-th value)
      const bool trow = TOPK && (row0 + lane) < epi_rows(epi) && (ROWDIV == 1 || (lane & 1) == 0);
      int tcnt = 0;
      unsigned long long tthr = ~0ull;
      float tthr_f = __uint_as_float(0x7F800000u);
      unsigned long long* tlist = reinterpret_cast<unsigned long long*>(stg);
      for (int tn = tn0; tn < tn1; ++tn) {
      const int n0 = tn * BN + ch;
      const auto pre = epi.template prefetch<CW>(row0 + lane, n0, lane);
      float acc[CW];
#pragma unroll
      for (int i = 0; i < CW; ++i) acc[i] = 0.0f;
      // optional per-(row, column) initial value, added once (by the split holding K-block 0);
      // loaded here so its latency hides under the first partial's MMAs
      if constexpr (Epi::INIT)
        if (kb0 == 0) epi.template init<CW>(row0 + lane, n0, acc);
      for (int gi = 0; gi < ng; ++gi) {
        const uint32_t g = g0 + gi, a = g & 1;
        mbar_wait_backoff(&accfull[a], (g >> 1) & 1);
        fence_after();
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + a * BN + ch;
#ifndef KGQ_TC_DBG_NO_DRAIN  // perf probe only: skip the TMEM reads
#pragma unroll
        for (int c = 0; c < CW; c += 16) {  // x16 loads: few live temporaries next to acc[CW]
          float v[16];
          tmem_ld16(tq + c, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c + i] = kFp16x2 ? fmaf(v[i], kLoInv, acc[c + i]) : acc[c + i] + v[i];
        }
#else
        (void)tq;
#endif
        fence_before();
        __syncwarp();
        // default .release.cta semantics: the TMEM reads are complete (tcgen05.wait::ld) and
        // fenced; a .cluster-scope release would cost a MEMBAR.ALL.GPU per drain
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(accempty_leader + a * 8) : "memory");
      }
      g0 += ng;
      if (warp == EPI_WARP0 && lane == 0 && leader) TC_TRACE(u, 3);
      if (v >= 0 && sc.s_tail > 1) {
        // ---- split tail tile: publish this split's partial sums; the last arriver reduces ----
        const int tt = v / sc.s_tail, slot = (int)rank * EPI_WARPS + (warp - EPI_WARP0);
        // workspace slot of (unit, warp): [CW / 4][32 lanes] float4, so every access is 512 B
        // contiguous per warp (row-per-lane addressing would cost one L2 request per lane)
        float4* mine = reinterpret_cast<float4*>(sc.ws) + ((size_t)v * 2 * EPI_WARPS + slot) * 8 * CW + lane;
#pragma unroll
        for (int c = 0; c < CW; c += 4) __stcg(mine + c * 8, make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]));
        fence_acq_rel_gpu();  // release: this lane's partials before the arrival count
        __syncwarp();
        if (warp == EPI_WARP0 && lane == 0 && leader) TC_TRACE(u, 5);
        int old = 0;
        if (lane == 0) old = atomicAdd(&sc.cnt[tt * 2 * EPI_WARPS + slot], 1);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (warp == EPI_WARP0 && lane == 0 && leader) TC_TRACE(u, 6);
        if (old != sc.s_tail - 1) {  // another split finishes this slice
          if (warp == EPI_WARP0 && lane == 0 && leader) TC_TRACE(u, 4);
          continue;
        }
        fence_acq_rel_gpu();  // acquire: the other splits' partials after their counts
        for (int s2 = 0; s2 < sc.s_tail; ++s2) {
          if (s2 == v % sc.s_tail) continue;
          const float4* other =
              reinterpret_cast<const float4*>(sc.ws) + ((size_t)(tt * sc.s_tail + s2) * 2 * EPI_WARPS + slot) * 8 * CW + lane;
#pragma unroll
          for (int c = 0; c < CW; c += 4) {
            const float4 o = __ldcg(other + c * 8);
            acc[c] += o.x;
            acc[c + 1] += o.y;
            acc[c + 2] += o.z;
            acc[c + 3] += o.w;
          }
        }
        if (lane == 0) sc.cnt[tt * 2 * EPI_WARPS + slot] = 0;  // ready for the next launch
        if (warp == EPI_WARP0 && lane == 0 && leader) TC_TRACE(u, 7);
      }
      // ---- epilogue of this tile (the MMA warp is already on the next tile's partials) ----
      if constexpr (TOPK) {
        static_assert(CH == 32 && L::BUF_BYTES >= 32 * 16 * 8, "top-k lists: 16 keys x 32 lanes per warp slot");
#pragma unroll
        for (int c = 0; c < CW; c += CH) {
          float* v = acc + c;
          epi.template chunk<CH>(pre, row0 + lane, c, v);
          if (ROWDIV == 2) {
#pragma unroll
            for (int i = 0; i < CH; ++i) v[i] = fminf(v[i], __shfl_xor_sync(0xffffffffu, v[i], 1));
          }
          // candidates of this chunk: a 32-bit mask of the values <= the lane's k-th (ties and NaN
          // are settled by the exact key test below), then a compact loop over the set bits -- one
          // copy of the insertion code per chunk instead of 32 unrolled ones (the unrolled form
          // overflowed the instruction cache: ncu stall_no_inst was the top epilogue stall)
          const int cb = n0 + c;
          unsigned pm = 0;
#pragma unroll
          for (int i = 0; i < CH; ++i) pm |= (v[i] <= tthr_f ? 1u : 0u) << i;
          const int64_t left = epi.nvalid - cb;
          if (left < CH) pm &= left > 0 ? (1u << left) - 1u : 0u;
          if (!trow) pm = 0;
          while (pm) {
            const int i = __ffs(pm) - 1;
            pm &= pm - 1;
            const float vi = pick32(v, i);
            const unsigned long long key = ((unsigned long long)topk_fkey(vi) << 32) | (uint32_t)(cb + i);
            if (key < tthr) {
              topk_list_insert(tlist, lane, epi.k, tcnt, tthr, key);
              tthr_f = tcnt == epi.k ? topk_fkey_inv((uint32_t)(tthr >> 32)) : __uint_as_float(0x7F800000u);
            }
          }
        }
        continue;
      }
      // output row of this warp's 32 / ROWDIV-row box (row0 / ROWDIV, or the remapped row; -1:
      // none): once per tile, not per chunk (the remap's segment search is ~50 instructions)
      const int orow = epi.out_row(row0);
#pragma unroll
      for (int c = 0; c < CW; c += CH, ++nchunk) {
        float* v = acc + c;  // in place (unrolled: stays in registers)
        epi.template chunk<CH>(pre, row0 + lane, c, v);
        if (ROWDIV == 2) {
#pragma unroll
          for (int i = 0; i < CH; ++i) v[i] = fminf(v[i], __shfl_xor_sync(0xffffffffu, v[i], 1));
        }
        if constexpr (Epi::CMIN) epi.template chunk_min<CH>(row0 + lane, n0 + c, v);
        uint8_t* buf = stg + (nchunk % L::NBUF) * (EPI_WARPS * L::BUF_BYTES);
        if (lane == 0) bulk_wait_read<L::NBUF - 1>();  // this buffer's previous store has read it
        __syncwarp();
        if (PLANES == 1) {
          const int r = ROWDIV == 2 ? lane >> 1 : lane;  // output row within the 32 / ROWDIV box
          if (ROWDIV == 1 || (lane & 1) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(buf + r * 128 + ((j ^ (r & 7)) << 4)) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
        } else {
          // 16 columns -> three bf16 planes of 32 rows x 32 B (1 KB each), 32-byte swizzle:
          // 16-byte chunk c of row r at r * 32 + ((c ^ ((r >> 2) & 1)) << 4)
          uint32_t q0[8], q1[8], q2[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) split3_pair(v[2 * i], v[2 * i + 1], q0[i], q1[i], q2[i]);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int o = lane * 32 + ((c ^ ((lane >> 2) & 1)) << 4);
            *reinterpret_cast<uint4*>(buf + o) = make_uint4(q0[4 * c], q0[4 * c + 1], q0[4 * c + 2], q0[4 * c + 3]);
            *reinterpret_cast<uint4*>(buf + 1024 + o) = make_uint4(q1[4 * c], q1[4 * c + 1], q1[4 * c + 2], q1[4 * c + 3]);
            *reinterpret_cast<uint4*>(buf + 2048 + o) = make_uint4(q2[4 * c], q2[4 * c + 1], q2[4 * c + 2], q2[4 * c + 3]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
#ifndef KGQ_TC_DBG_NO_STORE  // perf probe only: skip the output stores
        if (lane == 0) {
          if (orow >= 0) {
            if (Epi::STREAM_OUT)
              tma_store_2d_evict_first(&mO0, buf, n0 + c, orow);
            else
              tma_store_2d(&mO0, buf, n0 + c, orow);
            if (PLANES == 3) {
              tma_store_2d(&mO1, buf + 1024, n0 + c, orow);
              if constexpr (!kFp16x2) tma_store_2d(&mO2, buf + 2048, n0 + c, orow);
            }
          }
          bulk_commit();
        }
#endif
      }
      if (warp == EPI_WARP0 && lane == 0 && leader) TC_TRACE(u, 4);
      }  // tiles of the unit
      if constexpr (TOPK) {  // the stripe's list of this (row, column half)
        if (trow) {
          int tm2, stripe;
          tile_mn(u, m_pairs, sc.n_stripes, sc.group_m, tm2, stripe);
          const int half = (warp - EPI_WARP0) >> 2;
          unsigned long long* dst = epi.cand + (int64_t)((row0 + lane) / ROWDIV) * epi.ldcand +
                                    (int64_t)(stripe * 2 + half) * epi.k;
          for (int j = 0; j < epi.k; ++j) dst[j] = j < tcnt ? tlist[j * 32 + lane] : ~0ull;
        }
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  fence_before();
  cluster_sync_all();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(L::TMEM_COLS));
  }
  if (threadIdx.x == 0) kt_end(sc.kt);
}

// ---- host: tensor maps (cached per buffer) -----------------------------------------------
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)p;
  });
  return fn;
}

// rows x cols matrix (fp32 or bf16) with row stride ld (elements); box = box_rows x box_cols
inline bool make_map(CUtensorMap* m, const void* ptr, bool bf16, int64_t rows, int64_t cols, int64_t ld,
                     int box_rows, int box_cols, CUtensorMapSwizzle sw) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int64_t, int64_t, int64_t, int, int, int>, CUtensorMap> cache;
  const auto key = std::make_tuple(ptr, rows, cols, ld, box_rows, box_cols * (bf16 ? -1 : 1), (int)sw);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *m = it->second;
    return true;
  }
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  const size_t es = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "libkgq: cuTensorMapEncodeTiled(rows %lld, cols %lld, ld %lld, box %dx%d) = %d\n",
            (long long)rows, (long long)cols, (long long)ld, box_rows, box_cols, (int)r);
    return false;
  }
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *m);
  return true;
}
// bf16 operand plane: box rows x 32 columns (64 B), 64-byte swizzle (umma_desc_sw64)
inline bool make_operand_map(CUtensorMap* m, const __nv_bfloat16* p, int64_t rows, int64_t cols, int64_t ld,
                             int box_rows) {
  return make_map(m, p, true, rows, cols, ld, box_rows, BK, CU_TENSOR_MAP_SWIZZLE_64B);
}

// Output of a GEMM launch: rows x cols (rows = M / ROWDIV), either fp32 (f32, row stride ld;
// PLANES 1) or the three bf16 planes of a Split (PLANES 3).
struct OutDesc {
  float* f32;
  int64_t ld;
  Split sp;
  int64_t rows, cols;
};


// Per-context scratch of the split tail (kgq_internal.cuh GemmWs): at most kClustersMax tail
// units of 256 x 256 fp32 and kClustersMax x 16 counters.
static_assert(kGemmWsFloats >= (size_t)kClustersMax * 2 * BM * 256, "split-tail workspace");
static_assert(kGemmCntInts >= kClustersMax * 2 * EPI_WARPS, "split-tail counters");

template <int BN, class Epi>
int launch_gemm(const Split& A, int M, const Split& W, int N, int K, const OutDesc& o, const Epi& epi,
                cudaStream_t st, Sched sc, int max_clusters = 0) {
  if (max_clusters <= 0) max_clusters = gemm_clusters();
  constexpr int PLANES = Epi::PLANES, ROWDIV = Epi::ROWDIV;
  static_assert(PLANES == 1 || PLANES == 3, "fp32 or bf16x3 output");
  CUtensorMap mA[3], mW[3], mO[3];
  bool ok = true;
  for (int p = 0; p < 3; ++p) {
    ok = ok && make_operand_map(&mA[p], A.plane(p), M, K, A.ld, BM);
    ok = ok && make_operand_map(&mW[p], W.plane(p), N, K, W.ld, BN / 2);
  }
  if constexpr (epi_topk<Epi>::value) {  // no output tensor: the lists go to epi.cand
    mO[0] = mO[1] = mO[2] = mA[0];
  } else if (PLANES == 1) {
    ok = ok && make_map(&mO[0], o.f32, false, o.rows, o.cols, o.ld, 32 / ROWDIV, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    mO[1] = mO[2] = mO[0];
  } else {
    for (int p = 0; p < 3; ++p)
      ok = ok && make_map(&mO[p], o.sp.plane(p), true, o.rows, o.cols, o.sp.ld, 32, 16, CU_TENSOR_MAP_SWIZZLE_32B);
  }
  if (!ok) {
    fprintf(stderr, "libkgq: cuTensorMapEncodeTiled failed\n");
    return -1;
  }
  auto kern = k_gemm<BN, Epi>;
  static SmemAttr attr;
  smem_attr_once(kern, Layout<BN, Epi::PLANES == 3>::TOTAL, attr);
  const int tiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN);
  if (sc.s_tail <= 1 || !sc.ws || !sc.cnt || epi_topk<Epi>::value) {
    sc.full = tiles;
    sc.s_tail = 1;
  }
  if constexpr (epi_topk<Epi>::value) {
    const int nt = (N + BN - 1) / BN;
    sc.n_stripes = std::max(1, std::min(sc.n_stripes, nt));
  }
  const int units = epi_topk<Epi>::value ? ((M + 2 * BM - 1) / (2 * BM)) * sc.n_stripes
                                         : sc.full + (tiles - sc.full) * sc.s_tail;
  const int clusters = units < max_clusters ? units : max_clusters;
  if (sc.group_m == 0) sc.group_m = (Epi::CMIN || epi_topk<Epi>::value) ? gemm_group_m() : gemm_group_m_dense();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = Layout<BN, Epi::PLANES == 3>::TOTAL;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_gemm_enabled() ? 1 : 0;
  // KGQ_PLAN_LOG=1 (diagnostics, scripts/diag_gemm_launches.py): one stderr line per launch, in
  // launch order, to pair with the kgq_ktime_log spans of the same sequence
  static const bool plan_log = [] { const char* e = getenv("KGQ_PLAN_LOG"); return e && e[0] == '1'; }();
  if (plan_log)
    fprintf(stderr, "KGQ_PLAN M=%d N=%d K=%d BN=%d tiles=%d full=%d s_tail=%d kper=%d stripes=%d clusters=%d topk=%d planes=%d\n",
            M, N, K, BN, tiles, sc.full, sc.s_tail, sc.kper, sc.n_stripes, clusters, (int)epi_topk<Epi>::value,
            Epi::PLANES);
  cudaLaunchKernelEx(&cfg, kern, mA[0], mA[1], mW[0], mW[1], mA[2], mW[2], mO[0], mO[1], mO[2], M, N, K, sc, epi);
  return 1;
}

// Launch plan: tile width and tail split, from the measured cost model below.  Complete rounds
// of whole tiles run back to back (their epilogues overlap the next tile); a split tail tile
// costs its kper K-blocks + publishing its partials + adding the other splits' partials.
struct Plan {
  int bn, full, s_tail, kper;
};
// Cost model in us, least-squares fit (scripts/fit_plan.py) to every (BN, tail split) plan of 17
// dense / score shapes of the C2-C4 workloads measured on B200 (`PROBE_SPLITS=1
// scripts/tc_probe_base`, profiles/r01/tc_plan_fit.txt):
//   t = c0 + whole rounds x nk x kb[BN] + tail kper x kb[BN] + [split] (pub + (s-1) part) x BN
// (picks a plan within 3.4 us of the best over all 17 shapes; the previous clock-count model
// lost ~14 us, mostly on the N = 400 / 1600, K = 800 layers at M = 1-3K).
// bf16x3 operands (6 MMAs per K16 step; profiles/r01/tc_plan_fit.txt)
constexpr double kKbUsB[5] = {0.623, 0.675, 0.687, 0.760, 1.004};  // BN 64 128 160 192 256
// fp16x2 operands (3 MMAs per K16 step, DRAIN 8), refit on 26 shapes incl. the mixed step's M = 4-28K
// layers (profiles/r02/tc_plan_fit_fp16x2.txt): per column BN = 256 is now the cheapest tile
constexpr double kKbUsH[5] = {0.493, 0.494, 0.516, 0.533, 0.633};
constexpr const double* kKbUs = kFp16x2 ? kKbUsH : kKbUsB;
constexpr double kC0Us = kFp16x2 ? -1.12 : 3.40, kPubUs = kFp16x2 ? 0.0281 : 0.0230,
                 kPartUs = kFp16x2 ? 0.0163 : 0.0113;
// 160 (split-output dense layers only: 16-column chunks) tiles N = 800 / 1600 exactly
constexpr int kTileBN[5] = {64, 128, 160, 192, 256};
struct PlanKnobs {  // tuning experiments only (scripts/gpu_ab.sh): KGQ_GEMM_BN, KGQ_GEMM_KB128 (us per K-block)
  int force_bn = 0;
  double kb128 = 0.0, kb256 = 0.0;
  bool no160 = false;
  bool deterministic = true;  // KGQ_DETERMINISTIC=0 allows more than two K-splits (plan_gemm)
  PlanKnobs() {
    const char* dt = getenv("KGQ_DETERMINISTIC");
    if (dt && dt[0]) deterministic = dt[0] != '0';
    const char* n = getenv("KGQ_GEMM_NO160");
    no160 = n && n[0] && n[0] != '0';
    const char* e = getenv("KGQ_GEMM_BN");
    if (e) force_bn = atoi(e);
    e = getenv("KGQ_GEMM_KB128");
    if (e) kb128 = atof(e);
    e = getenv("KGQ_GEMM_KB256");
    if (e) kb256 = atof(e);
  }
};
inline Plan plan_gemm(int64_t M, int64_t N, int64_t K, bool can_split, bool allow160) {
  static const PlanKnobs knobs;
  const int64_t pairs_m = (M + 2 * BM - 1) / (2 * BM);
  const int nk = (int)((K + BK - 1) / BK);
  Plan best{kTileBN[0], 0, 1, nk};
  double best_cost = 1e300;
  for (int bn : kTileBN) {
    if (knobs.force_bn && bn != knobs.force_bn) continue;
    if (bn == 160 && (!allow160 || knobs.no160)) continue;
    const int64_t tiles = pairs_m * ((N + bn - 1) / bn);
    const int cl = gemm_clusters();
    const int64_t full = tiles / cl * cl, tail = tiles - full;
    double kb = kKbUs[bn == 64 ? 0 : bn == 128 ? 1 : bn == 160 ? 2 : bn == 192 ? 3 : 4];
    if (bn == 128 && knobs.kb128 > 0) kb = knobs.kb128;
    if (bn == 256 && knobs.kb256 > 0) kb = knobs.kb256;
    // Two partials commute exactly; with three or more the last-arriving split adds the others
    // after its own, so the fp32 grouping (and the last bit) depends on arrival order.
    // Default: at most two splits, so reruns are bit-identical (measured cost on C2: ~0.1%);
    // KGQ_DETERMINISTIC=0 lifts the cap.
    const int scap = knobs.deterministic ? 2 : 6;
    const int smax = can_split && tail > 0 ? (int)std::max<int64_t>(1, std::min<int64_t>(cl / tail, std::min(scap, nk / 4))) : 1;
    for (int s = 1; s <= smax; ++s) {
      const int kper = (nk + s - 1) / s;
      const int se = (nk + kper - 1) / kper;  // no empty split
      const double cost = kC0Us + (double)(full / cl) * nk * kb +
                          (tail ? kper * kb + (se > 1 ? (kPubUs + kPartUs * (se - 1)) * bn : 0.0) : 0.0);
      if (cost < best_cost) {
        best_cost = cost;
        best = Plan{bn, (int)full, se, kper};
      }
    }
  }
  return best;
}

// Fused top-k launch plan: tile width and the number of N stripes (units = M blocks x stripes,
// each unit's tiles run back to back on one cluster; <= 64 stripes: a row's 2 x stripes lists
// are merged by one warp holding 4 list heads per lane).  Cost = rounds over the clusters x the longest stripe's
// K-blocks (same per-K-block model as plan_gemm) + a per-unit list flush.
struct PlanTopk {
  int bn, n_stripes;
};
inline PlanTopk plan_gemm_topk(int64_t M, int64_t N, int64_t K, int min_tiles) {
  static const int force_s = [] { const char* e = getenv("KGQ_TOPK_STRIPES"); return e ? atoi(e) : 0; }();
  static const int force_bn = [] { const char* e = getenv("KGQ_TOPK_BN"); return e ? atoi(e) : 0; }();
  const int64_t pairs_m = (M + 2 * BM - 1) / (2 * BM);
  const int nk = (int)((K + BK - 1) / BK);
  const int cl = gemm_clusters();
  PlanTopk best{256, 1};
  double best_cost = 1e300;
  for (int bn : {128, 192, 256}) {
    if (force_bn && bn != force_bn) continue;
    const double kb = kKbUs[bn == 128 ? 1 : bn == 192 ? 3 : 4];
    const int nt = (int)((N + bn - 1) / bn);
    for (int s = 1; s <= std::min(64, std::max(1, nt / std::max(1, min_tiles))); ++s) {
      if (force_s && s != std::min(force_s, nt)) continue;
      // static round-robin of units over the clusters: the busiest cluster runs `rounds` units
      // of nt / s tiles on average (stripes are balanced to floor / ceil)
      const int64_t units = pairs_m * s;
      const int64_t rounds = (units + cl - 1) / cl;
      const double per = (double)nt / s;
      const double cost = kC0Us + (double)rounds * (per * nk * kb + 1.0);  // + list warm-up and flush per unit
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        best = PlanTopk{bn, s};
      }
    }
  }
  return best;
}

template <class Epi>
int launch_gemm_topk(const Split& A, int M, const Split& W, int N, int K, const Epi& epi, const GemmWs* ws,
                     cudaStream_t st, int* n_stripes_out, int min_tiles) {
  const PlanTopk p = plan_gemm_topk(M, N, K, min_tiles);
  Sched sc{0, 1, (K + BK - 1) / BK, nullptr, nullptr, ws && ws->kt ? ws->kt + 8 : nullptr};
  sc.n_stripes = std::min(p.n_stripes, (N + p.bn - 1) / p.bn);
  *n_stripes_out = sc.n_stripes;
  const OutDesc o{nullptr, 0, Split{}, 0, 0};
  switch (p.bn) {
    case 128: return launch_gemm<128>(A, M, W, N, K, o, epi, st, sc);
    case 192: return launch_gemm<192>(A, M, W, N, K, o, epi, st, sc);
    default: return launch_gemm<256>(A, M, W, N, K, o, epi, st, sc);
  }
}

template <class Epi>
int launch_gemm_auto(const Split& A, int M, const Split& W, int N, int K, const OutDesc& o, const Epi& epi,
                     const GemmWs* ws, cudaStream_t st) {
  static const bool no_split = [] {
    const char* e = getenv("KGQ_NO_SPLITK");
    return e && e[0] && e[0] != '0';
  }();
  const Plan p = plan_gemm(M, N, K, !no_split && ws != nullptr && ws->ws != nullptr, Epi::PLANES == 3);
  // launch-span accounting (kgq_ktime_enable): the scorer (the only epilogue with block minima)
  // in slot 1, every dense layer in slot 0
  const Sched sc{p.full, p.s_tail, p.kper, ws ? ws->ws : nullptr, ws ? ws->cnt : nullptr,
                 ws && ws->kt ? ws->kt + 8 * (Epi::CMIN ? 1 : 0) : nullptr};
  switch (p.bn) {
    case 64: return launch_gemm<64>(A, M, W, N, K, o, epi, st, sc);
    case 128: return launch_gemm<128>(A, M, W, N, K, o, epi, st, sc);
    case 160:
      if constexpr (Epi::PLANES == 3) return launch_gemm<160>(A, M, W, N, K, o, epi, st, sc);
      return -1;  // not planned for fp32 outputs
    case 192: return launch_gemm<192>(A, M, W, N, K, o, epi, st, sc);
    default: return launch_gemm<256>(A, M, W, N, K, o, epi, st, sc);
  }
}

}  // namespace tc
}  // namespace kgq
