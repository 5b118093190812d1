// tcgen05 3xTF32 GEMM core shared by the dense layers (linear_tc.cu) and the tensor-core
// BetaE scorer (score_tc.cu).  See linear_tc.cu for the design notes.
#pragma once
#include <cuda.h>
#include <stdio.h>

#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "common.cuh"
#include "kgq_internal.cuh"

namespace kgq {
namespace tc {
constexpr int BM = 128, BK = 32, EPI_WARPS = 8, THREADS = 64 + 32 * EPI_WARPS;  // TMA, MMA, 8 x epilogue

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
// Wait for a phase that is typically far away (the epilogue warps wait for a whole K-group of
// MMAs): test, then sleep between polls so that eight idle warps do not compete with the
// single-thread MMA issuer and the TMA producer for issue slots and shared-memory bandwidth.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) break;
#ifndef KGQ_TC_NO_SLEEP
    __nanosleep(256);
#endif
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
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
// K-major operand tile, 128-byte swizzle: rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;              // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
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

template <int BN>
struct Smem {
  static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static constexpr int A_BYTES = BM * BK * 4;  // 16 KB
  static constexpr int W_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * W_BYTES;
  static constexpr int FIT = (227 * 1024 - 2048) / STAGE_BYTES;  // stages that fit in 227 KB
  static constexpr int STAGES = FIT > 4 ? 4 : FIT;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;  // + barriers + alignment slack
  static_assert(TOTAL <= 227 * 1024, "shared memory budget");
  static_assert(EPI_WARPS * 32 * (BN / 2 + 1) * 4 <= STAGES * STAGE_BYTES, "epilogue staging fits");
};

// K-blocks per tensor-core partial sum.  The TMEM accumulate path truncates (measured: bias
// ~ 0.5 ulp per MMA accumulate, rms rel. error 1.8e-5 at K = 1600 with one chain), so each
// partial covers DRAIN*BK of K (DRAIN*3*BK/8 accumulates) and the epilogue warps add the
// partials in fp32 round-to-nearest registers, as a sequential FFMA loop would.
#ifndef KGQ_TC_DRAIN
#define KGQ_TC_DRAIN 2
#endif
constexpr int DRAIN = KGQ_TC_DRAIN;

// Generic 3xTF32 GEMM acc[m, n] = sum_k A[m, k] W[n, k] over a 128 x BN tile; the epilogue
// policy Epi receives each epilogue thread's row and its BN fp32 sums (all 128 rows of the
// tile, including rows >= M, so that policies may shuffle between lanes).  Each epilogue warp
// owns 32 rows (its TMEM lane quarter) and BN/2 columns: Epi::apply(row0, lane, n0, acc, stage)
// gets that warp's first row, the thread's lane (row row0 + lane), its BN/2 sums and a
// 32 x (BN/2 + 1) fp32 shared-memory staging tile for coalesced row stores.
template <int BN, class Epi>
__global__ void __launch_bounds__(THREADS, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
              const __grid_constant__ CUtensorMap mWh, const __grid_constant__ CUtensorMap mWl,
              int M, int N, int K, const Epi epi) {
  using L = Smem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
  constexpr int STAGES = L::STAGES;
  uint64_t* empty = full + STAGES;
  uint64_t* accfull = empty + STAGES;   // [2] partial sum ready in TMEM buffer a
  uint64_t* accempty = accfull + 2;     // [2] partial drained by the epilogue warps
  uint32_t* tmem_slot = (uint32_t*)(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;  // M fastest: W tiles shared in time
  const int nk = (K + BK - 1) / BK;
  const int ng = (nk + DRAIN - 1) / DRAIN;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mAh);
    tma_prefetch(&mAl);
    tma_prefetch(&mWh);
    tma_prefetch(&mWl);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&accfull[a], 1);
      mbar_init(&accempty[a], EPI_WARPS);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // two TMEM partial accumulators: 128 lanes x 2*BN fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        uint8_t* st = smem + s * L::STAGE_BYTES;
#ifdef KGQ_TC_DBG_NO_TMA  // perf probe only (scripts/tc_perf.cu): skip the loads
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        (void)st;
#else
        mbar_expect_tx(&full[s], L::STAGE_BYTES);
        tma_load_2d(st, &mAh, &full[s], kb * BK, m0);
        tma_load_2d(st + L::A_BYTES, &mAl, &full[s], kb * BK, m0);
        tma_load_2d(st + 2 * L::A_BYTES, &mWh, &full[s], kb * BK, n0);
        tma_load_2d(st + 2 * L::A_BYTES + L::W_BYTES, &mWl, &full[s], kb * BK, n0);
#endif
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      // instruction descriptor: D f32, A/B tf32, both K-major, N = BN, M = 128
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const int g = kb / DRAIN, a = g & 1;
        const bool first = (kb % DRAIN) == 0;
        if (first && g >= 2) mbar_wait(&accempty[a], ((g >> 1) - 1) & 1);
        mbar_wait(&full[s], (kb / STAGES) & 1);
        fence_after();
        const uint32_t d = tmem + (uint32_t)(a * BN);
        const uint32_t st = smem_u32(smem + s * L::STAGE_BYTES);
        const uint32_t ah = st, al = st + L::A_BYTES;
        const uint32_t wh = st + 2 * L::A_BYTES, wl = wh + L::W_BYTES;
#ifndef KGQ_TC_DBG_NO_MMA  // perf probe only (scripts/tc_perf.cu): skip the MMAs
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {  // 8 tf32 = 32 bytes per MMA along K
          const uint32_t off = kk * 32;
          mma_tf32(d, umma_desc_sw128(ah + off), umma_desc_sw128(wl + off), idesc,
                   (first && kk == 0) ? 0u : 1u);
          mma_tf32(d, umma_desc_sw128(al + off), umma_desc_sw128(wh + off), idesc, 1u);
          mma_tf32(d, umma_desc_sw128(ah + off), umma_desc_sw128(wh + off), idesc, 1u);
        }
#else
        (void)d; (void)ah; (void)al; (void)wh; (void)wl; (void)idesc; (void)first;
#endif
        mma_commit(&empty[s]);  // frees the smem stage once these MMAs have read it
        if ((kb % DRAIN) == DRAIN - 1 || kb == nk - 1) mma_commit(&accfull[a]);
      }
    }
  } else {
    // -------- epilogue warps 2..9: TMEM lane quarter = warp % 4, column half = (warp - 2) / 4 --------
    constexpr int CW = BN / 2;
    const int q = warp & 3;
    const int ch = ((warp - 2) >> 2) * CW;
    const int row = m0 + q * 32 + lane;
    float acc[CW];
#pragma unroll
    for (int i = 0; i < CW; ++i) acc[i] = 0.0f;
    for (int g = 0; g < ng; ++g) {
      const int a = g & 1;
      mbar_wait(&accfull[a], (g >> 1) & 1);
      fence_after();
      const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * BN + ch);
#pragma unroll
      for (int c = 0; c + 32 <= CW; c += 32) {
        float v[32];
        tmem_ld32(tq + c, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[c + i] += v[i];
      }
      if constexpr (CW % 32 == 16) {
        float v[16];
        tmem_ld16(tq + CW - 16, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[CW - 16 + i] += v[i];
      }
      fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&accempty[a])) : "memory");
    }
    // every MMA has completed (last accfull), so the pipeline buffers are free: each epilogue
    // warp stages its 32 x CW tile there and writes rows coalesced (Epi::apply)
    float* stage = reinterpret_cast<float*>(smem) + (warp - 2) * 32 * (CW + 1);
    epi.apply(m0 + q * 32, lane, n0 + ch, acc, stage);
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(L::TMEM_COLS));
  }
}

// ================================================================================================
// 2-CTA variant (cta_group::2): a cluster of two CTAs on one TPC computes a 256 x BN tile.  Each
// CTA stages its own 128 rows of A and half (BN/2 rows) of the W tile; the leader CTA (rank 0)
// issues tcgen05.mma.cta_group::2 (M 256), which reads A and B from both CTAs' shared memory and
// writes each CTA's 128 accumulator rows into that CTA's TMEM.  Per CTA the operand stream is
// (128 + BN/2) x 256 B per K-block instead of (128 + BN) x 256 B for the same 128 x BN outputs.
// TMA completions of both CTAs count on the leader's full barrier; MMA commits multicast to the
// empty / accfull barriers of both CTAs; both CTAs' epilogue warps release the leader's accempty.
// ================================================================================================
template <int BN>
struct Smem2 {
  static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int W_BYTES = (BN / 2) * BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * W_BYTES;
  static constexpr int FIT = (227 * 1024 - 2048) / STAGE_BYTES;
  static constexpr int STAGES = FIT > 4 ? 4 : FIT;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
  static_assert(TOTAL <= 227 * 1024, "shared memory budget");
  static_assert(EPI_WARPS * 32 * (BN / 2 + 1) * 4 <= STAGES * STAGE_BYTES, "epilogue staging fits");
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "N of a 2-CTA MMA: multiple of 16 per CTA");
};

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
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_2sm(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar) {  // arrive on bar in both CTAs
  const uint16_t mask = 3;
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

template <int BN, class Epi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_tc_gemm2(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
               const __grid_constant__ CUtensorMap mWh, const __grid_constant__ CUtensorMap mWl,
               int M, int N, int K, const Epi epi) {
  using L = Smem2<BN>;
  constexpr int STAGES = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* accfull = empty + STAGES;
  uint64_t* accempty = accfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int nk = (K + BK - 1) / BK;
  const int ng = (nk + DRAIN - 1) / DRAIN;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mAh);
    tma_prefetch(&mAl);
    tma_prefetch(&mWh);
    tma_prefetch(&mWl);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&accfull[a], 1);
      mbar_init(&accempty[a], 2 * EPI_WARPS);  // epilogue warps of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  cluster_sync_all();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs; completions counted by the leader) ----------------
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        uint8_t* st = smem + s * L::STAGE_BYTES;
        if (leader) mbar_expect_tx(&full[s], 2 * L::STAGE_BYTES);
        const uint32_t lb = mapa_shared(smem_u32(&full[s]), 0);
        tma_load_2d_2sm(st, &mAh, lb, kb * BK, m0);
        tma_load_2d_2sm(st + L::A_BYTES, &mAl, lb, kb * BK, m0);
        tma_load_2d_2sm(st + 2 * L::A_BYTES, &mWh, lb, kb * BK, n0 + (int)rank * (BN / 2));
        tma_load_2d_2sm(st + 2 * L::A_BYTES + L::W_BYTES, &mWl, lb, kb * BK, n0 + (int)rank * (BN / 2));
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader only): M = 256 over the pair, N = BN ----------------
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)((2 * BM) >> 4) << 24);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const int g = kb / DRAIN, a = g & 1;
        const bool first = (kb % DRAIN) == 0;
        if (first && g >= 2) mbar_wait(&accempty[a], ((g >> 1) - 1) & 1);
        mbar_wait(&full[s], (kb / STAGES) & 1);
        fence_after();
        const uint32_t d = tmem + (uint32_t)(a * BN);
        const uint32_t st = smem_u32(smem + s * L::STAGE_BYTES);
        const uint32_t ah = st, al = st + L::A_BYTES;
        const uint32_t wh = st + 2 * L::A_BYTES, wl = wh + L::W_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint32_t off = kk * 32;
          mma_tf32_2sm(d, umma_desc_sw128(ah + off), umma_desc_sw128(wl + off), idesc,
                       (first && kk == 0) ? 0u : 1u);
          mma_tf32_2sm(d, umma_desc_sw128(al + off), umma_desc_sw128(wh + off), idesc, 1u);
          mma_tf32_2sm(d, umma_desc_sw128(ah + off), umma_desc_sw128(wh + off), idesc, 1u);
        }
        mma_commit_2sm(&empty[s]);
        if ((kb % DRAIN) == DRAIN - 1 || kb == nk - 1) mma_commit_2sm(&accfull[a]);
      }
    }
  } else {
    // -------- epilogue warps 2..9: own 128 TMEM rows, lane quarter = warp % 4, column half --------
    constexpr int CW = BN / 2;
    const int q = warp & 3;
    const int ch = ((warp - 2) >> 2) * CW;
    float acc[CW];
#pragma unroll
    for (int i = 0; i < CW; ++i) acc[i] = 0.0f;
    for (int g = 0; g < ng; ++g) {
      const int a = g & 1;
      mbar_wait(&accfull[a], (g >> 1) & 1);
      fence_after();
      const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * BN + ch);
#pragma unroll
      for (int c = 0; c + 32 <= CW; c += 32) {
        float v[32];
        tmem_ld32(tq + c, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[c + i] += v[i];
      }
      if constexpr (CW % 32 == 16) {
        float v[16];
        tmem_ld16(tq + CW - 16, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[CW - 16 + i] += v[i];
      }
      fence_before();
      __syncwarp();
      if (lane == 0) {
        const uint32_t lb = mapa_shared(smem_u32(&accempty[a]), 0);
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(lb) : "memory");
      }
    }
    float* stage = reinterpret_cast<float*>(smem) + (warp - 2) * 32 * (CW + 1);
    epi.apply(m0 + q * 32, lane, n0 + ch, acc, stage);
  }
  fence_before();
  cluster_sync_all();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(L::TMEM_COLS));
  }
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

// rows x cols fp32 matrix with row stride ld (elements); box = box_rows x BK, 128B swizzle
inline bool make_map(CUtensorMap* m, const float* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  static std::mutex mu;
  static std::map<std::tuple<const float*, int64_t, int64_t, int64_t, int>, CUtensorMap> cache;
  const auto key = std::make_tuple(ptr, rows, cols, ld, box_rows);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *m = it->second;
    return true;
  }
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * sizeof(float))};
  cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "libkgq: cuTensorMapEncodeTiled(rows %lld, cols %lld, ld %lld, box %d) = %d\n", (long long)rows,
            (long long)cols, (long long)ld, box_rows, (int)r);
    return false;
  }
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *m);
  return true;
}


// Column-tile width: the mainloop is bound by the L2 -> SMEM operand stream, (128 + BN) x 256 B
// per K-block for a 128 x BN tile, so a tile costs ~ (128 + BN) and a launch ~ waves x that.
constexpr int kTileBN[7] = {32, 64, 96, 128, 160, 192, 256};
inline int choose_bn(int64_t M, int64_t N) {
  const int64_t mt = (M + BM - 1) / BM;
  int best = 0;
  int64_t best_cost = INT64_MAX;
  for (int i = 0; i < 7; ++i) {
    const int64_t tiles = mt * ((N + kTileBN[i] - 1) / kTileBN[i]);
    const int64_t cost = ((tiles + 147) / 148) * (128 + kTileBN[i]);
    if (cost < best_cost) {
      best_cost = cost;
      best = i;
    }
  }
  return kTileBN[best];
}

// Calls f(std::integral_constant<int, BN>{}) for the chosen tile width.
template <class F>
int dispatch_bn(int bn, F&& f) {
  switch (bn) {
    case 32: return f(std::integral_constant<int, 32>{});
    case 64: return f(std::integral_constant<int, 64>{});
    case 96: return f(std::integral_constant<int, 96>{});
    case 128: return f(std::integral_constant<int, 128>{});
    case 160: return f(std::integral_constant<int, 160>{});
    case 192: return f(std::integral_constant<int, 192>{});
    default: return f(std::integral_constant<int, 256>{});
  }
}

template <int BN, class Epi>
int launch_tc_gemm(const Split& A, int M, const float* Wh, const float* Wl, int N, int64_t ldw, int K,
                   const Epi& epi, cudaStream_t st) {
  CUtensorMap mAh, mAl, mWh, mWl;
  if (!make_map(&mAh, A.hi, M, K, A.ld, BM) || !make_map(&mAl, A.lo, M, K, A.ld, BM) ||
      !make_map(&mWh, Wh, N, K, ldw, BN) || !make_map(&mWl, Wl, N, K, ldw, BN)) {
    fprintf(stderr, "libkgq: cuTensorMapEncodeTiled failed\n");
    return -1;
  }
  auto kern = k_tc_gemm<BN, Epi>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<BN>::TOTAL);
    attr = true;
  }
  dim3 grid((M + BM - 1) / BM, (N + BN - 1) / BN);
  kern<<<grid, THREADS, Smem<BN>::TOTAL, st>>>(mAh, mAl, mWh, mWl, M, N, K, epi);
  return 1;
}

template <int BN, class Epi>
int launch_tc_gemm2(const Split& A, int M, const float* Wh, const float* Wl, int N, int64_t ldw, int K,
                    const Epi& epi, cudaStream_t st) {
  CUtensorMap mAh, mAl, mWh, mWl;
  if (!make_map(&mAh, A.hi, M, K, A.ld, BM) || !make_map(&mAl, A.lo, M, K, A.ld, BM) ||
      !make_map(&mWh, Wh, N, K, ldw, BN / 2) || !make_map(&mWl, Wl, N, K, ldw, BN / 2)) {
    fprintf(stderr, "libkgq: cuTensorMapEncodeTiled failed\n");
    return -1;
  }
  auto kern = k_tc_gemm2<BN, Epi>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem2<BN>::TOTAL);
    attr = true;
  }
  dim3 grid(2 * ((M + 2 * BM - 1) / (2 * BM)), (N + BN - 1) / BN);
  kern<<<grid, THREADS, Smem2<BN>::TOTAL, st>>>(mAh, mAl, mWh, mWl, M, N, K, epi);
  return 1;
}

// Tile choice for both variants: a CTA's mainloop costs ~ its operand stream per K-block,
// (128 + BN) for one CTA, (128 + BN/2) per CTA of a pair; a launch costs waves x that (74 CTA
// pairs per wave on 148 SMs).  Returns BN, with *pair set for the 2-CTA kernel.
constexpr int kPairBN[5] = {64, 128, 192, 224, 256};
inline int choose_tile(int64_t M, int64_t N, bool* pair) {
  const int64_t mt = (M + BM - 1) / BM;
  int best = 0;
  int64_t best_cost = INT64_MAX;
  bool best_pair = false;
  for (int i = 0; i < 7; ++i) {
    const int64_t ctas = mt * ((N + kTileBN[i] - 1) / kTileBN[i]);
    const int64_t cost = ((ctas + 147) / 148) * (128 + kTileBN[i]);
    if (cost < best_cost) { best_cost = cost; best = kTileBN[i]; best_pair = false; }
  }
  const int64_t pairs_m = (M + 2 * BM - 1) / (2 * BM);
  for (int i = 0; i < 5; ++i) {
    const int64_t pairs = pairs_m * ((N + kPairBN[i] - 1) / kPairBN[i]);
    const int64_t cost = ((pairs + 73) / 74) * (128 + kPairBN[i] / 2);
    if (cost < best_cost) { best_cost = cost; best = kPairBN[i]; best_pair = true; }
  }
  *pair = best_pair;
  return best;
}

// Launch the chosen variant; make(std::integral_constant<int, CW>) returns the epilogue policy
// for CW = columns per epilogue warp (= BN / 2 in both variants).
template <class Make>
int launch_gemm_auto(const Split& A, int M, const float* Wh, const float* Wl, int N, int64_t ldw, int K,
                     Make&& make, cudaStream_t st) {
  bool pair = false;
  const int bn = choose_tile(M, N, &pair);
  if (pair) {
    switch (bn) {
      case 64: return launch_tc_gemm2<64>(A, M, Wh, Wl, N, ldw, K, make(std::integral_constant<int, 32>{}), st);
      case 128: return launch_tc_gemm2<128>(A, M, Wh, Wl, N, ldw, K, make(std::integral_constant<int, 64>{}), st);
      case 192: return launch_tc_gemm2<192>(A, M, Wh, Wl, N, ldw, K, make(std::integral_constant<int, 96>{}), st);
      case 224: return launch_tc_gemm2<224>(A, M, Wh, Wl, N, ldw, K, make(std::integral_constant<int, 112>{}), st);
      default: return launch_tc_gemm2<256>(A, M, Wh, Wl, N, ldw, K, make(std::integral_constant<int, 128>{}), st);
    }
  }
  return dispatch_bn(bn, [&](auto c) {
    constexpr int B = decltype(c)::value;
    return launch_tc_gemm<B>(A, M, Wh, Wl, N, ldw, K, make(std::integral_constant<int, B / 2>{}), st);
  });
}

}  // namespace tc
}  // namespace kgq
