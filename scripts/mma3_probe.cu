// Microbenchmark (not part of the library): cycles per bf16x3 K-block (BK = 32: 2 K16 steps x 6
// tcgen05.mma.cta_group::2.kind::f16, M = 256, N = BN) issued back to back by the leader's
// thread, operands rotating over 4 smem stages like the GEMM mainloop, a commit per K-block.
// Variants of the issue order / operand source:
//   0 GEMM order     (a0 w2)(a1 w1)(a2 w0)(a0 w1)(a1 w0)(a0 w0)   A changes every MMA
//   1 A-grouped      (a2 w0)(a1 w1)(a1 w0)(a0 w2)(a0 w1)(a0 w0)
//   2 A-grouped + collector::a hints (fill / use / lastuse: A re-read from the collector)
//   3 GEMM order with A in TMEM (tcgen05.cp per plane and K16 step, then the "ts" MMA form)
//   4 one A plane and one B plane only (6 identical MMAs: the MMA pipe alone)
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
#define MMA_SS(OPT)                                                                                   \
  __device__ __forceinline__ void mma_##OPT(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) { \
    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::f16" MMA_Q_##OPT          \
                 " [%0], %1, %2, %3, p;}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));             \
  }
#define MMA_Q_plain ""
#define MMA_Q_fill ".collector::a::fill"
#define MMA_Q_use ".collector::a::use"
#define MMA_Q_last ".collector::a::lastuse"
MMA_SS(plain)
MMA_SS(fill)
MMA_SS(use)
MMA_SS(last)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void cp_2sm(uint32_t t, uint64_t s) {
  asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(t), "l"(s) : "memory");
}

template <int BN, int VAR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(int kblocks, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  constexpr int A_B = 128 * 64, W_B = (BN / 2) * 64, STAGE = 3 * A_B + 3 * W_B, NST = 4;
  const int warp = threadIdx.x >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < NST * STAGE / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | (16u << 24);
    long long t0 = clock64();
    for (int kb = 0; kb < kblocks; ++kb) {
      const uint32_t st = smem_u32(smem + (kb % NST) * STAGE);
      const uint32_t a0 = st, a1 = st + A_B, a2 = st + 2 * A_B, w0 = st + 3 * A_B, w1 = w0 + W_B, w2 = w1 + W_B;
      const uint32_t ta = tmem + 2 * BN <= tmem + 512 - 48 ? tmem + 2 * BN : tmem + 256;
      if (VAR == 3)
        for (int p = 0; p < 3; ++p)
          for (int kk = 0; kk < 2; ++kk) cp_2sm(ta + (p * 2 + kk) * 8, desc_sw64(st + p * A_B + kk * 32));
      for (int kk = 0; kk < 2; ++kk) {
        const uint32_t o = kk * 32;
        const uint32_t acc = (kb == 0 && kk == 0) ? 0u : 1u;
        auto D = [](uint32_t x) { return desc_sw64(x); };
        if (VAR == 0) {
          mma_plain(tmem, D(a0 + o), D(w2 + o), idesc, acc);
          mma_plain(tmem, D(a1 + o), D(w1 + o), idesc, 1);
          mma_plain(tmem, D(a2 + o), D(w0 + o), idesc, 1);
          mma_plain(tmem, D(a0 + o), D(w1 + o), idesc, 1);
          mma_plain(tmem, D(a1 + o), D(w0 + o), idesc, 1);
          mma_plain(tmem, D(a0 + o), D(w0 + o), idesc, 1);
        } else if (VAR == 1) {
          mma_plain(tmem, D(a2 + o), D(w0 + o), idesc, acc);
          mma_plain(tmem, D(a1 + o), D(w1 + o), idesc, 1);
          mma_plain(tmem, D(a1 + o), D(w0 + o), idesc, 1);
          mma_plain(tmem, D(a0 + o), D(w2 + o), idesc, 1);
          mma_plain(tmem, D(a0 + o), D(w1 + o), idesc, 1);
          mma_plain(tmem, D(a0 + o), D(w0 + o), idesc, 1);
        } else if (VAR == 2) {
          mma_plain(tmem, D(a2 + o), D(w0 + o), idesc, acc);
          mma_fill(tmem, D(a1 + o), D(w1 + o), idesc, 1);
          mma_last(tmem, D(a1 + o), D(w0 + o), idesc, 1);
          mma_fill(tmem, D(a0 + o), D(w2 + o), idesc, 1);
          mma_use(tmem, D(a0 + o), D(w1 + o), idesc, 1);
          mma_last(tmem, D(a0 + o), D(w0 + o), idesc, 1);
        } else if (VAR == 3) {
          const uint32_t t0a = ta + kk * 8, t1a = t0a + 16, t2a = t1a + 16;
          mma_ts(tmem, t0a, D(w2 + o), idesc, acc);
          mma_ts(tmem, t1a, D(w1 + o), idesc, 1);
          mma_ts(tmem, t2a, D(w0 + o), idesc, 1);
          mma_ts(tmem, t0a, D(w1 + o), idesc, 1);
          mma_ts(tmem, t1a, D(w0 + o), idesc, 1);
          mma_ts(tmem, t0a, D(w0 + o), idesc, 1);
        } else {
          for (int i = 0; i < 6; ++i) mma_plain(tmem, D(a0 + o), D(w0 + o), idesc, i || kk || kb ? 1u : 0u);
        }
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(smem_u32(&bar)), "h"((uint16_t)1));
    }
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                 ::"r"(smem_u32(&bar)), "r"((kblocks - 1) & 1));
    long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int BN, int VAR>
void run(unsigned long long* dc) {
  const int kblocks = 2048;
  constexpr int STAGE = 3 * 128 * 64 + 3 * (BN / 2) * 64;
  const int smem = 4 * STAGE + 2048;
  cudaFuncSetAttribute(probe<BN, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<BN, VAR><<<148, 128, smem>>>(kblocks, dc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[148];
  cudaMemcpy(c, dc, sizeof c, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; i += 2) avg += c[i];
  avg /= 74;
  const double cyc = avg / kblocks, ideal = 12.0 * 128 * BN * 16 / 4096.0;
  const char* nm[] = {"GEMM order", "A-grouped", "A-grouped+collector", "A in TMEM", "one A/B plane"};
  printf("BN=%3d %-22s %7.1f clk per K-block (ideal %5.0f, %4.0f%%)  %s\n", BN, nm[VAR], cyc, ideal,
         100.0 * ideal / cyc, cudaGetErrorString(e));
}

int main() {
  unsigned long long* dc;
  cudaMalloc(&dc, 148 * 8);
  run<128, 0>(dc); run<128, 1>(dc); run<128, 2>(dc); run<128, 3>(dc); run<128, 4>(dc);
  run<192, 0>(dc); run<192, 1>(dc); run<192, 2>(dc); run<192, 4>(dc);
  run<256, 0>(dc); run<256, 1>(dc); run<256, 2>(dc); run<256, 4>(dc);
  return 0;
}
