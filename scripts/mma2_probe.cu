// Microbenchmark: cycles per tcgen05.mma.cta_group::2.kind::f16 (CTA pair, M = 256, K = 16,
// bf16 operands from shared memory) issued back to back by the leader's thread, for several N,
// 74 pairs (all SMs busy).  Also the same with a commit every 12 MMAs (one K-block of the
// bf16x3 GEMM).  Not part of the library.
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

template <int N, int COMMIT, int ROT = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(int reps, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 192 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
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
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (16u << 24);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      // ROT > 1: operands rotate over ROT distinct 24 KB (A) / 24 KB (B) stage buffers, like a
      // pipelined GEMM (every MMA of a K-block reads another plane pair)
      const int stg = (r / 2) % ROT;
      const uint64_t da = desc_sw64(smem_u32(smem + stg * 8192));
      const uint64_t db = desc_sw64(smem_u32(smem + 96 * 1024 + stg * 8192));
      asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %4, p;}"
                   ::"r"(tmem), "l"(da + ((r & 1) << 1)), "l"(db + ((r & 1) << 1)), "r"(r), "r"(idesc));
      if (COMMIT && (r % 12) == 11)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&bar)), "h"((uint16_t)1));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)1));
    // wait for the last commit's phase: every commit flips the barrier, so poll until no MMA is
    // pending by waiting on a fresh barrier round (count = commits + 1)
    const int phases = (COMMIT ? reps / 12 : 0) + 1;
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                 ::"r"(smem_u32(&bar)), "r"((phases - 1) & 1));
    long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int COMMIT, int ROT = 1>
void run(unsigned long long* dc) {
  const int reps = 12 * 512;
  const int smem = 192 * 1024 + 2048;
  cudaFuncSetAttribute(probe<N, COMMIT, ROT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, COMMIT, ROT><<<148, 128, smem>>>(reps, dc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[148];
  cudaMemcpy(c, dc, sizeof c, cudaMemcpyDeviceToHost);
  double avg = 0;
  int n = 0;
  for (int i = 0; i < 148; i += 2) { avg += c[i]; ++n; }
  avg /= n;
  const double cyc = avg / reps;
  const double mac = 128.0 * N * 16;  // per SM per instruction
  printf("cta_group::2 f16 N=%3d rot %2d %s %7.1f cycles/MMA  %6.0f MAC/clk/SM (per-SM 128 x N x 16)  %s\n", N,
         ROT, COMMIT ? "commit/12" : "no commit", cyc, mac / cyc, cudaGetErrorString(e));
}

int main() {
  unsigned long long* dc;
  cudaMalloc(&dc, 148 * 8);
  run<64, 0>(dc); run<128, 0>(dc); run<192, 0>(dc); run<256, 0>(dc);
  run<128, 1>(dc); run<192, 1>(dc); run<256, 1>(dc);
  run<128, 1, 12>(dc); run<192, 1, 12>(dc); run<256, 1, 12>(dc);
  return 0;
}
