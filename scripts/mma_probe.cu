// Microbenchmark: cycles per tcgen05.mma (cta_group::1, M = 128) issued back to back by one
// thread, operands from shared memory (SS) or A from TMEM (TS), kind::tf32 vs kind::f16, for
// several N.  One CTA per SM, all SMs busy.  Not part of the library.
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int KIND, int N, bool TS>  // KIND 0 = tf32, 1 = f16 (bf16)
__global__ void __launch_bounds__(128, 1) probe(int reps, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t fmt = KIND == 0 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint64_t da = desc_sw128(smem_u32(smem));
    const uint64_t db = desc_sw128(smem_u32(smem + 128 * 128));
    const uint32_t d = tmem;             // accumulator columns [0, N)
    const uint32_t ta = tmem + 256;      // A operand in TMEM (TS variant), columns [256, 264)
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (TS) {
        if (KIND == 0)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;}"
                       ::"r"(d), "r"(ta), "l"(db), "r"(r), "r"(idesc));
        else
          asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, p;}"
                       ::"r"(d), "r"(ta), "l"(db), "r"(r), "r"(idesc));
      } else {
        if (KIND == 0)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;}"
                       ::"r"(d), "l"(da), "l"(db), "r"(r), "r"(idesc));
        else
          asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;}"
                       ::"r"(d), "l"(da), "l"(db), "r"(r), "r"(idesc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND, int N, bool TS>
void run(unsigned long long* dc) {
  const int reps = 4096;
  const int smem = (128 + 256) * 128 + 2048;
  cudaFuncSetAttribute(probe<KIND, N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<KIND, N, TS><<<148, 128, smem>>>(reps, dc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[148];
  cudaMemcpy(c, dc, sizeof c, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  const double cyc = avg / reps;
  const double kmac = 128.0 * N * (KIND == 0 ? 8 : 16);
  printf("%s %-4s N=%3d  %7.1f cycles/MMA  %7.0f MAC/clk/SM  (floor 128*N/256 = %4d cyc)  %s\n",
         KIND == 0 ? "tf32" : "f16 ", TS ? "TS" : "SS", N, cyc, kmac / cyc, 128 * N / 256, cudaGetErrorString(e));
}


// GEMM-like pattern: STAGES stage buffers of (A_hi, A_lo, W_hi, W_lo) tiles (BN = N rows of W),
// 4 K-steps of 3 MMAs per stage, descriptors advanced by 32 B per K-step, commit per stage.
template <int N, int MODE>  // MODE 0: MMAs only; 1: + commit per stage; 2: + 2 accum buffers drained by 4 warps
__global__ void __launch_bounds__(192, 1) gemm_pattern(int nk, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int ST = 3, A_B = 128 * 128, W_B = N * 128, STAGE = 2 * A_B + 2 * W_B;
  __shared__ uint64_t bar[ST + 4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < ST * STAGE / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST + 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(i >= ST + 2 ? 4 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    long long t0 = clock64();
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % ST;
      const int g = kb / 2, a = g & 1;
      if (MODE == 2 && (kb % 2) == 0 && g >= 2)
        asm volatile("{.reg .pred p; W1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W1;}" ::"r"(smem_u32(&bar[ST + 2 + a])), "r"(((g >> 1) - 1) & 1));
      const uint32_t st = smem_u32(smem + s * STAGE);
      const uint32_t ah = st, al = st + A_B, wh = st + 2 * A_B, wl = wh + W_B;
      const uint32_t d = tmem + (MODE == 2 ? a * 256 : 0);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t off = kk * 32;
        asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;}" ::"r"(d), "l"(desc_sw128(ah + off)), "l"(desc_sw128(wl + off)), "r"(kb | kk), "r"(idesc));
        asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;}" ::"r"(d), "l"(desc_sw128(al + off)), "l"(desc_sw128(wh + off)), "r"(1), "r"(idesc));
        asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;}" ::"r"(d), "l"(desc_sw128(ah + off)), "l"(desc_sw128(wh + off)), "r"(1), "r"(idesc));
      }
      if (MODE >= 1) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[s])));
      if (MODE == 2 && (kb % 2 == 1 || kb == nk - 1)) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[ST + a])));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[ST + 1 + (MODE == 2 ? 10 : 0) * 0])));
    long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  } else if (MODE == 2 && warp >= 2) {
    const int q = warp & 3;
    const int ng = (nk + 1) / 2;
    float acc = 0.f;
    for (int g = 0; g < ng; ++g) {
      const int a = g & 1;
      asm volatile("{.reg .pred p; W2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W2;}" ::"r"(smem_u32(&bar[ST + a])), "r"((g >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int c = 0; c < N; c += 32) {
        uint32_t r[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31])
          : "r"(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * 256 + c)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[ST + 2 + a])));
    }
    if (acc == 123.f) cycles[1000] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int MODE>
void run_pattern(unsigned long long* dc) {
  const int nk = 50;
  const int smem = 3 * (2 * 128 * 128 + 2 * N * 128) + 2048;
  cudaFuncSetAttribute(gemm_pattern<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  gemm_pattern<N, MODE><<<148, 192, smem>>>(nk, dc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[148];
  cudaMemcpy(c, dc, sizeof c, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  printf("pattern N=%3d mode=%d: %8.1f cycles per K-block of 12 MMAs (floor %d)  %s\n", N, MODE, avg / nk, 12 * 128 * N / 256, cudaGetErrorString(e));
}

int main() {
  unsigned long long* dc;
  cudaMalloc(&dc, 1024 * 8 * sizeof(unsigned long long));
  run<0, 64, false>(dc); run<0, 128, false>(dc); run<0, 256, false>(dc);
  run<1, 64, false>(dc); run<1, 128, false>(dc); run<1, 256, false>(dc);
  run<0, 64, true>(dc); run<0, 128, true>(dc); run<0, 256, true>(dc);
  run<1, 256, true>(dc);
  run_pattern<64, 0>(dc); run_pattern<64, 1>(dc); run_pattern<64, 2>(dc);
  run_pattern<128, 0>(dc); run_pattern<128, 1>(dc); run_pattern<128, 2>(dc);
  run_pattern<256, 0>(dc); run_pattern<256, 1>(dc);
  return 0;
}
