// Throughput probe for the tcgen05 3xTF32 GEMM core (not part of the library).  Built in
// variants with -DKGQ_TC_DBG_NO_TMA / -DKGQ_TC_DBG_NO_MMA / -DKGQ_TC_DRAIN=n to isolate the
// bound (results are garbage in the debug variants; only the timing matters).
#include <cstdio>
#include <vector>

#include "../paper_2503_02172_b200/csrc/chain.cu"
#include "../paper_2503_02172_b200/csrc/linear_tc.cu"

using namespace kgq;

int main() {
  struct Shape { int M, N, K; };
  for (Shape sh : {Shape{1024, 1600, 1200}, Shape{2048, 1600, 1600}, Shape{1024, 800, 1600}, Shape{3072, 1600, 1600}, Shape{1024, 1600, 1600}, Shape{2048, 800, 1600}, Shape{2048, 800, 800}, Shape{2048, 400, 800}, Shape{1024, 14592, 800}, Shape{2048, 14592, 800}, Shape{4096, 14976, 800}}) {
    const int M = sh.M, N = sh.N, K = sh.K;
    float *x, *xh, *xl, *w, *wh, *wl, *b, *y;
    cudaMalloc(&x, (size_t)M * K * 4); cudaMalloc(&xh, (size_t)M * K * 4); cudaMalloc(&xl, (size_t)M * K * 4);
    cudaMalloc(&w, (size_t)N * K * 4); cudaMalloc(&wh, (size_t)N * K * 4); cudaMalloc(&wl, (size_t)N * K * 4);
    cudaMalloc(&b, N * 4); cudaMalloc(&y, (size_t)M * N * 4 * 2);
    cudaMemset(x, 0, (size_t)M * K * 4); cudaMemset(w, 0, (size_t)N * K * 4); cudaMemset(b, 0, N * 4);
    launch_split_copy(x, (int64_t)M * K, xh, xl, 0);
    launch_split_copy(w, (int64_t)N * K, wh, wl, 0);
    Linear L; L.W = w; L.W_hi = wh; L.W_lo = wl; L.b = b; L.out_f = N; L.in_f = K;
    Split out{y, y + (size_t)M * N, N};
    Split A{xh, xl, K};
    auto time_it = [&](auto launch) {
      for (int i = 0; i < 3; ++i) launch();
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      const int reps = 20;
      for (int i = 0; i < reps; ++i) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      return ms / reps * 1e3;  // us
    };
    printf("M=%5d N=%5d K=%5d |", M, N, K);
    for (int bn : {32, 64, 96, 128, 160, 192, 256}) {
      const double us = tc::dispatch_bn(bn, [&](auto c) {
        constexpr int B = decltype(c)::value;
        return (int)(100 * time_it([&] { tc::launch_tc_gemm<B>(A, M, wh, wl, N, K, K, EpiLinear<B / 2, kEpiRelu, true>{b, out, M, N, 0, 0}, 0); }));
      }) / 100.0;
      printf(" 1x%d:%.1f", bn, us);
    }
    printf(" |");
    printf(" 2x64:%.1f", time_it([&] { tc::launch_tc_gemm2<64>(A, M, wh, wl, N, K, K, EpiLinear<32, kEpiRelu, true>{b, out, M, N, 0, 0}, 0); }));
    printf(" 2x128:%.1f", time_it([&] { tc::launch_tc_gemm2<128>(A, M, wh, wl, N, K, K, EpiLinear<64, kEpiRelu, true>{b, out, M, N, 0, 0}, 0); }));
    printf(" 2x192:%.1f", time_it([&] { tc::launch_tc_gemm2<192>(A, M, wh, wl, N, K, K, EpiLinear<96, kEpiRelu, true>{b, out, M, N, 0, 0}, 0); }));
    printf(" 2x224:%.1f", time_it([&] { tc::launch_tc_gemm2<224>(A, M, wh, wl, N, K, K, EpiLinear<112, kEpiRelu, true>{b, out, M, N, 0, 0}, 0); }));
    printf(" 2x256:%.1f", time_it([&] { tc::launch_tc_gemm2<256>(A, M, wh, wl, N, K, K, EpiLinear<128, kEpiRelu, true>{b, out, M, N, 0, 0}, 0); }));
    printf(" | auto:%.1f\n", time_it([&] { launch_linear(A, M, K, L, kEpiRelu, out, 0, 0, 0); }));
    cudaFree(x); cudaFree(xh); cudaFree(xl); cudaFree(w); cudaFree(wh); cudaFree(wl); cudaFree(b); cudaFree(y);
  }
  return 0;
}
