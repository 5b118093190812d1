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
  for (Shape sh : {Shape{1024, 1600, 1200}, Shape{2048, 1600, 1600}, Shape{1024, 800, 1600}, Shape{3072, 1600, 1600}}) {
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
    auto run = [&](int bn) {
      switch (bn) {
        case 64: launch_bn<64>(Split{xh, xl, K}, M, K, L, kEpiRelu, out, 0, 0, 0); break;
        case 128: launch_bn<128>(Split{xh, xl, K}, M, K, L, kEpiRelu, out, 0, 0, 0); break;
        case 256: launch_bn<256>(Split{xh, xl, K}, M, K, L, kEpiRelu, out, 0, 0, 0); break;
        default: launch_linear(Split{xh, xl, K}, M, K, L, kEpiRelu, out, 0, 0, 0);
      }
    };
    for (int bn : {0, 64, 128, 256}) {
      for (int i = 0; i < 3; ++i) run(bn);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      const int reps = 20;
      for (int i = 0; i < reps; ++i) run(bn);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double t = ms / reps;
      const int64_t ctas = (int64_t)((M + 127) / 128) * ((N + (bn ? bn : 96) - 1) / (bn ? bn : 96));
      printf("M=%5d N=%5d K=%5d BN=%3d (%4lld CTAs) %8.1f us  %7.1f TFLOP/s (useful fp32)  err=%s\n", M, N, K, bn,
             (long long)ctas, t * 1e3, 2.0 * M * N * K / (t * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(x); cudaFree(xh); cudaFree(xl); cudaFree(w); cudaFree(wh); cudaFree(wl); cudaFree(b); cudaFree(y);
  }
  return 0;
}
