// Correctness probe: every column-tile width of the tcgen05 GEMM core must give the same
// y = x W^T (vs an fp64 host reference).  Not part of the library.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2503_02172_b200/csrc/chain.cu"
#include "../paper_2503_02172_b200/csrc/linear_tc.cu"

using namespace kgq;

int main() {
  const int M = 300, N = 520, K = 100;
  std::mt19937 g(1);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> x((size_t)M * K), w((size_t)N * K), b(N, 0.f);
  for (auto& v : x) v = U(g);
  for (auto& v : w) v = U(g);
  float *dx, *dxh, *dxl, *dw, *dwh, *dwl, *db, *dy;
  cudaMalloc(&dx, x.size() * 4); cudaMalloc(&dxh, x.size() * 4); cudaMalloc(&dxl, x.size() * 4);
  cudaMalloc(&dw, w.size() * 4); cudaMalloc(&dwh, w.size() * 4); cudaMalloc(&dwl, w.size() * 4);
  cudaMalloc(&db, N * 4); cudaMalloc(&dy, (size_t)M * N * 4);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), N * 4, cudaMemcpyHostToDevice);
  launch_split_copy(dx, x.size(), dxh, dxl, 0);
  launch_split_copy(dw, w.size(), dwh, dwl, 0);
  Linear L; L.W = dw; L.W_hi = dwh; L.W_lo = dwl; L.b = db; L.out_f = N; L.in_f = K;
  auto check = [&](const char* what, int bn, auto launch) {
    cudaMemset(dy, 0, (size_t)M * N * 4);
    launch();
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> y((size_t)M * N);
    cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost);
    double mx = 0; int bad = 0, fr = -1, fc = -1;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0, sa = 0;
        for (int k = 0; k < K; ++k) { s += (double)x[(size_t)m * K + k] * w[(size_t)n * K + k]; sa += fabs((double)x[(size_t)m * K + k] * w[(size_t)n * K + k]); }
        const double r = fabs(y[(size_t)m * N + n] - s) / sa;
        if (r > 1e-5) { if (!bad) { fr = m; fc = n; } ++bad; }
        mx = fmax(mx, r);
      }
    printf("%s BN=%3d max err %.3e  bad %d (first row %d col %d)  %s\n", what, bn, mx, bad, fr, fc, cudaGetErrorString(e));
  };
  Split A{dxh, dxl, K};
  Split out{dy, nullptr, N};
  for (int bn : {32, 64, 96, 128, 160, 192, 256})
    tc::dispatch_bn(bn, [&](auto c) {
      constexpr int B = decltype(c)::value;
      check("1-CTA", B, [&] { tc::launch_tc_gemm<B>(A, M, dwh, dwl, N, K, K, EpiLinear<B / 2, kEpiNone, false>{db, out, M, N, 0, 0}, 0); });
      return 0;
    });
  check("2-CTA", 64, [&] { tc::launch_tc_gemm2<64>(A, M, dwh, dwl, N, K, K, EpiLinear<32, kEpiNone, false>{db, out, M, N, 0, 0}, 0); });
  check("2-CTA", 128, [&] { tc::launch_tc_gemm2<128>(A, M, dwh, dwl, N, K, K, EpiLinear<64, kEpiNone, false>{db, out, M, N, 0, 0}, 0); });
  check("2-CTA", 192, [&] { tc::launch_tc_gemm2<192>(A, M, dwh, dwl, N, K, K, EpiLinear<96, kEpiNone, false>{db, out, M, N, 0, 0}, 0); });
  check("2-CTA", 224, [&] { tc::launch_tc_gemm2<224>(A, M, dwh, dwl, N, K, K, EpiLinear<112, kEpiNone, false>{db, out, M, N, 0, 0}, 0); });
  check("2-CTA", 256, [&] { tc::launch_tc_gemm2<256>(A, M, dwh, dwl, N, K, K, EpiLinear<128, kEpiNone, false>{db, out, M, N, 0, 0}, 0); });
  check("auto ", 0, [&] { launch_linear(A, M, K, L, kEpiNone, out, 0, 0, 0); });
  return 0;
}
