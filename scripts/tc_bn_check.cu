// Correctness probe: every tile width of the persistent tcgen05 GEMM core, each epilogue form
// (fp32 plane, split hi/lo planes, DNF row-pair min), ragged M / N / K, and a grid smaller
// than the tile count (persistence), vs an fp64 host reference.  Not part of the library.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2503_02172_b200/csrc/chain.cu"
#include "../paper_2503_02172_b200/csrc/linear_tc.cu"
#include "../paper_2503_02172_b200/csrc/score_tc.cu"

using namespace kgq;

int main(int argc, char** argv) {
  const int M = 300, N = 520, K = argc > 1 ? atoi(argv[1]) : 100;
  std::mt19937 g(1);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> x((size_t)M * K), w((size_t)N * K), b(N);
  for (auto& v : x) v = U(g);
  for (auto& v : w) v = U(g);
  for (auto& v : b) v = U(g);
  std::vector<double> ref((size_t)M * N), mag((size_t)M * N);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0, sa = 0;
      for (int k = 0; k < K; ++k) {
        s += (double)x[(size_t)m * K + k] * w[(size_t)n * K + k];
        sa += fabs((double)x[(size_t)m * K + k] * w[(size_t)n * K + k]);
      }
      ref[(size_t)m * N + n] = s;
      mag[(size_t)m * N + n] = sa + fabs(b[n]);
    }
  float *dx, *dw, *db, *dy;
  float2 *dP, *dE;
  cudaMalloc(&dx, x.size() * 4); cudaMalloc(&dw, w.size() * 4);
  cudaMalloc(&db, N * 4); cudaMalloc(&dy, (size_t)M * N * 4 * 2);
  cudaMalloc(&dP, M * 8); cudaMalloc(&dE, 640 * 8);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), N * 4, cudaMemcpyHostToDevice);
  cudaMemset(dP, 0, M * 8); cudaMemset(dE, 0, 640 * 8);
  auto mk = [](int64_t rows, int64_t cols) {
    Split s;
    s.ld = (cols + 7) / 8 * 8;
    cudaMalloc(&s.b0, 3 * rows * s.ld * 2);
    s.b1 = s.b0 + rows * s.ld;
    s.b2 = s.b1 + rows * s.ld;
    return s;
  };
  Split A = mk(M, K), Wsp = mk(N, K), Ysp = mk(M, N);
  launch_split_copy_rows(dx, M, K, A, 0, 0, true);
  launch_split_copy_rows(dw, N, K, Wsp, 0);
  GemmWs gws;
  cudaMalloc(&gws.ws, kGemmWsFloats * 4);
  cudaMalloc(&gws.cnt, kGemmCntInts * 4);
  cudaMemset(gws.cnt, 0, kGemmCntInts * 4);
  const tc::Sched whole{0, 1, 0, nullptr, nullptr};
  int fails = 0;
  // form 0: fp32 + bias (no activation); 1: split (bf16x3) + bias + ReLU; 2: row-pair min (DNF union)
  std::vector<uint16_t> hb(3 * (size_t)M * Ysp.ld);
  auto bf = [](uint16_t u) { uint32_t v = (uint32_t)u << 16; float f; memcpy(&f, &v, 4); return f; };
  auto check = [&](const char* what, int bn, int form, auto launch) {
    cudaMemset(dy, 0xff, (size_t)M * N * 4 * 2);  // NaN fill: every output must be written
    cudaMemset(Ysp.b0, 0xff, hb.size() * 2);
    launch();
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> y((size_t)M * N * 2);
    cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hb.data(), Ysp.b0, hb.size() * 2, cudaMemcpyDeviceToHost);
    double mx = 0;
    int bad = 0;
    const int rows = form == 2 ? M / 2 : M;
    const size_t pl = (size_t)M * Ysp.ld;
    for (int m = 0; m < rows; ++m)
      for (int n = 0; n < N; ++n) {
        double want, scale;
        float got;
        if (form == 2) {
          want = fmin(ref[(size_t)(2 * m) * N + n], ref[(size_t)(2 * m + 1) * N + n]);
          scale = fmax(mag[(size_t)(2 * m) * N + n], mag[(size_t)(2 * m + 1) * N + n]);
          got = y[(size_t)m * N + n];
        } else {
          want = ref[(size_t)m * N + n] + b[n];
          if (form == 1) want = fmax(want, 0.0);
          scale = mag[(size_t)m * N + n];
          if (form == 1) {  // the activation split: three bf16 planes (exact sum) or fp16 hi + 2^11-scaled lo
            const size_t o = (size_t)m * Ysp.ld + n;
            if (kgq::kFp16x2) {
              auto hf = [](uint16_t u) {  // fp16 bits -> float
                const uint32_t sgn = (u & 0x8000u) << 16, ex = (u >> 10) & 0x1F, man = u & 0x3FF;
                if (ex == 0) return (sgn ? -1.0f : 1.0f) * ldexpf((float)man, -24);
                const uint32_t v = sgn | ((ex + 112) << 23) | (man << 13);
                float f;
                memcpy(&f, &v, 4);
                return f;
              };
              got = hf(hb[o]) + hf(hb[pl + o]) * (1.0f / 2048.0f);
            } else {
              got = (bf(hb[o]) + bf(hb[pl + o])) + bf(hb[2 * pl + o]);
            }
          } else {
            got = y[(size_t)m * N + n];
          }
        }
        const double r = fabs((double)got - want) / scale;
        if (!(r <= 1e-6)) ++bad;
        if (r > mx || r != r) mx = r != r ? 1e30 : r;
      }
    fails += bad > 0 || e != cudaSuccess;
    printf("%-28s BN=%3d max err %.3e (of sum|x w|)  bad %d  %s\n", what, bn, mx, bad, cudaGetErrorString(e));
  };
  auto each_bn = [&](auto f) {
    f(std::integral_constant<int, 64>{});
    f(std::integral_constant<int, 128>{});
    f(std::integral_constant<int, 160>{});
    f(std::integral_constant<int, 192>{});
    f(std::integral_constant<int, 256>{});
  };
  each_bn([&](auto c) {
    constexpr int B = decltype(c)::value;
    const tc::OutDesc o1{dy, N, Split{}, M, N}, o2{nullptr, 0, Ysp, M, N};
    if constexpr (B % 64 == 0)
      check("fp32 + bias", B, 0, [&] { tc::launch_gemm<B>(A, M, Wsp, N, K, o1, EpiLinear<kEpiNone, false>{db, N, 0, 0}, 0, whole); });
    check("split + bias + relu", B, 1, [&] { tc::launch_gemm<B>(A, M, Wsp, N, K, o2, EpiLinear<kEpiRelu, true>{db, N, 0, 0}, 0, whole); });
    if constexpr (B % 64 == 0)
      check("fp32, 2 clusters (persist)", B, 0, [&] { tc::launch_gemm<B>(A, M, Wsp, N, K, o1, EpiLinear<kEpiNone, false>{db, N, 0, 0}, 0, whole, 2); });
    const tc::OutDesc o3{dy, N, Split{}, M / 2, N};
    if constexpr (B % 64 == 0)
      check("row-pair min (union)", B, 2, [&] { tc::launch_gemm<B>(A, M, Wsp, N, K, o3, EpiBetaScore<2>{dP, dE, M, 640}, 0, whole); });
    // split tail: the last tiles (or all) split in K; K = 100 -> 4 K-blocks
    const int tiles = ((M + 255) / 256) * ((N + B - 1) / B);
    for (int sk : {2, 4}) {
      const int nkb = (K + 31) / 32, kper = (nkb + sk - 1) / sk;
      const tc::Sched all{0, sk, kper, gws.ws, gws.cnt}, tail{tiles / 2, sk, kper, gws.ws, gws.cnt};
      char nm[64];
      snprintf(nm, sizeof nm, "split-K %d, every tile", sk);
      check(nm, B, 1, [&] { tc::launch_gemm<B>(A, M, Wsp, N, K, o2, EpiLinear<kEpiRelu, true>{db, N, 0, 0}, 0, all); });
      snprintf(nm, sizeof nm, "split-K %d, tail, 3 clusters", sk);
      if constexpr (B % 64 == 0) check(nm, B, 0, [&] { tc::launch_gemm<B>(A, M, Wsp, N, K, o1, EpiLinear<kEpiNone, false>{db, N, 0, 0}, 0, tail, 3); });
      snprintf(nm, sizeof nm, "split-K %d, union rows", sk);
      if constexpr (B % 64 == 0) check(nm, B, 2, [&] { tc::launch_gemm<B>(A, M, Wsp, N, K, o3, EpiBetaScore<2>{dP, dE, M, 640}, 0, all); });
    }
    // counters must be back to zero after every launch
    std::vector<int> cnt(kGemmCntInts);
    cudaMemcpy(cnt.data(), gws.cnt, kGemmCntInts * 4, cudaMemcpyDeviceToHost);
    int nz = 0;
    for (int v : cnt) nz += v != 0;
    if (nz) { printf("BN=%d: %d split counters not reset\n", B, nz); ++fails; }
  });
  printf(fails ? "FAILED (%d)\n" : "all tile widths and epilogues OK\n", fails);
  return fails ? 1 : 0;
}
