// Throughput probe for the persistent tcgen05 3xTF32 GEMM core (not part of the library):
// the C2 step's shapes -- BetaE MLP layers (M = B x branches) and the tensor-core scorer
// (N = padded shard, K = 2d) -- timed per tile width and with the launch's own choice.
// With -DKGQ_TC_TRACE (scripts/tc_probe.sh) it also prints per-tile phase times.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "../paper_2503_02172_b200/csrc/chain.cu"
#include "../paper_2503_02172_b200/csrc/linear_tc.cu"
#include "../paper_2503_02172_b200/csrc/score_tc.cu"

using namespace kgq;

template <class F>
static double time_us(F&& launch) {
  for (int i = 0; i < 3; ++i) launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps * 1e3;
}

int main() {
  struct Shape { int M, N, K; bool score; };
  const Shape shapes[] = {{1024, 1600, 1200, false}, {3072, 1600, 1600, false}, {2048, 800, 1600, false},
                          {2048, 800, 800, false},   {1024, 14592, 800, true},  {2048, 14592, 800, true},
                          {1024, 14592, 32, true},   {1024, 1600, 32, false}, {2048, 400, 800, false},
                          {3072, 400, 800, false},   {1024, 800, 1600, false}, {1024, 1600, 1600, false},
                          {1024, 1600, 800, false},  {2048, 1600, 800, false},  {3072, 1600, 800, false},
                          {2048, 1600, 1600, false}, {3072, 800, 1600, false},  {3072, 800, 800, false},
                          {1024, 400, 800, false},
                          // the mixed-submit step's shapes (M = rows of all types' branches per hop)
                          {27648, 1600, 800, false}, {27648, 1600, 1600, false}, {27648, 800, 1600, false},
                          {7168, 1600, 800, false},  {7168, 1600, 1600, false},  {7168, 800, 1600, false},
                          {20480, 800, 800, false},  {20480, 400, 800, false},   {4096, 14592, 800, true}};
#ifdef KGQ_TC_TRACE
  unsigned long long* tr;
  cudaMalloc(&tr, 8192 * 64);
  cudaMemcpyToSymbol(tc::g_tc_trace, &tr, sizeof(tr));
#endif
  for (const Shape& sh : shapes) {
    const int M = sh.M, N = sh.N, K = sh.K;
    float *xf, *wf, *b, *y;
    float2 *P, *E;
    cudaMalloc(&xf, (size_t)M * K * 4); cudaMalloc(&wf, (size_t)N * K * 4);
    cudaMalloc(&b, N * 4); cudaMalloc(&y, (size_t)M * N * 4);
    cudaMalloc(&P, M * 8); cudaMalloc(&E, N * 8);
    std::vector<float> hx((size_t)M * K), hw((size_t)N * K);  // non-zero operands
    for (size_t i = 0; i < hx.size(); ++i) hx[i] = (float)((i * 2654435761u) % 1000) * 1e-3f - 0.5f;
    for (size_t i = 0; i < hw.size(); ++i) hw[i] = (float)((i * 40503u) % 1000) * 1e-3f - 0.5f;
    cudaMemcpy(xf, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(wf, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice);
    auto mk = [](int64_t rows, int64_t cols) {
      Split s;
      s.ld = (cols + 7) / 8 * 8;
      cudaMalloc(&s.b0, 3 * rows * s.ld * 2);
      s.b1 = s.b0 + rows * s.ld;
      s.b2 = s.b1 + rows * s.ld;
      return s;
    };
    Split A = mk(M, K), Wsp = mk(N, K), Ysp = mk(M, N);
    launch_split_copy_rows(xf, M, K, A, 0, 0, true);
    launch_split_copy_rows(wf, N, K, Wsp, 0);
    cudaMemset(b, 0, N * 4); cudaMemset(P, 0, M * 8); cudaMemset(E, 0, N * 8);
    static GemmWs gws;
    if (!gws.ws) {
      cudaMalloc(&gws.ws, kGemmWsFloats * 4);
      cudaMalloc(&gws.cnt, kGemmCntInts * 4);
      cudaMemset(gws.cnt, 0, kGemmCntInts * 4);
    }
    const tc::Plan plan = tc::plan_gemm(M, N, K, !getenv("KGQ_NO_SPLITK"), !sh.score);
    const tc::Sched whole{0, 1, 0, nullptr, nullptr};
    tc::Sched sc = whole;
    auto run = [&](int bn) {
      auto go = [&](auto c) {
        constexpr int B = decltype(c)::value;
        if constexpr (B % 64 != 0) {
          tc::launch_gemm<B>(A, M, Wsp, N, K, tc::OutDesc{nullptr, 0, Ysp, M, N},
                             EpiLinear<kEpiRelu, true>{b, N, 0, 0}, 0, sc);
        } else if (sh.score)
          tc::launch_gemm<B>(A, M, Wsp, N, K, tc::OutDesc{y, N, Split{}, M, N},
                             EpiBetaScore<1>{P, E, M, (int64_t)N}, 0, sc);
        else
          tc::launch_gemm<B>(A, M, Wsp, N, K, tc::OutDesc{nullptr, 0, Ysp, M, N},
                             EpiLinear<kEpiRelu, true>{b, N, 0, 0}, 0, sc);
      };
      switch (bn) {
        case 64: go(std::integral_constant<int, 64>{}); break;
        case 128: go(std::integral_constant<int, 128>{}); break;
        case 160: go(std::integral_constant<int, 160>{}); break;
        case 192: go(std::integral_constant<int, 192>{}); break;
        default: go(std::integral_constant<int, 256>{}); break;
      }
    };
    const int pick = plan.bn;
    printf("M=%5d N=%5d K=%5d %s |", M, N, K, sh.score ? "score " : "linear");
    for (int bn : {64, 128, 160, 192, 256})
      if (bn % 64 == 0 || !sh.score) printf(" %d:%.1f", bn, time_us([&] { run(bn); }));
    sc = tc::Sched{plan.full, plan.s_tail, plan.kper, gws.ws, gws.cnt};
    const double us = time_us([&] { run(pick); });
    printf(" | plan %d full %d split %d: %.1f us %.1f TFLOP/s useful\n", pick, plan.full, plan.s_tail, us,
           2.0 * M * N * K / us * 1e-6);
    if (getenv("PROBE_SPLITS")) {  // every (BN, tail split) combination: the planner's search space
      printf("    splits:");
      double best = 1e30;
      int bb = 0, bs = 0;
      for (int bn : {64, 128, 160, 192, 256}) {
        if (bn % 64 && sh.score) continue;
        const int nkb = (K + 31) / 32;
        const int tiles = ((M + 255) / 256) * ((N + bn - 1) / bn);
        const int full = tiles / 74 * 74, tail = tiles - full;
        for (int sp = 1; sp <= 4; ++sp) {
          if (tail == 0 && sp > 1) break;
          if (sp > 1 && tail * sp > 74) break;
          const int kper = (nkb + sp - 1) / sp;
          sc = sp == 1 ? whole : tc::Sched{full, sp, kper, gws.ws, gws.cnt};
          const double t = time_us([&] { run(bn); });
          printf(" %d/%d:%.1f", bn, sp, t);
          if (t < best) { best = t; bb = bn; bs = sp; }
        }
      }
      printf("  | best %d/%d %.1f us (plan %.1f)\n", bb, bs, best, us);
      sc = tc::Sched{plan.full, plan.s_tail, plan.kper, gws.ws, gws.cnt};
    }
#ifdef KGQ_TC_TRACE
    {
      const int tiles0 = ((M + 255) / 256) * ((N + pick - 1) / pick);
      const int tiles = sc.s_tail > 1 ? sc.full + (tiles0 - sc.full) * sc.s_tail : tiles0;  // units
      cudaMemset(tr, 0, 8192 * 64);
      run(pick);
      cudaDeviceSynchronize();
      std::vector<unsigned long long> h((size_t)tiles * 8);
      cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull, tend = 0;
      double ph[4] = {0};
      for (int t = 0; t < tiles; ++t) {
        t0 = std::min(t0, h[t * 8]);
        tend = std::max(tend, h[t * 8 + 4]);
        for (int i = 0; i < 4; ++i) ph[i] += (double)(h[t * 8 + i + 1] - h[t * 8 + i]) * 1e-3 / tiles;
      }
      printf("    trace: %d units, span %.1f us; per unit (us): wait-first-stage %.2f mainloop %.2f "
             "drain-tail %.2f epilogue %.2f\n", tiles, (tend - t0) * 1e-3, ph[0], ph[1], ph[2], ph[3]);
      if (sc.s_tail > 1)
        for (int t = sc.full; t < tiles && t < sc.full + 6; ++t) {
          const unsigned long long* x = &h[t * 8];
          printf("      unit %d: start %.1f first %.1f mma-done %.1f drained %.1f published %.1f counted %.1f reduced %.1f end %.1f\n",
                 t, (x[0] - t0) * 1e-3, (x[1] - t0) * 1e-3, (x[2] - t0) * 1e-3, (x[3] - t0) * 1e-3,
                 x[5] ? (x[5] - t0) * 1e-3 : -1.0, x[6] ? (x[6] - t0) * 1e-3 : -1.0, x[7] ? (x[7] - t0) * 1e-3 : -1.0,
                 (x[4] - t0) * 1e-3);
        }
    }
#endif
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    cudaFree(xf); cudaFree(wf); cudaFree(A.b0); cudaFree(Wsp.b0); cudaFree(Ysp.b0); cudaFree(b); cudaFree(y);
    cudaFree(P); cudaFree(E);
  }
  return 0;
}
