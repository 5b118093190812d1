// Accuracy probe for the tcgen05 3xTF32 dense layer (not part of the library).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../include
//        scripts/tc_accuracy.cu -o tc_acc
// Prints max / rms relative error (vs float64) of y = x W^T for several input classes.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2503_02172_b200/csrc/chain.cu"
#include "../paper_2503_02172_b200/csrc/linear_tc.cu"

using namespace kgq;

static float tf32_rna_host(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

int main() {
  const int M = 256, N = 128;
  for (int K : {32, 96, 400, 1600}) {
    for (int cls = 0; cls < 3; ++cls) {
      std::mt19937_64 g(K * 7 + cls);
      std::uniform_real_distribution<float> U(-1.f, 1.f);
      std::vector<float> x((size_t)M * K), w((size_t)N * K), b(N, 0.f);
      for (auto& v : x) v = U(g);
      for (auto& v : w) v = U(g);
      if (cls == 1) {  // exactly representable in tf32: isolates accumulation error
        for (auto& v : x) v = tf32_rna_host(v);
        for (auto& v : w) v = tf32_rna_host(v);
      }
      if (cls == 2) {  // positive inputs: no cancellation, sums grow like K
        for (auto& v : x) v = fabsf(v);
        for (auto& v : w) v = fabsf(v);
      }
      float *dx, *dxh, *dxl, *dw, *dwh, *dwl, *db, *dy;
      cudaMalloc(&dx, x.size() * 4); cudaMalloc(&dxh, x.size() * 4); cudaMalloc(&dxl, x.size() * 4);
      cudaMalloc(&dw, w.size() * 4); cudaMalloc(&dwh, w.size() * 4); cudaMalloc(&dwl, w.size() * 4);
      cudaMalloc(&db, N * 4); cudaMalloc(&dy, (size_t)M * N * 4);
      cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(db, b.data(), N * 4, cudaMemcpyHostToDevice);
      launch_split_copy(dx, x.size(), dxh, dxl, 0);
      launch_split_copy(dw, w.size(), dwh, dwl, 0);
      Linear L;
      L.W = dw; L.W_hi = dwh; L.W_lo = dwl; L.b = db; L.out_f = N; L.in_f = K;
      launch_linear(Split{dxh, dxl, K}, M, K, L, kEpiNone, Split{dy, nullptr, N}, 0, 0, 0);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
      std::vector<float> y((size_t)M * N);
      cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost);
      double maxrel = 0, rms = 0, maxrel_f32 = 0;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double s = 0, sa = 0;
          float sf = 0.f;
          for (int k = 0; k < K; ++k) {
            const double p = (double)x[(size_t)m * K + k] * w[(size_t)n * K + k];
            s += p; sa += fabs(p);
            sf = fmaf(x[(size_t)m * K + k], w[(size_t)n * K + k], sf);
          }
          const double r = fabs(y[(size_t)m * N + n] - s) / sa;   // error relative to sum|terms|
          maxrel = fmax(maxrel, r); rms += r * r;
          maxrel_f32 = fmax(maxrel_f32, fabs(sf - s) / sa);
        }
      printf("K=%5d class=%d  3xTF32 max %.3e rms %.3e | sequential fp32 FMA max %.3e  (error / sum|x w|)\n",
             K, cls, maxrel, sqrt(rms / (M * N)), maxrel_f32);
      cudaFree(dx); cudaFree(dxh); cudaFree(dxl); cudaFree(dw); cudaFree(dwh); cudaFree(dwl);
      cudaFree(db); cudaFree(dy);
    }
  }
  return 0;
}
