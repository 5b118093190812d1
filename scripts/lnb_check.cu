// Cross-check of the custom fp64 ln B(a, b) (common.cuh lnbeta_f64) against libdevice lgamma on
// log-uniform (a, b) in [0.01, 1e9] (not part of the library).
#include <cstdio>
#include <cmath>
#include "../paper_2503_02172_b200/csrc/common.cuh"
__global__ void k(const double* a, const double* b, double* o, double* r, int n, const double* tab, double* o2) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    o[i] = kgq::lnbeta_f64(a[i], b[i]);
    o2[i] = kgq::lnbeta_f64_tab(a[i], b[i], tab, tab + kgq::kLogTab);
    r[i] = lgamma(a[i]) + lgamma(b[i]) - lgamma(a[i] + b[i]);
  }
}
int main() {
  const int n = 1 << 16;
  double *a, *b, *o, *r;
  cudaMallocManaged(&a, n * 8); cudaMallocManaged(&b, n * 8); cudaMallocManaged(&o, n * 8); cudaMallocManaged(&r, n * 8);
  unsigned s = 1;
  for (int i = 0; i < n; ++i) {
    s = s * 1664525u + 1013904223u; double u = (s >> 8) / 16777216.0;
    s = s * 1664525u + 1013904223u; double v = (s >> 8) / 16777216.0;
    // log-uniform over [0.01, hi]: hi = 1e4 for the first half, 1e9 (the regulariser's clamp) for
    // the second; with one argument >~1e8 and the other O(0.1) both formulas lose ~1e-5 relative
    // to the lgamma(b) - lgamma(a + b) cancellation (scipy betaln as referee: same for libdevice)
    const double hi = i < n / 2 ? 1e4 : 1e9;
    a[i] = exp(log(0.01) + u * (log(hi) - log(0.01)));
    b[i] = exp(log(0.01) + v * (log(hi) - log(0.01)));
  }
  double *tab, *o2;
  cudaMallocManaged(&tab, 2 * kgq::kLogTab * 8);
  cudaMallocManaged(&o2, n * 8);
  for (int i = 0; i < kgq::kLogTab; ++i) {
    tab[i] = log(1.0 + (double)i / kgq::kLogTab);
    tab[kgq::kLogTab + i] = 1.0 / (1.0 + (double)i / kgq::kLogTab);
  }
  k<<<n / 256, 256>>>(a, b, o, r, n, tab, o2);
  cudaDeviceSynchronize();
  for (int h = 0; h < 2; ++h) {
    double mx = 0;
    for (int i = h * n / 2; i < (h + 1) * n / 2; ++i) mx = fmax(mx, fabs(o2[i] - r[i]) / fmax(1.0, fabs(r[i])));
    printf("lnbeta_f64_tab (table log) vs libdevice lgamma, (a, b) log-uniform in [0.01, %g]: max |diff|/max(1,|lnB|) %.3e\n",
           h ? 1e9 : 1e4, mx);
  }
  for (int h = 0; h < 2; ++h) {
    double mx = 0, mxr = 0;
    for (int i = h * n / 2; i < (h + 1) * n / 2; ++i) {
      const double e = fabs(o[i] - r[i]);
      const double rel = e / fmax(1.0, fabs(r[i]));
      if (rel > mxr) mxr = rel;
      if (e > mx) mx = e;
    }
    printf("lnbeta_f64 (shift-8, log_pos) vs libdevice lgamma, (a, b) log-uniform in [0.01, %g]: max |diff| %.3e, max |diff|/max(1,|lnB|) %.3e\n",
           h ? 1e9 : 1e4, mx, mxr);
  }
  return 0;
}
