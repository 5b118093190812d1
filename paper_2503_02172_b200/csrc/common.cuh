// Small device helpers shared by the kernels of libkgq.so.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace kgq {

// fp32 -> tf32 (round to nearest, ties away) kept in an fp32 container (low 13 bits zero).
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Store x as the split pair (hi, lo): hi = rna_tf32(x), lo = x - hi (exact in fp32).
__device__ __forceinline__ void store_split(float* hi, float* lo, int64_t i, float x) {
  float h = tf32_rna(x);
  hi[i] = h;
  lo[i] = x - h;
}

__device__ __forceinline__ float load_split(const float* hi, const float* lo, int64_t i) {
  return hi[i] + lo[i];
}

// Record the first out-of-range id: err = {flag, row, slot, kind(0 anchor, 1 relation)}.
__device__ __forceinline__ void report_range(int32_t* err, int32_t* invalid, int row, int slot,
                                             int kind) {
  if (atomicCAS(&err[0], 0, 1) == 0) {
    err[1] = row;
    err[2] = slot;
    err[3] = kind;
  }
  invalid[row] = 1;
}

__device__ __forceinline__ float beta_reg(float y) {  // Q2/Q12: clamp(y + 1, 0.05, 1e9)
  return fminf(fmaxf(y + 1.0f, 0.05f), 1e9f);
}

// fp64 digamma: recurrence psi(x) = psi(x+1) - 1/x up to x >= 10, then the asymptotic
// series ln x - 1/(2x) - sum_n B_2n / (2n x^2n) through x^-14 (truncation < 1e-16 there).
__device__ __forceinline__ double digamma_f64(double x) {
  double r = 0.0;
  while (x < 10.0) {
    r -= 1.0 / x;
    x += 1.0;
  }
  const double f = 1.0 / (x * x);
  const double t =
      f * (-1.0 / 12 +
           f * (1.0 / 120 +
                f * (-1.0 / 252 +
                     f * (1.0 / 240 + f * (-1.0 / 132 + f * (691.0 / 32760 + f * (-1.0 / 12)))))));
  return r + log(x) - 0.5 / x + t;
}

}  // namespace kgq

