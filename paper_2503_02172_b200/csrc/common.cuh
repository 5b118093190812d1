// Small device helpers shared by the kernels of libkgq.so.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include <utility>
#include <stdint.h>

namespace kgq {

// fp32 tensor held as three bf16 planes, the operand format of the tensor-core GEMMs
// (tc_gemm.cuh, bf16x3): b0 = RN_bf16(x), b1 = RN_bf16(x - b0), b2 = RN_bf16(x - b0 - b1).
// Each remainder is exact in fp32 and the last one has <= 8 significant bits, so
// b0 + b1 + b2 == x exactly (bf16 keeps fp32's exponent range).  6 bytes per element.
struct Split {
  __nv_bfloat16* b0 = nullptr;
  __nv_bfloat16* b1 = nullptr;
  __nv_bfloat16* b2 = nullptr;
  int64_t ld = 0;  // row stride in elements (all three planes)
  __host__ __device__ __nv_bfloat16* plane(int p) const { return p == 0 ? b0 : p == 1 ? b1 : b2; }
  __host__ __device__ bool valid() const { return b0 != nullptr; }
  // the view starting at (row, col): same planes, shifted
  __host__ __device__ Split at(int64_t row, int64_t col = 0) const {
    const int64_t o = row * ld + col;
    return Split{b0 + o, b1 + o, b2 + o, ld};
  }
};

// Programmatic dependent launch (PDL): every hot-path kernel is launched with programmatic
// stream serialization, waits for its predecessor's results with griddepcontrol.wait before
// reading them and lets its successor start launching right away (griddepcontrol.
// launch_dependents), so kernel launch latency overlaps the predecessor's tail.  Both are
// no-ops for a kernel launched without the attribute.  KGQ_NO_PDL=1 disables the attribute.
__device__ __forceinline__ void pdl_grid_sync() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
inline bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KGQ_NO_PDL");
    v = (e && e[0] && e[0] != '0') ? 0 : 1;
  }
  return v == 1;
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Column of the offset half in a Q2B split state [centre | offset]: 8-element (16-byte) aligned
// so that the offset half is itself a TMA-addressable GEMM operand.
__host__ __device__ constexpr int q2b_off(int d) { return (d + 7) & ~7; }

__device__ __forceinline__ void split3(float x, __nv_bfloat16& a, __nv_bfloat16& b, __nv_bfloat16& c) {
  a = __float2bfloat16_rn(x);
  const float r = x - __bfloat162float(a);
  b = __float2bfloat16_rn(r);
  c = __float2bfloat16_rn(r - __bfloat162float(b));
}
__device__ __forceinline__ uint32_t pack_bf16(__nv_bfloat16 lo, __nv_bfloat16 hi) {
  return (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
}

// Store x at element i of the split tensor (all three planes).
__device__ __forceinline__ void store_split(const Split& s, int64_t i, float x) {
  __nv_bfloat16 a, b, c;
  split3(x, a, b, c);
  s.b0[i] = a;
  s.b1[i] = b;
  s.b2[i] = c;
}

__device__ __forceinline__ float load_split(const Split& s, int64_t i) {
  return (__bfloat162float(s.b0[i]) + __bfloat162float(s.b1[i])) + __bfloat162float(s.b2[i]);
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

// ln Gamma(y) for y >= 8 by the Stirling series through y^-13 (the first dropped term is
// < 1e-15 there): (y - 1/2) ln y - y + ln(2 pi)/2 + sum_k B_2k / (2k (2k-1) y^(2k-1)).
__device__ __forceinline__ double lgamma_stirling8(double y) {
  const double r = 1.0 / y, z = r * r;
  const double s = r * (1.0 / 12 + z * (-1.0 / 360 + z * (1.0 / 1260 + z * (-1.0 / 1680 +
                   z * (1.0 / 1188 + z * (-691.0 / 360360 + z * (1.0 / 156)))))));
  return (y - 0.5) * log(y) - y + 0.91893853320467274178 + s;
}
// Shift x > 0 up to y = x + n >= 8: ln Gamma(x) = ln Gamma(y) - ln(x (x+1) ... (x+n-1)); the
// product is returned in *p (multiplied into it), y as the result.
__device__ __forceinline__ double lgamma_shift8(double x, double* p) {
  while (x < 8.0) {
    *p *= x;
    x += 1.0;
  }
  return x;
}
// ln B(a, b) = ln Gamma(a) + ln Gamma(b) - ln Gamma(a + b) for a, b > 0 (Eq. 3): three
// Stirling evaluations and ONE log of the combined shift products -- ~4x fewer instructions
// than three libdevice lgamma calls (the query-side P_q precompute of the tensor-core scorer).
__device__ __forceinline__ double lnbeta_f64(double a, double b) {
  double pa = 1.0, pb = 1.0, pab = 1.0;
  const double ya = lgamma_shift8(a, &pa), yb = lgamma_shift8(b, &pb), yab = lgamma_shift8(a + b, &pab);
  return lgamma_stirling8(ya) + lgamma_stirling8(yb) - lgamma_stirling8(yab) + log(pab / (pa * pb));
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

