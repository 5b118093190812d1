// Small device helpers shared by the kernels of libkgq.so.
#pragma once
#include <mutex>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include <utility>
#include <stdint.h>

namespace kgq {

// Opt a kernel into more than 48 KB of dynamic shared memory on the CURRENT device.  The
// attribute is per (function, device): a process-wide "done" flag would leave a second
// context on another device launching with the 48 KB default (every launch there fails), so
// the cache is per device, per call site (F = the kernel's function pointer type + the calling
// template instance).  It holds the LARGEST value set: the attribute is a limit, and a call
// site whose size depends on the problem (the streaming scorers: d x query rows) must never
// lower it -- caching only "done" once let a d = 40 context set 5 KB and a later d = 400 one
// launch 51 KB against it ("invalid argument").  cudaGetDevice is a host-side lookup.
struct SmemAttr {
  int set[64] = {};  // per device: the largest MaxDynamicSharedMemorySize set so far
};
template <class F>
inline void smem_attr_once(F* kern, int bytes, SmemAttr& a) {
  int dev = 0;
  cudaGetDevice(&dev);
  int* s = &a.set[dev & 63];
  if (__atomic_load_n(s, __ATOMIC_ACQUIRE) >= bytes) return;
  static std::mutex mu;  // set + record atomically, so racing callers never lower the limit
  std::lock_guard<std::mutex> g(mu);
  if (*s >= bytes) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  __atomic_store_n(s, bytes, __ATOMIC_RELEASE);
}

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
// no-ops for a kernel launched without the attribute (the default, see pdl_env).
__device__ __forceinline__ void pdl_grid_sync() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Defaults from same-box measurements (KGQ_PDL = 0|1 sets both classes, KGQ_PDL_SMALL /
// KGQ_PDL_GEMM = 0|1 one class): ON for the persistent GEMM -- neutral in the per-type graph
// replays, +8% for the eagerly launched mixed-structure submit (3.41M -> 3.68M q/s) -- and OFF for
// the small kernels, whose early-launched CTAs take SM slots the predecessor still needs
// (per-type C2 -2.6% with them on).
inline int pdl_env(const char* specific, int dflt) {
  const char* f = getenv(specific);
  if (f && f[0]) return f[0] == '1' ? 1 : 0;
  const char* e = getenv("KGQ_PDL");
  if (e && e[0]) return e[0] == '1' ? 1 : 0;
  return dflt;
}
inline bool pdl_enabled() {  // small kernels (launch_pdl)
  static const int v = pdl_env("KGQ_PDL_SMALL", 0);
  return v == 1;
}
inline bool pdl_gemm_enabled() {  // the persistent GEMM (tc_gemm.cuh launch_gemm)
  static const int v = pdl_env("KGQ_PDL_GEMM", 1);
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

// Operand format of the tensor-core GEMMs (compile time, KGQ_OPERAND_FP16X2):
//  0  bf16x3: every operand x = b0 + b1 + b2 (three bf16 planes, exact); 6 bf16 MMAs per fp32
//     multiply-add (tc_gemm.cuh).
//  1  fp16x2 (Ootomo-Yokota split): activations ("A" operands) hold b0 = h = RN_fp16(x) and
//     b1 = l' = RN_fp16((x - h) 2^11) (b2 unused), i.e. x~ = h + l' 2^-11 with |x~ - x| <= 2^-22 |x|;
//     weights ("W" operands: dense weights, the scorer's (u, v) table) hold b0 = h 2^11 (exact),
//     b1 = l' and b2 = h, and the GEMM forms 2^11 x w ~= a_h w_h' + a_h w_l' + a_l' w_h -- three
//     fp16 MMAs per multiply-add, one fp32 accumulator scaled by 2^11 (undone exactly in the
//     epilogue), dropped a_l w_l ~ 2^-22 |x w|.  Range: |x| < 65504 (fp16); the scaled weight plane
//     needs |w| < 32.
//  Measured against the float64 oracle (profiles/r02/operand_accuracy.txt) fp16x2 is the MORE
//  accurate of the two -- its three MMAs per K step truncate in TMEM half as often as bf16x3's six
//  -- and 40% faster end to end; values outside its range are detected (range_flag below) and
//  reported as KGQ_ERANGE, for which the bf16x3 build (libkgq_bf16x3.so) is the full-range one.
#ifndef KGQ_OPERAND_FP16X2
#define KGQ_OPERAND_FP16X2 1
#endif
constexpr bool kFp16x2 = KGQ_OPERAND_FP16X2 != 0;
constexpr int kSplitPlanesA = kFp16x2 ? 2 : 3;  // planes an activation operand uses
constexpr int kMmasPerFma = kFp16x2 ? 3 : 6;    // tensor-core MMAs per useful fp32 multiply-add
constexpr float kLoScale = 2048.0f, kLoInv = 1.0f / 2048.0f;
constexpr float kFp16Limit = 65504.0f;          // activations: |x| below the fp16 maximum
constexpr float kFp16LimitW = 65504.0f / 2048.0f;  // weights: the 2^11-scaled high plane too
// Range guard of the fp16x2 format: a conversion of a finite |x| >= the limit sets this flag
// (one per translation unit -- `static` -- read and cleared by range_flag_take() from the host,
// kgq_check_errors / kgq_finalize turn it into KGQ_ERANGE).
static __device__ unsigned int g_range_flag = 0;
__device__ __forceinline__ void range_check(float a, float limit) {
  if constexpr (kFp16x2)
    if (fabsf(a) >= limit) atomicOr(&g_range_flag, 1u);
}
static inline unsigned int range_flag_take() {
  unsigned int v = 0, z = 0;
  if (cudaMemcpyFromSymbol(&v, g_range_flag, sizeof v) != cudaSuccess) return 0;
  if (v) cudaMemcpyToSymbol(g_range_flag, &z, sizeof z);
  return v;
}
__device__ __forceinline__ __nv_bfloat16 h2b(__half h) { return __ushort_as_bfloat16(__half_as_ushort(h)); }
__device__ __forceinline__ float b2hf(__nv_bfloat16 b) { return __half2float(__ushort_as_half(__bfloat16_as_ushort(b))); }

__device__ __forceinline__ void split3(float x, __nv_bfloat16& a, __nv_bfloat16& b, __nv_bfloat16& c) {
  if constexpr (kFp16x2) {
    range_check(x, kFp16Limit);
    const __half h = __float2half_rn(x);
    a = h2b(h);
    b = h2b(__float2half_rn((x - __half2float(h)) * kLoScale));
    c = __ushort_as_bfloat16(0);
  } else {
    a = __float2bfloat16_rn(x);
    const float r = x - __bfloat162float(a);
    b = __float2bfloat16_rn(r);
    c = __float2bfloat16_rn(r - __bfloat162float(b));
  }
}
// the weight ("W") form of the split: fp16x2 adds the 2^11-scaled high plane (see above)
__device__ __forceinline__ void split3_w(float x, __nv_bfloat16& a, __nv_bfloat16& b, __nv_bfloat16& c) {
  if constexpr (kFp16x2) {
    range_check(x, kFp16LimitW);
    const __half h = __float2half_rn(x);
    a = h2b(__float2half_rn(__half2float(h) * kLoScale));
    b = h2b(__float2half_rn((x - __half2float(h)) * kLoScale));
    c = h2b(h);
  } else {
    split3(x, a, b, c);
  }
}
__device__ __forceinline__ uint32_t pack_bf16(__nv_bfloat16 lo, __nv_bfloat16 hi) {
  return (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
}
// split3 of two values at once with packed conversions (one F2FP per plane pair): q0/q1/q2 =
// the (x, y) bf16 pairs of planes 0/1/2, x in the low half -- bit-identical to
// pack_bf16(split3(x), split3(y)) plane by plane.
__device__ __forceinline__ void split3_pair(float x, float y, uint32_t& q0, uint32_t& q1, uint32_t& q2) {
  if constexpr (kFp16x2) {
    range_check(fmaxf(fabsf(x), fabsf(y)), kFp16Limit);
    const __half2 h = __floats2half2_rn(x, y);
    const float2 f = __half22float2(h);
    const __half2 l = __floats2half2_rn((x - f.x) * kLoScale, (y - f.y) * kLoScale);
    q0 = *reinterpret_cast<const uint32_t*>(&h);
    q1 = *reinterpret_cast<const uint32_t*>(&l);
    q2 = 0u;
    return;
  }
  auto pk = [](float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  };
  auto lo = [](uint32_t u) { return __uint_as_float(u << 16); };
  auto hi = [](uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); };
  q0 = pk(x, y);
  const float rx = x - lo(q0), ry = y - hi(q0);
  q1 = pk(rx, ry);
  q2 = pk(rx - lo(q1), ry - hi(q1));
}

// Store x at element i of the split tensor (all three planes).
__device__ __forceinline__ void store_split(const Split& s, int64_t i, float x) {
  __nv_bfloat16 a, b, c;
  split3(x, a, b, c);
  s.b0[i] = a;
  s.b1[i] = b;
  if constexpr (!kFp16x2) s.b2[i] = c;
}

__device__ __forceinline__ float load_split(const Split& s, int64_t i) {
  if constexpr (kFp16x2) return b2hf(s.b0[i]) + b2hf(s.b1[i]) * kLoInv;  // exact: 11 + 11 bits
  return (__bfloat162float(s.b0[i]) + __bfloat162float(s.b1[i])) + __bfloat162float(s.b2[i]);
}
__device__ __forceinline__ void store_split_w(const Split& s, int64_t i, float x) {
  __nv_bfloat16 a, b, c;
  split3_w(x, a, b, c);
  s.b0[i] = a;
  s.b1[i] = b;
  s.b2[i] = c;
}
// 8 consecutive elements [i, i + 8) of a split tensor at once: one 16-byte access per plane
// (i % 8 == 0 and rows 16-byte aligned: ld % 8 == 0).  Bit-identical to 8 store_split /
// load_split calls.
__device__ __forceinline__ void store_split8(const Split& s, int64_t i, const float* x) {
  uint32_t q0[4], q1[4], q2[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) split3_pair(x[2 * j], x[2 * j + 1], q0[j], q1[j], q2[j]);
  *reinterpret_cast<uint4*>(s.b0 + i) = make_uint4(q0[0], q0[1], q0[2], q0[3]);
  *reinterpret_cast<uint4*>(s.b1 + i) = make_uint4(q1[0], q1[1], q1[2], q1[3]);
  if constexpr (!kFp16x2) *reinterpret_cast<uint4*>(s.b2 + i) = make_uint4(q2[0], q2[1], q2[2], q2[3]);
}
__device__ __forceinline__ void load_split8(const Split& s, int64_t i, float* x) {
  const uint4 u0 = *reinterpret_cast<const uint4*>(s.b0 + i), u1 = *reinterpret_cast<const uint4*>(s.b1 + i);
  if constexpr (kFp16x2) {
    const uint32_t a0[4] = {u0.x, u0.y, u0.z, u0.w}, a1[4] = {u1.x, u1.y, u1.z, u1.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 h = __half22float2(*reinterpret_cast<const __half2*>(&a0[j]));
      const float2 l = __half22float2(*reinterpret_cast<const __half2*>(&a1[j]));
      x[2 * j] = h.x + l.x * kLoInv;
      x[2 * j + 1] = h.y + l.y * kLoInv;
    }
    return;
  }
  const uint4 u2 = *reinterpret_cast<const uint4*>(s.b2 + i);
  const uint32_t a0[4] = {u0.x, u0.y, u0.z, u0.w}, a1[4] = {u1.x, u1.y, u1.z, u1.w}, a2[4] = {u2.x, u2.y, u2.z, u2.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    x[2 * j] = (__uint_as_float(a0[j] << 16) + __uint_as_float(a1[j] << 16)) + __uint_as_float(a2[j] << 16);
    x[2 * j + 1] = (__uint_as_float(a0[j] & 0xFFFF0000u) + __uint_as_float(a1[j] & 0xFFFF0000u)) +
                   __uint_as_float(a2[j] & 0xFFFF0000u);
  }
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

// fp64 reciprocal: fp32 seed + two Newton steps (2^-23 -> 2^-46 -> ~2^-92: within an ulp);
// x normal and inside the fp32 range
__device__ __forceinline__ double rcp_nr(double x) {
  double r = (double)__frcp_rn((float)x);
  r = r * (2.0 - x * r);
  r = r * (2.0 - x * r);
  return r;
}
// fp64 natural log for normal x > 0 without libdevice's special-case handling: x = 2^e m,
// m in [sqrt(1/2), sqrt(2)), ln m = 2 atanh(s), s = (m - 1)/(m + 1), |s| <= 0.1716, odd series
// through s^19 (truncation < 4e-16 relative).
__device__ __forceinline__ double log_pos(double x) {
  int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  int e = (hi >> 20) - 1023;
  hi = (hi & 0x000FFFFF) | 0x3FF00000;
  double m = __hiloint2double(hi, lo);
  if (m > 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  const double f = m - 1.0, den = m + 1.0;
  const double r = rcp_nr(den);
  double sq = f * r;
  sq = sq + r * (f - sq * den);  // residual correction of the quotient
  const double z = sq * sq;
  const double p = 1.0 / 3 + z * (1.0 / 5 + z * (1.0 / 7 + z * (1.0 / 9 + z * (1.0 / 11 + z * (1.0 / 13 +
                   z * (1.0 / 15 + z * (1.0 / 17 + z * (1.0 / 19))))))));
  return (double)e * 0.69314718055994530942 + (2.0 * sq + 2.0 * sq * z * p);
}
// Rising factorial x (x + 1) ... (x + 7) for x > 0 in Horner form: x (x^7 + 28 x^6 + 322 x^5 +
// 1960 x^4 + 6769 x^3 + 13132 x^2 + 13068 x + 5040) (unsigned Stirling numbers of the first kind
// c(8, k)) -- 8 fp64 operations instead of the product's 14; every coefficient and x are
// positive, so no cancellation (a few ulp, like the product)
__device__ __forceinline__ double rise8(double x) {
  double t = x + 28.0;
  t = fma(t, x, 322.0);
  t = fma(t, x, 1960.0);
  t = fma(t, x, 6769.0);
  t = fma(t, x, 13132.0);
  t = fma(t, x, 13068.0);
  t = fma(t, x, 5040.0);
  return t * x;
}
// ln B(a, b) = ln Gamma(a) + ln Gamma(b) - ln Gamma(a + b) for a, b > 0 (Eq. 3), the
// query-side P_q precompute of the tensor-core scorer.  ln Gamma(y) for y >= 8 by Stirling:
// (y - 1/2) ln y - y + ln(2 pi)/2 + sum_k B_2k / (2k (2k-1) y^(2k-1)).  Branch-free: every argument x is shifted
// by exactly 8 (y = x + 8 >= 8, ln Gamma(x) = ln Gamma(y) - ln(x (x+1) ... (x+7))), Stirling's
// series at y through y^-9 (truncation <= 691/360360 y^-11 ~ 2e-13 at y = 8), one reciprocal for
// the three series, and ONE log of the combined shift-product ratio.  Against libdevice lgamma:
// scripts/lnb_check.cu (same ~1e-5 relative cancellation limit when one argument is > 1e8 and
// the other O(0.1), where the libdevice formula loses the same digits).
__device__ __forceinline__ double lnbeta_f64(double a, double b) {
  const double c = a + b;
  const double pa = rise8(a), pb = rise8(b), pc = rise8(c);
  const double ya = a + 8.0, yb = b + 8.0, yc = c + 8.0;
  const double yab = ya * yb;
  const double rall = rcp_nr(yab * yc);  // <= (2e9 + 8)^3: inside the fp32 seed range
  const double ra = rall * yb * yc, rb = rall * ya * yc, rc = rall * yab;
  auto ser = [](double r) {
    const double z = r * r;
    return r * (1.0 / 12 + z * (-1.0 / 360 + z * (1.0 / 1260 + z * (-1.0 / 1680 + z * (1.0 / 1188)))));
  };
  const double pab = pa * pb;
  const double ratio = pab < 1e30 ? pc * rcp_nr(pab) : pc / pab;
  return (ya - 0.5) * log_pos(ya) + (yb - 0.5) * log_pos(yb) - (yc - 0.5) * log_pos(yc) - ya - yb + yc +
         0.91893853320467274178 + ser(ra) + ser(rb) - ser(rc) + log_pos(ratio);
}

// Table-driven fp64 log for normal x > 0 (the P_q prep's FP64 pipe is its bound): x = 2^e m,
// m in [1, 2), c_i = 1 + i/128 from the top 7 mantissa bits, r = (m - c_i) / c_i in [0, 1/128)
// (m - c_i exact), ln x = e ln 2 + ln c_i + ln(1 + r) with the series through r^7 (truncation
// < 2e-18).  lnc / invc: ln c_i and 1 / c_i (host-computed, kLogTab entries each, in shared
// memory).  ~11 fp64 operations instead of ~20 for log_pos.
constexpr int kLogTab = 128;
__device__ __forceinline__ double log_tab(double x, const double* lnc, const double* invc) {
  int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  const int e = (hi >> 20) - 1023;
  const int i = (hi >> 13) & (kLogTab - 1);
  hi = (hi & 0x000FFFFF) | 0x3FF00000;
  const double m = __hiloint2double(hi, lo);
  const double r = (m - (1.0 + i * (1.0 / kLogTab))) * invc[i];
  const double p = r * (1.0 + r * (-1.0 / 2 + r * (1.0 / 3 + r * (-1.0 / 4 + r * (1.0 / 5 + r * (-1.0 / 6 + r * (1.0 / 7)))))));
  return (double)e * 0.69314718055994530942 + (lnc[i] + p);
}
// lnbeta_f64 with the table log (same formula and error budget)
__device__ __forceinline__ double lnbeta_f64_tab(double a, double b, const double* lnc, const double* invc) {
  const double c = a + b;
  const double pa = rise8(a), pb = rise8(b), pc = rise8(c);
  const double ya = a + 8.0, yb = b + 8.0, yc = c + 8.0;
  const double yab = ya * yb;
  const double rall = rcp_nr(yab * yc);
  const double ra = rall * yb * yc, rb = rall * ya * yc, rc = rall * yab;
  auto ser = [](double r) {
    const double z = r * r;
    return r * (1.0 / 12 + z * (-1.0 / 360 + z * (1.0 / 1260 + z * (-1.0 / 1680 + z * (1.0 / 1188)))));
  };
  const double pab = pa * pb;
  const double ratio = pab < 1e30 ? pc * rcp_nr(pab) : pc / pab;
  return (ya - 0.5) * log_tab(ya, lnc, invc) + (yb - 0.5) * log_tab(yb, lnc, invc) -
         (yc - 0.5) * log_tab(yc, lnc, invc) - ya - yb + yc + 0.91893853320467274178 + ser(ra) + ser(rb) - ser(rc) +
         log_tab(ratio, lnc, invc);
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

