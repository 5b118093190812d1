// Dense layer y = epi(x W^T + b) (nn.Linear, W [out, in]) on the 5th-gen tensor cores.
//
// Used by the BetaE projection MLP (Eq. 4) and the intersection attention nets
// -- the only dense contractions on the path.  B200 has no fp32-input MMA,
// and single-pass TF32 / BF16 miss the 1e-4 parity bound (SURVEY §0 finding 5), so operands are
// held split (common.cuh Split): by default fp16x2 (x = h + l' 2^-11, three fp16 MMAs per fp32
// multiply-add), in the full-range build bf16x3 (x = x0 + x1 + x2, exact;
//   x w ~= x0 w0 + x0 w1 + x1 w0 + x0 w2 + x1 w1 + x2 w0     (dropped terms <= 2^-23 |x w|)),
// accumulated in fp32 in TMEM (tc_gemm.cuh).  Operands are produced already split (every
// producer kernel writes the three planes), so the mainloop is a pure TMA -> tcgen05.mma
// pipeline; the GEMM core (persistent CTA-pair kernel, TMA-store epilogue) is tc_gemm.cuh.  This
// file supplies the epilogue: bias + ReLU / BetaE regulariser (+ negation) fused, split
// (split planes) or fp32 output.
#include <stdint.h>

#include "tc_gemm.cuh"

namespace kgq {

namespace {
using tc::BM;

// nn.Linear epilogue: + bias, ReLU / BetaE regulariser (clamp(y+1,.05,1e9)) with 1/x on rows
// [neg0, neg1) (negation fused, Q5); output split (PLANES 3) for a next dense layer,
// or fp32.
// REL: first BetaE projection layer with the relation input factored out (RelTerm below): the
// accumulator of row (group gi, query b) starts at RW[r] for r = rels[b, rel_slot[gi]].
template <int EPI, bool SPLIT, bool REL = false>
struct EpiLinear {
  static constexpr int PLANES = SPLIT ? 3 : 1, ROWDIV = 1;
  static constexpr bool CMIN = false, INIT = REL, STREAM_OUT = false;
  template <int CH>
  __device__ void chunk_min(int, int, const float*) const {}
  const float* bias;
  int N, neg0, neg1;
  RelTerm rt;
  RowMap rm{};   // optional output row remap (rm.n > 0): rows >= rows are not stored
  int rows = 0;
  // destination row of the 32-row output box starting at GEMM row row0 (-1: nothing to store)
  __device__ __forceinline__ int out_row(int row0) const {
    if (rm.n == 0) return row0;
    if (row0 >= rows) return -1;
    int i = 0;
    while (i + 1 < rm.n && rm.dst0[i + 1] <= row0) ++i;
    return rm.src0[i] + row0 - rm.dst0[i];
  }
  template <int CW>
  __device__ __forceinline__ void init(int row, int n0, float* acc) const {
    if (row >= rt.M) return;
    int r;
    if (rt.rid) {
      r = rt.rid[row];  // mixed batches: looked up and range-checked by the gather
    } else {
      const int gi = row / rt.B, b = row - gi * rt.B;
      const int slot = rt.rel_slot[gi];
      r = rt.rels[(int64_t)b * rt.n_r + slot];
      if (r < 0 || r >= rt.n_relation) {  // kgq.h: out-of-range id -> NaN row, KGQ_ERANGE
        if (atomicCAS(&rt.err[0], 0, 1) == 0) {
          rt.err[1] = b;
          rt.err[2] = slot;
          rt.err[3] = 1;
        }
        rt.invalid[b] = 1;
        r = 0;
      }
    }
    const float* w = rt.RW + (int64_t)r * rt.ldrw + n0;
#pragma unroll
    for (int i = 0; i < CW; i += 4) {
      if (n0 + i + 4 <= N) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(w + i));
        acc[i] = v.x;
        acc[i + 1] = v.y;
        acc[i + 2] = v.z;
        acc[i + 3] = v.w;
      }
    }
  }
  struct Pre {
    float b[4];  // bias of columns n0 + lane + 32 j
    bool neg;      // this lane's row is negated
    bool any_neg;  // some row of this warp's 32-row box is (warp-uniform)
  };
  template <int CW>
  __device__ __forceinline__ Pre prefetch(int row, int n0, int lane) const {
    Pre p;
#pragma unroll
    for (int j = 0; j < (CW + 31) / 32; ++j) p.b[j] = n0 + lane + 32 * j < N ? __ldg(bias + n0 + lane + 32 * j) : 0.0f;
    p.neg = row >= neg0 && row < neg1;
    p.any_neg = __any_sync(0xffffffffu, p.neg);
    return p;
  }
  template <int CH>
  __device__ __forceinline__ void chunk(const Pre& p, int row, int c, float* v) const {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      float y = v[i] + __shfl_sync(0xffffffffu, p.b[(c + i) >> 5], (c + i) & 31);
      if (EPI == kEpiRelu) y = fmaxf(y, 0.0f);
      if (EPI == kEpiBetaReg) y = beta_reg(y);
      v[i] = y;
    }
    // negation (1/x, Q5) behind a warp-uniform branch: the IEEE division is ~10 instructions with
    // a slow-path check, and only the negated branches' rows (a few 32-row boxes) need it -- as a
    // select on every element it made the regulariser layer's epilogue outlast the MMAs it
    // overlaps (hop-0 last layer: tensor pipe 55% active vs 88% for the ReLU layer before it)
    if (EPI == kEpiBetaReg && p.any_neg) {
#pragma unroll
      for (int i = 0; i < CH; ++i)
        if (p.neg) v[i] = 1.0f / v[i];
    }
  }
};

template <int EPI, bool SPLIT>
int launch_epi(const Split& A, int M, int K, const Linear& L, const Split& out_sp, float* out_f32, int64_t ld_f32,
               int neg0, int neg1, const GemmWs* ws, cudaStream_t st) {
  const tc::OutDesc o{out_f32, ld_f32, out_sp, M, L.out_f};
  return tc::launch_gemm_auto(A, M, L.Wsp, L.out_f, K, o, EpiLinear<EPI, SPLIT>{L.b, L.out_f, neg0, neg1, RelTerm{}},
                              ws, st);
}
}  // namespace

int launch_linear_rel(const Split& A, int M, int K, const Linear& L, const RelTerm& rt, const Split& out,
                      const GemmWs* ws, cudaStream_t st) {
  if (M <= 0) return 0;
  const tc::OutDesc o{nullptr, 0, out, M, L.out_f};
  return tc::launch_gemm_auto(A, M, L.Wsp, L.out_f, K, o, EpiLinear<kEpiRelu, true, true>{L.b, L.out_f, 0, 0, rt},
                              ws, st);
}

int launch_linear_map(const Split& A, int M, int K, const Linear& L, int epi, const Split& out, int64_t out_rows,
                      const RowMap& rm, int neg0, int neg1, const GemmWs* ws, cudaStream_t st) {
  if (M <= 0) return 0;
  const tc::OutDesc o{nullptr, 0, out, out_rows, L.out_f};
#define KGQ_EPI_MAP(E)                                                             \
  do {                                                                             \
    EpiLinear<E, true> e{L.b, L.out_f, neg0, neg1, RelTerm{}};                     \
    e.rm = rm;                                                                     \
    e.rows = M;                                                                    \
    return tc::launch_gemm_auto(A, M, L.Wsp, L.out_f, K, o, e, ws, st);            \
  } while (0)
  switch (epi) {
    case kEpiRelu: KGQ_EPI_MAP(kEpiRelu);
    case kEpiBetaReg: KGQ_EPI_MAP(kEpiBetaReg);
    default: KGQ_EPI_MAP(kEpiNone);
  }
#undef KGQ_EPI_MAP
}

int launch_linear(const Split& A, int M, int K, const Linear& L, int epi, const Split& out_sp, float* out_f32,
                  int64_t ld_f32, int neg0, int neg1, const GemmWs* ws, cudaStream_t st) {
  if (M <= 0) return 0;
  const bool split = out_sp.valid();
#define KGQ_EPI(E) (split ? launch_epi<E, true>(A, M, K, L, out_sp, out_f32, ld_f32, neg0, neg1, ws, st) \
                          : launch_epi<E, false>(A, M, K, L, out_sp, out_f32, ld_f32, neg0, neg1, ws, st))
  switch (epi) {
    case kEpiRelu: return KGQ_EPI(kEpiRelu);
    case kEpiBetaReg: return KGQ_EPI(kEpiBetaReg);
    default: return KGQ_EPI(kEpiNone);
  }
#undef KGQ_EPI
}

// this translation unit's fp16x2 range flag (common.cuh range_check), read and cleared
unsigned int range_flag_linear() { return range_flag_take(); }

}  // namespace kgq
