// Dense layer y = epi(x W^T + b) (nn.Linear, W [out, in]) on the 5th-gen tensor cores.
//
// Used by the BetaE projection MLP (Eq. 4) and the intersection attention nets
// -- the only dense contractions on the path.  B200 has no fp32-input MMA,
// and single-pass TF32 misses the 1e-4 parity bound (SURVEY §0 finding 5), so this is 3xTF32:
//   x = x_hi + x_lo, w = w_hi + w_lo (hi = rna_tf32, lo = remainder; both exact in fp32)
//   x w ~= x_hi w_lo + x_lo w_hi + x_hi w_hi          (x_lo w_lo, ~2^-22 relative, dropped)
// accumulated in fp32 in TMEM.  Operands are produced already split (every producer kernel
// writes hi/lo pairs), so the mainloop is a pure TMA -> tcgen05.mma pipeline:
//   warp 0 / one lane : TMA producer, 4 tiles per stage (A_hi, A_lo, W_hi, W_lo), 128B swizzle
//   warp 1 / one lane : MMA issuer, 3 x (BK/8) tcgen05.mma.kind::tf32 per stage, commit->empty
//   warps 2-9         : epilogue; tcgen05.ld 32x32b (warp w owns TMEM lanes 32(w%4)..+31 = rows
//                       and half of the BN columns),
//                       partial sums added in fp32 registers, bias + ReLU / BetaE regulariser
//                       (+ negation) fused, split (hi/lo) or fp32 store.
// CTA tile 128 x BN (BN = 64 or 128) x BK = 32 fp32 (one 128-byte swizzle row), 3-4 stages;
// TMEM holds two 128 x BN partial accumulators (ping-pong between MMA and epilogue).
#include <stdint.h>

#include "tc_gemm.cuh"

namespace kgq {

namespace {
using tc::launch_tc_gemm;
using tc::BM;

// nn.Linear epilogue: + bias, ReLU / BetaE regulariser (clamp(y+1,.05,1e9)) with 1/x on rows
// [neg0, neg1) (negation fused, Q5), output split (hi/lo) for a next dense layer or fp32.
template <int CW, int EPI, bool SPLIT>
struct EpiLinear {
  const float* bias;
  Split out;
  int M, N, neg0, neg1;
  __device__ __forceinline__ void apply(int row0, int lane, int n0, const float (&acc)[CW],
                                        float* stage) const {
    const int row = row0 + lane;
    const bool neg = row >= neg0 && row < neg1;
#pragma unroll
    for (int i = 0; i < CW; ++i) {
      const int n = n0 + i;
      float y = acc[i] + (n < N ? bias[n] : 0.0f);
      if (EPI == kEpiRelu) y = fmaxf(y, 0.0f);
      if (EPI == kEpiBetaReg) {
        y = beta_reg(y);
        if (neg) y = 1.0f / y;
      }
      stage[lane * (CW + 1) + i] = y;
    }
    __syncwarp();
    for (int r = 0; r < 32; ++r) {  // row by row: lanes write consecutive columns
      const int rr = row0 + r;
      if (rr >= M) break;
      const int64_t o = (int64_t)rr * out.ld + n0;
#pragma unroll
      for (int c = lane; c < CW; c += 32) {
        if (n0 + c >= N) break;
        const float y = stage[r * (CW + 1) + c];
        if (SPLIT)
          store_split(out.hi, out.lo, o + c, y);
        else
          out.hi[o + c] = y;
      }
    }
  }
};

template <int EPI, bool SPLIT>
int launch_epi(const Split& A, int M, int K, const Linear& L, Split out, int neg0, int neg1,
               cudaStream_t st) {
  return tc::launch_gemm_auto(A, M, L.W_hi, L.W_lo, L.out_f, L.in_f, K, [&](auto cw) {
    return EpiLinear<decltype(cw)::value, EPI, SPLIT>{L.b, out, M, L.out_f, neg0, neg1};
  }, st);
}
}  // namespace

int launch_linear(const Split& A, int M, int K, const Linear& L, int epi, Split out, int neg0,
                  int neg1, cudaStream_t st) {
  if (M <= 0) return 0;
  const bool split = out.lo != nullptr;
  switch (epi) {
    case kEpiRelu:
      return split ? launch_epi<kEpiRelu, true>(A, M, K, L, out, neg0, neg1, st)
                   : launch_epi<kEpiRelu, false>(A, M, K, L, out, neg0, neg1, st);
    case kEpiBetaReg:
      return split ? launch_epi<kEpiBetaReg, true>(A, M, K, L, out, neg0, neg1, st)
                   : launch_epi<kEpiBetaReg, false>(A, M, K, L, out, neg0, neg1, st);
    default:
      return split ? launch_epi<kEpiNone, true>(A, M, K, L, out, neg0, neg1, st)
                   : launch_epi<kEpiNone, false>(A, M, K, L, out, neg0, neg1, st);
  }
}

}  // namespace kgq
