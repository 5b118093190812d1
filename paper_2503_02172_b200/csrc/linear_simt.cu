// Dense layer y = epi(x W^T + b) (nn.Linear, W [out, in]) -- fp32 SIMT version.
//
// Used by the BetaE projection MLP (Eq. 4) and the intersection attention
// nets (Q6).  Operands arrive as split pairs (hi + lo == x exactly) so that the tensor-core
// 3xTF32 kernel (linear_tc.cu) can consume the same buffers; this kernel re-adds them and
// runs plain fp32 FFMA.  128x128x8 CTA tile, 8x8 per thread, register double buffering.
#include "common.cuh"
#include "kgq_internal.cuh"

namespace kgq {

namespace {
constexpr int BM = 128, BN = 128, BK = 8, PAD = 4;

template <int EPI, bool SPLIT>
__global__ void __launch_bounds__(256) k_linear_simt(Split A, int M, int K,
                                                     const float* __restrict__ W,
                                                     const float* __restrict__ bias, int N,
                                                     Split out, int neg0, int neg1) {
  __shared__ __align__(16) float As[2][BK][BM + PAD];
  __shared__ __align__(16) float Ws[2][BK][BN + PAD];
  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  // loader mapping: 128 rows x 8 k, 4 consecutive k per thread
  const int lr = tid >> 1, lk = (tid & 1) * 4;

  float ra[4], rw[4];
  auto load = [&](int kb) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = kb + lk + i;
      const int m = m0 + lr, n = n0 + lr;
      ra[i] = (m < M && k < K) ? load_split(A.hi, A.lo, (int64_t)m * A.ld + k) : 0.0f;
      rw[i] = (n < N && k < K) ? W[(int64_t)n * K + k] : 0.0f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      As[buf][lk + i][lr] = ra[i];
      Ws[buf][lk + i][lr] = rw[i];
    }
  };

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

  const int nk = (K + BK - 1) / BK;
  load(0);
  store(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load((t + 1) * BK);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[8], w[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
      const float4 w0 = *reinterpret_cast<const float4*>(&Ws[buf][k][tx * 4]);
      const float4 w1 = *reinterpret_cast<const float4*>(&Ws[buf][k][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
      w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    if (t + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= M) continue;
    const bool neg = m >= neg0 && m < neg1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n >= N) continue;
      float y = acc[i][j] + bias[n];
      if (EPI == kEpiRelu) y = fmaxf(y, 0.0f);
      if (EPI == kEpiBetaReg) {
        y = beta_reg(y);
        if (neg) y = 1.0f / y;
      }
      const int64_t o = (int64_t)m * out.ld + n;
      if (SPLIT)
        store_split(out.hi, out.lo, o, y);
      else
        out.hi[o] = y;
    }
  }
}

template <int EPI>
void launch_epi(const Split& A, int M, int K, const Linear& L, Split out, int neg0, int neg1,
                cudaStream_t st) {
  dim3 grid((L.out_f + BN - 1) / BN, (M + BM - 1) / BM);
  if (out.lo)
    k_linear_simt<EPI, true><<<grid, 256, 0, st>>>(A, M, K, L.W, L.b, L.out_f, out, neg0, neg1);
  else
    k_linear_simt<EPI, false><<<grid, 256, 0, st>>>(A, M, K, L.W, L.b, L.out_f, out, neg0, neg1);
}
}  // namespace

int launch_linear(const Split& A, int M, int K, const Linear& L, int epi, Split out, int neg0,
                  int neg1, cudaStream_t st) {
  if (M <= 0) return 0;
  switch (epi) {
    case kEpiRelu: launch_epi<kEpiRelu>(A, M, K, L, out, neg0, neg1, st); break;
    case kEpiBetaReg: launch_epi<kEpiBetaReg>(A, M, K, L, out, neg0, neg1, st); break;
    default: launch_epi<kEpiNone>(A, M, K, L, out, neg0, neg1, st); break;
  }
  return 1;
}

}  // namespace kgq
