// Tensor-core BetaE scorer (a6 + a7 for BetaE at batch sizes past the
// HBM ridge).
//
// Per dimension KL(Beta(ae,be) || Beta(aq,bq)) = L_q + C_e + aq U_e + bq V_e >= 0 (closed form
// of the Eq. 3 densities, entity-only and query-only lgamma/digamma terms; prep.cu), and a
// KL divergence is non-negative, so sum_d |KL_d| = sum_d KL_d exactly.  With per-dimension
// means Ubar_d, Vbar_d (over all N entities) and u = U - Ubar, v = V - Vbar:
//   dist(q, e) = P_q + E_e + sum_d (aq_d u_ed + bq_d v_ed)
//   P_q = sum_d (lnB(aq_d, bq_d) + aq_d Ubar_d + bq_d Vbar_d)     (fp64, per query row)
//   E_e = sum_d C_ed                                               (fp64, per entity, finalize)
// P_q and E_e are stored as fp32 pairs (hi = RN(x), lo = RN(x - hi)) and the epilogue forms
// (P_hi + E_hi) + ((P_lo + E_lo) + acc) in fp32: the first sum is exact when it cancels
// (Sterbenz; the usual case, P ~ -E) and otherwise errs by <= 2^-24 |P + E| ~ 2^-24 dist, the
// dropped lo-lo rounding is ~2^-48 |P|, so dist carries ~1e-7 relative -- three FADDs instead
// of fp64 adds and conversions, and no fp64 registers next to the row accumulators.
// The last term is a dense contraction [rows, 2d] x [2d, N] on tcgen05 with split fp32 operands
// (fp16x2 by default, bf16x3 in the full-range build; tc_gemm.cuh, common.cuh).
// Centring keeps its terms ~0.1 (|u|, |v| << |U|, |V| ~ 1), so the fp32 partial sums carry
// ~1e-7 of sum|terms| ~ 1e-5 absolute instead of ~1e-4 for the uncentred sum, and the large,
// cancelling P_q + E_e (~ +-800 at d = 400) are added in fp64 in the epilogue.  DNF union:
// rows are (b, branch) = 2b + br, so the two branches of a query are adjacent rows of the
// epilogue's staged tile and the min is taken while writing dist rows.
#include "tc_gemm.cuh"

namespace kgq {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Pass 1: per-dimension sums of U and V over all entities (means for centring).
__global__ void k_uv_dim_sums(const float* __restrict__ ent, int64_t e0, int64_t ns, int d,
                              double* __restrict__ sums /* [2][d] */) {
  const int j = blockIdx.y * blockDim.x + threadIdx.x;
  if (j >= d) return;
  double su = 0.0, sv = 0.0;
  for (int64_t e = blockIdx.x; e < ns; e += gridDim.x) {
    const double a = ent[(e0 + e) * 2 * d + j], b = ent[(e0 + e) * 2 * d + d + j];
    const double pab = digamma_f64(a + b);
    su += pab - digamma_f64(a);
    sv += pab - digamma_f64(b);
  }
  atomicAdd(&sums[j], su);
  atomicAdd(&sums[d + j], sv);
}

// Pass 2: centred split table uv [np][2d] = [u; v] (hi/lo) and E_e = sum_d C_ed (fp64).
__device__ __forceinline__ float2 split_f64(double x) {
  const float h = (float)x;
  return make_float2(h, (float)(x - (double)h));
}

__global__ void k_uv_table(const float* __restrict__ ent, int64_t e0, int64_t ns, int64_t np, int d,
                           int64_t n_all, const double* __restrict__ sums, Split uv,
                           float2* __restrict__ Esum, float* __restrict__ uvT) {
  const int64_t e = blockIdx.x;
  __shared__ double red[32];
  double c = 0.0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float u = 0.0f, v = 0.0f;
    if (e < ns) {
      const double a = ent[(e0 + e) * 2 * d + j], b = ent[(e0 + e) * 2 * d + d + j];
      const double pa = digamma_f64(a), pb = digamma_f64(b), pab = digamma_f64(a + b);
      c += -(lgamma(a) + lgamma(b) - lgamma(a + b)) + a * pa + b * pb - (a + b) * pab;
      u = (float)((pab - pa) - sums[j] / (double)n_all);
      v = (float)((pab - pb) - sums[d + j] / (double)n_all);
    }
    store_split_w(uv, e * 2 * d + j, u);  // the scorer GEMM's "W" operand
    store_split_w(uv, e * 2 * d + d + j, v);
    if (uvT) {  // dim-major fp32 copy for the small-batch streaming scorer: [d][2][np]
      uvT[(int64_t)(2 * j) * np + e] = u;
      uvT[(int64_t)(2 * j + 1) * np + e] = v;
    }
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) Esum[e] = split_f64(t);
  }
}

// Per batch: A = split [aq; bq] rows (query embedding rows, already (b, branch) ordered) and
// P_q in fp64.
__global__ void k_score_prep_tc(const float* __restrict__ q, int rows, int d,
                                const double* __restrict__ sums, int64_t ns, Split A,
                                float2* __restrict__ P) {
  pdl_grid_sync();
  const int r = blockIdx.x;
  __shared__ double red[32];
  __shared__ double tab[2 * kLogTab];  // ln c_i, 1 / c_i (stored after the [2][d] sums)
  for (int i = threadIdx.x; i < 2 * kLogTab; i += blockDim.x) tab[i] = sums[2 * d + i];
  __syncthreads();
  double p = 0.0;
  const double inv = 1.0 / (double)ns;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const float a = q[(int64_t)r * 2 * d + j], b = q[(int64_t)r * 2 * d + d + j];
    store_split(A, (int64_t)r * A.ld + j, a);
    store_split(A, (int64_t)r * A.ld + d + j, b);
    const double da = a, db = b;
    p += lnbeta_f64_tab(da, db, tab, tab + kLogTab) + da * sums[j] * inv + db * sums[d + j] * inv;
  }
  p = warp_sum(p);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = p;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) P[r] = split_f64(t);
  }
}

// Score epilogue: dist = (P_hi + E_hi) + ((P_lo + E_lo) + acc), DNF min over row pairs (NB 2),
// and, when cmin is set, the minimum of every 32-entity block of each output row over the
// shard's real entities (columns < nvalid): cmin[row][n / 32].  The top-k reads these block
// minima first and scans only the blocks that can hold one of the k best (k_topk_cmin).
// Mixed batches: score row r is the split state row srcrow[r] of S (no fp32 round trip).
// Single-structure submits (srcrow == nullptr): score row r of the chunk starting at query b0 is
// branch r % nout of query b0 + r / nout, i.e. state row (r % nout) * B + b0 + r / nout.
// One WARP per score row, four rows per 128-thread block (the log table staged once per block):
// d = 400 dims are 12-13 per lane instead of 3-4 per thread of a 128-thread block per row, whose
// 16 four-dim threads left the other 112 idle for the last chain (25% of the fp64 time), and the
// row sum is a shuffle tree without __syncthreads.
constexpr int kPrepRows = 4;
// Register cap: ten resident 128-thread blocks per SM (48 registers, 8 bytes spilled) instead of
// the 64-register default's eight -- more rows in flight for the latency-bound fp64 chains:
// 109 -> 92.5 us per C2 step (ncu), C2 +0.8%; twelve blocks (40 registers) spill 120 bytes
// (95.7 us), sixteen 276 (101.6 us)
#ifndef KGQ_PREP_MINB
#define KGQ_PREP_MINB 10
#endif
__global__ void __launch_bounds__(32 * kPrepRows, KGQ_PREP_MINB)
    k_mix_score_prep(const int64_t* __restrict__ srcrow, Split S, int d, const double* __restrict__ sums, int64_t ns,
                     Split A, float2* __restrict__ P, int64_t B, int64_t b0, int nout, int rows) {
  pdl_grid_sync();
  __shared__ double tab[2 * kLogTab];  // ln c_i, 1 / c_i (stored after the [2][d] sums)
  for (int i = threadIdx.x; i < 2 * kLogTab; i += blockDim.x) tab[i] = sums[2 * d + i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kPrepRows + (threadIdx.x >> 5);
  if (r >= rows) return;
  double p = 0.0;
  const double inv = 1.0 / (double)ns;
  const int64_t srow = srcrow ? srcrow[r] : (int64_t)(r % nout) * B + b0 + r / nout;
  const int64_t s0 = srow * S.ld, a0 = (int64_t)r * A.ld;
  if ((d & 7) == 0 && (S.ld & 7) == 0 && (A.ld & 7) == 0) {
    // the row copy as 16-byte plane accesses (a plain copy of the split planes), then the fp64
    // P_q terms from the fp32 values
    for (int j = 8 * lane; j < 2 * d; j += 8 * 32)
#pragma unroll
      for (int p3 = 0; p3 < kSplitPlanesA; ++p3)
        *reinterpret_cast<uint4*>(A.plane(p3) + a0 + j) = *reinterpret_cast<const uint4*>(S.plane(p3) + s0 + j);
    // two dims per iteration with two partial sums: independent fp64 chains in flight (the
    // FP64 pipe is this kernel's bound; one chain per lane left it ~58% busy)
    double p1 = 0.0;
    int j = lane;
    for (; j + 32 < d; j += 64) {
      const double da = load_split(S, s0 + j), db = load_split(S, s0 + d + j);
      const double ea = load_split(S, s0 + j + 32), eb = load_split(S, s0 + d + j + 32);
      const double t0 = lnbeta_f64_tab(da, db, tab, tab + kLogTab);
      const double t1 = lnbeta_f64_tab(ea, eb, tab, tab + kLogTab);
      p += t0 + da * sums[j] * inv + db * sums[d + j] * inv;
      p1 += t1 + ea * sums[j + 32] * inv + eb * sums[d + j + 32] * inv;
    }
    if (j < d) {
      const double da = load_split(S, s0 + j), db = load_split(S, s0 + d + j);
      p += lnbeta_f64_tab(da, db, tab, tab + kLogTab) + da * sums[j] * inv + db * sums[d + j] * inv;
    }
    p += p1;
  } else {
    for (int j = lane; j < d; j += 32) {
      const float a = load_split(S, s0 + j), b = load_split(S, s0 + d + j);
      store_split(A, a0 + j, a);
      store_split(A, a0 + d + j, b);
      const double da = a, db = b;
      p += lnbeta_f64_tab(da, db, tab, tab + kLogTab) + da * sums[j] * inv + db * sums[d + j] * inv;
    }
  }
  p = warp_sum(p);
  if (lane == 0) P[r] = split_f64(p);
}

// TK (fused top-k): no distance block; the epilogue keeps every output row's k
// smallest (dist, column) pairs per N stripe (tc_gemm.cuh TOPK) and writes only those lists.
template <int NB, bool TK = false>
struct EpiBetaScore {
  static constexpr int PLANES = 1, ROWDIV = NB;
  static constexpr bool CMIN = !TK, INIT = false, STREAM_OUT = true, TOPK = TK;
  // One TMEM partial per tile for K = 2d <= 800 (25 K-blocks): the scorer's epilogue (the fused
  // top-k lists above all) then runs once per tile instead of after every 8 K-blocks -- scorer
  // 458 -> 480 TFLOP/s, C2 +1.7% -- while the whole-row distance errors vs the oracle stay
  // unchanged to three digits (small / medium / C2 / C4: 2.4e-5 / 4.2e-5 / 1.6e-5 / 2.2e-5; they
  // are dominated by the query embedding, profiles/r02/score_drain_ab.txt)
#ifndef KGQ_SCORE_DRAIN
#define KGQ_SCORE_DRAIN 25
#endif
  static constexpr int DRAIN = KGQ_SCORE_DRAIN;
  template <int CW>
  __device__ void init(int, int, float*) const {}
  const float2* P;  // [rows] (hi, lo)
  const float2* E;  // [np] (hi, lo)
  int rows;
  int64_t ncols;    // np: the last column tile may overhang it
  float* cmin = nullptr;  // [rows / NB][ldc] block minima, or nullptr
  int64_t ldc = 0;
  int64_t nvalid = 0;     // the shard's entity count ns (columns >= ns are padding)
  unsigned long long* cand = nullptr;  // TK: [rows / NB][ldcand] per-stripe sorted key lists
  int64_t ldcand = 0;
  int k = 0;
  __device__ __forceinline__ int out_row(int row0) const { return row0 / NB; }  // no remap
  struct Pre {
    float2 p;       // P of this lane's row
    float2 e[4];    // E of columns n0 + lane + 32 j
  };
  template <int CW>
  __device__ __forceinline__ Pre prefetch(int row, int n0, int lane) const {
    Pre r;
    r.p = row < rows ? __ldg(P + row) : make_float2(0.0f, 0.0f);
#pragma unroll
    for (int j = 0; j < CW / 32; ++j)
      r.e[j] = n0 + lane + 32 * j < ncols ? __ldg(E + n0 + lane + 32 * j) : make_float2(0.0f, 0.0f);
    return r;
  }
  template <int CH>
  __device__ __forceinline__ void chunk(const Pre& r, int row, int c, float* v) const {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const float eh = __shfl_sync(0xffffffffu, r.e[(c + i) >> 5].x, (c + i) & 31);
      const float el = __shfl_sync(0xffffffffu, r.e[(c + i) >> 5].y, (c + i) & 31);
      v[i] = (r.p.x + eh) + ((r.p.y + el) + v[i]);
    }
  }
  template <int CH>
  __device__ __forceinline__ void chunk_min(int row, int n, const float* v) const {
    static_assert(CH == 32, "block minima are over 32 columns");
    if (!cmin || (NB == 2 && (row & 1)) || row >= rows || n >= nvalid) return;
    float m = __uint_as_float(0x7F800000u);
    if (n + CH <= nvalid) {  // interior block: pairwise tree, no column predicates
      float t[CH / 2];
#pragma unroll
      for (int i = 0; i < CH / 2; ++i) t[i] = fminf(v[2 * i], v[2 * i + 1]);
#pragma unroll
      for (int w = CH / 4; w >= 1; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) t[i] = fminf(t[i], t[i + w]);
      m = t[0];
    } else {
#pragma unroll
      for (int i = 0; i < CH; ++i)
        if (n + i < nvalid) m = fminf(m, v[i]);
    }
    cmin[(int64_t)(row / NB) * ldc + n / 32] = m;
  }
};

}  // namespace

int launch_betae_uv_table(const float* ent, int64_t n_all, int64_t e0, int64_t ns, int64_t np, int d,
                          double* sums, Split uv, float2* Esum, float* uvT, cudaStream_t st) {
  // centring means over ALL entities (every rank holds the full table), so that every shard
  // uses the same u, v and a sharded run is bit-identical to a single-GPU run
  cudaMemsetAsync(sums, 0, 2 * d * sizeof(double), st);
  const int gx = (int)(n_all < 1024 ? n_all : 1024);
  k_uv_dim_sums<<<dim3(gx, (d + 127) / 128), 128, 0, st>>>(ent, 0, n_all, d, sums);
  k_uv_table<<<(unsigned)np, 128, 0, st>>>(ent, e0, ns, np, d, n_all, sums, uv, Esum, uvT);
  return 2;
}

int launch_mix_score_prep(const int64_t* srcrow, Split S, int rows, int d, const double* sums, int64_t ns,
                          Split A, float2* P, cudaStream_t st, int64_t B, int64_t b0, int nout) {
  if (rows <= 0) return 0;
  launch_pdl(k_mix_score_prep, dim3((rows + kPrepRows - 1) / kPrepRows), dim3(32 * kPrepRows), 0, st, srcrow, S, d,
             sums, ns, A, P, B, b0, nout, rows);
  return 1;
}

int launch_score_tc_gemm(int rows, int nbq, int d, Split A, const float2* P, const Split& uv, const float2* Esum,
                         int64_t np, float* dist, int64_t ldd, float* cmin, int64_t ldc, int64_t nvalid,
                         const GemmWs* ws, cudaStream_t st) {
  if (rows <= 0) return 0;
  const tc::OutDesc o{dist, ldd, Split{}, rows / nbq, np};
  if (nbq == 2)
    return tc::launch_gemm_auto(A, rows, uv, (int)np, 2 * d, o, EpiBetaScore<2>{P, Esum, rows, np, cmin, ldc, nvalid},
                                ws, st);
  return tc::launch_gemm_auto(A, rows, uv, (int)np, 2 * d, o, EpiBetaScore<1>{P, Esum, rows, np, cmin, ldc, nvalid},
                              ws, st);
}

int launch_score_tc_topk(int rows, int nbq, int d, Split A, const float2* P, const Split& uv, const float2* Esum,
                         int64_t np, int64_t nvalid, int k, unsigned long long* cand, int64_t ldcand,
                         const GemmWs* ws, cudaStream_t st, int* nlists, int min_tiles) {
  if (rows <= 0) {
    *nlists = 0;
    return 0;
  }
  int ns = 1, L;
  if (nbq == 2) {
    EpiBetaScore<2, true> e{P, Esum, rows, np};
    e.nvalid = nvalid;
    e.cand = cand;
    e.ldcand = ldcand;
    e.k = k;
    L = tc::launch_gemm_topk(A, rows, uv, (int)np, 2 * d, e, ws, st, &ns, min_tiles);
  } else {
    EpiBetaScore<1, true> e{P, Esum, rows, np};
    e.nvalid = nvalid;
    e.cand = cand;
    e.ldcand = ldcand;
    e.k = k;
    L = tc::launch_gemm_topk(A, rows, uv, (int)np, 2 * d, e, ws, st, &ns, min_tiles);
  }
  *nlists = 2 * ns;  // one list per (stripe, column half)
  return L;
}

int launch_score_prep_tc(const float* q, int rows, int d, const double* sums, int64_t ns, Split A, float2* P,
                         cudaStream_t st) {
  if (rows <= 0) return 0;
  launch_pdl(k_score_prep_tc, dim3(rows), dim3(128), 0, st, q, rows, d, sums, ns, A, P);
  return 1;
}

int launch_score_betae_tc(const float* q, int rows, int nbq, int d, const double* sums, int64_t ns,
                          Split A, float2* P, const Split& uv, const float2* Esum,
                          int64_t np, float* dist, int64_t ldd, float* cmin, int64_t ldc, int64_t nvalid,
                          const GemmWs* ws, cudaStream_t st) {
  launch_pdl(k_score_prep_tc, dim3(rows), dim3(128), 0, st, q, rows, d, sums, ns, A, P);
  // dist rows: one per query (NB = 2: min over the two DNF branch rows 2b, 2b + 1)
  const tc::OutDesc o{dist, ldd, Split{}, rows / nbq, np};
  if (nbq == 2)
    return 1 + tc::launch_gemm_auto(A, rows, uv, (int)np, 2 * d, o,
                                    EpiBetaScore<2>{P, Esum, rows, np, cmin, ldc, nvalid}, ws, st);
  return 1 + tc::launch_gemm_auto(A, rows, uv, (int)np, 2 * d, o,
                                  EpiBetaScore<1>{P, Esum, rows, np, cmin, ldc, nvalid}, ws, st);
}

// this translation unit's fp16x2 range flag (common.cuh range_check), read and cleared
unsigned int range_flag_score_tc() { return range_flag_take(); }

}  // namespace kgq
