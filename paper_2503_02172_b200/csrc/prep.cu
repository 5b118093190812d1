// Table and operand preparation.
//
//  * finalize: BetaE regulariser on the entity table (Q12), the shard's
//    dim-major scoring layout, and the BetaE entity-side terms, computed in fp64 and stored
//    fp32 [d][3][np]:
//      KL(Beta(ae,be) || Beta(aq,bq)) = lnB(aq,bq) + C_e + aq*U_e + bq*V_e   (per dim)
//      C_e = -lnB(ae,be) + ae psi(ae) + be psi(be) - (ae+be) psi(ae+be)
//      U_e = psi(ae+be) - psi(ae),   V_e = psi(ae+be) - psi(be)
//    (algebra of the closed-form Beta KL, Eq. 3: every lgamma/digamma argument is
//    entity-only or query-only, SURVEY §0 finding 4).
//  * per batch: the scorer's query operand planes, k-major [plane][d][rpad]; BetaE also
//    L_q = lnB(aq, bq) in fp64 (a7).
#include "common.cuh"
#include "kgq_internal.cuh"

namespace kgq {

__device__ __forceinline__ double log_beta_f64(double a, double b) {
  return lgamma(a) + lgamma(b) - lgamma(a + b);
}

__global__ void k_beta_regularize(float* ent, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    ent[i] = beta_reg(ent[i]);
}

int launch_beta_regularize(float* ent, int64_t n, cudaStream_t st) {
  k_beta_regularize<<<2048, 256, 0, st>>>(ent, n);
  return 1;
}

// tab[j][e] = ent[e0+e][j] (GQE/Q2B), zero padding for e in [ns, np).
__global__ void k_transpose_shard(const float* __restrict__ ent, int64_t e0, int64_t ns, int d,
                                  float* __restrict__ tab, int64_t np) {
  __shared__ float t[32][33];
  const int64_t eb = (int64_t)blockIdx.x * 32;
  const int jb = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t e = eb + r;
    const int j = jb + threadIdx.x;
    t[r][threadIdx.x] = (e < ns && j < d) ? ent[(e0 + e) * d + j] : 0.0f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = jb + r;
    const int64_t e = eb + threadIdx.x;
    if (j < d && e < np) tab[(int64_t)j * np + e] = t[threadIdx.x][r];
  }
}

int launch_transpose_shard(const float* ent, int64_t e0, int64_t ns, int d, int ew, float* tab,
                           int64_t np, cudaStream_t st) {
  (void)ew;
  dim3 grid((unsigned)((np + 31) / 32), (d + 31) / 32);
  k_transpose_shard<<<grid, dim3(32, 8), 0, st>>>(ent, e0, ns, d, tab, np);
  return 1;
}

// BetaE entity terms, tab[(j*3 + {0,1,2}) * np + e] = {C, U, V}; padding rows get the terms of
// Beta(1,1) (finite; never ranked: top-k reads only [0, ns)).
__global__ void k_betae_entity_terms(const float* __restrict__ ent, int64_t e0, int64_t ns, int d,
                                     float* __restrict__ tab, int64_t np) {
  __shared__ float ta[32][33], tb[32][33];
  const int64_t eb = (int64_t)blockIdx.x * 32;
  const int jb = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t e = eb + r;
    const int j = jb + threadIdx.x;
    const bool ok = e < ns && j < d;
    ta[r][threadIdx.x] = ok ? ent[(e0 + e) * 2 * d + j] : 1.0f;
    tb[r][threadIdx.x] = ok ? ent[(e0 + e) * 2 * d + d + j] : 1.0f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = jb + r;
    const int64_t e = eb + threadIdx.x;
    if (j >= d || e >= np) continue;
    const double a = ta[threadIdx.x][r], b = tb[threadIdx.x][r];
    const double pa = digamma_f64(a), pb = digamma_f64(b), pab = digamma_f64(a + b);
    const double C = -log_beta_f64(a, b) + a * pa + b * pb - (a + b) * pab;
    float* base = tab + (int64_t)j * 3 * np;
    base[e] = (float)C;
    base[np + e] = (float)(pab - pa);
    base[2 * np + e] = (float)(pab - pb);
  }
}

int launch_betae_entity_terms(const float* ent, int64_t e0, int64_t ns, int d, float* tab,
                              int64_t np, cudaStream_t st) {
  dim3 grid((unsigned)((np + 31) / 32), (d + 31) / 32);
  k_betae_entity_terms<<<grid, dim3(32, 8), 0, st>>>(ent, e0, ns, d, tab, np);
  return 1;
}

// Query operand planes for the scorer, rows r = b*nbq + br (padding rows up to a multiple of
// kRowPad get neutral values).  GQE: {q}; Q2B: {c, o}; BetaE: {L = lnB(a,b), a, b}.
__global__ void k_score_prep(int model, const float* __restrict__ q, int rows, int rows_pad,
                             int d, float* __restrict__ Qt, int64_t rpad) {
  __shared__ float t0[32][33], t1[32][33];
  const int rb = blockIdx.x * 32;
  const int jb = blockIdx.y * 32;
  const int w = model == KGQ_GQE ? d : 2 * d;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int row = rb + r;
    const int j = jb + threadIdx.x;
    const bool ok = row < rows && j < d;
    t0[r][threadIdx.x] = ok ? q[(int64_t)row * w + j] : (model == KGQ_BETAE ? 1.0f : 0.0f);
    t1[r][threadIdx.x] =
        (ok && model != KGQ_GQE) ? q[(int64_t)row * w + d + j] : (model == KGQ_BETAE ? 1.0f : 0.0f);
  }
  __syncthreads();
  const int64_t plane = (int64_t)d * rpad;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = jb + r;
    const int row = rb + threadIdx.x;
    if (j >= d || row >= rows_pad) continue;
    const float v0 = t0[threadIdx.x][r], v1 = t1[threadIdx.x][r];
    const int64_t o = (int64_t)j * rpad + row;
    if (model == KGQ_GQE) {
      Qt[o] = v0;
    } else if (model == KGQ_Q2B) {
      Qt[o] = v0;
      Qt[plane + o] = v1;
    } else {
      Qt[o] = (float)log_beta_f64((double)v0, (double)v1);
      Qt[plane + o] = v0;
      Qt[2 * plane + o] = v1;
    }
  }
}

int launch_score_prep(int model, const float* q, int B, int nbq, int d, float* Qt, int64_t rpad,
                      cudaStream_t st) {
  const int rows = B * nbq;
  const int rows_pad = (rows + kRowPad - 1) / kRowPad * kRowPad;
  dim3 grid((rows_pad + 31) / 32, (d + 31) / 32);
  k_score_prep<<<grid, dim3(32, 8), 0, st>>>(model, q, rows, rows_pad, d, Qt, rpad);
  return 1;
}

}  // namespace kgq
