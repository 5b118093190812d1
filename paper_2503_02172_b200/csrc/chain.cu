// Operator-chain kernels: anchor/relation gathers, GQE/Q2B
// translation projections, BetaE MLP input assembly, negation, attention combine.
//
// Layouts: split states S are [rows, w] with rows = branch * B + b; final query
// embeddings q are [B, nb, w] fp32 (w = d GQE, 2d Q2B [centre; offset], 2d BetaE
// [alpha; beta]).  All index reads are range-checked on the device (kgq.h: dist NaN,
// id -1, KGQ_ERANGE), with the offending id clamped to 0 so no read is out of bounds.
#include <algorithm>

#include "common.cuh"
#include "kgq_internal.cuh"

namespace kgq {

__device__ __forceinline__ int checked_id(int v, int64_t n, int32_t* err, int32_t* invalid,
                                          int row, int slot, int kind) {
  if (v < 0 || v >= n) {
    if (threadIdx.x == 0) report_range(err, invalid, row, slot, kind);
    return 0;
  }
  return v;
}

// ---- GQE / Q2B: q = E[a] + R[r0] + R[r1] + ...; Q2B offset o = 0 + R_o[r0] + ... --------
// (horizontal fusion P:146: the whole projection chain of a branch in one pass; vertical
// fusion P:148: all branches of the query in one launch, blockIdx.y = branch)
__global__ void k_translate_chain(ChainArgs a, const float* __restrict__ ent,
                                  const float* __restrict__ rel,
                                  const float* __restrict__ rel_off, int B, Split out,
                                  float* __restrict__ q) {
  pdl_grid_sync();
  const int b = blockIdx.x;
  const int br = blockIdx.y;
  const BranchPlan& P = a.br[br];
  const int d = a.d;
  const int aid = checked_id(a.anchors[(int64_t)b * a.n_a + P.anchor], a.n_entity, a.err,
                             a.invalid, b, P.anchor, 0);
  int rid[kMaxOps];
#pragma unroll
  for (int o = 0; o < kMaxOps; ++o) {
    rid[o] = (o < P.nops && P.ops[o] >= 0)
                 ? checked_id(a.rels[(int64_t)b * a.n_r + P.ops[o]], a.n_relation, a.err,
                              a.invalid, b, P.ops[o], 1)
                 : 0;
  }
  const bool q2b = a.model == KGQ_Q2B;
  const int w = q2b ? 2 * d : d;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float c = ent[(int64_t)aid * d + j];
    float off = 0.0f;
    for (int o = 0; o < P.nops; ++o) {
      c += rel[(int64_t)rid[o] * d + j];
      if (q2b) off += rel_off[(int64_t)rid[o] * d + j];
    }
    if (out.valid()) {
      const int64_t row = (int64_t)br * B + b;
      store_split(out, row * out.ld + j, c);
      if (q2b) store_split(out, row * out.ld + q2b_off(d) + j, off);
    } else {
      float* dst = q + ((int64_t)b * a.nb + br) * w;
      dst[j] = c;
      if (q2b) dst[d + j] = off;
    }
  }
}

int launch_translate_chain(const ChainArgs& a, const float* ent, const float* rel,
                           const float* rel_off, int B, Split out_split, float* out_q,
                           cudaStream_t st) {
  dim3 grid(B, a.nb);
  launch_pdl(k_translate_chain, grid, dim3(128), 0, st, a, ent, rel, rel_off, B, out_split, out_q);
  return 1;
}

// ---- BetaE MLP input: z = [alpha; beta; R[r]] (Eq. 4 var_S with the relation, Q3) -------
// Group row g*B + b of Z; source = regularised anchor row or split state row.  One warp per
// row, 16-byte loads and 8-byte plane stores (d % 4 == 0 and every row stride % 8 == 0, so
// rows are 16-byte aligned).
__device__ __forceinline__ void store_split4(const Split& z, int64_t i, float4 x) {
  uint32_t a0, b0, c0, a1, b1, c1;
  split3_pair(x.x, x.y, a0, b0, c0);
  split3_pair(x.z, x.w, a1, b1, c1);
  *reinterpret_cast<uint2*>(z.b0 + i) = make_uint2(a0, a1);
  *reinterpret_cast<uint2*>(z.b1 + i) = make_uint2(b0, b1);
  if constexpr (!kFp16x2) *reinterpret_cast<uint2*>(z.b2 + i) = make_uint2(c0, c1);
}
constexpr int kMlpInRows = 4;  // rows (warps) per block
__global__ void k_betae_mlp_input(ChainArgs a, const float* __restrict__ ent,
                                  const float* __restrict__ rel, int B, MlpGroup g, Split src,
                                  Split z, int with_rel) {
  pdl_grid_sync();
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * kMlpInRows + (threadIdx.x >> 5);
  const int gi = blockIdx.y;
  if (b >= B) return;
  const int d = a.d;
  const int rslot = g.rel_slot[gi];
  int rid = a.rels[(int64_t)b * a.n_r + rslot];
  if (rid < 0 || rid >= a.n_relation) {
    if (lane == 0) report_range(a.err, a.invalid, b, rslot, 1);
    rid = 0;
  }
  const int aslot = g.anchor_slot[gi];
  const int64_t zrow = ((int64_t)gi * B + b) * z.ld;
  if (aslot >= 0) {
    int aid = a.anchors[(int64_t)b * a.n_a + aslot];
    if (aid < 0 || aid >= a.n_entity) {
      if (lane == 0) report_range(a.err, a.invalid, b, aslot, 0);
      aid = 0;
    }
    const float4* er = reinterpret_cast<const float4*>(ent + (int64_t)aid * 2 * d);
    for (int j = lane; j < (2 * d) / 4; j += 32) store_split4(z, zrow + 4 * j, __ldg(er + j));
  } else {  // split -> split: plane copies (exact)
    const int64_t srow = (g.src_row[gi] + b) * src.ld;
    for (int p = 0; p < kSplitPlanesA; ++p) {
      const uint2* sp = reinterpret_cast<const uint2*>(src.plane(p) + srow);
      uint2* dp = reinterpret_cast<uint2*>(z.plane(p) + zrow);
      for (int j = lane; j < (2 * d) / 4; j += 32) dp[j] = sp[j];
    }
  }
  if (with_rel) {
    const float4* rr = reinterpret_cast<const float4*>(rel + (int64_t)rid * d);
    for (int j = lane; j < d / 4; j += 32) store_split4(z, zrow + 2 * d + 4 * j, __ldg(rr + j));
  }
}

int launch_betae_mlp_input(const ChainArgs& a, const float* ent, const float* rel, int B,
                           const MlpGroup& g, Split src, Split z, cudaStream_t st, bool with_rel) {
  dim3 grid((B + kMlpInRows - 1) / kMlpInRows, g.n);
  launch_pdl(k_betae_mlp_input, grid, dim3(32 * kMlpInRows), 0, st, a, ent, rel, B, g, src, z, with_rel ? 1 : 0);
  return 1;
}

// ---- mixed-structure batches: hop gather / scatter over row blocks (MixSegs) ----------------
// the last segment with dst0 <= row (segments are in ascending dst0 order): a binary search --
// the linear scan over the ~27 segments of a hop-0 batch (dynamically indexed parameter loads)
// was a large share of the per-row instructions of the one-row-per-block kernels
__device__ __forceinline__ int mix_seg_of(const MixSegs& sg, int row) {
  int lo = 0, hi = sg.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sg.s[mid].dst0 <= row) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void k_mix_gather(MixSegs sg, const float* __restrict__ ent, Split S, Split Mst, Split Z,
                             int32_t* __restrict__ rid, int d, int64_t n_entity, int n_relation,
                             int32_t* err, int32_t* invalid) {
  pdl_grid_sync();
  const int row = blockIdx.x;
  const MixSeg& g = sg.s[mix_seg_of(sg, row)];
  const int b = row - g.dst0, q = g.q0 + b;
  int r = g.rels[(int64_t)b * g.n_r + g.rslot];
  if (r < 0 || r >= n_relation) {
    if (threadIdx.x == 0) report_range(err, invalid, q, g.rslot, 1);
    r = 0;
  }
  if (threadIdx.x == 0) rid[row] = r;
  const int64_t zrow = (int64_t)row * Z.ld;
  if (g.kind == 0) {
    int a = g.anchors[(int64_t)b * g.n_a + g.aslot];
    if (a < 0 || a >= n_entity) {
      if (threadIdx.x == 0) report_range(err, invalid, q, g.aslot, 0);
      a = 0;
    }
    const float* er = ent + (int64_t)a * 2 * d;
    if ((d & 3) == 0 && (Z.ld & 7) == 0) {  // 8 elements per thread: two float4 loads, 16-byte plane stores
      for (int j = 8 * threadIdx.x; j < 2 * d; j += 8 * blockDim.x) {
        const float4 x0 = *reinterpret_cast<const float4*>(er + j), x1 = *reinterpret_cast<const float4*>(er + j + 4);
        const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        store_split8(Z, zrow + j, x);
      }
    } else {
      for (int j = threadIdx.x; j < 2 * d; j += blockDim.x) store_split(Z, zrow + j, er[j]);
    }
  } else {  // split -> split: a plane-wise copy, 16-byte vectors when aligned
    // kind 1: the state rows src0 + b of S; kind 2: the combine's output rows q0 + b of M
    const Split& src = g.kind == 1 ? S : Mst;
    const int64_t srow = ((g.kind == 1 ? g.src0 : (int64_t)g.q0) + b) * src.ld;
    if (((2 * d) & 7) == 0) {
      const int nv = (2 * d) >> 3;
      for (int p = 0; p < kSplitPlanesA; ++p) {
        const uint4* sp = reinterpret_cast<const uint4*>(src.plane(p) + srow);
        uint4* dp = reinterpret_cast<uint4*>(Z.plane(p) + zrow);
        for (int j = threadIdx.x; j < nv; j += blockDim.x) dp[j] = sp[j];
      }
    } else {
      for (int j = threadIdx.x; j < 2 * d; j += blockDim.x) {
        Z.b0[zrow + j] = src.b0[srow + j];
        Z.b1[zrow + j] = src.b1[srow + j];
        Z.b2[zrow + j] = src.b2[srow + j];
      }
    }
  }
}

int launch_mix_gather(const MixSegs& sg, int M, const float* ent, Split S, Split Mst, Split Z, int32_t* rid, int d,
                      int64_t n_entity, int n_relation, int32_t* err, int32_t* invalid, cudaStream_t st) {
  if (M <= 0) return 0;
  launch_pdl(k_mix_gather, dim3(M), dim3(128), 0, st, sg, ent, S, Mst, Z, rid, d, n_entity, n_relation, err, invalid);
  return 1;
}

__global__ void k_mix_scatter(MixSegs sg, Split src, Split S, int w) {
  pdl_grid_sync();
  const int row = blockIdx.x;
  const MixSeg& g = sg.s[mix_seg_of(sg, row)];
  const int64_t o = (g.src0 + row - g.dst0) * S.ld, i = (int64_t)row * src.ld;
  if ((w & 7) == 0) {  // 16-byte vectors (row starts are 16-byte aligned: ld % 8 == 0)
    const int nv = w >> 3;
    for (int p = 0; p < kSplitPlanesA; ++p) {
      const uint4* sp = reinterpret_cast<const uint4*>(src.plane(p) + i);
      uint4* dp = reinterpret_cast<uint4*>(S.plane(p) + o);
      for (int j = threadIdx.x; j < nv; j += blockDim.x) dp[j] = sp[j];
    }
    return;
  }
  for (int j = threadIdx.x; j < w; j += blockDim.x) {
    S.b0[o + j] = src.b0[i + j];
    S.b1[o + j] = src.b1[i + j];
    S.b2[o + j] = src.b2[i + j];
  }
}

// ---- hop-0 first projection layer from the per-entity precompute ------------------------------
// Every hop-0 MLP row starts from an anchor entity e and a relation r, so its first layer is
// W1 [x_e; R_r] + b1 = Hpre[e] + RW[r] with Hpre = X W1[:, :2d]^T + b1 precomputed for every entity
// at finalize (kgq_api.cu) -- the distributive law, as the relation term RW already is.  One block
// per row: H0[row] = split(ReLU(Hpre[e] + RW[r])), 8 columns per thread; ids range-checked as
// in k_mix_gather (a bad id: row computed from id 0, query flagged).
__global__ void k_mix_h0_pre(MixSegs sg, const float* __restrict__ Hpre, const float* __restrict__ RW,
                             int H, Split H0, int64_t n_entity, int n_relation,
                             int32_t* err, int32_t* invalid) {
  pdl_grid_sync();
  const int row = blockIdx.x;
  const MixSeg& g = sg.s[mix_seg_of(sg, row)];
  const int b = row - g.dst0, q = g.q0 + b;
  int r = g.rels[(int64_t)b * g.n_r + g.rslot];
  if (r < 0 || r >= n_relation) {
    if (threadIdx.x == 0) report_range(err, invalid, q, g.rslot, 1);
    r = 0;
  }
  int a = g.anchors[(int64_t)b * g.n_a + g.aslot];
  if (a < 0 || a >= n_entity) {
    if (threadIdx.x == 0) report_range(err, invalid, q, g.aslot, 0);
    a = 0;
  }
  const float* hp = Hpre + (int64_t)a * H;
  const float* rw = RW + (int64_t)r * H;
  const int64_t o = (int64_t)row * H0.ld;
  if ((H & 7) == 0 && (H0.ld & 7) == 0) {
    for (int j = 8 * threadIdx.x; j < H; j += 8 * blockDim.x) {
      float x[8];
#pragma unroll
      for (int h = 0; h < 8; h += 4) {
        const float4 u = __ldg(reinterpret_cast<const float4*>(hp + j + h));
        const float4 v = __ldg(reinterpret_cast<const float4*>(rw + j + h));
        x[h] = fmaxf(u.x + v.x, 0.0f);
        x[h + 1] = fmaxf(u.y + v.y, 0.0f);
        x[h + 2] = fmaxf(u.z + v.z, 0.0f);
        x[h + 3] = fmaxf(u.w + v.w, 0.0f);
      }
      store_split8(H0, o + j, x);
    }
  } else {
    for (int j = threadIdx.x; j < H; j += blockDim.x) store_split(H0, o + j, fmaxf(hp[j] + rw[j], 0.0f));
  }
}

int launch_mix_h0_pre(const MixSegs& sg, int M, const float* Hpre, const float* RW, int H,
                      Split H0, int64_t n_entity, int n_relation, int32_t* err, int32_t* invalid, cudaStream_t st) {
  if (M <= 0) return 0;
  // one thread per 8 columns: H = 1600 -> 200 threads, a 224-thread block (89% of its lanes busy)
  const int threads = std::min(256, std::max(32, ((H / 8 + 31) / 32) * 32));
  launch_pdl(k_mix_h0_pre, dim3(M), dim3(threads), 0, st, sg, Hpre, RW, H, H0, n_entity, n_relation, err,
             invalid);
  return 1;
}

int launch_mix_scatter(const MixSegs& sg, int M, Split src, Split S, int w, cudaStream_t st) {
  if (M <= 0) return 0;
  launch_pdl(k_mix_scatter, dim3(M), dim3(128), 0, st, sg, src, S, w);
  return 1;
}

// ---- relation term of the first projection layer: RW[r, n] = sum_k W[n, col0 + k] R[r, k] ----
// fp64 accumulation, once per table load (finalize).  Block (r, 128 outputs); R[r] staged in smem.
__global__ void k_relation_term(const float* __restrict__ R, int d, const float* __restrict__ W, int64_t ldw,
                                int col0, int H, float* __restrict__ RW) {
  extern __shared__ double rr[];
  const int r = blockIdx.x;
  for (int k = threadIdx.x; k < d; k += blockDim.x) rr[k] = R[(int64_t)r * d + k];
  __syncthreads();
  const int n = blockIdx.y * blockDim.x + threadIdx.x;
  if (n >= H) return;
  const float* w = W + (int64_t)n * ldw + col0;
  double s = 0.0;
  for (int k = 0; k < d; ++k) s += (double)w[k] * rr[k];
  RW[(int64_t)r * H + n] = (float)s;
}

int launch_relation_term(const float* R, int n_relation, int d, const float* W, int64_t ldw, int col0, int H,
                         float* RW, cudaStream_t st) {
  k_relation_term<<<dim3(n_relation, (H + 127) / 128), 128, d * sizeof(double), st>>>(R, d, W, ldw, col0, H, RW);
  return 1;
}

// ---- BetaE Eq.-4 literal terminal: softmax over the 2d outputs, max(., 1e-6) -----------
__global__ void k_softmax_terminal(const float* __restrict__ T, int64_t ldt, int w, Split out,
                                   int64_t out_row0, int neg0, int neg1) {
  pdl_grid_sync();
  const int r = blockIdx.x;
  const float* t = T + (int64_t)r * ldt;
  __shared__ float red[32];
  float m = -INFINITY;
  for (int j = threadIdx.x; j < w; j += blockDim.x) m = fmaxf(m, t[j]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  m = red[0];
  __syncthreads();
  float s = 0.0f;
  for (int j = threadIdx.x; j < w; j += blockDim.x) s += expf(t[j] - m);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = 1.0f / red[0];
  const bool neg = r >= neg0 && r < neg1;
  for (int j = threadIdx.x; j < w; j += blockDim.x) {
    float y = fmaxf(expf(t[j] - m) * inv, 1e-6f);
    if (neg) y = 1.0f / y;
    store_split(out, (out_row0 + r) * out.ld + j, y);
  }
}

int launch_softmax_terminal(const float* T, int64_t ldt, int M, int w, Split out,
                            int64_t out_row0, int neg0, int neg1, cudaStream_t st) {
  launch_pdl(k_softmax_terminal, dim3(M), dim3(256), 0, st, T, ldt, w, out, out_row0, neg0, neg1);
  return 1;
}

// ---- negation (Q5): alpha -> 1/alpha, beta -> 1/beta, in place on split rows -----------
__global__ void k_negate(Split x, int64_t r0, int64_t nrows, int w) {
  pdl_grid_sync();
  const int64_t n = nrows * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = r0 + i / w, j = i % w;
    const int64_t o = r * x.ld + j;
    store_split(x, o, 1.0f / load_split(x, o));
  }
}

int launch_negate(Split x, int64_t r0, int64_t r1, int w, cudaStream_t st) {
  const int64_t n = (r1 - r0) * w;
  const int blocks = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  launch_pdl(k_negate, dim3(blocks), dim3(256), 0, st, x, r0, r1 - r0, w);
  return 1;
}

// ---- Q2B offset gate input: mean over branches of ReLU(V1 o_i + c1) --------------------
__global__ void k_branch_mean(const float* __restrict__ T, int64_t ldt, int nb, int B, int d,
                              Split out) {
  pdl_grid_sync();
  const int b = blockIdx.x;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float s = 0.0f;
    for (int i = 0; i < nb; ++i) s += T[((int64_t)i * B + b) * ldt + j];
    store_split(out, (int64_t)b * out.ld + j, s / (float)nb);
  }
}

int launch_branch_mean(const float* T, int64_t ldt, int nb, int B, int d, Split out,
                       cudaStream_t st) {
  launch_pdl(k_branch_mean, dim3(B), dim3(128), 0, st, T, ldt, nb, B, d, out);
  return 1;
}

// ---- attention combine (Q6): a_i = softmax_i(logit_i) per dim; out = sum_i a_i x_i --------
// GQE: x = state[:, :d].  BetaE: the same a_i weights alpha (cols [0,d)) and beta ([d,2d)).
// Q2B: centre as GQE; offset o = min_i o_i * sigmoid(G) (gate logits G [B, d]).
// Post projection (ip): + R[r] on the centre (GQE/Q2B; Q2B offset + R_o[r]).
__device__ __forceinline__ float4 load_split4(const Split& s, int64_t i) {  // i % 4 == 0
  const uint2 a = *reinterpret_cast<const uint2*>(s.b0 + i);
  const uint2 b = *reinterpret_cast<const uint2*>(s.b1 + i);
  if constexpr (kFp16x2) {
    const float2 h0 = __half22float2(*reinterpret_cast<const __half2*>(&a.x));
    const float2 h1 = __half22float2(*reinterpret_cast<const __half2*>(&a.y));
    const float2 l0 = __half22float2(*reinterpret_cast<const __half2*>(&b.x));
    const float2 l1 = __half22float2(*reinterpret_cast<const __half2*>(&b.y));
    return make_float4(h0.x + l0.x * kLoInv, h0.y + l0.y * kLoInv, h1.x + l1.x * kLoInv, h1.y + l1.y * kLoInv);
  }
  const uint2 c = *reinterpret_cast<const uint2*>(s.b2 + i);
  auto lo = [](uint32_t u) { return __uint_as_float(u << 16); };
  auto hi = [](uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); };
  return make_float4((lo(a.x) + lo(b.x)) + lo(c.x), (hi(a.x) + hi(b.x)) + hi(c.x),
                     (lo(a.y) + lo(b.y)) + lo(c.y), (hi(a.y) + hi(b.y)) + hi(c.y));
}
// One query per block; each thread owns 4 consecutive dimensions (d % 4 == 0, all row strides
// % 8 == 0: 16-byte logit / gate / relation loads, 8-byte plane loads and stores).
__device__ __forceinline__ void combine_query(const CombineArgs& c, const Split& S, const float* __restrict__ logits,
                                              const float* __restrict__ gate, const Split& out,
                                              float* __restrict__ q, int b) {
  const int d = c.d;
  const int B = c.B;
  const int nb = c.nb;
  int rid = 0;
  if (c.post_slot >= 0)
    rid = checked_id(c.rels[(int64_t)b * c.n_r + c.post_slot], c.n_relation, c.err, c.invalid,
                     b, c.post_slot, 1);
  for (int j = 4 * threadIdx.x; j < d; j += 4 * blockDim.x) {
    float l[kMaxBranches][4];
    float m[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int i = 0; i < kMaxBranches; ++i) {  // unrolled: l stays in registers
      if (i >= nb) break;
      const float4 v = *reinterpret_cast<const float4*>(logits + ((int64_t)i * B + b) * c.ldl + j);
      l[i][0] = v.x; l[i][1] = v.y; l[i][2] = v.z; l[i][3] = v.w;
#pragma unroll
      for (int u = 0; u < 4; ++u) m[u] = fmaxf(m[u], l[i][u]);
    }
    float sum[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int i = 0; i < kMaxBranches; ++i)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i >= nb) break;
        l[i][u] = expf(l[i][u] - m[u]);
        sum[u] += l[i][u];
      }
    float inv[4], x0[4] = {0.0f, 0.0f, 0.0f, 0.0f}, x1[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    float omin[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
#pragma unroll
    for (int u = 0; u < 4; ++u) inv[u] = 1.0f / sum[u];
#pragma unroll
    for (int i = 0; i < kMaxBranches; ++i) {
      if (i >= nb) break;
      const int64_t row = ((int64_t)i * B + b) * S.ld;
      const float4 s0 = load_split4(S, row + j);
      const float v0[4] = {s0.x, s0.y, s0.z, s0.w};
      float v1[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      if (c.model == KGQ_BETAE) {
        const float4 s1 = load_split4(S, row + d + j);
        v1[0] = s1.x; v1[1] = s1.y; v1[2] = s1.z; v1[3] = s1.w;
      }
      if (c.model == KGQ_Q2B) {
        const float4 o = load_split4(S, row + q2b_off(d) + j);
        const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) omin[u] = fminf(omin[u], ov[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float a = l[i][u] * inv[u];
        x0[u] += a * v0[u];
        if (c.model == KGQ_BETAE) x1[u] += a * v1[u];
      }
    }
    if (c.model == KGQ_Q2B) {
      const float4 g = *reinterpret_cast<const float4*>(gate + (int64_t)b * c.ldg + j);
      const float gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) x1[u] = omin[u] * (1.0f / (1.0f + expf(-gv[u])));
    }
    if (c.post_slot >= 0) {
      const float4 r0 = *reinterpret_cast<const float4*>(c.rel + (int64_t)rid * d + j);
      x0[0] += r0.x; x0[1] += r0.y; x0[2] += r0.z; x0[3] += r0.w;
      if (c.model == KGQ_Q2B) {
        const float4 r1 = *reinterpret_cast<const float4*>(c.rel_off + (int64_t)rid * d + j);
        x1[0] += r1.x; x1[1] += r1.y; x1[2] += r1.z; x1[3] += r1.w;
      }
    }
    if (c.negate_out) {  // De Morgan union: N(I(...)), alpha -> 1/alpha, beta -> 1/beta (Q5)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x0[u] = 1.0f / x0[u];
        x1[u] = 1.0f / x1[u];
      }
    }
    const bool two = c.model != KGQ_GQE;
    if (out.valid()) {
      store_split4(out, (int64_t)b * out.ld + j, make_float4(x0[0], x0[1], x0[2], x0[3]));
      if (two) store_split4(out, (int64_t)b * out.ld + d + j, make_float4(x1[0], x1[1], x1[2], x1[3]));
    } else {
      float* dst = q + (int64_t)b * (two ? 2 * d : d);
      *reinterpret_cast<float4*>(dst + j) = make_float4(x0[0], x0[1], x0[2], x0[3]);
      if (two) *reinterpret_cast<float4*>(dst + d + j) = make_float4(x1[0], x1[1], x1[2], x1[3]);
    }
  }
}

__global__ void k_attention_combine(CombineArgs c, Split S, const float* __restrict__ logits,
                                    const float* __restrict__ gate, Split out,
                                    float* __restrict__ q) {
  pdl_grid_sync();
  combine_query(c, S, logits, gate, out, q, blockIdx.x);
}

// Mixed batches: the attention combine of every intersection group in one launch.  Block i is
// query i of the concatenation of the groups (MixCombine::q_begin prefix).
// Register cap: 16 resident 128-thread blocks per SM (32 registers, ~100 bytes spilled) instead of
// ~10 at 48 registers -- more queries in flight for the latency-bound loads and exp / divide
// chains: 47.4 -> 31.2 us per C2 step (ncu; 12 blocks / 40 registers: 34.1 us)
#ifndef KGQ_COMBINE_MINB
#define KGQ_COMBINE_MINB 16
#endif
__global__ void __launch_bounds__(128, KGQ_COMBINE_MINB)
    k_mix_combine(MixCombine mc, Split S, const float* __restrict__ logits, int64_t ldl, Split Mst) {
  pdl_grid_sync();
  const int i = blockIdx.x;
  int g = 0;
  while (g + 1 < mc.n && mc.g[g + 1].q_begin <= i) ++g;
  const MixCombine::Group& G = mc.g[g];
  const Split src = S.at(G.srow0);
  const Split out = G.to_m ? Mst.at(G.q0) : src;
  combine_query(G.c, src, logits + G.srow0 * ldl, nullptr, out, nullptr, i - G.q_begin);
}

int launch_mix_combine(const MixCombine& mc, int total, Split S, const float* logits, int64_t ldl, Split Mst,
                       cudaStream_t st) {
  if (total <= 0) return 0;
  launch_pdl(k_mix_combine, dim3(total), dim3(128), 0, st, mc, S, logits, ldl, Mst);
  return 1;
}

int launch_attention_combine(const CombineArgs& c, Split S, const float* logits,
                             const float* gate, Split out_split, float* out_q, cudaStream_t st) {
  launch_pdl(k_attention_combine, dim3(c.B), dim3(128), 0, st, c, S, logits, gate, out_split, out_q);
  return 1;
}

// ---- split state rows -> q[b, br, :] ---------------------------------------------------
__global__ void k_state_to_q(Split S, int nb, int B, int w, float* __restrict__ q) {
  pdl_grid_sync();
  const int b = blockIdx.x, br = blockIdx.y;
  for (int j = threadIdx.x; j < w; j += blockDim.x)
    q[((int64_t)b * nb + br) * w + j] = load_split(S, ((int64_t)br * B + b) * S.ld + j);
}

int launch_state_to_q(Split S, int nb, int B, int w, float* q, cudaStream_t st) {
  launch_pdl(k_state_to_q, dim3(B, nb), dim3(128), 0, st, S, nb, B, w, q);
  return 1;
}

// ---- split copy (weights -> tensor-core operands) --------------------------------------
__global__ void k_split_copy(const float* __restrict__ src, int64_t n, Split dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    store_split_w(dst, i, src[i]);
}

int launch_split_copy(const float* src, int64_t n, Split dst, cudaStream_t st) {
  k_split_copy<<<1024, 256, 0, st>>>(src, n, dst);
  return 1;
}

// [rows, cols] fp32 with row stride lds -> split planes with row stride dst.ld (>= cols)
// weight form (store_split_w: the GEMMs' W operand) or, act = true, the activation form
__global__ void k_split_copy_rows(const float* __restrict__ src, int64_t lds, int64_t rows, int cols, Split dst,
                                  bool act) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (i / cols) * dst.ld + i % cols;
    const float x = src[(i / cols) * lds + i % cols];
    if (act)
      store_split(dst, o, x);
    else
      store_split_w(dst, o, x);
  }
}

int launch_split_copy_rows(const float* src, int64_t rows, int cols, Split dst, cudaStream_t st, int64_t lds,
                           bool act) {
  k_split_copy_rows<<<1024, 256, 0, st>>>(src, lds > 0 ? lds : cols, rows, cols, dst, act);
  return 1;
}

__global__ void k_empty() {}
int launch_empty(cudaStream_t st) {
  k_empty<<<148, 128, 0, st>>>();
  return 1;
}

// this translation unit's fp16x2 range flag (common.cuh range_check), read and cleared
unsigned int range_flag_chain() { return range_flag_take(); }

}  // namespace kgq
