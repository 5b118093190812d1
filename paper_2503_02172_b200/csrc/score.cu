// Entity scorer (SURVEY §8(a) a6 + a7): distance of every query embedding to every entity of
// this rank's shard, min over DNF branches (union, Eq. 1), written as dist[b, e].
//
//   GQE   sum_d |e - q|                                   2 FP32 ops per (q, e, d), issued as
//                                                         1 packed FADD2 per (q, e, d) (l1_pair)
//   Q2B   sum_d |e-c| - (1-cen) sum_d min(|e-c|, o)         4 ops  (== sum ReLU(|e-c|-o) +
//                                                                   cen * sum min(|e-c|, o)):
//                                                         1.5 FADD2 + 1 FMNMX per (q, e, d)
//   BetaE sum_d |L_q + C_e + a_q U_e + b_q V_e|             4 ops  (== sum_d |KL(e || q)|)
//
// Register-tiled SIMT "GEMM-like" kernel: the inner op is not a dot product, so tensor cores do
// not apply.  CTA tile 64 query rows x 128 entities, 256 threads, 4x8
// per thread; k-major operand planes staged through shared memory by cp.async, two stages.
// Query rows are (b, branch) pairs; for 2u/up (NB = 2) a thread owns both branches of its
// queries and takes the min in registers (a6 fused into a7).
#include "common.cuh"
#include "kgq_internal.cuh"

namespace kgq {

namespace {
constexpr int TQ = 64, TE = 128, DK = 16;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Packed FP32 pairs (sm_100 FADD2): (a0, a1) += (|e0 - q|, |e1 - q|) is two instructions for two
// entities -- a sub with q broadcast as a scalar operand, then an add whose |.| is an operand
// modifier -- instead of four scalar ones.  The same two RN operations per element in the same
// order as fabsf(e - q) then +=, so results are bit-identical to the scalar form.
__device__ __forceinline__ float2 fadd2(const float2 a, const float2 b) {
  float2 c;
  asm("{\n.reg .b64 x, y, z;\nmov.b64 x, {%2, %3};\nmov.b64 y, {%4, %5};\n"
      "add.rn.f32x2 z, x, y;\nmov.b64 {%0, %1}, z;\n}\n"
      : "=f"(c.x), "=f"(c.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return c;
}
__device__ __forceinline__ float2 fsub2(const float2 a, const float2 b) {
  float2 c;
  asm("{\n.reg .b64 x, y, z;\nmov.b64 x, {%2, %3};\nmov.b64 y, {%4, %5};\n"
      "sub.rn.f32x2 z, x, y;\nmov.b64 {%0, %1}, z;\n}\n"
      : "=f"(c.x), "=f"(c.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return c;
}
// GQE: acc += |e - q| for an entity pair.  Q2B (BOX): also acc2 += min(|e - c|, o) -- the min
// stays scalar (FMNMX, on the ALU pipe next to the FADD2s on the FMA pipe).
template <bool BOX>
__device__ __forceinline__ void l1_pair(float& a0, float& a1, float& b0, float& b1, float e0, float e1, float q,
                                        float o) {
  const float2 t = fsub2(make_float2(e0, e1), make_float2(q, q));
  const float2 at = make_float2(fabsf(t.x), fabsf(t.y));
  const float2 a = fadd2(make_float2(a0, a1), at);
  a0 = a.x;
  a1 = a.y;
  if (BOX) {
    const float2 b = fadd2(make_float2(b0, b1), make_float2(fminf(at.x, o), fminf(at.y, o)));
    b0 = b.x;
    b1 = b.y;
  }
}

template <int MODEL>
struct Planes {
  static constexpr int NQ = MODEL == KGQ_GQE ? 1 : (MODEL == KGQ_Q2B ? 2 : 3);
  static constexpr int NE = MODEL == KGQ_BETAE ? 3 : 1;
};

template <int MODEL, int NB>
__global__ void __launch_bounds__(256, 2)
    k_score(const float* __restrict__ Qt, int64_t rpad, const float* __restrict__ tab, int64_t np,
            int d, float cen, float* __restrict__ dist, int64_t ldd, int B) {
  constexpr int NQ = Planes<MODEL>::NQ, NE = Planes<MODEL>::NE;
  extern __shared__ __align__(16) float smem[];
  float* Qs = smem;                          // [2][NQ][DK][TQ]
  float* Es = smem + 2 * NQ * DK * TQ;       // [2][NE][DK][TE]
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t e0 = (int64_t)blockIdx.x * TE;
  const int64_t r0 = (int64_t)blockIdx.y * TQ;
  const int64_t qplane = (int64_t)d * rpad;
  // E tab plane p of dim j: GQE/Q2B tab + j*np; BetaE tab + (j*3+p)*np
  auto eptr = [&](int p, int j) -> const float* {
    return NE == 1 ? tab + (int64_t)j * np : tab + ((int64_t)j * 3 + p) * np;
  };
  auto load_stage = [&](int buf, int j0) {
    // Q: NQ planes x DK x TQ floats = NQ * 256 float4, one per thread per plane
#pragma unroll
    for (int p = 0; p < NQ; ++p) {
      const int k = tid >> 4, c = (tid & 15) * 4;
      const int j = j0 + k;
      const float* g = Qt + p * qplane + (int64_t)(j < d ? j : 0) * rpad + r0 + c;
      cp_async16(Qs + ((buf * NQ + p) * DK + k) * TQ + c, g, j < d);
    }
    // E: NE planes x DK x TE floats = NE * 512 float4, two per thread per plane
#pragma unroll
    for (int p = 0; p < NE; ++p)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int idx = tid + h * 256;
        const int k = idx >> 5, c = (idx & 31) * 4;
        const int j = j0 + k;
        const float* g = eptr(p, j < d ? j : 0) + e0 + c;
        cp_async16(Es + ((buf * NE + p) * DK + k) * TE + c, g, j < d);
      }
  };

  float acc[4][8], acc2[4][8];  // acc2: Q2B inside sums (dead code otherwise)
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = acc2[i][j] = 0.0f;

  const int nst = (d + DK - 1) / DK;
  load_stage(0, 0);
  cp_async_commit();
  for (int s = 0; s < nst; ++s) {
    const int buf = s & 1;
    if (s + 1 < nst) {
      load_stage(buf ^ 1, (s + 1) * DK);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < DK; ++k) {
      float q[NQ][4], e[NE][8];
#pragma unroll
      for (int p = 0; p < NQ; ++p) {
        const float4 v = *reinterpret_cast<const float4*>(Qs + ((buf * NQ + p) * DK + k) * TQ + ty * 4);
        q[p][0] = v.x; q[p][1] = v.y; q[p][2] = v.z; q[p][3] = v.w;
      }
#pragma unroll
      for (int p = 0; p < NE; ++p) {
        const float* row = Es + ((buf * NE + p) * DK + k) * TE;
        const float4 v0 = *reinterpret_cast<const float4*>(row + tx * 4);
        const float4 v1 = *reinterpret_cast<const float4*>(row + 64 + tx * 4);
        e[p][0] = v0.x; e[p][1] = v0.y; e[p][2] = v0.z; e[p][3] = v0.w;
        e[p][4] = v1.x; e[p][5] = v1.y; e[p][6] = v1.z; e[p][7] = v1.w;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (MODEL != KGQ_BETAE) {
            if (j % 2 == 0)
              l1_pair<MODEL == KGQ_Q2B>(acc[i][j], acc[i][j + 1], acc2[i][j], acc2[i][j + 1], e[0][j], e[0][j + 1],
                                        q[0][i], MODEL == KGQ_Q2B ? q[1][i] : 0.0f);
          } else {
            float t = e[0][j] + q[0][i];
            t = fmaf(q[1][i], e[1][j], t);
            t = fmaf(q[2][i], e[2][j], t);
            acc[i][j] += fabsf(t);
          }
        }
    }
    __syncthreads();
  }

  float res[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      res[i][j] = MODEL == KGQ_Q2B ? fmaf(-(1.0f - cen), acc2[i][j], acc[i][j]) : acc[i][j];

  constexpr int QPT = 4 / NB;  // queries per thread
#pragma unroll
  for (int u = 0; u < QPT; ++u) {
    const int64_t b = (r0 + ty * 4) / NB + u;
    if (b >= B) continue;
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      o[j] = res[u * NB][j];
      if (NB == 2) o[j] = fminf(o[j], res[u * NB + 1][j]);
    }
    float* drow = dist + b * ldd + e0;
    *reinterpret_cast<float4*>(drow + tx * 4) = make_float4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<float4*>(drow + 64 + tx * 4) = make_float4(o[4], o[5], o[6], o[7]);
  }
}

// ---- small-batch streaming variant (SURVEY §8(d) C5a latency regime: B*NB <= 16) ----------
// The tiled kernel pads the query tile to 64 rows; at B <= ~16 the sweep is HBM-bound
// (ridge ~11 queries for GQE, ~17 for BetaE-CUV), so here every thread streams 4 consecutive
// entities of the dim-major table with 16-byte loads (a warp reads 512 contiguous bytes per
// dim and plane) while the <= 16 query rows sit in shared memory and are read as broadcasts.
// Per (q, e, d) it evaluates exactly the expression of k_score, in the same order, so both
// variants return bit-identical distances.
// Tuned on the C5a sweep (2M entities, d 400; r02_stream_ab): GQE 1p B = 8 0.48 -> 0.79 of the
// measured HBM bandwidth with 16-byte query loads, a register cap of two CTAs per SM for the
// <= 8-row GQE variants and 8 dims of loads in flight (unroll 8); B = 1 stays at ~1.0.
#ifndef KGQ_STREAM_MINB  // min resident CTAs of the GQE <= 8-row variants (register cap)
#define KGQ_STREAM_MINB 2
#endif
#ifndef KGQ_STREAM_UNROLL
#define KGQ_STREAM_UNROLL 8
#endif
#ifndef KGQ_STREAM_QVEC
#define KGQ_STREAM_QVEC 1
#endif
constexpr int kStreamUnroll = KGQ_STREAM_UNROLL;
template <int MODEL, int NB, int QB>
__global__ void __launch_bounds__(256, MODEL == KGQ_GQE ? KGQ_STREAM_MINB : 1)
    k_score_stream(const float* __restrict__ Qt, int64_t rpad, const float* __restrict__ tab,
                   int64_t np, int d, float cen, float* __restrict__ dist, int64_t ldd, int B) {
  constexpr int NQ = Planes<MODEL>::NQ, NE = Planes<MODEL>::NE, R = QB * NB;
  extern __shared__ __align__(16) float qs[];  // [d][NQ][R]
  const int64_t qplane = (int64_t)d * rpad;
  for (int i = threadIdx.x; i < d * NQ * R; i += blockDim.x) {
    const int r = i % R, p = (i / R) % NQ, j = i / (R * NQ);
    qs[i] = Qt[p * qplane + (int64_t)j * rpad + r];
  }
  __syncthreads();
  const int64_t ngroups = np / 4;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = g * 4;
    float acc[R][4], acc2[R][4];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[r][i] = acc2[r][i] = 0.0f;
#pragma unroll kStreamUnroll
    for (int j = 0; j < d; ++j) {
      float e[NE][4];
#pragma unroll
      for (int p = 0; p < NE; ++p) {
        const float* src = NE == 1 ? tab + (int64_t)j * np + e0 : tab + ((int64_t)j * 3 + p) * np + e0;
        const float4 v = __ldg(reinterpret_cast<const float4*>(src));
        e[p][0] = v.x; e[p][1] = v.y; e[p][2] = v.z; e[p][3] = v.w;
      }
      const float* qjp = qs + j * NQ * R;
      float qj[NQ * R];  // this dim's query operands (16-byte broadcast loads when R % 4 == 0)
      if constexpr (KGQ_STREAM_QVEC && (NQ * R) % 4 == 0) {
#pragma unroll
        for (int i = 0; i < NQ * R; i += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(qjp + i);
          qj[i] = t4.x; qj[i + 1] = t4.y; qj[i + 2] = t4.z; qj[i + 3] = t4.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < NQ * R; ++i) qj[i] = qjp[i];
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (MODEL != KGQ_BETAE) {
            if (i % 2 == 0)
              l1_pair<MODEL == KGQ_Q2B>(acc[r][i], acc[r][i + 1], acc2[r][i], acc2[r][i + 1], e[0][i], e[0][i + 1],
                                        qj[r], MODEL == KGQ_Q2B ? qj[R + r] : 0.0f);
          } else {
            float t = e[0][i] + qj[r];
            t = fmaf(qj[R + r], e[1][i], t);
            t = fmaf(qj[2 * R + r], e[2][i], t);
            acc[r][i] += fabsf(t);
          }
        }
      }
    }
#pragma unroll
    for (int b = 0; b < QB; ++b) {
      if (b >= B) break;
      float o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        o[i] = MODEL == KGQ_Q2B ? fmaf(-(1.0f - cen), acc2[b * NB][i], acc[b * NB][i]) : acc[b * NB][i];
        if (NB == 2) {
          const float o1 = MODEL == KGQ_Q2B ? fmaf(-(1.0f - cen), acc2[b * NB + 1][i], acc[b * NB + 1][i])
                                            : acc[b * NB + 1][i];
          o[i] = fminf(o[i], o1);
        }
      }
      *reinterpret_cast<float4*>(dist + (int64_t)b * ldd + e0) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
}

// ---- BetaE small-batch streaming scorer on the centred (u, v) table -------------------------
// The per-dimension KL splits into query-only, entity-only and bilinear terms (score_tc.cu):
//   dist(q, e) = P_q + E_e + sum_d (a_qd u_ed + b_qd v_ed),  u = U - mean(U), v = V - mean(V),
// with P_q, E_e computed in fp64 and held as fp32 (hi, lo) pairs, and sum_d |KL_d| = sum_d KL_d
// (each KL_d >= 0).  So the sweep streams only u and v (8 bytes per entity and dimension instead
// of the C, U, V planes' 12) and does two fused multiply-adds per (query row, entity, dim), as
// packed FFMA2 over entity pairs (fma.rn.f32x2): one instruction per (q, e, d).  Thread = four
// consecutive entities (two 16-byte loads per dimension, coalesced 512 bytes per warp and
// plane); the query rows' (a, a, b, b) quadruples sit in shared memory and are read as 16-byte
// broadcasts.  Epilogue = the tensor-core scorer's: (P_hi + E_hi) + ((P_lo + E_lo) + acc).
__device__ __forceinline__ void ffma2(float2& c, const float2 a, const float2 b) {
  asm("{\n.reg .b64 x, y, z;\nmov.b64 x, {%2, %3};\nmov.b64 y, {%4, %5};\nmov.b64 z, {%0, %1};\n"
      "fma.rn.f32x2 z, x, y, z;\nmov.b64 {%0, %1}, z;\n}\n"
      : "+f"(c.x), "+f"(c.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
}

#ifndef KGQ_UV_UNROLL  // dims of (u, v) loads in flight per thread (r02_stream_ab2: 2 / 4 / 8 ->
#define KGQ_UV_UNROLL 8   // 2u B = 8 at 0.49 / 0.63 / 0.68 of the measured HBM bandwidth)
#endif
#ifndef KGQ_UV_MINB
#define KGQ_UV_MINB 2
#endif
constexpr int kUvUnroll = KGQ_UV_UNROLL;
// Thread = 4 consecutive entities x RS query rows.  With 16 rows (2u at B = 8) the two half-warps
// take rows 0-7 and 8-15 of the same 16 entity groups (their u, v loads hit the same 256 bytes:
// one request), so a thread keeps 32 accumulators instead of 64.
template <int NB, int QB>
__global__ void __launch_bounds__(256, KGQ_UV_MINB)
    k_score_uv_stream(Split A, const float2* __restrict__ P, const float* __restrict__ uvT, const float2* __restrict__ E,
                      int64_t np, int d, float* __restrict__ dist, int64_t ldd, int B) {
  constexpr int R = QB * NB;
  constexpr int HALVES = R >= 16 ? 2 : 1;
  constexpr int RS = R / HALVES;      // rows per thread
  constexpr int GPW = 32 / HALVES;    // entity groups per warp
  static_assert(R % 2 == 0 || R == 1, "query rows are read in pairs");
  extern __shared__ __align__(16) float2 qab[];  // [d][R] = (a, b); ptxas broadcasts a / b into FFMA2
  pdl_grid_sync();
  const int rows = B * NB;
  for (int i = threadIdx.x; i < d * R; i += blockDim.x) {
    const int r = i % R, j = i / R;
    float a = 0.0f, b = 0.0f;
    if (r < rows) {
      a = load_split(A, (int64_t)r * A.ld + j);
      b = load_split(A, (int64_t)r * A.ld + d + j);
    }
    qab[i] = make_float2(a, b);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, half = HALVES == 2 ? lane >> 4 : 0;
  const int r0 = half * RS;
  const int64_t ngroups = np / 4;
  const int64_t gpb = (int64_t)(blockDim.x >> 5) * GPW;  // entity groups per CTA pass
  for (int64_t gb = (int64_t)blockIdx.x * gpb; gb < ngroups; gb += (int64_t)gridDim.x * gpb) {
    const int64_t g = gb + (threadIdx.x >> 5) * GPW + (lane % GPW);
    if (g >= ngroups) continue;
    const int64_t e0 = g * 4;
    float2 acc[RS][2];
#pragma unroll
    for (int r = 0; r < RS; ++r) acc[r][0] = acc[r][1] = make_float2(0.0f, 0.0f);
    const float* up = uvT + e0;
#pragma unroll kUvUnroll
    for (int j = 0; j < d; ++j) {
      const float4 u4 = __ldg(reinterpret_cast<const float4*>(up + (int64_t)(2 * j) * np));
      const float4 v4 = __ldg(reinterpret_cast<const float4*>(up + (int64_t)(2 * j + 1) * np));
      const float2 u[2] = {make_float2(u4.x, u4.y), make_float2(u4.z, u4.w)};
      const float2 v[2] = {make_float2(v4.x, v4.y), make_float2(v4.z, v4.w)};
      const float2* qj = qab + j * R + r0;
      if constexpr (RS % 2 == 0) {
#pragma unroll
        for (int r = 0; r < RS; r += 2) {  // two rows' (a, b) per 16-byte broadcast
          const float4 q = *reinterpret_cast<const float4*>(qj + r);
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            ffma2(acc[r][p], u[p], make_float2(q.x, q.x));
            ffma2(acc[r][p], v[p], make_float2(q.y, q.y));
            ffma2(acc[r + 1][p], u[p], make_float2(q.z, q.z));
            ffma2(acc[r + 1][p], v[p], make_float2(q.w, q.w));
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < RS; ++r) {
          const float2 q = qj[r];
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            ffma2(acc[r][p], u[p], make_float2(q.x, q.x));
            ffma2(acc[r][p], v[p], make_float2(q.y, q.y));
          }
        }
      }
    }
    float2 ee[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) ee[i] = __ldg(E + e0 + i);
#pragma unroll
    for (int bl = 0; bl < RS / NB; ++bl) {
      const int b = r0 / NB + bl;
      if (b >= B) break;
      float o[4];
#pragma unroll
      for (int br = 0; br < NB; ++br) {
        const float2 p = __ldg(P + b * NB + br);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float s = (i & 1) ? acc[bl * NB + br][i >> 1].y : acc[bl * NB + br][i >> 1].x;
          const float v = (p.x + ee[i].x) + ((p.y + ee[i].y) + s);
          o[i] = br == 0 ? v : fminf(o[i], v);
        }
      }
      *reinterpret_cast<float4*>(dist + (int64_t)b * ldd + e0) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
}

template <int NB, int QB>
void launch_uv_stream_t(const Split& A, const float2* P, const float* uvT, const float2* E, int64_t np, int d,
                        float* dist, int64_t ldd, int B, cudaStream_t st) {
  constexpr int HALVES = QB * NB >= 16 ? 2 : 1;
  const size_t smem = (size_t)d * QB * NB * sizeof(float2);
  static SmemAttr attr;
  smem_attr_once(k_score_uv_stream<NB, QB>, (int)smem, attr);
  const int64_t gpb = 8 * 32 / HALVES;
  const int64_t want = (np / 4 + gpb - 1) / gpb;
  const int grid = (int)(want < 148 * 8 ? want : 148 * 8);
  launch_pdl(k_score_uv_stream<NB, QB>, dim3(grid), dim3(256), smem, st, A, P, uvT, E, np, d, dist, ldd, B);
}

template <int MODEL, int NB, int QB>
void launch_stream_t(const float* Qt, int64_t rpad, const float* tab, int64_t np, int d, float cen,
                     float* dist, int64_t ldd, int B, cudaStream_t st) {
  constexpr int NQ = Planes<MODEL>::NQ, R = QB * NB;
  const size_t smem = (size_t)d * NQ * R * sizeof(float);
  cudaFuncSetAttribute(k_score_stream<MODEL, NB, QB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t groups = np / 4;
  const int64_t want = (groups + 255) / 256;
  const int grid = (int)(want < 148 * 8 ? want : 148 * 8);
  k_score_stream<MODEL, NB, QB><<<grid, 256, smem, st>>>(Qt, rpad, tab, np, d, cen, dist, ldd, B);
}

template <int MODEL, int NB>
void launch_stream(const float* Qt, int64_t rpad, const float* tab, int64_t np, int d, float cen,
                   float* dist, int64_t ldd, int B, cudaStream_t st) {
  if (B <= 1) launch_stream_t<MODEL, NB, 1>(Qt, rpad, tab, np, d, cen, dist, ldd, B, st);
  else if (B <= 2) launch_stream_t<MODEL, NB, 2>(Qt, rpad, tab, np, d, cen, dist, ldd, B, st);
  else if (B <= 4) launch_stream_t<MODEL, NB, 4>(Qt, rpad, tab, np, d, cen, dist, ldd, B, st);
  else launch_stream_t<MODEL, NB, (MODEL == KGQ_Q2B ? 8 / NB : 8)>(Qt, rpad, tab, np, d, cen, dist, ldd, B, st);
}

template <int MODEL, int NB>
void launch_t(const float* Qt, int64_t rpad, const float* tab, int64_t np, int d, float cen,
              float* dist, int64_t ldd, int B, cudaStream_t st) {
  constexpr int NQ = Planes<MODEL>::NQ, NE = Planes<MODEL>::NE;
  const size_t smem = (size_t)2 * (NQ * DK * TQ + NE * DK * TE) * sizeof(float);
  static SmemAttr attr;
  smem_attr_once(k_score<MODEL, NB>, (int)smem, attr);
  const int rows = B * NB;
  dim3 grid((unsigned)(np / TE), (unsigned)((rows + TQ - 1) / TQ));
  k_score<MODEL, NB><<<grid, 256, smem, st>>>(Qt, rpad, tab, np, d, cen, dist, ldd, B);
}
}  // namespace

int launch_score_betae_stream(const Split& A, const float2* P, const float* uvT, const float2* E, int64_t np, int d,
                              float* dist, int64_t ldd, int B, int nbq, cudaStream_t st) {
  if (B <= 0) return 0;
#define KGQ_UV(NB)                                                                   \
  if (B <= 1) launch_uv_stream_t<NB, 1>(A, P, uvT, E, np, d, dist, ldd, B, st);      \
  else if (B <= 2) launch_uv_stream_t<NB, 2>(A, P, uvT, E, np, d, dist, ldd, B, st); \
  else if (B <= 4) launch_uv_stream_t<NB, 4>(A, P, uvT, E, np, d, dist, ldd, B, st); \
  else launch_uv_stream_t<NB, 8>(A, P, uvT, E, np, d, dist, ldd, B, st);
  if (nbq == 2) { KGQ_UV(2) } else { KGQ_UV(1) }
#undef KGQ_UV
  return 1;
}

// Small batches (<= 16 query rows; <= 8 for Q2B, which keeps two sums per pair) stream the
// table (HBM-bound regime); larger batches use the register-tiled kernel (FP32-ALU-bound).
bool score_uses_stream(int model, int nbq, int B) {
  return B * nbq <= (model == KGQ_Q2B ? 8 : 16) && B <= 8;
}

int launch_score(int model, int nbq, int B, int d, float cen, const float* Qt, int64_t rpad,
                 const float* tab, int64_t np, int64_t ns, float* dist, int64_t ldd,
                 cudaStream_t st) {
  (void)ns;
  const bool s = score_uses_stream(model, nbq, B);
#define KGQ_SCORE(M, NB)                                                  \
  (s ? launch_stream<M, NB>(Qt, rpad, tab, np, d, cen, dist, ldd, B, st) \
     : launch_t<M, NB>(Qt, rpad, tab, np, d, cen, dist, ldd, B, st))
  if (model == KGQ_GQE) {
    if (nbq == 2) KGQ_SCORE(KGQ_GQE, 2); else KGQ_SCORE(KGQ_GQE, 1);
  } else if (model == KGQ_Q2B) {
    if (nbq == 2) KGQ_SCORE(KGQ_Q2B, 2); else KGQ_SCORE(KGQ_Q2B, 1);
  } else {
    if (nbq == 2) KGQ_SCORE(KGQ_BETAE, 2); else KGQ_SCORE(KGQ_BETAE, 1);
  }
#undef KGQ_SCORE
  return 1;
}

}  // namespace kgq
