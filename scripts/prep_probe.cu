// Timing probe for the BetaE score prep (score_tc.cu k_score_prep_tc): per query row, the split
// [aq; bq] operand and P_q = sum_d lnB(aq, bq) + aq Ubar + bq Vbar in fp64.  Variants of the
// lnB evaluation and of the thread mapping, rows = 1024, d = 400 (not part of the library).
#include <cstdio>
#include <cmath>
#include <vector>
#include "../paper_2503_02172_b200/csrc/common.cuh"
using namespace kgq;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// branch-free: always shift by 8 (x > 0 -> y = x + 8 >= 8), one reciprocal for three Stirling
// series, one division for the shift products
__device__ __forceinline__ double lnbeta_b(double a, double b) {
  const double c = a + b;
  double pa = a, pb = b, pc = c;
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    pa *= a + i;
    pb *= b + i;
    pc *= c + i;
  }
  const double ya = a + 8.0, yb = b + 8.0, yc = c + 8.0;
  const double yab = ya * yb, rall = 1.0 / (yab * yc);
  const double ra = rall * yb * yc, rb = rall * ya * yc, rc = rall * yab;
  auto ser = [](double r) {
    const double z = r * r;
    return r * (1.0 / 12 + z * (-1.0 / 360 + z * (1.0 / 1260 + z * (-1.0 / 1680 +
           z * (1.0 / 1188 + z * (-691.0 / 360360 + z * (1.0 / 156)))))));
  };
  return (ya - 0.5) * log(ya) + (yb - 0.5) * log(yb) - (yc - 0.5) * log(yc) - ya - yb + yc +
         0.91893853320467274178 + ser(ra) + ser(rb) - ser(rc) + log(pc / (pa * pb));
}

// fp64 reciprocal: fp32 seed + two Newton steps (2^-23 -> 2^-46 -> ~2^-92, i.e. correctly
// rounded up to an ulp); x normal, |x| within fp32 range
__device__ __forceinline__ double rcp_nr_p(double x) {
  double r = (double)__frcp_rn((float)x);
  r = r * (2.0 - x * r);  // fma-contracted
  r = r * (2.0 - x * r);
  return r;
}
// fp64 natural log for normal x > 0: x = 2^e m, m in [sqrt(1/2), sqrt(2)), ln m = 2 atanh(s),
// s = (m - 1)/(m + 1), |s| <= 0.1716, series through s^19 (truncation < 4e-16 relative)
__device__ __forceinline__ double log_fast_p(double x) {
  int hi = __double2hiint(x), lo = __double2loint(x);
  int e = (hi >> 20) - 1023;
  hi = (hi & 0x000FFFFF) | 0x3FF00000;
  double m = __hiloint2double(hi, lo);
  if (m > 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  const double f = m - 1.0, den = m + 1.0;
  const double r = rcp_nr_p(den);
  double sq = f * r;
  sq = sq + r * (f - sq * den);  // residual correction
  const double z = sq * sq;
  const double p = 1.0 / 3 + z * (1.0 / 5 + z * (1.0 / 7 + z * (1.0 / 9 + z * (1.0 / 11 + z * (1.0 / 13 +
                   z * (1.0 / 15 + z * (1.0 / 17 + z * (1.0 / 19))))))));
  return (double)e * 0.69314718055994530942 + (2.0 * sq + 2.0 * sq * z * p);
}
__device__ __forceinline__ double lnbeta_c(double a, double b) {
  const double c = a + b;
  double pa = a, pb = b, pc = c;
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    pa *= a + i;
    pb *= b + i;
    pc *= c + i;
  }
  const double ya = a + 8.0, yb = b + 8.0, yc = c + 8.0;
  const double yab = ya * yb, yabc = yab * yc;
  const double rall = rcp_nr_p(yabc);
  const double ra = rall * yb * yc, rb = rall * ya * yc, rc = rall * yab;
  auto ser = [](double r) {
    const double z = r * r;
    return r * (1.0 / 12 + z * (-1.0 / 360 + z * (1.0 / 1260 + z * (-1.0 / 1680 + z * (1.0 / 1188)))));
  };
  const double pab = pa * pb;
  const double ratio = pab < 1e30 ? pc * rcp_nr_p(pab) : pc / pab;  // fp32 seed range
  return (ya - 0.5) * log_fast_p(ya) + (yb - 0.5) * log_fast_p(yb) - (yc - 0.5) * log_fast_p(yc) - ya - yb + yc +
         0.91893853320467274178 + ser(ra) + ser(rb) - ser(rc) + log_fast_p(ratio);
}

template <int V>
__global__ void k_prep(const float* __restrict__ q, int rows, int d, const double* __restrict__ sums, int64_t ns,
                       Split A, float2* __restrict__ P) {
  const int r = blockIdx.x;
  __shared__ double red[32];
  double p = 0.0;
  const double inv = 1.0 / (double)ns;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const float a = q[(int64_t)r * 2 * d + j], b = q[(int64_t)r * 2 * d + d + j];
    if (V != 3) {
      store_split(A, (int64_t)r * A.ld + j, a);
      store_split(A, (int64_t)r * A.ld + d + j, b);
    }
    const double da = a, db = b;
    double l = 0.0;
    if (V == 0 || V == 3) l = lnbeta_f64(da, db);
    if (V == 1) l = lnbeta_b(da, db);
    if (V == 4) l = lnbeta_c(da, db);
    p += l + da * sums[j] * inv + db * sums[d + j] * inv;
  }
  p = warp_sum(p);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = p;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) P[r] = make_float2((float)t, (float)(t - (double)(float)t));
  }
}

// warp per row, 8 rows per block, branch-free lnB
template <int V>
__global__ void k_prep_w(const float* __restrict__ q, int rows, int d, const double* __restrict__ sums, int64_t ns,
                         Split A, float2* __restrict__ P) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  double p = 0.0;
  const double inv = 1.0 / (double)ns;
  for (int j = lane; j < d; j += 32) {
    const float a = q[(int64_t)r * 2 * d + j], b = q[(int64_t)r * 2 * d + d + j];
    store_split(A, (int64_t)r * A.ld + j, a);
    store_split(A, (int64_t)r * A.ld + d + j, b);
    const double da = a, db = b;
    const double l = V == 0 ? lnbeta_f64(da, db) : lnbeta_b(da, db);
    p += l + da * sums[j] * inv + db * sums[d + j] * inv;
  }
  p = warp_sum(p);
  if (lane == 0) P[r] = make_float2((float)p, (float)(p - (double)(float)p));
}

int main() {
  const int rows = 1024, d = 400;
  std::vector<float> hq((size_t)rows * 2 * d);
  unsigned s = 7;
  for (auto& x : hq) {
    s = s * 1664525u + 1013904223u;
    const double u = (s >> 8) / 16777216.0;
    x = (float)exp(log(0.05) + u * (log(5.0) - log(0.05)));  // post-regulariser range
  }
  float* q; double* sums; float2* P; __nv_bfloat16* planes;
  cudaMalloc(&q, hq.size() * 4);
  cudaMemcpy(q, hq.data(), hq.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&sums, 2 * d * 8);
  cudaMemset(sums, 0, 2 * d * 8);
  cudaMalloc(&P, rows * 8);
  cudaMalloc(&planes, (size_t)3 * rows * 2 * d * 2);
  Split A{planes, planes + (size_t)rows * 2 * d, planes + (size_t)2 * rows * 2 * d, 2 * d};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float2> ref(rows), got(rows);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(got.data(), P, rows * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int r = 0; r < rows; ++r)
      mx = fmax(mx, fabs(((double)got[r].x + got[r].y) - ((double)ref[r].x + ref[r].y)));
    printf("%-40s %8.2f us   max |P - P_ref| %.3e  %s\n", name, ms * 1e3 / 20, mx, cudaGetErrorString(cudaGetLastError()));
  };
  k_prep<0><<<rows, 128>>>(q, rows, d, sums, 14505, A, P);
  cudaDeviceSynchronize();
  cudaMemcpy(ref.data(), P, rows * 8, cudaMemcpyDeviceToHost);
  run("block/row, lnbeta_f64 (common.cuh)", [&] { k_prep<0><<<rows, 128>>>(q, rows, d, sums, 14505, A, P); });
  run("block/row, lnbeta_f64, no stores", [&] { k_prep<3><<<rows, 128>>>(q, rows, d, sums, 14505, A, P); });
  run("block/row, branch-free lnB", [&] { k_prep<1><<<rows, 128>>>(q, rows, d, sums, 14505, A, P); });
  run("block/row, custom log/rcp lnB", [&] { k_prep<4><<<rows, 128>>>(q, rows, d, sums, 14505, A, P); });
  run("block/row, no lnB (stores only)", [&] { k_prep<2><<<rows, 128>>>(q, rows, d, sums, 14505, A, P); });
  run("warp/row x4, lnbeta_f64", [&] { k_prep_w<0><<<rows / 4, 128>>>(q, rows, d, sums, 14505, A, P); });
  run("warp/row x4, branch-free lnB", [&] { k_prep_w<1><<<rows / 4, 128>>>(q, rows, d, sums, 14505, A, P); });
  run("warp/row x8, branch-free lnB", [&] { k_prep_w<1><<<rows / 8, 256>>>(q, rows, d, sums, 14505, A, P); });
  run("warp/row x2, branch-free lnB", [&] { k_prep_w<1><<<rows / 2, 64>>>(q, rows, d, sums, 14505, A, P); });
  return 0;
}
