// N1: filtered ranking of given answers, the KGReasoning test protocol behind
// the paper's accuracy check (MRR, P:425 / P:450).  For query b with answer set A_b (easy and
// hard answers, global ids) and an answer a in A_b:
//   count(a) = #{entities e of this shard, e not in A_b : (dist_e, e) < (dist_a, a)}
// so the filtered rank is 1 + the sum of counts over shards (ties by ascending id, Q13).
#include <stdint.h>

#include "common.cuh"
#include "kgq_internal.cuh"

namespace kgq {

namespace {
constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t okey(float f) {  // order-preserving key (as in topk.cu)
  if (f != f) return 0xFFFFFFFFu;
  if (f == 0.0f) f = 0.0f;
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <typename T>
__device__ void block_bitonic(T* v, int P) {
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const T a = v[lo], b = v[hi];
        if ((a > b) == up) {
          v[lo] = b;
          v[hi] = a;
        }
      }
      __syncthreads();
    }
}

// number of elements of sorted v[0, n) that are <= x
template <typename T>
__device__ __forceinline__ int upper_bound(const T* v, int n, T x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (v[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Distances of the answers that live in this shard (mode 0/1); +inf for the others (mode 1,
// to be min-reduced across ranks) -- dist rows [b0, b0 + nb) of the chunk.
__global__ void k_answer_dist(const float* __restrict__ dist, int64_t ldd, int64_t e0, int64_t ns, int b0,
                              int nb, const int32_t* __restrict__ ans_off, const int32_t* __restrict__ ans_id,
                              float* __restrict__ ans_dist) {
  const int b = blockIdx.x;
  const int q = b0 + b;
  const int a0 = ans_off[q], a1 = ans_off[q + 1];
  for (int j = a0 + threadIdx.x; j < a1; j += blockDim.x) {
    const int64_t loc = (int64_t)ans_id[j] - e0;
    ans_dist[j] = (loc >= 0 && loc < ns) ? dist[(int64_t)b * ldd + loc] : __uint_as_float(0x7F800000u);
  }
  (void)nb;
}

__global__ void __launch_bounds__(kThreads)
    k_filtered_counts(const float* __restrict__ dist, int64_t ldd, int64_t e0, int64_t ns, int b0,
                      const int32_t* __restrict__ ans_off, const int32_t* __restrict__ ans_id,
                      const float* __restrict__ ans_dist, int32_t* __restrict__ count, int32_t* err) {
  __shared__ unsigned long long skey[kMaxAnswers];  // answers' (key, id), sorted
  __shared__ uint32_t sid[kMaxAnswers];             // answers' ids, sorted (membership)
  __shared__ uint32_t diff[kMaxAnswers + 1];
  const int b = blockIdx.x;
  const int q = b0 + b;
  const int a0 = ans_off[q], na = ans_off[q + 1] - a0;
  if (na <= 0) return;
  if (na > kMaxAnswers) {
    if (threadIdx.x == 0) atomicCAS(&err[0], 0, 2);  // reported as KGQ_EINVAL by the host
    return;
  }
  int P = 1;
  while (P < na) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    if (i < na) {
      skey[i] = ((unsigned long long)okey(ans_dist[a0 + i]) << 32) | (uint32_t)ans_id[a0 + i];
      sid[i] = (uint32_t)ans_id[a0 + i];
    } else {
      skey[i] = ~0ull;
      sid[i] = 0xFFFFFFFFu;
    }
  }
  for (int i = threadIdx.x; i <= na; i += blockDim.x) diff[i] = 0;
  __syncthreads();
  block_bitonic(skey, P);
  block_bitonic(sid, P);
  const float* row = dist + (int64_t)b * ldd;
  for (int64_t e = threadIdx.x; e < ns; e += blockDim.x) {
    const uint32_t id = (uint32_t)(e0 + e);
    const int m = upper_bound(sid, na, id);
    if (m > 0 && sid[m - 1] == id) continue;  // an answer: filtered
    const unsigned long long k = ((unsigned long long)okey(row[e]) << 32) | id;
    const int p = upper_bound(skey, na, k);   // answers at sorted positions >= p rank behind e
    if (p < na) atomicAdd(&diff[p], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int j = 0; j < na; ++j) {
      run += diff[j];
      diff[j] = run;  // count for the answer at sorted position j
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < na; i += blockDim.x) {
    const unsigned long long k = ((unsigned long long)okey(ans_dist[a0 + i]) << 32) | (uint32_t)ans_id[a0 + i];
    const int j = upper_bound(skey, na, k) - 1;  // its own position (keys are unique)
    count[a0 + i] = (int32_t)diff[j];
  }
}

__global__ void k_add_one(int32_t* v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] += 1;
}

// MRR / Hits@{1,3,10} (KGReasoning averaging): per query the mean over its scored answers, then
// the mean over the queries that have one.  One CTA; fp64 sums in registers then shared memory
// (batch <= max_batch, a few thousand queries: one pass).
__global__ void __launch_bounds__(256) k_rank_metrics(int B, const int32_t* __restrict__ ans_off,
                                                      const int32_t* __restrict__ ranks,
                                                      const uint8_t* __restrict__ hard, double* out) {
  double acc[5] = {0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    double s[4] = {0, 0, 0, 0};
    int n = 0;
    for (int j = ans_off[b]; j < ans_off[b + 1]; ++j) {
      if (hard && !hard[j]) continue;
      const int r = ranks[j];
      s[0] += 1.0 / r;
      s[1] += r <= 1;
      s[2] += r <= 3;
      s[3] += r <= 10;
      ++n;
    }
    if (n) {
      for (int i = 0; i < 4; ++i) acc[i] += s[i] / n;
      acc[4] += 1.0;
    }
  }
  __shared__ double red[5][256];
  for (int i = 0; i < 5; ++i) red[i][threadIdx.x] = acc[i];
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if ((int)threadIdx.x < w)
      for (int i = 0; i < 5; ++i) red[i][threadIdx.x] += red[i][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double q = red[4][0];
    for (int i = 0; i < 4; ++i) out[i] = q > 0 ? red[i][0] / q : 0.0;
    out[4] = q;
  }
}
}  // namespace

int launch_add_one(int32_t* v, int n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_add_one<<<(n + 255) / 256, 256, 0, st>>>(v, n);
  return 1;
}

int launch_rank_metrics(int B, const int32_t* ans_off, const int32_t* ranks, const uint8_t* hard, double* out,
                        cudaStream_t st) {
  k_rank_metrics<<<1, 256, 0, st>>>(B, ans_off, ranks, hard, out);
  return 1;
}

int launch_answer_dist(const float* dist, int64_t ldd, int64_t e0, int64_t ns, int b0, int nb,
                       const int32_t* ans_off, const int32_t* ans_id, float* ans_dist, cudaStream_t st) {
  k_answer_dist<<<nb, 128, 0, st>>>(dist, ldd, e0, ns, b0, nb, ans_off, ans_id, ans_dist);
  return 1;
}

int launch_filtered_counts(const float* dist, int64_t ldd, int64_t e0, int64_t ns, int b0, int nb,
                           const int32_t* ans_off, const int32_t* ans_id, const float* ans_dist,
                           int32_t* count, int32_t* err, cudaStream_t st) {
  k_filtered_counts<<<nb, kThreads, 0, st>>>(dist, ldd, e0, ns, b0, ans_off, ans_id, ans_dist, count, err);
  return 1;
}

}  // namespace kgq
