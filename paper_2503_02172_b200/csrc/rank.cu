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
}  // namespace

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
