// capture test for the library kernels: which launch fails inside stream capture?
#include <cstdio>
#include "/root/repo/paper_2503_02172_b200/csrc/chain.cu"
#include "/root/repo/paper_2503_02172_b200/csrc/linear_tc.cu"
using namespace kgq;
int main() {
  const int M = 1024, N = 1600, K = 1200;
  float *x, *xh, *xl, *w, *wh, *wl, *b, *y;
  cudaMalloc(&x, (size_t)M * K * 4); cudaMalloc(&xh, (size_t)M * K * 4); cudaMalloc(&xl, (size_t)M * K * 4);
  cudaMalloc(&w, (size_t)N * K * 4); cudaMalloc(&wh, (size_t)N * K * 4); cudaMalloc(&wl, (size_t)N * K * 4);
  cudaMalloc(&b, N * 4); cudaMalloc(&y, (size_t)M * N * 8);
  Linear L; L.W = w; L.W_hi = wh; L.W_lo = wl; L.b = b; L.out_f = N; L.in_f = K;
  Split A{xh, xl, K}; Split out{y, y + (size_t)M * N, N};
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  // eager first

  tc::launch_tc_gemm2<128>(A, M, wh, wl, N, K, K, EpiLinear<64, kEpiRelu, true>{b, out, M, N, 0, 0}, s);
  tc::launch_tc_gemm<128>(A, M, wh, wl, N, K, K, EpiLinear<64, kEpiRelu, true>{b, out, M, N, 0, 0}, s);
  printf("eager: %s\n", cudaGetErrorString(cudaStreamSynchronize(s)));
  cudaGraph_t g;
  printf("begin: %s\n", cudaGetErrorString(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal)));
  tc::launch_tc_gemm<128>(A, M, wh, wl, N, K, K, EpiLinear<64, kEpiRelu, true>{b, out, M, N, 0, 0}, s);
  printf("1cta in capture: %s\n", cudaGetErrorString(cudaGetLastError()));
  tc::launch_tc_gemm2<128>(A, M, wh, wl, N, K, K, EpiLinear<64, kEpiRelu, true>{b, out, M, N, 0, 0}, s);
  printf("2cta in capture: %s\n", cudaGetErrorString(cudaGetLastError()));
  printf("end: %s\n", cudaGetErrorString(cudaStreamEndCapture(s, &g)));
  return 0;
}
