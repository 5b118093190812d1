// FP32 issue-rate probe (the ALU roof of the SIMT / streaming scorers): lane-operations per
// clock per SM of FADD, FFMA, FADD2 (add.rn.f32x2), FFMA2 (fma.rn.f32x2), FADD2 with |.| operand
// modifiers (the L1 scorer's form) and FMNMX, each as 8 independent dependency chains per
// thread, 148 x 4 CTAs of 256 threads.  A packed op counts two lane-operations per lane.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_pipe_probe fp32_pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__device__ __forceinline__ void add2(float& x, float& y, float a, float b) {
  asm volatile("{\n.reg .b64 p, q;\nmov.b64 p, {%0, %1};\nmov.b64 q, {%2, %3};\nadd.rn.f32x2 p, p, q;\nmov.b64 {%0, %1}, p;\n}"
               : "+f"(x), "+f"(y) : "f"(a), "f"(b));
}
__device__ __forceinline__ void fma2(float& x, float& y, float a, float b, float c, float d) {
  asm volatile("{\n.reg .b64 p, q, r;\nmov.b64 p, {%0, %1};\nmov.b64 q, {%2, %3};\nmov.b64 r, {%4, %5};\n"
               "fma.rn.f32x2 p, q, r, p;\nmov.b64 {%0, %1}, p;\n}"
               : "+f"(x), "+f"(y) : "f"(a), "f"(b), "f"(c), "f"(d));
}

template <int OP>
__global__ void k(float* out, float s0, float s1) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 1e-3f + i;
  float a = s0 + threadIdx.x * 1e-7f, b = s1;
  float w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = threadIdx.x * 2e-3f - i;
  for (int it = 0; it < ITERS; ++it) {
    const float av = a + it * 1e-9f, bv = b - it * 1e-9f;  // OP 6's query value (one op per 16 elements)
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (OP == 0) { v[i] += a; v[i + 1] += b; }                       // 2 FADD
      if (OP == 1) { v[i] = fmaf(v[i], a, b); v[i + 1] = fmaf(v[i + 1], b, a); }  // 2 FFMA
      if (OP == 2) add2(v[i], v[i + 1], a, b);                          // 1 FADD2
      if (OP == 3) fma2(v[i], v[i + 1], a, b, b, a);                    // 1 FFMA2
      if (OP == 4) {                                                    // 1 FADD2 with |.|
        float2 t = make_float2(fabsf(v[(i + 2) & 15]), fabsf(v[(i + 3) & 15]));
        add2(v[i], v[i + 1], t.x, t.y);
      }
      if (OP == 5) { v[i] = fminf(v[i], v[(i + 3) & 15]); v[i + 1] = fmaxf(v[i + 1], v[(i + 6) & 15]); }  // 2 FMNMX
      if (OP == 6) {  // the min form of an L1 step: 2 FMNMX + 1 FADD2 per entity pair
        const float m0 = fminf(av, w[i]), m1 = fminf(bv, w[i + 1]);
        add2(v[i], v[i + 1], m0, m1);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  if (s == 123.456f) out[0] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const char* names[] = {"FADD", "FFMA", "FADD2", "FFMA2", "FADD2 |.|", "FMNMX", "2FMNMX+FADD2"};
  void (*fns[])(float*, float, float) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
  const int grid = 148 * 4, block = 256;
  for (int o = 0; o < 7; ++o) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fns[o]<<<grid, block>>>(out, 1.0001f, 0.9999f);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) fns[o]<<<grid, block>>>(out, 1.0001f, 0.9999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // two lane-ops per pair per iteration (OP 6: counted per element, i.e. per FMNMX + half FADD2)
    const double lane_ops = 5.0 * grid * block * ITERS * 16.0;
    const double per_s = lane_ops / (ms * 1e-3);
    printf("%-10s %8.2f T lane-ops/s = %6.1f lane-ops/clk/SM at %d MHz (max clock)\n", names[o], per_s / 1e12,
           per_s / (148.0 * clk_khz * 1e3), clk_khz / 1000);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
