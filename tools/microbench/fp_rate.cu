// FP32 issue-rate microbenchmark on B200: independent chains of FADD / FFMA (3-register) vs FADD2 / FFMA2.
// Prints per-SM ops/cycle for each; used to decide the emitter's arithmetic form.
#include <cstdio>
#include <cuda_runtime.h>
#define N 2048
__global__ void k_fadd(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  float y = a * 0.5f;
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    x0 = __fadd_rn(x0, y); x1 = __fadd_rn(x1, y); x2 = __fadd_rn(x2, y); x3 = __fadd_rn(x3, y);
    x4 = __fadd_rn(x4, y); x5 = __fadd_rn(x5, y); x6 = __fadd_rn(x6, y); x7 = __fadd_rn(x7, y);
    y = __fadd_rn(y, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_ffma(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  float y = a * 0.5f, z = b;
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    x0 = __fmaf_rn(x0, y, z); x1 = __fmaf_rn(x1, y, z); x2 = __fmaf_rn(x2, y, z); x3 = __fmaf_rn(x3, y, z);
    x4 = __fmaf_rn(x4, y, z); x5 = __fmaf_rn(x5, y, z); x6 = __fmaf_rn(x6, y, z); x7 = __fmaf_rn(x7, y, z);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_fadd2(float* out, float a, float b) {
  float2 x0 = make_float2(threadIdx.x, 1), x1 = make_float2(2, 3), x2 = make_float2(4, 5), x3 = make_float2(6, 7);
  float2 y = make_float2(a, b);
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    x0 = __fadd2_rn(x0, y); x1 = __fadd2_rn(x1, y); x2 = __fadd2_rn(x2, y); x3 = __fadd2_rn(x3, y);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0.x + x1.x + x2.x + x3.x + x0.y + x1.y + x2.y + x3.y;
}
__global__ void k_ffma2(float* out, float a, float b) {
  float2 x0 = make_float2(threadIdx.x, 1), x1 = make_float2(2, 3), x2 = make_float2(4, 5), x3 = make_float2(6, 7);
  float2 y = make_float2(a, b), z = make_float2(b, a);
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    x0 = __ffma2_rn(x0, y, z); x1 = __ffma2_rn(x1, y, z); x2 = __ffma2_rn(x2, y, z); x3 = __ffma2_rn(x3, y, z);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0.x + x1.x + x2.x + x3.x + x0.y + x1.y + x2.y + x3.y;
}
template <typename F>
void run(const char* name, F f, double ops_per_thread_iter) {
  float* out;
  cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
  int sms = 148, tpb = 1024;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    f<<<sms * 2, tpb>>>(out, 1.0001f, 0.999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ops = (double)sms * 2 * tpb * N * ops_per_thread_iter;
    double cycles = ms * 1e-3 * 1.965e9;
    if (rep) printf("%-6s %8.3f ms  %7.1f lane-ops/cycle/SM (at 1.965 GHz)\n", name, ms, ops / cycles / sms);
  }
  cudaFree(out);
}
int main() {
  run("FADD", k_fadd, 9);
  run("FFMA", k_ffma, 8);
  run("FADD2", k_fadd2, 8);
  run("FFMA2", k_ffma2, 8);
  return 0;
}
