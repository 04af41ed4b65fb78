// FP64 pipe microbenchmark: DFMA throughput and IEEE sqrt+div throughput on sm_100a.
// Used to derive the "alu" roofline peak for the entry-evaluation kernels.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void sqrtdiv_loop(double* out, int iters, double a) {
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  double d = 1.0 + threadIdx.x * 1e-3;
  for (int i = 0; i < iters; ++i) {
    double d0 = d + i, d1 = d0 + 0.25, d2 = d0 + 0.5, d3 = d0 + 0.75;
    acc0 += a / sqrt(d0); acc1 += a / sqrt(d1); acc2 += a / sqrt(d2); acc3 += a / sqrt(d3);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<<<sms * 8, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)sms * 8 * 256 * iters * 16 * 8;
    printf("{\"kernel\":\"dfma\",\"rep\":%d,\"ms\":%.3f,\"dfma_per_s\":%.4e,\"tflops\":%.3f,\"sms\":%d,\"clk_mhz\":%d}\n", rep, ms, fmas / (ms * 1e-3), 2 * fmas / (ms * 1e-3) / 1e12, sms, clk / 1000);
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    sqrtdiv_loop<<<sms * 8, 256>>>(out, iters * 4, 1.5);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 8 * 256 * iters * 4 * 4;
    printf("{\"kernel\":\"sqrt_div\",\"rep\":%d,\"ms\":%.3f,\"evals_per_s\":%.4e}\n", rep, ms, ops / (ms * 1e-3));
  }
  return 0;
}
