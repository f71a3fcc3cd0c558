// Microbenchmark: fp64 / fp32 FMA issue rates on the local B200 (diagnostic only).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void cvt_loop(double* out, int iters, float a) {
  float f = threadIdx.x; double acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) { acc += (double)f; f = f * a + 1.0f; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void rcp_loop(double* out, int iters) {
  double x = threadIdx.x + 1.5, acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc += 1.0 / x; x += 1.0; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  int blocks = sms * 8, threads = 256, iters = 4000;
  double* d; cudaMalloc(&d, blocks * threads * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); fma_loop<double><<<blocks, threads>>>(d, iters, 0.999999, 1e-7); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)blocks * threads * iters * 16 * 8;
    printf("DFMA: %.3f T fma/s  (%.1f per SM per clk at max clk)\n", n / ms / 1e9, n / (ms * 1e-3) / sms / (clk * 1e3));
    cudaEventRecord(e0); fma_loop<float><<<blocks, threads>>>((float*)d, iters, 0.999999f, 1e-7f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA: %.3f T fma/s  (%.1f per SM per clk)\n", n / ms / 1e9, n / (ms * 1e-3) / sms / (clk * 1e3));
    cudaEventRecord(e0); cvt_loop<<<blocks, threads>>>(d, iters, 0.999f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    n = (double)blocks * threads * iters * 16;
    printf("F2F.F64.F32+DADD+FFMA: %.3f T/s  (%.1f per SM per clk)\n", n / ms / 1e9, n / (ms * 1e-3) / sms / (clk * 1e3));
    cudaEventRecord(e0); rcp_loop<<<blocks, threads>>>(d, iters / 4); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    n = (double)blocks * threads * (iters / 4) * 8;
    printf("fp64 1.0/x: %.3f T/s  (%.1f per SM per clk)\n", n / ms / 1e9, n / (ms * 1e-3) / sms / (clk * 1e3));
  }
  return 0;
}
