// Diagnostic: dependent-chain latency (cycles) of a few instruction types on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* od, float* of, long long* cyc, int n) {
  double d = threadIdx.x * 1e-3 + 1.0; float f = d;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { d = fma(d, 0.9999999, 1e-9); }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { f = fmaf(f, 0.9999999f, 1e-9f); }
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) { f = (float)(d + (double)f * 1e-30); }   // F2F chain (+DFMA)
  long long t3 = clock64();
  double x = d;
  for (int i = 0; i < n; ++i) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y; }
  long long t4 = clock64();
  float g = f;
  for (int i = 0; i < n; ++i) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(g)); g = y; }
  long long t5 = clock64();
  od[threadIdx.x] = d + x; of[threadIdx.x] = f + g;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* od; float* of; long long* c; cudaMalloc(&od, 256 * 8); cudaMalloc(&of, 256 * 4); cudaMallocManaged(&c, 64);
  int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    lat<<<1, 32>>>(od, of, c, n); cudaDeviceSynchronize();
    printf("per-op latency (cycles): DFMA %.2f  FFMA %.2f  F2F+DFMA+F2F %.2f  MUFU.RCP64H %.2f  MUFU.RCP %.2f\n",
           (double)c[0] / n, (double)c[1] / n, (double)c[2] / n, (double)c[3] / n, (double)c[4] / n);
  }
  return 0;
}
