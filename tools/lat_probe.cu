// Latency probe (development): dependent-chain cycles of FP64 ops on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double x = a, y = b;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 125; ++i) {
#pragma unroll
 for (int u = 0; u < 8; ++u) x = fma(x, y, 1e-300); }
  t1 = clock64(); cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 125; ++i) {
#pragma unroll
 for (int u = 0; u < 8; ++u) x = x + y; }
  t1 = clock64(); cyc[1] = t1 - t0;
  // rsqrt.approx.f64
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 125; ++i)
#pragma unroll
 for (int u = 0; u < 8; ++u) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  t1 = clock64(); cyc[2] = t1 - t0;
  // rcp.approx.ftz.f64
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 125; ++i)
#pragma unroll
 for (int u = 0; u < 8; ++u) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  t1 = clock64(); cyc[3] = t1 - t0;
  // sqrt (IEEE)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = sqrt(x) + 1.0; }
  t1 = clock64(); cyc[4] = t1 - t0;
  // division
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = y / x + 1.0; }
  t1 = clock64(); cyc[5] = t1 - t0;
  // FFMA32 chain for reference
  float xf = (float)a, yf = (float)b;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 125; ++i) {
#pragma unroll
 for (int u = 0; u < 8; ++u) xf = fmaf(xf, yf, 1e-30f); }
  t1 = clock64(); cyc[6] = t1 - t0;
  // smem load chain
  __shared__ int sidx[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sidx[i] = (i + 1) & 63;
  __syncthreads();
  int j = 0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 125; ++i) {
#pragma unroll
 for (int u = 0; u < 8; ++u) j = sidx[j]; }
  t1 = clock64(); cyc[7] = t1 - t0;
  // empty loop
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { asm volatile(""); }
  t1 = clock64(); cyc[8] = t1 - t0;
  // double shuffle chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 125; ++i) {
#pragma unroll
 for (int u = 0; u < 8; ++u) x = __shfl_xor_sync(0xffffffffu, x, 1); }
  t1 = clock64(); cyc[9] = t1 - t0;
  // syncwarp + smem store->load
  __shared__ double sd[32];
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { sd[threadIdx.x & 31] = x; __syncwarp(); x = sd[(threadIdx.x + 1) & 31] + 1.0; __syncwarp(); }
  t1 = clock64(); cyc[10] = t1 - t0;
  out[threadIdx.x] = x + xf + j;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64 * 8);
  k<<<1, 32>>>(o, c, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  const char* nm[] = {"DFMA", "DADD", "rsqrt.approx.f64+DADD", "rcp.approx.f64+DADD", "sqrt+DADD", "div+DADD", "FFMA", "LDS chain", "empty loop", "SHFL f64", "STS/syncwarp/LDS+DADD"};
  for (int i = 0; i < 11; ++i) printf("%-26s %6.1f cyc/iter\n", nm[i], c[i] / 1000.0);
  return 0;
}
