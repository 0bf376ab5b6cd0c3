// Development probe: cost of the eig kernel's deferred window updates (one thread's pair of
// column segments) split into load / apply / store, on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int WIN = 32, BS = 5, SPW = 27, N = 200, SUB = 5;
__device__ __forceinline__ int band_lo(int i) { return i > SUB ? i - SUB : 0; }
__device__ __forceinline__ void apply2(double (&sa)[WIN], double (&sb)[WIN], const double* refl) {
#pragma unroll
  for (int u = 0; u < SPW; ++u) {
    const double* rf = refl + BS * u;
    double r[BS];
#pragma unroll
    for (int j = 0; j < BS; ++j) r[j] = rf[j];
    double xa = sa[u], xb = sb[u];
#pragma unroll
    for (int j = 1; j < BS; ++j) { xa = fma(r[j - 1], sa[u + j], xa); xb = fma(r[j - 1], sb[u + j], xb); }
    xa *= r[BS - 1]; xb *= r[BS - 1];
    sa[u] -= xa; sb[u] -= xb;
#pragma unroll
    for (int j = 1; j < BS; ++j) { sa[u + j] = fma(-xa, r[j - 1], sa[u + j]); sb[u + j] = fma(-xb, r[j - 1], sb[u + j]); }
  }
}
__global__ void k(long long* out, int w0, int nw) {
  extern __shared__ double sm[];
  __shared__ int rowoff[N + 1];
  __shared__ double refl[BS * SPW];
  const int tid = threadIdx.x;
  if (tid == 0) { int o = 0; for (int i = 0; i < N; ++i) { rowoff[i] = o - band_lo(i); o += N - band_lo(i); } rowoff[N] = o; }
  for (int e = tid; e < BS * SPW; e += blockDim.x) refl[e] = (e % BS == BS - 1) ? 1.5 : 0.01 * (e % 7);
  __syncthreads();
  for (int e = tid; e < rowoff[N]; e += blockDim.x) sm[e] = 1.0 / (1 + e % 13);
  __syncthreads();
  const int w1 = w0 + nw, nL = N - w1, nR = w0;
  long long t0 = clock64();
  double sa[WIN], sb[WIN];
  const int ta = tid, tb = tid + 128;
  auto load = [&](double (&seg)[WIN], int task) {
    if (task >= nL + nR) { for (int u = 0; u < WIN; ++u) seg[u] = 0.0; }
    else if (task < nL) { const int c = w1 + task;
#pragma unroll
      for (int u = 0; u < WIN; ++u) seg[u] = (u < nw) ? sm[rowoff[w0 + u] + c] : 0.0; }
    else { const double* row = sm + rowoff[task - nL] + w0;
#pragma unroll
      for (int u = 0; u < WIN; ++u) seg[u] = (u < nw) ? row[u] : 0.0; }
  };
  load(sa, ta); load(sb, tb);
  double chk = 0; for (int u = 0; u < WIN; ++u) chk += sa[u] + sb[u];
  long long t1 = clock64();
  apply2(sa, sb, refl);
  double chk2 = 0; for (int u = 0; u < WIN; ++u) chk2 += sa[u] + sb[u];
  long long t2 = clock64();
  auto store = [&](const double (&seg)[WIN], int task) {
    if (task >= nL + nR) return;
    if (task < nL) { const int c = w1 + task;
#pragma unroll
      for (int u = 0; u < WIN; ++u) if (u < nw) sm[rowoff[w0 + u] + c] = seg[u]; }
    else { double* row = sm + rowoff[task - nL] + w0;
#pragma unroll
      for (int u = 0; u < WIN; ++u) if (u < nw) row[u] = seg[u]; }
  };
  store(sa, ta); store(sb, tb);
  __syncthreads();
  long long t3 = clock64();
  if (tid == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = (long long)(chk + chk2); }
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[4];
  const int smem = 21400 * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int w0 : {0, 54, 108}) {
    k<<<1, 128, smem>>>(d, w0, 32); cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    k<<<1, 128, smem>>>(d, w0, 32);
    cudaError_t e = cudaDeviceSynchronize(); if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("w0=%d load %lld apply %lld store+sync %lld\n", w0, h[0], h[1], h[2]);
  }
  return 0;
}
