// FP64 DMMA GEMM: 64x64x16 CTA tile, 4 warps (2x2), 32x32 warp tile = 4x4 m8n8k4 MMAs,
// register-staged double buffering of the global->shared copy.
#include "gemm_f64.cuh"

namespace ssi {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 128;
constexpr int LDS = BM + 4;  // 68 doubles: conflict-free m8n8k4 fragment reads (LDS%16==4)

struct TileArgs {
  int64_t M, N, kb, ke;    // valid rows/cols, k range [kb, ke)
  Operand A, B;
};

template <bool AKC, bool BKC>
__device__ __forceinline__ void load_tile(const TileArgs& t, int64_t m0, int64_t n0, int64_t k0,
                                          double (&ra)[8], double (&rb)[8]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int mm, kk;
    if (AKC) { kk = tid % BK; mm = tid / BK + 8 * j; }
    else     { mm = tid % BM; kk = tid / BM + 2 * j; }
    const int64_t gi = m0 + mm, gk = k0 + kk;
    ra[j] = (gi < t.M && gk < t.ke) ? t.A.p[gi * t.A.s_r + gk * t.A.s_c] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int nn, kk;
    if (BKC) { kk = tid % BK; nn = tid / BK + 8 * j; }
    else     { nn = tid % BN; kk = tid / BN + 2 * j; }
    const int64_t gj = n0 + nn, gk = k0 + kk;
    rb[j] = (gj < t.N && gk < t.ke) ? t.B.p[gk * t.B.s_r + gj * t.B.s_c] : 0.0;
  }
}

template <bool AKC, bool BKC>
__device__ __forceinline__ void store_tile(double* As, double* Bs, const double (&ra)[8],
                                           const double (&rb)[8]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int mm, kk;
    if (AKC) { kk = tid % BK; mm = tid / BK + 8 * j; }
    else     { mm = tid % BM; kk = tid / BM + 2 * j; }
    As[kk * LDS + mm] = ra[j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int nn, kk;
    if (BKC) { kk = tid % BK; nn = tid / BK + 8 * j; }
    else     { nn = tid % BN; kk = tid / BN + 2 * j; }
    Bs[kk * LDS + nn] = rb[j];
  }
}

// Computes the 64x64 tile at (m0, n0) over k in [kb, ke); result in acc.
template <bool AKC, bool BKC>
__device__ __forceinline__ void tile_mma(const TileArgs& t, int64_t m0, int64_t n0,
                                         double (&acc)[4][4][2], double* smem) {
  double* As[2] = {smem, smem + 2 * BK * LDS};
  double* Bs[2] = {smem + BK * LDS, smem + 3 * BK * LDS};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  if (t.ke <= t.kb) return;
  double ra[8], rb[8];
  load_tile<AKC, BKC>(t, m0, n0, t.kb, ra, rb);
  store_tile<AKC, BKC>(As[0], Bs[0], ra, rb);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = t.kb; k0 < t.ke; k0 += BK) {
    const bool more = (k0 + BK) < t.ke;
    if (more) load_tile<AKC, BKC>(t, m0, n0, k0 + BK, ra, rb);
    const double* as = As[buf];
    const double* bs = Bs[buf];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(kk + (lane & 3)) * LDS + wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(kk + (lane & 3)) * LDS + wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (more) {
      store_tile<AKC, BKC>(As[buf ^ 1], Bs[buf ^ 1], ra, rb);
      __syncthreads();
      buf ^= 1;
    }
  }
}

__device__ __forceinline__ void store_acc(const double (&acc)[4][4][2], int64_t m0, int64_t n0,
                                          int64_t M, int64_t N, double alpha, double* C,
                                          int64_t ldc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t r = m0 + wm + i * 8 + (lane >> 2);
        const int64_t c = n0 + wn + j * 8 + 2 * (lane & 3) + e;
        if (r < M && c < N) C[r + c * ldc] = alpha * acc[i][j][e];
      }
}

template <bool AKC, bool BKC>
__global__ void __launch_bounds__(NT) gemm_kernel(int64_t M, int64_t N, int64_t K, double alpha,
                                                  Operand A, Operand B, double* C, int64_t ldc,
                                                  int64_t kchunk, double* partial, const int* run_if) {
  __shared__ __align__(16) double smem[4 * BK * LDS];
  if (!run_enabled(run_if)) return;
  const int64_t m0 = int64_t(blockIdx.x) * BM, n0 = int64_t(blockIdx.y) * BN;
  TileArgs t{M, N, int64_t(blockIdx.z) * kchunk, 0, A, B};
  t.ke = t.kb + kchunk < K ? t.kb + kchunk : K;
  double acc[4][4][2];
  tile_mma<AKC, BKC>(t, m0, n0, acc, smem);
  if (partial)
    store_acc(acc, m0, n0, M, N, 1.0, partial + int64_t(blockIdx.z) * M * N, M);
  else
    store_acc(acc, m0, n0, M, N, alpha, C, ldc);
}

__global__ void splitk_reduce(int64_t M, int64_t N, int splits, const double* __restrict__ part,
                              double alpha, double* __restrict__ C, int64_t ldc, const int* run_if) {
  if (!run_enabled(run_if)) return;
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    s = ordered_sum(part + e, total, splits);
    const int64_t r = e % M, c = e / M;
    C[r + c * ldc] = alpha * s;
  }
}

// Batched order GEMMs: blockIdx.z = order index.
__global__ void __launch_bounds__(NT) gemm_orders_kernel(int n0, int dn, const double* A,
                                                         int64_t lda, const double* B,
                                                         int64_t ldb, double* Cbase) {
  __shared__ __align__(16) double smem[4 * BK * LDS];
  const int b = blockIdx.z;
  const int64_t n = n0 + int64_t(b) * dn;
  const int64_t m0 = int64_t(blockIdx.x) * BM, c0 = int64_t(blockIdx.y) * BN;
  if (m0 >= n || c0 >= n) return;
  // off_b = sum_{b'<b} (n0 + b' dn)^2
  int64_t off = 0;
  for (int bb = 0; bb < b; ++bb) { const int64_t nb = n0 + int64_t(bb) * dn; off += nb * nb; }
  TileArgs t{n, n, 0, n, Operand{A, 1, lda}, Operand{B, 1, ldb}};
  double acc[4][4][2];
  tile_mma<false, true>(t, m0, c0, acc, smem);
  store_acc(acc, m0, c0, n, n, 1.0, Cbase + off, n);
}

}  // namespace

int gemm_pick_splits(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int64_t target = 148 * 4;
  int64_t s = (target + tiles - 1) / tiles;
  const int64_t kmax = (K + 255) / 256;   // keep >= 256 k per split
  if (s > kmax) s = kmax;
  if (s < 1) s = 1;
  if (s > 64) s = 64;
  return int(s);
}

size_t gemm_partial_elems(int64_t M, int64_t N, int splits) {
  return splits > 1 ? size_t(splits) * size_t(M) * size_t(N) : 0;
}

ssi_status gemm_f64(int64_t M, int64_t N, int64_t K, double alpha, Operand A, Operand B,
                    double* C, int64_t ldc, int splits, double* partial, cudaStream_t s, const int* run_if) {
  if (M <= 0 || N <= 0) return SSI_OK;
  const bool akc = (A.s_c == 1), bkc = (B.s_r == 1);
  if (splits < 1) splits = 1;
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  if (kchunk < BK) kchunk = BK;
  const int z = int((K + kchunk - 1) / kchunk > 0 ? (K + kchunk - 1) / kchunk : 1);
  double* part = (z > 1) ? partial : nullptr;
  dim3 grid((M + BM - 1) / BM, (N + BN - 1) / BN, z);
  if (akc && bkc) gemm_kernel<true, true><<<grid, NT, 0, s>>>(M, N, K, alpha, A, B, C, ldc, kchunk, part, run_if);
  else if (akc)   gemm_kernel<true, false><<<grid, NT, 0, s>>>(M, N, K, alpha, A, B, C, ldc, kchunk, part, run_if);
  else if (bkc)   gemm_kernel<false, true><<<grid, NT, 0, s>>>(M, N, K, alpha, A, B, C, ldc, kchunk, part, run_if);
  else            gemm_kernel<false, false><<<grid, NT, 0, s>>>(M, N, K, alpha, A, B, C, ldc, kchunk, part, run_if);
  SSI_TRY(launch_check("gemm_f64"));
  if (z > 1) {
    const int64_t tot = M * N;
    int blocks = int((tot + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    splitk_reduce<<<blocks, 256, 0, s>>>(M, N, z, partial, alpha, C, ldc, run_if);
    SSI_TRY(launch_check("splitk_reduce"));
  }
  return SSI_OK;
}

ssi_status gemm_f64_orders(int nb, int n0, int dn, const double* A, int64_t lda, const double* B,
                           int64_t ldb, double* Cbase, cudaStream_t s) {
  const int nmax = n0 + (nb - 1) * dn;
  dim3 grid((nmax + BM - 1) / BM, (nmax + BN - 1) / BN, nb);
  gemm_orders_kernel<<<grid, NT, 0, s>>>(n0, dn, A, lda, B, ldb, Cbase);
  return launch_check("gemm_f64_orders");
}

}  // namespace ssi
