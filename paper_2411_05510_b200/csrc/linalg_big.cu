// Sketch widths beyond one SM (NEXT-1: the paper's rank rule k = k̄(T) % of T, 25-30 %,
// PAPER.md:360-373 Eq. (empirical_formula) and :513 — e.g. k = 2880 at T = 11520):
//   * CholeskyQR2 with a blocked right-looking Cholesky (64-column panels: one CTA factors the
//     diagonal block and inverts it, DMMA tiles form the panel and the trailing update) and a
//     blocked right-looking triangular solve Q = Y L^{-T} (no explicit L^{-1}); the shifted
//     CholeskyQR3 fallback on breakdown, decided on the device (conditional launches);
//   * the small SVD of the k x k factor as a block one-sided (Hestenes) Jacobi over the whole GPU:
//     16-column blocks, round-robin pairing of the blocks, one persistent CTA per block pair
//     (grid barrier between rounds); per pair the 32 x 32 Gram matrix is formed on the FP64
//     tensor cores, diagonalised in shared memory by parallel-ordered two-sided Jacobi
//     rotations accumulated into V, and the pair's columns are replaced by X V (DMMA).
// Same results as the one-CTA kernels of linalg.cu up to rounding; used for k > kSvdMaxK.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <math_constants.h>

#include "linalg.cuh"

namespace cg = cooperative_groups;

namespace ssi {
namespace {

constexpr int PB = 64;                    // Cholesky / TRSM panel width
constexpr int TT = 64, TK = PB, TLD = TK + 4;
constexpr int kNtThreads = 256;

// C (M x N, col-major ldc) = alpha C + beta A B^T with A: M x K (col-major lda), B: N x K (col-major
// ldb), K <= 64. One 64 x 64 tile per CTA (A and B tiles staged whole: C may alias A when N <= 64,
// the tile reads its A rows before it writes them). lower: skip tiles strictly above the diagonal.
__global__ void __launch_bounds__(kNtThreads) gemm_nt_kernel(int64_t M, int64_t N, int K, const double* A, int64_t lda,
                                                             const double* B, int64_t ldb, double* C, int64_t ldc,
                                                             double alpha, double beta, int lower, const int* run_if) {
  if (!run_enabled(run_if)) return;
  if (lower && blockIdx.y > blockIdx.x) return;
  extern __shared__ double smb[];
  double* As = smb;             // [64][TLD]: As[r][k]
  double* Bs = smb + TT * TLD;  // [64][TLD]: Bs[n][k]
  const int64_t m0 = int64_t(blockIdx.x) * TT, n0 = int64_t(blockIdx.y) * TT;
  for (int e = threadIdx.x; e < TT * TK; e += kNtThreads) {
    const int r = e % TT, kk = e / TT;
    As[r * TLD + kk] = (m0 + r < M && kk < K) ? A[(m0 + r) + int64_t(kk) * lda] : 0.0;
    Bs[r * TLD + kk] = (n0 + r < N && kk < K) ? B[(n0 + r) + int64_t(kk) * ldb] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int kq = lane & 3, r8 = lane >> 2;
#pragma unroll 4
  for (int k4 = 0; k4 < TK; k4 += 4) {
    double af[2], bf[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) af[a] = As[(wr + 8 * a + r8) * TLD + k4 + kq];
#pragma unroll
    for (int b = 0; b < 4; ++b) bf[b] = Bs[(wc + 8 * b + r8) * TLD + k4 + kq];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
  }
  __syncthreads();
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = m0 + wr + 8 * a + r8, c = n0 + wc + 8 * b + 2 * kq + h;
        if (r < M && c < N) {
          double* p = C + r + c * ldc;
          *p = alpha == 0.0 ? beta * acc[a][b][h] : fma(beta, acc[a][b][h], alpha * *p);
        }
      }
}

ssi_status gemm_nt(int64_t M, int64_t N, int K, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double* C, int64_t ldc, double alpha, double beta, bool lower, cudaStream_t s,
                   const int* run_if = nullptr) {
  if (M <= 0 || N <= 0) return SSI_OK;
  const size_t smem = size_t(2) * TT * TLD * sizeof(double);
  cudaFuncSetAttribute(gemm_nt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  gemm_nt_kernel<<<dim3(unsigned((M + TT - 1) / TT), unsigned((N + TT - 1) / TT)), kNtThreads, smem, s>>>(
      M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, lower ? 1 : 0, run_if);
  return launch_check("gemm_nt_kernel");
}

// Diagonal panel [j0, j0 + jb) of the trailing-updated W: L11 = chol(W11) into L, L11^{-1} into
// D (jb x jb col-major, ld PB). A pivot below 64 k u times its original diagonal entry (the
// breakdown test of the one-CTA kernels) sets SSI_ERR_NUMERIC (no shifted retry at this size).
// probe != nullptr: a breakdown sets *probe (the first attempt of pass 1, which the shifted retry
// may replace); otherwise it sets SSI_ERR_NUMERIC in the status word.
__global__ void __launch_bounds__(256) chol_panel_kernel(const double* __restrict__ W, const double* __restrict__ W0diag,
                                                         int k, int j0, int jb, double* __restrict__ L,
                                                         double* __restrict__ D, int32_t* status, const int* run_if,
                                                         int* probe) {
  if (!run_enabled(run_if)) return;
  extern __shared__ double psm[];
  double (*a)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(psm);
  double (*x)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(psm + PB * (PB + 1));
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < PB * PB; e += 256) {
    const int r = e % PB, c = e / PB;
    a[r][c] = (r < jb && c < jb && r >= c) ? W[(j0 + r) + int64_t(j0 + c) * k] : 0.0;
  }
  __syncthreads();
  const double tol = 64.0 * k * 2.220446049250313e-16;
  for (int j = 0; j < jb; ++j) {
    if (tid == 0) {
      double d = a[j][j];
      if (!(d > tol * W0diag[j0 + j])) { bad = 1; d = fmax(fabs(W0diag[j0 + j]), 1e-300); }
      a[j][j] = sqrt(d);
    }
    __syncthreads();
    const double inv = 1.0 / a[j][j];
    for (int r = j + 1 + tid; r < jb; r += 256) a[r][j] *= inv;
    __syncthreads();
    // trailing rank-1 update of the lower part
    for (int e = tid; e < (jb - j - 1) * (jb - j - 1); e += 256) {
      const int r = j + 1 + e % (jb - j - 1), c = j + 1 + e / (jb - j - 1);
      if (r >= c) a[r][c] = fma(-a[r][j], a[c][j], a[r][c]);
    }
    __syncthreads();
  }
  // X = L11^{-1}: thread c solves column c by forward substitution
  if (tid < jb) {
    const int c = tid;
    for (int r = 0; r < jb; ++r) {
      double v = r == c ? 1.0 : 0.0;
      for (int p = c; p < r; ++p) v = fma(-a[r][p], x[p][c], v);
      x[r][c] = r < c ? 0.0 : v / a[r][r];
    }
  }
  __syncthreads();
  for (int e = tid; e < jb * jb; e += 256) {
    const int r = e % jb, c = e / jb;
    L[(j0 + r) + int64_t(j0 + c) * k] = r >= c ? a[r][c] : 0.0;
    D[r + c * PB] = x[r][c];
  }
  if (tid == 0 && bad) {
    if (probe) *probe = 1;
    else set_status(status, SSI_ERR_NUMERIC);
  }
}

__global__ void diag_copy_kernel(const double* __restrict__ W, int k, double* __restrict__ d, const int* run_if) {
  if (!run_enabled(run_if)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) d[i] = W[i + int64_t(i) * k];
}

__global__ void copy_cols_kernel(const double* __restrict__ src, int64_t lds, int64_t m, int64_t k,
                                 double* __restrict__ dst, const int* run_if) {
  if (!run_enabled(run_if)) return;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m * k; e += int64_t(gridDim.x) * blockDim.x)
    dst[e] = src[(e % m) + (e / m) * lds];
}

__global__ void zero_kernel(double* __restrict__ p, int64_t n, const int* run_if) {
  if (!run_enabled(run_if)) return;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    p[e] = 0.0;
}

// Shifted CholeskyQR (the one-CTA kernels' shift): W <- W0 + s I with
// s = 11 (m k + k (k + 1)) u tr(W0); one CTA.
__global__ void shift_kernel(const double* __restrict__ W0, int k, int64_t m, double* __restrict__ W,
                             const int* run_if) {
  if (!run_enabled(run_if)) return;
  __shared__ double red[32];
  double t = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) t += W0[i + int64_t(i) * k];
  t = warp_sum(t);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const double sh = 11.0 * (double(m) * k + double(k) * (k + 1)) * 1.1102230246251565e-16 * red[0];
  for (int64_t e = threadIdx.x; e < int64_t(k) * k; e += blockDim.x) {
    const int64_t r = e % k, c = e / k;
    W[e] = W0[e] + (r == c ? sh : 0.0);
  }
}

// ---------------------------------------------------------------- block one-sided Jacobi
constexpr int JB = 16;             // columns per block
constexpr int JP = 2 * JB;         // columns per pair
constexpr int JRC = 96;            // rows per staged chunk (static shared memory < 48 KB)
constexpr int kBjThreads = 256;
constexpr int kBjMaxSweeps = 40;
#ifndef SSI_BJ_INNER
#define SSI_BJ_INNER 1
#endif
constexpr int kBjInner = SSI_BJ_INNER;   // inner sweeps per pair and round (the outer sweeps revisit every pair)

struct BjArgs {
  double* G;               // k x k, col-major, leading dimension ld (even: 16-byte row pairs)
  int k, nb, ld;           // matrix size, blocks (even), leading dimension
  int* sweep_rot;          // [kBjMaxSweeps]: pairs that rotated in each sweep
  int32_t* status;
  int profile;
};

__device__ __forceinline__ int bj_col(int blk, int j, int k) {   // column of slot j of block blk, or -1
  const int c = blk * JB + j;
  return c < k ? c : -1;
}

// Row chunks of the pair's 32 columns go through a KST-stage ring of cp.async (16-byte pieces:
// the matrix is copied to an even leading dimension first) into column-major chunks
// Xc[pair column][row] (pitch XLD: m8n8k4 fragments conflict-free both ways).
constexpr int XLD = JRC + 4;                 // 100 doubles
constexpr int KST = 4;                       // ring stages
constexpr int XCH = JP * XLD;                // doubles per chunk
constexpr int PIECES = JP * (JRC / 2);       // 16-byte pieces per chunk (1536)
static_assert(PIECES % kBjThreads == 0, "pieces must split evenly");
constexpr size_t kBjSmem = size_t(KST) * XCH * sizeof(double);

__device__ __forceinline__ void bj_issue(const double* G, int k, int ld, const int (&cols)[2], int r0, double* Xc) {
#pragma unroll
  for (int u = 0; u < PIECES / kBjThreads; ++u) {
    const int q = threadIdx.x + u * kBjThreads;
    const int j = q / (JRC / 2), rr = (q % (JRC / 2)) * 2;
    const int c = bj_col(cols[j / JB], j % JB, k);
    const int rows = (c >= 0) ? min(2, k - (r0 + rr)) : 0;          // k - r0 - rr may be <= 0
    const bool ok = rows > 0;
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(Xc + j * XLD + rr));
    const double* src = ok ? G + int64_t(c) * ld + r0 + rr : G;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 * rows : 0)
                 : "memory");
  }
}
__device__ __forceinline__ void bj_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bj_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(kBjThreads) bjacobi_kernel(BjArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double xring[];   // KST chunks Xc[JP][XLD]
  __shared__ double Gm[JP][JP + 1];    // pair Gram
  __shared__ double V[JP][JP + 1];     // accumulated rotation
  __shared__ double cs_c[JP / 2], cs_s[JP / 2];
  __shared__ int cs_p[JP / 2], cs_q[JP / 2];
  __shared__ int any_rot, sweep_done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = a.k, nb = a.nb, ld = a.ld;
  const int nch = (k + JRC - 1) / JRC;
  const double tol = sqrt(double(k)) * 1.1102230246251565e-16;
  const int kq = lane & 3, r8 = lane >> 2;
  long long t_gram = 0, t_inner = 0, t_apply = 0, t_sync = 0, tc = clock64();
  for (int sweep = 0; sweep < kBjMaxSweeps; ++sweep) {
    if (tid == 0) any_rot = 0;
    for (int round = 0; round < nb - 1; ++round) {
      // round-robin: position 0 fixed, positions 1..nb-1 rotate
      const int pa = blockIdx.x, pb = nb - 1 - blockIdx.x;
      const int ba = pa == 0 ? 0 : 1 + (pa - 1 + round) % (nb - 1);
      const int bb = 1 + (pb - 1 + round) % (nb - 1);
      int cols[2] = {ba < bb ? ba : bb, ba < bb ? bb : ba};
      // ---- Gram of the pair's columns, row chunks through shared memory (DMMA, 16 tiles)
      // warp w: tile row ti = w & 3 (4 tiles of 8 x 8), row half w >> 2 of every chunk (4-way ILP);
      // the two halves are summed in a fixed order
      double g[4][2];
#pragma unroll
      for (int tj = 0; tj < 4; ++tj) g[tj][0] = g[tj][1] = 0.0;
      const int ti = warp & 3, kh = (warp >> 2) * (JRC / 2);
#pragma unroll
      for (int c0 = 0; c0 < KST - 1; ++c0) {
        if (c0 < nch) bj_issue(a.G, k, ld, cols, c0 * JRC, xring + c0 * XCH);
        bj_commit();
      }
      for (int ch = 0; ch < nch; ++ch) {
        bj_wait<KST - 2>();
        __syncthreads();                       // chunk ch landed; slot (ch - 1) % KST is free
        if (ch + KST - 1 < nch) bj_issue(a.G, k, ld, cols, (ch + KST - 1) * JRC, xring + ((ch + KST - 1) % KST) * XCH);
        bj_commit();
        const double* Xc = xring + (ch % KST) * XCH;
#pragma unroll 4
        for (int kk = kh; kk < kh + JRC / 2; kk += 4) {
          // A = X^T (pair column, row), B = X (row, pair column): both Xc[column][row]
          const double a0 = Xc[(8 * ti + r8) * XLD + kk + kq];
#pragma unroll
          for (int tj = 0; tj < 4; ++tj) dmma884(g[tj][0], g[tj][1], a0, Xc[(8 * tj + r8) * XLD + kk + kq]);
        }
      }
      bj_wait<0>();
      __syncthreads();
      { const long long t = clock64(); t_gram += t - tc; tc = t; }
      if (warp >= 4)
#pragma unroll
        for (int tj = 0; tj < 4; ++tj)
#pragma unroll
          for (int h = 0; h < 2; ++h) Gm[8 * ti + r8][8 * tj + 2 * kq + h] = g[tj][h];
      __syncthreads();
      if (warp < 4)
#pragma unroll
        for (int tj = 0; tj < 4; ++tj)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double& d = Gm[8 * ti + r8][8 * tj + 2 * kq + h];
            d = g[tj][h] + d;
          }
      for (int e = tid; e < JP * JP; e += kBjThreads) V[e / JP][e % JP] = (e / JP == e % JP) ? 1.0 : 0.0;
      __syncthreads();
      // ---- diagonalise the pair Gram: parallel-ordered Jacobi sweeps (16 disjoint pairs a step:
      // angles, then G <- J^T G, then G <- G J and V <- V J; a pair below the threshold keeps
      // c = 1, s = 0, which leaves its rows and columns bit-for-bit unchanged)
      int rotated = 0;
      for (int inner = 0; inner < kBjInner; ++inner) {
        int inner_rot = 0;
        for (int st = 0; st < JP - 1; ++st) {
          int on = 0;
          if (tid < JP / 2) {
            const int q0 = tid, q1 = JP - 1 - tid;
            int p = q0 == 0 ? 0 : 1 + (q0 - 1 + st) % (JP - 1);
            int q = 1 + (q1 - 1 + st) % (JP - 1);
            if (p > q) { const int t = p; p = q; q = t; }
            const double al = Gm[p][p], be = Gm[q][q], ga = Gm[p][q];
            double c = 1.0, s = 0.0;
            if (ga != 0.0 && ga * ga > tol * tol * (al * be)) {
              // zeta = (be - al) / (2 ga); t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2));
              // c = 1 / sqrt(1 + t^2), s = c t  (Newton-refined reciprocal / rsqrt: a few ulp)
              const double zeta = (be - al) * fast_rcp(2.0 * ga);
              const double r1 = fast_rsqrt(fma(zeta, zeta, 1.0));
              const double hyp = fma(zeta, zeta, 1.0) * r1;          // sqrt(1 + zeta^2)
              const double t = copysign(fast_rcp(fabs(zeta) + hyp), zeta);
              c = fast_rsqrt(fma(t, t, 1.0));
              s = c * t;
              on = 1;
            }
            cs_p[tid] = p; cs_q[tid] = q; cs_c[tid] = c; cs_s[tid] = s;
          }
          if (__syncthreads_or(on)) inner_rot = 1;
          // rows: G <- J^T G (thread: (pair, column))
          for (int e = tid; e < (JP / 2) * JP; e += kBjThreads) {
            const int pr = e / JP, j = e % JP;
            const int p = cs_p[pr], q = cs_q[pr];
            const double c = cs_c[pr], s = cs_s[pr];
            const double x = Gm[p][j], y = Gm[q][j];
            Gm[p][j] = c * x - s * y;
            Gm[q][j] = s * x + c * y;
          }
          __syncthreads();
          // columns: G <- G J, V <- V J
          for (int e = tid; e < (JP / 2) * JP * 2; e += kBjThreads) {
            const int which = e / ((JP / 2) * JP), f = e % ((JP / 2) * JP);
            const int pr = f / JP, j = f % JP;
            const int p = cs_p[pr], q = cs_q[pr];
            const double c = cs_c[pr], s = cs_s[pr];
            double (*Mx)[JP + 1] = which ? V : Gm;
            const double x = Mx[j][p], y = Mx[j][q];
            Mx[j][p] = c * x - s * y;
            Mx[j][q] = s * x + c * y;
          }
          __syncthreads();
        }
        rotated |= inner_rot;
        if (!inner_rot) break;
      }
      { const long long t = clock64(); t_inner += t - tc; tc = t; }
      // ---- X <- X V for the pair's columns (row chunks, DMMA: chunk (JRC x 32) * V (32 x 32))
      if (rotated) {
#pragma unroll
        for (int c0 = 0; c0 < KST - 1; ++c0) {
          if (c0 < nch) bj_issue(a.G, k, ld, cols, c0 * JRC, xring + c0 * XCH);
          bj_commit();
        }
        for (int ch = 0; ch < nch; ++ch) {
          const int r0 = ch * JRC;
          bj_wait<KST - 2>();
          __syncthreads();
          if (ch + KST - 1 < nch) bj_issue(a.G, k, ld, cols, (ch + KST - 1) * JRC, xring + ((ch + KST - 1) % KST) * XCH);
          bj_commit();
          const double* Xc = xring + (ch % KST) * XCH;
          // output tiles: (JRC/8) x 4, TPW per warp
          constexpr int TPW = JRC / 16;
          double acc[TPW][2];
#pragma unroll
          for (int u = 0; u < TPW; ++u) acc[u][0] = acc[u][1] = 0.0;
#pragma unroll
          for (int kk = 0; kk < JP; kk += 4) {
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
              const int t = warp * TPW + u, ti = t / 4, tj = t % 4;
              const double af = Xc[(kk + kq) * XLD + 8 * ti + r8];
              const double bf = V[kk + kq][8 * tj + r8];
              dmma884(acc[u][0], acc[u][1], af, bf);
            }
          }
#pragma unroll
          for (int u = 0; u < TPW; ++u) {
            const int t = warp * TPW + u, ti = t / 4, tj = t % 4;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int rr = 8 * ti + r8, j = 8 * tj + 2 * kq + h;
              const int c = bj_col(cols[j / JB], j % JB, k);
              if (c >= 0 && r0 + rr < k) __stcg(a.G + int64_t(c) * ld + r0 + rr, acc[u][h]);
            }
          }
        }
        bj_wait<0>();
        __syncthreads();
        if (tid == 0) any_rot = 1;
      }
      { const long long t = clock64(); t_apply += t - tc; tc = t; }
      grid.sync();
      { const long long t = clock64(); t_sync += t - tc; tc = t; }
    }
    if (tid == 0 && any_rot) atomicAdd(a.sweep_rot + sweep, 1);
    grid.sync();
    if (tid == 0) sweep_done = (__ldcg(a.sweep_rot + sweep) == 0);
    __syncthreads();
    if (sweep_done) {
      if (a.profile && blockIdx.x == 0 && tid == 0)
        printf("bjacobi k=%d: %d sweeps of %d rounds; cycles gram %lld inner %lld apply %lld sync %lld\n", k,
               sweep + 1, nb - 1, t_gram, t_inner, t_apply, t_sync);
      return;
    }
  }
  if (blockIdx.x == 0 && tid == 0) set_status(a.status, SSI_ERR_NUMERIC);
}

// singular values = column norms; ranks by counting (descending, ties by index); Ut columns
__global__ void bj_norms_kernel(const double* __restrict__ G, int k, int ld, double* __restrict__ nrm) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= k) return;
  double a = 0.0;
  for (int r = lane; r < k; r += 32) { const double x = G[int64_t(j) * ld + r]; a = fma(x, x, a); }
  a = warp_sum(a);
  if (lane == 0) nrm[j] = sqrt(a);
}

__global__ void bj_rank_kernel(const double* __restrict__ nrm, int k, int* __restrict__ rank, double* __restrict__ S) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const double v = nrm[j];
  int rk = 0;
  for (int i = 0; i < k; ++i) rk += (nrm[i] > v) || (nrm[i] == v && i < j);
  rank[j] = rk;
  S[rk] = v;
}

__global__ void bj_out_kernel(const double* __restrict__ G, int k, int ld, const double* __restrict__ nrm,
                              const int* __restrict__ rank, double* __restrict__ Ut) {
  const int j = blockIdx.y;
  const double inv = nrm[j] > 0.0 ? 1.0 / nrm[j] : 0.0;
  const int dst = rank[j];
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < k; r += gridDim.x * blockDim.x)
    Ut[int64_t(dst) * k + r] = G[int64_t(j) * ld + r] * inv;
}

__global__ void bj_copy_kernel(const double* __restrict__ src, int k, int ld, double* __restrict__ dst) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(k) * k;
       e += int64_t(gridDim.x) * blockDim.x)
    dst[(e % k) + (e / k) * ld] = src[e];
}

}  // namespace

constexpr size_t kPanelSmem = size_t(2) * PB * (PB + 1) * sizeof(double);

size_t cholqr_big_panel_elems(int k) { return size_t((k + PB - 1) / PB) * PB * PB + size_t(k); }

// Blocked right-looking Cholesky of W (k x k col-major, lower part; overwritten by the trailing
// updates) into L (lower, zero upper) with the panel inverses in D. run_if: conditional launch;
// probe: breakdown flag instead of the status word (see chol_panel_kernel).
ssi_status chol_big(double* W, int k, double* L, double* D, int32_t* status, cudaStream_t s,
                    const int* run_if = nullptr, int* probe = nullptr) {
  double* d0 = D + size_t((k + PB - 1) / PB) * PB * PB;    // original diagonal (breakdown test)
  cudaFuncSetAttribute(chol_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPanelSmem));
  diag_copy_kernel<<<(k + 255) / 256, 256, 0, s>>>(W, k, d0, run_if);
  SSI_TRY(launch_check("diag_copy_kernel"));
  zero_kernel<<<148 * 4, 256, 0, s>>>(L, int64_t(k) * k, run_if);
  SSI_TRY(launch_check("zero_kernel"));
  for (int j0 = 0; j0 < k; j0 += PB) {
    const int jb = k - j0 < PB ? k - j0 : PB;
    double* Dj = D + size_t(j0 / PB) * PB * PB;
    chol_panel_kernel<<<1, 256, kPanelSmem, s>>>(W, d0, k, j0, jb, L, Dj, status, run_if, probe);
    SSI_TRY(launch_check("chol_panel_kernel"));
    const int rest = k - j0 - jb;
    if (rest <= 0) break;
    // L21 = W21 L11^{-T}
    SSI_TRY(gemm_nt(rest, jb, jb, W + (j0 + jb) + int64_t(j0) * k, k, Dj, PB, L + (j0 + jb) + int64_t(j0) * k, k,
                    0.0, 1.0, false, s, run_if));
    // W22 -= L21 L21^T (lower tiles)
    SSI_TRY(gemm_nt(rest, rest, jb, L + (j0 + jb) + int64_t(j0) * k, k, L + (j0 + jb) + int64_t(j0) * k, k,
                    W + (j0 + jb) + int64_t(j0 + jb) * k, k, 1.0, -1.0, true, s, run_if));
  }
  return SSI_OK;
}

// In place X <- X L^{-T} (X m x k col-major, ld m): block column j: X_j <- X_j D_j^T, then
// X_{j+} -= X_j L_{j+, j}^T.
ssi_status trsm_big(double* X, int64_t m, int k, const double* L, const double* D, cudaStream_t s,
                    const int* run_if = nullptr) {
  for (int j0 = 0; j0 < k; j0 += PB) {
    const int jb = k - j0 < PB ? k - j0 : PB;
    const double* Dj = D + size_t(j0 / PB) * PB * PB;
    double* Xj = X + int64_t(j0) * m;
    SSI_TRY(gemm_nt(m, jb, jb, Xj, m, Dj, PB, Xj, m, 0.0, 1.0, false, s, run_if));
    const int rest = k - j0 - jb;
    if (rest <= 0) break;
    SSI_TRY(gemm_nt(m, rest, jb, Xj, m, L + (j0 + jb) + int64_t(j0) * k, k, X + int64_t(j0 + jb) * m, m, 1.0, -1.0,
                    false, s, run_if));
  }
  return SSI_OK;
}

// Cholesky with the shifted retry of the one-CTA path, as conditional launches: the first
// attempt (under run_if) only raises *flag on a breakdown; then W <- W0 + s I and a second
// attempt run only if *flag is set (a breakdown of that one sets SSI_ERR_NUMERIC).
static ssi_status chol_retry(double* W, double* W0, int k, int64_t m, double* L, double* D, int32_t* status,
                             cudaStream_t s, const int* run_if, int* flag) {
  copy_cols_kernel<<<148 * 4, 256, 0, s>>>(W, k, k, k, W0, run_if);
  SSI_TRY(launch_check("copy_cols_kernel"));
  SSI_TRY(chol_big(W, k, L, D, status, s, run_if, flag));
  shift_kernel<<<1, 1024, 0, s>>>(W0, k, m, W, flag);
  SSI_TRY(launch_check("shift_kernel"));
  return chol_big(W, k, L, D, status, s, flag, nullptr);
}

// CholeskyQR2 for k > kSvdMaxK, with the shifted-CholeskyQR fallback decided on the device. Pass 1
// retries its Cholesky on W0 + s I after a breakdown; then up to kCqExtraPasses extra passes run,
// each only if the previous pass shifted, each shifting again on a breakdown; the final pass must
// factor unshifted (else SSI_ERR_NUMERIC). Y = Q R with R^T = L1 (Lb_1 ... Lb_n) L2, the product
// of the extra passes' factors accumulated in La and folded into L2.
// Why more than one extra pass (unlike the one-CTA path's single pass, whose explicit inverses add
// error of order u kappa(L)^2): on an exactly rank-deficient Y the columns beyond the rank are
// rounding noise, which each shifted pass scales up by about 1 / sqrt(s) ~ 1e4 relative to the
// signal; the accurate blocked solves keep that noise small, so it takes two or three shifted
// passes before those columns are O(1) and the final pass completes an orthonormal basis.
ssi_status cholqr2_big(const double* Y, int64_t ldy, int64_t m, int k, double* Q, CholQRWork& w, int32_t* status,
                       cudaStream_t s) {
  const int splits = gemm_pick_splits(k, k, m);
  int* f = w.flag;   // f[0]: pass 1 shifted; f[j]: extra pass j shifted (gates extra pass j + 1)
  if (cudaMemsetAsync(w.flag, 0, (1 + kCqExtraPasses) * sizeof(int), s) != cudaSuccess)
    return launch_check("cholqr2_big flag");
  SSI_TRY(gemm_f64(k, k, m, 1.0, Operand{Y, ldy, 1}, Operand{Y, 1, ldy}, w.W, k, splits, w.partial, s));
  SSI_TRY(chol_retry(w.W, w.W0, k, m, w.L1, w.Dp1, status, s, nullptr, f));
  copy_cols_kernel<<<148 * 8, 256, 0, s>>>(Y, ldy, m, k, w.Q1, nullptr);
  SSI_TRY(launch_check("copy_cols_kernel"));
  SSI_TRY(trsm_big(w.Q1, m, k, w.L1, w.Dp1, s));
  for (int j = 1; j <= kCqExtraPasses; ++j) {   // extra pass j: Q1 <- Q1 Lb^{-T}, La <- La Lb
    const int* run = f + j - 1;
    SSI_TRY(gemm_f64(k, k, m, 1.0, Operand{w.Q1, m, 1}, Operand{w.Q1, 1, m}, w.W, k, splits, w.partial, s, run));
    SSI_TRY(chol_retry(w.W, w.W0, k, m, w.Lb, w.Dp2, status, s, run, f + j));
    SSI_TRY(trsm_big(w.Q1, m, k, w.Lb, w.Dp2, s, run));
    if (j == 1) {
      copy_cols_kernel<<<148 * 8, 256, 0, s>>>(w.Lb, k, k, k, w.La, run);
    } else {
      SSI_TRY(gemm_f64(k, k, k, 1.0, Operand{w.La, 1, k}, Operand{w.Lb, 1, k}, w.W, k, 1, nullptr, s, run));
      copy_cols_kernel<<<148 * 8, 256, 0, s>>>(w.W, k, k, k, w.La, run);
    }
    SSI_TRY(launch_check("copy_cols_kernel"));
  }
  // final pass
  SSI_TRY(gemm_f64(k, k, m, 1.0, Operand{w.Q1, m, 1}, Operand{w.Q1, 1, m}, w.W, k, splits, w.partial, s));
  SSI_TRY(chol_big(w.W, k, w.L2, w.Dp2, status, s));
  if (cudaMemcpyAsync(Q, w.Q1, sizeof(double) * size_t(m) * k, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return launch_check("cholqr2_big copy");
  SSI_TRY(trsm_big(Q, m, k, w.L2, w.Dp2, s));
  // fold: L2 <- La L2 (both lower triangular; only after a shift)
  SSI_TRY(gemm_f64(k, k, k, 1.0, Operand{w.La, 1, k}, Operand{w.L2, 1, k}, w.W, k, 1, nullptr, s, f));
  copy_cols_kernel<<<148 * 8, 256, 0, s>>>(w.W, k, k, k, w.L2, f);
  return launch_check("copy_cols_kernel");
}

size_t jacobi_big_scratch_elems(int k) {
  return size_t(k) + size_t(k) + kBjMaxSweeps + 2 + size_t(k + (k & 1)) * k;
}

int jacobi_big_ctas(int k) {
  int nb = (k + JB - 1) / JB;
  nb += nb & 1;
  return nb / 2;
}

ssi_status jacobi_big(double* G, int k, double* Ut, double* S, double* scratch, int32_t* status, cudaStream_t s) {
  int nb = (k + JB - 1) / JB;
  nb += nb & 1;
  double* nrm = scratch;
  int* rank = reinterpret_cast<int*>(scratch + k);
  int* flags = reinterpret_cast<int*>(scratch + 2 * size_t(k));
  if (cudaMemsetAsync(flags, 0, sizeof(int) * kBjMaxSweeps, s) != cudaSuccess) return launch_check("memset flags");
  // working copy with an even leading dimension (16-byte cp.async pieces of two rows)
  const int ld = k + (k & 1);
  double* Gp = scratch + 2 * size_t(k) + kBjMaxSweeps + 2;
  Gp = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(Gp) + 15) & ~uintptr_t(15));
  bj_copy_kernel<<<148 * 8, 256, 0, s>>>(G, k, ld, Gp);
  SSI_TRY(launch_check("bj_copy_kernel"));
  BjArgs a{Gp, k, nb, ld, flags, status, getenv("SSI_JAC_PROFILE") ? 1 : 0};
  void* args[] = {&a};
  cudaFuncSetAttribute(bjacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kBjSmem));
  if (cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bjacobi_kernel), dim3(unsigned(nb / 2)), dim3(kBjThreads),
                                  args, kBjSmem, s) != cudaSuccess)
    return launch_check("bjacobi_kernel (cooperative launch)");
  bj_norms_kernel<<<(k + 7) / 8, 256, 0, s>>>(Gp, k, ld, nrm);
  SSI_TRY(launch_check("bj_norms_kernel"));
  bj_rank_kernel<<<(k + 255) / 256, 256, 0, s>>>(nrm, k, rank, S);
  SSI_TRY(launch_check("bj_rank_kernel"));
  bj_out_kernel<<<dim3(unsigned((k + 255) / 256), unsigned(k)), 256, 0, s>>>(Gp, k, ld, nrm, rank, Ut);
  return launch_check("bj_out_kernel");
}

}  // namespace ssi
