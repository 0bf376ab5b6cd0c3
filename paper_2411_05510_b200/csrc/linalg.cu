// Small dense FP64 kernels of the RSVD (A5, A8): Cholesky + triangular inverse for
// CholeskyQR2, and a one-sided Jacobi SVD for the k x k factor of B = Q^T T
// (Eq. 16). One CTA per problem; latency-bound by construction.
#include "linalg.cuh"

namespace ssi {
namespace {

constexpr int kCholThreads = 256;
constexpr int kJacThreads = 1024;

__device__ __forceinline__ int64_t tri(int64_t i) { return i * (i + 1) / 2; }

// W (k x k col-major, lower part read) -> L (lower) and Linv = L^{-1} (lower), both
// col-major ld k with zeros above the diagonal. Packed row-major lower triangle P
// (P[i(i+1)/2 + c], c <= i) in shared memory when it fits, else in gscratch.
__global__ void __launch_bounds__(kCholThreads) chol_inv_kernel(const double* __restrict__ W, int k,
                                                                double* __restrict__ L,
                                                                double* __restrict__ Linv,
                                                                double* gscratch, int use_smem,
                                                                int32_t* status) {
  extern __shared__ __align__(16) double sm[];
  double* vec = sm;                  // k: scaled column j / row i of L
  double* P = use_smem ? sm + k : gscratch;
  __shared__ int fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) fail = 0;
  for (int64_t e = tid; e < tri(k); e += nt) {
    // row i, col c of packed index e
    int64_t i = int64_t((sqrt(8.0 * double(e) + 1.0) - 1.0) * 0.5);
    while (tri(i + 1) <= e) ++i;
    while (tri(i) > e) --i;
    const int64_t c = e - tri(i);
    P[e] = W[i + c * int64_t(k)];
  }
  __syncthreads();
  // Right-looking Cholesky, column by column.
  for (int j = 0; j < k; ++j) {
    if (tid == 0) {
      const double d = P[tri(j) + j];
      if (!(d > 0.0) || !isfinite(d)) { fail = 1; P[tri(j) + j] = 1.0; }
      else P[tri(j) + j] = sqrt(d);
    }
    __syncthreads();
    const double djj = P[tri(j) + j];
    for (int i = j + 1 + tid; i < k; i += nt) {
      const double v = P[tri(i) + j] / djj;
      P[tri(i) + j] = v;
      vec[i] = v;
    }
    __syncthreads();
    // trailing update P[i][c] -= L[i][j] L[c][j], j < c <= i: warp per row i
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (int i = j + 1 + warp; i < k; i += nw) {
      const double li = vec[i];
      double* row = P + tri(i);
      for (int c = j + 1 + lane; c <= i; c += 32) row[c] -= li * vec[c];
    }
    __syncthreads();
  }
  if (fail) set_status(status, SSI_ERR_NUMERIC);
  // write L (col-major, zero upper)
  for (int64_t e = tid; e < int64_t(k) * k; e += nt) {
    const int64_t r = e % k, c = e / k;
    L[e] = (c <= r) ? P[tri(r) + c] : 0.0;
  }
  __syncthreads();
  // In-place inverse: row i of X = L^{-1} overwrites row i of L.
  //   X[i][j] = (delta_ij - sum_{p=j}^{i-1} L[i][p] X[p][j]) / L[i][i]
  for (int i = 0; i < k; ++i) {
    for (int p = tid; p <= i; p += nt) vec[p] = P[tri(i) + p];
    __syncthreads();
    const double lii = vec[i];
    for (int j = tid; j <= i; j += nt) {
      double s0 = (j == i) ? 1.0 : 0.0, s1 = 0.0;
      int p = j;
      for (; p + 1 < i; p += 2) {
        s0 -= vec[p] * P[tri(p) + j];
        s1 -= vec[p + 1] * P[tri(p + 1) + j];
      }
      if (p < i) s0 -= vec[p] * P[tri(p) + j];
      P[tri(i) + j] = (s0 + s1) / lii;
    }
    __syncthreads();
  }
  for (int64_t e = tid; e < int64_t(k) * k; e += nt) {
    const int64_t r = e % k, c = e / k;
    Linv[e] = (c <= r) ? P[tri(r) + c] : 0.0;
  }
}

// One-sided Jacobi with the round-robin (circle) ordering; warp per column pair.
__global__ void __launch_bounds__(kJacThreads) jacobi_kernel(double* __restrict__ G, int k,
                                                             double* __restrict__ Ut,
                                                             double* __restrict__ S,
                                                             int32_t* status) {
  extern __shared__ __align__(16) double jsm[];
  double* nrm = jsm;                                    // k
  int* arr = reinterpret_cast<int*>(jsm + k);           // n (even)
  int* rank = arr + (k + 2);                            // k
  __shared__ int rot;
  const int n = (k + 1) & ~1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < n; i += blockDim.x) arr[i] = i;
  const double tol = sqrt(double(k)) * 1.1102230246251565e-16;
  int sweep = 0;
  bool converged = false;
  __syncthreads();
  for (; sweep < 60 && !converged; ++sweep) {
    if (tid == 0) rot = 0;
    __syncthreads();
    for (int round = 0; round < n - 1; ++round) {
      for (int pr = warp; pr < n / 2; pr += nw) {
        int p = arr[pr], q = arr[n - 1 - pr];
        if (p >= k || q >= k) continue;
        if (p > q) { const int t = p; p = q; q = t; }
        double* gp = G + int64_t(p) * k;
        double* gq = G + int64_t(q) * k;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = lane; r < k; r += 32) {
          const double x = gp[r], y = gq[r];
          al += x * x; be += y * y; ga += x * y;
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        if (fabs(ga) > tol * sqrt(al * be) && ga != 0.0) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int r = lane; r < k; r += 32) {
            const double x = gp[r], y = gq[r];
            gp[r] = c * x - s * y;
            gq[r] = s * x + c * y;
          }
          if (lane == 0) atomicAdd(&rot, 1);
        }
      }
      __syncthreads();
      // rotate positions 1..n-1 by one (position 0 fixed)
      if (tid == 0) {
        const int last = arr[n - 1];
        for (int i = n - 1; i > 1; --i) arr[i] = arr[i - 1];
        arr[1] = last;
      }
      __syncthreads();
    }
    converged = (rot == 0);
    __syncthreads();
  }
  if (!converged && tid == 0) set_status(status, SSI_ERR_NUMERIC);
  // singular values = column norms; sort descending (rank by counting, ties by index)
  for (int j = warp; j < k; j += nw) {
    double s = 0.0;
    for (int r = lane; r < k; r += 32) s += G[int64_t(j) * k + r] * G[int64_t(j) * k + r];
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < k; j += blockDim.x) {
    int rk = 0;
    const double v = nrm[j];
    for (int i = 0; i < k; ++i) rk += (nrm[i] > v) || (nrm[i] == v && i < j);
    rank[j] = rk;
    S[rk] = v;
  }
  __syncthreads();
  for (int j = warp; j < k; j += nw) {
    const double inv = nrm[j] > 0.0 ? 1.0 / nrm[j] : 0.0;
    const int dst = rank[j];
    for (int r = lane; r < k; r += 32) Ut[int64_t(dst) * k + r] = G[int64_t(j) * k + r] * inv;
  }
}

}  // namespace

size_t cholqr_partial_elems(int64_t m, int k) {
  return gemm_partial_elems(k, k, gemm_pick_splits(k, k, m));
}

void cholqr_carve(Carver& c, int64_t m, int k, CholQRWork& w) {
  w.W = c.take<double>(size_t(k) * k);
  w.L1 = c.take<double>(size_t(k) * k);
  w.Linv1 = c.take<double>(size_t(k) * k);
  w.L2 = c.take<double>(size_t(k) * k);
  w.Linv2 = c.take<double>(size_t(k) * k);
  w.Q1 = c.take<double>(size_t(m) * k);
  w.chol_g = c.take<double>(size_t(k) * (k + 1) / 2);
  w.partial = c.take<double>(cholqr_partial_elems(m, k) + 1);
}

static size_t chol_smem_bytes(int k) { return (size_t(k) + size_t(k) * (k + 1) / 2) * sizeof(double); }

ssi_status chol_inv(const double* W, int k, double* L, double* Linv, double* gscratch,
                    int32_t* status, cudaStream_t s) {
  const size_t smem_full = chol_smem_bytes(k);
  const bool use_smem = smem_full <= 220 * 1024;
  const size_t smem = use_smem ? smem_full : size_t(k) * sizeof(double);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  }
  chol_inv_kernel<<<1, kCholThreads, smem, s>>>(W, k, L, Linv, gscratch, use_smem ? 1 : 0, status);
  return launch_check("chol_inv_kernel");
}

ssi_status cholqr2(const double* Y, int64_t ldy, int64_t m, int k, double* Q, CholQRWork& w,
                   int32_t* status, cudaStream_t s) {
  const int splits = gemm_pick_splits(k, k, m);
  // W = Y^T Y : A(i,kk) = Y[kk + i*ldy] (k-contiguous), B(kk,j) = Y[kk + j*ldy]
  SSI_TRY(gemm_f64(k, k, m, 1.0, Operand{Y, ldy, 1}, Operand{Y, 1, ldy}, w.W, k, splits,
                   w.partial, s));
  SSI_TRY(chol_inv(w.W, k, w.L1, w.Linv1, w.chol_g, status, s));
  // Q1 = Y Linv1^T : B(kk,j) = Linv1[j + kk*k]
  SSI_TRY(gemm_f64(m, k, k, 1.0, Operand{Y, 1, ldy}, Operand{w.Linv1, k, 1}, w.Q1, m, 1,
                   nullptr, s));
  SSI_TRY(gemm_f64(k, k, m, 1.0, Operand{w.Q1, m, 1}, Operand{w.Q1, 1, m}, w.W, k, splits,
                   w.partial, s));
  SSI_TRY(chol_inv(w.W, k, w.L2, w.Linv2, w.chol_g, status, s));
  return gemm_f64(m, k, k, 1.0, Operand{w.Q1, 1, m}, Operand{w.Linv2, k, 1}, Q, m, 1, nullptr, s);
}

ssi_status jacobi_svd(double* G, int k, double* Ut, double* S, int32_t* status, cudaStream_t s) {
  const size_t smem = size_t(k) * sizeof(double) + size_t(2 * k + 4) * sizeof(int);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  jacobi_kernel<<<1, kJacThreads, smem, s>>>(G, k, Ut, S, status);
  return launch_check("jacobi_kernel");
}

}  // namespace ssi
