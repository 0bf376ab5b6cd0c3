// FP64 tensor-core GEMM (mma.sync m8n8k4 -> SASS DMMA) used by the RSVD passes
// T*Omega, T^T*Q, T*Z (Eqs. 14-15), the CholeskyQR2 Gram products
// and triangular multiplies, and U = Q*U~ (Eq. 18). FP64 is required for parity
// (a BF16x3 sketch moves physical poles by 1.6e-4).
#pragma once
#include "common.cuh"

namespace ssi {

// Strided operand: element (r, c) at p[r*s_r + c*s_c].
struct Operand {
  const double* p;
  int64_t s_r, s_c;
};

// Conditional launches: a kernel given run_if != nullptr returns at once unless *run_if != 0
// (a device flag written by an earlier kernel on the same stream; used by the CholeskyQR
// breakdown fallback, whose extra pass must not cost a host synchronisation).
__device__ __forceinline__ bool run_enabled(const int* run_if) {
  return run_if == nullptr || *reinterpret_cast<const volatile int*>(run_if) != 0;
}

// C (M x N, col-major, ldc) = alpha * A (M x K) * B (K x N).
// A is "k-contiguous" when s_c == 1 (row-major), otherwise s_r must be 1 (col-major);
// likewise B is k-contiguous when s_r == 1. splits > 1 partitions K, writes partials to
// `partial` ([splits][M*N]) and reduces them in fixed order (deterministic).
ssi_status gemm_f64(int64_t M, int64_t N, int64_t K, double alpha, Operand A, Operand B,
                    double* C, int64_t ldc, int splits, double* partial, cudaStream_t s,
                    const int* run_if = nullptr);

// Heuristic split count so that tiles*splits fills the 148 SMs a few times over.
int gemm_pick_splits(int64_t M, int64_t N, int64_t K);
size_t gemm_partial_elems(int64_t M, int64_t N, int splits);

// Batched "order" GEMM for the modal sweep: for b in [0, nb), n_b = n0 + b*dn,
// C_b (n_b x n_b col-major, at Cbase + off_b, off_b = sum_{b'<b} n_b'^2) =
//   A[:n_b, :n_b] * B[:n_b, :n_b] with A, B col-major (ld lda, ldb).
ssi_status gemm_f64_orders(int nb, int n0, int dn, const double* A, int64_t lda,
                           const double* B, int64_t ldb, double* Cbase, cudaStream_t s);

}  // namespace ssi

namespace ssi {
// Tall-skinny FP64 DMMA GEMM for the RSVD passes (N <= 224): C (M x N, col-major, ldc) =
// op(A) (M x K) * B (K x N); A row-major (a_rowmajor: A(i,k) = A[i*lda + k]) or col-major
// (A[i + k*lda]); B col-major (B(k,j) = B[k + j*ldb]). One 64 x 224 tile per CTA, 3-stage
// cp.async pipeline, split-K over whole waves with a fixed-order reduction.
ssi_status gemm_tall(int64_t M, int64_t N, int64_t K, bool a_rowmajor, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* C, int64_t ldc, double* partial, cudaStream_t s);
size_t gemm_tall_partial_elems(int64_t M, int64_t N, int64_t K);
constexpr int kTallMaxN = 224;
// Batched form without split-K: for b in [0, batch), C_b = op(A_b) B_b with
// A_b = A + b*sA, B_b = B + b*sB, C_b = C + b*sC (N <= kTallMaxN; lda, ldb even).
// Lower-triangular 64 x 64 tiles of C (n x n) = op(A) (n x K) B (K x n) (A row-major: op(A)(i,k) =
// A[i*lda + k]); the strictly-upper off-diagonal tiles of C are not written. partial: at least
// 64 n^2 doubles (split-K slabs).
ssi_status gemm_tall_syrk_lower(int64_t n, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                                double* C, int64_t ldc, double* partial, cudaStream_t s,
                                const int* run_if = nullptr);
// C (M x N) = A (M x K, col-major) B (K x N, col-major upper triangular, K == N): the N tile at
// j0 reads only K rows [0, j0 + 64).
ssi_status gemm_tall_triu(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                          int64_t ldb, double* C, int64_t ldc, cudaStream_t s, const int* run_if = nullptr);
ssi_status gemm_tall_batched(int64_t M, int64_t N, int64_t K, bool a_rowmajor, const double* A, int64_t lda,
                             int64_t sA, const double* B, int64_t ldb, int64_t sB, double* C, int64_t ldc,
                             int64_t sC, int batch, cudaStream_t s);
// max of gemm_tall_partial_elems(m, N, m) over m <= M (workspace for every smaller square size)
size_t gemm_tall_partial_elems_upto(int64_t M, int64_t N);
}  // namespace ssi
