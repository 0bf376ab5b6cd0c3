#pragma once
#include "common.cuh"
#include "gemm_f64.cuh"

namespace ssi {

// Scratch for one CholeskyQR2 of an m x k matrix.
struct CholQRWork {
  double* W;        // k x k Gram
  double* L1;       // k x k lower, first Cholesky factor
  double* Linv1;    // k x k lower, its inverse
  double* L2;
  double* Linv2;
  double* LinvT1;   // Linv1^T and Linv2^T (col-major k x k): B operands of the tall products
  double* LinvT2;
  double* Lb;       // k x k factors of the fallback pass (shifted CholeskyQR3)
  double* Linvb;
  double* LinvTb;
  int* flag;        // 1 when pass 1 needed the shift (device; read by the conditional launches);
                    //   k > kSvdMaxK: one flag per pass (1 + kCqExtraPasses)
  double* Q1;       // m x k intermediate
  double* chol_g;   // packed triangle when k is too large for shared memory
  double* partial;  // split-K partials
  double* tallp;    // split-K partials of the tall-skinny kernels
  double* Dp1;      // k > kSvdMaxK (linalg_big.cu): 64 x 64 panel inverses of L1 / L2 and the
  double* Dp2;      //   original Gram diagonal
  double* W0;       // k > kSvdMaxK: the unshifted Gram matrix of a pass (shifted retry)
  double* La;       // k > kSvdMaxK: product of the extra passes' factors
};
size_t cholqr_partial_elems(int64_t m, int k);
void cholqr_carve(Carver& c, int64_t m, int k, CholQRWork& w);

// CholeskyQR2 (A5; "qr(Y,0)"): Y = Q R, R = L2^T L1^T upper with
// positive diagonal (R^{-1} = Linv1^T Linv2^T). Y: m x k col-major (ldy); Q: m x k col-major
// (ld m). When the first Cholesky breaks down (Y numerically rank-deficient) it is redone with a
// diagonal shift and one extra CholeskyQR pass runs (shifted CholeskyQR3), decided on the device;
// the returned factors then include that pass.
ssi_status cholqr1(const double* Y, int64_t ldy, int64_t m, int k, double* Q, CholQRWork& w,
                   int32_t* status, cudaStream_t s);
ssi_status cholqr2(const double* Y, int64_t ldy, int64_t m, int k, double* Q, CholQRWork& w,
                   int32_t* status, cudaStream_t s);

// Single-CTA Cholesky W = L L^T and L^{-1} (lower, col-major ld k), k <= 512, with one shifted
// retry on breakdown (*shifted_out = 1); run_if: conditional launch; final: a shift is an error.
ssi_status chol_inv(const double* W, int k, int64_t m, double* L, double* Linv, double* LinvT, double* gscratch,
                    int32_t* status, cudaStream_t s, const int* run_if, int* shifted_out, int final);

// Largest sketch width of the one-SM kernels (Cholesky, one-sided Jacobi on one 8/16-CTA cluster);
// above it the blocked whole-GPU kernels of linalg_big.cu take over, up to kBigMaxK. The RSVD
// entry points reject larger k synchronously, before any launch.
constexpr int kSvdMaxK = 512;
constexpr int kBigMaxK = 4096;
constexpr int kCqExtraPasses = 3;   // k > kSvdMaxK: shifted extra CholeskyQR passes at most

// linalg_big.cu (k > kSvdMaxK)
size_t cholqr_big_panel_elems(int k);
ssi_status cholqr2_big(const double* Y, int64_t ldy, int64_t m, int k, double* Q, CholQRWork& w, int32_t* status,
                       cudaStream_t s);
size_t jacobi_big_scratch_elems(int k);
ssi_status jacobi_big(double* G, int k, double* Ut, double* S, double* scratch, int32_t* status, cudaStream_t s);

// One-sided (Hestenes) Jacobi SVD of a k x k matrix G (col-major, overwritten):
// G V = U Sigma; Ut = U sorted by descending sigma (col-major k x k), S = sigma.
// scratch: jacobi_scratch_elems(k) doubles of device memory (norms and sweep flags).
size_t jacobi_scratch_elems(int k);
ssi_status jacobi_svd(double* G, int k, double* Ut, double* S, double* scratch, int32_t* status, cudaStream_t s);

}  // namespace ssi
