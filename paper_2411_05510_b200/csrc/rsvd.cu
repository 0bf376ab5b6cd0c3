// A3-A8: randomized SVD of the block-Toeplitz T (Algorithm 1, with
// the north star's q power iterations; reading A-12). Host-side orchestration of the
// device kernels; every arithmetic step runs on the GPU.
#include "covariance.cuh"
#include "linalg.cuh"
#include "rsvd.cuh"
#include "toeplitz_dft.cuh"

#ifndef SSI_RSVD_MIDQR
#define SSI_RSVD_MIDQR cholqr1   // measured: 114.5 -> 121.1 records/s at c3 (cholqr2 for A/B)
#endif

namespace ssi {

struct RsvdWork {
  double *Omega, *Y, *Q, *Q2, *G, *Ut, *Sk, *tall, *jac;
  CholQRWork cq;
};

static void rsvd_carve(Carver& c, int64_t m, int k, RsvdWork& w) {
  w.Omega = c.take<double>(size_t(m) * k);
  w.Y = c.take<double>(size_t(m) * k);
  w.Q = c.take<double>(size_t(m) * k);
  w.Q2 = c.take<double>(size_t(m) * k);
  w.G = c.take<double>(size_t(k) * k);
  w.Ut = c.take<double>(size_t(k) * k);
  w.Sk = c.take<double>(size_t(k));
  w.jac = c.take<double>(jacobi_scratch_elems(k));
  w.tall = c.take<double>((k <= kTallMaxN ? gemm_tall_partial_elems_upto(m, k) : 0) + 1);
  cholqr_carve(c, m, k, w.cq);
}

size_t rsvd_ws_bytes(int64_t m, int k) {
  Carver c(nullptr);
  RsvdWork w;
  rsvd_carve(c, m, k, w);
  return c.bytes();
}

// Algorithm 1 with q power iterations, given the operator pass(trans, X, out): out = T X or
// T^T X (X and out m x k col-major, ld m).
template <typename Pass>
static ssi_status rsvd_core(Pass&& pass, int64_t m, int k, int q, uint64_t seed, uint64_t sid,
                            int n_keep, double* U, int64_t ldU, double* S, RsvdWork& w,
                            int32_t* status, cudaStream_t s) {
  // line 1: Omega ~ N(0,1), Philox on device (Eq. 14 input; reading A-11)
  SSI_TRY(sketch_launch(int(m), k, seed, sid, w.Omega, m, s));
  // line 2: Y = T Omega (Eq. 14)
  SSI_TRY(pass(false, w.Omega, w.Y));
  // line 3: Q = qr(Y). Between the power iterations' products only span(Q) carries forward, so
  // those re-orthonormalisations are one CholeskyQR pass (SSI_RSVD_MIDQR); the Q that enters
  // B = Q^T T (line 4) is always CholeskyQR2 (reading A-12).
  SSI_TRY(q > 0 ? SSI_RSVD_MIDQR(w.Y, m, m, k, w.Q, w.cq, status, s) : cholqr2(w.Y, m, m, k, w.Q, w.cq, status, s));
  // power iterations: Z = qr(T^T Q); Q = qr(T Z)
  for (int it = 0; it < q; ++it) {
    SSI_TRY(pass(true, w.Q, w.Y));
    SSI_TRY(SSI_RSVD_MIDQR(w.Y, m, m, k, w.Q2, w.cq, status, s));
    SSI_TRY(pass(false, w.Q2, w.Y));
    if (it + 1 < q) {
      SSI_TRY(SSI_RSVD_MIDQR(w.Y, m, m, k, w.Q, w.cq, status, s));
    } else {
      SSI_TRY(cholqr2(w.Y, m, m, k, w.Q, w.cq, status, s));
    }
  }
  // line 4: B = Q^T T, formed as B^T = T^T Q (m x k) (Eq. 15)
  SSI_TRY(pass(true, w.Q, w.Y));
  // line 5: B^T = Qb Rb (CholeskyQR2) -> B = Rb^T Qb^T; SVD(Rb^T) = U~ Sigma W^T
  SSI_TRY(cholqr2(w.Y, m, m, k, w.Q2, w.cq, status, s));
  // Rb^T = (L2^T L1^T)^T = L1 L2
  SSI_TRY(gemm_f64(k, k, k, 1.0, Operand{w.cq.L1, 1, k}, Operand{w.cq.L2, 1, k}, w.G, k, 1,
                   nullptr, s));
  SSI_TRY(jacobi_svd(w.G, k, w.Ut, w.Sk, w.jac, status, s));
  // line 6: U = Q U~ (Eq. 18), leading n_keep columns
  if (n_keep <= kTallMaxN && m % 2 == 0 && k % 2 == 0 && ldU % 2 == 0 &&
      (reinterpret_cast<uintptr_t>(U) & 15) == 0) {
    // tall-skinny DMMA kernel, one M tile per CTA (no split-K)
    SSI_TRY(gemm_tall_batched(m, n_keep, k, false, w.Q, m, 0, w.Ut, k, 0, U, ldU, 0, 1, s));
  } else {
    SSI_TRY(gemm_f64(m, n_keep, k, 1.0, Operand{w.Q, 1, m}, Operand{w.Ut, 1, k}, U, ldU, 1,
                     nullptr, s));
  }
  if (cudaMemcpyAsync(S, w.Sk, sizeof(double) * k, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return launch_check("rsvd S copy");
  return SSI_OK;
}

ssi_status rsvd_run(const double* T, int64_t ldT, int64_t m, int k, int q, uint64_t seed,
                    uint64_t sid, int n_keep, double* U, int64_t ldU, double* S, void* ws,
                    int32_t* status, cudaStream_t s) {
  Carver c(ws);
  RsvdWork w;
  rsvd_carve(c, m, k, w);
  // dedicated tall-skinny kernel (whole width in one tile; 16-byte cp.async alignment)
  const bool tall = k <= 224 && m % 2 == 0 && ldT % 2 == 0 && (reinterpret_cast<uintptr_t>(T) & 15) == 0;
  const Operand Tn{T, ldT, 1};   // T(i,j) = T[i*ldT + j]  (row-major, k-contiguous)
  const Operand Tt{T, 1, ldT};   // T^T(i,j) = T[j*ldT + i]
  // X -> T X (trans = false) or T^T X (trans = true), X and the result m x k col-major
  auto pass = [&](bool trans, const double* X, double* out) -> ssi_status {
    if (tall) return gemm_tall(m, k, m, !trans, T, ldT, X, m, out, m, w.tall, s);
    return gemm_f64(m, k, m, 1.0, trans ? Tt : Tn, Operand{X, 1, m}, out, m, 1, nullptr, s);
  };
  return rsvd_core(pass, m, k, q, seed, sid, n_keep, U, ldU, S, w, status, s);
}

// ---------------------------------------------------------------- structured (T never formed)
struct RsvdBtWork {
  RsvdWork base;
  double *Bb, *Xh, *Yh, *tables;
};

static void rsvd_bt_carve(Carver& c, int l, int i, int k, RsvdBtWork& w) {
  const int64_t m = int64_t(l) * i;
  w.base.Omega = c.take<double>(size_t(m) * k);
  w.base.Y = c.take<double>(size_t(m) * k);
  w.base.Q = c.take<double>(size_t(m) * k);
  w.base.Q2 = c.take<double>(size_t(m) * k);
  w.base.G = c.take<double>(size_t(k) * k);
  w.base.Ut = c.take<double>(size_t(k) * k);
  w.base.Sk = c.take<double>(size_t(k));
  w.base.jac = c.take<double>(jacobi_scratch_elems(k));
  w.base.tall = nullptr;
  cholqr_carve(c, m, k, w.base.cq);
  w.Bb = c.take<double>(bt_spectrum_elems(l, i));
  w.Xh = c.take<double>(bt_freq_elems(l, i, k));
  w.Yh = c.take<double>(bt_freq_elems(l, i, k));
  w.tables = c.take<double>(bt_table_elems(i));
}

size_t rsvd_bt_ws_bytes(int l, int i, int k) {
  Carver c(nullptr);
  RsvdBtWork w;
  rsvd_bt_carve(c, l, i, k, w);
  return c.bytes();
}

ssi_status rsvd_bt_run(const double* R, int l, int i, int k, int q, uint64_t seed, uint64_t sid,
                       int n_keep, double* U, int64_t ldU, double* S, void* ws, int32_t* status,
                       cudaStream_t s) {
  Carver c(ws);
  RsvdBtWork w;
  rsvd_bt_carve(c, l, i, k, w);
  const int64_t m = int64_t(l) * i;
  // spectrum of the block sequence B_d = R_{i+d}, once per call
  // the spectrum GEMM's l^2 x 2i output lives in Xh when it fits (Xh is first written by the
  // first pass, after the spectrum is formed)
  const bool zfit = bt_freq_elems(l, i, k) >= size_t(l) * l * 2 * i;
  SSI_TRY(bt_spectrum(R, l, i, w.Bb, w.tables, s, zfit ? w.Xh : nullptr));
  auto pass = [&](bool trans, const double* X, double* out) -> ssi_status {
    return bt_apply(w.Bb, w.tables, l, i, k, trans, X, m, out, m, w.Xh, w.Yh, s);
  };
  return rsvd_core(pass, m, k, q, seed, sid, n_keep, U, ldU, S, w.base, status, s);
}

}  // namespace ssi
