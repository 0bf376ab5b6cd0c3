#pragma once
#include "common.cuh"

namespace ssi {

// Block-Toeplitz operator T of Eq. (6) applied through its block DFT (toeplitz_dft.cu).
// Spectrum: i blocks of (2l)^2 doubles; per-pass frequency buffers: i * 2l * k doubles each.
size_t bt_spectrum_elems(int l, int i);
size_t bt_freq_elems(int l, int i, int k);
size_t bt_table_elems(int i);
// spectrum of the block sequence + the forward / inverse DFT tables
// Z: optional scratch of >= l^2 * 2i doubles (the GEMM form of the spectrum; nullptr: direct sums)
ssi_status bt_spectrum(const double* R, int l, int i, double* Bb, double* tables, cudaStream_t s,
                       double* Z = nullptr);
// Y (m x k col-major, ldy) = T X or T^T X (trans), X m x k col-major (ldx), m = l i.
ssi_status bt_apply(const double* Bb, const double* tables, int l, int i, int k, bool trans, const double* X,
                    int64_t ldx, double* Y, int64_t ldy, double* Xh, double* Yh, cudaStream_t s);

}  // namespace ssi
