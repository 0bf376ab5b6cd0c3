#pragma once
#include "common.cuh"

namespace ssi {

// FP64 DMMA covariance (SSI_COV_FP64). partial: cov_fp64_partial_elems() doubles.
ssi_status cov_fp64(const void* Y, int dtype, int64_t N, int l, int64_t ldY, int lag_lo,
                    int lag_hi, int64_t t_begin, int64_t t_end, int normalize, double* R,
                    double* partial, int32_t* status, cudaStream_t s);
size_t cov_fp64_partial_elems(int64_t span, int rows, int l);
int cov_fp64_splits(int64_t span, int rows, int l);
// In-place R[k - lag_lo] /= (N - k) for k = lag_lo .. lag_lo + n_lags - 1.
ssi_status cov_normalize(double* R, int l, int lag_lo, int n_lags, int64_t N, cudaStream_t s);

// Toeplitz assembly (A2).
ssi_status toeplitz_launch(const double* R, int l, int i, double* T, int64_t ldT, cudaStream_t s);

// Philox sketch (A3).
ssi_status sketch_launch(int m, int k, uint64_t seed, uint64_t stream_id, double* omega,
                         int64_t ldo, cudaStream_t s);
ssi_status philox_words_launch(uint64_t seed, uint64_t stream_id, int64_t n_pairs,
                               uint32_t* words, cudaStream_t s);

}  // namespace ssi
