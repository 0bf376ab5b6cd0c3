#pragma once
#include "common.cuh"

namespace ssi {

// SSI_COV_INT8X3: exact int8-slice covariance on tcgen05 (kind::i8). See cov_i8.cu.
bool cov_i8_supported(int l, int n_lags, int64_t ldY, int dtype);
void cov_i8_carve(Carver& c, int64_t N, int l, int lag_lo, int lag_hi);
ssi_status cov_i8(const void* Y, int dtype, int64_t N, int l, int64_t ldY, int lag_lo, int lag_hi,
                  int64_t t_begin, int64_t t_end, int normalize, double* R, void* ws,
                  int32_t* status, cudaStream_t s);

}  // namespace ssi
