#pragma once
#include "common.cuh"

namespace ssi {

// SSI_COV_SPECTRAL (cov_spectral.cu): segment cross-spectra, FP64.
constexpr int kSpecMaxF = 2048;   // FFT length limit (lag_hi < kSpecMaxF)
constexpr int kSpecChunk = 512;   // segments per chunk (bounds the spectra workspace)

struct SpecPlan {
  int F, B, lp, n_lags;   // FFT length, segment length F - lag_hi, l rounded up to even, lags
  int64_t S;              // segments covering the time shard
  int64_t Sc;             // segments per chunk (spectra buffer capacity)
};
struct SpecBufs {
  double2* tw;
  double *W, *A, *Bs, *G, *partial, *Rp;
};

SpecPlan spec_plan(int64_t N, int64_t span, int l, int lag_lo, int lag_hi);
void cov_spec_carve(Carver& c, int64_t N, int64_t span, int l, int lag_lo, int lag_hi, SpecBufs& b);
bool cov_spec_supported(int lag_hi);
// G[f] (Re, Im blocks, (b, a) at b + a lp) (+)= sum over nseg segments of Ye_a conj(X_b), three
// real DMMA products per complex one (cross_spectral.cu)
ssi_status cross_spectral_3m(const double* A, const double* B, int64_t sF, int64_t nseg, int lp, int nfreq,
                             double* G, bool accumulate, cudaStream_t s);
ssi_status cov_spectral(const void* Y, int dtype, int64_t N, int l, int64_t ldY, int lag_lo, int lag_hi,
                        int64_t t_begin, int64_t t_end, int normalize, double* R, void* ws, int32_t* status,
                        cudaStream_t s, int phases = 7);

}  // namespace ssi
