// NEXT-4 preprocessing and shear-frame generator (preprocess.cu, frame.cu).
// PAPER.md:482 (§3.2), :314 (§3.1), :349 (§3.1.2).
#pragma once
#include "common.cuh"

namespace ssi {

constexpr int kFrameMaxDof = 12;

size_t preprocess_ws_bytes(int64_t N, int l, int L, int order);
ssi_status preprocess_run(const void* Y, int dtype, int64_t N, int l, int64_t ldY, double fs_in, int L, int M,
                          int order, double rp_db, double fc, void* Z, int zdtype, int64_t ldZ, void* ws,
                          cudaStream_t s);
ssi_status lowpass_design(int order, double rp_db, double fc, double fs, double* sos, cudaStream_t s);

size_t frame_ws_bytes(int n, int64_t N, int64_t n_burn);
ssi_status frame_model_run(int n, double m, double k, double xi, int mode_a, int mode_b, double fs, double* Ad,
                           double* Bd, double* Co, double* ab, cudaStream_t s);
ssi_status frame_simulate_run(int n, double m, double k, double xi, int mode_a, int mode_b, double fs, int64_t N,
                              int64_t n_burn, double snr_db, uint64_t seed, uint64_t stream_id, void* Y, int dtype,
                              int64_t ldY, double* clean, void* ws, cudaStream_t s);

}  // namespace ssi
