#pragma once
#include "common.cuh"

namespace ssi {

size_t rsvd_ws_bytes(int64_t m, int k);
ssi_status rsvd_run(const double* T, int64_t ldT, int64_t m, int k, int q, uint64_t seed,
                    uint64_t sid, int n_keep, double* U, int64_t ldU, double* S, void* ws,
                    int32_t* status, cudaStream_t s);

// RSVD of the block-Toeplitz T defined by R (lags 1..2i-1) without forming T.
size_t rsvd_bt_ws_bytes(int l, int i, int k);
ssi_status rsvd_bt_run(const double* R, int l, int i, int k, int q, uint64_t seed, uint64_t sid,
                       int n_keep, double* U, int64_t ldU, double* S, void* ws, int32_t* status,
                       cudaStream_t s);

size_t modal_ws_bytes(int l, int i, int n_min, int n_max, int n_step);
ssi_status modal_run(const double* U, int64_t ldU, const double* S, int l, int i, int n_min,
                     int n_max, int n_step, double dt, const ssi_pole_table& tab, void* ws,
                     int32_t* status, cudaStream_t s);
constexpr size_t kModalSmemMax = 227 * 1024;
constexpr int kModalMaxOrder = 512;     // Householder vector of the Hessenberg kernel in shared memory
size_t modal_smem_bytes(int n_max, int cap, bool band_global);
bool modal_band_global(int n_max);

ssi_status stab3d_run(const ssi_pole_table* tables, int n_lags, const ssi_criteria& crit,
                      uint8_t* flags, int32_t* stable_count, cudaStream_t s);

}  // namespace ssi
