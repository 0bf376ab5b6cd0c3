// NEXT-2 clustering + tracking (cluster.cu). PAPER.md:293, :402-415, :541-544.
#pragma once
#include "common.cuh"

namespace ssi {

// Pole tables of a 3D diagram passed by value as a kernel parameter (capture-safe, no
// host-to-device copy); SSI_MAX_LAGS of include/ssi.h bounds the lag count.
struct TableSet {
  ssi_pole_table t[SSI_MAX_LAGS];
};

size_t cluster_stage1_ws_bytes(int n_lags, int n_orders);
ssi_status cluster_stage1_run(const TableSet& ts, int n_lags, const ssi_criteria& crit, const uint8_t* flags,
                              int max_poles, double fcm_tol, int fcm_max_iter, int32_t* pole_idx, double* X,
                              double* Umem, int32_t* retained, ssi_cluster_info* info, void* ws, int32_t* status,
                              cudaStream_t s);
size_t cluster_stage2_ws_bytes(int n, int l);
ssi_status cluster_stage2_run(const TableSet& ts, const int32_t* pole_idx, const int32_t* retained, int n,
                              double cutoff, int min_size, int max_clusters, int32_t* labels, double* cl_f,
                              double* cl_xi, int32_t* cl_size, int32_t* cl_medoid, double* cl_shape,
                              int32_t* merges_ab, double* merges_h, ssi_cluster_info* info, void* ws,
                              cudaStream_t s);
ssi_status track_run(const double* ref_f, const double* ref_shape, int n_ref, const double* f, const double* shape,
                     const int32_t* count, int n_sess, int max_modes, int l, double df_max, double macd_max,
                     int32_t* match, double* success, cudaStream_t s);

}  // namespace ssi
