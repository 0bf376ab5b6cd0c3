// libssi.so C ABI (include/ssi.h): synchronous argument checks, workspace carving and
// stream plumbing around the device kernels. No arithmetic of the method runs here.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "covariance.cuh"
#include "cov_i8.cuh"
#include "cov_spectral.cuh"
#include "linalg.cuh"
#include "rsvd.cuh"
#include "cluster.cuh"
#include "preprocess.cuh"

namespace ssi {

static thread_local char g_err[512] = "";

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

ssi_status launch_check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error("%s: %s", what, cudaGetErrorString(e));
    return SSI_ERR_CUDA;
  }
  return SSI_OK;
}

static cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }


static size_t cov_ws(int64_t N, int l, int lag_lo, int lag_hi, int mode, int64_t span) {
  Carver c(nullptr);
  const int rows = (lag_hi - lag_lo + 1) * l;
  if (mode == SSI_COV_FP64) {
    c.take<double>(cov_fp64_partial_elems(span, rows, l));
  } else if (mode == SSI_COV_SPECTRAL) {
    SpecBufs sb;
    cov_spec_carve(c, N, span, l, lag_lo, lag_hi, sb);
  } else {
    cov_i8_carve(c, N, l, lag_lo, lag_hi);
  }
  return c.bytes();
}

}  // namespace ssi

using namespace ssi;

extern "C" {

const char* ssi_last_error(void) { return g_err; }

const char* ssi_version(void) { return "ssi 0.1 (sm_100a)"; }

const char* ssi_status_string(ssi_status s) {
  switch (s) {
    case SSI_OK: return "ok";
    case SSI_ERR_INVALID_ARG: return "invalid argument";
    case SSI_ERR_SHAPE: return "leading dimension too small";
    case SSI_ERR_DTYPE: return "unsupported dtype or mode";
    case SSI_ERR_WORKSPACE: return "workspace too small";
    case SSI_ERR_CUDA: return "CUDA error";
    case SSI_ERR_NONFINITE: return "non-finite input";
    case SSI_ERR_NUMERIC: return "numerical failure (CholeskyQR2 breakdown or non-convergence)";
    default: return "unknown status";
  }
}

ssi_status ssi_clear_status(void* ws, void* stream) {
  SSI_REQUIRE(ws, SSI_ERR_INVALID_ARG, "ssi_clear_status: NULL ws");
  if (cudaMemsetAsync(ws, 0, kWsHeader, S(stream)) != cudaSuccess) return launch_check("ssi_clear_status");
  return SSI_OK;
}

ssi_status ssi_fetch_device_status(const void* ws, ssi_status* code) {
  SSI_REQUIRE(ws && code, SSI_ERR_INVALID_ARG, "ssi_fetch_device_status: NULL pointer");
  int32_t v = 0;
  if (cudaMemcpy(&v, ws, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess)
    return launch_check("ssi_fetch_device_status");
  *code = v;
  return SSI_OK;
}

ssi_status ssi_covariances_ws(int64_t N, int32_t l, int32_t lag_lo, int32_t lag_hi,
                              int32_t cov_mode, size_t* bytes) {
  SSI_REQUIRE(bytes, SSI_ERR_INVALID_ARG, "ssi_covariances_ws: NULL bytes");
  SSI_REQUIRE(N > 0 && l > 0 && lag_lo >= 1 && lag_hi >= lag_lo, SSI_ERR_INVALID_ARG,
              "ssi_covariances_ws: bad sizes");
  SSI_REQUIRE(cov_mode == SSI_COV_FP64 || cov_mode == SSI_COV_INT8X3 || cov_mode == SSI_COV_SPECTRAL, SSI_ERR_DTYPE,
              "ssi_covariances_ws: unknown cov_mode %d", cov_mode);
  SSI_REQUIRE(cov_mode != SSI_COV_SPECTRAL || cov_spec_supported(lag_hi), SSI_ERR_DTYPE,
              "ssi_covariances_ws: SSI_COV_SPECTRAL needs lag_hi < %d", kSpecMaxF);
  // the int8x3 plan tiles channels by pick_nb(l); an unsupported l has no plan (and no size)
  SSI_REQUIRE(cov_mode != SSI_COV_INT8X3 || cov_i8_supported(l, lag_hi - lag_lo + 1, l, SSI_F32), SSI_ERR_DTYPE,
              "ssi_covariances_ws: SSI_COV_INT8X3 needs l %% 64 == 0, or l %% 16 == 0 and l <= 64");
  *bytes = cov_ws(N, l, lag_lo, lag_hi, cov_mode, N);
  return SSI_OK;
}

ssi_status ssi_cov_spectral_plan(int64_t N, int32_t l, int32_t lag_lo, int32_t lag_hi, int32_t* F,
                                 int64_t* S) {
  SSI_REQUIRE(F && S, SSI_ERR_INVALID_ARG, "ssi_cov_spectral_plan: NULL pointer");
  SSI_REQUIRE(N > 0 && l > 0 && lag_lo >= 1 && lag_hi >= lag_lo, SSI_ERR_INVALID_ARG,
              "ssi_cov_spectral_plan: bad sizes");
  SSI_REQUIRE(cov_spec_supported(lag_hi), SSI_ERR_DTYPE, "ssi_cov_spectral_plan: lag_hi >= %d", kSpecMaxF);
  const SpecPlan p = spec_plan(N, N, l, lag_lo, lag_hi);
  *F = p.F;
  *S = p.S;
  return SSI_OK;
}

ssi_status ssi_covariances(const void* Y, int32_t dtype, int64_t N, int32_t l, int64_t ldY,
                           int32_t lag_lo, int32_t lag_hi, int32_t cov_mode, int64_t t_begin,
                           int64_t t_end, int32_t normalize, double* R, void* ws,
                           size_t ws_bytes, void* stream) {
  SSI_REQUIRE(Y && R && ws, SSI_ERR_INVALID_ARG, "ssi_covariances: NULL pointer");
  SSI_REQUIRE(N > 0 && l > 0, SSI_ERR_INVALID_ARG, "ssi_covariances: N and l must be positive");
  SSI_REQUIRE(lag_lo >= 1 && lag_hi >= lag_lo, SSI_ERR_INVALID_ARG,
              "ssi_covariances: need 1 <= lag_lo <= lag_hi");
  SSI_REQUIRE(lag_hi < N, SSI_ERR_INVALID_ARG, "ssi_covariances: record too short (N=%lld, lag %d)",
              (long long)N, lag_hi);
  SSI_REQUIRE(0 <= t_begin && t_begin <= t_end && t_end <= N, SSI_ERR_INVALID_ARG,
              "ssi_covariances: bad time shard [%lld, %lld)", (long long)t_begin, (long long)t_end);
  SSI_REQUIRE(!normalize || (t_begin == 0 && t_end == N), SSI_ERR_INVALID_ARG,
              "ssi_covariances: normalize=1 requires the full record");
  SSI_REQUIRE(ldY >= l, SSI_ERR_SHAPE, "ssi_covariances: ldY < l");
  SSI_REQUIRE(dtype == SSI_F32 || dtype == SSI_F64, SSI_ERR_DTYPE, "ssi_covariances: bad dtype");
  SSI_REQUIRE(cov_mode == SSI_COV_FP64 || cov_mode == SSI_COV_INT8X3 || cov_mode == SSI_COV_SPECTRAL, SSI_ERR_DTYPE,
              "ssi_covariances: unknown cov_mode %d", cov_mode);
  SSI_REQUIRE(cov_mode != SSI_COV_INT8X3 || cov_i8_supported(l, lag_hi - lag_lo + 1, ldY, dtype),
              SSI_ERR_DTYPE, "ssi_covariances: SSI_COV_INT8X3 needs l %% 64 == 0, or l %% 16 == 0 and l <= 64");
  SSI_REQUIRE(cov_mode != SSI_COV_SPECTRAL || cov_spec_supported(lag_hi), SSI_ERR_DTYPE,
              "ssi_covariances: SSI_COV_SPECTRAL needs lag_hi < %d", kSpecMaxF);
  const size_t need = cov_ws(N, l, lag_lo, lag_hi, cov_mode, t_end - t_begin);
  SSI_REQUIRE(ws_bytes >= need, SSI_ERR_WORKSPACE, "ssi_covariances: workspace %zu < %zu",
              ws_bytes, need);
  cudaStream_t s = S(stream);
  int32_t* st = static_cast<int32_t*>(ws);
  if (cov_mode == SSI_COV_FP64) {
    Carver c(ws);
    const int rows = (lag_hi - lag_lo + 1) * l;
    double* part = c.take<double>(cov_fp64_partial_elems(t_end - t_begin, rows, l));
    return cov_fp64(Y, dtype, N, l, ldY, lag_lo, lag_hi, t_begin, t_end, normalize, R, part, st, s);
  }
  if (cov_mode == SSI_COV_SPECTRAL)
    return cov_spectral(Y, dtype, N, l, ldY, lag_lo, lag_hi, t_begin, t_end, normalize, R, ws, st, s);
  return cov_i8(Y, dtype, N, l, ldY, lag_lo, lag_hi, t_begin, t_end, normalize, R, ws, st, s);
}

ssi_status ssi_cov_normalize(double* R, int32_t l, int32_t lag_lo, int32_t n_lags, int64_t N, void* stream) {
  SSI_REQUIRE(R, SSI_ERR_INVALID_ARG, "ssi_cov_normalize: NULL R");
  SSI_REQUIRE(l > 0 && lag_lo >= 1 && n_lags >= 1, SSI_ERR_INVALID_ARG, "ssi_cov_normalize: bad sizes");
  SSI_REQUIRE(int64_t(lag_lo) + n_lags - 1 < N, SSI_ERR_INVALID_ARG,
              "ssi_cov_normalize: record too short (N=%lld, lag %d)", (long long)N, lag_lo + n_lags - 1);
  return cov_normalize(R, l, lag_lo, n_lags, N, S(stream));
}

ssi_status ssi_cov_spectral_phases(const void* Y, int32_t dtype, int64_t N, int32_t l, int64_t ldY,
                                   int32_t lag_lo, int32_t lag_hi, int64_t t_begin, int64_t t_end,
                                   int32_t normalize, double* R, void* ws, size_t ws_bytes, int32_t phases,
                                   void* stream) {
  SSI_REQUIRE(phases >= 1 && phases <= 7, SSI_ERR_INVALID_ARG, "ssi_cov_spectral_phases: phases must be 1..7");
  SSI_REQUIRE(Y && R && ws, SSI_ERR_INVALID_ARG, "ssi_cov_spectral_phases: NULL pointer");
  SSI_REQUIRE(N > 0 && l > 0 && lag_lo >= 1 && lag_hi >= lag_lo && lag_hi < N, SSI_ERR_INVALID_ARG,
              "ssi_cov_spectral_phases: bad sizes");
  SSI_REQUIRE(0 <= t_begin && t_begin <= t_end && t_end <= N, SSI_ERR_INVALID_ARG,
              "ssi_cov_spectral_phases: bad time shard");
  SSI_REQUIRE(!normalize || (t_begin == 0 && t_end == N), SSI_ERR_INVALID_ARG,
              "ssi_cov_spectral_phases: normalize=1 requires the full record");
  SSI_REQUIRE(ldY >= l, SSI_ERR_SHAPE, "ssi_cov_spectral_phases: ldY < l");
  SSI_REQUIRE(dtype == SSI_F32 || dtype == SSI_F64, SSI_ERR_DTYPE, "ssi_cov_spectral_phases: bad dtype");
  SSI_REQUIRE(cov_spec_supported(lag_hi), SSI_ERR_DTYPE, "ssi_cov_spectral_phases: lag_hi >= %d", kSpecMaxF);
  const size_t need = cov_ws(N, l, lag_lo, lag_hi, SSI_COV_SPECTRAL, t_end - t_begin);
  SSI_REQUIRE(ws_bytes >= need, SSI_ERR_WORKSPACE, "ssi_cov_spectral_phases: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = S(stream);
  return cov_spectral(Y, dtype, N, l, ldY, lag_lo, lag_hi, t_begin, t_end, normalize, R, ws,
                      static_cast<int32_t*>(ws), s, phases);
}

ssi_status ssi_toeplitz(const double* R, int32_t l, int32_t i, double* T, int64_t ldT, void* stream) {
  SSI_REQUIRE(R && T, SSI_ERR_INVALID_ARG, "ssi_toeplitz: NULL pointer");
  SSI_REQUIRE(l > 0 && i > 0, SSI_ERR_INVALID_ARG, "ssi_toeplitz: l and i must be positive");
  SSI_REQUIRE(ldT >= int64_t(l) * i, SSI_ERR_SHAPE, "ssi_toeplitz: ldT < l*i");
  return toeplitz_launch(R, l, i, T, ldT, S(stream));
}

ssi_status ssi_rsvd_ws(int32_t m, int32_t k, int32_t n_keep, size_t* bytes) {
  SSI_REQUIRE(bytes, SSI_ERR_INVALID_ARG, "ssi_rsvd_ws: NULL bytes");
  SSI_REQUIRE(m > 0 && k >= 1 && k <= m && n_keep >= 1 && n_keep <= k, SSI_ERR_INVALID_ARG,
              "ssi_rsvd_ws: bad sizes");
  SSI_REQUIRE(k <= kBigMaxK, SSI_ERR_INVALID_ARG, "ssi_rsvd_ws: k = %d > %d unsupported", k, kBigMaxK);
  *bytes = rsvd_ws_bytes(m, k);
  return SSI_OK;
}

ssi_status ssi_rsvd(const double* T, int64_t ldT, int32_t m, int32_t k, int32_t q, uint64_t seed,
                    uint64_t stream_id, int32_t n_keep, double* U, int64_t ldU, double* S_,
                    void* ws, size_t ws_bytes, void* stream) {
  SSI_REQUIRE(T && U && S_ && ws, SSI_ERR_INVALID_ARG, "ssi_rsvd: NULL pointer");
  SSI_REQUIRE(m > 0 && k >= 1 && k <= m, SSI_ERR_INVALID_ARG, "ssi_rsvd: need 1 <= k <= m");
  SSI_REQUIRE(k <= kBigMaxK, SSI_ERR_INVALID_ARG, "ssi_rsvd: k = %d > %d unsupported", k, kBigMaxK);
  SSI_REQUIRE(n_keep >= 1 && n_keep <= k, SSI_ERR_INVALID_ARG, "ssi_rsvd: need 1 <= n_keep <= k");
  SSI_REQUIRE(q >= 0, SSI_ERR_INVALID_ARG, "ssi_rsvd: q < 0");
  SSI_REQUIRE(ldT >= m && ldU >= m, SSI_ERR_SHAPE, "ssi_rsvd: ldT or ldU < m");
  const size_t need = rsvd_ws_bytes(m, k);
  SSI_REQUIRE(ws_bytes >= need, SSI_ERR_WORKSPACE, "ssi_rsvd: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = S(stream);
  return rsvd_run(T, ldT, m, k, q, seed, stream_id, n_keep, U, ldU, S_, ws,
                  static_cast<int32_t*>(ws), s);
}

ssi_status ssi_rsvd_toeplitz_ws(int32_t l, int32_t i, int32_t k, int32_t n_keep, size_t* bytes) {
  SSI_REQUIRE(bytes, SSI_ERR_INVALID_ARG, "ssi_rsvd_toeplitz_ws: NULL bytes");
  SSI_REQUIRE(l > 0 && i > 0 && k >= 1 && int64_t(k) <= int64_t(l) * i && n_keep >= 1 && n_keep <= k,
              SSI_ERR_INVALID_ARG, "ssi_rsvd_toeplitz_ws: bad sizes");
  SSI_REQUIRE(k <= kBigMaxK, SSI_ERR_INVALID_ARG, "ssi_rsvd_toeplitz_ws: k = %d > %d unsupported", k, kBigMaxK);
  *bytes = rsvd_bt_ws_bytes(l, i, k);
  return SSI_OK;
}

ssi_status ssi_rsvd_toeplitz(const double* R, int32_t l, int32_t i, int32_t k, int32_t q, uint64_t seed,
                             uint64_t stream_id, int32_t n_keep, double* U, int64_t ldU, double* S_,
                             void* ws, size_t ws_bytes, void* stream) {
  SSI_REQUIRE(R && U && S_ && ws, SSI_ERR_INVALID_ARG, "ssi_rsvd_toeplitz: NULL pointer");
  SSI_REQUIRE(l > 0 && i > 0, SSI_ERR_INVALID_ARG, "ssi_rsvd_toeplitz: l and i must be positive");
  const int64_t m = int64_t(l) * i;
  SSI_REQUIRE(m <= INT32_MAX, SSI_ERR_INVALID_ARG, "ssi_rsvd_toeplitz: l*i too large");
  SSI_REQUIRE(k >= 1 && k <= m, SSI_ERR_INVALID_ARG, "ssi_rsvd_toeplitz: need 1 <= k <= l*i");
  SSI_REQUIRE(k <= kBigMaxK, SSI_ERR_INVALID_ARG, "ssi_rsvd_toeplitz: k = %d > %d unsupported", k, kBigMaxK);
  SSI_REQUIRE(n_keep >= 1 && n_keep <= k, SSI_ERR_INVALID_ARG, "ssi_rsvd_toeplitz: need 1 <= n_keep <= k");
  SSI_REQUIRE(q >= 0, SSI_ERR_INVALID_ARG, "ssi_rsvd_toeplitz: q < 0");
  SSI_REQUIRE(ldU >= m, SSI_ERR_SHAPE, "ssi_rsvd_toeplitz: ldU < l*i");
  const size_t need = rsvd_bt_ws_bytes(l, i, k);
  SSI_REQUIRE(ws_bytes >= need, SSI_ERR_WORKSPACE, "ssi_rsvd_toeplitz: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = S(stream);
  return rsvd_bt_run(R, l, i, k, q, seed, stream_id, n_keep, U, ldU, S_, ws,
                     static_cast<int32_t*>(ws), s);
}

ssi_status ssi_philox_words(uint64_t seed, uint64_t stream_id, int64_t n_pairs, uint32_t* words,
                            void* stream) {
  SSI_REQUIRE(words && n_pairs > 0, SSI_ERR_INVALID_ARG, "ssi_philox_words: bad arguments");
  return philox_words_launch(seed, stream_id, n_pairs, words, S(stream));
}

ssi_status ssi_gaussian_sketch(int32_t m, int32_t k, uint64_t seed, uint64_t stream_id,
                               double* omega, int64_t ldo, void* stream) {
  SSI_REQUIRE(omega && m > 0 && k > 0, SSI_ERR_INVALID_ARG, "ssi_gaussian_sketch: bad arguments");
  SSI_REQUIRE(ldo >= m, SSI_ERR_SHAPE, "ssi_gaussian_sketch: ldo < m");
  return sketch_launch(m, k, seed, stream_id, omega, ldo, S(stream));
}

static ssi_status check_orders(int32_t n_min, int32_t n_max, int32_t n_step) {
  SSI_REQUIRE(n_min >= 2 && n_min % 2 == 0 && n_step >= 2 && n_step % 2 == 0 && n_max >= n_min,
              SSI_ERR_INVALID_ARG,
              "orders must be even: n_min >= 2, n_step >= 2 even, n_max >= n_min (SPEC.md:312)");
  return SSI_OK;
}

ssi_status ssi_modal_sweep_ws(int32_t l, int32_t i, int32_t n_min, int32_t n_max, int32_t n_step,
                              size_t* bytes) {
  SSI_REQUIRE(bytes && l > 0 && i >= 2, SSI_ERR_INVALID_ARG, "ssi_modal_sweep_ws: bad sizes");
  SSI_TRY(check_orders(n_min, n_max, n_step));
  SSI_REQUIRE(n_max <= kModalMaxOrder && modal_smem_bytes(n_max, n_max / 2, modal_band_global(n_max)) <= kModalSmemMax,
              SSI_ERR_INVALID_ARG, "ssi_modal_sweep_ws: n_max %d > %d", n_max, kModalMaxOrder);
  *bytes = modal_ws_bytes(l, i, n_min, n_max, n_step);
  return SSI_OK;
}

ssi_status ssi_modal_sweep(const double* U, int64_t ldU, const double* S_, int32_t l, int32_t i,
                           int32_t n_min, int32_t n_max, int32_t n_step, double dt,
                           const ssi_pole_table* out, void* ws, size_t ws_bytes, void* stream) {
  SSI_REQUIRE(U && S_ && out && ws, SSI_ERR_INVALID_ARG, "ssi_modal_sweep: NULL pointer");
  SSI_REQUIRE(l > 0 && i >= 2 && dt > 0.0, SSI_ERR_INVALID_ARG, "ssi_modal_sweep: need l > 0, i >= 2, dt > 0");
  SSI_TRY(check_orders(n_min, n_max, n_step));
  const int64_t m = int64_t(l) * i;
  SSI_REQUIRE(n_max <= m - l, SSI_ERR_INVALID_ARG, "ssi_modal_sweep: n_max > l(i-1)");
  SSI_REQUIRE(ldU >= m, SSI_ERR_SHAPE, "ssi_modal_sweep: ldU < l*i");
  const int no = (n_max - n_min) / n_step + 1;
  SSI_REQUIRE(out->n_orders == no && out->cap >= n_max / 2 && out->l == l &&
                  out->n_min == n_min && out->n_step == n_step,
              SSI_ERR_INVALID_ARG, "ssi_modal_sweep: pole table header does not match the sweep");
  SSI_REQUIRE(out->count && out->f && out->xi && out->mu_re && out->mu_im && out->mpc && out->mpd &&
                  out->shape,
              SSI_ERR_INVALID_ARG, "ssi_modal_sweep: NULL pole-table array");
  SSI_REQUIRE(n_max <= kModalMaxOrder &&
                  modal_smem_bytes(n_max, out->cap, modal_band_global(n_max)) <= kModalSmemMax,
              SSI_ERR_INVALID_ARG, "ssi_modal_sweep: n_max %d > %d or pole-table cap %d too large", n_max,
              kModalMaxOrder, out->cap);
  const size_t need = modal_ws_bytes(l, i, n_min, n_max, n_step);
  SSI_REQUIRE(ws_bytes >= need, SSI_ERR_WORKSPACE, "ssi_modal_sweep: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = S(stream);
  return modal_run(U, ldU, S_, l, i, n_min, n_max, n_step, dt, *out, ws, static_cast<int32_t*>(ws), s);
}

ssi_status ssi_stab3d(const ssi_pole_table* tables, int32_t n_lags, const ssi_criteria* crit,
                      uint8_t* flags, int32_t* stable_count, void* stream) {
  SSI_REQUIRE(tables && crit && flags && stable_count && n_lags >= 1, SSI_ERR_INVALID_ARG,
              "ssi_stab3d: bad arguments");
  for (int g = 1; g < n_lags; ++g)
    SSI_REQUIRE(tables[g].n_orders == tables[0].n_orders && tables[g].cap == tables[0].cap &&
                    tables[g].l == tables[0].l && tables[g].n_min == tables[0].n_min &&
                    tables[g].n_step == tables[0].n_step,
                SSI_ERR_INVALID_ARG, "ssi_stab3d: pole tables differ in shape");
  return stab3d_run(tables, n_lags, *crit, flags, stable_count, S(stream));
}

static ssi_status table_set(const ssi_pole_table* tables, int32_t n_lags, const char* fn, TableSet& ts) {
  SSI_REQUIRE(tables && n_lags >= 1 && n_lags <= SSI_MAX_LAGS, SSI_ERR_INVALID_ARG,
              "%s: need 1 <= n_lags <= %d tables", fn, SSI_MAX_LAGS);
  for (int g = 0; g < n_lags; ++g) {
    const ssi_pole_table& t = tables[g];
    SSI_REQUIRE(t.count && t.f && t.xi && t.mpc && t.mpd && t.shape && t.n_orders >= 1 && t.cap >= 1 && t.l >= 1,
                SSI_ERR_INVALID_ARG, "%s: bad pole table %d", fn, g);
    SSI_REQUIRE(t.n_orders == tables[0].n_orders && t.cap == tables[0].cap && t.l == tables[0].l &&
                    t.n_min == tables[0].n_min && t.n_step == tables[0].n_step,
                SSI_ERR_INVALID_ARG, "%s: pole tables differ in shape", fn);
    ts.t[g] = t;
  }
  for (int g = n_lags; g < SSI_MAX_LAGS; ++g) ts.t[g] = tables[0];
  return SSI_OK;
}

ssi_status ssi_cluster_stage1_ws(int32_t n_lags, int32_t n_orders, size_t* bytes) {
  SSI_REQUIRE(bytes && n_lags >= 1 && n_orders >= 1, SSI_ERR_INVALID_ARG, "ssi_cluster_stage1_ws: bad arguments");
  *bytes = cluster_stage1_ws_bytes(n_lags, n_orders);
  return SSI_OK;
}

ssi_status ssi_cluster_stage1(const ssi_pole_table* tables, int32_t n_lags, const ssi_criteria* crit,
                              const uint8_t* flags, int32_t max_poles, double fcm_tol, int32_t fcm_max_iter,
                              int32_t* pole_idx, double* X, double* U, int32_t* retained,
                              ssi_cluster_info* info, void* ws, size_t ws_bytes, void* stream) {
  TableSet ts;
  SSI_TRY(table_set(tables, n_lags, "ssi_cluster_stage1", ts));
  SSI_REQUIRE(crit && flags && pole_idx && X && U && retained && info && ws, SSI_ERR_INVALID_ARG,
              "ssi_cluster_stage1: NULL pointer");
  SSI_REQUIRE(max_poles >= 1 && fcm_tol >= 0.0 && fcm_max_iter >= 0, SSI_ERR_INVALID_ARG,
              "ssi_cluster_stage1: need max_poles >= 1, fcm_tol >= 0, fcm_max_iter >= 0");
  const size_t need = cluster_stage1_ws_bytes(n_lags, tables[0].n_orders);
  SSI_REQUIRE(ws_bytes >= need, SSI_ERR_WORKSPACE, "ssi_cluster_stage1: workspace %zu < %zu", ws_bytes, need);
  return cluster_stage1_run(ts, n_lags, *crit, flags, max_poles, fcm_tol, fcm_max_iter, pole_idx, X, U, retained,
                            info, ws, static_cast<int32_t*>(ws), S(stream));
}

ssi_status ssi_cluster_stage2_ws(int32_t n_retained, int32_t l, size_t* bytes) {
  SSI_REQUIRE(bytes && n_retained >= 0 && l >= 1, SSI_ERR_INVALID_ARG, "ssi_cluster_stage2_ws: bad arguments");
  *bytes = cluster_stage2_ws_bytes(n_retained, l);
  return SSI_OK;
}

ssi_status ssi_cluster_stage2(const ssi_pole_table* tables, int32_t n_lags, const int32_t* pole_idx,
                              const int32_t* retained, int32_t n_retained, double cutoff, int32_t min_size,
                              int32_t max_clusters, int32_t* labels, double* cl_f, double* cl_xi, int32_t* cl_size,
                              int32_t* cl_medoid, double* cl_shape, int32_t* merges_ab, double* merges_h,
                              ssi_cluster_info* info, void* ws, size_t ws_bytes, void* stream) {
  TableSet ts;
  SSI_TRY(table_set(tables, n_lags, "ssi_cluster_stage2", ts));
  SSI_REQUIRE(pole_idx && retained && labels && cl_f && cl_xi && cl_size && cl_medoid && cl_shape && info && ws,
              SSI_ERR_INVALID_ARG, "ssi_cluster_stage2: NULL pointer");
  SSI_REQUIRE(n_retained >= 0 && min_size >= 1 && max_clusters >= 1 && isfinite(cutoff), SSI_ERR_INVALID_ARG,
              "ssi_cluster_stage2: need n_retained >= 0, min_size >= 1, max_clusters >= 1, finite cutoff");
  const size_t need = cluster_stage2_ws_bytes(n_retained, tables[0].l);
  SSI_REQUIRE(ws_bytes >= need, SSI_ERR_WORKSPACE, "ssi_cluster_stage2: workspace %zu < %zu", ws_bytes, need);
  return cluster_stage2_run(ts, pole_idx, retained, n_retained, cutoff, min_size, max_clusters, labels, cl_f, cl_xi,
                            cl_size, cl_medoid, cl_shape, merges_ab, merges_h, info, ws, S(stream));
}

ssi_status ssi_track(const double* ref_f, const double* ref_shape, int32_t n_ref, const double* f,
                     const double* shape, const int32_t* count, int32_t n_sess, int32_t max_modes, int32_t l,
                     double df_max, double macd_max, int32_t* match, double* success, void* stream) {
  SSI_REQUIRE(ref_f && ref_shape && f && shape && count && match, SSI_ERR_INVALID_ARG, "ssi_track: NULL pointer");
  SSI_REQUIRE(n_ref >= 1 && n_sess >= 1 && max_modes >= 1 && l >= 1 && int64_t(n_ref) * max_modes <= 16384,
              SSI_ERR_INVALID_ARG, "ssi_track: need n_ref, n_sess, max_modes, l >= 1 and n_ref * max_modes <= 16384");
  return track_run(ref_f, ref_shape, n_ref, f, shape, count, n_sess, max_modes, l, df_max, macd_max, match, success,
                   S(stream));
}

ssi_status ssi_preprocess_ws(int64_t N, int32_t l, int32_t L, int32_t order, size_t* bytes) {
  SSI_REQUIRE(bytes && N >= 2 && l >= 1 && L >= 1 && order >= 2 && order <= 16 && order % 2 == 0,
              SSI_ERR_INVALID_ARG, "ssi_preprocess_ws: bad arguments");
  *bytes = preprocess_ws_bytes(N, l, L, order);
  return SSI_OK;
}

ssi_status ssi_preprocess(const void* Y, int32_t dtype, int64_t N, int32_t l, int64_t ldY, double fs_in, int32_t L,
                          int32_t M, int32_t order, double rp_db, double fc_hz, void* Z, int32_t out_dtype,
                          int64_t ldZ, void* ws, size_t ws_bytes, void* stream) {
  SSI_REQUIRE(Y && Z && ws, SSI_ERR_INVALID_ARG, "ssi_preprocess: NULL pointer");
  SSI_REQUIRE((dtype == SSI_F32 || dtype == SSI_F64) && (out_dtype == SSI_F32 || out_dtype == SSI_F64),
              SSI_ERR_DTYPE, "ssi_preprocess: dtype must be SSI_F32 or SSI_F64");
  SSI_REQUIRE(N >= 2 && l >= 1 && L >= 1 && M >= 1 && fs_in > 0.0 && order >= 2 && order <= 16 && order % 2 == 0 &&
                  rp_db > 0.0 && fc_hz > 0.0 && fc_hz < 0.5 * L * fs_in && (N * L) / M >= 1,
              SSI_ERR_INVALID_ARG, "ssi_preprocess: bad sizes, rates or filter parameters");
  SSI_REQUIRE(ldY >= l && ldZ >= l, SSI_ERR_SHAPE, "ssi_preprocess: ldY or ldZ < l");
  const size_t need = preprocess_ws_bytes(N, l, L, order);
  SSI_REQUIRE(ws_bytes >= need, SSI_ERR_WORKSPACE, "ssi_preprocess: workspace %zu < %zu", ws_bytes, need);
  return preprocess_run(Y, dtype, N, l, ldY, fs_in, L, M, order, rp_db, fc_hz, Z, out_dtype, ldZ, ws, S(stream));
}

ssi_status ssi_lowpass_design(int32_t order, double rp_db, double fc_hz, double fs_hz, double* sos, void* stream) {
  SSI_REQUIRE(sos && order >= 2 && order <= 16 && order % 2 == 0 && rp_db > 0.0 && fc_hz > 0.0 &&
                  fc_hz < 0.5 * fs_hz,
              SSI_ERR_INVALID_ARG, "ssi_lowpass_design: bad arguments");
  return lowpass_design(order, rp_db, fc_hz, fs_hz, sos, S(stream));
}

static ssi_status frame_check(int32_t n_dof, double m, double k, double xi, int32_t mode_a, int32_t mode_b, double fs,
                              const char* fn) {
  SSI_REQUIRE(n_dof >= 1 && n_dof <= kFrameMaxDof && m > 0.0 && k > 0.0 && fs > 0.0 && xi > 0.0 && xi < 1.0 &&
                  mode_a >= 1 && mode_a <= n_dof && mode_b >= 1 && mode_b <= n_dof && mode_a != mode_b,
              SSI_ERR_INVALID_ARG, "%s: bad frame parameters", fn);
  return SSI_OK;
}

ssi_status ssi_frame_simulate_ws(int32_t n_dof, int64_t N, int64_t n_burn, size_t* bytes) {
  SSI_REQUIRE(bytes && n_dof >= 1 && n_dof <= kFrameMaxDof && N >= 1 && n_burn >= 0, SSI_ERR_INVALID_ARG,
              "ssi_frame_simulate_ws: bad arguments");
  *bytes = frame_ws_bytes(n_dof, N, n_burn);
  return SSI_OK;
}

ssi_status ssi_frame_model(int32_t n_dof, double m, double k, double xi, int32_t mode_a, int32_t mode_b, double fs,
                           double* Ad, double* Bd, double* Co, double* ab, void* stream) {
  SSI_TRY(frame_check(n_dof, m, k, xi, mode_a, mode_b, fs, "ssi_frame_model"));
  SSI_REQUIRE(Ad && Bd && Co && ab, SSI_ERR_INVALID_ARG, "ssi_frame_model: NULL pointer");
  return frame_model_run(n_dof, m, k, xi, mode_a, mode_b, fs, Ad, Bd, Co, ab, S(stream));
}

ssi_status ssi_frame_simulate(int32_t n_dof, double m, double k, double xi, int32_t mode_a, int32_t mode_b, double fs,
                              int64_t N, int64_t n_burn, double snr_db, uint64_t seed, uint64_t stream_id, void* Y,
                              int32_t dtype, int64_t ldY, double* clean, void* ws, size_t ws_bytes, void* stream) {
  SSI_TRY(frame_check(n_dof, m, k, xi, mode_a, mode_b, fs, "ssi_frame_simulate"));
  SSI_REQUIRE(Y && ws && N >= 1 && n_burn >= 0 && (N + n_burn) * n_dof < (int64_t(1) << 31) && isfinite(snr_db),
              SSI_ERR_INVALID_ARG, "ssi_frame_simulate: bad arguments");
  SSI_REQUIRE(dtype == SSI_F32 || dtype == SSI_F64, SSI_ERR_DTYPE, "ssi_frame_simulate: dtype");
  SSI_REQUIRE(ldY >= n_dof, SSI_ERR_SHAPE, "ssi_frame_simulate: ldY < n_dof");
  const size_t need = frame_ws_bytes(n_dof, N, n_burn);
  SSI_REQUIRE(ws_bytes >= need, SSI_ERR_WORKSPACE, "ssi_frame_simulate: workspace %zu < %zu", ws_bytes, need);
  return frame_simulate_run(n_dof, m, k, xi, mode_a, mode_b, fs, N, n_burn, snr_db, seed, stream_id, Y, dtype, ldY,
                            clean, ws, S(stream));
}

}  // extern "C"
