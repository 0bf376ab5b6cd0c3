// A1: lagged output covariances (§2.1), FP64 mode.
//   C[(k,a)][b] = sum_{t in shard, t+k<N} Y[t+k][a] * Y[t][b]
// as one long-K GEMM over lag-shifted views of the record: rows (k, a) flattened,
// columns b, K = time. FP64 DMMA (mma.sync m8n8k4) on 64x64x16 tiles; FP32 records are
// widened exactly on the way into shared memory. Split-K over time writes partials that
// a second kernel reduces in fixed order and divides by (N - k) (reading A-6).
#include "common.cuh"
#include "covariance.cuh"

namespace ssi {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 128, LDS = BM + 4;

struct CovArgs {
  const void* Y;
  int64_t N, ldY;
  int l, lag_lo, rows;     // rows = (lag_hi - lag_lo + 1) * l
  int64_t t_begin, t_end;  // shard
  int64_t tchunk;          // time per split
  double* out;             // direct output (splits == 1) or partial base
  int32_t* status;
};

template <typename T>
__device__ __forceinline__ double ld(const T* p) { return double(__ldg(p)); }

template <typename T>
__global__ void __launch_bounds__(NT) cov_fp64_kernel(CovArgs a) {
  __shared__ __align__(16) double smem[4 * BK * LDS];
  double* As[2] = {smem, smem + 2 * BK * LDS};
  double* Bs[2] = {smem + BK * LDS, smem + 3 * BK * LDS};
  const T* Y = static_cast<const T*>(a.Y);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int r0 = blockIdx.x * BM, b0 = blockIdx.y * BN;
  const int64_t tb = a.t_begin + int64_t(blockIdx.z) * a.tchunk;
  const int64_t te = min(a.t_end, tb + a.tchunk);

  // Row this thread loads for A: fixed across k-steps (mm = tid % 64).
  const int mm = tid % BM;
  const int r = r0 + mm;
  const bool rvalid = r < a.rows;
  const int lag = rvalid ? a.lag_lo + r / a.l : 0;
  const int ach = rvalid ? r % a.l : 0;
  const int64_t tmax_r = rvalid ? min(te, a.N - lag) : tb;  // t < tmax_r contributes
  const int nn = tid % BN;
  const bool bvalid = (b0 + nn) < a.l;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[8], rb[8];
  bool bad = false;
  auto load = [&](int64_t t0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int kk = tid / BM + 2 * j;
      const int64_t t = t0 + kk;
      ra[j] = (rvalid && t < tmax_r) ? ld(Y + (t + lag) * a.ldY + ach) : 0.0;
      rb[j] = (bvalid && t < te) ? ld(Y + t * a.ldY + b0 + nn) : 0.0;
      bad |= !isfinite(ra[j]) || !isfinite(rb[j]);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int kk = tid / BM + 2 * j;
      As[buf][kk * LDS + mm] = ra[j];
      Bs[buf][kk * LDS + nn] = rb[j];
    }
  };
  if (te > tb) {
    load(tb);
    store(0);
    __syncthreads();
    int buf = 0;
    for (int64_t t0 = tb; t0 < te; t0 += BK) {
      const bool more = t0 + BK < te;
      if (more) load(t0 + BK);
      const double* as = As[buf];
      const double* bs = Bs[buf];
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = as[(kk + (lane & 3)) * LDS + wm + i * 8 + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = bs[(kk + (lane & 3)) * LDS + wn + j * 8 + (lane >> 2)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      if (more) {
        store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
  if (bad) set_status(a.status, SSI_ERR_NONFINITE);
  double* out = a.out + int64_t(blockIdx.z) * int64_t(a.rows) * a.l;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int rr = r0 + wm + i * 8 + (lane >> 2);
        const int cc = b0 + wn + j * 8 + 2 * (lane & 3) + e;
        if (rr < a.rows && cc < a.l) out[int64_t(rr) * a.l + cc] = acc[i][j][e];
      }
}

// R[k-lag_lo][a][b] = sum_z part[z] (fixed order), optionally / (N - k).
__global__ void cov_finalize(const double* __restrict__ part, int splits, int rows, int l,
                             int lag_lo, int64_t N, int normalize, double* __restrict__ R) {
  const int64_t total = int64_t(rows) * l;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    s = ordered_sum(part + e, total, splits);
    if (normalize) {
      const int k = lag_lo + int(e / (int64_t(l) * l));
      s /= double(N - k);
    }
    R[e] = s;
  }
}

}  // namespace

int cov_fp64_splits(int64_t span, int rows, int l) {
  const int64_t tiles = int64_t((rows + BM - 1) / BM) * ((l + BN - 1) / BN);
  int64_t s = (148 * 4 + tiles - 1) / tiles;
  const int64_t smax = (span + 1023) / 1024;
  if (s > smax) s = smax;
  if (s < 1) s = 1;
  if (s > 256) s = 256;
  return int(s);
}

ssi_status cov_fp64(const void* Y, int dtype, int64_t N, int l, int64_t ldY, int lag_lo,
                    int lag_hi, int64_t t_begin, int64_t t_end, int normalize, double* R,
                    double* partial, int32_t* status, cudaStream_t s) {
  const int rows = (lag_hi - lag_lo + 1) * l;
  const int64_t span = t_end - t_begin;
  const int splits = cov_fp64_splits(span, rows, l);
  int64_t tchunk = (span + splits - 1) / splits;
  tchunk = (tchunk + BK - 1) / BK * BK;
  if (tchunk < BK) tchunk = BK;
  const int z = span > 0 ? int((span + tchunk - 1) / tchunk) : 1;
  CovArgs a{Y, N, ldY, l, lag_lo, rows, t_begin, t_end, tchunk, partial, status};
  dim3 grid((rows + BM - 1) / BM, (l + BN - 1) / BN, z);
  if (dtype == SSI_F32) cov_fp64_kernel<float><<<grid, NT, 0, s>>>(a);
  else                  cov_fp64_kernel<double><<<grid, NT, 0, s>>>(a);
  SSI_TRY(launch_check("cov_fp64_kernel"));
  const int64_t tot = int64_t(rows) * l;
  int blocks = int((tot + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  cov_finalize<<<blocks, 256, 0, s>>>(partial, z, rows, l, lag_lo, N, normalize, R);
  return launch_check("cov_finalize");
}

// R[k - lag_lo][a][b] /= (N - k) in place (reading A-6): the raw sums of time-sharded calls,
// all-reduced over ranks, become the covariances of the whole record.
__global__ void cov_normalize_kernel(double* __restrict__ R, int l, int lag_lo, int64_t n_lags, int64_t N) {
  const int64_t per = int64_t(l) * l, total = n_lags * per;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x)
    R[e] /= double(N - (lag_lo + e / per));
}

ssi_status cov_normalize(double* R, int l, int lag_lo, int n_lags, int64_t N, cudaStream_t s) {
  const int64_t tot = int64_t(n_lags) * l * l;
  int blocks = int((tot + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  cov_normalize_kernel<<<blocks, 256, 0, s>>>(R, l, lag_lo, n_lags, N);
  return launch_check("cov_normalize_kernel");
}

size_t cov_fp64_partial_elems(int64_t span, int rows, int l) {
  return size_t(cov_fp64_splits(span, rows, l)) * size_t(rows) * size_t(l);
}

}  // namespace ssi
