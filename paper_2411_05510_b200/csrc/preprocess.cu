// NEXT-4: preprocessing of raw acceleration records (§3.2; readings P-1..P-3 of
// DESIGN.md §3): least-squares detrend, upsampling by L, zero-phase Chebyshev-I low-pass at the
// rate L fs_in, keep every M-th sample.
//
// The IIR cascade is a linear recurrence in time, so one channel is one dependent chain. To use
// the whole GPU on one record the time axis is cut into chunks and every (chunk, channel) pair is
// a thread, in two passes per filter direction:
//   pass A  each thread runs its chunk from a zero state and keeps only the final state F_c;
//   scan    per channel, the true chunk-start states S_{c+1} = Phi S_c + F_c, S_0 = 0, where
//           Phi = A^Lc is the cascade's state transition over one chunk;
//   pass B  each thread re-runs its chunk from S_c and writes the outputs.
// By linearity pass B reproduces the sequential recursion up to rounding (the chunk-start states
// differ by rounding only). The forward output v (FP64, rate L fs_in) is materialised; the
// backward pass B writes only the kept samples, converted to the output type.
#include <math_constants.h>

#include "preprocess.cuh"

namespace ssi {
namespace {

constexpr int kMaxSec = 8;            // order <= 16
constexpr int kMaxD = 2 * kMaxSec;    // cascade state size (DF2T: two per section)

struct Sos {
  int nsec;
  double b0[kMaxSec], b1[kMaxSec], b2[kMaxSec], a1[kMaxSec], a2[kMaxSec];
};

// ---------------------------------------------------------------- P-2 design (one thread)
// Chebyshev-I analog prototype (poles -sinh(mu + j theta_m), theta_m = pi m / (2n),
// m = -n+1, -n+3, ..., n-1; mu = asinh(1/eps)/n; gain prod(-p), / sqrt(1 + eps^2) for even n),
// low-pass scaled to the prewarped edge 2 tan(pi fc / fs) (in units of fs), bilinear transform
// (z = (2 + p)/(2 - p), zeros at -1), conjugate pairs -> biquads, gain spread evenly.
__global__ void design_kernel(int order, double rp_db, double fc, double fs, double* sos_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int n = order, nsec = n / 2;
  const double eps = sqrt(pow(10.0, 0.1 * rp_db) - 1.0);
  const double mu = asinh(1.0 / eps) / n;
  const double wo = 2.0 * tan(CUDART_PI * fc / fs);       // prewarped edge, fs = 1
  // analog gain of the scaled prototype: prod(-p') with p' = wo p
  double kre = 1.0, kim = 0.0;
  // digital: k_d = k' / prod(2 - p') (real), poles z = (2 + p') / (2 - p')
  double dre = 1.0, dim = 0.0;
  int s = 0;
  double zr[kMaxSec], zi[kMaxSec];
  for (int m = -n + 1; m <= n - 1; m += 2) {
    const double th = CUDART_PI * m / (2.0 * n);
    // -sinh(mu + j th) = -(sinh mu cos th + j cosh mu sin th)
    const double pr = -sinh(mu) * cos(th) * wo, pi = -cosh(mu) * sin(th) * wo;
    double t = kre * (-pr) - kim * (-pi);
    kim = kre * (-pi) + kim * (-pr);
    kre = t;
    const double qr = 2.0 - pr, qi = -pi;
    t = dre * qr - dim * qi;
    dim = dre * qi + dim * qr;
    dre = t;
    if (m < 0) {                                            // Im p > 0: one per conjugate pair
      const double nr = 2.0 + pr, ni = pi;                  // z = (2 + p)/(2 - p)
      const double den = qr * qr + qi * qi;
      zr[s] = (nr * qr + ni * qi) / den;
      zi[s] = (ni * qr - nr * qi) / den;
      ++s;
    }
  }
  double k = kre;
  if ((n & 1) == 0) k /= sqrt(1.0 + eps * eps);
  const double kd = k / dre;                                // prod(2 - p) is real
  const double g = pow(kd, 1.0 / nsec);
  for (int j = 0; j < nsec; ++j) {
    double* o = sos_out + 5 * j;
    o[0] = g; o[1] = 2.0 * g; o[2] = g;
    o[3] = -2.0 * zr[j];
    o[4] = zr[j] * zr[j] + zi[j] * zi[j];
  }
}

__device__ __forceinline__ void load_sos(const double* __restrict__ p, int nsec, Sos& f) {
  f.nsec = nsec;
#pragma unroll
  for (int j = 0; j < kMaxSec; ++j)
    if (j < nsec) {
      f.b0[j] = p[5 * j]; f.b1[j] = p[5 * j + 1]; f.b2[j] = p[5 * j + 2];
      f.a1[j] = p[5 * j + 3]; f.a2[j] = p[5 * j + 4];
    }
}

// One step of the DF2T cascade: returns the output, updates the state z[2 nsec].
template <int NSEC>
__device__ __forceinline__ double cascade_step(const Sos& f, double* z, double x) {
#pragma unroll
  for (int j = 0; j < NSEC; ++j) {
    const double y = fma(f.b0[j], x, z[2 * j]);
    z[2 * j] = fma(f.b1[j], x, fma(-f.a1[j], y, z[2 * j + 1]));
    z[2 * j + 1] = fma(f.b2[j], x, -f.a2[j] * y);
    x = y;
  }
  return x;
}

// Phi[D][D] (column j = state after Lc zero-input steps from e_j); D threads.
template <int NSEC>
__global__ void phi_kernel(const double* __restrict__ sos, int64_t Lc, double* __restrict__ Phi) {
  constexpr int D = 2 * NSEC;
  const int j = threadIdx.x;
  if (j >= D) return;
  Sos f;
  load_sos(sos, NSEC, f);
  double z[D];
#pragma unroll
  for (int q = 0; q < D; ++q) z[q] = q == j ? 1.0 : 0.0;
  for (int64_t t = 0; t < Lc; ++t) cascade_step<NSEC>(f, z, 0.0);
#pragma unroll
  for (int q = 0; q < D; ++q) Phi[q * D + j] = z[q];
}

// ---------------------------------------------------------------- P-1 detrend statistics
constexpr int kDetNT = 128;

template <typename T>
__global__ void __launch_bounds__(kDetNT) detrend_partial_kernel(const T* __restrict__ Y, int64_t N, int l,
                                                                  int64_t ldY, int64_t tchunk,
                                                                  double* __restrict__ part) {
  const int64_t t0 = int64_t(blockIdx.x) * tchunk, t1 = min(N, t0 + tchunk);
  const double hbar = 0.5 * double(N - 1);
  for (int c = threadIdx.x; c < l; c += kDetNT) {
    double s0 = 0.0, s1 = 0.0;
    for (int64_t t = t0; t < t1; ++t) {
      const double y = double(Y[t * ldY + c]);
      s0 += y;
      s1 = fma(double(t) - hbar, y, s1);
    }
    part[(int64_t(blockIdx.x) * l + c) * 2] = s0;
    part[(int64_t(blockIdx.x) * l + c) * 2 + 1] = s1;
  }
}

// alpha, beta per channel: beta = sum (h - hbar) y / sum (h - hbar)^2, alpha = mean - beta hbar.
__global__ void detrend_coef_kernel(const double* __restrict__ part, int nchunk, int64_t N, int l,
                                    double* __restrict__ ab) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= l) return;
  double s0 = 0.0, s1 = 0.0;
  for (int q = 0; q < nchunk; ++q) {
    s0 += part[(int64_t(q) * l + c) * 2];
    s1 += part[(int64_t(q) * l + c) * 2 + 1];
  }
  const double n = double(N), hbar = 0.5 * (n - 1.0);
  const double shh = n * (n * n - 1.0) / 12.0;              // sum (h - hbar)^2
  const double beta = N > 1 ? s1 / shh : 0.0;
  ab[2 * c] = s0 / n - beta * hbar;
  ab[2 * c + 1] = beta;
}

// ---------------------------------------------------------------- passes
struct PassArgs {
  const void* Y;       // forward input: raw record
  int ydtype;
  int64_t ldY;
  const double* ab;    // detrend coefficients
  int L, M;
  int64_t N, NH;       // input samples, high-rate samples (N L)
  int l;
  int64_t Lc, nchunk;
  double* v;           // forward output [NH][l]
  void* Z;             // decimated output [N_out][ldZ]
  int zdtype;
  int64_t ldZ, n_out;
  const double* sos;
  double* F;           // [nchunk][l][D] zero-state final states
  double* S;           // [nchunk][l][D] chunk-start states
};

__device__ __forceinline__ double load_y(const PassArgs& a, int64_t h, int c) {
  return a.ydtype == SSI_F32 ? double(static_cast<const float*>(a.Y)[h * a.ldY + c])
                             : static_cast<const double*>(a.Y)[h * a.ldY + c];
}

// DIR 0: forward over n = 0..NH-1, input L (y_h - alpha - beta h) at n = h L and 0 between;
// DIR 1: backward, r = 0..NH-1 <-> n = NH-1-r, input v[n]; kept samples n = j M, j < n_out.
// PASS 0: zero state, store the final state; PASS 1: start from S, write outputs.
// The phases n mod L / n mod M are carried as counters (no 64-bit division per sample).
template <int NSEC, int DIR, int PASS>
__global__ void __launch_bounds__(128) iir_pass_kernel(PassArgs a) {
  constexpr int D = 2 * NSEC;
  const int64_t tid = int64_t(blockIdx.x) * 128 + threadIdx.x;
  if (tid >= a.nchunk * a.l) return;
  const int c = int(tid % a.l);
  const int64_t ch = tid / a.l;
  Sos f;
  load_sos(a.sos, NSEC, f);
  double z[D];
  const double* s0 = a.S + (ch * a.l + c) * D;
#pragma unroll
  for (int q = 0; q < D; ++q) z[q] = PASS == 0 ? 0.0 : s0[q];
  const int64_t r0 = ch * a.Lc, r1 = min(a.NH, r0 + a.Lc);
  if (DIR == 0) {
    const double al = a.ab[2 * c], be = a.ab[2 * c + 1], gl = double(a.L);
    int64_t h = r0 / a.L;
    int ph = int(r0 - h * a.L);
    for (int64_t n = r0; n < r1; ++n) {
      const double x = ph == 0 ? gl * (load_y(a, h, c) - fma(be, double(h), al)) : 0.0;
      const double y = cascade_step<NSEC>(f, z, x);
      if (PASS == 1) a.v[n * a.l + c] = y;
      if (++ph == a.L) { ph = 0; ++h; }
    }
  } else {
    int64_t n = a.NH - 1 - r0;
    int64_t j = n / a.M;
    int dm = int(n - j * a.M);
    for (int64_t r = r0; r < r1; ++r, --n) {
      const double y = cascade_step<NSEC>(f, z, a.v[n * a.l + c]);
      if (PASS == 1 && dm == 0 && j < a.n_out) {
        if (a.zdtype == SSI_F32) static_cast<float*>(a.Z)[j * a.ldZ + c] = float(y);
        else static_cast<double*>(a.Z)[j * a.ldZ + c] = y;
      }
      if (dm == 0) { dm = a.M - 1; --j; } else { --dm; }
    }
  }
  if (PASS == 0) {
    double* fo = a.F + (ch * a.l + c) * D;
#pragma unroll
    for (int q = 0; q < D; ++q) fo[q] = z[q];
  }
}

// S_0 = 0, S_{c+1} = Phi S_c + F_c, one thread per channel (sequential over chunks).
template <int NSEC>
__global__ void chunk_scan_kernel(const double* __restrict__ Phi, const double* __restrict__ F,
                                  double* __restrict__ S, int64_t nchunk, int l) {
  constexpr int D = 2 * NSEC;
  __shared__ double P[D * D];
  for (int e = threadIdx.x; e < D * D; e += blockDim.x) P[e] = Phi[e];
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= l) return;
  double s[D];
#pragma unroll
  for (int q = 0; q < D; ++q) s[q] = 0.0;
  for (int64_t ch = 0; ch < nchunk; ++ch) {
    double* so = S + (ch * l + c) * D;
    const double* fi = F + (ch * l + c) * D;
#pragma unroll
    for (int q = 0; q < D; ++q) so[q] = s[q];
    double t[D];
#pragma unroll
    for (int q = 0; q < D; ++q) {
      double acc = fi[q];
#pragma unroll
      for (int p = 0; p < D; ++p) acc = fma(P[q * D + p], s[p], acc);
      t[q] = acc;
    }
#pragma unroll
    for (int q = 0; q < D; ++q) s[q] = t[q];
  }
}

template <int NSEC>
ssi_status run_filter(PassArgs a, double* Phi, cudaStream_t st) {
  const int64_t threads = a.nchunk * a.l;
  const int blocks = int((threads + 127) / 128);
  phi_kernel<NSEC><<<1, 32, 0, st>>>(a.sos, a.Lc, Phi);
  SSI_TRY(launch_check("phi_kernel"));
  iir_pass_kernel<NSEC, 0, 0><<<blocks, 128, 0, st>>>(a);
  SSI_TRY(launch_check("iir_pass_kernel fwd A"));
  chunk_scan_kernel<NSEC><<<(a.l + 127) / 128, 128, 0, st>>>(Phi, a.F, a.S, a.nchunk, a.l);
  SSI_TRY(launch_check("chunk_scan_kernel fwd"));
  iir_pass_kernel<NSEC, 0, 1><<<blocks, 128, 0, st>>>(a);
  SSI_TRY(launch_check("iir_pass_kernel fwd B"));
  iir_pass_kernel<NSEC, 1, 0><<<blocks, 128, 0, st>>>(a);
  SSI_TRY(launch_check("iir_pass_kernel bwd A"));
  chunk_scan_kernel<NSEC><<<(a.l + 127) / 128, 128, 0, st>>>(Phi, a.F, a.S, a.nchunk, a.l);
  SSI_TRY(launch_check("chunk_scan_kernel bwd"));
  iir_pass_kernel<NSEC, 1, 1><<<blocks, 128, 0, st>>>(a);
  return launch_check("iir_pass_kernel bwd B");
}

}  // namespace

int64_t preprocess_chunk_len(int64_t NH, int l) {
  // ~150k (chunk, channel) threads, chunks of 64..8192 samples
  int64_t want = NH * int64_t(l) / 150000;
  int64_t Lc = 64;
  while (Lc < want && Lc < 8192) Lc <<= 1;
  return Lc;
}

namespace {
struct PreBufs {
  double *sos, *Phi, *part, *ab, *F, *S, *v;
};
void carve_pre(Carver& c, int64_t N, int l, int L, int order, PreBufs& b, int64_t& nchunk, int64_t& Lc,
               int64_t& ndet, int64_t& tdet) {
  const int64_t NH = N * L;
  Lc = preprocess_chunk_len(NH, l);
  nchunk = (NH + Lc - 1) / Lc;
  tdet = 4096;
  ndet = (N + tdet - 1) / tdet;
  const int D = order;
  b.sos = c.take<double>(5 * kMaxSec);
  b.Phi = c.take<double>(kMaxD * kMaxD);
  b.part = c.take<double>(size_t(ndet) * l * 2);
  b.ab = c.take<double>(2 * size_t(l));
  b.F = c.take<double>(size_t(nchunk) * l * D);
  b.S = c.take<double>(size_t(nchunk) * l * D);
  b.v = c.take<double>(size_t(NH) * l);
}
}  // namespace

size_t preprocess_ws_bytes(int64_t N, int l, int L, int order) {
  Carver c(nullptr);
  PreBufs b;
  int64_t nchunk, Lc, ndet, tdet;
  carve_pre(c, N, l, L, order, b, nchunk, Lc, ndet, tdet);
  return c.bytes();
}

ssi_status lowpass_design(int order, double rp_db, double fc, double fs, double* sos, cudaStream_t s) {
  design_kernel<<<1, 1, 0, s>>>(order, rp_db, fc, fs, sos);
  return launch_check("design_kernel");
}

ssi_status preprocess_run(const void* Y, int dtype, int64_t N, int l, int64_t ldY, double fs_in, int L, int M,
                          int order, double rp_db, double fc, void* Z, int zdtype, int64_t ldZ, void* ws,
                          cudaStream_t s) {
  Carver c(ws);
  PreBufs b;
  int64_t nchunk, Lc, ndet, tdet;
  carve_pre(c, N, l, L, order, b, nchunk, Lc, ndet, tdet);
  SSI_TRY(lowpass_design(order, rp_db, fc, fs_in * L, b.sos, s));
  if (dtype == SSI_F32)
    detrend_partial_kernel<float><<<int(ndet), kDetNT, 0, s>>>(static_cast<const float*>(Y), N, l, ldY, tdet, b.part);
  else
    detrend_partial_kernel<double><<<int(ndet), kDetNT, 0, s>>>(static_cast<const double*>(Y), N, l, ldY, tdet,
                                                                 b.part);
  SSI_TRY(launch_check("detrend_partial_kernel"));
  detrend_coef_kernel<<<(l + 127) / 128, 128, 0, s>>>(b.part, int(ndet), N, l, b.ab);
  SSI_TRY(launch_check("detrend_coef_kernel"));
  PassArgs a;
  a.Y = Y; a.ydtype = dtype; a.ldY = ldY; a.ab = b.ab; a.L = L; a.M = M; a.N = N; a.NH = N * L; a.l = l;
  a.Lc = Lc; a.nchunk = nchunk; a.v = b.v; a.Z = Z; a.zdtype = zdtype; a.ldZ = ldZ;
  a.n_out = (N * L) / M; a.sos = b.sos; a.F = b.F; a.S = b.S;
  switch (order / 2) {
    case 1: return run_filter<1>(a, b.Phi, s);
    case 2: return run_filter<2>(a, b.Phi, s);
    case 3: return run_filter<3>(a, b.Phi, s);
    case 4: return run_filter<4>(a, b.Phi, s);
    case 5: return run_filter<5>(a, b.Phi, s);
    case 6: return run_filter<6>(a, b.Phi, s);
    case 7: return run_filter<7>(a, b.Phi, s);
    case 8: return run_filter<8>(a, b.Phi, s);
  }
  set_last_error("ssi_preprocess: order %d not supported", order);
  return SSI_ERR_INVALID_ARG;
}

}  // namespace ssi
