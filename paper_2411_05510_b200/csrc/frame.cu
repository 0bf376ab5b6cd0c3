// NEXT-4: the paper's 10-DOF shear-frame generator on the GPU (§3.1; PAPER.md:349,
// §3.1.2; readings F-1..F-4 of DESIGN.md §3).
//   model_kernel      one CTA: M = m I, K tridiagonal, Rayleigh C = a M + b K (undamped
//                     frequencies of the uniform fixed-free chain in closed form,
//                     w_j = 2 sqrt(k/m) sin((2j-1) pi / (4n+2))), state-space A_c, B_c, C_o and the
//                     zero-order hold [[A_d, B_d], [0, I]] = exp([[A_c, B_c], [0, 0]] dt) by scaling
//                     and squaring of a degree-24 Taylor polynomial, in shared memory.
//   sim kernels       x_{h+1} = A_d x_h + B_d u_h, y_h = C_o x_h: one warp per time chunk (lane q
//                     holds state component q, the mat-vecs broadcast the state by shuffles);
//                     pass A from a zero state keeps the final state, a per-chunk scan of
//                     S_{c+1} = A_d^Lc S_c + F_c gives the true chunk-start states, pass B re-runs
//                     each chunk from S_c and writes the kept clean outputs.
//   noise kernels     P_c = mean square of the kept clean channel (fixed-order reduction),
//                     Y = clean + sqrt(P_c / 10^(SNR/10)) v.
// Draws: u and v from the reading-A-11 Philox/Box-Muller stream (sketch_launch), u_h = column h of
// an n x (n_burn + N) sketch (stream 2 s_id), v_h = column h of an l x N sketch (stream 2 s_id + 1).
#include <math_constants.h>

#include "covariance.cuh"
#include "preprocess.cuh"

namespace ssi {
namespace {

constexpr int kMaxN = kFrameMaxDof;
constexpr int kMaxD = 2 * kMaxN;     // state size <= 32: one warp
constexpr int kE = 3 * kMaxN;        // augmented matrix size bound
constexpr int kModelNT = 256;

// C (q x q) = A B, all row-major in shared memory with leading dimension ld.
__device__ void smem_gemm(const double* A, const double* B, double* C, int q, int ld) {
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) {
    const int r = e / q, c = e % q;
    double s = 0.0;
    for (int t = 0; t < q; ++t) s = fma(A[r * ld + t], B[t * ld + c], s);
    C[r * ld + c] = s;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kModelNT) model_kernel(int n, double m, double k, double xi, int mode_a, int mode_b,
                                                         double fs, double* Ad, double* Bd, double* Co, double* ab) {
  __shared__ double E[kE * kE], P[kE * kE], T[kE * kE], W[kE * kE];
  __shared__ double coef[2];
  __shared__ int s_scale;
  const int D = 2 * n, q = 3 * n, ld = kE;
  if (threadIdx.x == 0) {
    const double w0 = 2.0 * sqrt(k / m);
    const double wa = w0 * sin((2 * mode_a - 1) * CUDART_PI / (4.0 * n + 2.0));
    const double wb = w0 * sin((2 * mode_b - 1) * CUDART_PI / (4.0 * n + 2.0));
    // xi = a/(2w) + b w/2 at wa and wb
    coef[0] = 2.0 * xi * wa * wb / (wa + wb);
    coef[1] = 2.0 * xi / (wa + wb);
    ab[0] = coef[0];
    ab[1] = coef[1];
  }
  __syncthreads();
  const double a = coef[0], b = coef[1], dt = 1.0 / fs;
  // K: 2k on the diagonal except k at the roof, -k off the diagonal; M^-1 = I/m
  auto Kel = [&](int r, int c) -> double {
    if (r == c) return r < n - 1 ? 2.0 * k : k;
    return (r - c == 1 || c - r == 1) ? -k : 0.0;
  };
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) {
    const int r = e / q, c = e % q;
    double v = 0.0;
    if (r < n) {
      v = (c == n + r) ? 1.0 : 0.0;                               // [0, I, 0]
    } else if (r < D) {
      const int i = r - n;
      if (c < n) v = -Kel(i, c) / m;                              // -M^-1 K
      else if (c < D) v = -(a * (i == c - n ? m : 0.0) + b * Kel(i, c - n)) / m;   // -M^-1 C
      else v = (c - D == i) ? 1.0 / m : 0.0;                      // M^-1
    }
    E[r * ld + c] = v * dt;
    if (r < n && c < D) {
      const double ck = -Kel(r, c < n ? c : 0) / m;
      Co[r * D + c] = c < n ? ck : -(a * (r == c - n ? m : 0.0) + b * Kel(r, c - n)) / m;
    }
  }
  __syncthreads();
  // scaling: ||E||_1 / 2^s <= 1/4
  if (threadIdx.x == 0) {
    double nrm = 0.0;
    for (int c = 0; c < q; ++c) {
      double sc = 0.0;
      for (int r = 0; r < q; ++r) sc += fabs(E[r * ld + c]);
      nrm = fmax(nrm, sc);
    }
    int s = 0;
    while (nrm > 0.25) { nrm *= 0.5; ++s; }
    s_scale = s;
  }
  __syncthreads();
  const double sc = ldexp(1.0, -s_scale);
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) {
    const int r = e / q, c = e % q;
    E[r * ld + c] *= sc;
    P[r * ld + c] = (r == c) ? 1.0 : 0.0;   // result
    T[r * ld + c] = (r == c) ? 1.0 : 0.0;   // current term
  }
  __syncthreads();
  // Taylor: P = sum_{p=0}^{24} E^p / p!   (||E|| <= 1/4: remainder < 4^-25 / 25!)
  for (int p = 1; p <= 24; ++p) {
    smem_gemm(T, E, W, q, ld);
    const double inv = 1.0 / p;
    for (int e = threadIdx.x; e < q * q; e += blockDim.x) {
      const int r = e / q, c = e % q;
      T[r * ld + c] = W[r * ld + c] * inv;
      P[r * ld + c] += T[r * ld + c];
    }
    __syncthreads();
  }
  for (int s = 0; s < s_scale; ++s) {
    smem_gemm(P, P, W, q, ld);
    for (int e = threadIdx.x; e < q * q; e += blockDim.x) P[(e / q) * ld + e % q] = W[(e / q) * ld + e % q];
    __syncthreads();
  }
  for (int e = threadIdx.x; e < D * D; e += blockDim.x) Ad[e] = P[(e / D) * ld + e % D];
  for (int e = threadIdx.x; e < D * n; e += blockDim.x) Bd[e] = P[(e / n) * ld + D + e % n];
}

// Phi = A_d^Lc (D x D row-major) by repeated squaring (Lc a power of two), one CTA.
__global__ void __launch_bounds__(kModelNT) power_kernel(const double* Ad, int D, int log2Lc, double* Phi) {
  __shared__ double P[kMaxD * kMaxD], W[kMaxD * kMaxD];
  for (int e = threadIdx.x; e < D * D; e += blockDim.x) P[(e / D) * kMaxD + e % D] = Ad[e];
  __syncthreads();
  for (int s = 0; s < log2Lc; ++s) {
    smem_gemm(P, P, W, D, kMaxD);
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) P[(e / D) * kMaxD + e % D] = W[(e / D) * kMaxD + e % D];
    __syncthreads();
  }
  for (int e = threadIdx.x; e < D * D; e += blockDim.x) Phi[e] = P[(e / D) * kMaxD + e % D];
}

struct SimArgs {
  int n, D;
  int64_t H, n_burn, Lc, nchunk;
  const double *Ad, *Bd, *Co, *U;   // U: [H][n]
  double *F, *S, *clean;            // F, S: [nchunk][D]; clean: [N][n]
};

// One warp per chunk. PASS 0: zero start, store the final state. PASS 1: start from S, write the
// kept outputs y_h = C_o x_h (h >= n_burn) before the update of step h.
template <int PASS>
__global__ void __launch_bounds__(128) sim_pass_kernel(SimArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t ch = (int64_t(blockIdx.x) * 128 + threadIdx.x) >> 5;
  if (ch >= a.nchunk) return;
  const int n = a.n, D = a.D;
  double arow[kMaxD], brow[kMaxN], crow[kMaxD];
#pragma unroll
  for (int j = 0; j < kMaxD; ++j) {
    arow[j] = (lane < D && j < D) ? a.Ad[lane * D + j] : 0.0;
    crow[j] = (lane < n && j < D) ? a.Co[lane * D + j] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < kMaxN; ++j) brow[j] = (lane < D && j < n) ? a.Bd[lane * n + j] : 0.0;
  double x = (PASS == 1 && lane < D) ? a.S[ch * D + lane] : 0.0;
  const int64_t h0 = ch * a.Lc, h1 = min(a.H, h0 + a.Lc);
  for (int64_t h = h0; h < h1; ++h) {
    const double u = lane < n ? a.U[h * n + lane] : 0.0;
    double xn = 0.0, y = 0.0;
#pragma unroll
    for (int j = 0; j < kMaxD; ++j) {
      if (j < D) {
        const double xj = __shfl_sync(0xffffffffu, x, j);
        xn = fma(arow[j], xj, xn);
        if (PASS == 1) y = fma(crow[j], xj, y);
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxN; ++j) {
      if (j < n) xn = fma(brow[j], __shfl_sync(0xffffffffu, u, j), xn);
    }
    if (PASS == 1 && h >= a.n_burn && lane < n) a.clean[(h - a.n_burn) * n + lane] = y;
    x = xn;
  }
  if (PASS == 0 && lane < D) a.F[ch * D + lane] = x;
}

// S_0 = 0, S_{c+1} = Phi S_c + F_c; one warp, lane q holds component q.
__global__ void sim_scan_kernel(const double* __restrict__ Phi, const double* __restrict__ F, double* __restrict__ S,
                                int D, int64_t nchunk) {
  const int lane = threadIdx.x & 31;
  double prow[kMaxD];
#pragma unroll
  for (int j = 0; j < kMaxD; ++j) prow[j] = (lane < D && j < D) ? Phi[lane * D + j] : 0.0;
  double s = 0.0;
  for (int64_t c = 0; c < nchunk; ++c) {
    if (lane < D) S[c * D + lane] = s;
    double t = lane < D ? F[c * D + lane] : 0.0;
#pragma unroll
    for (int j = 0; j < kMaxD; ++j)
      if (j < D) t = fma(prow[j], __shfl_sync(0xffffffffu, s, j), t);
    s = t;
  }
}

// mean square of each kept clean channel: one CTA per channel, fixed-order reduction
__global__ void __launch_bounds__(256) power_ms_kernel(const double* __restrict__ clean, int64_t N, int n,
                                                       double* __restrict__ P) {
  __shared__ double red[256];
  const int c = blockIdx.x;
  double s = 0.0;
  for (int64_t h = threadIdx.x; h < N; h += 256) {
    const double y = clean[h * n + c];
    s = fma(y, y, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) P[c] = red[0] / double(N);
}

__global__ void add_noise_kernel(const double* __restrict__ clean, const double* __restrict__ V,
                                 const double* __restrict__ P, int64_t N, int n, double snr_lin, void* Y, int dtype,
                                 int64_t ldY) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= N * n) return;
  const int64_t h = e / n;
  const int c = int(e - h * n);
  const double v = clean[e] + sqrt(P[c] / snr_lin) * V[e];
  if (dtype == SSI_F32) static_cast<float*>(Y)[h * ldY + c] = float(v);
  else static_cast<double*>(Y)[h * ldY + c] = v;
}

struct FrameBufs {
  double *Ad, *Bd, *Co, *ab, *Phi, *U, *V, *F, *S, *P, *clean;
};

void carve_frame(Carver& c, int n, int64_t N, int64_t n_burn, int64_t Lc, FrameBufs& b) {
  const int D = 2 * n;
  const int64_t H = N + n_burn;
  const int64_t nchunk = (H + Lc - 1) / Lc;
  b.Ad = c.take<double>(D * D); b.Bd = c.take<double>(D * n); b.Co = c.take<double>(n * D);
  b.ab = c.take<double>(2); b.Phi = c.take<double>(D * D);
  b.U = c.take<double>(size_t(H) * n); b.V = c.take<double>(size_t(N) * n);
  b.F = c.take<double>(size_t(nchunk) * D); b.S = c.take<double>(size_t(nchunk) * D);
  b.P = c.take<double>(n); b.clean = c.take<double>(size_t(N) * n);
}

int frame_log2_chunk(int64_t H) {
  // ~H / 256 chunks (one warp each), chunks of 2^6 .. 2^10 steps
  int lg = 6;
  while (lg < 10 && (H >> lg) > 512) ++lg;
  return lg;
}

}  // namespace

size_t frame_ws_bytes(int n, int64_t N, int64_t n_burn) {
  Carver c(nullptr);
  FrameBufs b;
  carve_frame(c, n, N, n_burn, int64_t(1) << frame_log2_chunk(N + n_burn), b);
  return c.bytes();
}

ssi_status frame_model_run(int n, double m, double k, double xi, int mode_a, int mode_b, double fs, double* Ad,
                           double* Bd, double* Co, double* ab, cudaStream_t s) {
  model_kernel<<<1, kModelNT, 0, s>>>(n, m, k, xi, mode_a, mode_b, fs, Ad, Bd, Co, ab);
  return launch_check("model_kernel");
}

ssi_status frame_simulate_run(int n, double m, double k, double xi, int mode_a, int mode_b, double fs, int64_t N,
                              int64_t n_burn, double snr_db, uint64_t seed, uint64_t stream_id, void* Y, int dtype,
                              int64_t ldY, double* clean_out, void* ws, cudaStream_t s) {
  const int D = 2 * n;
  const int64_t H = N + n_burn;
  const int lg = frame_log2_chunk(H);
  const int64_t Lc = int64_t(1) << lg;
  Carver c(ws);
  FrameBufs b;
  carve_frame(c, n, N, n_burn, Lc, b);
  double* clean = clean_out ? clean_out : b.clean;
  SSI_TRY(frame_model_run(n, m, k, xi, mode_a, mode_b, fs, b.Ad, b.Bd, b.Co, b.ab, s));
  power_kernel<<<1, kModelNT, 0, s>>>(b.Ad, D, lg, b.Phi);
  SSI_TRY(launch_check("power_kernel"));
  SSI_TRY(sketch_launch(n, int(H), seed, 2 * stream_id, b.U, n, s));
  SSI_TRY(sketch_launch(n, int(N), seed, 2 * stream_id + 1, b.V, n, s));
  SimArgs a;
  a.n = n; a.D = D; a.H = H; a.n_burn = n_burn; a.Lc = Lc; a.nchunk = (H + Lc - 1) / Lc;
  a.Ad = b.Ad; a.Bd = b.Bd; a.Co = b.Co; a.U = b.U; a.F = b.F; a.S = b.S; a.clean = clean;
  const int blocks = int((a.nchunk * 32 + 127) / 128);
  sim_pass_kernel<0><<<blocks, 128, 0, s>>>(a);
  SSI_TRY(launch_check("sim_pass_kernel A"));
  sim_scan_kernel<<<1, 32, 0, s>>>(b.Phi, b.F, b.S, D, a.nchunk);
  SSI_TRY(launch_check("sim_scan_kernel"));
  sim_pass_kernel<1><<<blocks, 128, 0, s>>>(a);
  SSI_TRY(launch_check("sim_pass_kernel B"));
  power_ms_kernel<<<n, 256, 0, s>>>(clean, N, n, b.P);
  SSI_TRY(launch_check("power_ms_kernel"));
  const int64_t tot = N * n;
  add_noise_kernel<<<int((tot + 255) / 256), 256, 0, s>>>(clean, b.V, b.P, N, n, pow(10.0, snr_db / 10.0), Y, dtype,
                                                         ldY);
  return launch_check("add_noise_kernel");
}

}  // namespace ssi
