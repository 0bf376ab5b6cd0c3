// SSI_COV_SPECTRAL: the lagged covariances of A1 (§2.1; R_k with 1/(N-k),
// DESIGN.md reading A-6) through cross-spectra of time segments, FP64 throughout — the
// structure-exploiting product SURVEY.md §8(f) NEXT-3 names.
//
// The record is cut into segments of B = F - K samples (K = lag_hi). For segment s, channel c:
//   x_s[r]  = y[sB + r][c] for r < B (zero for r >= B and past the shard end),
//   ye_s[r] = y[sB + r][c] for r < F (the segment plus a K-sample halo, zero past N).
// For 0 <= k <= K no circular wrap occurs (r + k < B + K = F), so
//   sum_t y[t+k][a] y[t][b] = (1/F) sum_f G_ab(f) e^{+2 pi i f k / F},
//   G_ab(f) = sum_s Ye_{s,a}(f) conj(X_{s,b}(f))
// exactly (up to rounding). Per segment and channel ONE complex FFT of z = x + i*ye gives
// both spectra (X = (Z(f) + conj Z(F-f))/2, Ye = (Z(f) - conj Z(F-f))/2i). The sum over
// segments is, per frequency, three real products on the FP64 tensor cores (cross_spectral.cu):
//   T1 = sum Xr Yr, T2 = sum Xi Yi, T3 = sum (Xr + Xi)(Yi - Yr); Re G = T1 + T2, Im G = T3 + T1 - T2
// (6 lp^2 S flops per frequency; the spectra are stored [f][s][channel][Re, Im], so the FFT writes
// 16-byte (Re, Im) pairs and the product reads them as 16-byte fragments).
// The inverse DFT at the K needed lags (hermitian half spectrum, weights 1 / 2 / 1, 1/(N-k)
// folded in) is a second GEMM R (l^2 x n_lags) = G (l^2 x (F+2)) W ((F+2) x n_lags).
// Work: 3 l^2 N F/B (cross-spectra) + 2 l^2 n_lags (F+2) (inverse) flops against
// 2 l^2 sum_k (N-k) for direct summation (60x fewer at c3), and the products run at FP64
// accuracy (no slicing).
#include <cmath>
#include <cstdlib>

#include "cov_spectral.cuh"
#include "gemm_f64.cuh"

namespace ssi {
namespace {

constexpr int kFftThreads = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// twiddles tw[j] = e^{-2 pi i j / F}; inverse weights W[kk + col*(F+2)], kk = 2f + part.
__global__ void spec_tables_kernel(int F, int n_lags, int lag_lo, int64_t N, int normalize, double2* tw,
                                   double* W) {
  const int64_t ld = F + 2;
  const int64_t total = F + ld * n_lags;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    if (e < F) {
      double sn, cs;
      sincospi(2.0 * double(e) / double(F), &sn, &cs);   // exact argument: e / F is a dyadic
      tw[e] = make_double2(cs, -sn);
    } else {
      const int64_t q = e - F;
      const int col = int(q / ld), kk = int(q % ld);
      const int f = kk >> 1, part = kk & 1;
      const int64_t k = lag_lo + col;
      const double wf = (f == 0 || 2 * f == F) ? 1.0 : 2.0;
      double sn, cs;
      sincospi(2.0 * double((int64_t(f) * k) % F) / double(F), &sn, &cs);
      const double v = part ? -wf * sn : wf * cs;
      const double den = double(F) * (normalize ? double(N - k) : 1.0);   // exact product
      W[q] = v / den;
    }
  }
}

// position of frequency k in the in-place decimation-in-frequency output (mixed radix 2 / 4
// digit reversal: one radix-2 stage first when log2 F is odd).
__device__ __forceinline__ int dif_pos(int k, int F, bool r2) {
  int p = 0, L = F;
  if (r2) { p += (k & 1) * (L >> 1); k >>= 1; L >>= 1; }
  while (L > 1) { p += (k & 3) * (L >> 2); k >>= 2; L >>= 2; }
  return p;
}

struct FftArgs {
  const void* Y;
  int dtype;
  int64_t N, ldY, t_begin, t_end;
  int l, lp, F, B;
  int64_t S;    // segment capacity of the spectra buffers (per-frequency stride 2 S lp)
  int64_t s0;   // first segment of this chunk (blockIdx.y = segment within the chunk)
  int64_t nseg; // segments in this chunk
  const double2* tw;
  double* A;   // [F/2+1][2S][lp]: column 2s = Re X_s, 2s+1 = Im X_s (channel contiguous)
  double* Bs;  // [F/2+1][2S][lp]: row 2s = Re Ye_s, 2s+1 = Im Ye_s
  int32_t* status;
};

// One CTA: CH channels of one segment. Load z = x + i ye, radix-2/4 DIF FFT in shared memory,
// split the two real spectra and write them in the cross-spectral GEMM's operand layouts.
// F is a compile-time constant so every loop unrolls: the record rows are loaded as CH-wide
// vectors, all of a thread's loads issued before the first use.
template <int F>
__global__ void __launch_bounds__(kFftThreads, 3) spec_fft_kernel(FftArgs g) {
  constexpr int CH = F <= 1024 ? 4 : 2;
  constexpr int FP = F + 2;                        // padded channel row (distinct banks)
  constexpr bool R2 = (__builtin_ctz(F) & 1) != 0;
  extern __shared__ __align__(16) double2 z[];     // [CH][FP]
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * CH;
  const int64_t s = blockIdx.y;
  const int64_t t0 = g.t_begin + (g.s0 + s) * g.B;
  bool bad = false;
  // ---- load: row r of the segment, CH channels per row
  constexpr int RPT = (F + kFftThreads - 1) / kFftThreads;   // rows per thread
  const bool vec = g.dtype == SSI_F32 && CH == 4 && c0 + 4 <= g.l &&
                   ((reinterpret_cast<uintptr_t>(g.Y) | uintptr_t(g.ldY * 4)) & 15) == 0;
  double v[RPT][CH];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = tid + u * kFftThreads;
    const int64_t t = t0 + r;
    const bool in = r < F && t < g.N;
    if (vec) {
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (in) q = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(g.Y) + t * g.ldY + c0));
      v[u][0] = q.x; v[u][1 % CH] = q.y; v[u][2 % CH] = q.z; v[u][3 % CH] = q.w;
    } else {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int ch = c0 + c;
        double x = 0.0;
        if (in && ch < g.l)
          x = g.dtype == SSI_F32 ? double(static_cast<const float*>(g.Y)[t * g.ldY + ch])
                                 : static_cast<const double*>(g.Y)[t * g.ldY + ch];
        v[u][c] = x;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = tid + u * kFftThreads;
    if (r < F) {
      const int64_t t = t0 + r;
      const bool xin = r < g.B && t < g.t_end;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        bad |= !isfinite(v[u][c]);
        z[c * FP + r] = make_double2(xin ? v[u][c] : 0.0, v[u][c]);
      }
    }
  }
  if (bad) set_status(g.status, SSI_ERR_NONFINITE);
  __syncthreads();
  // ---- decimation-in-frequency stages
  if (R2) {
    constexpr int q = F >> 1;
#pragma unroll
    for (int e0 = 0; e0 < q * CH; e0 += kFftThreads) {
      const int e = e0 + tid;
      if (q * CH % kFftThreads == 0 || e < q * CH) {
        const int c = e / q, n = e % q;
        double2* zc = z + c * FP;
        const double2 x0 = zc[n], x1 = zc[n + q];
        zc[n] = cadd(x0, x1);
        zc[n + q] = cmul(csub(x0, x1), __ldg(&g.tw[n]));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int L = R2 ? (F >> 1) : F; L >= 4; L >>= 2) {
    const int q = L >> 2, m = F / L;
#pragma unroll
    for (int e0 = 0; e0 < (F >> 2) * CH; e0 += kFftThreads) {
      const int e = e0 + tid;
      if ((F >> 2) * CH % kFftThreads == 0 || e < (F >> 2) * CH) {
        const int c = e / (F >> 2), b = e % (F >> 2);
        const int n = b % q, base = (b / q) * L + n;
        double2* zc = z + c * FP;
        const double2 w1 = __ldg(&g.tw[n * m]), w2 = __ldg(&g.tw[2 * n * m]), w3 = __ldg(&g.tw[3 * n * m]);
        const double2 x0 = zc[base], x1 = zc[base + q], x2 = zc[base + 2 * q], x3 = zc[base + 3 * q];
        const double2 a0 = cadd(x0, x2), a1 = csub(x0, x2), a2 = cadd(x1, x3);
        const double2 d = csub(x1, x3);
        const double2 a3 = make_double2(d.y, -d.x);   // -i (x1 - x3)
        zc[base] = cadd(a0, a2);
        zc[base + q] = cmul(cadd(a1, a3), w1);
        zc[base + 2 * q] = cmul(csub(a0, a2), w2);
        zc[base + 3 * q] = cmul(csub(a1, a3), w3);
      }
    }
    __syncthreads();
  }
  // ---- spectra of x (real part of z) and ye (imaginary part), frequencies 0..F/2
  constexpr int NF = (F >> 1) + 1;
  const int64_t sS = 2 * g.S * g.lp;   // per-frequency stride of both spectra
#pragma unroll 4
  for (int e = tid; e < NF * CH; e += kFftThreads) {
    const int f = e / CH, c = e % CH, ch = c0 + c;
    if (ch >= g.lp) continue;   // ch = l < lp (odd l): the zero padding channel
    const double2 zf = z[c * FP + dif_pos(f, F, R2)];
    const double2 zm = z[c * FP + dif_pos((F - f) & (F - 1), F, R2)];
    const int64_t off = f * sS + (s * g.lp + ch) * 2;
    __stcs(reinterpret_cast<double2*>(g.A + off), make_double2(0.5 * (zf.x + zm.x), 0.5 * (zf.y - zm.y)));    // X
    __stcs(reinterpret_cast<double2*>(g.Bs + off), make_double2(0.5 * (zf.y + zm.y), -0.5 * (zf.x - zm.x)));  // Ye
  }
}

// ---------------------------------------------------------------- F = 1024 fast path
// Three in-register DIF passes (radix 16, 16, 4) instead of five shared-memory radix-4 stages;
// shared rows padded by one element per 16 and the last pass's butterflies permuted so each
// quarter-warp hits distinct banks; a butterfly's 15 twiddles w^{rn} are formed from two table
// entries (w^n, w^{4n}) by at most two complex products; spectra written as 32-byte vectors.
__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }
#ifndef SSI_FFT_SEGS
#define SSI_FFT_SEGS 2
#endif
constexpr int kFftSegs = SSI_FFT_SEGS;   // segments per CTA of the F = 1024 kernel
constexpr int kF = 1024, kFP = kF + kF / 16 + 1;   // odd row stride: the 4 channels on distinct banks

// in-register radix-2 DIF DFT of length R (R = 16 or 4): x[bitrev(r)] = sum_m x[m] w_R^{rm}
template <int R>
__device__ __forceinline__ void dft_dif(double2 (&x)[R]) {
  // w_16^j, j < 8
  constexpr double C16[8] = {1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508974,
                             0.0, -0.38268343236508974, -0.70710678118654752, -0.92387953251128674};
  constexpr double S16[8] = {0.0, 0.38268343236508974, 0.70710678118654752, 0.92387953251128674,
                             1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508974};
#pragma unroll
  for (int h = R / 2; h >= 1; h >>= 1) {
#pragma unroll
    for (int b0 = 0; b0 < R; b0 += 2 * h) {
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const double2 a = x[b0 + j], b = x[b0 + j + h];
        x[b0 + j] = cadd(a, b);
        const double2 d = csub(a, b);
        const int t = j * (16 / (2 * h));          // w_{2h}^j = w_16^t = cos - i sin
        if (t == 0) x[b0 + j + h] = d;
        else if (t == 4) x[b0 + j + h] = make_double2(d.y, -d.x);
        else x[b0 + j + h] = cmul(d, make_double2(C16[t], -S16[t]));
      }
    }
  }
}
template <int R>
__device__ __forceinline__ constexpr int bitrev(int r) {
  int v = 0;
  for (int b = 1; b < R; b <<= 1) v = (v << 1) | ((r & b) ? 1 : 0);
  return v;
}

// y_r = x[bitrev(r)] * w^{r n} stored at base + r q; w^{rn} = (w^{4n})^{r/4} (w^n)^{r%4}
__device__ __forceinline__ void store_twiddled(double2* zc, int base, int q, const double2 (&x)[16], double2 w1,
                                               double2 w4) {
  const double2 w2 = cmul(w1, w1), w3 = cmul(w2, w1);
  const double2 w8 = cmul(w4, w4), w12 = cmul(w8, w4);
  zc[pad16(base)] = x[0];
#pragma unroll
  for (int r = 1; r < 16; ++r) {
    const int e = r & 3, hq = r >> 2;
    const double2 we = e == 1 ? w1 : (e == 2 ? w2 : w3);
    const double2 wq = hq == 1 ? w4 : (hq == 2 ? w8 : w12);
    const double2 w = e == 0 ? wq : (hq == 0 ? we : cmul(wq, we));
    zc[pad16(base + q * r)] = cmul(x[bitrev<16>(r)], w);
  }
}

template <int SEGS>
#ifndef SSI_FFT_MINB
#define SSI_FFT_MINB 2   // resident CTAs per SM declared for the 2-segment kernel
#endif
__global__ void __launch_bounds__(kFftThreads, SEGS == 1 ? 3 : SSI_FFT_MINB) spec_fft1024_kernel(FftArgs g) {
  constexpr int CH = 4;
  extern __shared__ __align__(16) double2 z[];     // [CH][kFP]
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * CH;
  const bool vec = g.dtype == SSI_F32 && c0 + 4 <= g.l &&
                   ((reinterpret_cast<uintptr_t>(g.Y) | uintptr_t(g.ldY * 4)) & 15) == 0;
  // SEGS > 1: a CTA handles SEGS consecutive segments; the next segment's rows are loaded into
  // registers while the current one is transformed (the load latency leaves the critical path)
  float4 pf[4];
  auto fetch = [&](int64_t sg) {
    const int64_t tq = g.t_begin + (g.s0 + sg) * g.B;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = tq + tid + u * kFftThreads;
      pf[u] = t < g.N ? __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(g.Y) + t * g.ldY + c0))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  const int64_t sfirst = int64_t(blockIdx.y) * SEGS;
  if (vec) fetch(sfirst);
  for (int kseg = 0; kseg < SEGS; ++kseg) {
  const int64_t s = sfirst + kseg;
  if (s >= g.nseg) break;                          // uniform over the CTA
  const int64_t t0 = g.t_begin + (g.s0 + s) * g.B;
  // ---- rows tid + 256u, CH channels per row
  {
    double v[4][CH];
    if (vec) {
#pragma unroll
      for (int u = 0; u < 4; ++u) { v[u][0] = pf[u].x; v[u][1] = pf[u].y; v[u][2] = pf[u].z; v[u][3] = pf[u].w; }
      if (kseg + 1 < SEGS && s + 1 < g.nseg) fetch(s + 1);
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t t = t0 + tid + u * kFftThreads;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int ch = c0 + c;
          double x = 0.0;
          if (t < g.N && ch < g.l)
            x = g.dtype == SSI_F32 ? double(static_cast<const float*>(g.Y)[t * g.ldY + ch])
                                   : static_cast<const double*>(g.Y)[t * g.ldY + ch];
          v[u][c] = x;
        }
      }
    }
    bool bad = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = tid + u * kFftThreads;
      const bool xin = r < g.B && t0 + r < g.t_end;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        bad |= !isfinite(v[u][c]);
        z[c * kFP + pad16(r)] = make_double2(xin ? v[u][c] : 0.0, v[u][c]);
      }
    }
    if (bad) set_status(g.status, SSI_ERR_NONFINITE);
  }
  __syncthreads();
  const int c = tid >> 6, b = tid & 63;
  double2* zc = z + c * kFP;
  // ---- pass 1: radix 16 over L = 1024 (q = 64), butterfly n = b
  {
    const double2 w1 = __ldg(&g.tw[b]), w4 = __ldg(&g.tw[4 * b]);   // w_1024^n, w_1024^{4n}
    double2 x[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) x[m] = zc[pad16(b + 64 * m)];
    dft_dif<16>(x);
    store_twiddled(zc, b, 64, x, w1, w4);
  }
  __syncthreads();
  // ---- pass 2: radix 16 over L = 64 (q = 4): block b >> 2, n = b & 3
  {
    const int n = b & 3, base = (b >> 2) * 64 + n;
    const double2 w1 = __ldg(&g.tw[16 * n]), w4 = __ldg(&g.tw[64 * n]);   // w_64^n, w_64^{4n}
    double2 x[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) x[m] = zc[pad16(base + 4 * m)];
    dft_dif<16>(x);
    store_twiddled(zc, base, 4, x, w1, w4);
  }
  __syncthreads();
  // ---- pass 3 fused with the spectrum extraction. Position d0*64 + d1*4 + r holds frequency
  // f = d0 + 16 d1 + 256 r after pass 3, and F - f sits in the partner group (d0', d1') =
  // (16 - d0, 15 - d1) (d0 > 0) or (0, 16 - d1) (d0 = 0), at r' = 3 - r: a thread loads a group
  // and its partner (the two radix-4 butterflies), transforms both in registers and writes the
  // four conjugate couples' spectra. 127 group pairs + the self-paired groups (0, 0), (0, 8) per
  // channel; lane = 4 * pair + channel, so 4 lanes write one 32-byte run.
  {
    const int cq = tid & 3;
    const double2* zq = z + cq * kFP;
    const int64_t sS = 2 * g.S * g.lp;
    double* Ab = g.A + (s * g.lp + c0 + cq) * 2;
    double* Bb = g.Bs + (s * g.lp + c0 + cq) * 2;
    auto put = [&](int f, double2 zf, double2 zm) {
      __stcs(reinterpret_cast<double2*>(Ab + f * sS), make_double2(0.5 * (zf.x + zm.x), 0.5 * (zf.y - zm.y)));  // X
      __stcs(reinterpret_cast<double2*>(Bb + f * sS), make_double2(0.5 * (zf.y + zm.y), -0.5 * (zf.x - zm.x)));  // Ye
    };
    auto group = [&](int d0, int d1, double2 (&y)[4]) {
      const int base = d0 * 64 + d1 * 4;
      double2 x[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) x[m] = zq[pad16(base + m)];
      dft_dif<4>(x);
#pragma unroll
      for (int r = 0; r < 4; ++r) y[r] = x[bitrev<4>(r)];
    };
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int pidx = (tid >> 2) + 64 * u;
      if (pidx > 128) break;
      int d0, d1;
      if (pidx < 112) { d0 = 1 + (pidx >> 4); d1 = pidx & 15; }
      else if (pidx < 120) { d0 = 8; d1 = pidx - 112; }
      else if (pidx < 127) { d0 = 0; d1 = pidx - 119; }
      else { d0 = 0; d1 = (pidx == 127) ? 0 : 8; }
      double2 ya[4];
      group(d0, d1, ya);
      if (pidx < 127) {
        const int e0 = d0 ? 16 - d0 : 0, e1 = d0 ? 15 - d1 : 16 - d1;
        double2 yb[4];
        group(e0, e1, yb);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int fa = d0 + 16 * d1 + 256 * r;     // partner frequency F - fa at (e0, e1, 3 - r)
          if (fa <= kF / 2) put(fa, ya[r], yb[3 - r]);
          else put(kF - fa, yb[3 - r], ya[r]);
        }
      } else if (d1 == 0) {                            // f = 0, 256 (with 768), 512
        put(0, ya[0], ya[0]);
        put(256, ya[1], ya[3]);
        put(512, ya[2], ya[2]);
      } else {                                         // f = 128 (with 896), 384 (with 640)
        put(128, ya[0], ya[3]);
        put(384, ya[1], ya[2]);
      }
    }
  }
  __syncthreads();                                 // z is reused by the next segment
  }
}

// ---------------------------------------------------------------- inverse transform, F = 1024
// R_k(e) = (1/den_k) Re sum_{f=0}^{F-1} G^_f(e) e^{+2 pi i f k / F}, G^ the hermitian extension of
// the half spectrum G_0..G_{F/2} (Im G_0 and Im G_{F/2} taken as 0, the weights 1 / 2 / 1 of the
// GEMM form), den_k = F (N - k) or F: the same sum as the GEMM R = G W, evaluated by an FFT
// (5 F log2 F / 2 flop per element pair instead of 2 (F + 2) n_lags). Two real outputs per
// complex transform: z_f = G^_f(e1) + i G^_f(e2) gives x(e1) + i x(e2); the inverse is the
// forward transform of conj(z), conjugated. One CTA: 4 transforms = 8 consecutive elements e
// (= (b, a) at b + a lp) of every frequency; the three in-register DIF passes of the forward
// kernel, and only the groups holding the wanted lags are finished (radix 4) and written.
#ifndef SSI_SPEC_IFFT
#define SSI_SPEC_IFFT 1   // 0: the inverse as the GEMM R = G W for every F (A/B)
#endif
struct IfftArgs {
  const double* G;     // [F/2+1][2][lp2]
  int64_t lp2;
  int lag_lo, n_lags;
  int64_t N;
  int normalize;
  const double2* tw;
  double* R;           // R[(k - lag_lo) lp2 + e]
};

__global__ void __launch_bounds__(kFftThreads, 2) spec_ifft1024_kernel(IfftArgs g) {
  constexpr int CH = 4;
  extern __shared__ __align__(16) double2 z[];     // [CH][kFP]
  const int tid = threadIdx.x;
  const int64_t e0 = int64_t(blockIdx.x) * (2 * CH);
  // ---- conj(z_f) for f = 0..F-1 from G_f (f <= F/2) and its hermitian extension
  {
    constexpr int NF = kF / 2 + 1;
    const int c = tid & 3;
    const int64_t e = e0 + 2 * c;
    const bool ok = e < g.lp2;                     // lp2 even: e + 1 < lp2 too
    double2* zc = z + c * kFP;
#pragma unroll 3
    for (int f = tid >> 2; f < NF; f += kFftThreads / 4) {
      double2 re = make_double2(0.0, 0.0), im = make_double2(0.0, 0.0);   // (a1, a2), (b1, b2)
      if (ok) {
        const double* src = g.G + int64_t(f) * 2 * g.lp2 + e;
        re = __ldcs(reinterpret_cast<const double2*>(src));
        im = __ldcs(reinterpret_cast<const double2*>(src + g.lp2));
      }
      if (f == 0 || f == kF / 2) im = make_double2(0.0, 0.0);
      // z_f = (a1 - b2) + i (b1 + a2);  z_{F-f} = (a1 + b2) + i (a2 - b1)
      zc[pad16(f)] = make_double2(re.x - im.y, -(im.x + re.y));
      if (f != 0 && f != kF / 2) zc[pad16(kF - f)] = make_double2(re.x + im.y, -(re.y - im.x));
    }
  }
  __syncthreads();
  const int c = tid >> 6, b = tid & 63;
  double2* zc = z + c * kFP;
  // ---- pass 1: radix 16 over L = 1024 (q = 64), butterfly n = b
  {
    const double2 w1 = __ldg(&g.tw[b]), w4 = __ldg(&g.tw[4 * b]);
    double2 x[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) x[m] = zc[pad16(b + 64 * m)];
    dft_dif<16>(x);
    store_twiddled(zc, b, 64, x, w1, w4);
  }
  __syncthreads();
  // ---- pass 2: radix 16 over L = 64 (q = 4): block b >> 2, n = b & 3
  {
    const int n = b & 3, base = (b >> 2) * 64 + n;
    const double2 w1 = __ldg(&g.tw[16 * n]), w4 = __ldg(&g.tw[64 * n]);
    double2 x[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) x[m] = zc[pad16(base + 4 * m)];
    dft_dif<16>(x);
    store_twiddled(zc, base, 4, x, w1, w4);
  }
  __syncthreads();
  // ---- pass 3 (radix 4) only for the wanted lags: lag k = d0 + 16 d1 + 256 r is output r of the
  // group at d0 * 64 + d1 * 4; y_r = sum_m x_m w_4^{rm}; x(e1) = Re y, x(e2) = -Im y
  for (int it = tid; it < g.n_lags * CH; it += kFftThreads) {
    const int cq = it & 3, kk = it >> 2;
    const int k = g.lag_lo + kk;
    const int64_t e = e0 + 2 * cq;
    if (e >= g.lp2) continue;
    const int d0 = k & 15, d1 = (k >> 4) & 15, r = (k >> 8) & 3;
    const double2* zq = z + cq * kFP;
    const int base = d0 * 64 + d1 * 4;
    const double2 x0 = zq[pad16(base)], x1 = zq[pad16(base + 1)], x2 = zq[pad16(base + 2)],
                  x3 = zq[pad16(base + 3)];
    double2 y;
    if (r == 0) y = make_double2((x0.x + x2.x) + (x1.x + x3.x), (x0.y + x2.y) + (x1.y + x3.y));
    else if (r == 2) y = make_double2((x0.x + x2.x) - (x1.x + x3.x), (x0.y + x2.y) - (x1.y + x3.y));
    else if (r == 1) y = make_double2((x0.x - x2.x) + (x1.y - x3.y), (x0.y - x2.y) - (x1.x - x3.x));   // -i x1, +i x3
    else y = make_double2((x0.x - x2.x) - (x1.y - x3.y), (x0.y - x2.y) + (x1.x - x3.x));
    const double den = double(kF) * (g.normalize ? double(g.N - k) : 1.0);   // as spec_tables_kernel
    __stcs(reinterpret_cast<double2*>(g.R + int64_t(kk) * g.lp2 + e), make_double2(y.x / den, -y.y / den));
  }
}

// R[lag][a][b] (l x l blocks) <- Rp[lag][a][b] (lp x lp blocks) for odd l
__global__ void spec_compact_kernel(const double* __restrict__ Rp, int l, int lp, int n_lags, double* __restrict__ R) {
  const int64_t total = int64_t(n_lags) * l * l;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = e / (int64_t(l) * l), r = e % (int64_t(l) * l);
    const int a = int(r / l), b = int(r % l);
    R[e] = Rp[k * lp * lp + int64_t(a) * lp + b];
  }
}

template <int F>
ssi_status launch_fft(const FftArgs& g, int l, int64_t nseg, cudaStream_t s) {
  constexpr int CH = F <= 1024 ? 4 : 2;
  const size_t smem = size_t(CH) * (F + 2) * sizeof(double2);
  cudaFuncSetAttribute(spec_fft_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  spec_fft_kernel<F><<<dim3(unsigned((l + CH - 1) / CH), unsigned(nseg)), kFftThreads, smem, s>>>(g);
  return launch_check("spec_fft_kernel");
}

}  // namespace

// F minimises the flop model on the full record length N (so a time shard of the same record
// uses the same F and never needs more workspace than the full record); S covers the shard.
SpecPlan spec_plan(int64_t N, int64_t span, int l, int lag_lo, int lag_hi) {
  SpecPlan p{};
  p.lp = l + (l & 1);
  p.n_lags = lag_hi - lag_lo + 1;
  double best = -1.0;
  for (int F = 64; F <= kSpecMaxF; F *= 2) {
    if (F <= lag_hi) continue;
    const int B = F - lag_hi;
    const int64_t S = (N + B - 1) / B;
    const double main = 2.0 * (2.0 * p.lp) * p.lp * (2.0 * S) * (F / 2 + 1);
    const double inv = 2.0 * double(p.lp) * p.lp * p.n_lags * (F + 2);
    if (best < 0 || main + inv < best) {
      best = main + inv;
      p.F = F;
      p.B = B;
    }
  }
  p.S = span > 0 ? (span + p.B - 1) / p.B : 1;
  // segments are processed in chunks of at most kSpecChunk (the cross-spectral product
  // accumulates over chunks), so the workspace does not grow with the record length
  const int64_t Sfull = (N + p.B - 1) / p.B;
  p.Sc = Sfull < kSpecChunk ? Sfull : kSpecChunk;
  if (p.Sc < 1) p.Sc = 1;
  return p;
}

void cov_spec_carve(Carver& c, int64_t N, int64_t span, int l, int lag_lo, int lag_hi, SpecBufs& b) {
  const SpecPlan p = spec_plan(N, span, l, lag_lo, lag_hi);
  const int64_t nf = p.F / 2 + 1;
  b.tw = c.take<double2>(size_t(p.F));
  b.W = c.take<double>(size_t(p.F + 2) * p.n_lags);
  b.A = c.take<double>(size_t(nf) * 2 * p.Sc * p.lp);
  b.Bs = c.take<double>(size_t(nf) * 2 * p.Sc * p.lp);
  b.G = c.take<double>(size_t(nf) * 2 * p.lp * p.lp);
  const int chunk = p.n_lags < kTallMaxN ? p.n_lags : kTallMaxN;
  b.partial = c.take<double>(gemm_tall_partial_elems(int64_t(p.lp) * p.lp, chunk, p.F + 2) + 1);
  b.Rp = (p.lp != l) ? c.take<double>(size_t(p.n_lags) * p.lp * p.lp) : nullptr;
}

bool cov_spec_supported(int lag_hi) { return lag_hi < kSpecMaxF; }

ssi_status cov_spectral(const void* Y, int dtype, int64_t N, int l, int64_t ldY, int lag_lo, int lag_hi,
                        int64_t t_begin, int64_t t_end, int normalize, double* R, void* ws, int32_t* status,
                        cudaStream_t s, int phases) {
  Carver c(ws);
  SpecBufs b;
  cov_spec_carve(c, N, t_end - t_begin, l, lag_lo, lag_hi, b);
  const SpecPlan p = spec_plan(N, t_end - t_begin, l, lag_lo, lag_hi);
  const int64_t nf = p.F / 2 + 1, lp2 = int64_t(p.lp) * p.lp;
  // phases: bit mask of 1 tables + FFT, 2 cross-spectral product, 4 inverse. ssi_covariances
  // always runs all three; the measurement entry point ssi_cov_spectral_phases re-runs a subset
  // on the spectra an earlier full call left in the same workspace (bench.py times the product
  // kernel alone that way).
  if (phases & 1) {
    const int64_t total = p.F + int64_t(p.F + 2) * p.n_lags;
    int blocks = int((total + 255) / 256);
    if (blocks > 148 * 4) blocks = 148 * 4;
    spec_tables_kernel<<<blocks, 256, 0, s>>>(p.F, p.n_lags, lag_lo, N, normalize, b.tw, b.W);
    SSI_TRY(launch_check("spec_tables_kernel"));
  }
  for (int64_t s0 = 0; t_end > t_begin && s0 < p.S; s0 += p.Sc) {
    const int64_t nseg = (p.S - s0 < p.Sc) ? p.S - s0 : p.Sc;
    if (phases & 1) {
      FftArgs g{Y, dtype, N, ldY, t_begin, t_end, l, p.lp, p.F, p.B, p.Sc, s0, nseg, b.tw, b.A, b.Bs, status};
      if (p.F == kF && p.lp % 4 == 0) {
        const size_t smem = size_t(4) * kFP * sizeof(double2);
        cudaFuncSetAttribute(spec_fft1024_kernel<kFftSegs>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        spec_fft1024_kernel<kFftSegs><<<dim3(unsigned((l + 3) / 4), unsigned((nseg + kFftSegs - 1) / kFftSegs)),
                                         kFftThreads, smem, s>>>(g);
        SSI_TRY(launch_check("spec_fft1024_kernel"));
      } else switch (p.F) {
        case 64: SSI_TRY(launch_fft<64>(g, l, nseg, s)); break;
        case 128: SSI_TRY(launch_fft<128>(g, l, nseg, s)); break;
        case 256: SSI_TRY(launch_fft<256>(g, l, nseg, s)); break;
        case 512: SSI_TRY(launch_fft<512>(g, l, nseg, s)); break;
        case 1024: SSI_TRY(launch_fft<1024>(g, l, nseg, s)); break;
        default: SSI_TRY(launch_fft<2048>(g, l, nseg, s)); break;
      }
    }
    if (phases & 2) {
      // G_f (+)= sum over the chunk's segments (Re G to G, Im G to G + lp^2)
      SSI_TRY(cross_spectral_3m(b.A, b.Bs, 2 * p.Sc * p.lp, nseg, p.lp, int(nf), b.G, s0 > 0, s));
    }
  }
  if (t_end <= t_begin) {

    if (cudaMemsetAsync(b.G, 0, sizeof(double) * nf * 2 * lp2, s) != cudaSuccess) return launch_check("memset G");
  }
  // R (lp^2 x n_lags) = G (lp^2 x (F+2), col-major, ld lp^2) * W ((F+2) x n_lags)
  if (!(phases & 4)) return SSI_OK;
  double* Rout = b.Rp ? b.Rp : R;
  if (SSI_SPEC_IFFT && p.F == kF && lag_hi < kF) {
    const size_t smem = size_t(4) * kFP * sizeof(double2);
    cudaFuncSetAttribute(spec_ifft1024_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const IfftArgs ia{b.G, lp2, lag_lo, p.n_lags, N, normalize, b.tw, Rout};
    spec_ifft1024_kernel<<<unsigned((lp2 + 7) / 8), kFftThreads, smem, s>>>(ia);
    SSI_TRY(launch_check("spec_ifft1024_kernel"));
  } else for (int c0 = 0; c0 < p.n_lags; c0 += kTallMaxN) {
    const int nc = p.n_lags - c0 < kTallMaxN ? p.n_lags - c0 : kTallMaxN;
    SSI_TRY(gemm_tall(lp2, nc, p.F + 2, false, b.G, lp2, b.W + int64_t(c0) * (p.F + 2), p.F + 2,
                      Rout + int64_t(c0) * lp2, lp2, b.partial, s));
  }
  if (b.Rp) {
    const int64_t total = int64_t(p.n_lags) * l * l;
    int blocks = int((total + 255) / 256);
    if (blocks > 148 * 4) blocks = 148 * 4;
    spec_compact_kernel<<<blocks, 256, 0, s>>>(b.Rp, l, p.lp, p.n_lags, R);
    SSI_TRY(launch_check("spec_compact_kernel"));
  }
  return SSI_OK;
}

}  // namespace ssi
