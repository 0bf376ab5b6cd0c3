// A9-A11: per-order modal sweep (§2.1, Eqs. 9-12), one CTA per order.
//
// S-free nested form (pin P10): with U^up = U[0:l(i-1), :n_max] = Q R
// (CholeskyQR2, diag R > 0) and W = Q^T U[l:li, :n_max],
//     A_n = S_n^{-1/2} (R_n^{-1} W_n) S_n^{1/2},   M_n := R_n^{-1} W_n = Rinv[:n,:n] W[:n,:n]
// (Rinv upper triangular, so its leading block is R_n^{-1}). eig(A_n) = eig(M_n) and
// Phi = C_n psi_A = U[0:l, :n] psi_M. Per order the CTA then runs
//   Householder Hessenberg reduction (global, L2-resident) with C <- C Q_H,
//   Francis double-shift QR on a banded copy in shared memory (real Schur form T,
//   LAPACK dlahqr/dlanv2 structure) with C <- C Z,
//   complex back substitution on T for every pole (Im mu > 0, 0 < xi < 1),
//   Phi = C x, normalization (reading A-15), MPC / MPD (A-16), f / xi (A-1),
// and writes the poles sorted by (f, xi).
#include <cstdio>
#include <cstdlib>

#include "linalg.cuh"
#include "rsvd.cuh"

namespace ssi {
namespace {

constexpr int NT = 256;
#ifndef SSI_ORDER_REV
#define SSI_ORDER_REV 1
#endif
constexpr bool kOrderRev = SSI_ORDER_REV != 0;   // CTAs of the largest orders launch first
constexpr int NW = NT / 32;
constexpr int WIN = 32;        // bulge-chase window (rows/cols) of the windowed Francis sweep
constexpr int BS = 5;          // reflector length: a bulge of BS - 1 shifts (6 shifts measured slower: per-sweep overhead)
constexpr int NSH = BS - 1;    // shifts per sweep (even)
constexpr int SUB = BS;        // sub-diagonals the band holds (Hessenberg + bulge)
constexpr int SPW = WIN - BS;  // bulge steps per window
constexpr int TLD = WIN + BS + 2;   // tile row stride (doubles): columns w0-1 .. (zero padded)
constexpr int TROWS = WIN + BS;     // tile rows (zero-padded rows below the window)
constexpr int HG_WARPS = 4;     // H group (band QR) warps; the rest form the C group
constexpr int HG_T = HG_WARPS * 32;
#ifndef SSI_EIG_CG_W0
#define SSI_EIG_CG_W0 (HG_WARPS + 1)
#endif
constexpr int CG_W0 = SSI_EIG_CG_W0;   // C group: warps CG_W0..7 (warp 4 shares warp 0's SMSP)
constexpr int CG_T = NT - CG_W0 * 32;
#ifndef SSI_EIG_NSLOT
#define SSI_EIG_NSLOT 8
#endif
constexpr int NSLOT = SSI_EIG_NSLOT;        // H -> C queue depth
enum { QWIN = 0, QEND = 2 };
struct QEntry {
  int type, w0, nw, nsteps;
  int chi;                      // columns > chi (deflated, never read again by the H group) are the C group's
  double r[BS * SPW];           // window reflectors (v_1..v_{BS-1}, tau) or rotation (cs, sn)
};
constexpr double kUlp = 2.220446049250313e-16;
constexpr double kSafeMin = 2.2250738585072014e-308;

// eigenvector scratch (NW complex vectors), also the windowed sweep's tile
__host__ __device__ inline size_t x_elems(int n_max) {
  const size_t a = size_t(NW) * 2 * n_max, b = size_t(TROWS) * TLD;
  return a > b ? a : b;
}
__host__ __device__ inline int band_lo(int i) { return i > SUB ? i - SUB : 0; }

__device__ __forceinline__ void hsync() { asm volatile("bar.sync 1, %0;" ::"n"(HG_T) : "memory"); }
__device__ __forceinline__ void csync() { asm volatile("bar.sync 2, %0;" ::"n"(CG_T) : "memory"); }
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a), "r"(parity)
      : "memory");
}

// seg (a row segment for right updates, a column segment for left updates: element u is index
// w0 + u) <- seg after the window's reflectors 0..nsteps-1, reflector t acting on u = t..t+BS-1
// (refl: v_1..v_{BS-1}, tau per reflector; v_j = 0 past the reflector's length).
// Branch-free: the window's unused reflector slots (u >= nsteps) hold zeros (tau = 0, v = 0),
// which leave seg bit-for-bit unchanged, so every slot is applied and the loop is one basic
// block the scheduler can pipeline.
__device__ __forceinline__ void apply_window(double (&seg)[WIN], const double* refl) {
#pragma unroll
  for (int u = 0; u < SPW; ++u) {
    const double* rf = refl + BS * u;
    double sum = seg[u];
#pragma unroll
    for (int j = 1; j < BS; ++j) sum = fma(rf[j - 1], seg[u + j], sum);
    sum *= rf[BS - 1];
    seg[u] -= sum;
#pragma unroll
    for (int j = 1; j < BS; ++j) seg[u + j] = fma(-sum, rf[j - 1], seg[u + j]);
  }
}

// apply_window on two independent segments, the two update chains interleaved
__device__ __forceinline__ void apply_window2(double (&sa)[WIN], double (&sb)[WIN], const double* refl) {
#pragma unroll
  for (int u = 0; u < SPW; ++u) {
    const double* rf = refl + BS * u;
    double r[BS];
#pragma unroll
    for (int j = 0; j < BS; ++j) r[j] = rf[j];
    double xa = sa[u], xb = sb[u];
#pragma unroll
    for (int j = 1; j < BS; ++j) { xa = fma(r[j - 1], sa[u + j], xa); xb = fma(r[j - 1], sb[u + j], xb); }
    xa *= r[BS - 1];
    xb *= r[BS - 1];
    sa[u] -= xa;
    sb[u] -= xb;
#pragma unroll
    for (int j = 1; j < BS; ++j) { sa[u + j] = fma(-xa, r[j - 1], sa[u + j]); sb[u + j] = fma(-xb, r[j - 1], sb[u + j]); }
  }
}

__host__ __device__ inline size_t band_elems(int n) {
  size_t s = 0;
  for (int i = 0; i < n; ++i) s += size_t(n - band_lo(i));
  return s;
}
__host__ __device__ inline int64_t order_off_sq(int n0, int dn, int b) {
  int64_t off = 0;
  for (int bb = 0; bb < b; ++bb) { const int64_t nb = n0 + int64_t(bb) * dn; off += nb * nb; }
  return off;
}

struct EigArgs {
  double* M;            // order slabs (col-major n x n), overwritten
  double* C;            // order slabs l x n
  const double* U;
  int64_t ldU;
  const double* S;
  int l, n_min, n_step, n_orders, n_max, cap;
  double dt;
  ssi_pole_table tab;
  int profile;          // development: print phase clocks of the largest order
  double* band_g;       // non-null: the banded H of order o lives in global memory (L2) at
                        // band_g + o * band_elems(n_max) (orders whose band exceeds shared memory)
};

struct Smem {
  double* H;      // banded Hessenberg / Schur
  int* rowoff;    // n+1
  double* x;      // NW * 2 * n: per-warp complex eigenvector
  int* cj;        // cap: block start of candidate
  int* blk;       // n_max / 2 + 1: first rows of the deflated 2 x 2 blocks (standardized after the QR)
  QEntry* q;      // NSLOT queue entries (H group -> C group)
  uint64_t* q_full;
  uint64_t* q_empty;
  uint64_t* q_rdone;   // C group finished an entry's rows above the block
  double* cre; double* cim; double* cf; double* cxi;  // cap each
};

// LAPACK dlanv2: Schur factorization of a real 2x2 nonsymmetric matrix in standardized
// form. Returns rotation (cs, sn) with [a b; c d]_in = [cs -sn; sn cs][a b; c d]_out[cs sn; -sn cs].
__device__ void dlanv2(double& a, double& b, double& c, double& d, double& cs, double& sn) {
  const double eps = kUlp * 0.5;
  if (c == 0.0) {
    cs = 1.0; sn = 0.0;
  } else if (b == 0.0) {
    cs = 0.0; sn = 1.0;
    const double t = d; d = a; a = t; b = -c; c = 0.0;
  } else if ((a - d) == 0.0 && (copysign(1.0, b) != copysign(1.0, c))) {
    cs = 1.0; sn = 0.0;
  } else {
    const double temp = a - d;
    double p = 0.5 * temp;
    const double bcmax = fmax(fabs(b), fabs(c));
    const double bcmis = fmin(fabs(b), fabs(c)) * copysign(1.0, b) * copysign(1.0, c);
    const double scale = fmax(fabs(p), bcmax);
    double z = (p / scale) * p + (bcmax / scale) * bcmis;
    if (z >= 4.0 * eps) {
      z = p + copysign(sqrt(scale) * sqrt(z), p);
      a = d + z;
      d = d - (bcmax / z) * bcmis;
      const double tau = hypot(c, z);
      cs = z / tau; sn = c / tau;
      b = b - c; c = 0.0;
    } else {
      const double sigma = b + c;
      const double tau = hypot(sigma, temp);
      cs = sqrt(0.5 * (1.0 + fabs(sigma) / tau));
      sn = -(p / (tau * cs)) * copysign(1.0, sigma);
      const double aa = a * cs + b * sn, bb = -a * sn + b * cs;
      const double cc = c * cs + d * sn, dd = -c * sn + d * cs;
      a = aa * cs + cc * sn; b = bb * cs + dd * sn;
      c = -aa * sn + cc * cs; d = -bb * sn + dd * cs;
      const double t2 = 0.5 * (a + d);
      a = t2; d = t2;
      if (c != 0.0) {
        if (b != 0.0) {
          if (copysign(1.0, b) == copysign(1.0, c)) {
            const double sab = sqrt(fabs(b)), sac = sqrt(fabs(c));
            p = copysign(sab * sac, c);
            const double tt = 1.0 / sqrt(fabs(b + c));
            a = t2 + p; d = t2 - p;
            b = b - c; c = 0.0;
            const double cs1 = sab * tt, sn1 = sac * tt;
            const double t3 = cs * cs1 - sn * sn1;
            sn = cs * sn1 + sn * cs1;
            cs = t3;
          }
        } else {
          b = -c; c = 0.0;
          const double t3 = cs; cs = -sn; sn = t3;
        }
      }
    }
  }
}

__device__ __forceinline__ bool order_truncated(const EigArgs& g, int n) {
  // orders above the numerical rank are reported (count = -1), not solved
  return !(g.S[n - 1] >= 1e-12 * g.S[0]);
}

__device__ __forceinline__ double* order_A(const EigArgs& g, int o) {
  return g.M + order_off_sq(g.n_min, g.n_step, o);
}
__device__ __forceinline__ double* order_C(const EigArgs& g, int o) {
  return g.C + int64_t(g.l) * (int64_t(o) * g.n_min + int64_t(g.n_step) * (int64_t(o) * (o - 1) / 2));
}

// ---------------------------------------------------------------- Householder Hessenberg
// One CTA (1024 threads) per order: A <- Q_H^T A Q_H in place (global, L2-resident) and
// C <- U[0:l, :n] Q_H. Left update: warp per column (coalesced, lanes over rows); right update:
// 4 warps per 32-row block split the columns (coalesced, many loads in flight).
#ifndef SSI_HESS_THREADS
#define SSI_HESS_THREADS 1024
#endif
constexpr int HT = SSI_HESS_THREADS;   // threads of the Hessenberg CTA
#ifndef SSI_HESS_QS
#define SSI_HESS_QS 2
#endif
constexpr int HQS = SSI_HESS_QS;   // warps sharing a 32-row block of the right update (column split)
constexpr int HW = HT / 32;
constexpr int kHessMaxN = 512;   // Householder vector in shared memory: orders up to 513

__global__ void __launch_bounds__(HT) hess_order_kernel(EigArgs g) {
  __shared__ double v[kHessMaxN + 8];
  __shared__ double red[HW];
  __shared__ double part[HQS][(HW / HQS) * 32];
  __shared__ double sh_tau, sh_scal, sh_beta;
  const int o = kOrderRev ? int(gridDim.x) - 1 - int(blockIdx.x) : int(blockIdx.x);   // largest order first
  const int n = g.n_min + o * g.n_step;
  if (order_truncated(g, n)) return;
  const int l = g.l;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = order_A(g, o);
  double* C = order_C(g, o);
  for (int64_t e = tid; e < int64_t(l) * n; e += HT) {
    const int64_t a = e % l, c = e / l;
    C[e] = g.U[a + c * g.ldU];
  }
  __syncthreads();
  for (int j = 0; j + 2 < n; ++j) {
    const int L = n - j - 1;   // rows j+1..n-1
    double pt = 0.0;
    for (int r = j + 2 + tid; r < n; r += HT) { const double t = A[r + int64_t(j) * n]; pt += t * t; }
    pt = warp_sum(pt);
    if (lane == 0) red[warp] = pt;
    __syncthreads();
    if (tid == 0) {
      double xn2 = 0.0;
      for (int w = 0; w < HW; ++w) xn2 += red[w];
      const double alpha = A[j + 1 + int64_t(j) * n];
      if (xn2 == 0.0) {
        sh_tau = 0.0;
      } else {
        const double beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        sh_tau = (beta - alpha) / beta;
        sh_scal = 1.0 / (alpha - beta);
        sh_beta = beta;
      }
    }
    __syncthreads();
    const double tau = sh_tau;
    if (tau == 0.0) continue;
    {
      double* col = A + int64_t(j) * n;
      const double scal = sh_scal;
      for (int r = tid; r < L; r += HT) {
        if (r == 0) { v[0] = 1.0; col[j + 1] = sh_beta; }
        else { v[r] = col[j + 1 + r] * scal; col[j + 1 + r] = 0.0; }
      }
    }
    __syncthreads();
    // left: columns j+1..n-1, two columns per warp iteration
    for (int c = j + 1 + 2 * warp; c < n; c += 2 * HW) {
      const bool two = c + 1 < n;
      double* c0 = A + int64_t(c) * n + j + 1;
      double* c1 = c0 + n;
      double w0 = 0.0, w1 = 0.0;
      for (int r = lane; r < L; r += 32) {
        const double vr = v[r];
        w0 += vr * c0[r];
        if (two) w1 += vr * c1[r];
      }
      w0 = warp_sum(w0) * tau;
      w1 = warp_sum(w1) * tau;
      for (int r = lane; r < L; r += 32) {
        const double vr = v[r];
        c0[r] -= w0 * vr;
        if (two) c1[r] -= w1 * vr;
      }
    }
    __syncthreads();
    // right: rows of A (0..n-1) then rows of C (n..n+l-1); HQS warps share a 32-row block
    const int q = warp % HQS;
    for (int rb0 = 0; rb0 < n + l; rb0 += (HW / HQS) * 32) {   // uniform trip count (barriers)
      const int rb = rb0 + (warp / HQS) * 32;
      const int r = rb + lane;
      const bool valid = r < n + l;
      double* base = nullptr;
      int64_t ld = 0;
      if (valid) {
        if (r < n) { base = A + r; ld = n; }
        else { base = C + (r - n); ld = l; }
      }
      double w = 0.0;
      if (valid) {
        // four independent partial sums, 16 loads in flight (L2 latency, not FMA, bounds this)
        double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
        int c = q;
        for (; c + 3 * HQS < L; c += 4 * HQS) {
          const double x0 = base[(j + 1 + c) * ld], x1 = base[(j + 1 + HQS + c) * ld];
          const double x2 = base[(j + 1 + 2 * HQS + c) * ld], x3 = base[(j + 1 + 3 * HQS + c) * ld];
          w0 = fma(x0, v[c], w0); w1 = fma(x1, v[c + HQS], w1);
          w2 = fma(x2, v[c + 2 * HQS], w2); w3 = fma(x3, v[c + 3 * HQS], w3);
        }
        for (; c < L; c += HQS) w0 = fma(base[(j + 1 + c) * ld], v[c], w0);
        w = (w0 + w1) + (w2 + w3);
      }
      part[q][(warp / HQS) * 32 + lane] = w;
      __syncthreads();
      if (valid) {
        const int pi = (warp / HQS) * 32 + lane;
        double ws = 0.0;
#pragma unroll
        for (int qq = 0; qq < HQS; ++qq) ws += part[qq][pi];
        ws *= tau;
        // read-modify-writes 4 in flight per thread (the row does not fit the registers)
        int c = q;
        for (; c + 3 * HQS < L; c += 4 * HQS) {
          double* p0 = base + (j + 1 + c) * ld;
          const int64_t d4 = HQS * ld;
          const double x0 = p0[0], x1 = p0[d4], x2 = p0[2 * d4], x3 = p0[3 * d4];
          p0[0] = fma(-ws, v[c], x0); p0[d4] = fma(-ws, v[c + HQS], x1);
          p0[2 * d4] = fma(-ws, v[c + 2 * HQS], x2); p0[3 * d4] = fma(-ws, v[c + 3 * HQS], x3);
        }
        for (; c < L; c += HQS) base[(j + 1 + c) * ld] -= ws * v[c];
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- Francis QR + vectors
// One CTA (256 threads) per order. The Hessenberg matrix lives in shared memory with SUB
// sub-diagonals (room for the bulge); warps 0-3 iterate on it (warp 0 chases the bulge), warps
// 5-7 apply the same transformations to the Schur vectors C.
__device__ __forceinline__ int band_off(int n, int i) {
  // offset of row i: rows 0..SUB have n entries, row r > SUB has n - r + SUB
  return i <= SUB + 1 ? i * n
                      : (SUB + 1) * n + (i - SUB - 1) * (n + SUB) - ((i - 1) * i / 2 - SUB * (SUB + 1) / 2);
}
struct Band {
  double* H;
  int n;
  __device__ __forceinline__ double& operator()(int i, int c) const {
    return H[band_off(n, i) + c - band_lo(i)];
  }
};

// Eigenvector of the quasi-triangular Schur form T for mu = wr + i wi (wi > 0) of the 2 x 2 block
// at rows (j, j + 1), by column-oriented (axpy) back substitution on one warp: x_j = 1,
// x_{j+1} = (wr - T_jj + i wi) / T_{j,j+1}, x_p = 0 beyond; the residual r_p = -sum_{q > i} T_pq x_q
// of every row p above the current one lives in registers (row p on lane p % 32, slot p / 32) and
// is updated as soon as x_i is known, so a row costs one shuffle, one complex division and one
// FMA on the dependent path (the row-oriented form needs a warp reduction per row). 1 x 1 and 2 x 2
// diagonal blocks as in LAPACK dtrevc (perturbed to smin when singular). x into xr / xim [0, j+1].
template <int KM>
__device__ __forceinline__ void eigvec_axpy(const Band& H, int j, double wr, double wi, double smin, double* xr,
                                            double* xim, int lane) {
  double rr[KM], ri[KM];
  const double b = H(j, j + 1);
  const double x1r = (wr - H(j, j)) / b, x1i = wi / b;
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    const int p = lane + 32 * k;
    rr[k] = 0.0; ri[k] = 0.0;
    if (p < j) {
      const double h0 = H(p, j), h1 = H(p, j + 1);
      rr[k] = -fma(h1, x1r, h0);
      ri[k] = -(h1 * x1i);
    }
  }
  if (lane == 0) { xr[j] = 1.0; xim[j] = 0.0; xr[j + 1] = x1r; xim[j + 1] = x1i; }
  // r_p of the (uniform) row p from its owner lane
  auto pick = [&](int p, double& vr, double& vi) {
    const int k = p >> 5;
    double sr = 0.0, si = 0.0;
#pragma unroll
    for (int kk = 0; kk < KM; ++kk)
      if (kk == k) { sr = rr[kk]; si = ri[kk]; }
    vr = __shfl_sync(0xffffffffu, sr, p & 31);
    vi = __shfl_sync(0xffffffffu, si, p & 31);
  };
  int i = j - 1;
  while (i >= 0) {
    const bool two = (i >= 1) && (H(i, i - 1) != 0.0);
    if (!two) {
      double r2r, r2i;
      pick(i, r2r, r2i);
      double dr = H(i, i) - wr, di = -wi;
      if (fma(dr, dr, di * di) < smin * smin) { dr = smin; di = 0.0; }
      const double iden = fast_rcp(fma(dr, dr, di * di));
      const double xir = (r2r * dr + r2i * di) * iden, xii = (r2i * dr - r2r * di) * iden;
      if (lane == (i & 31)) { xr[i] = xir; xim[i] = xii; }
#pragma unroll
      for (int k = 0; k < KM; ++k) {
        const int p = lane + 32 * k;
        if (p < i) {
          const double h = H(p, i);
          rr[k] = fma(-h, xir, rr[k]);
          ri[k] = fma(-h, xii, ri[k]);
        }
      }
      i -= 1;
    } else {
      // [[m00, m01], [m10, m11]] [x_{i-1}; x_i] = [r_{i-1}; r_i]
      double r1r, r1i, r2r, r2i;
      pick(i - 1, r1r, r1i);
      pick(i, r2r, r2i);
      const double m00r = H(i - 1, i - 1) - wr, m00i = -wi, m01 = H(i - 1, i);
      const double m10 = H(i, i - 1), m11r = H(i, i) - wr, m11i = -wi;
      double detr = (m00r * m11r - m00i * m11i) - m01 * m10;
      double deti = (m00r * m11i + m00i * m11r);
      if (fma(detr, detr, deti * deti) < smin * smin) { detr = smin; deti = 0.0; }
      const double iden = fast_rcp(fma(detr, detr, deti * deti));
      const double n1r = (r1r * m11r - r1i * m11i) - m01 * r2r;
      const double n1i = (r1r * m11i + r1i * m11r) - m01 * r2i;
      const double n2r = (m00r * r2r - m00i * r2i) - m10 * r1r;
      const double n2i = (m00r * r2i + m00i * r2r) - m10 * r1i;
      const double ar = (n1r * detr + n1i * deti) * iden, ai = (n1i * detr - n1r * deti) * iden;
      const double br = (n2r * detr + n2i * deti) * iden, bi = (n2i * detr - n2r * deti) * iden;
      if (lane == ((i - 1) & 31)) { xr[i - 1] = ar; xim[i - 1] = ai; }
      if (lane == (i & 31)) { xr[i] = br; xim[i] = bi; }
#pragma unroll
      for (int k = 0; k < KM; ++k) {
        const int p = lane + 32 * k;
        if (p < i - 1) {
          const double h0 = H(p, i - 1), h1 = H(p, i);
          rr[k] = fma(-h1, br, fma(-h0, ar, rr[k]));
          ri[k] = fma(-h1, bi, fma(-h0, ai, ri[k]));
        }
      }
      i -= 2;
    }
  }
  __syncwarp();
}

#ifndef SSI_EIG_MINB
#define SSI_EIG_MINB 1
#endif
// BG: the banded matrix lives in global memory (orders beyond shared memory); a separate
// instantiation so the shared-memory one addresses the band with LDS/STS, not generic accesses
template <bool BG>
__global__ void __launch_bounds__(NT, SSI_EIG_MINB) eig_order_kernel(EigArgs g) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ int sh_nblk;
  __shared__ int sh_l, sh_fail, sh_ncand;

  const int o = kOrderRev ? int(gridDim.x) - 1 - int(blockIdx.x) : int(blockIdx.x);   // largest order first
  const int n = g.n_min + o * g.n_step;
  const int l = g.l;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  ssi_pole_table T = g.tab;
  const int cap = T.cap;
  long long clk0 = clock64(), clk1 = 0, clk2 = 0, qr_its = 0;

  for (int sidx = tid; sidx < cap; sidx += NT) {
    const int64_t e = int64_t(o) * cap + sidx;
    T.f[e] = 0.0; T.xi[e] = 0.0; T.mu_re[e] = 0.0; T.mu_im[e] = 0.0; T.mpc[e] = 0.0; T.mpd[e] = 0.0;
  }
  // unused pole slots hold zeros (deterministic tables, independent of earlier contents)
  auto zero_shapes = [&](int from) {
    double* sh = T.shape + int64_t(o) * cap * l * 2;
    for (int64_t e = int64_t(from) * l * 2 + tid; e < int64_t(cap) * l * 2; e += NT) sh[e] = 0.0;
  };
  if (order_truncated(g, n)) {
    if (tid == 0) T.count[o] = -1;
    zero_shapes(0);
    return;
  }

  Smem s;
  {
    char* p = reinterpret_cast<char*>(dsm);
    const int nm = g.n_max;
    if (BG) {
      s.H = g.band_g + int64_t(o) * int64_t(band_elems(nm));
    } else {
      s.H = reinterpret_cast<double*>(p);    p += sizeof(double) * band_elems(nm);
    }
    s.x = reinterpret_cast<double*>(p);      p += sizeof(double) * x_elems(nm);
    s.cre = reinterpret_cast<double*>(p);    p += sizeof(double) * cap;
    s.cim = reinterpret_cast<double*>(p);    p += sizeof(double) * cap;
    s.cf = reinterpret_cast<double*>(p);     p += sizeof(double) * cap;
    s.cxi = reinterpret_cast<double*>(p);    p += sizeof(double) * cap;
    s.q = reinterpret_cast<QEntry*>(p);      p += sizeof(QEntry) * NSLOT;
    s.q_full = reinterpret_cast<uint64_t*>(p); p += sizeof(uint64_t) * NSLOT;
    s.q_empty = reinterpret_cast<uint64_t*>(p); p += sizeof(uint64_t) * NSLOT;
    s.q_rdone = reinterpret_cast<uint64_t*>(p); p += sizeof(uint64_t) * NSLOT;
    s.rowoff = reinterpret_cast<int*>(p);    p += sizeof(int) * (nm + 1);
    s.cj = reinterpret_cast<int*>(p);        p += sizeof(int) * cap;
    s.blk = reinterpret_cast<int*>(p);
  }
  if (tid == 0) {
    for (int i = 0; i < NSLOT; ++i) { mbar_init1(&s.q_full[i]); mbar_init1(&s.q_empty[i]); mbar_init1(&s.q_rdone[i]); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const Band H{s.H, n};
  if (tid == 0) sh_fail = 0;
  const double* A = order_A(g, o);
  double* C = order_C(g, o);
  for (int i = tid; i < n; i += NT) s.rowoff[i] = band_off(n, i) - band_lo(i);   // H(i, c) = H[rowoff[i] + c]
  for (int i = 0; i < n; ++i)
    for (int c = band_lo(i) + tid; c < n; c += NT) H(i, c) = A[i + int64_t(c) * n];
  __syncthreads();
  clk1 = clock64();

  // ---------------- Francis double-shift QR: warps 0-3 (H group) iterate on the band in shared
  // memory; warps 4-7 (C group) apply the same transformations, in the same order, to the Schur
  // vectors C (l x n, global/L2), fed through a queue of window-reflector / rotation entries.
  long long t_scan = 0, t_chase = 0, t_2x2 = 0, steps = 0, t_wchase = 0, t_wdef = 0, t_cwait = 0, t_shift = 0;
  int total_its = 0;
  if (warp < HG_WARPS) {
    const int htid = tid;
    int ihi = n - 1;
    int its = 0;
    int qslot = 0, quse = 0;          // next queue slot to fill and its use count
    int nblk = 0;                     // deflated 2 x 2 blocks so far
    const int itmax = 30 * (n > 10 ? n : 10);
    // acquire the next queue slot (all H threads call; thread 0 waits for the C group)
    auto acquire = [&]() -> QEntry* {
      if (htid == 0) { const long long tq = clock64(); mbar_wait_parity(&s.q_empty[qslot], (quse & 1) ^ 1); t_cwait += clock64() - tq; }
      hsync();
      return s.q + qslot;
    };
    int npub = 0;
    auto publish = [&]() {
      hsync();
      if (htid == 0) mbar_arrive(&s.q_full[qslot]);
      if (++qslot == NSLOT) { qslot = 0; ++quse; }
      ++npub;
    };
    // wait until the C group has finished every published entry (it also applies the windows'
    // right updates to the rows above each window; the next sweep and the 2 x 2 handling read them)
    auto drain = [&]() {
      if (npub == 0) return;
      if (htid == 0) {
        const int ls = (qslot + NSLOT - 1) % NSLOT;
        const int us = (qslot == 0) ? quse - 1 : quse;
        const long long tq = clock64();
        mbar_wait_parity(&s.q_rdone[ls], us & 1);
        t_cwait += clock64() - tq;
      }
      hsync();
    };
    while (ihi >= 0) {
      long long ta = clock64();
      // deflation test, in parallel: largest ll in (0, ihi] with a negligible subdiagonal
      if (htid == 0) sh_l = 0;
      hsync();
      for (int ll = ihi - htid; ll > 0; ll -= HG_T) {
        const double h = fabs(H(ll, ll - 1));
        bool small = h <= kSafeMin;
        if (!small) {
          double tst = fabs(H(ll - 1, ll - 1)) + fabs(H(ll, ll));
          if (tst == 0.0) {
            if (ll - 2 >= 0) tst += fabs(H(ll - 1, ll - 2));
            if (ll + 1 <= ihi) tst += fabs(H(ll + 1, ll));
          }
          small = h <= kUlp * tst;
        }
        if (small) { atomicMax(&sh_l, ll); break; }
      }
      hsync();
      const int lo = sh_l;
      long long tb = clock64();
      t_scan += tb - ta;
      if (lo > 0 && htid == 0) H(lo, lo - 1) = 0.0;
      if (lo == ihi) { ihi -= 1; its = 0; hsync(); continue; }
      if (lo == ihi - 1) {
        // a deflated 2 x 2 block: its standardization (dlanv2) and the rotation of the rows beyond
        // it, the columns above it and C are deferred to the end of the QR — rows p, q are frozen
        // from here on, and the later sweeps only apply row operations to columns p, q (which
        // commute with the deferred column rotation)
        if (htid == 0) s.blk[nblk] = ihi - 1;
        ++nblk;
        ihi -= 2; its = 0;
        t_2x2 += clock64() - tb;
        hsync();                       // sh_l is read by every H thread before thread 0 resets it
        continue;
      }
      drain();
      ++its; ++total_its;
      if (its > 100 || total_its > itmax) {
        if (htid == 0) sh_fail = 1;
        hsync();
        break;
      }
      // ---------------- one double-shift sweep over [lo, ihi], in windows of WIN rows/cols.
      // Inside a window [w0, w1) (dense tile in shared memory) warp 0 chases the bulge alone
      // (warp-synchronous); the parts of each reflector outside the window -- rows [w0, w1) x
      // columns >= w1 (left) and rows < w0 x columns [w0, w1) (right) -- are applied afterwards by
      // the H group, each row / column segment held in registers while the window's reflectors
      // stream through it; the C group applies them to the Schur vectors. Same arithmetic per
      // element as applying each reflector in turn (dlahqr); only independent updates reorder.
      {
        // First column of the shift polynomial. Normally NSH shifts per sweep (one bulge of
        // length BS = NSH + 1): the eigenvalues of the trailing NSH x NSH block, through its
        // characteristic polynomial (below). Exceptional sweeps (its = 10, 20) and small active blocks use one double shift from the
        // trailing 2 x 2 (w has 3 nonzeros; the same chase code runs with the other v_j = 0).
        double w0v[BS];
        const long long tsh0 = clock64();
        {
          double h11, h12, h21, h22;
          const bool exc = (its == 10 || its == 20);
          if (its == 10) {
            const double ex = fabs(H(lo + 1, lo)) + fabs(H(lo + 2, lo + 1));
            h11 = 0.75 * ex + H(lo, lo); h12 = -0.4375 * ex; h21 = ex; h22 = h11;
          } else if (its == 20) {
            const double ex = fabs(H(ihi, ihi - 1)) + fabs(H(ihi - 1, ihi - 2));
            h11 = 0.75 * ex + H(ihi, ihi); h12 = -0.4375 * ex; h21 = ex; h22 = h11;
          } else {
            h11 = H(ihi - 1, ihi - 1); h12 = H(ihi - 1, ihi);
            h21 = H(ihi, ihi - 1); h22 = H(ihi, ihi);
          }
          const double t1 = h11 + h22, d1 = h11 * h22 - h12 * h21;
          const bool four = !exc && (ihi - lo + 1 >= NSH + 2);
          // leading BS x NSH block of the active part
          double hh[BS][NSH];
#pragma unroll
          for (int r = 0; r < BS; ++r)
#pragma unroll
            for (int c = 0; c < NSH; ++c)
              hh[r][c] = (lo + r <= ihi && lo + c <= ihi && r <= c + 1) ? H(lo + r, lo + c) : 0.0;
          // y = (H^2 - t H + d) x for x supported on rows 0..BS-3
          auto quad = [&](const double* x, double t, double d, double* y) {
            double hx[BS], h2x[BS];
#pragma unroll
            for (int r = 0; r < BS; ++r) {
              double acc = 0.0;
#pragma unroll
              for (int c = 0; c < NSH; ++c) acc = fma(hh[r][c], x[c], acc);
              hx[r] = acc;
            }
#pragma unroll
            for (int r = 0; r < BS; ++r) {
              double acc = 0.0;
#pragma unroll
              for (int c = 0; c < NSH; ++c) acc = fma(hh[r][c], hx[c], acc);
              h2x[r] = acc;
            }
#pragma unroll
            for (int r = 0; r < BS; ++r) y[r] = fma(d, x[r], fma(-t, hx[r], h2x[r]));
          };
          double u[BS];
#pragma unroll
          for (int r = 0; r < BS; ++r) u[r] = r == 0 ? 1.0 : 0.0;
          // NSH = 4 shifts = the eigenvalues of the trailing 4 x 4 block G: the first column of
          // prod_q (H - s_q) is p(H) e_lo with p the characteristic polynomial of G, so the shifts
          // never need to be computed — every H thread forms p's coefficients (trace, principal
          // minors, det) from the broadcast-read block and evaluates p(H) e_lo by Horner's rule
          // with a running scale (no one-thread eigen-solve, no barrier).
          static_assert(NSH == 4, "characteristic-polynomial shifts assume 4 shifts");
          if (four) {
            double G[4][4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = 0; c < 4; ++c) G[r][c] = (r <= c + 1) ? H(ihi - 3 + r, ihi - 3 + c) : 0.0;
            auto m2 = [&](int a, int b) { return G[a][a] * G[b][b] - G[a][b] * G[b][a]; };
            auto m3 = [&](int a, int b, int c) {   // principal minor on rows / columns {a, b, c}
              return G[a][a] * (G[b][b] * G[c][c] - G[b][c] * G[c][b]) -
                     G[a][b] * (G[b][a] * G[c][c] - G[b][c] * G[c][a]) +
                     G[a][c] * (G[b][a] * G[c][b] - G[b][b] * G[c][a]);
            };
            const double a3 = -(G[0][0] + G[1][1] + G[2][2] + G[3][3]);
            const double a2 = m2(0, 1) + m2(0, 2) + m2(0, 3) + m2(1, 2) + m2(1, 3) + m2(2, 3);
            const double a1 = -(m3(1, 2, 3) + m3(0, 2, 3) + m3(0, 1, 3) + m3(0, 1, 2));
            // det by the first column (G[2][0] = G[3][0] = 0: Hessenberg)
            const double a0 = G[0][0] * m3(1, 2, 3) -
                              G[1][0] * (G[0][1] * (G[2][2] * G[3][3] - G[2][3] * G[3][2]) -
                                         G[0][2] * (G[2][1] * G[3][3] - G[2][3] * G[3][1]) +
                                         G[0][3] * (G[2][1] * G[3][2] - G[2][2] * G[3][1]));
            const double coef[4] = {a3, a2, a1, a0};
            double sc_run = 1.0;                   // u = (true Horner vector) * sc_run
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              double y[BS];
#pragma unroll
              for (int r = 0; r < BS; ++r) {
                double acc = 0.0;
#pragma unroll
                for (int c = 0; c < NSH; ++c) acc = fma(hh[r][c], u[c], acc);
                y[r] = acc;
              }
              y[0] = fma(coef[q], sc_run, y[0]);
              double sc = 0.0;
#pragma unroll
              for (int r = 0; r < BS; ++r) sc += fabs(y[r]);
              const double isc = sc > 0.0 ? 1.0 / sc : 1.0;
#pragma unroll
              for (int r = 0; r < BS; ++r) u[r] = y[r] * isc;
              sc_run *= isc;
            }
#pragma unroll
            for (int r = 0; r < BS; ++r) w0v[r] = u[r];
          } else {
            quad(u, t1, d1, w0v);
          }
          double sc = 0.0;
#pragma unroll
          for (int r = 0; r < BS; ++r) sc += fabs(w0v[r]);
          if (sc > 0.0) {
#pragma unroll
            for (int r = 0; r < BS; ++r) w0v[r] /= sc;
          }
        }
        t_shift += clock64() - tsh0;
        double* D = s.x;                 // TROWS x TLD tile (aliases the eigenvector scratch)
        for (int w0 = lo; w0 < ihi; ) {
          const int kend = (w0 + SPW < ihi) ? w0 + SPW : ihi;           // steps k in [w0, kend)
          const int w1 = (w0 + WIN < ihi + 1) ? w0 + WIN : ihi + 1;    // window rows [w0, w1)
          const int nw = w1 - w0;
          const int nsteps = kend - w0;
          QEntry* qe = acquire();
          // tile D[lr][lc] = H(w0 + lr, w0 - 1 + lc), lr < nw, lc <= nw (structural zeros as 0)
          for (int e = htid; e < TROWS * TLD; e += HG_T) {
            const int lr = e / TLD, lc = e - lr * TLD;
            const int r = w0 + lr, c = w0 - 1 + lc;
            D[e] = (lr < nw && lc <= nw && c >= 0 && c >= band_lo(r)) ? s.H[s.rowoff[r] + c] : 0.0;
          }
          hsync();
          const long long tw0 = clock64();
          if (warp == 0) {
            double* refl = qe->r;
            // Branch-free step (predicated code, the warp stays converged): components past the
            // reflector's length nr = min(BS, ihi - k + 1) are 0 and their row / column updates
            // are exact no-ops on the zero-padded tile; when y = 0 (tau = 0) every update is a no-op.
            for (int k = w0; k < kend; ++k) {
              const int t = k - w0;
              const int nr = (ihi - k + 1) < BS ? (ihi - k + 1) : BS;
              const bool first = (k == lo);
              // the left update's operands are final once the previous step's right update is done:
              // load them with x, so their latency overlaps the reflector's
              const int lc = t + 1 + lane;
              double bL[BS];
#pragma unroll
              for (int j = 0; j < BS; ++j) bL[j] = D[(t + j) * TLD + (lc <= nw ? lc : t + 1)];
              double xv[BS];
#pragma unroll
              for (int j = 0; j < BS; ++j) {
                const double dv = first ? w0v[j] : D[(t + j) * TLD + t];
                xv[j] = j < nr ? dv : 0.0;
              }
              const double x = xv[0];
              static_assert(BS == 5, "tree sums below assume a bulge of 5");
              // two-level trees instead of 4-long FMA chains (the step is one dependent chain)
              const double yz = fma(xv[1], xv[1], xv[2] * xv[2]) + fma(xv[3], xv[3], xv[4] * xv[4]);
              const bool refl_on = (yz != 0.0);
              // beta = -sign(x) sqrt(s); tau = 1 + |x|/sqrt(s); v = sign(x) y/(|x| + sqrt(s))
              const double ss = fma(x, x, yz);
              // rsqrt and the reciprocal of |x| + sqrt(ss) start together: the reciprocal's
              // hardware estimate uses the estimated sqrt, and its two Newton steps run on the
              // refined denominator (estimate error ~2^-21 -> ~2^-84)
              const double ssr = refl_on ? ss : 1.0;
              double rs, r0;
              asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rs) : "d"(ssr));
              asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(fabs(x) + ssr * rs));
              // Goldschmidt: g -> sqrt(ssr), h -> 1 / (2 sqrt(ssr)); one dependent FMA per step
              double g = ssr * rs, h = 0.5 * rs;
#pragma unroll
              for (int it = 0; it < 3; ++it) {
                const double rr = fma(-g, h, 0.5);
                g = fma(g, rr, g);
                h = fma(h, rr, h);
              }
              rs = h + h;
              const double sq = g;                 // (only used when refl_on, where ssr = ss)
              const double beta = -copysign(sq, x);
              const double tau = refl_on ? fma(fabs(x), rs, 1.0) : 0.0;
              const double den = fabs(x) + sq;
              r0 = fma(r0, fma(-den, r0, 1.0), r0);
              r0 = fma(r0, fma(-den, r0, 1.0), r0);
              const double inv = refl_on ? copysign(r0, x) : 0.0;
              double v[BS];
              v[0] = 1.0;
#pragma unroll
              for (int j = 1; j < BS; ++j) v[j] = xv[j] * inv;
              __syncwarp();
              // one predicated store per lane (no divergent lane-0 blocks): lanes 0..BS-1 write the
              // reduced column (beta, zeros), lanes 0..BS-1 the reflector (v_1..v_4, tau)
              if (lane < BS) {
                if (refl_on && !first && lane < nr) D[(t + lane) * TLD + t] = lane == 0 ? beta : 0.0;
                double rv = tau;
#pragma unroll
                for (int j = 1; j < BS; ++j) rv = (lane == j - 1) ? v[j] : rv;
                refl[BS * t + lane] = rv;
              }
              // left: rows t..t+BS-1, columns k..w1-1 (local t+1 .. nw)
              {
                if (lc <= nw) {
                  double* p0 = D + t * TLD + lc;
                  const double (&b)[BS] = bL;
                  double sum = fma(v[1], b[1], b[0]) + fma(v[2], b[2], fma(v[3], b[3], v[4] * b[4]));
                  sum *= tau;
                  p0[0] = b[0] - sum;
#pragma unroll
                  for (int j = 1; j < BS; ++j) p0[j * TLD] = fma(-sum, v[j], b[j]);
                }
              }
              __syncwarp();
              // right: columns k..k+BS-1 (local t+1..t+BS), rows w0..min(k+BS, ihi)
              {
                const int rmax = (k + BS < ihi ? k + BS : ihi) - w0;
                if (lane <= rmax) {
                  double* p0 = D + lane * TLD + t + 1;
                  double b[BS];
#pragma unroll
                  for (int j = 0; j < BS; ++j) b[j] = p0[j];
                  double sum = fma(v[1], b[1], b[0]) + fma(v[2], b[2], fma(v[3], b[3], v[4] * b[4]));
                  sum *= tau;
                  p0[0] = b[0] - sum;
#pragma unroll
                  for (int j = 1; j < BS; ++j) p0[j] = fma(-sum, v[j], b[j]);
                }
              }
              __syncwarp();
            }
            for (int e = BS * nsteps + lane; e < BS * SPW; e += 32) refl[e] = 0.0;   // unused slots: no-ops
            if (lane == 0) { qe->type = QWIN; qe->w0 = w0; qe->nw = nw; qe->nsteps = nsteps; qe->chi = ihi; }
          }
          publish();                     // the C group may start on this window
          const long long tw1 = clock64();
          t_wchase += tw1 - tw0;
          const double* refl = qe->r;
          // write the tile back
          for (int e = htid; e < TROWS * TLD; e += HG_T) {
            const int lr = e / TLD, lc = e - lr * TLD;
            const int r = w0 + lr, c = w0 - 1 + lc;
            if (lr < nw && lc <= nw && c >= 0 && c >= band_lo(r)) s.H[s.rowoff[r] + c] = D[e];
          }
          // deferred parts: (L) columns c in [w1, n), rows [w0, w1); (R) rows r in [0, w0),
          // columns [w0, w1)
          // columns beyond ihi (deflated: the H group never reads them again) and the rows above
          // the window are the C group's, in queue order
          const int nL = ihi + 1 - w1 > 0 ? ihi + 1 - w1 : 0, nR = 0;
          // two segments per thread, their reflector chains interleaved (independent: 2x ILP on
          // the latency-bound update chain)
          auto seg_load = [&](double (&seg)[WIN], int task) {
            if (task >= nL + nR) {
#pragma unroll
              for (int u = 0; u < WIN; ++u) seg[u] = 0.0;
            } else if (task < nL) {
              const int c = w1 + task;
#pragma unroll
              for (int u = 0; u < WIN; ++u) seg[u] = (u < nw) ? s.H[s.rowoff[w0 + u] + c] : 0.0;
            } else {
              const double* row = s.H + s.rowoff[task - nL] + w0;
#pragma unroll
              for (int u = 0; u < WIN; ++u) seg[u] = (u < nw) ? row[u] : 0.0;
            }
          };
          auto seg_store = [&](const double (&seg)[WIN], int task) {
            if (task >= nL + nR) return;
            if (task < nL) {
              const int c = w1 + task;
#pragma unroll
              for (int u = 0; u < WIN; ++u) if (u < nw) s.H[s.rowoff[w0 + u] + c] = seg[u];
            } else {
              double* row = s.H + s.rowoff[task - nL] + w0;
#pragma unroll
              for (int u = 0; u < WIN; ++u) if (u < nw) row[u] = seg[u];
            }
          };
          for (int t0 = htid; t0 < nL + nR; t0 += 2 * HG_T) {
            double sa[WIN], sb[WIN];
            seg_load(sa, t0);
            seg_load(sb, t0 + HG_T);
            apply_window2(sa, sb, refl);
            seg_store(sa, t0);
            seg_store(sb, t0 + HG_T);
          }
          hsync();
          t_wdef += clock64() - tw1;
          w0 = kend;
        }
      }
      long long tc = clock64();
      t_chase += tc - tb;
      steps += ihi - lo;
    }
    if (htid == 0) sh_nblk = nblk;
    // end of the queue
    acquire();
    if (htid == 0) s.q[qslot].type = QEND;
    publish();
  } else if (warp >= CG_W0) {
    // ---------------- C group: C[:, w0:w0+nw) <- C[:, w0:w0+nw) P_w0 ... P_{kend-1}, rotations.
    // Warp 4 stays idle: warps w and w+4 share a sub-partition, and warp 0 runs the
    // latency-bound bulge chase.
    const int ctid = tid - CG_W0 * 32;
    int slot = 0, use = 0;
    long long c_busy = 0, c_wait = 0, c_n = 0;
    while (true) {
      const long long cq0 = clock64();
      mbar_wait_parity(&s.q_full[slot], use & 1);
      const long long cq1 = clock64();
      c_wait += cq1 - cq0;
      const QEntry* e = s.q + slot;
      const int type = e->type;
      if (type == QEND) break;
      const int w0 = e->w0, nw = e->nw;
      const int chi = e->chi;
      // (1) H rows above the block (read by the H group's next sweep / 2 x 2 block): first, then
      // signal q_rdone so the H group's drain does not wait for (2)
      if (type == QWIN) {
        for (int r = ctid; r < w0; r += CG_T) {
          double* row = s.H + s.rowoff[r] + w0;
          double seg[WIN];
#pragma unroll
          for (int u = 0; u < WIN; ++u) seg[u] = (u < nw) ? row[u] : 0.0;
          apply_window(seg, e->r);
#pragma unroll
          for (int u = 0; u < WIN; ++u) if (u < nw) row[u] = seg[u];
        }
      }
      csync();
      if (ctid == 0) mbar_arrive(&s.q_rdone[slot]);
      // (2) rows of C (right) and H columns beyond chi (left; deflated, never read by the H group)
      if (type == QWIN) {
        for (int a = ctid; a < l; a += CG_T) {
          double* cr = C + a + int64_t(w0) * l;
          double seg[WIN];
#pragma unroll
          for (int u = 0; u < WIN; ++u) seg[u] = (u < nw) ? cr[int64_t(u) * l] : 0.0;
          apply_window(seg, e->r);
#pragma unroll
          for (int u = 0; u < WIN; ++u) if (u < nw) cr[int64_t(u) * l] = seg[u];
        }
        for (int c = chi + 1 + ctid; c < n; c += CG_T) {
          double seg[WIN];
#pragma unroll
          for (int u = 0; u < WIN; ++u) seg[u] = (u < nw) ? s.H[s.rowoff[w0 + u] + c] : 0.0;
          apply_window(seg, e->r);
#pragma unroll
          for (int u = 0; u < WIN; ++u) if (u < nw) s.H[s.rowoff[w0 + u] + c] = seg[u];
        }
      }
      csync();
      if (ctid == 0) mbar_arrive(&s.q_empty[slot]);
      if (++slot == NSLOT) { slot = 0; ++use; }
      c_busy += clock64() - cq1; ++c_n;
    }
    if (g.profile && ctid == 0 && (g.profile > 1 || o == g.n_orders - 1 || o == g.n_orders / 2))
      printf("eig order n=%d C group: %lld entries, busy %lld wait %lld cycles\n", n, c_n, c_busy, c_wait);
  }
  __syncthreads();
  clk2 = clock64();
  qr_its = total_its;
  if (sh_fail) {
    if (tid == 0) T.count[o] = -1;
    zero_shapes(0);
    return;
  }
  // ---------------- the deferred 2 x 2 standardizations: dlanv2 per block (one thread each), then
  // the rotations — rows p, q beyond q (left), then rows above p and the Schur vectors C in
  // columns p, q (right); blocks are disjoint index pairs, so each phase is race-free
  {
    const int nbk = sh_nblk;
    double* rcs = s.x;
    double* rsn = s.x + (g.n_max / 2 + 1);
    for (int t = tid; t < nbk; t += NT) {
      const int p = s.blk[t], q = p + 1;
      double a = H(p, p), b = H(p, q), c = H(q, p), d = H(q, q), cs, sn;
      dlanv2(a, b, c, d, cs, sn);
      H(p, p) = a; H(p, q) = b; H(q, p) = c; H(q, q) = d;
      rcs[t] = cs; rsn[t] = sn;
    }
    __syncthreads();
    for (int t = warp; t < nbk; t += NT / 32) {
      const int p = s.blk[t], q = p + 1;
      const double cs = rcs[t], sn = rsn[t];
      for (int c = q + 1 + lane; c < n; c += 32) {
        const double x = H(p, c), y = H(q, c);
        H(p, c) = cs * x + sn * y;
        H(q, c) = cs * y - sn * x;
      }
    }
    __syncthreads();
    for (int t = warp; t < nbk; t += NT / 32) {
      const int p = s.blk[t], q = p + 1;
      const double cs = rcs[t], sn = rsn[t];
      for (int r = lane; r < p; r += 32) {
        const double x = H(r, p), y = H(r, q);
        H(r, p) = cs * x + sn * y;
        H(r, q) = cs * y - sn * x;
      }
      for (int a = lane; a < l; a += 32) {
        double* cr = C + a;
        const double x = cr[int64_t(p) * l], y = cr[int64_t(q) * l];
        cr[int64_t(p) * l] = cs * x + sn * y;
        cr[int64_t(q) * l] = cs * y - sn * x;
      }
    }
    __syncthreads();
  }

  // ---------------- poles: complex pairs of the standardized Schur form. Thread 0 finds the 2 x 2
  // block starts (top-down scan, as dlahqr leaves them); the eigenvalue -> (f, xi) conversions
  // (log / atan2 / hypot) run one block per thread; the first `cap` valid poles in block order are
  // kept and ranked by (f, xi), ties by block order (a stable sort), in parallel.
  double* cand = s.x;                        // scratch (free after the QR): 6 arrays of n / 2
  const int half = n / 2 + 1;
  double *cb = cand, *cfv = cand + half, *cxv = cand + 2 * half, *crv = cand + 3 * half, *civ = cand + 4 * half,
         *cok = cand + 5 * half;
  if (tid == 0) {
    int nb = 0;
    for (int i = 0; i + 1 < n;) {
      if (H(i + 1, i) != 0.0) { cb[nb++] = double(i); i += 2; }
      else i += 1;
    }
    sh_ncand = nb;
  }
  __syncthreads();
  const int nb = sh_ncand;
  for (int t = tid; t < nb; t += NT) {
    const int i = int(cb[t]);
    const double wr = H(i, i);
    const double wi = sqrt(fabs(H(i, i + 1))) * sqrt(fabs(H(i + 1, i)));
    // lambda = ln(mu)/dt (principal branch); f = |lambda|/2pi; xi = -Re/|lambda|
    const double lr = log(hypot(wr, wi)) / g.dt, li = atan2(wi, wr) / g.dt;
    const double al = hypot(lr, li);
    const double f = al / (2.0 * 3.141592653589793), xi = -lr / al;
    cfv[t] = f; cxv[t] = xi; crv[t] = wr; civ[t] = wi;
    cok[t] = (wi > 0.0 && xi > 0.0 && xi < 1.0) ? 1.0 : 0.0;
  }
  __syncthreads();
  int kept_here = 0;
  for (int t = tid; t < nb; t += NT) {
    if (cok[t] == 0.0) continue;
    int ord = 0;                                   // valid poles before t (block order)
    for (int u = 0; u < t; ++u) ord += cok[u] != 0.0;
    if (ord >= cap) continue;
    const double f = cfv[t], xi = cxv[t];
    int rank = 0, seen = 0;
    for (int u = 0; u < nb && seen < cap; ++u) {
      if (cok[u] == 0.0) continue;
      ++seen;
      const double fu = cfv[u], xu = cxv[u];
      rank += (fu < f || (fu == f && (xu < xi || (xu == xi && u < t))));
    }
    s.cf[rank] = f; s.cxi[rank] = xi; s.cre[rank] = crv[t]; s.cim[rank] = civ[t]; s.cj[rank] = int(cb[t]);
    ++kept_here;
  }
  __syncthreads();
  if (tid == 0) sh_ncand = 0;
  __syncthreads();
  if (kept_here) atomicAdd(&sh_ncand, kept_here);
  __syncthreads();
  if (tid == 0) T.count[o] = sh_ncand;
  __syncthreads();
  const int nc = sh_ncand;
  if (tid == 0) sh_l = 0;               // reused as the pole counter of the vectors phase
  zero_shapes(nc);

  // ---------------- eigenvectors (warp per pole): back substitution on T, Phi = C x
  double* xr = s.x + warp * 2 * g.n_max;
  double* xim = xr + g.n_max;
  __syncthreads();
  // poles handed out dynamically, largest block index first (the back substitution and Phi cost
  // grow with it): the slowest warp no longer sets the phase length
  while (true) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&sh_l, 1);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= nc) break;
    c = nc - 1 - c;
    const int j = s.cj[c];
    const double wr = s.cre[c], wi = s.cim[c];
    const double smin = fmax(kUlp * hypot(wr, wi), kSafeMin);
    if (g.n_max <= 256) eigvec_axpy<8>(H, j, wr, wi, smin, xr, xim, lane);
    else eigvec_axpy<16>(H, j, wr, wi, smin, xr, xim, lane);
    // Phi = C x (C: l x n col-major), raw into the output slot
    double* shp = T.shape + (int64_t(o) * cap + c) * int64_t(l) * 2;
    double nrm2 = 0.0, best = -1.0;
    int besti = 0;
    for (int a0 = 0; a0 < l; a0 += 32 * 8) {
      // channels a0 + lane + 32 u, u < 8, accumulated together (independent chains, 8 loads of C
      // in flight per column); x_p broadcast from shared memory
      double pr[8], pi[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) { pr[u] = 0.0; pi[u] = 0.0; }
      const double* Ca = C + a0 + lane;
      for (int p = 0; p <= j + 1; ++p) {
        const double xpr = xr[p], xpi = xim[p];
        const double* Cp = Ca + int64_t(p) * l;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (a0 + lane + 32 * u < l) {
            const double cv = Cp[32 * u];
            pr[u] = fma(cv, xpr, pr[u]);
            pi[u] = fma(cv, xpi, pi[u]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int a = a0 + lane + 32 * u;
        if (a < l) {
          shp[2 * a] = pr[u]; shp[2 * a + 1] = pi[u];
          const double m2 = pr[u] * pr[u] + pi[u] * pi[u];
          nrm2 += m2;
          if (m2 > best) { best = m2; besti = a; }
        }
      }
    }
    nrm2 = warp_sum(nrm2);
#pragma unroll
    for (int ofs = 16; ofs > 0; ofs >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, ofs);
      const int oi = __shfl_xor_sync(0xffffffffu, besti, ofs);
      if (ob > best || (ob == best && oi < besti)) { best = ob; besti = oi; }
    }
    __syncwarp();
    const double pmr = shp[2 * besti], pmi = shp[2 * besti + 1];
    const double am = hypot(pmr, pmi), inv = 1.0 / sqrt(nrm2);
    const double rr = pmr / am * inv, ri = -pmi / am * inv;   // conj(phi_max)/|phi_max|/||phi||
    double sxx = 0.0, syy = 0.0, sxy = 0.0;
    __syncwarp();
    for (int a = lane; a < l; a += 32) {
      const double pr = shp[2 * a], pi = shp[2 * a + 1];
      const double qr = pr * rr - pi * ri, qi = pr * ri + pi * rr;
      shp[2 * a] = qr; shp[2 * a + 1] = qi;
      sxx += qr * qr; syy += qi * qi; sxy += qr * qi;
    }
    sxx = warp_sum(sxx); syy = warp_sum(syy); sxy = warp_sum(sxy);
    const double mpc = ((sxx - syy) * (sxx - syy) + 4.0 * sxy * sxy) / ((sxx + syy) * (sxx + syy));
    const double th = 0.5 * atan2(2.0 * sxy, sxx - syy);
    const double dx = cos(th), dy = sin(th);
    double wsum = 0.0, dsum = 0.0;
    __syncwarp();
    for (int a = lane; a < l; a += 32) {
      const double qr = shp[2 * a], qi = shp[2 * a + 1];
      const double dot = qr * dx + qi * dy, crs = qr * dy - qi * dx;
      const double mag = hypot(qr, qi);
      wsum += mag; dsum += mag * atan2(fabs(crs), fabs(dot));
    }
    wsum = warp_sum(wsum); dsum = warp_sum(dsum);
    if (lane == 0) {
      const int64_t e = int64_t(o) * cap + c;
      double mpd = dsum / wsum / (3.141592653589793 / 4.0);
      mpd = fmin(fmax(mpd, 0.0), 1.0);
      T.f[e] = s.cf[c]; T.xi[e] = s.cxi[c]; T.mu_re[e] = wr; T.mu_im[e] = wi;
      T.mpc[e] = mpc; T.mpd[e] = mpd;
    }
  }
  if (g.profile && tid == 0 && (g.profile > 1 || o == g.n_orders - 1 || o == g.n_orders / 2))
    printf("eig order n=%d: band load %lld qr %lld (its %lld) vectors %lld cycles | scan %lld chase %lld (steps %lld) cwait %lld 2x2 %lld | wchase %lld wdef %lld shift %lld\n", n, clk1 - clk0,
           clk2 - clk1, qr_its, clock64() - clk2, t_scan, t_chase, steps, t_cwait, t_2x2, t_wchase, t_wdef, t_shift);
}

}  // namespace

// dynamic shared memory of eig_order_kernel; band_global: the banded H is in global memory
size_t modal_smem_bytes(int n_max, int cap, bool band_global) {
  return sizeof(QEntry) * NSLOT + 3 * sizeof(uint64_t) * NSLOT +
         sizeof(double) * ((band_global ? 0 : band_elems(n_max)) + x_elems(n_max) +
                           4 * size_t(cap)) +
         sizeof(int) * (size_t(n_max) + 1 + cap + size_t(n_max) / 2 + 1) + 64;
}

// Orders up to ~230 keep the banded Hessenberg/Schur matrix in shared memory; beyond that (the
// paper's bridge sweeps reach order 400) it lives in an L2-resident global slab per
// order and the same kernel addresses it through generic pointers.
#ifndef SSI_EIG_BAND_GLOBAL
#define SSI_EIG_BAND_GLOBAL 0
#endif
bool modal_band_global(int n_max) {
  return SSI_EIG_BAND_GLOBAL || modal_smem_bytes(n_max, n_max / 2, false) > kModalSmemMax;
}

struct ModalWork {
  double *Rinv, *W, *M, *C, *Qup, *band;
  CholQRWork cq;
  double* partial;
};

static void modal_carve(Carver& c, int l, int i, int n_min, int n_max, int n_step, ModalWork& w) {
  const int64_t m = int64_t(l) * i, mu = m - l;
  const int no = (n_max - n_min) / n_step + 1;
  int64_t sq = 0, lin = 0;
  for (int b = 0; b < no; ++b) { const int64_t nb = n_min + int64_t(b) * n_step; sq += nb * nb; lin += nb; }
  w.Rinv = c.take<double>(size_t(n_max) * n_max);
  w.W = c.take<double>(size_t(n_max) * n_max);
  w.M = c.take<double>(size_t(sq));
  w.C = c.take<double>(size_t(lin) * l);
  w.Qup = c.take<double>(size_t(mu) * n_max);
  w.band = modal_band_global(n_max) ? c.take<double>(size_t(no) * band_elems(n_max)) : nullptr;
  {
    const size_t pg = gemm_partial_elems(n_max, n_max, gemm_pick_splits(n_max, n_max, mu));
    const size_t pt = n_max <= kTallMaxN ? gemm_tall_partial_elems(n_max, n_max, mu) : 0;
    w.partial = c.take<double>((pg > pt ? pg : pt) + 1);
  }
  cholqr_carve(c, mu, n_max, w.cq);
}

size_t modal_ws_bytes(int l, int i, int n_min, int n_max, int n_step) {
  Carver c(nullptr);
  ModalWork w;
  modal_carve(c, l, i, n_min, n_max, n_step, w);
  return c.bytes();
}

ssi_status modal_run(const double* U, int64_t ldU, const double* S, int l, int i, int n_min,
                     int n_max, int n_step, double dt, const ssi_pole_table& tab, void* ws,
                     int32_t* status, cudaStream_t st) {
  Carver c(ws);
  ModalWork w;
  modal_carve(c, l, i, n_min, n_max, n_step, w);
  const int64_t m = int64_t(l) * i, mu = m - l;
  const int no = (n_max - n_min) / n_step + 1;
  // U^up = Q R (CholeskyQR2); R^{-1} = Linv1^T Linv2^T (upper triangular)
  SSI_TRY(cholqr2(U, ldU, mu, n_max, w.Qup, w.cq, status, st));
  SSI_TRY(gemm_f64(n_max, n_max, n_max, 1.0, Operand{w.cq.Linv1, n_max, 1},
                   Operand{w.cq.Linv2, n_max, 1}, w.Rinv, n_max, 1, nullptr, st));
  // W = Q^T U^down, U^down = U[l:m, :n_max]
  // (tall-skinny DMMA kernel, split-K, when the shapes allow its 16-byte pieces)
  if (n_max <= kTallMaxN && mu % 2 == 0 && l % 2 == 0 && ldU % 2 == 0 &&
      (reinterpret_cast<uintptr_t>(U) & 15) == 0 && (reinterpret_cast<uintptr_t>(w.Qup) & 15) == 0) {
    SSI_TRY(gemm_tall(n_max, n_max, mu, true, w.Qup, mu, U + l, ldU, w.W, n_max, w.partial, st));
  } else {
    const int splits = gemm_pick_splits(n_max, n_max, mu);
    SSI_TRY(gemm_f64(n_max, n_max, mu, 1.0, Operand{w.Qup, mu, 1}, Operand{U + l, 1, ldU}, w.W,
                     n_max, splits, w.partial, st));
  }
  // M_n = Rinv[:n,:n] W[:n,:n] for every order
  SSI_TRY(gemm_f64_orders(no, n_min, n_step, w.Rinv, n_max, w.W, n_max, w.M, st));
  EigArgs g{w.M, w.C, U, ldU, S, l, n_min, n_step, no, n_max, tab.cap, dt, tab,
            getenv("SSI_EIG_PROFILE") ? atoi(getenv("SSI_EIG_PROFILE")) : 0, w.band};
  const size_t smem = modal_smem_bytes(n_max, tab.cap, w.band != nullptr);
  hess_order_kernel<<<no, HT, 0, st>>>(g);
  SSI_TRY(launch_check("hess_order_kernel"));
  if (w.band) {
    cudaFuncSetAttribute(eig_order_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    eig_order_kernel<true><<<no, NT, smem, st>>>(g);
  } else {
    cudaFuncSetAttribute(eig_order_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    eig_order_kernel<false><<<no, NT, smem, st>>>(g);
  }
  return launch_check("eig_order_kernel");
}

}  // namespace ssi
