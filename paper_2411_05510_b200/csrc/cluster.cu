// NEXT-2: two-stage clustering of the stable poles of a 3D stabilization diagram and modal
// tracking over a monitoring campaign (§2.3 step iii; §3.1.3;
// PAPER.md:541-544, §3.2.2). Readings C-1..C-5 of DESIGN.md §3.
//
// Stage I (ssi_cluster_stage1):
//   cell_scan_kernel   one CTA: stable poles (flag 2) per (lag, order) cell -> row offsets
//   features_kernel    one CTA per cell, one warp per stable pole: best soft-criteria
//                      neighbour on the order axis (g, o-1) then the lag axis (g-1, o) ->
//                      x = (d_f, d_xi, 1-MAC, 1-MPC, MPD)                          (C-1)
//   fcm_kernel         one CTA: fuzzy C-means, c = 2, m = 2, min/max initialisation, fixed-
//                      order block reductions; physical cluster = smaller centroid norm,
//                      retained iff membership >= 0.5              (C-2, C-3)
// Stage II (ssi_cluster_stage2), on the n retained poles:
//   gather_kernel      f, xi, shape planes (re / im, channel-padded) and |shape|^2
//   rank_f_kernel      f order of the retained poles (rank by counting)
//   band_link_kernel   union-find over the edges d <= cutoff (single-linkage components), with
//                      d = d_f + d_xi + (1 - MAC) from the complex Gram
//                      S S^H on the FP64 tensor cores (DMMA) with a fused epilogue. An edge needs
//                      d_f <= cutoff, so only 64 x 64 tiles inside that f band (in f order) are
//                      formed. An average-linkage merge at height <= cutoff needs one pair
//                      <= cutoff, so every flat cluster lies inside one component and the
//                      components are clustered independently and in parallel.
//   comp_dist_kernel   each component's dense distance block (DMMA tiles from a tile list)
//   nnchain_kernel     one CTA per component: average linkage (UPGMA) by the nearest-neighbour
//                      chain with the Lance-Williams update, restricted to heights <= cutoff
//                      (a cluster whose nearest neighbour is farther than the cutoff is final:
//                      by reducibility no later merge can bring it under the cutoff)      (C-4)
//   cluster kernels    flat clusters, min_size filter, lower-median f / xi, medoid shape,
//                      order by (f, first member)                                           (C-4)
// Tracking (ssi_track): one CTA per session, candidates d_f <= df_max and 1-MAC <= macd_max,
//   greedy one-to-one assignment by ascending d_f + (1-MAC)             (C-5)
#include <math_constants.h>

#include "cluster.cuh"

namespace ssi {
namespace {

// ------------------------------------------------------------------ block helpers (1024 thr)
template <int NT>
__device__ int block_excl_scan(int v, int* sh, int& total) {
  // sh: NT/32 + 1 ints. Returns the exclusive prefix of v in thread order.
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < NT / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) sh[lane] = s;            // inclusive warp totals
  }
  __syncthreads();
  total = sh[NT / 32 - 1];
  const int before = w > 0 ? sh[w - 1] : 0;
  __syncthreads();
  return before + x - v;
}

// 1 - MAC(a, b), MAC = |a^H b|^2 / (|a|^2 |b|^2); a, b interleaved (re, im); warp-collective.
__device__ double one_minus_mac(const double* a, const double* b, int l) {
  const int lane = threadIdx.x & 31;
  double re = 0.0, im = 0.0, na = 0.0, nb = 0.0;
  for (int i = lane; i < l; i += 32) {
    const double ar = a[2 * i], ai = a[2 * i + 1], br = b[2 * i], bi = b[2 * i + 1];
    re += ar * br + ai * bi;
    im += ar * bi - ai * br;
    na += ar * ar + ai * ai;
    nb += br * br + bi * bi;
  }
  re = warp_sum(re); im = warp_sum(im); na = warp_sum(na); nb = warp_sum(nb);
  return 1.0 - (re * re + im * im) / (na * nb);
}

__device__ __forceinline__ bool hard_ok(const ssi_pole_table& t, int64_t e, const ssi_criteria& c) {
  return t.xi[e] <= c.xi_max && t.mpc[e] > c.mpc_min && t.mpd[e] < c.mpd_max;
}

__device__ __forceinline__ double rel_diff(double a, double b) { return fabs(a - b) / fmax(a, b); }

// ------------------------------------------------------------------ stage I
constexpr int kScanNT = 1024;

// Stable poles per cell (recounted from flags) -> exclusive offsets cell_off[G*O + 1].
__global__ void __launch_bounds__(kScanNT) cell_scan_kernel(const uint8_t* __restrict__ flags, int n_cells,
                                                            int cap, int* cell_off, ssi_cluster_info* info) {
  __shared__ int sh[kScanNT / 32 + 1];
  int base = 0;
  for (int c0 = 0; c0 < n_cells; c0 += kScanNT) {
    const int c = c0 + threadIdx.x;
    int cnt = 0;
    if (c < n_cells)
      for (int s = 0; s < cap; ++s) cnt += flags[int64_t(c) * cap + s] == 2;
    int total;
    const int ex = block_excl_scan<kScanNT>(cnt, sh, total);
    if (c < n_cells) cell_off[c] = base + ex;
    base += total;
  }
  if (threadIdx.x == 0) {
    cell_off[n_cells] = base;
    info->n_stable = base;
  }
}

constexpr int kFeatNT = 256;

__global__ void __launch_bounds__(kFeatNT) features_kernel(TableSet ts, int n_orders, const uint8_t* __restrict__ flags,
                                                           const int* __restrict__ cell_off, ssi_criteria c,
                                                           int max_poles, int32_t* __restrict__ pole_idx,
                                                           double* __restrict__ X, ssi_cluster_info* info,
                                                           int32_t* status) {
  const int cell = blockIdx.x;
  const int g = cell / n_orders, o = cell % n_orders;
  const ssi_pole_table& t = ts.t[g];
  const int cap = t.cap, l = t.l;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint8_t* fl = flags + int64_t(cell) * cap;
  for (int s = warp; s < cap; s += kFeatNT / 32) {
    if (fl[s] != 2) continue;
    int rank = 0;
    for (int s0 = 0; s0 < s; s0 += 32) {
      const int q = s0 + lane;
      rank += __popc(__ballot_sync(0xffffffffu, q < s && fl[q] == 2));
    }
    const int row = cell_off[cell] + rank;
    if (row >= max_poles) {
      if (lane == 0) atomicMax(&info->overflow, 1);
      continue;
    }
    const int64_t e = int64_t(o) * cap + s;
    const double f = t.f[e], xi = t.xi[e];
    const double* sh = t.shape + e * l * 2;
    bool found = false;
    double best = 0.0, bdf = 0.0, bdxi = 0.0, bdm = 0.0;
    for (int axis = 0; axis < 2; ++axis) {
      const int gg = axis == 0 ? g : g - 1, oo = axis == 0 ? o - 1 : o;
      if (gg < 0 || oo < 0) continue;
      const ssi_pole_table& u = ts.t[gg];
      const int nn = u.count[oo] > 0 ? u.count[oo] : 0;
      for (int q = 0; q < nn; ++q) {
        const int64_t eq = int64_t(oo) * cap + q;
        if (!hard_ok(u, eq, c)) continue;
        const double df = rel_diff(f, u.f[eq]);
        const double dxi = rel_diff(xi, u.xi[eq]);
        if (!(df <= c.alpha_f && dxi <= c.alpha_xi)) continue;
        const double dm = one_minus_mac(sh, u.shape + eq * l * 2, l);
        if (!(dm <= c.alpha_mac)) continue;
        const double sum = df + dxi + dm;
        if (!found || sum < best) {
          found = true;
          best = sum; bdf = df; bdxi = dxi; bdm = dm;
        }
      }
    }
    if (lane == 0) {
      pole_idx[3 * row] = g;
      pole_idx[3 * row + 1] = o;
      pole_idx[3 * row + 2] = s;
      double* x = X + 5 * int64_t(row);
      if (found) {
        x[0] = bdf; x[1] = bdxi; x[2] = bdm;
      } else {  // flag 2 without a qualifying neighbour: flags were not made with these criteria
        x[0] = x[1] = x[2] = CUDART_NAN;
        set_status(status, SSI_ERR_NUMERIC);
      }
      x[3] = 1.0 - t.mpc[e];
      x[4] = t.mpd[e];
    }
  }
}

constexpr int kFcmNT = 1024;
constexpr int kF = 5;           // features
constexpr int kRed = 2 * (1 + kF);

// Memberships of point x to centroids V (c = 2, m = 2): u_j = 1 / sum_k d_j^2 / d_k^2; a zero
// distance takes the whole membership (first such centroid).
__device__ __forceinline__ void fcm_u(const double* x, const double (*V)[kF], double& u0, double& u1) {
  double d0 = 0.0, d1 = 0.0;
#pragma unroll
  for (int f = 0; f < kF; ++f) {
    const double a = x[f] - V[0][f], b = x[f] - V[1][f];
    d0 = __dadd_rn(d0, __dmul_rn(a, a));
    d1 = __dadd_rn(d1, __dmul_rn(b, b));
  }
  if (d0 == 0.0) { u0 = 1.0; u1 = 0.0; return; }
  if (d1 == 0.0) { u0 = 0.0; u1 = 1.0; return; }
  u0 = 1.0 / (d0 / d0 + d0 / d1);
  u1 = 1.0 / (d1 / d0 + d1 / d1);
}

// Fixed-order block reduction of kRed doubles (warp xor trees, then warps in order).
__device__ void block_reduce(double* v, double (*sh)[kRed]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < kRed; ++r) v[r] = warp_sum(v[r]);
  if (lane == 0)
#pragma unroll
    for (int r = 0; r < kRed; ++r) sh[w][r] = v[r];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int r = 0; r < kRed; ++r) {
      double x = sh[lane][r];
      x = warp_sum(x);
      v[r] = x;
    }
  }
  __syncthreads();
  if (w == 0 && lane == 0)
#pragma unroll
    for (int r = 0; r < kRed; ++r) sh[0][r] = v[r];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRed; ++r) v[r] = sh[0][r];
  __syncthreads();
}

__global__ void __launch_bounds__(kFcmNT) fcm_kernel(const double* __restrict__ X, int max_poles, double tol,
                                                     int max_iter, double* __restrict__ Umem,
                                                     int32_t* __restrict__ retained, ssi_cluster_info* info) {
  __shared__ double red[kFcmNT / 32][kRed];
  __shared__ double V[2][kF];
  __shared__ double mm[kFcmNT / 32][2 * kF];
  __shared__ int sh_scan[kFcmNT / 32 + 1];
  __shared__ int done;
  const int n = min(info->n_stable, max_poles);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (n == 0) {
    if (threadIdx.x == 0) {
      info->n_retained = 0; info->fcm_iters = 0; info->phys = 0;
      for (int j = 0; j < 2 * kF; ++j) info->V[j / kF][j % kF] = 0.0;
    }
    return;
  }
  // feature-wise min / max (exact, any order)
  double lo[kF], hi[kF];
#pragma unroll
  for (int f = 0; f < kF; ++f) { lo[f] = CUDART_INF; hi[f] = -CUDART_INF; }
  for (int p = threadIdx.x; p < n; p += kFcmNT)
#pragma unroll
    for (int f = 0; f < kF; ++f) {
      const double x = X[5 * int64_t(p) + f];
      lo[f] = fmin(lo[f], x); hi[f] = fmax(hi[f], x);
    }
#pragma unroll
  for (int f = 0; f < kF; ++f)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[f] = fmin(lo[f], __shfl_xor_sync(0xffffffffu, lo[f], o));
      hi[f] = fmax(hi[f], __shfl_xor_sync(0xffffffffu, hi[f], o));
    }
  if (lane == 0)
#pragma unroll
    for (int f = 0; f < kF; ++f) { mm[w][f] = lo[f]; mm[w][kF + f] = hi[f]; }
  __syncthreads();
  if (threadIdx.x < kF) {
    const int f = threadIdx.x;
    double a = mm[0][f], b = mm[0][kF + f];
    for (int j = 1; j < kFcmNT / 32; ++j) { a = fmin(a, mm[j][f]); b = fmax(b, mm[j][kF + f]); }
    V[0][f] = a + (b - a) * 0.0;          // lo + (hi - lo) * j / (c - 1), j = 0, 1
    V[1][f] = a + (b - a) * 1.0;
  }
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  int it = 0;
  for (it = 1; it <= max_iter; ++it) {
    double acc[kRed];
#pragma unroll
    for (int r = 0; r < kRed; ++r) acc[r] = 0.0;
    for (int p = threadIdx.x; p < n; p += kFcmNT) {
      double x[kF];
#pragma unroll
      for (int f = 0; f < kF; ++f) x[f] = X[5 * int64_t(p) + f];
      double u0, u1;
      fcm_u(x, V, u0, u1);
      const double w0 = u0 * u0, w1 = u1 * u1;
      acc[0] += w0;
      acc[1 + kF] += w1;
#pragma unroll
      for (int f = 0; f < kF; ++f) { acc[1 + f] += w0 * x[f]; acc[2 + kF + f] += w1 * x[f]; }
    }
    block_reduce(acc, red);
    if (threadIdx.x == 0) {
      double delta = 0.0;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int f = 0; f < kF; ++f) {
          const double vn = acc[j * (1 + kF) + 1 + f] / acc[j * (1 + kF)];
          delta = fmax(delta, fabs(vn - V[j][f]));
          V[j][f] = vn;
        }
      done = delta < tol;
    }
    __syncthreads();
    if (done) break;
  }
  if (it > max_iter) it = max_iter;
  // physical cluster: the centroid nearer the origin (first on ties)
  __shared__ int phys;
  if (threadIdx.x == 0) {
    double nr[2];
    for (int j = 0; j < 2; ++j) {
      double s = 0.0;
      for (int f = 0; f < kF; ++f) s += V[j][f] * V[j][f];
      nr[j] = sqrt(s);
    }
    phys = nr[1] < nr[0] ? 1 : 0;
  }
  __syncthreads();
  int base = 0;
  for (int p0 = 0; p0 < n; p0 += kFcmNT) {
    const int p = p0 + threadIdx.x;
    int keep = 0;
    if (p < n) {
      double x[kF];
#pragma unroll
      for (int f = 0; f < kF; ++f) x[f] = X[5 * int64_t(p) + f];
      double u[2];
      fcm_u(x, V, u[0], u[1]);
      Umem[2 * int64_t(p)] = u[0];
      Umem[2 * int64_t(p) + 1] = u[1];
      keep = u[phys] >= 0.5;
    }
    int total;
    const int ex = block_excl_scan<kFcmNT>(keep, sh_scan, total);
    if (keep) retained[base + ex] = p;
    base += total;
  }
  if (threadIdx.x == 0) {
    info->n_retained = base;
    info->fcm_iters = it;
    info->phys = phys;
    for (int j = 0; j < 2; ++j)
      for (int f = 0; f < kF; ++f) info->V[j][f] = V[j][f];
  }
}

// ------------------------------------------------------------------ stage II
constexpr int kGathNT = 256;

// Retained pole r -> F[r], XI[r], Sre[r][lp], Sim[r][lp] (zero-padded), NRM[r] = |shape|^2.
__global__ void __launch_bounds__(kGathNT) gather_kernel(TableSet ts, const int32_t* __restrict__ pole_idx,
                                                         const int32_t* __restrict__ retained, int n, int lp,
                                                         double* F, double* XI, double* Sre, double* Sim,
                                                         double* NRM) {
  const int warp = (blockIdx.x * kGathNT + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const int pi = retained[warp];
  const int g = pole_idx[3 * pi], o = pole_idx[3 * pi + 1], s = pole_idx[3 * pi + 2];
  const ssi_pole_table& t = ts.t[g];
  const int64_t e = int64_t(o) * t.cap + s;
  const double* sh = t.shape + e * t.l * 2;
  double nr = 0.0;
  for (int c = lane; c < lp; c += 32) {
    const double re = c < t.l ? sh[2 * c] : 0.0, im = c < t.l ? sh[2 * c + 1] : 0.0;
    Sre[int64_t(warp) * lp + c] = re;
    Sim[int64_t(warp) * lp + c] = im;
    nr += re * re + im * im;
  }
  nr = warp_sum(nr);
  if (lane == 0) {
    F[warp] = t.f[e];
    XI[warp] = t.xi[e];
    NRM[warp] = nr;
  }
}

// Distance tile: d between 64 row poles ri[] and 64 column poles cj[] (retained indices, -1 =
// none; shared arrays) into Ct [64][65] (shared, aliases the staging buffers). 8 warps, warp w owns
// rows 16 (w>>1) .. +16 and columns 32 (w&1) .. +32 as 2 x 4 DMMA 8x8 blocks (re and im).
constexpr int kDT = 64, kDK = 32, kDS = kDK + 4;   // stride 36 doubles: conflict-free fragments
constexpr int kDistNT = 256;
constexpr size_t kDistSmem = size_t(4) * kDT * kDS * sizeof(double);

__device__ void dist_tile(const double* __restrict__ F, const double* __restrict__ XI,
                          const double* __restrict__ Sre, const double* __restrict__ Sim,
                          const double* __restrict__ NRM, int lp, const int* ri, const int* cj, double* smem) {
  double* Ar = smem;                 // [64][kDS]
  double* Ai = Ar + kDT * kDS;
  double* Br = Ai + kDT * kDS;
  double* Bi = Br + kDT * kDS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;
  double cre[2][4][2], cim[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) { cre[a][b][0] = cre[a][b][1] = cim[a][b][0] = cim[a][b][1] = 0.0; }
  for (int k0 = 0; k0 < lp; k0 += kDK) {
    const int kw = min(kDK, lp - k0);
    for (int e = threadIdx.x; e < kDT * kDK; e += kDistNT) {
      const int r = e / kDK, k = e % kDK;
      const bool okk = k < kw;
      const int gi = ri[r], gj = cj[r];
      Ar[r * kDS + k] = okk && gi >= 0 ? Sre[int64_t(gi) * lp + k0 + k] : 0.0;
      Ai[r * kDS + k] = okk && gi >= 0 ? Sim[int64_t(gi) * lp + k0 + k] : 0.0;
      Br[r * kDS + k] = okk && gj >= 0 ? Sre[int64_t(gj) * lp + k0 + k] : 0.0;
      Bi[r * kDS + k] = okk && gj >= 0 ? Sim[int64_t(gj) * lp + k0 + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kDK; kk += 4) {
      double ar[2], ai[2], nai[2], br[4], bi[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int r = wr + 8 * a + (lane >> 2);
        ar[a] = Ar[r * kDS + kk + (lane & 3)];
        ai[a] = Ai[r * kDS + kk + (lane & 3)];
        nai[a] = -ai[a];
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int r = wc + 8 * b + (lane >> 2);
        br[b] = Br[r * kDS + kk + (lane & 3)];
        bi[b] = Bi[r * kDS + kk + (lane & 3)];
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          // (conj(s_i) . s_j): re = ar br + ai bi, im = ar bi - ai br
          dmma884(cre[a][b][0], cre[a][b][1], ar[a], br[b]);
          dmma884(cre[a][b][0], cre[a][b][1], ai[a], bi[b]);
          dmma884(cim[a][b][0], cim[a][b][1], ar[a], bi[b]);
          dmma884(cim[a][b][0], cim[a][b][1], nai[a], br[b]);
        }
    }
    __syncthreads();
  }
  // d = d_f + d_xi + (1 - MAC); 0 on the diagonal (same pole)
  double* Ct = smem;   // [64][65]
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = wr + 8 * a + (lane >> 2), cc = wc + 8 * b + 2 * (lane & 3) + h;
        const int gi = ri[r], gj = cj[cc];
        double d = 0.0;
        if (gi >= 0 && gj >= 0 && gi != gj) {
          const double re = cre[a][b][h], im = cim[a][b][h];
          const double mac = (re * re + im * im) / (NRM[gi] * NRM[gj]);
          d = (rel_diff(F[gi], F[gj]) + rel_diff(XI[gi], XI[gj])) + (1.0 - mac);
        }
        Ct[r * (kDT + 1) + cc] = d;
      }
  __syncthreads();
}

// f-order of the retained poles: rank by counting (ties by index), ord[rank] = i, fs[rank] = f_i.
__global__ void __launch_bounds__(256) rank_f_kernel(const double* __restrict__ F, int n, int* __restrict__ ord,
                                                     double* __restrict__ fs) {
  __shared__ double fb[2048];
  const int i = blockIdx.x * 256 + threadIdx.x;
  const double fi = i < n ? F[i] : 0.0;
  int rk = 0;
  for (int j0 = 0; j0 < n; j0 += 2048) {
    const int nj = min(2048, n - j0);
    for (int e = threadIdx.x; e < nj; e += 256) fb[e] = F[j0 + e];
    __syncthreads();
    if (i < n)
      for (int e = 0; e < nj; ++e) rk += fb[e] < fi || (fb[e] == fi && j0 + e < i);
    __syncthreads();
  }
  if (i < n) { ord[rk] = i; fs[rk] = fi; }
}

// Band of candidate edges: an edge needs d <= cutoff, hence d_f <= cutoff, hence (f ascending)
// f_q <= f_p / (1 - cutoff); tile row ti needs column tiles whose first f is below
// lim[ti] = f(last pole of ti) / (1 - cutoff), widened by 1e-12 relative (rounding of d).
__global__ void band_lim_kernel(const double* __restrict__ fs, int n, double cutoff, double* __restrict__ lim) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nt = (n + kDT - 1) / kDT;
  if (t >= nt) return;
  const double fmax = fs[min(n - 1, t * kDT + kDT - 1)];
  lim[t] = cutoff < 1.0 ? fmax / (1.0 - cutoff) * (1.0 + 1e-12) : CUDART_INF;
}

__device__ void uf_union(int* parent, int a, int b);

// Edges of the band: tile (ti, tj), tj >= ti, in f order; pairs p < q (f order) with d <= cutoff
// are joined in the union-find forest (retained indices).
__global__ void __launch_bounds__(kDistNT) band_link_kernel(const double* __restrict__ F, const double* __restrict__ XI,
                                                            const double* __restrict__ Sre,
                                                            const double* __restrict__ Sim,
                                                            const double* __restrict__ NRM, int n, int lp,
                                                            const int* __restrict__ ord, const double* __restrict__ fs,
                                                            const double* __restrict__ lim, double cutoff,
                                                            int* parent) {
  const int ti = blockIdx.y, tj = blockIdx.x;
  if (tj < ti || fs[tj * kDT] > lim[ti]) return;
  extern __shared__ double smem[];
  __shared__ int ri[kDT], cj[kDT];
  if (threadIdx.x < kDT) {
    const int p = ti * kDT + threadIdx.x, q = tj * kDT + threadIdx.x;
    ri[threadIdx.x] = p < n ? ord[p] : -1;
    cj[threadIdx.x] = q < n ? ord[q] : -1;
  }
  __syncthreads();
  dist_tile(F, XI, Sre, Sim, NRM, lp, ri, cj, smem);
  const double* Ct = smem;
  for (int e = threadIdx.x; e < kDT * kDT; e += kDistNT) {
    const int r = e / kDT, cc = e % kDT;
    const int p = ti * kDT + r, q = tj * kDT + cc;
    if (p < q && q < n && Ct[r * (kDT + 1) + cc] <= cutoff) uf_union(parent, ri[r], cj[cc]);
  }
}

// Tile list of the per-component distance blocks: (component, ti, tj), tj >= ti, components of
// >= 2 members. One CTA; the count goes to *ntiles.
__global__ void __launch_bounds__(256) comp_tiles_kernel(const int* __restrict__ comp_size, const ssi_cluster_info* info,
                                                         int* __restrict__ tiles, int* ntiles) {
  __shared__ int sh[256 / 32 + 1];
  const int K = info->n_components;
  int base = 0;
  for (int c0 = 0; c0 < K; c0 += 256) {
    const int c = c0 + threadIdx.x;
    const int s = c < K ? comp_size[c] : 0;
    const int nt = s >= 2 ? (s + kDT - 1) / kDT : 0;
    const int cnt = nt * (nt + 1) / 2;
    int total;
    const int ex = block_excl_scan<256>(cnt, sh, total);
    int w = base + ex;
    for (int a = 0; a < nt; ++a)
      for (int b = a; b < nt; ++b, ++w) { tiles[3 * w] = c; tiles[3 * w + 1] = a; tiles[3 * w + 2] = b; }
    base += total;
  }
  if (threadIdx.x == 0) *ntiles = base;
}

// Per-component distance blocks from the tile list: Dco (original distances, 0 diagonal, for the
// medoids) and Dc (+inf diagonal, consumed by the nearest-neighbour chains), s x s row-major at
// comp_doff[c], rows in the component's member order (ascending retained index).
__global__ void __launch_bounds__(kDistNT) comp_dist_kernel(const double* __restrict__ F, const double* __restrict__ XI,
                                                            const double* __restrict__ Sre,
                                                            const double* __restrict__ Sim,
                                                            const double* __restrict__ NRM, int lp,
                                                            const int* __restrict__ tiles, const int* ntiles,
                                                            const int* __restrict__ comp_off,
                                                            const int* __restrict__ comp_size,
                                                            const int64_t* __restrict__ comp_doff,
                                                            const int* __restrict__ members, double* __restrict__ Dc,
                                                            double* __restrict__ Dco) {
  extern __shared__ double smem[];
  __shared__ int ri[kDT], cj[kDT];
  const int T = *ntiles;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const int c = tiles[3 * t], ti = tiles[3 * t + 1], tj = tiles[3 * t + 2];
    const int s = comp_size[c], off = comp_off[c];
    if (threadIdx.x < kDT) {
      const int p = ti * kDT + threadIdx.x, q = tj * kDT + threadIdx.x;
      ri[threadIdx.x] = p < s ? members[off + p] : -1;
      cj[threadIdx.x] = q < s ? members[off + q] : -1;
    }
    __syncthreads();
    dist_tile(F, XI, Sre, Sim, NRM, lp, ri, cj, smem);
    const double* Ct = smem;
    double* D1 = Dc + comp_doff[c];
    double* D0 = Dco + comp_doff[c];
    for (int e = threadIdx.x; e < kDT * kDT; e += kDistNT) {
      const int r = e / kDT, cc = e % kDT;
      const int p = ti * kDT + r, q = tj * kDT + cc;
      if (p < s && q < s) {
        const double d = Ct[r * (kDT + 1) + cc];
        D0[int64_t(p) * s + q] = d;
        D1[int64_t(p) * s + q] = p == q ? CUDART_INF : d;
      }
    }
    if (ti != tj)
      for (int e = threadIdx.x; e < kDT * kDT; e += kDistNT) {
        const int r = e / kDT, cc = e % kDT;     // (q, p) = tile[cc][r] transposed
        const int q = tj * kDT + r, p = ti * kDT + cc;
        if (p < s && q < s) {
          const double d = Ct[cc * (kDT + 1) + r];
          D0[int64_t(q) * s + p] = d;
          D1[int64_t(q) * s + p] = d;
        }
      }
    __syncthreads();
  }
}

// local position of every retained pole inside its component's member list
__global__ void local_index_kernel(const int* __restrict__ members, const int* __restrict__ key,
                                   const int* __restrict__ comp_off, int n, int* __restrict__ g2l) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int i = members[p];
  g2l[i] = p - comp_off[key[i]];
}

__device__ int uf_find(int* parent, int x) {
  volatile int* vp = parent;
  int p = vp[x];
  while (p != x) {
    const int gp = vp[p];
    if (gp != p) atomicCAS(&parent[x], p, gp);   // path halving
    x = p;
    p = vp[x];
  }
  return x;
}

__device__ void uf_union(int* parent, int a, int b) {
  while (true) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (a < b) { const int t = a; a = b; b = t; }      // link the larger root under the smaller
    if (atomicCAS(&parent[a], a, b) == a) return;
  }
}

__global__ void uf_init_kernel(int* parent, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) parent[i] = i;
}

__global__ void uf_flatten_kernel(int* parent, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    int x = i;
    while (parent[x] != x) x = parent[x];
    parent[i] = x;       // final root = smallest index of the component
  }
}

// One warp: stable grouping of 0..n-1 by key[i] (keys are group ids 0..K-1 with counters
// ctr[K] preset to group offsets): pos[...] in ascending i within each group.
__device__ void warp_stable_place(const int* key, int n, int* ctr, int* out) {
  const int lane = threadIdx.x & 31;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const int k = i < n ? key[i] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, k);
    const int leader = __ffs(grp) - 1;
    int base = 0;
    if (lane == leader && k >= 0) {
      base = ctr[k];
      ctr[k] = base + __popc(grp);
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    if (k >= 0) out[base + __popc(grp & ((1u << lane) - 1))] = i;
    __syncwarp();
  }
}

// Components: roots (parent[i] == i) in index order get ids; sizes, member offsets, D-block
// offsets (sum of squared sizes) and the member lists (ascending) of every component.
__global__ void __launch_bounds__(kScanNT) components_kernel(const int* __restrict__ parent, int n, int* comp_id,
                                                             int* comp_off, int* comp_size, int64_t* comp_doff,
                                                             int* ctr, int* members, int* key,
                                                             ssi_cluster_info* info) {
  __shared__ int sh[kScanNT / 32 + 1];
  int base = 0;
  for (int i0 = 0; i0 < n; i0 += kScanNT) {
    const int i = i0 + threadIdx.x;
    const int is_root = i < n && parent[i] == i;
    int total;
    const int ex = block_excl_scan<kScanNT>(is_root, sh, total);
    if (is_root) comp_id[i] = base + ex;
    base += total;
  }
  const int K = base;
  for (int c = threadIdx.x; c < K; c += kScanNT) comp_size[c] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kScanNT) {
    const int c = comp_id[parent[i]];
    key[i] = c;
    atomicAdd(&comp_size[c], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {      // offsets (K is at most n; sequential scan keeps this simple)
    int off = 0;
    int64_t doff = 0;
    for (int c = 0; c < K; ++c) {
      comp_off[c] = off;
      ctr[c] = off;
      comp_doff[c] = doff;
      off += comp_size[c];
      doff += int64_t(comp_size[c]) * comp_size[c];
    }
    comp_off[K] = off;
    comp_doff[K] = doff;
    info->n_components = K;
  }
  __syncthreads();
  if (threadIdx.x < 32) warp_stable_place(key, n, ctr, members);
}

constexpr int kChainNT = 256;

// Average linkage restricted to heights <= cutoff, one CTA per component (see header).
// Local arrays at the component's member offset: csize, chain, par (local parent), act.
// merges: (a, b) global retained indices and the height, at the component's member offset.
__global__ void __launch_bounds__(kChainNT) nnchain_kernel(double* __restrict__ Dc, const int* __restrict__ comp_off,
                                                           const int* __restrict__ comp_size,
                                                           const int64_t* __restrict__ comp_doff,
                                                           const int* __restrict__ members, ssi_cluster_info* info,
                                                           double cutoff, int* csize, int* chain, int* par,
                                                           uint8_t* act, int* m_ab, double* m_h, int* m_cnt) {
  __shared__ double wv[kChainNT / 32];
  __shared__ int wi[kChainNT / 32];
  __shared__ int s_x, s_y, s_action, s_len, s_ptr;
  const int K = info->n_components;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c = blockIdx.x; c < K; c += gridDim.x) {
    const int s = comp_size[c], off = comp_off[c];
    int* sz = csize + off;
    int* ch = chain + off;
    int* pa = par + off;
    uint8_t* ac = act + off;
    for (int i = threadIdx.x; i < s; i += kChainNT) { sz[i] = 1; pa[i] = -1; ac[i] = 1; }
    if (threadIdx.x == 0) { s_len = 0; s_ptr = 0; }
    int nm = 0;
    __syncthreads();
    if (s < 2) {
      if (threadIdx.x == 0) m_cnt[c] = 0;
      __syncthreads();
      continue;
    }
    double* Dm = Dc + comp_doff[c];
    while (true) {
      if (threadIdx.x == 0) {
        if (s_len == 0) {
          while (s_ptr < s && !ac[s_ptr]) ++s_ptr;
          if (s_ptr < s) { ch[0] = s_ptr; s_len = 1; }
        }
      }
      __syncthreads();
      if (s_len == 0) break;
      const int x = ch[s_len - 1];
      const double* row = Dm + int64_t(x) * s;
      double bv = CUDART_INF;
      int bi = 0x7fffffff;
      for (int i = threadIdx.x; i < s; i += kChainNT) {
        const double v = row[i];                 // inactive columns and the diagonal hold +inf
        if (v < bv) { bv = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { wv[w] = bv; wi[w] = bi; }
      __syncthreads();
      if (threadIdx.x == 0) {
        double dmin = wv[0];
        int imin = wi[0];
        for (int j = 1; j < kChainNT / 32; ++j)
          if (wv[j] < dmin || (wv[j] == dmin && wi[j] < imin)) { dmin = wv[j]; imin = wi[j]; }
        const int y0 = s_len > 1 ? ch[s_len - 2] : -1;
        double cm = y0 >= 0 ? row[y0] : CUDART_INF;
        int y = y0;
        if (dmin < cm) { cm = dmin; y = imin; }
        if (y0 < 0 && !(cm <= cutoff)) {
          s_action = 0; s_x = x;                 // final: no neighbour within the cutoff
          ac[x] = 0;
          s_len = 0;
        } else if (y == y0) {
          const int a = min(x, y), b = max(x, y);
          s_action = 1; s_x = a; s_y = b;
          m_ab[2 * (off + nm)] = members[off + a];
          m_ab[2 * (off + nm) + 1] = members[off + b];
          m_h[off + nm] = cm;
          pa[a] = b;
          ac[a] = 0;
          s_len -= 2;
        } else {
          s_action = 2;
          ch[s_len] = y;
          s_len += 1;
        }
      }
      __syncthreads();
      const int action = s_action;
      if (action == 0) {
        const int xx = s_x;
        for (int i = threadIdx.x; i < s; i += kChainNT) Dm[int64_t(i) * s + xx] = CUDART_INF;
      } else if (action == 1) {
        const int a = s_x, b = s_y;
        const double na = sz[a], nb = sz[b];
        const double inv = na + nb;
        for (int i = threadIdx.x; i < s; i += kChainNT) {
          const double da = Dm[int64_t(a) * s + i], db = Dm[int64_t(b) * s + i];
          // Lance-Williams, average linkage: (n_a d_ia + n_b d_ib) / (n_a + n_b), no FMA
          const double v = __ddiv_rn(__dadd_rn(__dmul_rn(na, da), __dmul_rn(nb, db)), inv);
          Dm[int64_t(b) * s + i] = v;
          Dm[int64_t(i) * s + b] = v;
          Dm[int64_t(i) * s + a] = CUDART_INF;
        }
        ++nm;
        __syncthreads();
        if (threadIdx.x == 0) sz[b] = sz[a] + sz[b];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      m_cnt[c] = nm;
      atomicAdd(&info->n_merges, nm);
    }
    __syncthreads();
  }
}

// root[i] (global retained index of the flat cluster's representative: the component member
// that absorbed the others) and the flat cluster size, for every retained pole.
__global__ void roots_kernel(const int* __restrict__ comp_off, const int* __restrict__ comp_size,
                             const int* __restrict__ members, const int* __restrict__ par,
                             const int* __restrict__ csize, const ssi_cluster_info* info, int* root,
                             int* rsize) {
  const int K = info->n_components;
  for (int c = blockIdx.x; c < K; c += gridDim.x) {
    const int s = comp_size[c], off = comp_off[c];
    for (int k = threadIdx.x; k < s; k += blockDim.x) {
      int x = k;
      while (par[off + x] >= 0) x = par[off + x];
      const int gi = members[off + k];
      root[gi] = members[off + x];
      if (x == k) rsize[gi] = s < 2 ? 1 : csize[off + x];
    }
  }
}

// Kept flat clusters (size >= min_size) in root-index order, their member lists (ascending).
__global__ void __launch_bounds__(kScanNT) flat_kernel(const int* __restrict__ root, const int* __restrict__ rsize,
                                                       int n, int min_size, int* cid, int* cl_root, int* cl_off,
                                                       int* ctr, int* key, int* cl_members,
                                                       ssi_cluster_info* info) {
  __shared__ int sh[kScanNT / 32 + 1];
  int base = 0;
  for (int i0 = 0; i0 < n; i0 += kScanNT) {
    const int i = i0 + threadIdx.x;
    const int kept = i < n && root[i] == i && rsize[i] >= min_size;
    int total;
    const int ex = block_excl_scan<kScanNT>(kept, sh, total);
    if (i < n) cid[i] = kept ? base + ex : -1;
    if (kept) cl_root[base + ex] = i;
    base += total;
  }
  const int K = base;
  __syncthreads();
  if (threadIdx.x == 0) {
    int off = 0;
    for (int k = 0; k < K; ++k) {
      cl_off[k] = off;
      ctr[k] = off;
      off += rsize[cl_root[k]];
    }
    cl_off[K] = off;
    info->n_clusters = K;
  }
  for (int i = threadIdx.x; i < n; i += kScanNT) key[i] = cid[root[i]];
  __syncthreads();
  if (threadIdx.x < 32) warp_stable_place(key, n, ctr, cl_members);
}

// Per kept cluster: lower median of f and xi (rank selection), medoid (least summed original
// distance to the other members, lowest index on ties), first member.
__global__ void __launch_bounds__(256) summary_kernel(const double* __restrict__ Dco,
                                                      const int64_t* __restrict__ comp_doff,
                                                      const int* __restrict__ comp_size, const int* __restrict__ key,
                                                      const int* __restrict__ g2l,
                                                      const double* __restrict__ F, const double* __restrict__ XI,
                                                      const int* __restrict__ cl_off,
                                                      const int* __restrict__ cl_members, const ssi_cluster_info* info,
                                                      double* kf, double* kxi, int* kmed, int* kfirst, int* ksize) {
  __shared__ double bv[8];
  __shared__ int bi[8];
  const int K = info->n_clusters;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = blockIdx.x; k < K; k += gridDim.x) {
    const int off = cl_off[k], s = cl_off[k + 1] - off;
    const int* mem = cl_members + off;
    const int med = (s - 1) / 2;
    for (int a = threadIdx.x; a < s; a += 256) {
      const double fa = F[mem[a]], xa = XI[mem[a]];
      int rf = 0, rx = 0;
      for (int b = 0; b < s; ++b) {
        const double fb = F[mem[b]], xb = XI[mem[b]];
        rf += fb < fa || (fb == fa && b < a);
        rx += xb < xa || (xb == xa && b < a);
      }
      if (rf == med) kf[k] = fa;
      if (rx == med) kxi[k] = xa;
    }
    double best = CUDART_INF;
    int besti = 0x7fffffff;
    // a flat cluster lies inside one component: its original distances are in that component's
    // block (rows / columns in the component's member order)
    const int comp = key[mem[0]];
    const int cs = comp_size[comp];
    const double* Db = Dco + comp_doff[comp];
    for (int a = threadIdx.x; a < s; a += 256) {
      double sum = 0.0;
      if (cs >= 2) {
        const double* row = Db + int64_t(g2l[mem[a]]) * cs;
        for (int b = 0; b < s; ++b) sum += row[g2l[mem[b]]];
      }
      if (sum < best || (sum == best && a < besti)) { best = sum; besti = a; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, besti, o);
      if (ov < best || (ov == best && oi < besti)) { best = ov; besti = oi; }
    }
    if (lane == 0) { bv[w] = best; bi[w] = besti; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int j = 1; j < 8; ++j)
        if (bv[j] < bv[0] || (bv[j] == bv[0] && bi[j] < bi[0])) { bv[0] = bv[j]; bi[0] = bi[j]; }
      kmed[k] = mem[bi[0]];
      kfirst[k] = mem[0];
      ksize[k] = s;
    }
    __syncthreads();
  }
}

// Order clusters by (f, first member); write outputs and labels.
__global__ void __launch_bounds__(256) order_kernel(TableSet ts, const int32_t* __restrict__ pole_idx,
                                                    const int32_t* __restrict__ retained, int n,
                                                    const int* __restrict__ root, const int* __restrict__ cid,
                                                    const double* kf, const double* kxi, const int* kmed,
                                                    const int* kfirst, const int* ksize, int* krank,
                                                    ssi_cluster_info* info, int max_clusters, int32_t* labels,
                                                    double* cl_f, double* cl_xi, int32_t* cl_size,
                                                    int32_t* cl_medoid, double* cl_shape) {
  const int K = info->n_clusters;
  for (int k = threadIdx.x; k < K; k += 256) {
    int r = 0;
    for (int j = 0; j < K; ++j) r += kf[j] < kf[k] || (kf[j] == kf[k] && kfirst[j] < kfirst[k]);
    krank[k] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0 && K > max_clusters) atomicMax(&info->overflow, 1);
  const int l = ts.t[0].l;
  for (int k = 0; k < K; ++k) {
    const int r = krank[k];
    if (r >= max_clusters) continue;
    if (threadIdx.x == 0) {
      cl_f[r] = kf[k];
      cl_xi[r] = kxi[k];
      cl_size[r] = ksize[k];
      cl_medoid[r] = kmed[k];
    }
    const int pi = retained[kmed[k]];
    const ssi_pole_table& t = ts.t[pole_idx[3 * pi]];
    const int64_t e = int64_t(pole_idx[3 * pi + 1]) * t.cap + pole_idx[3 * pi + 2];
    for (int c = threadIdx.x; c < 2 * l; c += 256) cl_shape[int64_t(r) * 2 * l + c] = t.shape[e * 2 * l + c];
  }
  for (int i = threadIdx.x; i < n; i += 256) {
    const int k = cid[root[i]];
    labels[i] = k >= 0 && krank[k] < max_clusters ? krank[k] : -1;
  }
}

// ------------------------------------------------------------------ tracking (C-5)
constexpr int kTrackNT = 256;

__global__ void __launch_bounds__(kTrackNT) track_kernel(const double* __restrict__ ref_f,
                                                         const double* __restrict__ ref_shape, int n_ref,
                                                         const double* __restrict__ f, const double* __restrict__ shape,
                                                         const int32_t* __restrict__ count, int max_modes, int l,
                                                         double df_max, double macd_max, int32_t* match) {
  extern __shared__ double tsm[];
  const int sess = blockIdx.x;
  const int nc = min(max(count[sess], 0), max_modes);
  const int P = n_ref * nc;
  double* score = tsm;                                   // [P]
  int* ok = reinterpret_cast<int*>(score + P);           // [P]
  int* order = ok + P;                                   // [P]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* sf = f + int64_t(sess) * max_modes;
  const double* ss = shape + int64_t(sess) * max_modes * l * 2;
  for (int p = warp; p < P; p += kTrackNT / 32) {
    const int r = p / nc, c = p % nc;
    const double df = rel_diff(sf[c], ref_f[r]);
    const double dm = one_minus_mac(ss + int64_t(c) * l * 2, ref_shape + int64_t(r) * l * 2, l);
    if (lane == 0) {
      ok[p] = df <= df_max && dm <= macd_max;
      score[p] = df + dm;
    }
  }
  __syncthreads();
  // ascending (score, r, c): p = r * nc + c, so (r, c) order is p order
  for (int p = threadIdx.x; p < P; p += kTrackNT) {
    if (!ok[p]) continue;
    int rk = 0;
    for (int q = 0; q < P; ++q)
      rk += ok[q] && (score[q] < score[p] || (score[q] == score[p] && q < p));
    order[rk] = p;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t* mt = match + int64_t(sess) * n_ref;
    int n_ok = 0;
    for (int p = 0; p < P; ++p) n_ok += ok[p];
    for (int r = 0; r < n_ref; ++r) mt[r] = -1;
    // used flags of the candidates reuse ok[] (a pair's ok is no longer needed once ranked)
    for (int c = 0; c < nc; ++c) ok[c] = 0;
    for (int j = 0; j < n_ok; ++j) {
      const int p = order[j], r = p / nc, c = p % nc;
      if (mt[r] < 0 && !ok[c]) {
        mt[r] = c;
        ok[c] = 1;
      }
    }
  }
}

__global__ void success_kernel(const int32_t* __restrict__ match, int n_sess, int n_ref, double* success) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_ref) return;
  int cnt = 0;
  for (int s = 0; s < n_sess; ++s) cnt += match[int64_t(s) * n_ref + r] >= 0;
  success[r] = 100.0 * double(cnt) / double(n_sess);
}

__global__ void merges_kernel(const int* __restrict__ comp_off, const int* __restrict__ m_cnt,
                              const int* __restrict__ m_ab, const double* __restrict__ m_h,
                              const ssi_cluster_info* info, int n, int32_t* out_ab, double* out_h) {
  __shared__ int base;
  const int K = info->n_components;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int c = 0; c < K; ++c) {
    const int cnt = m_cnt[c], off = comp_off[c];
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
      if (out_ab) { out_ab[2 * (base + j)] = m_ab[2 * (off + j)]; out_ab[2 * (base + j) + 1] = m_ab[2 * (off + j) + 1]; }
      if (out_h) out_h[base + j] = m_h[off + j];
    }
    __syncthreads();
    if (threadIdx.x == 0) base += cnt;
    __syncthreads();
  }
  for (int j = base + threadIdx.x; j < n; j += blockDim.x) {
    if (out_ab) { out_ab[2 * j] = -1; out_ab[2 * j + 1] = -1; }
    if (out_h) out_h[j] = CUDART_NAN;
  }
}

__global__ void info_reset2_kernel(ssi_cluster_info* info) {
  info->n_components = 0;
  info->n_clusters = 0;
  info->n_merges = 0;
}

}  // namespace

// ------------------------------------------------------------------ host side
size_t cluster_stage1_ws_bytes(int n_lags, int n_orders) {
  Carver c(nullptr);
  c.take<int>(size_t(n_lags) * n_orders + 1);
  return c.bytes();
}

ssi_status cluster_stage1_run(const TableSet& ts, int n_lags, const ssi_criteria& crit, const uint8_t* flags,
                              int max_poles, double fcm_tol, int fcm_max_iter, int32_t* pole_idx, double* X,
                              double* Umem, int32_t* retained, ssi_cluster_info* info, void* ws, int32_t* status,
                              cudaStream_t s) {
  const int no = ts.t[0].n_orders, cap = ts.t[0].cap;
  Carver c(ws);
  int* cell_off = c.take<int>(size_t(n_lags) * no + 1);
  if (cudaMemsetAsync(info, 0, sizeof(ssi_cluster_info), s) != cudaSuccess) return launch_check("memset info");
  cell_scan_kernel<<<1, kScanNT, 0, s>>>(flags, n_lags * no, cap, cell_off, info);
  SSI_TRY(launch_check("cell_scan_kernel"));
  features_kernel<<<n_lags * no, kFeatNT, 0, s>>>(ts, no, flags, cell_off, crit, max_poles, pole_idx, X, info,
                                                  status);
  SSI_TRY(launch_check("features_kernel"));
  fcm_kernel<<<1, kFcmNT, 0, s>>>(X, max_poles, fcm_tol, fcm_max_iter, Umem, retained, info);
  return launch_check("fcm_kernel");
}

namespace {
struct Stage2Bufs {
  double *F, *XI, *Sre, *Sim, *NRM, *Dco, *Dc, *kf, *kxi, *m_h, *fs, *lim;
  int *ord, *tiles, *ntiles, *g2l;
  int *parent, *comp_id, *comp_off, *comp_size, *ctr, *members, *key, *key2, *csize, *chain, *par, *root, *rsize,
      *cid, *cl_root, *cl_off, *cl_members, *kmed, *kfirst, *ksize, *krank, *m_cnt, *m_ab;
  int64_t* comp_doff;
  uint8_t* act;
};

void carve2(Carver& c, int n, int l, Stage2Bufs& b) {
  const int lp = (l + 31) / 32 * 32;
  const size_t nn = size_t(n) * n;
  b.F = c.take<double>(n); b.XI = c.take<double>(n); b.NRM = c.take<double>(n);
  b.Sre = c.take<double>(size_t(n) * lp); b.Sim = c.take<double>(size_t(n) * lp);
  // per-component distance blocks: sum of squared component sizes <= n^2
  b.Dco = c.take<double>(nn); b.Dc = c.take<double>(nn);
  const size_t ntl = size_t((n + 63) / 64);
  b.fs = c.take<double>(n); b.lim = c.take<double>(ntl);
  b.ord = c.take<int>(n); b.g2l = c.take<int>(n);
  b.tiles = c.take<int>(3 * (ntl * (ntl + 1) / 2 + ntl)); b.ntiles = c.take<int>(1);
  b.kf = c.take<double>(n); b.kxi = c.take<double>(n); b.m_h = c.take<double>(n);
  b.parent = c.take<int>(n); b.comp_id = c.take<int>(n); b.comp_off = c.take<int>(n + 1);
  b.comp_size = c.take<int>(n); b.ctr = c.take<int>(n + 1); b.members = c.take<int>(n); b.key = c.take<int>(n); b.key2 = c.take<int>(n);
  b.csize = c.take<int>(n); b.chain = c.take<int>(n); b.par = c.take<int>(n); b.root = c.take<int>(n);
  b.rsize = c.take<int>(n); b.cid = c.take<int>(n); b.cl_root = c.take<int>(n); b.cl_off = c.take<int>(n + 1);
  b.cl_members = c.take<int>(n); b.kmed = c.take<int>(n); b.kfirst = c.take<int>(n); b.ksize = c.take<int>(n);
  b.krank = c.take<int>(n); b.m_cnt = c.take<int>(n); b.m_ab = c.take<int>(2 * size_t(n));
  b.comp_doff = c.take<int64_t>(n + 1);
  b.act = c.take<uint8_t>(n);
}
}  // namespace

size_t cluster_stage2_ws_bytes(int n, int l) {
  Carver c(nullptr);
  Stage2Bufs b;
  carve2(c, n < 1 ? 1 : n, l, b);
  return c.bytes();
}

ssi_status cluster_stage2_run(const TableSet& ts, const int32_t* pole_idx, const int32_t* retained, int n,
                              double cutoff, int min_size, int max_clusters, int32_t* labels, double* cl_f,
                              double* cl_xi, int32_t* cl_size, int32_t* cl_medoid, double* cl_shape,
                              int32_t* merges_ab, double* merges_h, ssi_cluster_info* info, void* ws,
                              cudaStream_t s) {
  const int l = ts.t[0].l;
  const int lp = (l + 31) / 32 * 32;
  Carver c(ws);
  Stage2Bufs b;
  carve2(c, n < 1 ? 1 : n, l, b);
  // stage-II counters of info are reset here; stage-I fields are kept
  info_reset2_kernel<<<1, 1, 0, s>>>(info);
  SSI_TRY(launch_check("info_reset2_kernel"));
  if (n == 0) return SSI_OK;
  gather_kernel<<<(n * 32 + kGathNT - 1) / kGathNT, kGathNT, 0, s>>>(ts, pole_idx, retained, n, lp, b.F, b.XI,
                                                                    b.Sre, b.Sim, b.NRM);
  SSI_TRY(launch_check("gather_kernel"));
  const int nt = (n + kDT - 1) / kDT;
  // components of {d <= cutoff}: only pairs inside the f band can be edges
  rank_f_kernel<<<(n + 255) / 256, 256, 0, s>>>(b.F, n, b.ord, b.fs);
  SSI_TRY(launch_check("rank_f_kernel"));
  band_lim_kernel<<<(nt + 127) / 128, 128, 0, s>>>(b.fs, n, cutoff, b.lim);
  SSI_TRY(launch_check("band_lim_kernel"));
  uf_init_kernel<<<(n + 255) / 256, 256, 0, s>>>(b.parent, n);
  SSI_TRY(launch_check("uf_init_kernel"));
  cudaFuncSetAttribute(band_link_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kDistSmem));
  band_link_kernel<<<dim3(nt, nt), kDistNT, kDistSmem, s>>>(b.F, b.XI, b.Sre, b.Sim, b.NRM, n, lp, b.ord, b.fs,
                                                             b.lim, cutoff, b.parent);
  SSI_TRY(launch_check("band_link_kernel"));
  uf_flatten_kernel<<<(n + 255) / 256, 256, 0, s>>>(b.parent, n);
  SSI_TRY(launch_check("uf_flatten_kernel"));
  components_kernel<<<1, kScanNT, 0, s>>>(b.parent, n, b.comp_id, b.comp_off, b.comp_size, b.comp_doff, b.ctr,
                                          b.members, b.key, info);
  SSI_TRY(launch_check("components_kernel"));
  local_index_kernel<<<(n + 255) / 256, 256, 0, s>>>(b.members, b.key, b.comp_off, n, b.g2l);
  SSI_TRY(launch_check("local_index_kernel"));
  // every component's dense distance block (original and chain copies)
  comp_tiles_kernel<<<1, 256, 0, s>>>(b.comp_size, info, b.tiles, b.ntiles);
  SSI_TRY(launch_check("comp_tiles_kernel"));
  const int grid = 148 * 4;
  cudaFuncSetAttribute(comp_dist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kDistSmem));
  comp_dist_kernel<<<grid, kDistNT, kDistSmem, s>>>(b.F, b.XI, b.Sre, b.Sim, b.NRM, lp, b.tiles, b.ntiles, b.comp_off,
                                                    b.comp_size, b.comp_doff, b.members, b.Dc, b.Dco);
  SSI_TRY(launch_check("comp_dist_kernel"));
  nnchain_kernel<<<grid, kChainNT, 0, s>>>(b.Dc, b.comp_off, b.comp_size, b.comp_doff, b.members, info, cutoff,
                                           b.csize, b.chain, b.par, b.act, b.m_ab, b.m_h, b.m_cnt);
  SSI_TRY(launch_check("nnchain_kernel"));
  roots_kernel<<<grid, 128, 0, s>>>(b.comp_off, b.comp_size, b.members, b.par, b.csize, info, b.root, b.rsize);
  SSI_TRY(launch_check("roots_kernel"));
  flat_kernel<<<1, kScanNT, 0, s>>>(b.root, b.rsize, n, min_size, b.cid, b.cl_root, b.cl_off, b.ctr, b.key2,
                                    b.cl_members, info);
  SSI_TRY(launch_check("flat_kernel"));
  summary_kernel<<<grid, 256, 0, s>>>(b.Dco, b.comp_doff, b.comp_size, b.key, b.g2l, b.F, b.XI, b.cl_off,
                                      b.cl_members, info, b.kf, b.kxi, b.kmed, b.kfirst, b.ksize);
  SSI_TRY(launch_check("summary_kernel"));
  order_kernel<<<1, 256, 0, s>>>(ts, pole_idx, retained, n, b.root, b.cid, b.kf, b.kxi, b.kmed, b.kfirst, b.ksize,
                                 b.krank, info, max_clusters, labels, cl_f, cl_xi, cl_size, cl_medoid, cl_shape);
  SSI_TRY(launch_check("order_kernel"));
  if (merges_ab || merges_h) {
    // merges of component c sit at its member offset; compact them in component order
    merges_kernel<<<1, 256, 0, s>>>(b.comp_off, b.m_cnt, b.m_ab, b.m_h, info, n, merges_ab, merges_h);
    SSI_TRY(launch_check("merges_kernel"));
  }
  return SSI_OK;
}

ssi_status track_run(const double* ref_f, const double* ref_shape, int n_ref, const double* f, const double* shape,
                     const int32_t* count, int n_sess, int max_modes, int l, double df_max, double macd_max,
                     int32_t* match, double* success, cudaStream_t s) {
  const size_t P = size_t(n_ref) * max_modes;
  const size_t smem = P * (sizeof(double) + 2 * sizeof(int));
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(track_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  track_kernel<<<n_sess, kTrackNT, smem, s>>>(ref_f, ref_shape, n_ref, f, shape, count, max_modes, l, df_max,
                                              macd_max, match);
  SSI_TRY(launch_check("track_kernel"));
  if (success) {
    success_kernel<<<(n_ref + 127) / 128, 128, 0, s>>>(match, n_sess, n_ref, success);
    SSI_TRY(launch_check("success_kernel"));
  }
  return SSI_OK;
}

}  // namespace ssi
