// Small dense FP64 kernels of the RSVD (A5, A8): Cholesky + triangular inverse for
// CholeskyQR2, and a one-sided Jacobi SVD for the k x k factor of B = Q^T T
// (Eq. 16). One CTA per problem; latency-bound by construction.
#include <cstdio>
#include <cstdlib>

#include "linalg.cuh"

namespace ssi {
namespace {

constexpr int kJacThreads = 512;
constexpr int JC = 8;                // Jacobi cluster size (CTAs); 16 (non-portable) for k > 256
constexpr int kJacMaxSweeps = 60;
#ifndef SSI_JAC_RING
#define SSI_JAC_RING 1   // 0: columns re-read from L2 every round, cluster barrier per round (A/B)
#endif


// Blocked variant (k <= 224): 32-wide block columns; the diagonal block is factored and
// inverted by one warp in registers (shuffles, no barriers), the panel below is L_IJ = A_IJ L_JJ^-T
// (one thread per row), the trailing lower triangle gets a rank-32 update in 4 x 4 register
// tiles; three barriers per block column instead of three per column. The inverse is then
// formed by block rows, X_IJ = -X_II sum_{K=J}^{I-1} L_IK X_KJ (one thread per column of X_IJ),
// (kp = k rounded up to 32; the padding is an identity block). The nb diagonal-block inverses are
// cached in the scratch X (nb CB x (CB + 1) blocks; for k > 224 the packed triangle follows them).
constexpr int CB = 32;
constexpr int kCholBlkMax = 224;    // packed triangle in shared memory
constexpr int kCholBlkGMax = 512;   // packed triangle in the L2-resident scratch
constexpr int kCholBlkThreads = 256;
constexpr unsigned FULLM = 0xffffffffu;

__device__ __forceinline__ int tri(int r) { return r * (r + 1) / 2; }

// One warp, register-resident right-looking Cholesky of the 32 x 32 diagonal block at (j0, j0)
// of the packed P (lane i holds row i; every index is a compile-time constant, so the row stays
// in registers): per column one shuffle of the pivot, an inline rsqrt, and the rank-1 update
// with the scaled column broadcast through a 2 x 32 shared-memory buffer `cb` (one store per
// lane, broadcast loads: a single warp issues a shuffle only every ~15 cycles, and the 496
// shuffled column entries made this 3x slower). The two halves of cb alternate by column, so a
// lane's store of column j + 2 cannot overtake another lane's loads of column j.
// Breakdown test: pivot j must exceed thr_j = tau * (diagonal of the Gram matrix at row j), lane j
// holding thr_j; a smaller pivot means column j is numerically in the span of the previous ones.
#ifndef SSI_CHOL32_SHFL
#define SSI_CHOL32_SHFL 0   // 1: the column broadcast by shuffles (round 1; A/B)
#endif
__device__ __noinline__ void chol32(double* P, int j0, int lane, double thr, int& bad, double* cb) {
  double* Li = P + tri(j0 + lane) + j0;
  double a[CB];
#pragma unroll
  for (int c = 0; c < CB; ++c) a[c] = (c <= lane) ? Li[c] : 0.0;
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    double d = __shfl_sync(FULLM, a[j], j);
    const double tj = __shfl_sync(FULLM, thr, j);
    if (!(d > tj) || !isfinite(d)) { bad = 1; d = 1.0; }
    const double r = fast_rsqrt(d);
    a[j] = (lane == j) ? d * r : a[j] * r;          // lanes < j hold 0 in a[j]
    double* col = cb + (j & 1) * CB;
    if (!SSI_CHOL32_SHFL) {
      col[lane] = a[j];
      __syncwarp();
    }
#pragma unroll
    for (int c = j + 1; c < CB; ++c) {
      const double lcj = SSI_CHOL32_SHFL ? __shfl_sync(FULLM, a[j], c) : col[c];
      if (lane >= c) a[c] = fma(-a[j], lcj, a[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < CB; ++c)
    if (c <= lane) Li[c] = a[c];
  __syncwarp();
}

// One warp: X = L^{-1} of the lower-triangular 32 x 32 block at (j0, j0) of P into Xd (ld CB + 1),
// lane c computing column c by forward substitution in registers (L entries are warp-wide
// broadcasts from shared memory; X[q][c] = 0 for q < c falls out of the recurrence).
__device__ __noinline__ void inv32(const double* P, int j0, double* Xd, int lane) {
  const double myr = fast_rcp(P[tri(j0 + lane) + j0 + lane]);
  double x[CB];
#pragma unroll
  for (int p = 0; p < CB; ++p) {
    const double* Lp = P + tri(j0 + p) + j0;
    double s0 = (lane == p) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int q = 0; q < p; ++q) {
      const double l = Lp[q];
      if ((q & 3) == 0) s0 = fma(-l, x[q], s0);
      else if ((q & 3) == 1) s1 = fma(-l, x[q], s1);
      else if ((q & 3) == 2) s2 = fma(-l, x[q], s2);
      else s3 = fma(-l, x[q], s3);
    }
    x[p] = ((s0 + s1) + (s2 + s3)) * __shfl_sync(FULLM, myr, p);
  }
#pragma unroll
  for (int p = 0; p < CB; ++p) Xd[p * (CB + 1) + lane] = x[p];
  __syncwarp();
}

// GLOBALP (kCholBlkMax < k <= kCholBlkGMax): the packed triangle (1.05 MB at k = 512) does not
// fit shared memory and lives in the L2-resident scratch instead (X + the diagonal-inverse
// cache); the algorithm is the same, and each thread forms up to two columns of a block row
// of the inverse (block rows are up to kp - 32 = 480 columns wide).
//
// Breakdown fallback (shifted CholeskyQR, Fukaya et al.'s shift): when a pivot fails the relative
// test of chol32 (tau = 64 k u of the row's Gram diagonal, i.e. Y is numerically rank-deficient or
// kappa(Y) >~ 1e6), the factorization restarts once on W + s I with s = 11 (m k + k (k + 1)) u tr(W),
// which always factors; *shifted_out = 1 then tells cholqr2 to run its extra (third) pass. A
// failure of the shifted attempt (non-finite input), or any shift in the final pass of a QR
// (final != 0), sets SSI_ERR_NUMERIC.
template <bool GLOBALP>
__global__ void __launch_bounds__(kCholBlkThreads, 1) chol_blk_kernel(const double* __restrict__ W, int k,
                                                                   int64_t m,
                                                                   double* __restrict__ L,
                                                                   double* __restrict__ Linv,
                                                                   double* __restrict__ LinvT,
                                                                   double* __restrict__ X,   // diagonal-inverse cache (+ packed triangle)
                                                                   int32_t* status, int profile,
                                                                   const int* run_if, int* shifted_out,
                                                                   int final) {
  if (!run_enabled(run_if)) return;
  long long tdiag = 0, tpanel = 0, ttrail = 0, tinv = 0, t0c = clock64(), tc;
  extern __shared__ __align__(16) double sm[];
  const int kp = (k + CB - 1) / CB * CB, nb = kp / CB;
  constexpr int NCOL = GLOBALP ? 2 : 1;        // inverse columns per thread
  // packed lower triangle, tri(kp) doubles; the diagonal-inverse cache follows it when global
  double* P = GLOBALP ? X + size_t(nb) * CB * (CB + 1) : sm;
  double* Xd = GLOBALP ? sm : sm + tri(kp);    // CB x (CB + 1): inverse of the current diagonal block
  double* Z = GLOBALP ? P + tri(kp) : nullptr; // CB x kp staging of a block row of the inverse
  // global variant: shared-memory copies of what the inner loops re-read — the panel below the
  // diagonal block (CB columns of up to kp - CB rows, column-major, so a 4 x 4 tile reads its
  // rows with 16-byte loads) for the trailing update, and the block row L_I* (CB x i0) for the
  // inverse; both fit in (kp - CB) (CB + 1) doubles
  double* Ps = GLOBALP ? sm + CB * (CB + 1) : nullptr;
  __shared__ int fail;
  __shared__ double shift;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const double tau = 64.0 * double(k) * 1.1102230246251565e-16;
  int attempt = 0;
  for (;; ++attempt) {
  const double sh = attempt ? shift : 0.0;
  if (tid == 0) fail = 0;
  for (int i = warp; i < kp; i += nw)
    for (int c = lane; c <= i; c += 32)
      P[tri(i) + c] = (i < k) ? W[i + int64_t(c) * k] + (i == c ? sh : 0.0) : (i == c ? 1.0 : 0.0);
  __syncthreads();
  // ---------------- factorization
  for (int J = 0; J < nb; ++J) {
    const int j0 = J * CB;
    if (warp == 0) {
      int bad = 0;
      const int r = j0 + lane;
      chol32(P, j0, lane, tau * (r < k ? W[r + int64_t(r) * k] + sh : 1.0), bad, Xd);   // Xd: column buffer
      if (bad && lane == 0) fail = 1;
      inv32(P, j0, Xd, lane);
      // keep L_JJ^{-1} for the inverse phase (L2-resident scratch; saves recomputing it)
      for (int e = lane; e < CB * (CB + 1); e += 32) X[J * CB * (CB + 1) + e] = Xd[e];
    }
    __syncthreads();
    tc = clock64(); tdiag += tc - t0c; t0c = tc;
    // panel: L[r][j0 + c] = sum_{p <= c} A[r][j0 + p] X_JJ[c][p]
    for (int r = j0 + CB + tid; r < kp; r += nt) {
      double* rowp = P + tri(r) + j0;
      double av[CB];
#pragma unroll
      for (int p = 0; p < CB; ++p) av[p] = rowp[p];
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int p = 0; p <= c; ++p) acc = fma(av[p], Xd[c * (CB + 1) + p], acc);
        rowp[c] = acc;
        if (GLOBALP) Ps[c * (kp - CB) + (r - j0 - CB)] = acc;   // column-major panel
      }
    }
    __syncthreads();
    tc = clock64(); tpanel += tc - t0c; t0c = tc;
    // trailing rank-32 update of the lower triangle, 4 x 4 tiles
    const int n4 = (kp - j0 - CB) / 4;
    const int ntile = n4 * (n4 + 1) / 2;
    for (int t = tid; t < ntile; t += nt) {
      int ti = int((sqrtf(8.0f * float(t) + 1.0f) - 1.0f) * 0.5f);
      while (tri(ti + 1) <= t) ++ti;
      while (tri(ti) > t) --ti;
      const int tj = t - tri(ti);
      const int r0 = j0 + CB + 4 * ti, c0 = j0 + CB + 4 * tj;
      const double* lr[4];
      const double* lc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { lr[u] = P + tri(r0 + u) + j0; lc[u] = P + tri(c0 + u) + j0; }
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
#pragma unroll 4
      for (int p = 0; p < CB; ++p) {
        double xr[4], xc[4];
        if (GLOBALP) {   // column-major panel: the tile's 4 rows are two 16-byte loads
          const double2* pr = reinterpret_cast<const double2*>(Ps + p * (kp - CB) + (r0 - j0 - CB));
          const double2* pc = reinterpret_cast<const double2*>(Ps + p * (kp - CB) + (c0 - j0 - CB));
          const double2 r01 = pr[0], r23 = pr[1], c01 = pc[0], c23 = pc[1];
          xr[0] = r01.x; xr[1] = r01.y; xr[2] = r23.x; xr[3] = r23.y;
          xc[0] = c01.x; xc[1] = c01.y; xc[2] = c23.x; xc[3] = c23.y;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) { xr[u] = lr[u][p]; xc[u] = lc[u][p]; }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(xr[u], xc[v], acc[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (c0 + v <= r0 + u) P[tri(r0 + u) + c0 + v] -= acc[u][v];
    }
    __syncthreads();
    tc = clock64(); ttrail += tc - t0c; t0c = tc;
  }
  if (!fail || attempt == 1) break;               // fail is read after the loop's last barrier
  if (warp == 0) {                                // s = 11 (m k + k (k + 1)) u tr(W)
    double t = 0.0;
    for (int c = lane; c < k; c += 32) t += W[c + int64_t(c) * k];
    t = warp_sum(t);
    if (lane == 0) shift = 11.0 * (double(m) * k + double(k) * (k + 1)) * 1.1102230246251565e-16 * t;
  }
  __syncthreads();
  }
  if (tid == 0) {
    if (shifted_out) *shifted_out = attempt;
    if (fail || (final && attempt)) set_status(status, SSI_ERR_NUMERIC);
  }
  // L out (col-major k x k, zeros above the diagonal) before P is overwritten by the inverse
  for (int64_t e = tid; e < int64_t(k) * k; e += nt) {
    const int r = int(e % k), c = int(e / k);
    L[e] = (c <= r) ? P[tri(r) + c] : 0.0;
  }
  // ---------------- inverse in place, by block rows: X_IJ = -X_II sum_{K=J}^{I-1} L_IK X_KJ
  // (rows above i0 of P already hold X; all T of a block row are formed before any write)
  for (int I = 0; I < nb; ++I) {
    const int i0 = I * CB;
    if (warp == 0)
      for (int e = lane; e < CB * (CB + 1); e += 32) Xd[e] = X[I * CB * (CB + 1) + e];
    const int ntask = I * CB;
    if (GLOBALP) {
      for (int e = tid; e < CB * i0; e += nt) {            // L_I* -> shared (row-major CB x i0)
        const int i = e / i0, q = e - i * i0;
        Ps[e] = P[tri(i0 + i) + q];
      }
      __syncthreads();                                     // Xd and L_I* ready
    }
#pragma unroll 1
    for (int u = 0; u < NCOL; ++u) {
      const int col = tid + u * nt;                        // columns tid, tid + nt of X_I*
      double T[CB];
#pragma unroll
      for (int i = 0; i < CB; ++i) T[i] = 0.0;
      if (col < ntask) {
        // q runs warp-uniformly from the warp's first column, so the L_I* entries are
        // broadcasts; X[q][col] = 0 for q < col (masked: the packed row q ends at column q)
#pragma unroll (GLOBALP ? 4 : 1)
        for (int q = col & ~31; q < i0; ++q) {
          const double xq = (q >= col) ? P[tri(q) + col] : 0.0;
#pragma unroll
          for (int i = 0; i < CB; ++i) T[i] = fma(GLOBALP ? Ps[i * i0 + q] : P[tri(i0 + i) + q], xq, T[i]);
        }
      }
      if (!GLOBALP) __syncthreads();                       // Xd ready, every L_I* read
      if (col < ntask) {
#pragma unroll
        for (int i = 0; i < CB; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int p = 0; p <= i; ++p) acc = fma(Xd[i * (CB + 1) + p], T[p], acc);
          // global variant: staged in Z (other threads still read L_I*), copied after the barrier
          if (GLOBALP) Z[i * int64_t(kp) + col] = -acc;
          else P[tri(i0 + i) + col] = -acc;
        }
      }
    }
    if (GLOBALP) {
      __syncthreads();                                     // every L_I* read
      for (int e = tid; e < CB * ntask; e += nt) {
        const int i = e / ntask, col = e - i * ntask;
        P[tri(i0 + i) + col] = Z[i * int64_t(kp) + col];
      }
    }
    if (warp == 0) {
#pragma unroll 4
      for (int r = 0; r < CB; ++r)
        if (lane <= r) P[tri(i0 + r) + i0 + lane] = Xd[r * (CB + 1) + lane];
    }
    __syncthreads();
  }
  tc = clock64(); tinv += tc - t0c; t0c = tc;
  if (profile && tid == 0) printf("chol_blk k=%d: diag %lld panel %lld trail %lld inv %lld cycles\n", k, tdiag, tpanel, ttrail, tinv);
  // ---------------- inverse out (col-major k x k)
  for (int64_t e = tid; e < int64_t(k) * k; e += nt) {
    const int r = int(e % k), c = int(e / k);
    Linv[e] = (c <= r) ? P[tri(r) + c] : 0.0;
    if (LinvT) LinvT[e] = (r <= c) ? P[tri(c) + r] : 0.0;
  }
}

// One-sided (Hestenes) Jacobi with the round-robin (circle) ordering; warp per column
// pair. Round r pairs positions (i, n-1-i); position 0 holds column 0, position p >= 1
// holds column 1 + (p - 1 + r) mod (n - 1). Column norms are updated with Rutishauser's
// formulas (|p'|^2 = a - t g, |q'|^2 = b + t g), so a pair costs one dot product; norms are
// recomputed exactly at the start of every sweep.
// The k x k matrix (387 KB at k = 220) does not fit one SM, and one SM's L2 bandwidth bounds a
// round (every column is read and written once per round), so the pairs of a round are spread
// over a cluster of JC CTAs that meet at a cluster barrier after every round; G and the norms
// live in L2 (ld/st.global.cg, coherent across the cluster's SMs).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int KPL, int JCT>   // column elements per lane (k <= 32 * KPL), cluster size
__global__ void __launch_bounds__(kJacThreads, 1) jacobi_kernel(double* __restrict__ G, int k,
                                                             double* __restrict__ Ut,
                                                             double* __restrict__ S,
                                                             double* __restrict__ gnrm,   // k
                                                             int* __restrict__ gflag,     // kJacMaxSweeps
                                                             int32_t* status, int profile) {
  extern __shared__ __align__(16) double jsm[];
  double* nrm = jsm;                                    // k (final phase, CTA 0)
  int* rank = reinterpret_cast<int*>(jsm + k);          // k
  __shared__ int rot;
  const int n = (k + 1) & ~1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int cr = int(cluster_rank());
  const int gw = cr * nw + warp, gnw = JCT * nw;         // warp index / count over the cluster
  const double tol = sqrt(double(k)) * 1.1102230246251565e-16;
  if (cr == 0)
    for (int i = tid; i < kJacMaxSweeps; i += blockDim.x) gflag[i] = 0;
  bool converged = false;
  int sweeps = 0;
  const long long c0 = clock64();
  for (int sweep = 0; sweep < kJacMaxSweeps && !converged; ++sweep) {
    ++sweeps;
    for (int j = gw; j < k; j += gnw) {
      double a = 0.0;
      for (int r = lane; r < k; r += 32) { const double x = __ldcg(G + int64_t(j) * k + r); a += x * x; }
      a = warp_sum(a);
      if (lane == 0) __stcg(gnrm + j, a);
    }
    if (tid == 0) rot = 0;
    cluster_sync_all();
    for (int round = 0; round < n - 1; ++round) {
      for (int pr = gw; pr < n / 2; pr += gnw) {
        const int pa = pr, pb = n - 1 - pr;
        int p = pa == 0 ? 0 : 1 + (pa - 1 + round) % (n - 1);
        int q = 1 + (pb - 1 + round) % (n - 1);
        if (p >= k || q >= k) continue;
        if (p > q) { const int t = p; p = q; q = t; }
        double* gp = G + int64_t(p) * k;
        double* gq = G + int64_t(q) * k;
        double x[KPL], y[KPL];
#pragma unroll
        for (int u = 0; u < KPL; ++u) {
          const int r = lane + 32 * u;
          x[u] = r < k ? __ldcg(gp + r) : 0.0;
          y[u] = r < k ? __ldcg(gq + r) : 0.0;
        }
        const double al = __ldcg(gnrm + p), be = __ldcg(gnrm + q);
        double ga = 0.0;
#pragma unroll
        for (int u = 0; u < KPL; ++u) ga += x[u] * y[u];
        ga = warp_sum(ga);
        if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
#pragma unroll
          for (int u = 0; u < KPL; ++u) {
            const int r = lane + 32 * u;
            if (r < k) {
              __stcg(gp + r, c * x[u] - sn * y[u]);
              __stcg(gq + r, sn * x[u] + c * y[u]);
            }
          }
          if (lane == 0) {
            __stcg(gnrm + p, al - t * ga);
            __stcg(gnrm + q, be + t * ga);
            rot = 1;
          }
        }
      }
      cluster_sync_all();
    }
    __syncthreads();
    if (tid == 0 && rot) atomicAdd(gflag + sweep, 1);
    cluster_sync_all();
    converged = (__ldcg(gflag + sweep) == 0);
  }
  if (cr != 0) return;
  if (!converged && tid == 0) set_status(status, SSI_ERR_NUMERIC);
  if (profile && tid == 0) printf("jacobi k=%d: %d sweeps, %lld cycles\n", k, sweeps, clock64() - c0);
  // singular values = column norms; sort descending (rank by counting, ties by index)
  for (int j = warp; j < k; j += nw) {
    double a = 0.0;
    for (int r = lane; r < k; r += 32) { const double x = __ldcg(G + int64_t(j) * k + r); a += x * x; }
    a = warp_sum(a);
    if (lane == 0) nrm[j] = sqrt(a);
  }
  __syncthreads();
  for (int j = tid; j < k; j += blockDim.x) {
    int rk = 0;
    const double v = nrm[j];
    for (int i = 0; i < k; ++i) rk += (nrm[i] > v) || (nrm[i] == v && i < j);
    rank[j] = rk;
    S[rk] = v;
  }
  __syncthreads();
  for (int j = warp; j < k; j += nw) {
    const double inv = nrm[j] > 0.0 ? 1.0 / nrm[j] : 0.0;
    const int dst = rank[j];
    for (int r = lane; r < k; r += 32) Ut[int64_t(dst) * k + r] = __ldcg(G + int64_t(j) * k + r) * inv;
  }
}

// Ring variant of jacobi_kernel (k <= 256): the same pairs, rounds, rotation formulas and
// convergence test — bit-identical results — but the columns stay in the registers of the warp
// that owns their pair: warp g owns positions g (top) and n-1-g (bottom) of the round-robin
// ordering, and between rounds the positions shift by one (new[p] = old[p+1] for p in [1, n-2],
// new[n-1] = old[1], position 0 fixed), so every warp sends its top column to warp g-1 (warp 1:
// to warp 0's bottom) and its bottom column to warp g+1 (the middle warp: to its own top)
// through a double-buffered mailbox in the receiving CTA's shared memory (DSMEM stores and a
// remote mbarrier arrive with release semantics at cluster scope). A round costs one dot
// product, the rotation and two 32-lane DSMEM hand-offs instead of two L2 column reads, two
// writes and a cluster barrier (k = 220: 10.5M -> 7.7M cycles; st.async with complete_tx per
// 16-byte piece measured 16.8M, one release-arrive per warp after a warp sync 12.8M). A mailbox buffer is rewritten only after its reader has
// consumed it: the writer of round t has received the reader's own round t-1 output (the two
// neighbours exchange in both directions). Column norms travel with their columns.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t map_rank(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster2(uint32_t a, double v0, double v1) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v0), "d"(v1) : "memory");
}
__device__ __forceinline__ void st_cluster1(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t a) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
// st.async: store to a CTA of the cluster and signal its mbarrier with the bytes (complete_tx)
__device__ __forceinline__ void st_async2(uint32_t a, double v0, double v1, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               ::"r"(a), "d"(v0), "d"(v1), "r"(bar) : "memory");
}
__device__ __forceinline__ void st_async1(uint32_t a, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
               ::"r"(a), "d"(v), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
#ifndef SSI_JAC_STASYNC
#define SSI_JAC_STASYNC 0
#endif
__device__ __forceinline__ void mbar_wait_cluster(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a), "r"(parity) : "memory");
}

template <int KPL, int JCT>
__global__ void __launch_bounds__(kJacThreads, 1) jacobi_ring_kernel(double* __restrict__ G, int k,
                                                                  double* __restrict__ Ut,
                                                                  double* __restrict__ S,
                                                                  int* __restrict__ gflag,
                                                                  int32_t* status, int profile) {
  constexpr int NWC = kJacThreads / 32;             // warps per CTA
  constexpr int MB = KPL * 32 + 2;                   // mailbox: column + norm (+ pad to 16 bytes)
  static_assert(KPL % 2 == 0, "16-byte pairs");
  extern __shared__ __align__(16) double jsm[];      // [NWC][2 slots][2 buffers][MB]
  __shared__ __align__(8) uint64_t mbar[NWC][2][2];
  __shared__ int rot;
  const int n = (k + 1) & ~1, np = n / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cr = int(cluster_rank());
  const int g = cr * NWC + warp;                     // pair index
  const bool active = g < np;
  const double tol = sqrt(double(k)) * 1.1102230246251565e-16;
  if (tid == 0) {
    for (int w = 0; w < NWC; ++w)
      for (int sl = 0; sl < 2; ++sl)
        for (int b = 0; b < 2; ++b)
          asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&mbar[w][sl][b])), "r"(SSI_JAC_STASYNC ? 1 : 32) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (cr == 0)
    for (int i = tid; i < kJacMaxSweeps; i += blockDim.x) gflag[i] = 0;
  cluster_sync_all();
  // destinations of this warp's top / bottom column (pair index, slot 0 = top, 1 = bottom)
  // and the sources of its own new columns
  const int top_dst = g >= 2 ? g - 1 : (g == 1 ? 0 : -1), top_slot = g >= 2 ? 0 : 1;
  const int bot_dst = g <= np - 2 ? g + 1 : -1;      // -1: the middle warp keeps it as its top
  const bool top_in = g >= 1 && g <= np - 2;         // new top arrives in slot 0
  const bool bot_in = (g >= 1) || (g == 0 && np >= 2);   // new bottom arrives in slot 1
  auto mbox = [&](int pair, int slot, int buf) -> double* {
    return jsm + ((size_t(pair % NWC) * 2 + slot) * 2 + buf) * MB;
  };
  double x[KPL], y[KPL];                             // top / bottom column
  double nx = 0.0, ny = 0.0;
  const int ct0 = g, cb0 = n - 1 - g;                // columns at round 0
  if (active) {
#pragma unroll
    for (int u = 0; u < KPL; ++u) {
      const int r = lane + 32 * u;
      x[u] = (r < k && ct0 < k) ? __ldcg(G + int64_t(ct0) * k + r) : 0.0;
      y[u] = (r < k && cb0 < k) ? __ldcg(G + int64_t(cb0) * k + r) : 0.0;
    }
  }
  bool converged = false;
  int sweeps = 0;
  long long t = 0;                                   // global round counter (mailbox phases)
  const long long c0 = clock64();
  for (int sweep = 0; sweep < kJacMaxSweeps && !converged; ++sweep) {
    ++sweeps;
    if (tid == 0) rot = 0;
    int myrot = 0;
    if (active) {                                    // exact norms at the start of every sweep
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int u = 0; u < KPL; ++u) {
        const int r = lane + 32 * u;
        if (r < k) { a += x[u] * x[u]; b += y[u] * y[u]; }
      }
      nx = warp_sum(a);
      ny = warp_sum(b);
    }
    for (int round = 0; round < n - 1; ++round, ++t) {
      if (!active) continue;
      const int ct = g == 0 ? 0 : 1 + (g - 1 + round) % (n - 1);
      const int cb = 1 + (n - 2 - g + round) % (n - 1);
      if (np >= 2 && ct < k && cb < k) {
        const bool sw = ct > cb;                     // x must hold column p = min(ct, cb)
        if (sw) {
#pragma unroll
          for (int u = 0; u < KPL; ++u) { const double tmp = x[u]; x[u] = y[u]; y[u] = tmp; }
        }
        const double al = sw ? ny : nx, be = sw ? nx : ny;
        double ga = 0.0;
#pragma unroll
        for (int u = 0; u < KPL; ++u) ga += x[u] * y[u];
        ga = warp_sum(ga);
        double na = al, nb = be;
        if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + tt * tt), sn = c * tt;
#pragma unroll
          for (int u = 0; u < KPL; ++u) {
            const int r = lane + 32 * u;
            if (r < k) {
              const double xp = c * x[u] - sn * y[u], yq = sn * x[u] + c * y[u];
              x[u] = xp;
              y[u] = yq;
            }
          }
          na = al - tt * ga;
          nb = be + tt * ga;
          myrot = 1;
        }
        if (sw) {
#pragma unroll
          for (int u = 0; u < KPL; ++u) { const double tmp = x[u]; x[u] = y[u]; y[u] = tmp; }
          nx = nb; ny = na;
        } else {
          nx = na; ny = nb;
        }
      }
      if (np < 2) continue;
      // hand-off for round t + 1 (buffer (t + 1) & 1)
      const int buf = int((t + 1) & 1);
      // mailbox layout: pair j = (x[2j], x[2j+1]) of lane L at 16-byte slot j * 32 + L (a warp's
      // store covers 512 contiguous bytes; lane-major 64-byte runs measured 1.7x slower), norm last
      if (top_dst >= 0) {
        const uint32_t rk = uint32_t(top_dst / NWC);
        const uint32_t dst = map_rank(smem_addr(mbox(top_dst, top_slot, buf)), rk);
        const uint32_t bar = map_rank(smem_addr(&mbar[top_dst % NWC][top_slot][buf]), rk);
        if (SSI_JAC_STASYNC) {
#pragma unroll
          for (int u = 0; u < KPL; u += 2) st_async2(dst + 16u * ((u / 2) * 32 + lane), x[u], x[u + 1], bar);
          if (lane == 0) st_async1(dst + 8u * (KPL * 32), nx, bar);
        } else {
#pragma unroll
          for (int u = 0; u < KPL; u += 2) st_cluster2(dst + 16u * ((u / 2) * 32 + lane), x[u], x[u + 1]);
          if (lane == 0) st_cluster1(dst + 8u * (KPL * 32), nx);
          mbar_arrive_cluster(bar);                    // every lane releases its own stores (count 32;
        }                                            // one lane's release after a warp sync measured slower)
      }
      if (bot_dst >= 0) {
        const uint32_t rk = uint32_t(bot_dst / NWC);
        const uint32_t dst = map_rank(smem_addr(mbox(bot_dst, 1, buf)), rk);
        const uint32_t bar = map_rank(smem_addr(&mbar[bot_dst % NWC][1][buf]), rk);
        if (SSI_JAC_STASYNC) {
#pragma unroll
          for (int u = 0; u < KPL; u += 2) st_async2(dst + 16u * ((u / 2) * 32 + lane), y[u], y[u + 1], bar);
          if (lane == 0) st_async1(dst + 8u * (KPL * 32), ny, bar);
        } else {
#pragma unroll
          for (int u = 0; u < KPL; u += 2) st_cluster2(dst + 16u * ((u / 2) * 32 + lane), y[u], y[u + 1]);
          if (lane == 0) st_cluster1(dst + 8u * (KPL * 32), ny);
          mbar_arrive_cluster(bar);
        }
      } else {                                       // middle warp: bottom becomes its top
#pragma unroll
        for (int u = 0; u < KPL; ++u) x[u] = y[u];
        nx = ny;
      }
      const uint32_t ph = uint32_t((t >> 1) & 1);       // use (t >> 1) of buffer (t + 1) & 1
      if (top_in) {
        const uint32_t bar = smem_addr(&mbar[warp][0][buf]);
        if (SSI_JAC_STASYNC && lane == 0) mbar_expect_tx(bar, (KPL * 32 + 1) * 8);
        mbar_wait_cluster(bar, ph);
        const double2* src = reinterpret_cast<const double2*>(mbox(g, 0, buf)) + lane;
#pragma unroll
        for (int u = 0; u < KPL; u += 2) { const double2 v = src[(u / 2) * 32]; x[u] = v.x; x[u + 1] = v.y; }
        nx = mbox(g, 0, buf)[KPL * 32];
      }
      if (bot_in) {
        const uint32_t bar = smem_addr(&mbar[warp][1][buf]);
        if (SSI_JAC_STASYNC && lane == 0) mbar_expect_tx(bar, (KPL * 32 + 1) * 8);
        mbar_wait_cluster(bar, ph);
        const double2* src = reinterpret_cast<const double2*>(mbox(g, 1, buf)) + lane;
#pragma unroll
        for (int u = 0; u < KPL; u += 2) { const double2 v = src[(u / 2) * 32]; y[u] = v.x; y[u + 1] = v.y; }
        ny = mbox(g, 1, buf)[KPL * 32];
      }
    }
    if (myrot && lane == 0) rot = 1;
    __syncthreads();
    if (tid == 0 && rot) atomicAdd(gflag + sweep, 1);
    cluster_sync_all();
    converged = (__ldcg(gflag + sweep) == 0);
  }
  // the columns are back at their round-0 positions: write them out for the final phase
  if (active) {
#pragma unroll
    for (int u = 0; u < KPL; ++u) {
      const int r = lane + 32 * u;
      if (r < k) {
        if (ct0 < k) __stcg(G + int64_t(ct0) * k + r, x[u]);
        if (cb0 < k) __stcg(G + int64_t(cb0) * k + r, y[u]);
      }
    }
  }
  cluster_sync_all();
  if (cr != 0) return;
  if (!converged && tid == 0) set_status(status, SSI_ERR_NUMERIC);
  if (profile && tid == 0) printf("jacobi(ring) k=%d: %d sweeps, %lld cycles\n", k, sweeps, clock64() - c0);
  double* nrm = jsm;                                 // the mailboxes are no longer used
  int* rank = reinterpret_cast<int*>(jsm + k);
  const int nw = blockDim.x >> 5;
  for (int j = warp; j < k; j += nw) {
    double a = 0.0;
    for (int r = lane; r < k; r += 32) { const double v = __ldcg(G + int64_t(j) * k + r); a += v * v; }
    a = warp_sum(a);
    if (lane == 0) nrm[j] = sqrt(a);
  }
  __syncthreads();
  for (int j = tid; j < k; j += blockDim.x) {
    int rk = 0;
    const double v = nrm[j];
    for (int i = 0; i < k; ++i) rk += (nrm[i] > v) || (nrm[i] == v && i < j);
    rank[j] = rk;
    S[rk] = v;
  }
  __syncthreads();
  for (int j = warp; j < k; j += nw) {
    const double inv = nrm[j] > 0.0 ? 1.0 / nrm[j] : 0.0;
    const int dst = rank[j];
    for (int r = lane; r < k; r += 32) Ut[int64_t(dst) * k + r] = __ldcg(G + int64_t(j) * k + r) * inv;
  }
}

}  // namespace

size_t cholqr_partial_elems(int64_t m, int k) {
  return gemm_partial_elems(k, k, gemm_pick_splits(k, k, m));
}

void cholqr_carve(Carver& c, int64_t m, int k, CholQRWork& w) {
  if (k > kSvdMaxK) {   // blocked whole-GPU path (linalg_big.cu): no explicit inverses
    w.W = c.take<double>(size_t(k) * k);
    w.W0 = c.take<double>(size_t(k) * k);
    w.L1 = c.take<double>(size_t(k) * k);
    w.L2 = c.take<double>(size_t(k) * k);
    w.Lb = c.take<double>(size_t(k) * k);
    w.La = c.take<double>(size_t(k) * k);
    w.Linv1 = w.Linv2 = w.LinvT1 = w.LinvT2 = w.Linvb = w.LinvTb = nullptr;
    w.flag = c.take<int>(1 + kCqExtraPasses);
    w.Q1 = c.take<double>(size_t(m) * k);
    w.chol_g = nullptr;
    w.partial = c.take<double>(cholqr_partial_elems(m, k) + 1);
    w.tallp = nullptr;
    w.Dp1 = c.take<double>(cholqr_big_panel_elems(k));
    w.Dp2 = c.take<double>(cholqr_big_panel_elems(k));
    return;
  }
  w.Dp1 = w.Dp2 = nullptr;
  w.W0 = w.La = nullptr;
  w.W = c.take<double>(size_t(k) * k);
  w.L1 = c.take<double>(size_t(k) * k);
  w.Linv1 = c.take<double>(size_t(k) * k);
  w.L2 = c.take<double>(size_t(k) * k);
  w.Linv2 = c.take<double>(size_t(k) * k);
  w.LinvT1 = c.take<double>(size_t(k) * k);
  w.LinvT2 = c.take<double>(size_t(k) * k);
  w.Lb = c.take<double>(size_t(k) * k);
  w.Linvb = c.take<double>(size_t(k) * k);
  w.LinvTb = c.take<double>(size_t(k) * k);
  w.flag = c.take<int>(1);
  w.Q1 = c.take<double>(size_t(m) * k);
  const size_t kp = size_t(k + 31) / 32 * 32;
  const size_t nbk = kp / 32;
  // k <= kCholBlkMax: chol_blk_kernel<false> keeps the packed triangle in shared memory and
  // caches the nb diagonal-block inverses (CB x (CB + 1) each) here
  w.chol_g = c.take<double>(k <= kCholBlkMax ? nbk * 32 * 33
                            : k <= kCholBlkGMax ? nbk * 32 * 33 + kp * (kp + 1) / 2 + 32 * kp
                                                : size_t(k) * (k + 1) / 2);
  w.partial = c.take<double>(cholqr_partial_elems(m, k) + 1);
  // gemm_tall uses s <= min(64, K/64) splits: upper bounds, non-decreasing in m
  const size_t s2 = size_t(k / 64 > 1 ? (k / 64 < 64 ? k / 64 : 64) : 1);
  const size_t t1 = size_t(64) * k * k, t2 = s2 > 1 ? s2 * size_t(m) * k : 0;
  w.tallp = c.take<double>((t1 > t2 ? t1 : t2) + 1);
}

ssi_status chol_inv(const double* W, int k, int64_t m, double* L, double* Linv, double* LinvT, double* gscratch,
                    int32_t* status, cudaStream_t s, const int* run_if, int* shifted_out, int final) {
  static const int profile = getenv("SSI_CHOL_PROFILE") ? 1 : 0;
  const int kp = (k + CB - 1) / CB * CB;
  if (k <= kCholBlkMax) {
    const size_t smem = (size_t(kp) * (kp + 1) / 2 + size_t(CB) * (CB + 1)) * sizeof(double);
    cudaFuncSetAttribute(chol_blk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    chol_blk_kernel<false><<<1, kCholBlkThreads, smem, s>>>(W, k, m, L, Linv, LinvT, gscratch, status, profile,
                                                           run_if, shifted_out, final);
    return launch_check("chol_blk_kernel");
  }
  if (k <= kCholBlkGMax) {
    const size_t smem = (size_t(CB) * (CB + 1) + size_t(kp - CB) * (CB + 1)) * sizeof(double);
    cudaFuncSetAttribute(chol_blk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    chol_blk_kernel<true><<<1, kCholBlkThreads, smem, s>>>(W, k, m, L, Linv, LinvT, gscratch, status, profile,
                                                          run_if, shifted_out, final);
    return launch_check("chol_blk_kernel");
  }
  set_last_error("chol_inv: k = %d > %d unsupported", k, kCholBlkGMax);
  return SSI_ERR_INVALID_ARG;
}

namespace {
// Q1 <- Q (m x k, both ld m) when *run_if (the extra pass of the breakdown fallback wrote Q).
__global__ void cq_copy_kernel(const int* run_if, int64_t n, const double* __restrict__ src, double* __restrict__ dst) {
  if (!run_enabled(run_if)) return;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    dst[e] = src[e];
}

// After a fallback QR, Y = Q L2^T Lb^T L1^T: fold the extra pass's factor into the second one so
// R^T = L1 L2 and R^{-1} = Linv1^T Linv2^T keep holding for the callers:
//   L2 <- Lb L2 (CTA c < k: column c, which only reads column c of L2), and
//   Linv2 <- Linv2 Linvb (CTA k + r: row r, which only reads row r of Linv2);
// each CTA forms its whole column / row before writing it back, so the update is in place.
__global__ void cq_fold_kernel(const int* run_if, int k, const double* __restrict__ Lb,
                               const double* __restrict__ Linvb, double* L2, double* Linv2) {
  if (!run_enabled(run_if)) return;
  extern __shared__ double v[];
  const int b = blockIdx.x;
  if (b < k) {
    const int c = b;
    for (int r = threadIdx.x; r < k; r += blockDim.x) {
      double a = 0.0;
      for (int p = c; p <= r; ++p) a = fma(Lb[r + int64_t(p) * k], L2[p + int64_t(c) * k], a);
      v[r] = a;
    }
    __syncthreads();
    for (int r = c + threadIdx.x; r < k; r += blockDim.x) L2[r + int64_t(c) * k] = v[r];
  } else {
    const int r = b - k;
    for (int c = threadIdx.x; c <= r; c += blockDim.x) {
      double a = 0.0;
      for (int p = c; p <= r; ++p) a = fma(Linv2[r + int64_t(p) * k], Linvb[p + int64_t(c) * k], a);
      v[c] = a;
    }
    __syncthreads();
    for (int c = threadIdx.x; c <= r; c += blockDim.x) Linv2[r + int64_t(c) * k] = v[c];
  }
}
}  // namespace

// CholeskyQR2 with the shifted-CholeskyQR3 fallback: pass 1 (shift on breakdown) -> [extra pass,
// launched always, run only when pass 1 shifted] -> pass 2. The conditional launches read a
// device flag, so a healthy QR costs no host synchronisation and no arithmetic for the fallback.
ssi_status cholqr2(const double* Y, int64_t ldy, int64_t m, int k, double* Q, CholQRWork& w,
                   int32_t* status, cudaStream_t s) {
  if (k > kSvdMaxK) return cholqr2_big(Y, ldy, m, k, Q, w, status, s);
  // tall-skinny DMMA kernels (cp.async 16-byte pieces) when the shapes and alignment allow
  const bool tall = k <= kTallMaxN && ldy % 2 == 0 && m % 2 == 0 && k % 2 == 0 &&
                    (reinterpret_cast<uintptr_t>(Y) & 15) == 0 && (reinterpret_cast<uintptr_t>(Q) & 15) == 0;
  const int splits = gemm_pick_splits(k, k, m);
  auto gram = [&](const double* X, int64_t ldx, const int* run_if) -> ssi_status {   // W = X^T X (lower)
    if (tall) return gemm_tall_syrk_lower(k, m, X, ldx, X, ldx, w.W, k, w.tallp, s, run_if);
    return gemm_f64(k, k, m, 1.0, Operand{X, ldx, 1}, Operand{X, 1, ldx}, w.W, k, splits, w.partial, s, run_if);
  };
  auto trmul = [&](const double* X, int64_t ldx, const double* Linv, const double* LinvT, double* out,
                   const int* run_if) {
    // out = X Linv^T  (B(kk, j) = Linv(j, kk) = LinvT[kk + j k])
    if (tall) return gemm_tall_triu(m, k, k, X, ldx, LinvT, k, out, m, s, run_if);
    return gemm_f64(m, k, k, 1.0, Operand{X, 1, ldx}, Operand{Linv, k, 1}, out, m, 1, nullptr, s, run_if);
  };
  const int* shifted = w.flag;
  SSI_TRY(gram(Y, ldy, nullptr));
  SSI_TRY(chol_inv(w.W, k, m, w.L1, w.Linv1, w.LinvT1, w.chol_g, status, s, nullptr, w.flag, 0));
  SSI_TRY(trmul(Y, ldy, w.Linv1, w.LinvT1, w.Q1, nullptr));
#ifndef SSI_NO_CQ_FALLBACK
  // fallback pass: Q1 = Q_b Lb^T (CholeskyQR of the shifted pass's output), result through Q
  SSI_TRY(gram(w.Q1, m, shifted));
  SSI_TRY(chol_inv(w.W, k, m, w.Lb, w.Linvb, w.LinvTb, w.chol_g, status, s, shifted, nullptr, 0));
  SSI_TRY(trmul(w.Q1, m, w.Linvb, w.LinvTb, Q, shifted));
  cq_copy_kernel<<<148 * 4, 256, 0, s>>>(shifted, m * k, Q, w.Q1);
  SSI_TRY(launch_check("cq_copy_kernel"));
#endif
  SSI_TRY(gram(w.Q1, m, nullptr));
  SSI_TRY(chol_inv(w.W, k, m, w.L2, w.Linv2, w.LinvT2, w.chol_g, status, s, nullptr, nullptr, 1));
  SSI_TRY(trmul(w.Q1, m, w.Linv2, w.LinvT2, Q, nullptr));
#ifdef SSI_NO_CQ_FALLBACK
  return SSI_OK;
#endif
  cq_fold_kernel<<<2 * k, 128, size_t(k) * sizeof(double), s>>>(shifted, k, w.Lb, w.Linvb, w.L2, w.Linv2);
  return launch_check("cq_fold_kernel");
}

// One CholeskyQR pass (with the shift on breakdown): the re-orthonormalisation between the
// power iterations' passes, where only span(Q) matters (the next pass and the final CholeskyQR2
// see the same subspace); its orthogonality error ~ kappa(Y)^2 u is removed by the next QR.
ssi_status cholqr1(const double* Y, int64_t ldy, int64_t m, int k, double* Q, CholQRWork& w,
                   int32_t* status, cudaStream_t s) {
  if (k > kSvdMaxK) return cholqr2_big(Y, ldy, m, k, Q, w, status, s);
  const bool tall = k <= kTallMaxN && ldy % 2 == 0 && m % 2 == 0 && k % 2 == 0 &&
                    (reinterpret_cast<uintptr_t>(Y) & 15) == 0 && (reinterpret_cast<uintptr_t>(Q) & 15) == 0;
  if (tall) {
    SSI_TRY(gemm_tall_syrk_lower(k, m, Y, ldy, Y, ldy, w.W, k, w.tallp, s, nullptr));
  } else {
    SSI_TRY(gemm_f64(k, k, m, 1.0, Operand{Y, ldy, 1}, Operand{Y, 1, ldy}, w.W, k, gemm_pick_splits(k, k, m),
                     w.partial, s, nullptr));
  }
  SSI_TRY(chol_inv(w.W, k, m, w.L1, w.Linv1, w.LinvT1, w.chol_g, status, s, nullptr, w.flag, 0));
  if (tall) return gemm_tall_triu(m, k, k, Y, ldy, w.LinvT1, k, Q, m, s, nullptr);
  return gemm_f64(m, k, k, 1.0, Operand{Y, 1, ldy}, Operand{w.Linv1, k, 1}, Q, m, 1, nullptr, s, nullptr);
}

template <int KPL, int JCT>
static ssi_status jacobi_launch(double* G, int k, double* Ut, double* S, double* scratch, int32_t* status,
                                cudaStream_t s) {
  const size_t smem = size_t(k) * (sizeof(double) + sizeof(int));
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(jacobi_kernel<KPL, JCT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (JCT > 8) cudaFuncSetAttribute(jacobi_kernel<KPL, JCT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  static const int profile = getenv("SSI_JAC_PROFILE") ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(JCT);
  cfg.blockDim = dim3(kJacThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = JCT;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (JCT > 8) {   // a 16-CTA cluster is opt-in: fall back to the portable 8 when it cannot be placed
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, jacobi_kernel<KPL, JCT>, &cfg) != cudaSuccess || nc < 1) {
      cudaGetLastError();
      return jacobi_launch<KPL, 8>(G, k, Ut, S, scratch, status, s);
    }
  }
  double* gnrm = scratch;
  int* gflag = reinterpret_cast<int*>(scratch + k);
  if constexpr (SSI_JAC_RING && JCT == 8 && KPL <= 8) if (k >= 3) {
    // ring variant: mailboxes for 16 warps x 2 slots x 2 buffers per CTA
    const size_t rsmem = size_t(kJacThreads / 32) * 4 * (KPL * 32 + 2) * sizeof(double);
    const size_t fsmem = size_t(k) * (sizeof(double) + sizeof(int));
    cfg.dynamicSmemBytes = rsmem > fsmem ? rsmem : fsmem;
    cudaFuncSetAttribute(jacobi_ring_kernel<KPL, JCT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(cfg.dynamicSmemBytes));
    if (cudaLaunchKernelEx(&cfg, jacobi_ring_kernel<KPL, JCT>, G, k, Ut, S, gflag, status, profile) != cudaSuccess)
      return launch_check("jacobi_ring_kernel (cluster launch)");
    return SSI_OK;
  }
  if (cudaLaunchKernelEx(&cfg, jacobi_kernel<KPL, JCT>, G, k, Ut, S, gnrm, gflag, status, profile) != cudaSuccess)
    return launch_check("jacobi_kernel (cluster launch)");
  return SSI_OK;
}

size_t jacobi_scratch_elems(int k) {
  return k > kSvdMaxK ? jacobi_big_scratch_elems(k) : size_t(k) + kJacMaxSweeps / 2 + 1;
}

ssi_status jacobi_svd(double* G, int k, double* Ut, double* S, double* scratch, int32_t* status, cudaStream_t s) {
  ssi_status st;
  if (k <= 64) st = jacobi_launch<2, JC>(G, k, Ut, S, scratch, status, s);
  else if (k <= 128) st = jacobi_launch<4, JC>(G, k, Ut, S, scratch, status, s);
  else if (k <= 256) st = jacobi_launch<8, JC>(G, k, Ut, S, scratch, status, s);
  else if (k <= 512) st = jacobi_launch<16, 16>(G, k, Ut, S, scratch, status, s);
  else if (k <= kBigMaxK) return jacobi_big(G, k, Ut, S, scratch, status, s);
  else {
    set_last_error("jacobi_svd: k = %d > %d unsupported", k, kBigMaxK);
    return SSI_ERR_INVALID_ARG;
  }
  if (st != SSI_OK) return st;
  return launch_check("jacobi_kernel");
}

}  // namespace ssi
