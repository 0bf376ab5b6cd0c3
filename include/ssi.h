/*
 * ssi.h — C ABI of libssi.so, the B200 (sm_100a) hot path of covariance-driven
 * Stochastic Subspace Identification with Randomized SVD (arXiv 2411.05510,
 * Tomassini, García-Macías, Ubertini). Citations are /root/reference/PAPER.md line
 * numbers followed by the paper section / equation.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Every array pointer is DEVICE memory owned by the caller (in Python: torch CUDA
 *    tensors). The library never allocates or frees caller memory and keeps no
 *    pointer past the completion of the enqueued work. Scratch comes from the caller's
 *    workspace `ws` of `ws_bytes` bytes, sized by the matching *_ws() query.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream). All
 *    work is enqueued on it; a call returns once enqueued. Outputs are valid after the
 *    stream orders past them. The caller selects the device (cudaSetDevice).
 *  - No global mutable state: calls are reentrant across host threads and devices.
 *  - Matrices are FP64. "col-major" means element (r, c) at ptr[r + c*ld];
 *    "row-major" means ptr[r*ld + c].
 *  - Synchronous argument checks run before any launch and leave outputs untouched:
 *    NULL pointers / bad sizes -> SSI_ERR_INVALID_ARG, leading dimension too small ->
 *    SSI_ERR_SHAPE, unsupported dtype / mode -> SSI_ERR_DTYPE, workspace too small ->
 *    SSI_ERR_WORKSPACE, a failed launch -> SSI_ERR_CUDA (detail in ssi_last_error()).
 *  - Asynchronous numeric failures (a Cholesky breakdown that the shifted-CholeskyQR3
 *    fallback below could not absorb, Jacobi or Francis-QR non-convergence, non-finite
 *    input) are recorded in a device status word at the start of `ws` (its first 256 bytes
 *    are a header). The word is STICKY: every call max-combines its failures into it and no
 *    call clears it, so a workspace reused by many calls (a record pipeline, a lag sweep)
 *    reports a failure of any of them; zero it once before first use (ssi_clear_status, or
 *    zero the 256-byte header) and read it with ssi_fetch_device_status() after
 *    synchronizing the stream.
 *  - QR (CholeskyQR2, "qr(Y,0)") on a numerically rank-deficient panel
 *    (e.g. a sketch width k above the rank of T): the first Cholesky of the Gram matrix
 *    W = Y^T Y breaks down when a pivot falls below 64 k u times its diagonal entry; it is
 *    then redone on W + s I, s = 11 (m k + k (k + 1)) u tr(W) (shifted CholeskyQR), and one
 *    extra CholeskyQR pass runs before the usual second one (shifted CholeskyQR3). The
 *    decision is taken on the device (conditional launches), so it costs no host
 *    synchronisation; the status stays SSI_OK. Only a breakdown of the final pass, or a
 *    non-finite Gram matrix, sets SSI_ERR_NUMERIC. Sketch widths k > 512 (the paper's rank rule
 *    at bridge sizes, blocked whole-GPU Cholesky) take the same fallback through conditional
 *    launches of the blocked kernels (the shift uses the trace of the unshifted Gram matrix),
 *    with up to three shifted extra passes, each run only if the previous one shifted (an
 *    exactly rank-deficient panel needs two or three; see linalg_big.cu).
 *  - Determinism: fixed inputs, seed and launch configuration give bit-identical
 *    outputs run to run (fixed reduction orders, no floating-point atomics).
 */
#ifndef SSI_H_
#define SSI_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SSI_API __attribute__((visibility("default")))
#else
#define SSI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t ssi_status;
enum {
  SSI_OK = 0,
  SSI_ERR_INVALID_ARG = 1,
  SSI_ERR_SHAPE = 2,
  SSI_ERR_DTYPE = 3,
  SSI_ERR_WORKSPACE = 4,
  SSI_ERR_CUDA = 5,
  SSI_ERR_NONFINITE = 6,
  SSI_ERR_NUMERIC = 7
};

/* Record storage types. */
enum { SSI_F32 = 0, SSI_F64 = 1 };

/* Covariance arithmetic (ssi_covariances cov_mode).
 *  SSI_COV_FP64   : FP64 products and sums (DMMA tensor-core path).
 *  SSI_COV_INT8X3 : each sample is cut into three int8 slices against a per-channel
 *                   power-of-two scale; the eight leading slice products (all but d3*d3) are summed
 *                   EXACTLY in int32 on the 5th-gen tensor cores (tcgen05 kind::i8)
 *                   and promoted to FP64. Error is the slicing rounding only
 *                   (<= 2^-22 of the channel's max |y| per sample); see DESIGN.md.
 *                   Channel counts: l % 64 == 0, or l % 16 == 0 and l <= 64; any other l
 *                   -> SSI_ERR_DTYPE from ssi_covariances and ssi_covariances_ws.
 *  SSI_COV_SPECTRAL : the same sums through segment cross-spectra, FP64 throughout: the record
 *                   is cut into segments of B = F - lag_hi samples (F a power of two <= 2048
 *                   chosen by a flop model), one FFT per segment and channel gives the spectra
 *                   of the segment and of the segment plus its lag_hi halo, their cross-spectra
 *                   are summed over segments on the FP64 tensor cores (DMMA) and an inverse DFT
 *                   at the requested lags yields R_k exactly up to FP64 rounding (relative error
 *                   ~1e-15 of the lag-0 scale). Segments are processed in chunks of at most
 *                   512, so the workspace is bounded independently of N. Needs lag_hi < 2048.
 *                   See DESIGN.md. */
enum { SSI_COV_FP64 = 0, SSI_COV_INT8X3 = 1, SSI_COV_SPECTRAL = 2 };

/* ------------------------------------------------------------------------------
 * A1. Lagged output covariances (§2.1; normalization 1/(N-k), reading
 * A-6 of DESIGN.md):
 *     R_k[a][b] = (1/(N-k)) * sum_{t=0}^{N-k-1} Y[t+k][a] * Y[t][b],  k = lag_lo..lag_hi
 *  Y       : record, time-major [N][ldY] (channel a of sample t at Y[t*ldY + a]),
 *            dtype SSI_F32 or SSI_F64, ldY >= l. Must be finite.
 *  R       : output [(lag_hi-lag_lo+1)][l][l] row-major FP64, R_k at block k-lag_lo.
 *  t_begin, t_end : time shard of the sum, 0 <= t_begin <= t_end <= N: only terms with
 *            t in [t_begin, t_end) and t+k < N are summed (the kernel reads the halo
 *            rows t_end .. t_end+lag_hi-1 itself). Used by time-sharded multi-GPU runs.
 *  normalize : 1 = divide by (N-k) (requires t_begin = 0, t_end = N);
 *            0 = raw FP64 sums (to be all-reduced across shards, then divided).
 *  Errors: lag_lo < 1, lag_hi < lag_lo or lag_hi >= N -> INVALID_ARG ("record too
 *  short"); bad shard -> INVALID_ARG; dtype/mode pairs not supported ->
 *  DTYPE. Non-finite samples set SSI_ERR_NONFINITE in the device status word.
 * ---------------------------------------------------------------------------- */
SSI_API ssi_status ssi_covariances(const void* Y, int32_t dtype, int64_t N, int32_t l, int64_t ldY,
                           int32_t lag_lo, int32_t lag_hi, int32_t cov_mode,
                           int64_t t_begin, int64_t t_end, int32_t normalize,
                           double* R, void* ws, size_t ws_bytes, void* stream);
SSI_API ssi_status ssi_covariances_ws(int64_t N, int32_t l, int32_t lag_lo, int32_t lag_hi,
                              int32_t cov_mode, size_t* bytes);
/* SSI_COV_SPECTRAL plan for a record of N samples (pure host function): FFT length F (the
 * segment length is F - lag_hi) and the number of segments S covering the full record. The
 * cross-spectral product then costs 6 lp^2 S (F/2 + 1) flops and the inverse transform
 * 2 lp^2 (lag_hi - lag_lo + 1) (F + 2), lp = l rounded up to even. */
SSI_API ssi_status ssi_cov_spectral_plan(int64_t N, int32_t l, int32_t lag_lo, int32_t lag_hi,
                                 int32_t* F, int64_t* S);
/* A1 across time shards: in place R[k - lag_lo][a][b] /= (N - k), k = lag_lo .. lag_lo + n_lags - 1
 * (reading A-6), turning the raw sums of time-sharded ssi_covariances(normalize = 0) calls,
 * summed over the shards (e.g. one NCCL all-reduce across ranks), into the covariances of the
 * whole N-sample record. R: [n_lags][l][l] FP64 device. Errors: lag_lo < 1, n_lags < 1, l < 1
 * or lag_lo + n_lags - 1 >= N -> INVALID_ARG. */
SSI_API ssi_status ssi_cov_normalize(double* R, int32_t l, int32_t lag_lo, int32_t n_lags, int64_t N,
                                     void* stream);
/* Measurement entry point of SSI_COV_SPECTRAL (not part of the method): runs the phases in the
 * bit mask `phases` (1 = twiddle/weight tables + segment FFTs, 2 = cross-spectral product,
 * 4 = inverse DFT at the lags) with the arguments of ssi_covariances. phases = 7 is
 * ssi_covariances(cov_mode = SSI_COV_SPECTRAL); a partial mask re-runs those phases on the
 * spectra an earlier full call left in the same workspace (bench.py times the product kernel
 * alone this way). */
SSI_API ssi_status ssi_cov_spectral_phases(const void* Y, int32_t dtype, int64_t N, int32_t l, int64_t ldY,
                                           int32_t lag_lo, int32_t lag_hi, int64_t t_begin, int64_t t_end,
                                           int32_t normalize, double* R, void* ws, size_t ws_bytes,
                                           int32_t phases, void* stream);

/* ------------------------------------------------------------------------------
 * A2. Block-Toeplitz matrix T_{1|i}, Eq. (6) (§2.1):
 *     T[r*l + a][c*l + b] = R_{i+r-c}[a][b],   r, c in [0, i)
 *  R : [2i-1][l][l] row-major FP64 holding R_1..R_{2i-1} (R_k at block k-1), e.g. the
 *      output of ssi_covariances with lag_lo = 1, lag_hi >= 2i-1.
 *  T : output, row-major, m = l*i rows and columns, ldT >= m. Pure copy (bit-exact).
 * ---------------------------------------------------------------------------- */
SSI_API ssi_status ssi_toeplitz(const double* R, int32_t l, int32_t i, double* T, int64_t ldT,
                        void* stream);

/* ------------------------------------------------------------------------------
 * A3-A8. Randomized SVD of T (§2.2, Algorithm 1 at PAPER.md:255-268,
 * Eqs. 13-18) with q power iterations (north star; reading A-12):
 *   Omega = N(0,1) m x k sketch from Philox4x32-10 (key = seed, counter = (element
 *           pair index, stream_id); reading A-11), generated on the device;
 *   Y = T Omega; Q = qr(Y) (CholeskyQR2, diag(R) > 0);
 *   q times: Z = qr(T^T Q); Q = qr(T Z);
 *   B = Q^T T; small SVD B = U~ S V^T (CholeskyQR2 of B^T + one-sided Jacobi);
 *   U = Q U~.
 *  T : m x m row-major FP64, ldT >= m.   k : sketch width (n_max + p, or the paper's rank rule
 *      k = ceil(kbar(T) % T)), 1 <= k <= min(m, 4096): k <= 512 runs the small
 *      SVD on one thread-block cluster, larger k the blocked whole-GPU Cholesky / triangular solve
 *      and a block one-sided Jacobi (one persistent CTA per 32-column block pair); larger k ->
 *      INVALID_ARG, synchronously.
 *  U : output m x n_keep col-major FP64 (leading left singular vectors), ldU >= m,
 *      1 <= n_keep <= k. Column signs are arbitrary (reading A-13).
 *  S : output [k] FP64, descending.
 *  Errors: k or n_keep out of range -> INVALID_ARG. A rank-deficient sketch (k above the
 *  numerical rank of T) is handled by the shifted-CholeskyQR3 fallback (see the conventions
 *  above) and returns SSI_OK with S[j] ~ 0 beyond the rank. A final-pass Cholesky breakdown or
 *  Jacobi non-convergence -> SSI_ERR_NUMERIC in the device status word.
 * ---------------------------------------------------------------------------- */
SSI_API ssi_status ssi_rsvd(const double* T, int64_t ldT, int32_t m, int32_t k, int32_t q,
                    uint64_t seed, uint64_t stream_id, int32_t n_keep,
                    double* U, int64_t ldU, double* S, void* ws, size_t ws_bytes,
                    void* stream);
/* Workspace bytes of ssi_rsvd; pure host function. The size is non-decreasing in m, so a
 * workspace sized for the largest m of a lag sweep serves every smaller lag. */
SSI_API ssi_status ssi_rsvd_ws(int32_t m, int32_t k, int32_t n_keep, size_t* bytes);

/* ------------------------------------------------------------------------------
 * A2-A8 without forming T: the same randomized SVD (same Omega, same steps and outputs as
 * ssi_rsvd on T = ssi_toeplitz(R, l, i)), with every product T X / T^T X applied through
 * the block structure of Eq. (6): (T X)_r = sum_c R_{i+r-c} X_c is a
 * block convolution, evaluated exactly as a length-(2i-1) block DFT, i complex (l x l)(l x k)
 * products per pass on the FP64 tensor cores, and the inverse DFT (north star (b): "exploit
 * its block-Toeplitz structure"). Results equal ssi_rsvd's up to FP64 rounding order.
 *  R : [>= 2i-1][l][l] row-major FP64, R_k at block k-1 (ssi_covariances, lag_lo = 1).
 *  m = l*i; k, q, seed, stream_id, n_keep, U, ldU, S as in ssi_rsvd.
 *  Errors: as ssi_rsvd (k <= min(l*i, 4096)); i < 1 or l < 1 -> INVALID_ARG.
 * ---------------------------------------------------------------------------- */
SSI_API ssi_status ssi_rsvd_toeplitz(const double* R, int32_t l, int32_t i, int32_t k, int32_t q,
                             uint64_t seed, uint64_t stream_id, int32_t n_keep,
                             double* U, int64_t ldU, double* S, void* ws, size_t ws_bytes,
                             void* stream);
/* Workspace bytes of ssi_rsvd_toeplitz; pure host function, non-decreasing in i. */
SSI_API ssi_status ssi_rsvd_toeplitz_ws(int32_t l, int32_t i, int32_t k, int32_t n_keep, size_t* bytes);

/* Raw Philox words and the Gaussian sketch, exposed for bit-exact verification
 * (P13). words: [n_pairs][4] uint32 for pairs 0..n_pairs-1; omega: m x k col-major. */
SSI_API ssi_status ssi_philox_words(uint64_t seed, uint64_t stream_id, int64_t n_pairs,
                            uint32_t* words, void* stream);
SSI_API ssi_status ssi_gaussian_sketch(int32_t m, int32_t k, uint64_t seed, uint64_t stream_id,
                               double* omega, int64_t ldo, void* stream);

/* ------------------------------------------------------------------------------
 * A9-A11. Modal sweep over model orders n = n_min, n_min+n_step, ..., <= n_max (even),
 * PAPER.md:156-206 (§2.1, Eqs. 9-12):
 *   O_n = U_n S_n^{1/2}; A_n = pinv(O_n^up) O_n^down (first / last l(i-1) rows,
 *   reading A-2); C_n = first l rows; A_n = Psi M Psi^{-1} (reading A-4);
 *   lambda = ln(mu)/dt, f = |lambda|/(2 pi), xi = -Re(lambda)/|lambda| (reading A-1);
 *   Phi = C_n Psi. Computed in the S-free nested form: thin QR U^up = Q R, W = Q^T U^down,
 *   M_n = R[:n,:n]^{-1} W[:n,:n] has the eigenvalues of A_n and Phi = U[0:l,:n] psi_M.
 *   Poles: Im(mu) > 0, 0 < xi < 1 (reading A-14), shapes unit-norm with the largest
 *   component real positive (A-15), MPC / MPD (A-16), sorted by (f, xi).
 *  U : m x n_max col-major (m = l*i, ldU >= m), S : [>= n_max] descending (ssi_rsvd).
 *  n_max <= 512 (PAPER.md:518 sweeps orders up to 400); orders whose banded Schur matrix
 *  exceeds shared memory (n_max above ~230) keep it in the workspace (L2-resident).
 *  out : caller-allocated pole table (device arrays) with n_orders = number of orders,
 *        cap >= n_max/2, l = channels. count[o] = number of poles, or -1 when
 *        S[n-1] < 1e-12 S[0] (order above the numerical rank) or when the
 *        order's eigen-solve did not converge. Slots past count[o] hold zeros (every array),
 *        so tables are bit-reproducible whatever the buffers held before.
 * ---------------------------------------------------------------------------- */
typedef struct {
  int32_t n_orders;  /* number of model orders (rows) */
  int32_t cap;       /* pole slots per order (>= n_max/2) */
  int32_t l;         /* channels (mode-shape length) */
  int32_t n_min;     /* first order */
  int32_t n_step;    /* order step (2) */
  int32_t* count;    /* [n_orders] */
  double* f;         /* [n_orders][cap] Hz */
  double* xi;        /* [n_orders][cap] damping ratio */
  double* mu_re;     /* [n_orders][cap] discrete pole, real part */
  double* mu_im;     /* [n_orders][cap] discrete pole, imaginary part */
  double* mpc;       /* [n_orders][cap] */
  double* mpd;       /* [n_orders][cap] */
  double* shape;     /* [n_orders][cap][l][2] (re, im) */
} ssi_pole_table;

SSI_API ssi_status ssi_modal_sweep(const double* U, int64_t ldU, const double* S, int32_t l,
                           int32_t i, int32_t n_min, int32_t n_max, int32_t n_step,
                           double dt, const ssi_pole_table* out, void* ws, size_t ws_bytes,
                           void* stream);
SSI_API ssi_status ssi_modal_sweep_ws(int32_t l, int32_t i, int32_t n_min, int32_t n_max,
                              int32_t n_step, size_t* bytes);

/* ------------------------------------------------------------------------------
 * A13. Hard + 3D soft stability criteria (§2.1 and Eq.
 * (stabcriteria3D), §2.3 step ii):
 *   HC: keep iff xi <= xi_max && mpc > mpc_min && mpd < mpd_max (reading A-17).
 *   SC: a kept pole at (lag g, order o) is stable iff one kept pole at (g, o-1) OR at
 *       (g-1, o) has d_f <= alpha_f && d_xi <= alpha_xi && 1-MAC <= alpha_mac
 *       (readings A-18..A-21).
 *  tables : host array of n_lags pole tables (device arrays inside), lags in increasing
 *           i, all with equal n_orders, cap, l, n_min, n_step.
 *  flags  : output [n_lags][n_orders][cap] uint8: 0 rejected / empty, 1 new, 2 stable.
 *  stable_count : output [n_lags][n_orders] int32 (number of flag-2 poles).
 * ---------------------------------------------------------------------------- */
typedef struct {
  double xi_max, mpc_min, mpd_max;     /* hard criteria */
  double alpha_f, alpha_xi, alpha_mac; /* soft criteria */
} ssi_criteria;

SSI_API ssi_status ssi_stab3d(const ssi_pole_table* tables, int32_t n_lags, const ssi_criteria* crit,
                      uint8_t* flags, int32_t* stable_count, void* stream);

/* ------------------------------------------------------------------------------
 * NEXT-2. Two-stage clustering of the stable poles of a 3D stabilization diagram
 * (§2.3 step iii; §3.1.3; §3.2.2) and modal
 * tracking (§3.2.2, Table 4). Readings C-1..C-5 of DESIGN.md §3:
 *  Stage I  (ssi_cluster_stage1): every pole with flag 2 (stable) gets the features of its
 *           best soft-criteria neighbour (order axis (g, o-1) first, then lag axis (g-1, o),
 *           slots ascending, least d_f + d_xi + (1-MAC), first on ties):
 *           x = (d_f, d_xi, 1-MAC, 1-MPC, MPD) (C-1). Fuzzy C-means with c = 2, m = 2,
 *           centroids initialised at the feature-wise min and max, until the largest centroid
 *           move is < fcm_tol or fcm_max_iter iterations (C-2). The "possibly physical"
 *           cluster is the one whose centroid is nearer the origin; a pole is
 *           retained iff its membership there is >= 0.5 (C-3).
 *  Stage II (ssi_cluster_stage2): d(i, j) = d_f + d_xi + (1 - MAC) between retained poles
 *           (PAPER.md:293, :405); average linkage (UPGMA); flat clusters = merges at height
 *           <= cutoff; clusters with < min_size members are dropped; per cluster the lower
 *           median f and xi and the medoid's shape (least summed distance, lowest index on
 *           ties); clusters ordered by (f, smallest member index) (C-4).
 *  Tracking (ssi_track): a session mode c is a candidate for reference mode r iff
 *           |f_c - f_r| / max(f_c, f_r) <= df_max and 1 - MAC <= macd_max; candidates are
 *           assigned one-to-one in ascending d_f + (1 - MAC) order (ties: lower r, then lower
 *           c); success[r] = 100 * (sessions where r was matched) / n_sess (C-5).
 * The pole table layout is the one of ssi_modal_sweep; tables as for ssi_stab3d, at most
 * SSI_MAX_LAGS lags. All arrays are device memory. Indices of stable poles ("pole rows") are
 * in (lag, order, slot) lexicographic order; "retained rows" index the retained poles in
 * increasing pole-row order.
 * ---------------------------------------------------------------------------- */
#define SSI_MAX_LAGS 64

typedef struct {
  int32_t n_stable;      /* stable poles (flag 2) in the diagram */
  int32_t n_retained;    /* poles with membership >= 0.5 in the physical FCM cluster */
  int32_t fcm_iters;     /* fuzzy C-means iterations run */
  int32_t phys;          /* index (0 / 1) of the possibly-physical FCM cluster */
  int32_t n_components;  /* stage II: connected components of {d <= cutoff} (diagnostic) */
  int32_t n_clusters;    /* stage II: clusters with >= min_size members */
  int32_t n_merges;      /* stage II: average-linkage merges at height <= cutoff */
  int32_t overflow;      /* 1: n_stable > max_poles or n_clusters > max_clusters (truncated) */
  double V[2][5];        /* FCM centroids */
} ssi_cluster_info;

/* Stage I. flags: [n_lags][n_orders][cap] from ssi_stab3d with the same crit.
 *  pole_idx [max_poles][3] int32 (lag, order index, slot); X [max_poles][5] features;
 *  U [max_poles][2] final memberships; retained [max_poles] int32 pole rows of the retained
 *  poles; info: device struct (all fields of stage I written). Rows past info.n_stable (or
 *  max_poles) are not written.
 *  Errors: n_lags outside [1, SSI_MAX_LAGS], tables of different shape, max_poles < 1,
 *  fcm_tol < 0 or fcm_max_iter < 0 -> INVALID_ARG; ws_bytes below ssi_cluster_stage1_ws ->
 *  WORKSPACE. A flag-2 pole without a qualifying neighbour (flags made with other criteria)
 *  gets NaN features and sets SSI_ERR_NUMERIC in the device status word. */
SSI_API ssi_status ssi_cluster_stage1(const ssi_pole_table* tables, int32_t n_lags, const ssi_criteria* crit,
                                      const uint8_t* flags, int32_t max_poles, double fcm_tol,
                                      int32_t fcm_max_iter, int32_t* pole_idx, double* X, double* U,
                                      int32_t* retained, ssi_cluster_info* info, void* ws, size_t ws_bytes,
                                      void* stream);
SSI_API ssi_status ssi_cluster_stage1_ws(int32_t n_lags, int32_t n_orders, size_t* bytes);

/* Stage II on the n_retained poles listed by stage I (n_retained = info.n_retained, read by the
 * caller after stage I; the workspace, O(n_retained^2) doubles, depends on it).
 *  labels [n_retained] int32: cluster of each retained row (0..), -1 if its cluster was dropped.
 *  cl_f, cl_xi [max_clusters], cl_size, cl_medoid (retained row) [max_clusters] int32,
 *  cl_shape [max_clusters][l][2]: the clusters in output order; info.n_clusters of them.
 *  merges_ab [n_retained][2] int32 (retained rows; the surviving cluster keeps the larger
 *  row) and merges_h [n_retained]: the merges at height <= cutoff, component by component,
 *  padded with -1 / NaN; either may be NULL.
 *  Errors: n_retained < 0, min_size < 1, max_clusters < 1, cutoff not finite -> INVALID_ARG;
 *  ws_bytes below ssi_cluster_stage2_ws -> WORKSPACE. */
SSI_API ssi_status ssi_cluster_stage2(const ssi_pole_table* tables, int32_t n_lags, const int32_t* pole_idx,
                                      const int32_t* retained, int32_t n_retained, double cutoff,
                                      int32_t min_size, int32_t max_clusters, int32_t* labels, double* cl_f,
                                      double* cl_xi, int32_t* cl_size, int32_t* cl_medoid, double* cl_shape,
                                      int32_t* merges_ab, double* merges_h, ssi_cluster_info* info, void* ws,
                                      size_t ws_bytes, void* stream);
SSI_API ssi_status ssi_cluster_stage2_ws(int32_t n_retained, int32_t l, size_t* bytes);

/* Tracking over n_sess sessions against n_ref reference modes.
 *  ref_f [n_ref], ref_shape [n_ref][l][2]; f [n_sess][max_modes], shape
 *  [n_sess][max_modes][l][2], count [n_sess] int32 (modes of each session; clamped to
 *  [0, max_modes]). match [n_sess][n_ref] int32: the session mode assigned to r, or -1.
 *  success [n_ref] (may be NULL): percentage of sessions in which r was matched.
 *  Errors: n_ref < 1, n_sess < 1, max_modes < 1, l < 1, n_ref * max_modes > 16384 ->
 *  INVALID_ARG. */
SSI_API ssi_status ssi_track(const double* ref_f, const double* ref_shape, int32_t n_ref, const double* f,
                             const double* shape, const int32_t* count, int32_t n_sess, int32_t max_modes,
                             int32_t l, double df_max, double macd_max, int32_t* match, double* success,
                             void* stream);

/* ------------------------------------------------------------------------------
 * NEXT-4. Upstream preprocessing of raw acceleration records (§3.2): "elimination
 * of linear trends and downsampling to 40 Hz (eighth-order low-pass Chebyshev Type I filter with
 * a cut-off frequency of 0.8·20 Hz followed by a decimation to 40 Hz)". Readings P-1..P-3 of
 * DESIGN.md §3:
 *  P-1 per channel, subtract the least-squares line alpha + beta h (h = 0..N-1);
 *  P-2 Chebyshev-I low-pass of the given even order (2..16) and passband ripple rp_db, passband
 *      edge fc_hz, designed by the bilinear transform (prewarped) for the rate L fs_in, applied
 *      zero-phase: forward, then backward, zero initial state, no padding;
 *  P-3 upsample by L (L x[n] at n L, zeros between), filter (P-2), keep every M-th sample
 *      starting with the first: Z has N_out = floor(N L / M) rows (125 -> 40 Hz: L = 8, M = 25;
 *      an integer decimation by q: L = 1, M = q).
 *  Y : [N][ldY] SSI_F32 / SSI_F64, ldY >= l. Z : [N_out][ldZ] of out_dtype, ldZ >= l.
 *  Errors: N < 2, l < 1, L < 1, M < 1, fs_in <= 0, odd order or order outside 2..16, rp_db <= 0,
 *  fc_hz outside (0, L fs_in / 2), N_out < 1 -> INVALID_ARG; ld too small -> SHAPE; workspace
 *  (O(N L l) doubles: the forward-filtered signal at the high rate) too small -> WORKSPACE.
 * ---------------------------------------------------------------------------- */
SSI_API ssi_status ssi_preprocess(const void* Y, int32_t dtype, int64_t N, int32_t l, int64_t ldY, double fs_in,
                                  int32_t L, int32_t M, int32_t order, double rp_db, double fc_hz, void* Z,
                                  int32_t out_dtype, int64_t ldZ, void* ws, size_t ws_bytes, void* stream);
SSI_API ssi_status ssi_preprocess_ws(int64_t N, int32_t l, int32_t L, int32_t order, size_t* bytes);
/* The filter of P-2 as second-order sections: sos [order/2][5] = (b0, b1, b2, a1, a2) with
 * a0 = 1 (verification entry point; same design kernel as ssi_preprocess). */
SSI_API ssi_status ssi_lowpass_design(int32_t order, double rp_db, double fc_hz, double fs_hz, double* sos,
                                      void* stream);

/* ------------------------------------------------------------------------------
 * NEXT-4. The paper's shear-type frame generator (§3.1; §3.1.2;
 * readings F-1..F-4 of DESIGN.md §3): n_dof storeys of mass m and stiffness k (K tridiagonal:
 * 2k on the diagonal except k at the roof, -k off it), Rayleigh damping C = a M + b K with
 * damping ratio xi at undamped modes mode_a and mode_b; state x = (q, dq/dt), a Gaussian force
 * at every DOF held over each step (zero-order hold: [[A_d, B_d], [0, I]] = exp([[A_c, B_c],
 * [0, 0]] / fs)); x_0 = 0, x_{h+1} = A_d x_h + B_d u_h; outputs the accelerations
 * y_h = C_o x_h, C_o = [-M^-1 K, -M^-1 C]; the first n_burn samples are discarded; channel c
 * gets Gaussian noise of variance P_c / 10^(snr_db/10), P_c the mean square of the kept clean
 * channel. u_h: column h of the reading-A-11 Philox Gaussian sketch n_dof x (n_burn + N) with
 * (seed, stream 2 stream_id); v_h: column h of the l x N sketch with (seed, stream 2 stream_id + 1).
 *  Y : [N][ldY] (dtype), clean (may be NULL): [N][n_dof] FP64 noise-free outputs.
 *  Errors: n_dof outside 1..12, m, k, fs <= 0, xi outside (0, 1), modes outside 1..n_dof or
 *  equal, N < 1, n_burn < 0, (N + n_burn) n_dof >= 2^31 -> INVALID_ARG; ldY < n_dof -> SHAPE.
 * ssi_frame_model writes the model: Ad [2n][2n], Bd [2n][n], Co [n][2n] row-major, ab = (a, b).
 * ---------------------------------------------------------------------------- */
SSI_API ssi_status ssi_frame_simulate(int32_t n_dof, double m, double k, double xi, int32_t mode_a, int32_t mode_b,
                                      double fs, int64_t N, int64_t n_burn, double snr_db, uint64_t seed,
                                      uint64_t stream_id, void* Y, int32_t dtype, int64_t ldY, double* clean,
                                      void* ws, size_t ws_bytes, void* stream);
SSI_API ssi_status ssi_frame_simulate_ws(int32_t n_dof, int64_t N, int64_t n_burn, size_t* bytes);
SSI_API ssi_status ssi_frame_model(int32_t n_dof, double m, double k, double xi, int32_t mode_a, int32_t mode_b,
                                   double fs, double* Ad, double* Bd, double* Co, double* ab, void* stream);

/* ------------------------------------------------------------------------------
 * Status helpers.
 * ---------------------------------------------------------------------------- */
/* Zeroes the 256-byte header of ws (the sticky status word), enqueued on stream. */
SSI_API ssi_status ssi_clear_status(void* ws, void* stream);
/* Reads the device status word at the start of ws (synchronous copy; call after the
 * stream finished the work that used ws). */
SSI_API ssi_status ssi_fetch_device_status(const void* ws, ssi_status* code);
SSI_API const char* ssi_status_string(ssi_status s);
/* Thread-local detail of the last synchronous failure on this host thread. */
SSI_API const char* ssi_last_error(void);
/* Library version string and the compiled target ("sm_100a"). */
SSI_API const char* ssi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SSI_H_ */
