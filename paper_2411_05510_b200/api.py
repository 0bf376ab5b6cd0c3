"""Thin torch-facing binding over the libssi.so C ABI (include/ssi.h).

PyTorch supplies device memory and the current CUDA stream; every step of the method
runs in the library's sm_100a kernels. Functions mirror the C entry points:

    covariances(Y, lag_hi, ...)      -> R [L][l][l] FP64            (A1)
    toeplitz(R, i)                   -> T [m][m] FP64 row-major     (A2, Eq. 6)
    rsvd(T, k, q, seed, stream_id)   -> U [m][n_keep] (col-major), S [k]   (A3-A8, Alg. 1)
    rsvd_toeplitz(R, l, i, k, ...)   -> same RSVD, T applied through its block structure (A2-A8)
    modal_sweep(U, S, l, i, ...)     -> PoleTable                   (A9-A11, Eqs. 9-12)
    stab3d(tables, criteria)         -> flags, stable_count         (A13)
    cluster3d(tables, flags, crit)   -> Clustering (two-stage: fuzzy C-means + average linkage)
                                                                    (NEXT-2)
    track(ref_f, ref_shape, f, shape, count) -> match, success      (NEXT-2)
    preprocess(Y, fs_in, fs_out)     -> detrended, low-passed, resampled record (NEXT-4)
    frame_simulate(N, fs, snr_db, ...) -> shear-frame acceleration record      (NEXT-4)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import PoleTableC, CriteriaC, ClusterInfoC, call, SSI_F32, SSI_F64, SSI_COV_FP64, SSI_COV_INT8X3, SSI_COV_SPECTRAL

COV_MODES = {"fp64": SSI_COV_FP64, "int8x3": SSI_COV_INT8X3, "spectral": SSI_COV_SPECTRAL}


def _ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if not (isinstance(t, torch.Tensor) and t.is_cuda):
            raise TypeError("libssi operates on CUDA tensors only (no CPU fallback)")


def _workspace(nbytes: int, device) -> torch.Tensor:
    """Workspace of nbytes with its status header cleared (the status word is sticky)."""
    ws = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
    clear_status(ws)
    return ws


def clear_status(ws: torch.Tensor) -> None:
    """Zero the sticky device status word of ws (ssi_clear_status), on the current stream."""
    call("ssi_clear_status", _ptr(ws), _stream())


def device_status(ws: torch.Tensor) -> int:
    """Status word of the last call that used `ws` (synchronizes the stream)."""
    torch.cuda.current_stream().synchronize()
    v = C.c_int32(0)
    call("ssi_fetch_device_status", _ptr(ws), C.byref(v))
    return v.value


def _check_device(fn, ws, check):
    if check:
        code = device_status(ws)
        if code != 0:
            raise _lib.SSIError(fn + " (device status)", code)


def covariances_ws_bytes(N, l, lag_hi, lag_lo=1, mode="fp64") -> int:
    b = C.c_size_t(0)
    call("ssi_covariances_ws", N, l, lag_lo, lag_hi, COV_MODES[mode], C.byref(b))
    return b.value


def cov_spectral_plan(N, l, lag_hi, lag_lo=1):
    """(F, S): FFT length and segment count SSI_COV_SPECTRAL uses for an N-sample record."""
    F, S = C.c_int32(0), C.c_int64(0)
    call("ssi_cov_spectral_plan", N, l, lag_lo, lag_hi, C.byref(F), C.byref(S))
    return F.value, S.value


def cov_spectral_flops(N, l, lag_hi, lag_lo=1):
    """Algorithmic flops of SSI_COV_SPECTRAL: (cross-spectral product -- three real products per
    complex one, 6 lp^2 S (F/2+1) -- and the inverse transform: for F = 1024 one complex FFT per
    two elements, 5 F log2 F lp^2 / 2; otherwise the GEMM 2 lp^2 n_lags (F + 2))."""
    F, S = cov_spectral_plan(N, l, lag_hi, lag_lo)
    lp = l + (l & 1)
    if F == 1024 and lag_hi < F:
        inv = 5.0 * F * 10 * lp * lp / 2
    else:
        inv = 2.0 * lp * lp * (lag_hi - lag_lo + 1) * (F + 2)
    return 6.0 * lp * lp * S * (F // 2 + 1), inv


def covariances(Y: torch.Tensor, lag_hi: int, lag_lo: int = 1, mode: str = "fp64",
                t_begin: int = 0, t_end: int | None = None, normalize: bool = True,
                out: torch.Tensor | None = None, ws: torch.Tensor | None = None,
                check: bool = False) -> torch.Tensor:
    _require_cuda(Y)
    if Y.dim() != 2 or Y.stride(1) != 1:
        raise ValueError("Y must be [N][l] with unit channel stride")
    dtype = {torch.float32: SSI_F32, torch.float64: SSI_F64}.get(Y.dtype)
    if dtype is None:
        raise TypeError("Y must be float32 or float64")
    N, l = Y.shape
    t_end = N if t_end is None else t_end
    L = lag_hi - lag_lo + 1
    R = out if out is not None else torch.empty((L, l, l), dtype=torch.float64, device=Y.device)
    if ws is None:
        ws = _workspace(covariances_ws_bytes(N, l, lag_hi, lag_lo, mode), Y.device)
    call("ssi_covariances", _ptr(Y), dtype, N, l, Y.stride(0), lag_lo, lag_hi, COV_MODES[mode],
         t_begin, t_end, 1 if normalize else 0, _ptr(R), _ptr(ws), ws.numel(), _stream())
    _check_device("ssi_covariances", ws, check)
    return R


def cov_normalize(R: torch.Tensor, N: int, lag_lo: int = 1) -> torch.Tensor:
    """In place R[k - lag_lo] /= (N - k) on the device (ssi_cov_normalize): the all-reduced raw sums
    of time-sharded covariances(..., normalize=False) calls become the record's covariances."""
    _require_cuda(R)
    if R.dtype != torch.float64 or not R.is_contiguous() or R.dim() != 3:
        raise ValueError("R must be contiguous FP64 [L][l][l]")
    call("ssi_cov_normalize", _ptr(R), R.shape[1], lag_lo, R.shape[0], N, _stream())
    return R


def cov_spectral_phases(Y: torch.Tensor, lag_hi: int, phases: int, out: torch.Tensor, ws: torch.Tensor,
                        lag_lo: int = 1) -> torch.Tensor:
    """Measurement entry point (ssi_cov_spectral_phases): re-runs the SSI_COV_SPECTRAL phases in the
    bit mask (1 FFT, 2 cross-spectral product, 4 inverse DFT) on the workspace of an earlier full
    covariances(..., mode="spectral", ws=ws) call."""
    _require_cuda(Y, out, ws)
    dtype = {torch.float32: SSI_F32, torch.float64: SSI_F64}[Y.dtype]
    N, l = Y.shape
    call("ssi_cov_spectral_phases", _ptr(Y), dtype, N, l, Y.stride(0), lag_lo, lag_hi, 0, N, 1, _ptr(out),
         _ptr(ws), ws.numel(), phases, _stream())
    return out


def toeplitz(R: torch.Tensor, i: int, out: torch.Tensor | None = None) -> torch.Tensor:
    _require_cuda(R)
    l = R.shape[1]
    if R.shape[0] < 2 * i - 1 or not R.is_contiguous() or R.dtype != torch.float64:
        raise ValueError("R must be contiguous FP64 [>= 2i-1][l][l]")
    m = l * i
    T = out if out is not None else torch.empty((m, m), dtype=torch.float64, device=R.device)
    call("ssi_toeplitz", _ptr(R), l, i, _ptr(T), T.stride(0), _stream())
    return T


def rsvd_ws_bytes(m, k, n_keep) -> int:
    b = C.c_size_t(0)
    call("ssi_rsvd_ws", m, k, n_keep, C.byref(b))
    return b.value


def rsvd(T: torch.Tensor, k: int, q: int, seed: int, stream_id: int, n_keep: int | None = None,
         ws: torch.Tensor | None = None, check: bool = False):
    """Returns (U, S): U is an (m, n_keep) column-major view, S has k entries."""
    _require_cuda(T)
    m = T.shape[0]
    n_keep = k if n_keep is None else n_keep
    if T.dtype != torch.float64 or T.stride(1) != 1:
        raise ValueError("T must be FP64 row-major")
    Ucm = torch.empty((n_keep, m), dtype=torch.float64, device=T.device)   # col-major storage
    S = torch.empty(k, dtype=torch.float64, device=T.device)
    if ws is None:
        ws = _workspace(rsvd_ws_bytes(m, k, n_keep), T.device)
    call("ssi_rsvd", _ptr(T), T.stride(0), m, k, q, C.c_uint64(seed), C.c_uint64(stream_id),
         n_keep, _ptr(Ucm), m, _ptr(S), _ptr(ws), ws.numel(), _stream())
    _check_device("ssi_rsvd", ws, check)
    return Ucm.t(), S


def rsvd_into(T: torch.Tensor, k: int, q: int, seed: int, stream_id: int, n_keep: int,
              U: torch.Tensor, S: torch.Tensor, ws: torch.Tensor | None = None, check: bool = False):
    """rsvd() into caller buffers: U (m, n_keep) column-major view, S [k]."""
    _require_cuda(T, U, S)
    m = T.shape[0]
    if U.stride(0) != 1 or U.shape != (m, n_keep) or S.numel() < k:
        raise ValueError("U must be an (m, n_keep) column-major view and S hold k values")
    if ws is None:
        ws = _workspace(rsvd_ws_bytes(m, k, n_keep), T.device)
    call("ssi_rsvd", _ptr(T), T.stride(0), m, k, q, C.c_uint64(seed), C.c_uint64(stream_id),
         n_keep, _ptr(U), U.stride(1), _ptr(S), _ptr(ws), ws.numel(), _stream())
    _check_device("ssi_rsvd", ws, check)
    return U, S


def rsvd_toeplitz_ws_bytes(l, i, k, n_keep) -> int:
    b = C.c_size_t(0)
    call("ssi_rsvd_toeplitz_ws", l, i, k, n_keep, C.byref(b))
    return b.value


def rsvd_toeplitz(R: torch.Tensor, i: int, k: int, q: int, seed: int, stream_id: int,
                  n_keep: int | None = None, U: torch.Tensor | None = None, S: torch.Tensor | None = None,
                  ws: torch.Tensor | None = None, check: bool = False):
    """RSVD of the block-Toeplitz T of R (lags 1..2i-1) without forming T. Returns (U, S) as
    rsvd(toeplitz(R, i), ...) does: U an (m, n_keep) column-major view, S [k]."""
    _require_cuda(R)
    if R.dtype != torch.float64 or not R.is_contiguous() or R.dim() != 3 or R.shape[0] < 2 * i - 1:
        raise ValueError("R must be contiguous FP64 [>= 2i-1][l][l]")
    l = R.shape[1]
    m = l * i
    n_keep = k if n_keep is None else n_keep
    if U is None:
        U = torch.empty((n_keep, m), dtype=torch.float64, device=R.device).t()
    if S is None:
        S = torch.empty(k, dtype=torch.float64, device=R.device)
    _require_cuda(U, S)
    if U.stride(0) != 1 or U.shape != (m, n_keep) or S.numel() < k:
        raise ValueError("U must be an (m, n_keep) column-major view and S hold k values")
    if ws is None:
        ws = _workspace(rsvd_toeplitz_ws_bytes(l, i, k, n_keep), R.device)
    call("ssi_rsvd_toeplitz", _ptr(R), l, i, k, q, C.c_uint64(seed), C.c_uint64(stream_id), n_keep,
         _ptr(U), U.stride(1), _ptr(S), _ptr(ws), ws.numel(), _stream())
    _check_device("ssi_rsvd_toeplitz", ws, check)
    return U, S


def philox_words(seed: int, stream_id: int, n_pairs: int, device="cuda") -> torch.Tensor:
    w = torch.empty((n_pairs, 4), dtype=torch.int32, device=device)
    call("ssi_philox_words", C.c_uint64(seed), C.c_uint64(stream_id), n_pairs, _ptr(w), _stream())
    return w


def gaussian_sketch(m: int, k: int, seed: int, stream_id: int, device="cuda") -> torch.Tensor:
    om = torch.empty((k, m), dtype=torch.float64, device=device)
    call("ssi_gaussian_sketch", m, k, C.c_uint64(seed), C.c_uint64(stream_id), _ptr(om), m, _stream())
    return om.t()


@dataclass
class PoleTable:
    """Device pole table of one (record, lag): rows = model orders n_min..n_max."""
    n_min: int
    n_step: int
    l: int
    cap: int
    count: torch.Tensor      # [O] int32 (-1 = order not solved)
    f: torch.Tensor          # [O][cap] f64
    xi: torch.Tensor
    mu_re: torch.Tensor
    mu_im: torch.Tensor
    mpc: torch.Tensor
    mpd: torch.Tensor
    shape: torch.Tensor      # [O][cap][l][2] f64

    @classmethod
    def empty(cls, n_min, n_max, n_step, l, device, cap=None):
        O = (n_max - n_min) // n_step + 1
        cap = cap or n_max // 2
        z = lambda *s, dt=torch.float64: torch.zeros(s, dtype=dt, device=device)
        return cls(n_min, n_step, l, cap, z(O, dt=torch.int32), z(O, cap), z(O, cap), z(O, cap),
                   z(O, cap), z(O, cap), z(O, cap), z(O, cap, l, 2))

    @property
    def n_orders(self):
        return self.count.shape[0]

    @property
    def orders(self):
        return [self.n_min + j * self.n_step for j in range(self.n_orders)]

    def as_c(self) -> PoleTableC:
        return PoleTableC(self.n_orders, self.cap, self.l, self.n_min, self.n_step,
                          self.count.data_ptr(), self.f.data_ptr(), self.xi.data_ptr(),
                          self.mu_re.data_ptr(), self.mu_im.data_ptr(), self.mpc.data_ptr(),
                          self.mpd.data_ptr(), self.shape.data_ptr())

    def tensors(self):
        return [self.count, self.f, self.xi, self.mu_re, self.mu_im, self.mpc, self.mpd, self.shape]

    def to(self, device):
        return PoleTable(self.n_min, self.n_step, self.l, self.cap,
                         *[t.to(device) for t in self.tensors()])


def modal_sweep_ws_bytes(l, i, n_min, n_max, n_step) -> int:
    b = C.c_size_t(0)
    call("ssi_modal_sweep_ws", l, i, n_min, n_max, n_step, C.byref(b))
    return b.value


def modal_sweep(U: torch.Tensor, S: torch.Tensor, l: int, i: int, n_min: int, n_max: int,
                n_step: int, dt: float, out: PoleTable | None = None,
                ws: torch.Tensor | None = None, check: bool = False) -> PoleTable:
    _require_cuda(U, S)
    if U.stride(0) != 1:
        raise ValueError("U must be column-major (as returned by rsvd)")
    tab = out if out is not None else PoleTable.empty(n_min, n_max, n_step, l, U.device)
    if ws is None:
        ws = _workspace(modal_sweep_ws_bytes(l, i, n_min, n_max, n_step), U.device)
    ct = tab.as_c()
    call("ssi_modal_sweep", _ptr(U), U.stride(1), _ptr(S), l, i, n_min, n_max, n_step, float(dt),
         C.byref(ct), _ptr(ws), ws.numel(), _stream())
    _check_device("ssi_modal_sweep", ws, check)
    return tab


@dataclass(frozen=True)
class Criteria:
    """Hard (xi_max, mpc_min, mpd_max; reading A-17) and soft (alpha_f, alpha_xi, alpha_mac;
    readings A-18..A-21) stabilization criteria of ssi_stab3d. The default is the paper's 10-DOF
    3D set; the presets below are the sets the paper states."""
    xi_max: float = 0.10
    mpc_min: float = 0.60
    mpd_max: float = 0.50
    alpha_f: float = 0.01
    alpha_xi: float = 0.03
    alpha_mac: float = 0.02


# The paper's criteria sets (HC: xi > 10 %, MPC <= 60 %, MPD >= 50 % discarded everywhere).
#  - 2D order-axis SC of the rank study (Fig. 3): 2 %, 2 %, 5 % (§3.1.1)
#  - 10-DOF 3D diagram: alpha_f, alpha_xi, alpha_MAC = 1 %, 3 %, 2 % (§3.1.3)
#  - San Faustino 2D continuous identification: 2 %, 3 %, 2 % (§3.2.2)
#  - San Faustino 3D diagram: 2.5 %, 5 %, 3 % (§3.2.2)
CRITERIA_2D_RANK_STUDY = Criteria(alpha_f=0.02, alpha_xi=0.02, alpha_mac=0.05)
CRITERIA_10DOF_3D = Criteria(alpha_f=0.01, alpha_xi=0.03, alpha_mac=0.02)
CRITERIA_BRIDGE_2D = Criteria(alpha_f=0.02, alpha_xi=0.03, alpha_mac=0.02)
CRITERIA_BRIDGE_3D = Criteria(alpha_f=0.025, alpha_xi=0.05, alpha_mac=0.03)


def stab3d(tables: list, crit: Criteria):
    """flags [G][O][cap] uint8 (0 rejected, 1 new, 2 stable) and stable_count [G][O]."""
    G = len(tables)
    t0 = tables[0]
    dev = t0.count.device
    flags = torch.zeros((G, t0.n_orders, t0.cap), dtype=torch.uint8, device=dev)
    counts = torch.zeros((G, t0.n_orders), dtype=torch.int32, device=dev)
    arr = (PoleTableC * G)(*[t.as_c() for t in tables])
    cc = CriteriaC(crit.xi_max, crit.mpc_min, crit.mpd_max, crit.alpha_f, crit.alpha_xi, crit.alpha_mac)
    call("ssi_stab3d", arr, G, C.byref(cc), _ptr(flags), _ptr(counts), _stream())
    return flags, counts


# ------------------------------------------------------------------ NEXT-2: clustering + tracking
@dataclass
class Clustering:
    """Result of cluster3d (device tensors; readings C-1..C-4, include/ssi.h NEXT-2).
    pole_idx [n_stable][3] (lag, order index, slot) of the stable poles; X [n_stable][5] stage-I
    features; U [n_stable][2] fuzzy memberships; V [2][5] centroids; phys: index of the possibly-
    physical FCM cluster; retained [n_retained] rows of pole_idx kept for stage II; labels
    [n_retained] cluster of each retained pole (-1: dropped); f, xi, size, medoid (retained row),
    shape [K][l][2] of the K clusters ordered by (f, first member); merges_ab / merges_h: the
    average-linkage merges at height <= cutoff."""
    n_stable: int
    n_retained: int
    fcm_iters: int
    phys: int
    n_components: int
    n_merges: int
    overflow: int
    pole_idx: torch.Tensor
    X: torch.Tensor
    U: torch.Tensor
    V: torch.Tensor
    retained: torch.Tensor
    labels: torch.Tensor
    f: torch.Tensor
    xi: torch.Tensor
    size: torch.Tensor
    medoid: torch.Tensor
    shape: torch.Tensor
    merges_ab: torch.Tensor
    merges_h: torch.Tensor

    @property
    def n_clusters(self):
        return int(self.f.shape[0])


def _table_array(tables):
    if not 1 <= len(tables) <= _lib.SSI_MAX_LAGS:
        raise ValueError(f"1..{_lib.SSI_MAX_LAGS} pole tables expected")
    return (PoleTableC * len(tables))(*[t.as_c() for t in tables])


def cluster3d(tables: list, flags: torch.Tensor, crit: Criteria, cutoff: float = 0.10, min_size: int = 1,
              max_clusters: int = 4096, fcm_tol: float = 1e-10, fcm_max_iter: int = 1000,
              check: bool = True) -> Clustering:
    """Two-stage clustering of the stable poles (flag 2) of the diagram `tables` (lags in increasing
    i) with `flags` from stab3d(tables, crit) (ssi_cluster_stage1 + ssi_cluster_stage2). Stage I
    reads back the retained-pole count (one synchronisation) to size stage II's O(n^2) workspace."""
    t0 = tables[0]
    dev = t0.count.device
    _require_cuda(flags)
    arr = _table_array(tables)
    G = len(tables)
    cc = CriteriaC(crit.xi_max, crit.mpc_min, crit.mpd_max, crit.alpha_f, crit.alpha_xi, crit.alpha_mac)
    max_poles = max(1, G * t0.n_orders * t0.cap)
    pole_idx = torch.empty((max_poles, 3), dtype=torch.int32, device=dev)
    X = torch.empty((max_poles, 5), dtype=torch.float64, device=dev)
    U = torch.empty((max_poles, 2), dtype=torch.float64, device=dev)
    retained = torch.empty(max_poles, dtype=torch.int32, device=dev)
    info = torch.zeros(C.sizeof(ClusterInfoC), dtype=torch.uint8, device=dev)
    b = C.c_size_t(0)
    call("ssi_cluster_stage1_ws", G, t0.n_orders, C.byref(b))
    ws1 = _workspace(b.value, dev)
    call("ssi_cluster_stage1", arr, G, C.byref(cc), _ptr(flags), max_poles, float(fcm_tol), int(fcm_max_iter),
         _ptr(pole_idx), _ptr(X), _ptr(U), _ptr(retained), _ptr(info), _ptr(ws1), ws1.numel(), _stream())
    if check:
        _check_device("ssi_cluster_stage1", ws1, True)
    h = ClusterInfoC.from_buffer_copy(bytes(info.cpu().numpy()))
    n_ret = h.n_retained
    call("ssi_cluster_stage2_ws", n_ret, t0.l, C.byref(b))
    ws2 = _workspace(b.value, dev)
    labels = torch.empty(max(n_ret, 1), dtype=torch.int32, device=dev)
    cl_f = torch.empty(max_clusters, dtype=torch.float64, device=dev)
    cl_xi = torch.empty_like(cl_f)
    cl_size = torch.empty(max_clusters, dtype=torch.int32, device=dev)
    cl_med = torch.empty_like(cl_size)
    cl_shape = torch.empty((max_clusters, t0.l, 2), dtype=torch.float64, device=dev)
    m_ab = torch.empty((max(n_ret, 1), 2), dtype=torch.int32, device=dev)
    m_h = torch.empty(max(n_ret, 1), dtype=torch.float64, device=dev)
    call("ssi_cluster_stage2", arr, G, _ptr(pole_idx), _ptr(retained), n_ret, float(cutoff), int(min_size),
         int(max_clusters), _ptr(labels), _ptr(cl_f), _ptr(cl_xi), _ptr(cl_size), _ptr(cl_med), _ptr(cl_shape),
         _ptr(m_ab), _ptr(m_h), _ptr(info), _ptr(ws2), ws2.numel(), _stream())
    if check:
        _check_device("ssi_cluster_stage2", ws2, True)
    h = ClusterInfoC.from_buffer_copy(bytes(info.cpu().numpy()))
    K = min(h.n_clusters, max_clusters)
    ns = min(h.n_stable, max_poles)
    return Clustering(h.n_stable, n_ret, h.fcm_iters, h.phys, h.n_components, h.n_merges, h.overflow,
                      pole_idx[:ns], X[:ns], U[:ns], torch.tensor(list(h.V), dtype=torch.float64).view(2, 5),
                      retained[:n_ret], labels[:n_ret], cl_f[:K], cl_xi[:K], cl_size[:K], cl_med[:K],
                      cl_shape[:K], m_ab[:h.n_merges], m_h[:h.n_merges])


def track(ref_f: torch.Tensor, ref_shape: torch.Tensor, f: torch.Tensor, shape: torch.Tensor,
          count: torch.Tensor, df_max: float = 0.05, macd_max: float = 0.15):
    """Modal tracking (ssi_track, reading C-5): ref_f [R], ref_shape [R][l][2]; f [S][M],
    shape [S][M][l][2], count [S] int32 modes per session. Returns (match [S][R] int32 with the
    session mode assigned to each reference mode or -1, success [R] percentages)."""
    _require_cuda(ref_f, ref_shape, f, shape, count)
    R, l = ref_shape.shape[0], ref_shape.shape[1]
    S, M = f.shape
    for t in (ref_f, ref_shape, f, shape):
        if t.dtype != torch.float64 or not t.is_contiguous():
            raise ValueError("ref_f, ref_shape, f, shape must be contiguous FP64")
    if count.dtype != torch.int32 or shape.shape != (S, M, l, 2) or ref_shape.shape != (R, l, 2):
        raise ValueError("shape mismatch")
    match = torch.empty((S, R), dtype=torch.int32, device=f.device)
    success = torch.empty(R, dtype=torch.float64, device=f.device)
    call("ssi_track", _ptr(ref_f), _ptr(ref_shape), R, _ptr(f), _ptr(shape), _ptr(count), S, M, l,
         float(df_max), float(macd_max), _ptr(match), _ptr(success), _stream())
    return match, success


# ------------------------------------------------------------------ NEXT-4: preprocessing + generator
def rate_ratio(fs_in: float, fs_out: float):
    """(L, M) with fs_out / fs_in = L / M in lowest terms (integral rates in Hz)."""
    from fractions import Fraction
    fr = Fraction(int(round(fs_out)), int(round(fs_in)))
    return fr.numerator, fr.denominator


def preprocess_ws_bytes(N, l, L, order=8) -> int:
    b = C.c_size_t(0)
    call("ssi_preprocess_ws", N, l, L, order, C.byref(b))
    return b.value


def preprocess(Y: torch.Tensor, fs_in: float, fs_out: float, order: int = 8, rp_db: float = 0.05,
               fc_hz: float | None = None, out_dtype=torch.float64, out: torch.Tensor | None = None,
               ws: torch.Tensor | None = None) -> torch.Tensor:
    """ssi_preprocess (readings P-1..P-3): detrend, upsample by L, zero-phase Chebyshev-I low-pass
    (edge 0.8 fs_out / 2 unless fc_hz is given) at L fs_in, keep every M-th sample."""
    _require_cuda(Y)
    if Y.dim() != 2 or Y.stride(1) != 1:
        raise ValueError("Y must be [N][l] with unit channel stride")
    dt = {torch.float32: SSI_F32, torch.float64: SSI_F64}
    N, l = Y.shape
    L, M = rate_ratio(fs_in, fs_out)
    fc = 0.8 * fs_out / 2.0 if fc_hz is None else fc_hz
    n_out = (N * L) // M
    Z = out if out is not None else torch.empty((n_out, l), dtype=out_dtype, device=Y.device)
    if ws is None:
        ws = _workspace(preprocess_ws_bytes(N, l, L, order), Y.device)
    call("ssi_preprocess", _ptr(Y), dt[Y.dtype], N, l, Y.stride(0), float(fs_in), L, M, order, float(rp_db),
         float(fc), _ptr(Z), dt[Z.dtype], Z.stride(0), _ptr(ws), ws.numel(), _stream())
    return Z


def lowpass_design(order: int, rp_db: float, fc_hz: float, fs_hz: float, device="cuda") -> torch.Tensor:
    """Second-order sections [order/2][5] = (b0, b1, b2, a1, a2) of ssi_preprocess's filter."""
    sos = torch.empty((order // 2, 5), dtype=torch.float64, device=device)
    call("ssi_lowpass_design", order, float(rp_db), float(fc_hz), float(fs_hz), _ptr(sos), _stream())
    return sos


@dataclass(frozen=True)
class Frame:
    """Shear-type frame of PAPER.md:314 (defaults: the paper's 10-DOF case)."""
    n_dof: int = 10
    m: float = 100.0
    k: float = 5.0e6
    xi: float = 0.01
    mode_a: int = 1
    mode_b: int = 4


def frame_model(frame: Frame, fs: float, device="cuda"):
    """(A_d [2n][2n], B_d [2n][n], C_o [n][2n], (a, b)) computed by ssi_frame_model."""
    n = frame.n_dof
    z = lambda *s: torch.empty(s, dtype=torch.float64, device=device)
    Ad, Bd, Co, ab = z(2 * n, 2 * n), z(2 * n, n), z(n, 2 * n), z(2)
    call("ssi_frame_model", n, frame.m, frame.k, frame.xi, frame.mode_a, frame.mode_b, float(fs), _ptr(Ad), _ptr(Bd),
         _ptr(Co), _ptr(ab), _stream())
    return Ad, Bd, Co, ab


def frame_simulate(N: int, fs: float, snr_db: float, seed: int, stream_id: int = 0, frame: Frame = Frame(),
                   n_burn: int | None = None, dtype=torch.float64, device="cuda", with_clean: bool = False):
    """ssi_frame_simulate (readings F-1..F-4): an [N][n_dof] acceleration record of the frame at fs Hz
    (burn-in 10 s unless n_burn is given); with_clean also returns the noise-free outputs."""
    n = frame.n_dof
    nb = int(round(10.0 * fs)) if n_burn is None else n_burn
    Y = torch.empty((N, n), dtype=dtype, device=device)
    clean = torch.empty((N, n), dtype=torch.float64, device=device) if with_clean else None
    b = C.c_size_t(0)
    call("ssi_frame_simulate_ws", n, N, nb, C.byref(b))
    ws = _workspace(b.value, device)
    call("ssi_frame_simulate", n, frame.m, frame.k, frame.xi, frame.mode_a, frame.mode_b, float(fs), N, nb,
         float(snr_db), C.c_uint64(seed), C.c_uint64(stream_id), _ptr(Y),
         {torch.float32: SSI_F32, torch.float64: SSI_F64}[dtype], Y.stride(0),
         _ptr(clean) if clean is not None else None, _ptr(ws), ws.numel(), _stream())
    return (Y, clean) if with_clean else Y
