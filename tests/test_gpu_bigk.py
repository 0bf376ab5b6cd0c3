"""Sketch widths above one SM (-m gpu): the paper's own rank rule k = ⌈k̄(T) % · T⌉ with
k̄(T) = max{30 − 0.00156 T; 25} % (Eq. empirical_formula) in the regime the
paper reports for the bridge ("Toeplitz matrix of 11400"): at T = 2880 (c2) k = 735,
at T = 11520 (c3) k = 2880 — Algorithm 1 verbatim (q = p = 0). These k run the
blocked whole-GPU Cholesky / triangular solve and the block one-sided Jacobi of linalg_big.cu.
GPU vs oracle (Householder QR + dgesdd) with the same Philox sketch."""
import numpy as np
import pytest

import oracle
import synth
from tests.parity import gpu_cells, compare_tables

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.fixture(scope="module")
def api():
    from paper_2411_05510_b200 import api, build
    build.build()
    return api


def _svd_parity(U, S, Uo, So, n, k):
    rel = np.abs(S[:n] - So[:n]) / So[:n]
    print(f"leading {n}: max rel dsigma {rel.max():.2e}; all {k}: max |dsigma|/sigma_1 "
          f"{np.abs(S[:k] - So[:k]).max() / So[0]:.2e}")
    assert rel.max() <= 1e-5                                     # contract
    assert rel.max() <= 1e-9                                     # internal FP64 tripwire
    assert np.abs(S[:k] - So[:k]).max() <= 1e-11 * So[0]         # every sigma of the k x k factor
    np.testing.assert_allclose(U.T @ U, np.eye(n), atol=1e-10)
    gap = np.minimum(np.abs(np.diff(So[:n + 1]))[:n], np.r_[np.inf, np.abs(np.diff(So[:n]))]) / So[0]
    d = np.abs(np.sum(U * Uo, axis=0))
    assert np.all(d[gap > 1e-6] > 1 - 1e-6)


@pytest.fixture(scope="module")
def c2_big():
    cfg = synth.config("c2")
    Y, _ = synth.make_record(cfg)
    m = cfg.m
    k = oracle.sample_count(oracle.min_rank_percent(m), m)
    assert k == 735
    R = oracle.covariances(Y, 2 * cfg.i - 1)
    U, S, _ = oracle.rsvd(oracle.toeplitz(R, cfg.i), k, 0, cfg.philox_key, cfg.i, cfg.n_max)
    cells = oracle.modal_sweep(U, S, cfg.l, cfg.i, cfg.orders, cfg.dt)
    return cfg, Y, k, R, U, S, cells


def test_c2_rank_rule_explicit_t(api, c2_big):
    cfg, _, k, R, Uo, So, _ = c2_big
    U, S = api.rsvd(api.toeplitz(_dev(R), cfg.i), k, 0, cfg.philox_key, cfg.i, cfg.n_max, check=True)
    _svd_parity(U.cpu().numpy(), S.cpu().numpy(), Uo, So, cfg.n_max, k)


def test_c2_rank_rule_structured_whole_chain(api, c2_big):
    """Record -> spectral covariances -> structured RSVD (k = 735, q = 0) -> modal sweep."""
    cfg, Y, k, _, Uo, So, cells = c2_big
    R = api.covariances(_dev(Y), 2 * cfg.i - 1, 1, "spectral", check=True)
    U, S = api.rsvd_toeplitz(R, cfg.i, k, 0, cfg.philox_key, cfg.i, cfg.n_max, check=True)
    _svd_parity(U.cpu().numpy(), S.cpu().numpy(), Uo, So, cfg.n_max, k)
    tab = api.modal_sweep(U, S, cfg.l, cfg.i, cfg.n_min, cfg.n_max, cfg.n_step, cfg.dt, check=True)
    flags, _ = oracle.stab3d([cells], oracle.SC_10DOF_3D, cfg.n_max // 2)
    st = compare_tables(gpu_cells(tab), cells, flags[0])
    assert st["count_mismatch"] == []
    assert st["n_stable"] > 0
    assert st["max_df_stable"] <= 1e-5 and st["max_dxi_stable"] <= 1e-4


@pytest.mark.parametrize("m,k", [(1500, 1037), (700, 513), (1200, 1200)])
def test_big_k_random_operator(api, m, k):
    """Full-rank random T (orthogonal factors, singular values 1 .. 1e-3) at awkward widths (not
    multiples of the 16-column Jacobi blocks or the 64-column Cholesky panels; k = m: the sketch
    spans everything), q = 1."""
    rng = np.random.default_rng([m, k])
    Qa, _ = np.linalg.qr(rng.standard_normal((m, m)))
    Qb, _ = np.linalg.qr(rng.standard_normal((m, m)))
    T = (Qa * np.logspace(0, -3, m)) @ Qb.T
    Uo, So, _ = oracle.rsvd(T, k, 1, 77, 5, 50)
    U, S = api.rsvd(_dev(T), k, 1, 77, 5, 50, check=True)
    _svd_parity(U.cpu().numpy(), S.cpu().numpy(), Uo, So, 50, k)


def test_c3_rank_rule_full_size(api):
    """T = 11520 (the metric's record, i = 60): k̄ = 25 %, k = 2880, Algorithm 1 verbatim through
    the structured path; the leading 200 singular values / vectors and the k x k factor's spectrum
    against the oracle's dense RSVD with the same sketch."""
    cfg = synth.config("c3")
    Y, _ = synth.make_record(cfg)
    m = cfg.m
    k = oracle.sample_count(oracle.min_rank_percent(m), m)
    assert k == 2880
    R = oracle.covariances(Y, 2 * cfg.i - 1)
    Uo, So, _ = oracle.rsvd(oracle.toeplitz(R, cfg.i), k, 0, cfg.philox_key, cfg.i, cfg.n_max)
    U, S = api.rsvd_toeplitz(_dev(R), cfg.i, k, 0, cfg.philox_key, cfg.i, cfg.n_max, check=True)
    torch.cuda.synchronize()
    _svd_parity(U.cpu().numpy(), S.cpu().numpy(), Uo, So, cfg.n_max, k)


def test_bridge_record_2d_full_size(api):
    """The paper's bridge workload at its own sizes: a 2-hour 114-channel record,
    j_b = 76 (T = 8664), Algorithm 1 verbatim with k = 25 % of T = 2166, orders 250..400. GPU chain
    (covariances -> structured RSVD -> modal sweep) against the oracle chain on the same
    preprocessed record (uploaded from the GPU's preprocessing, itself parity-tested in
    test_gpu_next4.py: the oracle cannot run the 2-hour filter at 1 kHz in a test's time):
    singular values and the poles of a sample of orders."""
    from paper_2411_05510_b200 import drivers
    from synth.raw import make_bridge_raw
    from tests.parity import gpu_cells, compare_tables
    raw, modes = make_bridge_raw()
    P = drivers.bridge_params()
    Yd = api.preprocess(torch.from_numpy(raw).cuda(), 125.0, 40.0, out_dtype=torch.float32)
    Y = Yd.cpu().numpy()
    assert P.k == 2166 and Y.shape == (288000, 114)
    R = api.covariances(Yd, 2 * P.i - 1, 1, "spectral", check=True)
    U, S = api.rsvd_toeplitz(R, P.i, P.k, 0, P.seed, P.i, P.n_max, check=True)
    Ro = oracle.covariances(Y, 2 * P.i - 1)
    assert np.linalg.norm(R.cpu().numpy() - Ro) / np.linalg.norm(Ro) <= 1e-12
    Uo, So, _ = oracle.rsvd(oracle.toeplitz(Ro, P.i), P.k, 0, P.seed, P.i, P.n_max)
    _svd_parity(U.cpu().numpy(), S.cpu().numpy(), Uo, So, P.n_max, P.k)
    orders = [250, 300, 350, 400]
    cells = oracle.modal_sweep(Uo, So, P.l, P.i, orders, P.dt)
    for n, c in zip(orders, cells):
        tab = api.modal_sweep(U, S, P.l, P.i, n, n, 2, P.dt, check=True)
        st = compare_tables(gpu_cells(tab), [c])
        assert st["count_mismatch"] == [], n
        assert st["max_df_all"] <= 1e-6 and st["max_dxi_all"] <= 1e-5, (n, st)


def test_big_k_rank_deficient_sketch_takes_the_shifted_fallback(api):
    """k = 600 > 512 columns on an operator of rank 100: the first Cholesky breaks down, the
    blocked path's shifted CholeskyQR3 fallback runs (conditional launches), the call returns
    SSI_OK and the 100 nonzero singular values equal the full SVD's."""
    rng = np.random.default_rng(606)
    m, r = 1200, 100
    A = np.linalg.qr(rng.standard_normal((m, r)))[0] * np.logspace(0, -2, r)
    T = A @ np.linalg.qr(rng.standard_normal((m, r)))[0].T
    So = np.linalg.svd(T, compute_uv=False)
    U, S = api.rsvd(_dev(T), 600, 0, 9, 1, 50, check=True)          # raises on a device failure
    S = S.cpu().numpy()
    np.testing.assert_allclose(S[:r], So[:r], rtol=1e-11)
    assert np.abs(S[r:]).max() <= 1e-10 * So[0]


def test_full_svd_as_k_equal_T_on_the_e3_frame(api):
    """The classical CoV-SSI decomposition (Eq. 8) is the same path with the
    sketch spanning all of T (k = T = 1890, q = 0): every singular value against the oracle's
    dgesdd, and the leading 30 singular vectors (E3 setting, Table 1 frame)."""
    from synth.records import _simulate
    from tests.analytic import shear_frame_modes
    modes = shear_frame_modes(200.0)
    Y = _simulate(modes, 60000, 0.1, np.random.default_rng([27, 0xE3]))
    R = oracle.covariances(Y, 2 * 189 - 1)
    T = oracle.toeplitz(R, 189)
    Uo, So = oracle.full_svd(T)
    U, S = api.rsvd_toeplitz(_dev(R), 189, 1890, 0, 1, 189, 30, check=True)
    S = S.cpu().numpy()
    assert np.abs(S - So).max() <= 1e-12 * So[0]
    np.testing.assert_allclose(S[:30], So[:30], rtol=1e-10)
    d = np.abs(np.sum(U.cpu().numpy() * Uo[:, :30], axis=0))
    gap = np.minimum(np.abs(np.diff(So[:31]))[:30], np.r_[np.inf, np.abs(np.diff(So[:30]))]) / So[0]
    assert np.all(d[gap > 1e-6] > 1 - 1e-8)
