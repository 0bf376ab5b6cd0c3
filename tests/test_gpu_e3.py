"""E3 workload: Algorithm 1 verbatim (q = p = 0) on
the 10-DOF shear frame of Table 1, with the sketch width from the paper's own
rank rule k = ⌈k̄(T) % · T⌉ (Eq. empirical_formula): j_b = 189, T = 1890 rows,
k = 512, orders 2..30 step 2, fs = 200 Hz, 5 min, SNR 20 dB. This is the "tall-and-wide" regime:
k = 512 > 224 runs the generic GEMM, packed Cholesky and 16-column-per-lane Jacobi kernels
instead of the c3 ones. GPU vs oracle through the C ABI; tolerances as in test_gpu_parity.py."""
import numpy as np
import pytest

import oracle
from synth.records import _simulate
from tests.analytic import shear_frame_modes
from tests.parity import gpu_cells, compare_tables

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FS, N, L, I, SEED = 200.0, 60000, 10, 189, 0xE3
ORDERS = list(range(2, 31, 2))


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.fixture(scope="module")
def e3():
    from paper_2411_05510_b200 import api, build
    build.build()
    modes = shear_frame_modes(FS)
    Y = _simulate(modes, N, 0.1, np.random.default_rng([27, 0xE3]))    # SNR 20 dB (amplitude 10 %)
    m = L * I
    k = oracle.sample_count(oracle.min_rank_percent(m), m)
    assert k == 512                                                    # PAPER.md:391 (k = 512)
    R = oracle.covariances(Y, 2 * I - 1)
    U, S, _ = oracle.rsvd(oracle.toeplitz(R, I), k, 0, SEED, I, ORDERS[-1])
    cells = oracle.modal_sweep(U, S, L, I, ORDERS, 1.0 / FS)
    return api, modes, Y, k, R, U, S, cells


def _svd_parity(U, S, Uo, So, n):
    rel = np.abs(S[:n] - So[:n]) / So[:n]
    assert rel.max() <= 1e-5                  # contract: leading singular values
    assert rel.max() <= 1e-9                  # internal FP64 tripwire
    np.testing.assert_allclose(U.T @ U, np.eye(n), atol=1e-10)
    gap = np.minimum(np.abs(np.diff(So[:n + 1]))[:n], np.r_[np.inf, np.abs(np.diff(So[:n]))]) / So[0]
    d = np.abs(np.sum(U * Uo, axis=0))
    assert np.all(d[gap > 1e-6] > 1 - 1e-6)


def test_e3_covariances_spectral(e3):
    api, _, Y, _, R, *_ = e3
    Rg = api.covariances(_dev(Y), 2 * I - 1, 1, "spectral", check=True).cpu().numpy()
    rel = np.linalg.norm(Rg - R) / np.linalg.norm(R)
    assert rel <= 1e-6                        # contract
    assert rel <= 1e-12                       # internal FP64 tripwire


def test_e3_algorithm1_verbatim_explicit_t(e3):
    api, _, _, k, R, Uo, So, _ = e3
    T = api.toeplitz(_dev(R), I)
    U, S = api.rsvd(T, k, 0, SEED, I, ORDERS[-1], check=True)
    _svd_parity(U.cpu().numpy(), S.cpu().numpy(), Uo, So, ORDERS[-1])


def test_e3_algorithm1_verbatim_structured(e3):
    api, _, _, k, R, Uo, So, _ = e3
    U, S = api.rsvd_toeplitz(_dev(R), I, k, 0, SEED, I, ORDERS[-1], check=True)
    _svd_parity(U.cpu().numpy(), S.cpu().numpy(), Uo, So, ORDERS[-1])


def test_e3_whole_chain_and_model_recovery(e3):
    """Record in HBM → spectral covariances → structured RSVD (k = 512, q = 0) → modal sweep, vs
    the oracle chain; then the identified order-30 poles against the shear frame's exact modes."""
    api, modes, Y, k, _, _, _, cells = e3
    R = api.covariances(_dev(Y), 2 * I - 1, 1, "spectral", check=True)
    U, S = api.rsvd_toeplitz(R, I, k, 0, SEED, I, ORDERS[-1], check=True)
    tab = api.modal_sweep(U, S, L, I, ORDERS[0], ORDERS[-1], 2, 1.0 / FS, check=True)
    flags, _ = oracle.stab3d([cells], oracle.SC_10DOF_3D, len(ORDERS))
    g = gpu_cells(tab)
    st = compare_tables(g, cells, flags[0])
    assert st["count_mismatch"] == []                                       # contract
    assert st["n_stable"] > 0
    assert st["max_df_stable"] <= 1e-5 and st["max_dxi_stable"] <= 1e-4    # contract
    f_id = np.array([p.f for p in g[-1].poles])
    for f in modes.f:                         # every one of the 10 modes within 1 % at n = 30
        assert np.min(np.abs(f_id - f) / f) < 0.01
