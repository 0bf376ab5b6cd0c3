"""GPU-vs-oracle parity through the C ABI (-m gpu). Tolerances are the north star's
(BASELINE.json): covariances rel. Frobenius 1e-6 (FP64 path), leading singular values
1e-5, frequencies 1e-5 relative and damping 1e-4 absolute for every oracle-stable pole,
bit-exact Philox words, Toeplitz copies and stabilization pole counts. Tighter internal
tripwires (FP64 everywhere) are asserted alongside and named as such."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle
import synth
from tests.parity import gpu_cells, compare_tables

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def ssi():
    from paper_2411_05510_b200 import api, drivers, build
    build.build()
    return api, drivers


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ------------------------------------------------------------------ A3 Philox / sketch
def test_philox_words_bit_exact_vs_oracle_and_curand(ssi):
    api, _ = ssi
    seed, sid, n = 0x5EED0003_12345678, (7 << 32) | 60, 100003
    w = api.philox_words(seed, sid, n).cpu().numpy().view(np.uint32)
    ref = oracle.philox_words(np.arange(n), seed, sid)
    assert np.array_equal(w, ref)
    so = os.path.join("/tmp", "curand_philox_ref.so")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-shared", "-Xcompiler", "-fPIC", "-o", so,
                           os.path.join(HERE, "cuda", "curand_philox_ref.cu")])
    lib = C.CDLL(so)
    out = torch.empty((n, 4), dtype=torch.int32, device="cuda")
    assert lib.curand_ref_words(C.c_uint64(seed), C.c_uint64(sid), C.c_int64(n), C.c_void_p(out.data_ptr())) == 0
    assert np.array_equal(out.cpu().numpy().view(np.uint32), w)


def test_gaussian_sketch_matches_oracle(ssi):
    api, _ = ssi
    for (m, k) in ((120, 40), (2881, 7), (1, 1)):
        om = api.gaussian_sketch(m, k, 0xABCDEF, 99).cpu().numpy()
        ref = oracle.gaussian_sketch(m, k, 0xABCDEF, 99)
        assert np.max(np.abs(om - ref)) <= 1e-13       # uniforms bit-exact; log/sincos ulps


# ------------------------------------------------------------------ A1 covariances
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_covariances_match_oracle(ssi, name):
    api, _ = ssi
    cfg = synth.config(name)
    Y, _ = synth.make_record(cfg)
    L = 2 * cfg.i - 1
    R = api.covariances(_dev(Y), L, check=True).cpu().numpy()
    Ro = oracle.covariances(Y, L)
    err = _rel(R, Ro)
    assert err <= 1e-6                        # contract (north star)
    assert err <= 1e-12                       # internal FP64 tripwire
    for k in range(L):                        # per-lag check catches N-k / tail bugs
        assert _rel(R[k], Ro[k]) <= 1e-11


def test_covariance_edge_cases(ssi):
    api, _ = ssi
    rng = np.random.default_rng(21)
    # ragged sizes, max lag = N-1, strided record (ldY > l), FP64 input
    for (N, l, lo, hi, dt) in ((1013, 7, 1, 40, np.float32), (50, 3, 1, 49, np.float64),
                               (3000, 65, 3, 17, np.float32), (129, 1, 1, 128, np.float64)):
        Y = rng.standard_normal((N, l)).astype(dt)
        R = api.covariances(_dev(Y), hi, lo, check=True).cpu().numpy()
        Ro = oracle.covariances(Y, hi, lo)
        np.testing.assert_allclose(R, Ro, rtol=1e-11, atol=1e-13)
    Ywide = rng.standard_normal((800, 12))
    Yd = _dev(Ywide)[:, :9]
    R = api.covariances(Yd, 11, check=True).cpu().numpy()
    np.testing.assert_allclose(R, oracle.covariances(Ywide[:, :9], 11), rtol=1e-11, atol=1e-13)


def test_covariance_time_shards_sum_to_full(ssi):
    """Raw shard sums (normalize=0) add up to the oracle's full sums (multi-GPU split)."""
    api, drivers = ssi
    rng = np.random.default_rng(22)
    Y = rng.standard_normal((5000, 10)).astype(np.float32)
    Yd = _dev(Y)
    tot = 0
    for tb, te in drivers.time_shards(5000, 3):
        tot = tot + api.covariances(Yd, 25, 1, t_begin=tb, t_end=te, normalize=False).cpu().numpy()
    np.testing.assert_allclose(tot, oracle.covariance_partial_sums(Y, 1, 25), rtol=1e-11, atol=1e-9)


def test_covariance_nonfinite_is_flagged(ssi):
    api, _ = ssi
    from paper_2411_05510_b200._lib import SSIError
    Y = np.ones((100, 4), np.float32)
    Y[37, 2] = np.nan
    with pytest.raises(SSIError) as e:
        api.covariances(_dev(Y), 5, check=True)
    assert e.value.code == 6


# ------------------------------------------------------------------ A1 spectral (NEXT-3)
def _rel_scale(R, Ro):
    """max over lags of ||R_k - Ro_k||_F relative to the largest ||Ro_k||_F: the segment
    cross-spectral path's rounding is relative to the record's energy, not to each lag."""
    scale = max(np.linalg.norm(Ro[k]) for k in range(Ro.shape[0]))
    return max(np.linalg.norm(R[k] - Ro[k]) for k in range(Ro.shape[0])) / scale


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_covariances_spectral_match_oracle(ssi, name):
    api, _ = ssi
    cfg = synth.config(name)
    Y, _ = synth.make_record(cfg)
    L = 2 * cfg.i - 1
    R = api.covariances(_dev(Y), L, mode="spectral", check=True).cpu().numpy()
    Ro = oracle.covariances(Y, L)
    assert _rel(R, Ro) <= 1e-6                # contract (north star)
    assert _rel(R, Ro) <= 1e-12               # internal FP64 tripwire
    assert _rel_scale(R, Ro) <= 1e-12
    if name == "c2":                          # c2 plans F = 1024 (fast kernel): its FP64-record branch
        assert api.cov_spectral_plan(cfg.N, cfg.l, L)[0] == 1024
        R64 = api.covariances(_dev(Y.astype(np.float64)), L, mode="spectral", check=True).cpu().numpy()
        assert _rel_scale(R64, Ro) <= 1e-12


def test_covariance_spectral_edge_cases(ssi):
    """Ragged / odd channel counts (padding channel), one channel, max lag = N-1 (segments of
    one sample), lag_lo > 1, FP64 and strided records, lags past one GEMM N tile (> 224)."""
    api, _ = ssi
    rng = np.random.default_rng(31)
    for (N, l, lo, hi, dt) in ((1013, 7, 1, 40, np.float32), (50, 3, 1, 49, np.float64),
                               (3000, 65, 3, 17, np.float32), (129, 1, 1, 128, np.float64),
                               (7000, 4, 1, 300, np.float32), (20000, 33, 5, 5, np.float64),
                               (30000, 6, 1, 1500, np.float32),           # F = 2048 (two-channel FFT CTAs)
                               (20000, 2, 1, 2000, np.float32)):          # lag_hi near the 2047 limit
        Y = rng.standard_normal((N, l)).astype(dt)
        R = api.covariances(_dev(Y), hi, lo, mode="spectral", check=True).cpu().numpy()
        Ro = oracle.covariances(Y, hi, lo)
        assert _rel_scale(R, Ro) <= 1e-12, (N, l, lo, hi)
    Ywide = rng.standard_normal((800, 12))
    Yd = _dev(Ywide)[:, :9]
    R = api.covariances(Yd, 11, mode="spectral", check=True).cpu().numpy()
    assert _rel_scale(R, oracle.covariances(Ywide[:, :9], 11)) <= 1e-12


def test_covariance_spectral_inverse_fft(ssi):
    """The F = 1024 inverse transform (spec_ifft1024_kernel): odd channel counts (padding channel,
    a partial last CTA of 8 elements), lag_lo > 1, and lags in every radix-4 output quarter
    (k >= 256, 512, 768), against the oracle's direct sums; normalised and raw sums."""
    api, _ = ssi
    rng = np.random.default_rng(35)
    for (N, l, lo, hi) in ((200000, 9, 3, 300), (100000, 6, 1, 600), (50000, 3, 1, 850),
                           (30000, 2, 1, 800), (200000, 11, 1, 119)):
        assert api.cov_spectral_plan(N, l, hi, lo)[0] == 1024, (N, l, lo, hi)
        Y = rng.standard_normal((N, l)).astype(np.float32)
        R = api.covariances(_dev(Y), hi, lo, mode="spectral", check=True).cpu().numpy()
        Ro = oracle.covariances(Y, hi, lo)
        assert _rel_scale(R, Ro) <= 1e-12, (N, l, lo, hi)
        S = api.covariances(_dev(Y), hi, lo, mode="spectral", normalize=False).cpu().numpy()
        So = oracle.covariance_partial_sums(Y, lo, hi)
        assert np.max(np.abs(S - So)) <= 1e-12 * np.max(np.abs(So)), (N, l, lo, hi)


def test_covariance_spectral_long_record_chunks(ssi):
    """A record long enough that its segments are processed in several chunks (the product
    accumulates over chunks in a fixed order), against the oracle."""
    api, _ = ssi
    N, l, hi = 1_200_000, 8, 60
    F, S = api.cov_spectral_plan(N, l, hi)
    assert S > 512                                   # more than one chunk of segments
    rng = np.random.default_rng(33)
    Y = rng.standard_normal((N, l)).astype(np.float32)
    R = api.covariances(_dev(Y), hi, mode="spectral", check=True).cpu().numpy()
    assert _rel_scale(R, oracle.covariances(Y, hi)) <= 1e-12


def test_covariance_spectral_time_shards_sum_to_full(ssi):
    api, drivers = ssi
    rng = np.random.default_rng(32)
    Y = rng.standard_normal((5000, 10)).astype(np.float32)
    Yd = _dev(Y)
    tot = 0
    for tb, te in list(drivers.time_shards(5000, 3)) + [(5000, 5000)]:   # + an empty shard
        tot = tot + api.covariances(Yd, 25, 1, mode="spectral", t_begin=tb, t_end=te,
                                    normalize=False).cpu().numpy()
    ref = oracle.covariance_partial_sums(Y, 1, 25)
    assert np.max(np.abs(tot - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_covariance_spectral_chunked_time_shards(ssi):
    """Time shards of a record whose segments span several chunks: the raw shard sums add up to
    the oracle's full sums (multi-GPU split of the spectral path)."""
    api, drivers = ssi
    N, l, hi = 600_000, 4, 100
    assert api.cov_spectral_plan(N, l, hi)[1] > 512
    rng = np.random.default_rng(34)
    Y = rng.standard_normal((N, l)).astype(np.float32)
    Yd = _dev(Y)
    tot = 0
    for tb, te in drivers.time_shards(N, 3):
        tot = tot + api.covariances(Yd, hi, 1, mode="spectral", t_begin=tb, t_end=te, normalize=False).cpu().numpy()
    ref = oracle.covariance_partial_sums(Y, 1, hi)
    assert np.max(np.abs(tot - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_covariance_spectral_nonfinite_is_flagged(ssi):
    api, _ = ssi
    from paper_2411_05510_b200._lib import SSIError
    Y = np.ones((100, 4), np.float32)
    Y[37, 2] = np.inf
    with pytest.raises(SSIError) as e:
        api.covariances(_dev(Y), 5, mode="spectral", check=True)
    assert e.value.code == 6


# ------------------------------------------------------------------ A2 Toeplitz
def test_toeplitz_bit_exact(ssi):
    api, _ = ssi
    rng = np.random.default_rng(23)
    for (l, i) in ((1, 2), (6, 20), (48, 7), (5, 33)):
        R = rng.standard_normal((2 * i - 1, l, l))
        T = api.toeplitz(_dev(R), i).cpu().numpy()
        assert np.array_equal(T, oracle.toeplitz(R, i))
    # padded leading dimension
    R = rng.standard_normal((9, 3, 3))
    out = torch.full((15, 17), -1.0, dtype=torch.float64, device="cuda")
    api.toeplitz(_dev(R), 5, out=out[:, :15])
    o = out.cpu().numpy()
    assert np.array_equal(o[:, :15], oracle.toeplitz(R, 5)) and np.all(o[:, 15:] == -1.0)


# ------------------------------------------------------------------ A3-A8 RSVD
def _rsvd_case(api, T, k, q, seed, sid, n_keep):
    U, S = api.rsvd(_dev(T), k, q, seed, sid, n_keep, check=True)
    Uo, So, _ = oracle.rsvd(T, k, q, seed, sid, n_keep)
    return U.cpu().numpy(), S.cpu().numpy(), Uo, So


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_rsvd_matches_oracle_same_sketch(ssi, name):
    api, _ = ssi
    cfg = synth.config(name)
    Y, _ = synth.make_record(cfg)
    T = oracle.toeplitz(oracle.covariances(Y, 2 * cfg.i - 1), cfg.i)
    U, S, Uo, So = _rsvd_case(api, T, cfg.k, cfg.q, cfg.philox_key, cfg.i, cfg.n_max)
    rel = np.abs(S[:cfg.n_max] - So[:cfg.n_max]) / So[:cfg.n_max]
    assert rel.max() <= 1e-5                  # contract: leading singular values
    assert rel.max() <= 1e-9                  # internal FP64 tripwire
    np.testing.assert_allclose(U.T @ U, np.eye(cfg.n_max), atol=1e-10)
    # columns up to sign, where the singular value is separated from its neighbours
    gap = np.minimum(np.abs(np.diff(So[:cfg.n_max + 1]))[:cfg.n_max],
                     np.r_[np.inf, np.abs(np.diff(So[:cfg.n_max]))]) / So[0]
    ok = gap > 1e-6
    d = np.abs(np.sum(U * Uo, axis=0))
    assert np.all(d[ok] > 1 - 1e-6)


def test_rsvd_edge_cases(ssi):
    api, _ = ssi
    cfg = synth.config("c1")
    modes = synth.make_modes(cfg)
    from tests.analytic import exact_covariances
    T = oracle.toeplitz(exact_covariances(modes, 2 * cfg.i - 1), cfg.i)
    Sf = oracle.full_svd(T)[1]
    # exact rank 6 captured for k >= 6, q = 0 (Algorithm 1 verbatim) and q = 2
    for q in (0, 2):
        _, S, _, So = _rsvd_case(api, T, 6, q, 5, 1, 6)
        np.testing.assert_allclose(S, Sf[:6], rtol=1e-12)
    # k = m (full width) and n_keep = 1
    rng = np.random.default_rng(24)
    A = rng.standard_normal((37, 37))
    U, S, Uo, So = _rsvd_case(api, A, 37, 1, 3, 3, 1)
    np.testing.assert_allclose(S, np.linalg.svd(A, compute_uv=False), rtol=1e-11)
    assert abs(abs(U[:, 0] @ Uo[:, 0]) - 1) < 1e-10


def test_rsvd_small_svd_widths(ssi):
    """The small SVD (ring Jacobi on an 8-CTA cluster, k <= 256; 16-CTA L2 variant above) at odd,
    even and tile-edge widths: a rank-r matrix with r <= k is captured exactly, so the leading r
    singular values equal the full SVD's and U's leading columns are orthonormal."""
    api, _ = ssi
    rng = np.random.default_rng(36)
    m = 600
    for k in (3, 5, 33, 64, 65, 127, 129, 255, 256, 257):
        r = min(k, 24)
        A = rng.standard_normal((m, r)) @ (rng.standard_normal((r, m)) * np.logspace(0, -3, m))
        Sf = np.linalg.svd(A, compute_uv=False)
        U, S, Uo, So = _rsvd_case(api, A, k, 1, 7, k, r)
        np.testing.assert_allclose(S[:r], Sf[:r], rtol=1e-9, err_msg=f"k = {k}")
        np.testing.assert_allclose(S[:r], So[:r], rtol=1e-9, err_msg=f"k = {k}")
        np.testing.assert_allclose(U.T @ U, np.eye(r), atol=1e-10, err_msg=f"k = {k}")


# ------------------------------------------------------------------ A2-A8 structured RSVD
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_rsvd_toeplitz_matches_oracle_same_sketch(ssi, name):
    """ssi_rsvd_toeplitz (T applied through its block structure, never formed) vs the oracle's
    RSVD of the explicit Toeplitz, same Philox sketch."""
    api, _ = ssi
    cfg = synth.config(name)
    Y, _ = synth.make_record(cfg)
    R = oracle.covariances(Y, 2 * cfg.i - 1)
    U, S = api.rsvd_toeplitz(_dev(R), cfg.i, cfg.k, cfg.q, cfg.philox_key, cfg.i, cfg.n_max, check=True)
    U, S = U.cpu().numpy(), S.cpu().numpy()
    Uo, So, _ = oracle.rsvd(oracle.toeplitz(R, cfg.i), cfg.k, cfg.q, cfg.philox_key, cfg.i, cfg.n_max)
    rel = np.abs(S[:cfg.n_max] - So[:cfg.n_max]) / So[:cfg.n_max]
    assert rel.max() <= 1e-5                  # contract: leading singular values
    assert rel.max() <= 1e-9                  # internal FP64 tripwire
    np.testing.assert_allclose(U.T @ U, np.eye(cfg.n_max), atol=1e-10)
    gap = np.minimum(np.abs(np.diff(So[:cfg.n_max + 1]))[:cfg.n_max],
                     np.r_[np.inf, np.abs(np.diff(So[:cfg.n_max]))]) / So[0]
    ok = gap > 1e-6
    d = np.abs(np.sum(U * Uo, axis=0))
    assert np.all(d[ok] > 1 - 1e-6)


def test_rsvd_toeplitz_edge_cases(ssi):
    """Ragged l (not a multiple of 32), i = 1 and 2 (DFT periods 1 and 3), l = 1, k > 224
    (column chunks of the batched product), full width k = m (exact SVD of T), exact rank."""
    api, _ = ssi
    rng = np.random.default_rng(31)
    for (l, i, k, q, n_keep) in ((5, 7, 12, 2, 10), (3, 1, 3, 1, 3), (4, 2, 8, 0, 8), (1, 9, 9, 2, 9),
                                 (3, 4, 12, 1, 12), (20, 15, 250, 1, 240), (33, 3, 40, 2, 30)):
        R = rng.standard_normal((2 * i - 1, l, l))
        U, S = api.rsvd_toeplitz(_dev(R), i, k, q, 77, i, n_keep, check=True)
        U, S = U.cpu().numpy(), S.cpu().numpy()
        T = oracle.toeplitz(R, i)
        Uo, So, _ = oracle.rsvd(T, k, q, 77, i, n_keep)
        np.testing.assert_allclose(S, So, rtol=1e-9, atol=1e-12 * So[0])
        if k == l * i:
            np.testing.assert_allclose(S, np.linalg.svd(T, compute_uv=False), rtol=1e-10, atol=1e-12 * So[0])
        np.testing.assert_allclose(U.T @ U, np.eye(n_keep), atol=1e-9)
    cfg = synth.config("c1")
    from tests.analytic import exact_covariances
    R = exact_covariances(synth.make_modes(cfg), 2 * cfg.i - 1)
    Sf = oracle.full_svd(oracle.toeplitz(R, cfg.i))[1]
    for q in (0, 2):
        _, S = api.rsvd_toeplitz(_dev(R), cfg.i, 6, q, 5, 1, 6, check=True)
        np.testing.assert_allclose(S.cpu().numpy(), Sf[:6], rtol=1e-12)


# ------------------------------------------------------------------ A9-A11 modal sweep
@pytest.fixture(scope="module")
def c2_chain():
    cfg = synth.config("c2")
    Y, _ = synth.make_record(cfg)
    R = oracle.covariances(Y, 2 * cfg.i - 1)
    T = oracle.toeplitz(R, cfg.i)
    U, S, _ = oracle.rsvd(T, cfg.k, cfg.q, cfg.philox_key, cfg.i, cfg.n_max)
    cells = oracle.modal_sweep(U, S, cfg.l, cfg.i, cfg.orders, cfg.dt)
    return cfg, Y, T, U, S, cells


@pytest.fixture(scope="module")
def c1_chain():
    cfg = synth.config("c1")
    Y, _ = synth.make_record(cfg)
    R = oracle.covariances(Y, 2 * cfg.i - 1)
    T = oracle.toeplitz(R, cfg.i)
    U, S, _ = oracle.rsvd(T, cfg.k, cfg.q, cfg.philox_key, cfg.i, cfg.n_max)
    cells = oracle.modal_sweep(U, S, cfg.l, cfg.i, cfg.orders, cfg.dt)
    return cfg, Y, T, U, S, cells


def _modal_parity(api, chain, crit):
    cfg, Y, T, U, S, cells = chain
    tab = api.modal_sweep(_dev(U.T).t(), _dev(S), cfg.l, cfg.i, cfg.n_min, cfg.n_max, cfg.n_step,
                          cfg.dt, check=True)
    flags, _ = oracle.stab3d([cells], crit, cfg.n_max // 2)
    st = compare_tables(gpu_cells(tab), cells, flags[0])
    return st


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_modal_sweep_matches_oracle(ssi, which, c1_chain, c2_chain):
    """Stage parity: both sides take the oracle's (U, S)."""
    api, _ = ssi
    chain = c1_chain if which == "c1" else c2_chain
    st = _modal_parity(api, chain, oracle.SC_10DOF_3D)
    assert st["count_mismatch"] == []                       # contract: pole counts exact
    assert st["n_stable"] > 0
    assert st["max_df_stable"] <= 1e-5 and st["max_dxi_stable"] <= 1e-4   # contract
    assert st["min_mac_stable"] >= 1 - 1e-6
    assert st["max_df_all"] <= 1e-7 and st["max_dxi_all"] <= 1e-7           # internal tripwire
    assert st["max_dmpc"] <= 1e-7 and st["max_dmpd"] <= 1e-7


def test_modal_rank_deficient_orders_reported(ssi):
    """Analytic T of rank 6: orders above the numerical rank come back count = -1 on both sides."""
    api, _ = ssi
    cfg = synth.config("c1")
    from tests.analytic import exact_covariances
    T = oracle.toeplitz(exact_covariances(synth.make_modes(cfg), 2 * cfg.i - 1), cfg.i)
    U, S = oracle.full_svd(T)
    tab = api.modal_sweep(_dev(U[:, :cfg.n_max].T).t(), _dev(S), cfg.l, cfg.i, 2, cfg.n_max, 2,
                          cfg.dt, check=True)
    cells = oracle.modal_sweep(U, S, cfg.l, cfg.i, cfg.orders, cfg.dt)
    g = gpu_cells(tab)
    assert [c.count for c in g] == [c.count for c in cells]
    assert g[2].count == 3 and g[-1].count == -1
    f, xi = synth.exact_poles(synth.make_modes(cfg))
    np.testing.assert_allclose([p.f for p in g[2].poles], f, rtol=1e-10)
    np.testing.assert_allclose([p.xi for p in g[2].poles], xi, atol=1e-10)


# ------------------------------------------------------------------ end to end + stab3d
@pytest.mark.parametrize("which", ["c1", "c2"])
def test_end_to_end_and_stab3d(ssi, which, c1_chain, c2_chain):
    """The whole GPU path (record in HBM -> pole table -> flags) vs the whole oracle path."""
    api, drivers = ssi
    cfg, Y, T, U, S, cells = c1_chain if which == "c1" else c2_chain
    P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs,
                            seed=cfg.philox_key)
    eng = drivers.Engine(P, cfg.N)
    tab = eng.identify(_dev(Y), stream_id=cfg.i)
    crit = oracle.SC_10DOF_3D
    flags_o, counts_o = oracle.stab3d([cells], crit, cfg.n_max // 2)
    st = compare_tables(gpu_cells(tab), cells, flags_o[0])
    assert st["count_mismatch"] == []
    assert st["max_df_stable"] <= 1e-5 and st["max_dxi_stable"] <= 1e-4
    flags, counts = api.stab3d([tab], api.Criteria(**crit.__dict__))
    assert np.array_equal(counts.cpu().numpy(), counts_o)
    fo = flags_o[0]
    fg = flags.cpu().numpy()[0]
    assert np.array_equal(fg, fo)


def test_stab3d_two_lags_vs_oracle(ssi, c2_chain):
    """3D soft criteria over two lags (i = 56, 60) of the c2 record."""
    api, drivers = ssi
    cfg, Y, *_ = c2_chain
    crit = oracle.SC_BRIDGE_3D
    R = oracle.covariances(Y, 2 * 60 - 1)
    tabs_o, tabs_g = [], []
    for i in (56, 60):
        T = oracle.toeplitz(R, i)
        U, S, _ = oracle.rsvd(T, cfg.k, cfg.q, cfg.philox_key, i, cfg.n_max)
        tabs_o.append(oracle.modal_sweep(U, S, cfg.l, i, cfg.orders, cfg.dt))
        tabs_g.append(api.modal_sweep(_dev(U.T).t(), _dev(S), cfg.l, i, cfg.n_min, cfg.n_max,
                                      cfg.n_step, cfg.dt, check=True))
    fo, co = oracle.stab3d(tabs_o, crit, cfg.n_max // 2)
    fg, cg = api.stab3d(tabs_g, api.Criteria(**crit.__dict__))
    assert np.array_equal(cg.cpu().numpy(), co)
    assert np.array_equal(fg.cpu().numpy(), fo)


@pytest.mark.parametrize("which", ["c2"])      # c1 (l = 6) has no int8x3 plan (test_abi.py)
def test_end_to_end_int8x3_covariances(ssi, which, c1_chain, c2_chain):
    """The int8x3 covariance path (exact int8 slices on tcgen05, `--cov int8x3`) carried through
    the whole chain to the pole table and stab3d flags, against the FP64 oracle path. Contract of
    the north star: pole counts exact, stable poles |df|/f <= 1e-5 and |dxi| <= 1e-4, flags and
    stable counts identical (int8x3 covariances are within ~4e-9 of FP64)."""
    api, drivers = ssi
    cfg, Y, T, U, S, cells = c1_chain if which == "c1" else c2_chain
    P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs,
                            seed=cfg.philox_key, cov_mode="int8x3")
    eng = drivers.Engine(P, cfg.N)
    tab = eng.identify(_dev(Y), stream_id=cfg.i)
    crit = oracle.SC_10DOF_3D
    flags_o, counts_o = oracle.stab3d([cells], crit, cfg.n_max // 2)
    st = compare_tables(gpu_cells(tab), cells, flags_o[0])
    print(f"{which} int8x3 end to end: stable {st['n_stable']}, max df {st['max_df_stable']:.1e}, "
          f"max dxi {st['max_dxi_stable']:.1e}")
    assert st["count_mismatch"] == []
    assert st["n_stable"] > 0
    assert st["max_df_stable"] <= 1e-5 and st["max_dxi_stable"] <= 1e-4
    flags, counts = api.stab3d([tab], api.Criteria(**crit.__dict__))
    assert np.array_equal(counts.cpu().numpy(), counts_o)
    assert np.array_equal(flags.cpu().numpy()[0], flags_o[0])
