"""GPU tests of the round-2 boundary additions (-m gpu), all through the C ABI:

* the shifted-CholeskyQR3 fallback of the RSVD's QR (A5; "qr(Y,0)") on a
  sketch wider than the rank of T — the analytic c1 Toeplitz has rank exactly 2M = 6
  (north star: "in the noise-free limit T has rank 2·(number of modes)"), so k = 8 and k = 40
  make every Gram matrix of the RSVD singular;
* ssi_cov_normalize (reading A-6, 1/(N-k)) after time-sharded raw sums;
* ssi_cov_spectral_phases (measurement entry point) reproducing ssi_covariances bit for bit;
* synchronous rejection of k > 4096 (kBigMaxK) before any launch (ssi.h conventions);
* the multi-rank drivers (time-sharded covariances + all-reduce + on-device normalisation,
  LPT lags, one packed all_gather, ssi_stab3d; round-robin record batch) run as two processes
  on one GPU over gloo (host-staged collectives: no kernel of one rank waits on the other)
  against world = 1.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from tests.analytic import exact_covariances

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ssi():
    from paper_2411_05510_b200 import api, drivers, build
    build.build()
    return api, drivers


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


# ------------------------------------------------------------------ A5 breakdown fallback
@pytest.mark.parametrize("k", [8, 40])
@pytest.mark.parametrize("q", [0, 2])
@pytest.mark.parametrize("structured", [False, True])
def test_rsvd_sketch_wider_than_rank(ssi, k, q, structured):
    """k > rank(T) = 6: sigma_1..6 equal the full SVD's within 1e-12, the rest are at the
    rounding floor, the leading 6 singular vectors span the full SVD's, status stays SSI_OK."""
    api, _ = ssi
    cfg = synth.config("c1")
    R = exact_covariances(synth.make_modes(cfg), 2 * cfg.i - 1)
    T = oracle.toeplitz(R, cfg.i)
    Uf, Sf, _ = np.linalg.svd(T)
    assert Sf[6] / Sf[0] < 1e-14                 # rank 6 (pin P3)
    n_keep = min(k, 30)
    if structured:
        U, S = api.rsvd_toeplitz(_dev(R), cfg.i, k, q, 11, 3, n_keep, check=True)
    else:
        U, S = api.rsvd(_dev(T), k, q, 11, 3, n_keep, check=True)
    U, S = U.cpu().numpy(), S.cpu().numpy()
    np.testing.assert_allclose(S[:6], Sf[:6], rtol=1e-12)
    assert np.all(S[6:] <= 1e-12 * S[0])
    P = Uf[:, :6] @ Uf[:, :6].T                  # the signal subspace is captured exactly
    np.testing.assert_allclose(P @ U[:, :6], U[:, :6], atol=1e-10)
    np.testing.assert_allclose(U[:, :6].T @ U[:, :6], np.eye(6), atol=1e-10)
    Uo, So, _ = oracle.rsvd(T, k, q, 11, 3, n_keep)   # oracle (Householder QR) agrees
    np.testing.assert_allclose(S[:6], So[:6], rtol=1e-12)


def test_modal_sweep_after_rank_deficient_rsvd(ssi):
    """The poles of the analytic T at n = 2M = 6 are the generator's (pin P4) also when the
    sketch (k = 40) is wider than the rank; orders above the rank report count = -1."""
    api, _ = ssi
    cfg = synth.config("c1")
    modes = synth.make_modes(cfg)
    R = exact_covariances(modes, 2 * cfg.i - 1)
    U, S = api.rsvd_toeplitz(_dev(R), cfg.i, 40, 2, 11, 3, 30, check=True)
    tab = api.modal_sweep(U, S, cfg.l, cfg.i, 2, 30, 2, cfg.dt, check=True)
    cnt = tab.count.cpu().numpy()
    assert cnt[2] == 3                            # order 6: three conjugate pairs
    assert np.all(cnt[3:] == -1)                  # sigma_n < 1e-12 sigma_1 above the rank
    f = np.sort(tab.f.cpu().numpy()[2, :3])
    np.testing.assert_allclose(f, np.sort(modes.f), rtol=1e-9)


def test_rsvd_k_above_4096_rejected_before_any_launch(ssi):
    api, _ = ssi
    from paper_2411_05510_b200 import _lib
    lib = _lib.get()
    l, i, k = 64, 70, 4097
    R = torch.zeros((2 * i - 1, l, l), dtype=torch.float64, device="cuda")
    U = torch.full((k * l * i,), -7.0, dtype=torch.float64, device="cuda")
    S = torch.full((k,), -7.0, dtype=torch.float64, device="cuda")
    ws = torch.full((1 << 20,), 0x55, dtype=torch.uint8, device="cuda")
    sz = C.c_size_t(0)
    assert lib.ssi_rsvd_toeplitz_ws(l, i, k, k, C.byref(sz)) == 1
    assert lib.ssi_rsvd_ws(l * i, k, k, C.byref(sz)) == 1
    code = lib.ssi_rsvd_toeplitz(C.c_void_p(R.data_ptr()), l, i, k, 1, C.c_uint64(1), C.c_uint64(1), k,
                                 C.c_void_p(U.data_ptr()), l * i, C.c_void_p(S.data_ptr()),
                                 C.c_void_p(ws.data_ptr()), ws.numel(), None)
    assert code == 1 and b"4096" in lib.ssi_last_error()
    torch.cuda.synchronize()
    assert torch.all(U == -7.0) and torch.all(S == -7.0) and torch.all(ws == 0x55)


# ------------------------------------------------------------------ A1 normalisation + phases
@pytest.mark.parametrize("mode", ["spectral", "fp64"])
def test_cov_normalize_after_time_shards(ssi, mode):
    api, _ = ssi
    cfg = synth.config("c2")
    Y, _ = synth.make_record(cfg, N=40000)
    L = 2 * cfg.i - 1
    Yd = _dev(Y)
    N = Y.shape[0]
    S = None
    for tb, te in ((0, 13001), (13001, 27000), (27000, N)):
        part = api.covariances(Yd, L, 1, mode, t_begin=tb, t_end=te, normalize=False, check=True)
        S = part if S is None else S + part
    R = api.cov_normalize(S, N, 1).cpu().numpy()
    Ro = oracle.covariances(Y, L)
    assert np.linalg.norm(R - Ro) / np.linalg.norm(Ro) <= 1e-12
    # lag_lo > 1 and the synchronous checks
    S2 = api.covariances(Yd, 9, 4, mode, normalize=False)
    np.testing.assert_allclose(api.cov_normalize(S2, N, 4).cpu().numpy(), Ro[3:9], rtol=1e-11, atol=1e-14)
    from paper_2411_05510_b200 import _lib
    with pytest.raises(_lib.SSIError):
        api.cov_normalize(S2, 9, 4)                # lag 9 >= N


def test_cov_spectral_phases_reproduce_the_full_call(ssi):
    api, _ = ssi
    cfg = synth.config("c2")
    Y, _ = synth.make_record(cfg)
    L = 2 * cfg.i - 1
    Yd = _dev(Y)
    ws = api._workspace(api.covariances_ws_bytes(Y.shape[0], cfg.l, L, 1, "spectral"), Yd.device)
    R = api.covariances(Yd, L, 1, "spectral", ws=ws, check=True).clone()
    out = torch.empty_like(R)
    api.cov_spectral_phases(Yd, L, 7, out, ws)
    assert torch.equal(out, R)
    out.zero_()
    api.cov_spectral_phases(Yd, L, 2 | 4, out, ws)   # product + inverse on the kept spectra
    assert torch.equal(out, R)


# ------------------------------------------------------------------ multi-rank drivers
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


LAGS = (24, 28, 32)


def _params():
    from paper_2411_05510_b200 import drivers
    cfg = synth.config("c2")
    return cfg, drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=60, p=20, q=cfg.q, fs=cfg.fs,
                                    seed=cfg.philox_key)


def _host_tables(tabs):
    return {int(k): [x.cpu().numpy() for x in t.tensors()] for k, t in tabs.items()}


def _world_job(rank, world, port, q):
    import torch.distributed as dist
    from paper_2411_05510_b200 import api, drivers
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg, P = _params()
        Y, _ = synth.make_record(cfg, N=60000)
        Yd = _dev(Y)
        tabs, flags, counts, cl = drivers.identify_3d(Yd, P, LAGS, api.CRITERIA_BRIDGE_3D, rank=rank, world=world)
        recs = [_dev(synth.make_record(synth.config("c2", seed=cfg.seed + 7 * r), N=20000)[0]) for r in range(3)]
        btabs = drivers.record_batch(recs, P, rank, world, n_streams=2)
        match, succ, _, _ = drivers.track_campaign([btabs[j] for j in range(3)], api.CRITERIA_BRIDGE_3D)
        clus = (cl.labels.cpu().numpy(), cl.f.cpu().numpy(), cl.size.cpu().numpy())
        if world > 1 and rank == 0:
            # a world = 1 call on one rank inside the process group (bench.py's rank-0 legs) must
            # run no collective (the other rank never joins one): it equals the world = 1 sweep
            solo = drivers.lag_sweep_3d(Yd, P, LAGS, api.CRITERIA_BRIDGE_3D, rank=0, world=1)[2]
            assert torch.equal(solo.cpu(), drivers.lag_sweep_3d(Yd, P, LAGS, api.CRITERIA_BRIDGE_3D)[2].cpu())
        q.put((rank, (_host_tables(tabs), flags.cpu().numpy(), counts.cpu().numpy(), _host_tables(btabs), clus,
                      match.cpu().numpy())))
    finally:
        if world > 1:
            dist.destroy_process_group()


def _run_world(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_world_job, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


def test_two_ranks_match_one_rank(ssi):
    """world = 2 (two processes on one GPU, gloo) vs world = 1: the lag sweep's tables agree to
    FP64 rounding of the re-associated covariance sum (1e-9 relative on every pole's f and xi,
    identical pole counts, stab3d flags and stable counts) and so does the clustering of the
    gathered diagram (identical memberships); the record batch, whose records are independent, is
    bit-identical, and so is its tracking; both ranks hold identical gathered tables."""
    one = _run_world(1)[0]
    two = _run_world(2)
    for r in (0, 1):
        t1, f1, c1, b1, k1, m1 = one
        t2, f2, c2, b2, k2, m2 = two[r]
        assert np.array_equal(k1[0], k2[0]) and np.array_equal(k1[2], k2[2])       # memberships, sizes
        np.testing.assert_allclose(k2[1], k1[1], rtol=1e-9)                         # cluster f
        assert np.array_equal(m1, m2)
        assert sorted(t2) == sorted(t1) == list(LAGS)
        for lag in LAGS:
            cnt1, cnt2 = t1[lag][0], t2[lag][0]
            assert np.array_equal(cnt1, cnt2)
            for a, b in zip(t1[lag][1:3], t2[lag][1:3]):          # f, xi
                np.testing.assert_allclose(b, a, rtol=1e-9, atol=1e-12)
        assert np.array_equal(f1, f2) and np.array_equal(c1, c2)
        assert sorted(b2) == sorted(b1) == [0, 1, 2]
        for key in b1:
            for a, b in zip(b1[key], b2[key]):
                assert np.array_equal(a, b)
    for lag in LAGS:                                              # ranks agree bit for bit
        for a, b in zip(two[0][0][lag], two[1][0][lag]):
            assert np.array_equal(a, b)


def test_status_word_is_sticky_until_cleared(ssi):
    """A failure stays in the workspace's status word across later successful calls (so a
    pipeline that reuses the workspace sees it at its final check) until ssi_clear_status."""
    api, _ = ssi
    bad = np.ones((200, 4), np.float32)
    bad[37, 2] = np.nan
    good = np.random.default_rng(3).standard_normal((200, 4)).astype(np.float32)
    ws = api._workspace(api.covariances_ws_bytes(200, 4, 5, 1, "spectral"), "cuda")
    assert api.device_status(ws) == 0
    api.covariances(_dev(bad), 5, 1, "spectral", ws=ws)
    api.covariances(_dev(good), 5, 1, "spectral", ws=ws)
    assert api.device_status(ws) == 6
    api.clear_status(ws)
    api.covariances(_dev(good), 5, 1, "spectral", ws=ws)
    assert api.device_status(ws) == 0
