"""NEXT-2 GPU parity (-m gpu): two-stage clustering (ssi_cluster_stage1 / _stage2) and modal
tracking (ssi_track) against oracle/cluster.py and oracle/track.py on the same inputs.

Inputs come from synth/ (seeded synthetic diagrams, synth/poles.py) or from the oracle's own
identification of a synth record (the paper's 10-DOF frame), uploaded to device pole tables;
flags come from the oracle's stab3d. Exact parts are compared exactly: the stable-pole list,
the FCM physical cluster, the retained set, every cluster membership and size, the
representative f / xi (lower medians of the same table values). Floating-point parts at
rounding level: features (<= 1e-12), memberships (<= 1e-9), merge heights (<= 1e-12)."""
import numpy as np
import pytest

import oracle
import synth
from synth.poles import make_diagram
from tests.parity import cells_to_table, diagram_cells, compare_clustering

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2411_05510_b200 import api, build
    build.build()
    return api


def _crit(api, c):
    return api.Criteria(**c.__dict__)


def _run_both(api, cells, crit, cutoff, min_size, cap, l):
    flags, _ = oracle.stab3d(cells, crit, cap)
    oc = oracle.cluster_3d(cells, flags, crit, cutoff=cutoff, min_size=min_size)
    tabs = [cells_to_table(c, api, "cuda", cap=cap, l=l) for c in cells]
    gc = api.cluster3d(tabs, torch.from_numpy(flags).cuda(), _crit(api, crit), cutoff=cutoff, min_size=min_size)
    torch.cuda.synchronize()
    return gc, oc


@pytest.mark.parametrize("seed,G,O,cap,l,modes,cutoff,min_size", [
    (1, 1, 12, 8, 6, 3, 0.10, 1),         # 2D diagram (one lag)
    (2, 4, 25, 20, 12, 8, 0.10, 3),       # several D tiles, ragged tail
    (3, 6, 30, 24, 33, 10, 0.15, 5),      # odd channel count
    (4, 3, 20, 16, 8, 6, 0.30, 1),        # loose cutoff: large components
    (5, 8, 50, 40, 24, 15, 0.10, 5),      # ~4400 stable poles, ~2200 retained (35 D tiles a side)
])
def test_cluster_synthetic_diagrams(api, seed, G, O, cap, l, modes, cutoff, min_size):
    d = make_diagram(seed, G, list(range(2, 2 * O + 1, 2)), cap, l, modes)
    cells = diagram_cells(d)
    gc, oc = _run_both(api, cells, oracle.SC_10DOF_3D, cutoff, min_size, cap, l)
    st = compare_clustering(gc, oc, cutoff)
    print(st)
    assert st["max_dX"] <= 1e-12 and st["max_dU"] <= 1e-9
    assert st.get("max_dh", 0.0) <= 1e-12
    assert gc.overflow == 0


def test_cluster_edge_cases(api):
    """No stable pole at all (nothing to cluster: empty outputs, SSI_OK), and a diagram whose
    stable poles are one tight cloud."""
    d = make_diagram(9, 2, [2, 4, 6], 6, 5, 0, spurious=1.0)
    cells = diagram_cells(d)
    flags, _ = oracle.stab3d(cells, oracle.SC_10DOF_3D, 6)
    assert not (flags == 2).any()
    idx, X = oracle.stable_pole_features(cells, flags, oracle.SC_10DOF_3D)
    assert len(idx) == 0
    tabs = [cells_to_table(c, api, "cuda", cap=6, l=5) for c in cells]
    gc = api.cluster3d(tabs, torch.from_numpy(flags).cuda(), _crit(api, oracle.SC_10DOF_3D))
    assert (gc.n_stable, gc.n_retained, gc.n_clusters, gc.fcm_iters) == (0, 0, 0, 0)
    d = make_diagram(10, 3, list(range(2, 21, 2)), 4, 7, 1, spurious=0.0)
    cells = diagram_cells(d)
    gc, oc = _run_both(api, cells, oracle.SC_10DOF_3D, 0.1, 1, 4, 7)
    compare_clustering(gc, oc, 0.1)
    assert gc.n_clusters >= 1


def test_cluster_paper_frame_end_to_end(api):
    """The oracle's end-to-end NEXT-2 pin (tests/test_oracle_cluster.py): the paper's 10-DOF frame
    (Table 1), three lags of the paper's grid, orders 2..40,
    identified by the oracle; the GPU clustering of the same tables returns the same ten clusters."""
    from synth.records import _simulate
    from tests.analytic import shear_frame_modes
    modes = shear_frame_modes(200.0)
    Y = _simulate(modes, 60000, 0.1, np.random.default_rng([27, 0xE3]))
    l, n_max = 10, 40
    orders = list(range(2, n_max + 1, 2))
    lags = (170, 179, 188)
    R = oracle.covariances(Y, 2 * lags[-1] - 1)
    cells = []
    for i in lags:
        U, S, _ = oracle.rsvd(oracle.toeplitz(R, i), n_max + 20, 2, 0xE3, i, n_max)
        cells.append(oracle.modal_sweep(U, S, l, i, orders, 1 / 200.0))
    min_size = int(0.2 * len(orders) * len(lags))
    gc, oc = _run_both(api, cells, oracle.SC_10DOF_3D, 0.10, min_size, n_max // 2, l)
    st = compare_clustering(gc, oc, 0.10)
    print(st)
    assert gc.n_clusters == 10
    np.testing.assert_allclose(gc.f.cpu().numpy(), np.sort(modes.f), rtol=0.01)


def _shapes_dev(shapes):
    a = np.stack([np.asarray(shapes).real, np.asarray(shapes).imag], axis=-1)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_track_random_sessions(api, seed):
    """ssi_track vs oracle.track_session on random campaigns: competing candidates, misses,
    sessions with no mode, exact-threshold ties left to the oracle's reading."""
    rng = np.random.default_rng([seed, 77])
    R, S, M, l = 6, 40, 9, 7
    rf = np.sort(rng.uniform(2, 8, R))
    rs = [rng.standard_normal(l) + 0.05j * rng.standard_normal(l) for _ in range(R)]
    f = np.zeros((S, M))
    sh = np.zeros((S, M, l), complex)
    cnt = rng.integers(0, M + 1, S).astype(np.int32)
    cnt[0] = 0
    matches = []
    for s in range(S):
        for c in range(cnt[s]):
            r = rng.integers(0, R)
            f[s, c] = rf[r] * (1 + rng.uniform(-0.08, 0.08))
            sh[s, c] = rs[r] + rng.uniform(0.0, 0.6) * rng.standard_normal(l)
        matches.append(oracle.track_session(rf, rs, f[s, :cnt[s]], list(sh[s, :cnt[s]])))
    match, success = api.track(torch.from_numpy(rf).cuda(), _shapes_dev(rs), torch.from_numpy(f).cuda(),
                               _shapes_dev(sh), torch.from_numpy(cnt).cuda())
    assert np.array_equal(match.cpu().numpy(), np.array(matches))
    np.testing.assert_array_equal(success.cpu().numpy(), oracle.success_ratio(np.array(matches)))


# ------------------------------------------------------------------ full size (bench.py's configs)
def _params(drivers, cfg, i=None):
    return drivers.SweepParams(l=cfg.l, i=i or cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs,
                               n_min=cfg.n_min, n_step=cfg.n_step, seed=cfg.philox_key, cov_mode="spectral")


def test_c4_identify_3d_full_size(api):
    """The c4 workload end to end on the GPU (16 lags, orders 2..200, bridge 3D criteria,
    PAPER.md:541): drivers.identify_3d. The oracle clusters the same 16 device tables (they are
    parity-gated against the oracle's own identification in test_gpu_fullsize.py, and ssi_stab3d's
    flags against oracle.stab3d on them there; the oracle cannot identify 16 lags of c4 from the
    record within a test's time). Exact: stable-pole list, retained set, every membership."""
    from paper_2411_05510_b200 import drivers
    from tests.parity import gpu_cells
    cfg = synth.config("c4")
    lags = list(cfg.lags)
    Y, modes = synth.make_record(cfg)
    P = _params(drivers, cfg, i=max(lags))
    crit = oracle.SC_BRIDGE_3D
    tables, flags, counts, gc = drivers.identify_3d(torch.from_numpy(Y).cuda(), P, lags, _crit(api, crit))
    torch.cuda.synchronize()
    gcells = [gpu_cells(tables[i]) for i in lags]
    fl = flags.cpu().numpy()
    min_size = max(1, int(0.2 * len(cfg.orders) * len(lags)))
    oc = oracle.cluster_3d(gcells, fl, crit, cutoff=0.10, min_size=min_size)
    st = compare_clustering(gc, oc, 0.10)
    print("c4 clustering:", st)
    assert st["max_dX"] <= 1e-12 and st["max_dU"] <= 1e-9 and st.get("max_dh", 0.0) <= 1e-12
    # the generating modes are among the clusters (20 bridge modes, 0.5..15 Hz)
    reps = gc.f.cpu().numpy()
    hit = [np.min(np.abs(reps - f) / f) for f in modes.f]
    print("c4 clusters", len(reps), "max rel. distance of a true mode to a cluster", max(hit))
    assert max(hit) <= 0.01


def test_c5_campaign_tracking(api):
    """Continuous monitoring: 8 drifting c5 records identified by the
    record pipeline; per-session two-stage clustering and tracking against the first session
    (drivers.track_campaign) vs the oracle's cluster_3d + track_session on the same tables."""
    from paper_2411_05510_b200 import drivers
    from tests.parity import gpu_cells
    cfg = synth.config("c5")
    recs = [torch.from_numpy(synth.make_record(cfg, r)[0]).cuda() for r in range(8)]
    P = _params(drivers, cfg)
    tabs = drivers.record_batch(recs, P, n_streams=8)
    tabs = [tabs[j] for j in range(8)]
    crit = oracle.SC_BRIDGE_3D
    match, success, ref_f, ref_shape = drivers.track_campaign(tabs, _crit(api, crit))
    torch.cuda.synchronize()
    min_size = max(1, int(0.2 * len(cfg.orders)))
    modes = []
    for j, t in enumerate(tabs):
        cells = gpu_cells(t)
        fl, _ = oracle.stab3d([cells], crit, t.cap)
        oc = oracle.cluster_3d([cells], fl, crit, cutoff=0.10, min_size=min_size)
        gc = drivers.session_modes(t, _crit(api, crit))
        compare_clustering(gc, oc, 0.10)
        modes.append(([c["f"] for c in oc["clusters"]],
                      [oc["shapes"][c["medoid"]] for c in oc["clusters"]]))
    ref = modes[0]
    m_o = np.array([oracle.track_session(np.array(ref[0]), ref[1], np.array(f), sh) for f, sh in modes])
    assert np.array_equal(match.cpu().numpy(), m_o)
    np.testing.assert_array_equal(success.cpu().numpy(), oracle.success_ratio(m_o))
    print("c5 campaign: reference modes", len(ref[0]), "success", success.cpu().numpy().round(1).tolist())


def test_cluster_degenerate_settings(api):
    """Cutoff >= 1 (no f band pruning), a min_size above every cluster (nothing kept, all labels
    -1), max_clusters below the cluster count (overflow flagged, outputs truncated), and orders
    reported as truncated (count = -1) inside the diagram."""
    d = make_diagram(31, 3, list(range(2, 41, 2)), 16, 10, 6)
    d.count[1, 5] = -1                     # an order above the numerical rank (count = -1)
    d.count[2, 7] = -1
    cells = diagram_cells(d)
    for c in (cells[1][5], cells[2][7]):
        c.poles = []
    crit = oracle.SC_10DOF_3D
    gc, oc = _run_both(api, cells, crit, 1.5, 1, 16, 10)
    compare_clustering(gc, oc, 1.5)
    gc, oc = _run_both(api, cells, crit, 0.1, 10 ** 6, 16, 10)
    compare_clustering(gc, oc, 0.1)
    assert gc.n_clusters == 0 and (gc.labels.cpu().numpy() == -1).all()
    flags, _ = oracle.stab3d(cells, crit, 16)
    tabs = [cells_to_table(c, api, "cuda", cap=16, l=10) for c in cells]
    full = api.cluster3d(tabs, torch.from_numpy(flags).cuda(), _crit(api, crit), cutoff=0.1, min_size=1)
    few = api.cluster3d(tabs, torch.from_numpy(flags).cuda(), _crit(api, crit), cutoff=0.1, min_size=1,
                        max_clusters=3)
    assert full.n_clusters > 3 and full.overflow == 0
    assert few.overflow == 1 and few.n_clusters == 3
    np.testing.assert_array_equal(few.f.cpu().numpy(), full.f.cpu().numpy()[:3])
    lab = few.labels.cpu().numpy()
    lab_full = full.labels.cpu().numpy()
    assert np.array_equal(lab[lab_full < 3], lab_full[lab_full < 3]) and (lab[lab_full >= 3] == -1).all()
