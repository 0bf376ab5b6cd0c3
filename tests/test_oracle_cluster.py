"""Pins of the NEXT-2 oracle (oracle/cluster.py, oracle/track.py), -m "not gpu".

Each function is checked against something other than itself: hand-built grids whose
best neighbours are known, the closed-form symmetric fixed point of fuzzy C-means solved by
an independent root finder, a brute-force UPGMA written from the definition (mean of the
original pairwise distances, globally closest pair merged first), SPEC.md's worked examples
 and, end to end, the ten Table 1 modes of the paper's shear frame
 recovered by the 3D diagram + two-stage clustering on a synthetic record."""
import itertools

import numpy as np
import pytest
from scipy.optimize import brentq

import oracle
import synth


def _pole(f, xi, shape, mpc=0.99, mpd=0.01):
    return oracle.Pole(f, xi, complex(0.9, 0.1), oracle.normalize_shape(np.asarray(shape, complex)), mpc, mpd)


def _cell(n, ps):
    return oracle.OrderCell(n, len(ps), ps)


# ------------------------------------------------------------------ stage I features (C-1)
def test_features_identical_neighbour_is_zero():
    """a pole identical to its neighbour has d_f = d_xi = 1 - MAC = 0."""
    s = [1.0, 0.4, -0.3]
    g0 = [_cell(2, [_pole(5.0, 0.02, s, mpc=0.9, mpd=0.05)]), _cell(4, [_pole(5.0, 0.02, s, mpc=0.9, mpd=0.05)])]
    flags, _ = oracle.stab3d([g0], oracle.SC_10DOF_3D, 2)
    idx, X = oracle.stable_pole_features([g0], flags, oracle.SC_10DOF_3D)
    assert idx.tolist() == [[0, 1, 0]]
    np.testing.assert_allclose(X[0], [0.0, 0.0, 0.0, 0.1, 0.05], atol=1e-15)


def test_features_pick_the_closest_qualifying_neighbour():
    """Two predecessors satisfy the soft criteria: the order-axis one at d_f = 0.1/5.1 (SPEC.md:452
    arithmetic: 0.019608 > alpha_f = 1 %, so it does NOT qualify) and a lag-axis one; a third
    candidate is rejected by the hard criteria. The features are the lag-axis neighbour's."""
    C = oracle.SC_10DOF_3D
    s = [1.0, 0.5, 0.2]
    p = _pole(5.1, 0.0200, s)
    order_nb = _pole(5.0, 0.0200, s)                       # d_f = 0.019608 > 0.01
    lag_nb = _pole(5.12, 0.0201, s)                         # d_f = 0.003906, d_xi = 0.004975
    hard_bad = _pole(5.1, 0.0200, s, mpc=0.5)               # MPC <= 60 %: not kept
    g0 = [_cell(2, []), _cell(4, [lag_nb])]
    g1 = [_cell(2, [order_nb, hard_bad]), _cell(4, [p])]
    flags, _ = oracle.stab3d([g0, g1], C, 2)
    assert flags[1, 1, 0] == 2
    idx, X = oracle.stable_pole_features([g0, g1], flags, C)
    assert idx.tolist() == [[1, 1, 0]]
    assert abs(0.1 / 5.1 - 0.019608) < 5e-7                # SPEC.md:452 printed value
    np.testing.assert_allclose(X[0, :3], [0.02 / 5.12, 0.0001 / 0.0201, 0.0], rtol=1e-12, atol=1e-15)


def test_features_tie_keeps_the_order_axis():
    C = oracle.SC_10DOF_3D
    s = [1.0, 0.5, 0.2]
    q = _pole(5.0, 0.02, s)
    g0 = [_cell(2, []), _cell(4, [_pole(5.0, 0.02, s, mpc=0.95)])]
    g1 = [_cell(2, [q]), _cell(4, [_pole(5.0, 0.02, s, mpc=0.97, mpd=0.02)])]
    flags, _ = oracle.stab3d([g0, g1], C, 1)
    idx, X = oracle.stable_pole_features([g0, g1], flags, C)
    assert idx.tolist() == [[1, 1, 0]]
    np.testing.assert_allclose(X[0], [0, 0, 0, 0.03, 0.02], atol=1e-15)


# ------------------------------------------------------------------ fuzzy C-means (C-2, C-3)
def test_fcm_two_tight_clouds():
    """two tight clouds -> each point's membership >= 0.95 in its own cluster."""
    X = np.array([[0, 0], [0.01, 0.01], [1, 1], [0.99, 1.01]], float)
    U, V, it = oracle.fuzzy_cmeans(X)
    assert np.all(U[:2, 0] >= 0.95) and np.all(U[2:, 1] >= 0.95)
    np.testing.assert_allclose(U.sum(axis=1), 1.0, rtol=1e-14)


def test_fcm_point_at_a_centroid_takes_full_membership():
    """SPEC.md:462 singularity rule."""
    U = oracle.fcm_memberships(np.array([[0.0, 1.0], [0.5, 0.5]]), np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert U[0].tolist() == [1.0, 0.0]
    np.testing.assert_allclose(U[1], [0.5, 0.5], rtol=1e-15)


def test_fcm_symmetric_fixed_point_closed_form():
    """Points {-1, -0.5, 0.5, 1}: by symmetry the centroids converge to -v*, +v* where v* > 0 is the
    non-trivial root of v = sum_x (u_x^2 - (1-u_x)^2) x / sum_x (u_x^2 + (1-u_x)^2), x in {0.5, 1},
    u_x = (x + v)^2 / ((x - v)^2 + (x + v)^2) (m = 2) — solved here by Brent's method."""
    X = np.array([[-1.0], [-0.5], [0.5], [1.0]])
    U, V, it = oracle.fuzzy_cmeans(X)

    def g(v):
        num = den = 0.0
        for x in (0.5, 1.0):
            u = (x + v) ** 2 / ((x - v) ** 2 + (x + v) ** 2)
            num += (u * u - (1 - u) ** 2) * x
            den += u * u + (1 - u) ** 2
        return num / den - v

    vstar = brentq(g, 1e-3, 0.999, xtol=1e-15)
    np.testing.assert_allclose(np.sort(V[:, 0]), [-vstar, vstar], atol=1e-9)
    assert it < 1000


def test_fcm_is_deterministic_and_permutation_equivariant():
    rng = np.random.default_rng(5)
    X = np.vstack([rng.normal(0.02, 0.01, (30, 5)), rng.normal(0.4, 0.1, (20, 5))]).clip(0)
    U1, V1, _ = oracle.fuzzy_cmeans(X)
    U2, V2, _ = oracle.fuzzy_cmeans(X)
    assert np.array_equal(U1, U2) and np.array_equal(V1, V2)
    perm = rng.permutation(len(X))
    U3, V3, _ = oracle.fuzzy_cmeans(X[perm])
    np.testing.assert_allclose(U3, U1[perm], atol=1e-9)
    j, keep = oracle.select_physical(U1, V1)
    assert j == int(np.argmin(np.linalg.norm(V1, axis=1)))
    assert keep[:30].all() and not keep[30:].any()       # the cloud near the origin is physical


def test_select_physical_keeps_p_exactly_half():
    """PAPER.md:415 'possibly physical poles if P >= 0.5'."""
    U = np.array([[0.5, 0.5], [0.49, 0.51], [0.9, 0.1]])
    V = np.array([[0.01, 0.0], [0.4, 0.3]])
    j, keep = oracle.select_physical(U, V)
    assert j == 0 and keep.tolist() == [True, False, True]


# ------------------------------------------------------------------ stage II (C-4)
def _upgma_bruteforce(D, cutoff):
    """Definition: clusters start as singletons; repeatedly merge the pair of clusters whose mean
    ORIGINAL pairwise distance is smallest (lowest (a, b) on ties) while it is <= cutoff."""
    cl = [[i] for i in range(D.shape[0])]
    while len(cl) > 1:
        best = None
        for a, b in itertools.combinations(range(len(cl)), 2):
            d = D[np.ix_(cl[a], cl[b])].mean()
            if best is None or d < best[0]:
                best = (d, a, b)
        if best[0] > cutoff:
            break
        _, a, b = best
        cl[a] = sorted(cl[a] + cl[b])
        del cl[b]
    return sorted(sorted(c) for c in cl)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_hierarchical_matches_bruteforce_upgma(seed):
    rng = np.random.default_rng(seed)
    n = 24
    f = np.concatenate([rng.normal(mu, 0.02 * mu, n // 3) for mu in (2.0, 2.3, 6.0)])
    xi = rng.uniform(0.01, 0.03, n)
    sh = rng.standard_normal((n, 6)) + 1j * 0.05 * rng.standard_normal((n, 6))
    sh[n // 3: 2 * n // 3] = sh[n // 3] + 0.1 * rng.standard_normal((n // 3, 6))
    D = oracle.pole_distances(f, xi, sh)
    for cutoff in (0.05, 0.2, 0.5, 1.0):
        labels, clusters = oracle.hierarchical_clusters(D, f, xi, cutoff, 1)
        got = sorted(sorted(c["members"]) for c in clusters)
        assert got == _upgma_bruteforce(D, cutoff)
        assert (labels >= 0).all()


def test_hierarchical_spec_examples_and_representatives():
    """three poles at 5.312 +- 0.001 Hz with MAC >= 0.999 and similar xi form one
    cluster; 5.3 Hz and 15.8 Hz never merge for cutoff <= 0.5 (d_f alone = 0.664). Representative
    f / xi = lower median, shape = medoid; min_size drops small clusters."""
    s = np.array([1.0, 0.5, 0.2], complex)
    f = np.array([5.311, 5.312, 5.313, 5.3, 15.8])
    xi = np.array([0.020, 0.0201, 0.0199, 0.02, 0.02])
    sh = np.array([s, s + 0.01, s - 0.01, s, [0.2, -1.0, 0.4]])
    D = oracle.pole_distances(f, xi, sh)
    assert abs(D[3, 4] - (10.5 / 15.8 + 1 - oracle.mac(sh[3], sh[4]))) < 1e-12
    assert abs(10.5 / 15.8 - 0.664) < 1e-3                  # SPEC.md:482 prints 0.664 (truncated)
    labels, cl = oracle.hierarchical_clusters(D, f, xi, 0.5, 1)
    assert len(cl) == 2 and cl[0]["members"] == [0, 1, 2, 3] and cl[1]["members"] == [4]
    assert cl[0]["f"] == 5.311 and cl[0]["xi"] == 0.02      # lower median of 4 members
    assert cl[0]["medoid"] in (0, 1, 2)
    labels, cl = oracle.hierarchical_clusters(D, f, xi, 0.01, 3)
    assert [c["members"] for c in cl] == [[0, 1, 2, 3]] and labels.tolist() == [0, 0, 0, 0, -1]
    labels, cl = oracle.hierarchical_clusters(D, f, xi, 0.01, 5)
    assert cl == [] and labels.tolist() == [-1] * 5


# ------------------------------------------------------------------ tracking (C-5)
def test_tracking_spec_examples():
    """SPEC.md:528-530 and Table 4's reference mode 1 (2.628 Hz)."""
    ref = np.array([2.628])
    s = np.array([1.0, 0.0, 0.0])
    t95 = np.array([1.0, np.sqrt(1 / 0.95 - 1), 0.0])         # MAC(s, t95) = 0.95
    t80 = np.array([1.0, np.sqrt(1 / 0.80 - 1), 0.0])
    assert abs(oracle.mac(s, t95) - 0.95) < 1e-12
    assert oracle.track_session(ref, [s], np.array([2.65]), [t95]).tolist() == [0]
    assert oracle.track_session(ref, [s], np.array([2.80]), [t80]).tolist() == [-1]
    # two candidates competing for one reference: the lower score wins, the other is free
    ref2 = np.array([2.628, 2.70])
    m = oracle.track_session(ref2, [s, s], np.array([2.64, 2.66]), [s, s])
    assert m.tolist() == [0, 1]


def test_tracking_greedy_equals_exhaustive_on_small_instances():
    """on small instances the greedy one-to-one assignment agrees with an
    exhaustive search whenever the optimum is unique and every reference has a candidate."""
    rng = np.random.default_rng(11)
    for _ in range(60):
        nr, nc = rng.integers(1, 5), rng.integers(1, 5)
        rf = np.sort(rng.uniform(2, 3, nr))
        cf = rf[rng.integers(0, nr, nc)] * (1 + rng.uniform(-0.03, 0.03, nc))
        rs = [rng.standard_normal(4) for _ in range(nr)]
        cs = [rs[rng.integers(0, nr)] + 0.05 * rng.standard_normal(4) for _ in range(nc)]
        m = oracle.track_session(rf, rs, cf, cs)
        assert len(set(x for x in m if x >= 0)) == (m >= 0).sum()          # one-to-one
        for r, c in enumerate(m):
            if c >= 0:
                assert abs(cf[c] - rf[r]) / max(cf[c], rf[r]) <= 0.05 and 1 - oracle.mac(cs[c], rs[r]) <= 0.15
        # monotonicity: loosening thresholds never loses a match count
        m2 = oracle.track_session(rf, rs, cf, cs, df_max=0.1, macd_max=0.3)
        assert (m2 >= 0).sum() >= (m >= 0).sum()


def test_success_ratio_arithmetic():
    """384 of 384 -> 100.0 (Table 4 mode 1, 3D-RSVD); 304 of 384 -> 79.17."""
    m = -np.ones((384, 2), int)
    m[:, 0] = 0
    m[:304, 1] = 1
    r = oracle.success_ratio(m)
    assert r[0] == 100.0 and round(r[1], 2) == 79.17


# ------------------------------------------------------------------ end to end on the paper's frame
def test_3d_clustering_recovers_the_table1_modes():
    """The paper's 10-DOF frame (Table 1), 5 min at 200 Hz with SNR 20 dB: the
    3D diagram over three lags of the paper's grid (j_b = 170, 179, 188), orders
    2..40, the 10-DOF 3D criteria and the two-stage clustering give exactly ten
    clusters, one per Table 1 mode, each representative within 1 % in frequency (statistical
    pin of the whole NEXT-2 chain, cf. Table 2's f_3D column)."""
    from synth.records import _simulate
    from tests.analytic import shear_frame_modes
    modes = shear_frame_modes(200.0)
    Y = _simulate(modes, 60000, 0.1, np.random.default_rng([27, 0xE3]))
    l, n_max = 10, 40
    orders = list(range(2, n_max + 1, 2))
    lags = (170, 179, 188)
    R = oracle.covariances(Y, 2 * lags[-1] - 1)
    tables = []
    for i in lags:
        U, S, _ = oracle.rsvd(oracle.toeplitz(R, i), n_max + 20, 2, 0xE3, i, n_max)
        tables.append(oracle.modal_sweep(U, S, l, i, orders, 1 / 200.0))
    crit = oracle.SC_10DOF_3D
    flags, counts = oracle.stab3d(tables, crit, n_max // 2)
    min_size = int(0.2 * len(orders) * len(lags))
    out = oracle.cluster_3d(tables, flags, crit, cutoff=0.10, min_size=min_size)
    assert out["keep"].sum() < len(out["keep"])                 # stage I rejects some poles
    reps = np.array([c["f"] for c in out["clusters"]])
    assert len(reps) == 10, reps
    np.testing.assert_allclose(reps, np.sort(modes.f), rtol=0.01)
