"""Helpers for GPU-vs-oracle parity (test infrastructure)."""
import numpy as np
from scipy.optimize import linear_sum_assignment

import oracle


def gpu_cells(tab):
    """Device PoleTable -> list per order of (count, [(f, xi, mu, shape, mpc, mpd)])."""
    cnt = tab.count.cpu().numpy()
    f, xi = tab.f.cpu().numpy(), tab.xi.cpu().numpy()
    mr, mi = tab.mu_re.cpu().numpy(), tab.mu_im.cpu().numpy()
    mpc, mpd = tab.mpc.cpu().numpy(), tab.mpd.cpu().numpy()
    sh = tab.shape.cpu().numpy()
    out = []
    for o in range(len(cnt)):
        poles = []
        for s in range(max(cnt[o], 0)):
            poles.append(oracle.Pole(f[o, s], xi[o, s], complex(mr[o, s], mi[o, s]),
                                     sh[o, s, :, 0] + 1j * sh[o, s, :, 1], mpc[o, s], mpd[o, s]))
        out.append(oracle.OrderCell(tab.n_min + o * tab.n_step, int(cnt[o]), poles))
    return out


def match_cell(a, b):
    """Minimum-cost assignment on d_f + d_xi + (1 - MAC) (SURVEY.md §8(c) parity contract)."""
    if not a or not b:
        return []
    cost = np.zeros((len(a), len(b)))
    for i, p in enumerate(a):
        for j, q in enumerate(b):
            cost[i, j] = (abs(p.f - q.f) / max(p.f, q.f) + abs(p.xi - q.xi) / max(p.xi, q.xi)
                          + 1 - oracle.mac(p.shape, q.shape))
    r, c = linear_sum_assignment(cost)
    return list(zip(r, c))


def compare_tables(gpu, ora, stable_flags=None):
    """Returns dict of parity statistics between GPU cells and oracle cells (same orders).
    stable_flags[o][s] (oracle stab3d flags) marks the poles the contract gates."""
    st = dict(count_mismatch=[], max_df_all=0.0, max_dxi_all=0.0, max_df_stable=0.0,
              max_dxi_stable=0.0, min_mac_stable=1.0, n_poles=0, n_stable=0,
              max_dmpc=0.0, max_dmpd=0.0)
    for o, (g, r) in enumerate(zip(gpu, ora)):
        if g.count != r.count:
            st["count_mismatch"].append((r.n, g.count, r.count))
            continue
        for i, j in match_cell(r.poles, g.poles):
            p, q = r.poles[i], g.poles[j]
            df = abs(p.f - q.f) / p.f
            dxi = abs(p.xi - q.xi)
            st["max_df_all"] = max(st["max_df_all"], df)
            st["max_dxi_all"] = max(st["max_dxi_all"], dxi)
            st["max_dmpc"] = max(st["max_dmpc"], abs(p.mpc - q.mpc))
            st["max_dmpd"] = max(st["max_dmpd"], abs(p.mpd - q.mpd))
            st["n_poles"] += 1
            if stable_flags is not None and stable_flags[o][i] == 2:
                st["n_stable"] += 1
                st["max_df_stable"] = max(st["max_df_stable"], df)
                st["max_dxi_stable"] = max(st["max_dxi_stable"], dxi)
                st["min_mac_stable"] = min(st["min_mac_stable"], oracle.mac(p.shape, q.shape))
    return st


def cells_to_table(cells, api, device, cap=None, l=None):
    """Oracle cells of one lag (list of OrderCell, orders with a constant step) -> device
    PoleTable (upload only; slots past count are zero)."""
    import torch
    n = [c.n for c in cells]
    step = n[1] - n[0] if len(n) > 1 else 2
    cap = cap or max(1, max(max(c.count, 0) for c in cells))
    l = l or next(len(p.shape) for c in cells for p in c.poles)
    t = api.PoleTable.empty(n[0], n[-1], step, l, "cpu", cap=cap)
    for o, c in enumerate(cells):
        t.count[o] = c.count
        for s, p in enumerate(c.poles):
            t.f[o, s], t.xi[o, s] = p.f, p.xi
            t.mu_re[o, s], t.mu_im[o, s] = p.mu.real, p.mu.imag
            t.mpc[o, s], t.mpd[o, s] = p.mpc, p.mpd
            sh = np.asarray(p.shape)
            t.shape[o, s, :, 0] = torch.from_numpy(sh.real.copy())
            t.shape[o, s, :, 1] = torch.from_numpy(sh.imag.copy())
    return t.to(device)


def diagram_cells(d):
    """synth.poles.Diagram -> per lag, list of oracle OrderCell."""
    G, O = d.count.shape
    out = []
    for g in range(G):
        cells = []
        for o, n in enumerate(d.orders):
            ps = [oracle.Pole(float(d.f[g, o, s]), float(d.xi[g, o, s]), 0j, d.shape[g, o, s].copy(),
                              float(d.mpc[g, o, s]), float(d.mpd[g, o, s])) for s in range(d.count[g, o])]
            cells.append(oracle.OrderCell(n, int(d.count[g, o]), ps))
        out.append(cells)
    return out


def compare_clustering(gc, oc, cutoff):
    """GPU Clustering vs oracle.cluster_3d output; returns a dict of statistics and asserts the
    exact parts (stable-pole list, FCM cluster choice, retained set, cluster memberships)."""
    from scipy.cluster.hierarchy import linkage
    from scipy.spatial.distance import squareform
    st = {}
    idx = gc.pole_idx.cpu().numpy()
    assert gc.n_stable == len(oc["idx"]) and np.array_equal(idx, oc["idx"])
    X = gc.X.cpu().numpy()
    st["max_dX"] = float(np.abs(X - oc["X"]).max()) if len(X) else 0.0
    U = gc.U.cpu().numpy()
    st["max_dU"] = float(np.abs(U - oc["U"]).max()) if len(U) else 0.0
    st["max_dV"] = float(np.abs(gc.V.numpy() - oc["V"]).max()) if len(X) else 0.0
    st["fcm_iters"] = (gc.fcm_iters, oc["iters"])
    if len(X):
        st["min_margin_P"] = float(np.abs(oc["U"][:, oc["phys"]] - 0.5).min())
        assert gc.phys == oc["phys"]
    ret = gc.retained.cpu().numpy()
    assert np.array_equal(ret, np.flatnonzero(oc["keep"]))
    labels = gc.labels.cpu().numpy()
    assert np.array_equal(labels, oc["labels"]), (labels, oc["labels"])
    cl = oc["clusters"]
    assert gc.n_clusters == len(cl)
    assert np.array_equal(gc.size.cpu().numpy(), [c["size"] for c in cl])
    assert np.array_equal(gc.f.cpu().numpy(), [c["f"] for c in cl])
    assert np.array_equal(gc.xi.cpu().numpy(), [c["xi"] for c in cl])
    n = len(ret)
    st["n_retained"], st["n_clusters"], st["n_components"] = n, len(cl), gc.n_components
    if n >= 2:
        D = oracle.pole_distances(oc["f"], oc["xi"], oc["shapes"])
        # medoids: equal, or a tie within rounding of the oracle's summed distances
        med = gc.medoid.cpu().numpy()
        for k, c in enumerate(cl):
            if med[k] != c["medoid"]:
                sums = D[np.ix_(c["members"], c["members"])].sum(axis=1)
                a, b = sums[c["members"].index(med[k])], sums[c["members"].index(c["medoid"])]
                assert abs(a - b) <= 1e-12 * max(abs(b), 1e-300), (k, a, b)
        Z = linkage(squareform(D, checks=False), method="average")
        h_o = np.sort(Z[Z[:, 2] <= cutoff, 2])
        h_g = np.sort(gc.merges_h.cpu().numpy())
        assert len(h_o) == len(h_g) == gc.n_merges
        st["max_dh"] = float(np.abs(h_o - h_g).max()) if len(h_o) else 0.0
        above = Z[:, 2][Z[:, 2] > cutoff]
        st["cut_margin"] = float(min(np.abs(Z[:, 2] - cutoff).min(), 1.0))
    return st
