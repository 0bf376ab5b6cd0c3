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
