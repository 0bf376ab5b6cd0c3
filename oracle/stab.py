"""Hard criteria + 3D soft criteria (§2.1, Eq. (stabcriteria3D) at
PAPER.md:283-291 §2.3 step ii).

Hard criteria (thresholds PAPER.md:356): "discarding poles with damping
ratios ξ_i > 10%, MPC ≤ 60%, and MPD ≥ 50%" → keep iff ξ ≤ ξ_max ∧ MPC > MPC_min ∧
MPD < MPD_max (reading A-17).

Soft criteria: a kept pole at (lag g, order n) is stable iff ONE
kept pole at the previous order of the same lag (g, n − n_step) OR at the previous lag
of the same order (g − 1, n) satisfies all three of
    d_f = |f_i − f_j| / max(f_i, f_j) ≤ α_f,
    d_ξ = |ξ_i − ξ_j| / max(ξ_i, ξ_j) ≤ α_ξ,           (reading A-21)
    1 − MAC(φ_i, φ_j) ≤ α_MAC                          (printed "MAC ≤ α", reading A-18)
(readings A-19, A-20). Flags: 0 rejected by HC (or empty slot), 1 kept but not
stable ("new"), 2 stable.
"""
from dataclasses import dataclass
import numpy as np

from .indicators import mac


@dataclass(frozen=True)
class Criteria:
    xi_max: float = 0.10
    mpc_min: float = 0.60
    mpd_max: float = 0.50
    alpha_f: float = 0.01
    alpha_xi: float = 0.03
    alpha_mac: float = 0.02


HC_DEFAULT = dict(xi_max=0.10, mpc_min=0.60, mpd_max=0.50)
SC_10DOF_3D = Criteria(**HC_DEFAULT, alpha_f=0.01, alpha_xi=0.03, alpha_mac=0.02)   # :402
SC_BRIDGE_3D = Criteria(**HC_DEFAULT, alpha_f=0.025, alpha_xi=0.05, alpha_mac=0.03)  # :541


def _hard_ok(p, c: Criteria) -> bool:
    return p.xi <= c.xi_max and p.mpc > c.mpc_min and p.mpd < c.mpd_max


def _soft_match(p, q, c: Criteria) -> bool:
    d_f = abs(p.f - q.f) / max(p.f, q.f)
    d_xi = abs(p.xi - q.xi) / max(p.xi, q.xi)
    return d_f <= c.alpha_f and d_xi <= c.alpha_xi and (1.0 - mac(p.shape, q.shape)) <= c.alpha_mac


def stab3d(tables, crit: Criteria, cap: int):
    """tables[g][o] = OrderCell for lag g (increasing i) and order index o (increasing n).
    Returns flags [G][O][cap] uint8 and stable_count [G][O] int32."""
    G, O = len(tables), len(tables[0])
    flags = np.zeros((G, O, cap), dtype=np.uint8)
    kept = [[[_hard_ok(p, crit) for p in tables[g][o].poles] for o in range(O)]
            for g in range(G)]
    for g in range(G):
        for o in range(O):
            for s, p in enumerate(tables[g][o].poles):
                if not kept[g][o][s]:
                    continue
                stable = False
                for (gg, oo) in ((g, o - 1), (g - 1, o)):
                    if gg < 0 or oo < 0:
                        continue
                    for t, q in enumerate(tables[gg][oo].poles):
                        if kept[gg][oo][t] and _soft_match(p, q, crit):
                            stable = True
                            break
                    if stable:
                        break
                flags[g, o, s] = 2 if stable else 1
    return flags, (flags == 2).sum(axis=2).astype(np.int32)
