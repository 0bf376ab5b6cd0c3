"""Seeded synthetic stabilization diagrams: inputs of the NEXT-2 clustering tests (no method
arithmetic: every pole field is drawn directly, nothing is identified from a record).

A diagram has G lags x O model orders; cell (g, o) holds up to `cap` poles sorted by (f, xi)
like a modal-sweep table. Physical modes m = 0..M-1 (f ~ U[1, 20] Hz with >= 5 % spacing,
xi ~ U[0.5, 3] %, complex shapes with a small imaginary part) appear from order 2(m+1) on with
probability 0.9 per cell, jittered (f x (1 + 2e-3 N), xi x (1 + 0.01 N), shape + complex
noise of norm ~0.04, MPC ~ U[0.85, 1], MPD ~ U[0, 0.15]); each cell adds Poisson(spurious) spurious poles
(f ~ U[1, 20], xi ~ U[0.1, 20] %, random complex shapes, MPC ~ U[0.2, 1], MPD ~ U[0, 0.8]).
Shapes are scaled to unit 2-norm (the criteria use MAC, which ignores scale and phase).
"""
from dataclasses import dataclass

import numpy as np


@dataclass
class Diagram:
    orders: list
    count: np.ndarray      # [G][O] int32
    f: np.ndarray          # [G][O][cap]
    xi: np.ndarray
    mpc: np.ndarray
    mpd: np.ndarray
    shape: np.ndarray      # [G][O][cap][l] complex128
    mode_f: np.ndarray     # [M] generating frequencies


def _unit(v):
    return v / np.linalg.norm(v)


def make_diagram(seed: int, G: int, orders, cap: int, l: int, n_modes: int, spurious: float = 3.0) -> Diagram:
    rng = np.random.default_rng([seed, 0xD1A6])
    while True:
        mf = np.sort(rng.uniform(1.0, 20.0, n_modes))
        if n_modes < 2 or np.all(np.diff(mf) / mf[1:] >= 0.05):
            break
    mxi = rng.uniform(0.005, 0.03, n_modes)
    msh = [_unit(rng.standard_normal(l) + 0.02j * rng.standard_normal(l)) for _ in range(n_modes)]
    O = len(orders)
    count = np.zeros((G, O), np.int32)
    f = np.zeros((G, O, cap))
    xi = np.zeros((G, O, cap))
    mpc = np.zeros((G, O, cap))
    mpd = np.zeros((G, O, cap))
    shape = np.zeros((G, O, cap, l), np.complex128)
    for g in range(G):
        for o, n in enumerate(orders):
            poles = []
            for m in range(n_modes):
                if n >= 2 * (m + 1) and rng.uniform() < 0.9:
                    sh = _unit(msh[m] + 0.03 / np.sqrt(l) * (rng.standard_normal(l) + 1j * rng.standard_normal(l)))
                    poles.append((mf[m] * (1 + 2e-3 * rng.standard_normal()),
                                  mxi[m] * (1 + 0.01 * rng.standard_normal()),
                                  rng.uniform(0.85, 1.0), rng.uniform(0.0, 0.15), sh))
            for _ in range(rng.poisson(spurious)):
                sh = _unit(rng.standard_normal(l) + 1j * rng.standard_normal(l))
                poles.append((rng.uniform(1.0, 20.0), rng.uniform(0.001, 0.2), rng.uniform(0.2, 1.0),
                              rng.uniform(0.0, 0.8), sh))
            poles = sorted(poles[:cap], key=lambda p: (p[0], p[1]))
            count[g, o] = len(poles)
            for s, p in enumerate(poles):
                f[g, o, s], xi[g, o, s], mpc[g, o, s], mpd[g, o, s], shape[g, o, s] = p
    return Diagram(list(orders), count, f, xi, mpc, mpd, shape, mf)
