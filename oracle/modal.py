"""Per-order modal identification, literal form (§2.1, Eqs. 9-12).

For each model order n ("iteratively retaining n₂ ∈ [N_min, N_max]"):
  Eq. (9)  O = U_n S_n^{1/2}
  Eq. (10) C = first l rows of O;  A = pinv(O^to) O^bo, O^to / O^bo = first / last
           l(i−1) rows of O (printed "n_o(j_b−1)", reading A-2)
           pinv by SVD with cutoff 1e−10·σ1
  Eq. (11) A = Ψ M Ψ⁻¹ (printed "ΨMΨᵀ", reading A-4), dense eigensolver (dgeev)
  Eq. (12) λ = ln μ / Δt; f = |λ|/2π, ξ = −Re λ/|λ| (printed forms garbled, reading A-1,
           consistent with Eq. (3)); Φ = C Ψ.
Pole selection (reading A-14): Im μ > 0 strictly, then keep 0 < ξ < 1.
Shapes normalized (A-15); MPC/MPD per indicators.py (A-16). Poles in a cell are sorted
by (f, ξ). An order whose σ_n < 1e−12 σ_1 is above the numerical rank and reported as
count = −1 ("order truncated with warning").
"""
from dataclasses import dataclass, field
import numpy as np

from .indicators import normalize_shape, mpc, mpd


@dataclass
class Pole:
    f: float
    xi: float
    mu: complex
    shape: np.ndarray
    mpc: float
    mpd: float


@dataclass
class OrderCell:
    n: int
    count: int
    poles: list = field(default_factory=list)


def poles_from_eigs(mu, shapes, dt: float):
    """Eq. (12) + reading A-14: (μ_j, Φ_j) → sorted list of Pole."""
    out = []
    for j in range(len(mu)):
        if not (mu[j].imag > 0):
            continue
        lam = np.log(mu[j]) / dt                     # principal branch
        f = abs(lam) / (2 * np.pi)
        xi = -lam.real / abs(lam)
        if not (0.0 < xi < 1.0):
            continue
        phi = normalize_shape(shapes[:, j])
        out.append(Pole(float(f), float(xi), complex(mu[j]), phi, mpc(phi), mpd(phi)))
    out.sort(key=lambda p: (p.f, p.xi))
    return out


def modal_sweep(U, S, l: int, i: int, orders, dt: float):
    """List of OrderCell, one per order in `orders`."""
    U = np.asarray(U, dtype=np.float64)
    S = np.asarray(S, dtype=np.float64)
    cells = []
    for n in orders:
        if S[n - 1] < 1e-12 * S[0]:
            cells.append(OrderCell(n, -1))
            continue
        O = U[:, :n] * np.sqrt(S[:n])                          # Eq. (9)
        C = O[:l]                                              # first l rows
        O_to, O_bo = O[: l * (i - 1)], O[l:]                   # Eq. (10), A-2
        A = np.linalg.pinv(O_to, rcond=1e-10) @ O_bo
        mu, Psi = np.linalg.eig(A)                             # Eq. (11)
        poles = poles_from_eigs(mu, C @ Psi, dt)               # Eq. (12), Φ = CΨ
        cells.append(OrderCell(n, len(poles), poles))
    return cells
