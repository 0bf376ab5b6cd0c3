"""Shear-type frame generator of the paper's 10-DOF case (§3.1; PAPER.md:349,
§3.1.2) — SURVEY.md NEXT-4. TEST INFRASTRUCTURE (see oracle/__init__.py).

PAPER.md:314: "a damped shear-type 10-storey frame, where the structural mass M and stiffness K
matrices are constructed based on each floor having a mass and a stiffness, set at 100 kg and
5000 kN/m ... The damping matrix C is defined proportionally to the mass matrix M ... and the
stiffness matrix K ... using the Rayleigh method, imposing that the first and fourth angular
frequencies of the system have a damping ratio ξ of 1%."  PAPER.md:349: "The matrices A and C in
Eq. (5) were used to generate the observation matrix Y. Noise was simulated as a zero-mean
Gaussian process with signal-to-noise ratio (SNR) ... sampled at 200 Hz."

Readings (F-1 .. F-4):
  F-1 M = m I; K tridiagonal with 2k on the diagonal except k at the roof and −k off the diagonal;
      C = a M + b K with ξ(ω) = a/(2ω) + bω/2 equal to ξ at the undamped modes 1 and 4.
  F-2 state x = (q, q̇): A_c = [[0, I], [−M⁻¹K, −M⁻¹C]]; a force at every DOF, B_c = [[0], [M⁻¹]],
      held over each step (zero-order hold): [[A_d, B_d], [0, I]] = exp([[A_c, B_c], [0, 0]] Δt).
  F-3 x_0 = 0, x_{h+1} = A_d x_h + B_d u_h, u_h ~ N(0, I_n); outputs are the accelerations
      y_h = C_o x_h with C_o = [−M⁻¹K, −M⁻¹C] (no feedthrough); the first n_burn samples are
      discarded (10 s).
  F-4 measurement noise: channel c gets v ~ N(0, P_c / 10^{SNR/10}) with P_c the mean square of
      the kept clean channel. Draws use the reading-A-11 Philox/Box–Muller stream: u from
      (seed, stream 2 s_id), element e = h n + j over all n_burn + N steps; v from (seed,
      stream 2 s_id + 1), element e = h l + c over the kept samples.
Library primitives: numpy.linalg.eigvalsh (undamped frequencies), scipy.linalg.expm.
"""
import numpy as np
from scipy.linalg import expm

from .philox import gaussian_sketch


def frame_matrices(n: int = 10, m: float = 100.0, k: float = 5.0e6, xi: float = 0.01,
                   mode_a: int = 1, mode_b: int = 4):
    """F-1. Returns (M, K, C, (a, b))."""
    M = m * np.eye(n)
    K = np.zeros((n, n))
    for j in range(n):
        K[j, j] = 2.0 * k if j < n - 1 else k
        if j + 1 < n:
            K[j, j + 1] = K[j + 1, j] = -k
    w = np.sqrt(np.linalg.eigvalsh(K / m))            # M = m I: eigenvalues of M^-1 K
    wa, wb = w[mode_a - 1], w[mode_b - 1]
    a, b = np.linalg.solve([[1 / (2 * wa), wa / 2], [1 / (2 * wb), wb / 2]], [xi, xi])
    return M, K, a * M + b * K, (a, b)


def discretize(M, K, C, fs: float):
    """F-2. Returns (A_d, B_d, C_o)."""
    n = M.shape[0]
    Mi = np.linalg.inv(M)
    Ac = np.block([[np.zeros((n, n)), np.eye(n)], [-Mi @ K, -Mi @ C]])
    Bc = np.vstack([np.zeros((n, n)), Mi])
    E = np.zeros((3 * n, 3 * n))
    E[:2 * n, :2 * n] = Ac
    E[:2 * n, 2 * n:] = Bc
    F = expm(E / fs)
    return F[:2 * n, :2 * n], F[:2 * n, 2 * n:], np.hstack([-Mi @ K, -Mi @ C])


def simulate(Ad, Bd, Co, N: int, n_burn: int, snr_db: float, seed: int, stream_id: int):
    """F-3 + F-4. Returns (Y [N][l] with noise, clean [N][l])."""
    n = Bd.shape[1]
    l = Co.shape[0]
    H = n_burn + N
    U = gaussian_sketch(n, H, seed, 2 * stream_id)          # column h = u_h
    x = np.zeros(Ad.shape[0])
    clean = np.zeros((N, l))
    for h in range(H):
        if h >= n_burn:
            clean[h - n_burn] = Co @ x
        x = Ad @ x + Bd @ U[:, h]
    P = (clean ** 2).mean(axis=0)
    sd = np.sqrt(P / 10.0 ** (snr_db / 10.0))
    V = gaussian_sketch(l, N, seed, 2 * stream_id + 1)      # column h = v_h
    return clean + V.T * sd[None, :], clean
