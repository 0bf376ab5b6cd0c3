"""Closed forms used to pin the oracle (test infrastructure; no oracle code here).

For the synth/ modal generator with unit-variance modal coordinates, the exact output
covariance at lag k ≥ 1 is (PAPER.md:137 R_j = C A^{j−1} G):
    R_k = Σ_m |μ_m|^k cos(k arg μ_m) φ_m φ_mᵀ
(measurement noise enters only R_0, which T never uses)."""
import numpy as np


def exact_covariances(modes, lag_hi: int) -> np.ndarray:
    mu = modes.mu
    r, th = np.abs(mu), np.angle(mu)
    l = modes.phi.shape[1]
    R = np.zeros((lag_hi, l, l))
    for k in range(1, lag_hi + 1):
        w = r ** k * np.cos(k * th)
        R[k - 1] = (modes.phi.T * w) @ modes.phi
    return R


def shear_frame_10dof(m=100.0, k=5.0e6, xi=0.01):
    """10-storey shear frame of PAPER.md:314 with Rayleigh damping ξ = 1% at modes 1, 4.
    Returns (M, K, C, omega_sorted)."""
    n = 10
    M = m * np.eye(n)
    K = np.zeros((n, n))
    for j in range(n):
        K[j, j] = 2 * k if j < n - 1 else k
        if j + 1 < n:
            K[j, j + 1] = K[j + 1, j] = -k
    w2 = np.sort(np.linalg.eigvals(np.linalg.solve(M, K)).real)
    w = np.sqrt(w2)
    # ξ_i = a/(2 ω_i) + b ω_i / 2 at i = 1, 4
    A = np.array([[1 / (2 * w[0]), w[0] / 2], [1 / (2 * w[3]), w[3] / 2]])
    a, b = np.linalg.solve(A, [xi, xi])
    return M, K, a * M + b * K, w, (a, b)


def shear_frame_modes(fs: float):
    """The 10-DOF shear frame (Table 1 model) as synth.Modes: undamped modes of
    (M, K) (proportional damping keeps them real), natural frequencies ω/2π, Rayleigh ξ_i =
    a/(2ω_i) + b ω_i/2, unit-norm shapes with the largest component positive. The E2/E3 workload
     is this model sampled at 200 Hz."""
    import synth
    M, K, C, w, (a, b) = shear_frame_10dof()
    w2, V = np.linalg.eigh(np.linalg.solve(np.sqrt(M), np.linalg.solve(np.sqrt(M), K).T))
    order = np.argsort(w2)
    V = np.linalg.solve(np.sqrt(M), V[:, order])
    om = np.sqrt(w2[order])
    phi = V.T / np.linalg.norm(V.T, axis=1, keepdims=True)
    phi *= np.sign(phi[np.arange(10), np.argmax(np.abs(phi), axis=1)])[:, None]
    return synth.Modes(om / (2 * np.pi), a / (2 * om) + b * om / 2, phi, fs)
