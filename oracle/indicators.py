"""Pole-quality indicators used by the hard and soft criteria (§2.1).

PAPER.md:207 names MPC [Pappa 1993] ("assesses the linear relationship between the
real and imaginary parts of the modal components") and MPD [Dederichs 2023] ("evaluates
the statistical variation of the phase angles of each modal component"), "both ...
dimensionless and range from 0 to 1"; PAPER.md:208 names MAC [Allemang]. No formula is
printed; the readings (A-15, A-16) are:

  MAC(a, b) = |aᴴ b|² / (‖a‖² ‖b‖²)
  MPC(φ)    = ((λ1 − λ2)/(λ1 + λ2))², λ1 ≥ λ2 eigenvalues of the UNCENTERED 2×2 scatter
              [[ReᵀRe, ReᵀIm], [ReᵀIm, ImᵀIm]]
  MPD(φ)    = (Σ_j |φ_j| δ_j / Σ_j |φ_j|) / (π/4), clamped to [0, 1], where δ_j ∈ [0, π/2]
              is the angle between component j and the total-least-squares line through
              the origin (principal direction of the same scatter, from its SVD).
  Shape normalization: unit 2-norm, largest-|·| component rotated to the positive real
  axis (reading A-15).
"""
import numpy as np


def mac(a, b) -> float:
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    num = abs(np.vdot(a, b)) ** 2
    return float(num / (np.vdot(a, a).real * np.vdot(b, b).real))


def normalize_shape(phi):
    phi = np.asarray(phi, dtype=np.complex128)
    phi = phi / np.linalg.norm(phi)
    j = int(np.argmax(np.abs(phi)))
    return phi * (np.conj(phi[j]) / abs(phi[j]))


def _scatter(phi):
    X = np.stack([phi.real, phi.imag], axis=1)        # l × 2
    return X, X.T @ X                                 # uncentered 2×2 scatter


def mpc(phi) -> float:
    _, S = _scatter(np.asarray(phi, dtype=np.complex128))
    lam = np.linalg.eigvalsh(S)                        # ascending
    l1, l2 = lam[1], lam[0]
    return float(((l1 - l2) / (l1 + l2)) ** 2)


def mpd(phi) -> float:
    phi = np.asarray(phi, dtype=np.complex128)
    X, _ = _scatter(phi)
    _, _, Vt = np.linalg.svd(X, full_matrices=False)   # TLS line direction = Vt[0]
    d = Vt[0]
    dot = X @ d
    cross = X[:, 0] * d[1] - X[:, 1] * d[0]
    delta = np.arctan2(np.abs(cross), np.abs(dot))    # angle to the (undirected) line
    w = np.abs(phi)
    val = float((w * delta).sum() / w.sum() / (np.pi / 4))
    return min(max(val, 0.0), 1.0)
