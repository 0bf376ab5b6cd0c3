"""Randomized SVD of T (§2.2, Algorithm 1 at PAPER.md:255-268) and the
classical full SVD of Eq. (8).

Algorithm 1, rsvd(A, k):
  1  Ω ← randn(m, k)            (n×k for A ∈ R^{m×n}; T is square, reading A-5)
  2  Y ← A Ω                    Eq. (14)
  3  (Q, R) ← qr(Y, 0)          economy QR
  4  P ← Qᵀ A                   Eq. (15)
  5  (Ũ, S, V) ← svd(P, 'econ') Eq. (16)
  6  U ← Q Ũ                    Eq. (18)
The north star adds q power iterations with re-orthonormalisation (reading A-12):
between lines 3 and 4, q times: Z = qr(Aᵀ Q).Q ; Q = qr(A Z).Q. With q = 0 the function
is Algorithm 1 verbatim (pin P7). k = n_max + p (reading A-26).

QR is LAPACK Householder (numpy.linalg.qr) with column signs fixed so diag(R) > 0
(reading A-13); SVD is LAPACK dgesdd (numpy.linalg.svd).
"""
import numpy as np

from .philox import gaussian_sketch


def householder_qr(Y):
    """Economy QR, Y = Q R, diag(R) > 0 (reading A-13)."""
    Q, R = np.linalg.qr(Y, mode="reduced")
    d = np.sign(np.diag(R))
    d[d == 0] = 1.0
    return Q * d, R * d[:, None]


def rsvd(T, k: int, q: int, seed: int, stream_id: int, n_keep: int | None = None,
         Omega=None):
    """Returns (U [m×n_keep], S [k], Q [m×k]) following Algorithm 1 (+ q power iterations)."""
    T = np.asarray(T, dtype=np.float64)
    m, n = T.shape
    if not (1 <= k <= min(m, n)):
        raise ValueError("k out of range (SPEC.md:161)")
    if Omega is None:
        Omega = gaussian_sketch(n, k, seed, stream_id)          # line 1
    Y = T @ Omega                                               # line 2, Eq. (14)
    Q, _ = householder_qr(Y)                                    # line 3
    for _ in range(q):                                          # power iterations (A-12)
        Z, _ = householder_qr(T.T @ Q)
        Q, _ = householder_qr(T @ Z)
    P = Q.T @ T                                                 # line 4, Eq. (15)
    Ut, S, _ = np.linalg.svd(P, full_matrices=False)            # line 5, Eq. (16)
    U = Q @ Ut                                                  # line 6, Eq. (18)
    n_keep = k if n_keep is None else n_keep
    return U[:, :n_keep], S, Q


def full_svd(T):
    """Classical CoV-SSI decomposition, Eq. (8): (U, S) by dgesdd."""
    U, S, _ = np.linalg.svd(np.asarray(T, dtype=np.float64), full_matrices=False)
    return U, S
