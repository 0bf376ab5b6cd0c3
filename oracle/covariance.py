"""Output correlation matrices R_1 .. R_{2 j_b - 1} (§2.1).

PAPER.md:126: "Considering positive time intervals ranging from Δt to (2j_b − 1)Δt ...
the output correlation matrices R_1 ∈ R^{l×l} to R_{2j_b−1} can be directly derived
from the acceleration records." The normalization is unstated; reading A-6
takes the unbiased 1/(N−k) of the north star and SPEC.md:82:

    R_k[a][b] = (1/(N−k)) Σ_{t=0}^{N−k−1} Y[t+k][a] · Y[t][b],   k = lag_lo .. lag_hi.

Each lag's sum is one library matmul of the two lag-shifted views in FP64 (FP32 inputs
are converted exactly; FP32×FP32 products are exact in FP64).
"""
import numpy as np


def covariance_partial_sums(Y, lag_lo: int, lag_hi: int, t_begin: int = 0,
                            t_end: int | None = None) -> np.ndarray:
    """Raw sums S_k[a][b] = Σ_{t ∈ [t_begin, t_end), t+k < N} Y[t+k][a] Y[t][b] for
    k = lag_lo..lag_hi (time shard of the sum in PAPER.md:126; used by the multi-GPU
    time-sharded covariance). Returns [lag_hi-lag_lo+1][l][l] FP64."""
    Y = np.asarray(Y, dtype=np.float64)
    N, l = Y.shape
    t_end = N if t_end is None else t_end
    out = np.zeros((lag_hi - lag_lo + 1, l, l))
    for k in range(lag_lo, lag_hi + 1):
        hi = min(t_end, N - k)
        if hi > t_begin:
            out[k - lag_lo] = Y[t_begin + k:hi + k].T @ Y[t_begin:hi]
    return out


def covariances(Y, lag_hi: int, lag_lo: int = 1) -> np.ndarray:
    """R[k - lag_lo] = R_k for k = lag_lo..lag_hi (1/(N−k), reading A-6).
    For a Toeplitz of time-lag step i use lag_hi = 2i − 1 (reading A-7)."""
    N = np.asarray(Y).shape[0]
    if N <= lag_hi:
        raise ValueError("record too short for requested lags (SPEC.md:83)")
    S = covariance_partial_sums(Y, lag_lo, lag_hi)
    for k in range(lag_lo, lag_hi + 1):
        S[k - lag_lo] /= (N - k)
    return S
