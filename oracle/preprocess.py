"""Upstream preprocessing of an acceleration record (§3.2) — SURVEY.md NEXT-4.
TEST INFRASTRUCTURE (see oracle/__init__.py).

PAPER.md:482: "The acceleration records are processed through a simple filtering sequence
involving the elimination of linear trends and downsampling to 40 Hz (eighth-order low-pass
Chebyshev Type I filter with a cut-off frequency of 0.8·20 Hz followed by a decimation to 40 Hz)."

Readings (P-1 .. P-3):
  P-1 detrend: per channel, subtract the least-squares line α + β h over the sample index
      h = 0..N−1.
  P-2 filter: Chebyshev Type I low-pass, order 8, passband ripple 0.05 dB (not printed; the
      default of MATLAB's / scipy's decimate, whose description the paper's matches), passband
      edge f_c = 0.8 · f_out / 2 (16 Hz for 40 Hz), designed for the rate L·f_in by the bilinear
      transform with prewarping; applied zero-phase: forward, then backward over
      the reversed sequence, zero initial state both ways, no padding.
  P-3 rate change f_out = f_in · L / M, L/M in lowest terms (125 → 40 Hz is 8/25): the
      detrended channel is upsampled by L (L·x[n] at index n·L, zeros between), filtered at L·f_in
      (P-2), and every M-th sample kept starting with the first; N_out = floor(N L / M)
      (SPEC.md:68). With L = 1 this is SPEC.md's integer decimate.
Library primitives used as single steps: scipy.signal.cheby1 (design, output='sos') and
scipy.signal.sosfilt (the biquad recursion).
"""
from fractions import Fraction

import numpy as np
from scipy.signal import cheby1, sosfilt


def detrend(Y):
    """P-1. Y [N][l] → Y − (α + β h) per channel (FP64), least squares by the normal equations."""
    Y = np.asarray(Y, dtype=np.float64)
    N = Y.shape[0]
    h = np.arange(N, dtype=np.float64)
    hbar = (N - 1) / 2.0
    beta = ((h - hbar)[:, None] * Y).sum(axis=0) / ((h - hbar) ** 2).sum()
    alpha = Y.mean(axis=0) - beta * hbar
    return Y - (alpha[None, :] + beta[None, :] * h[:, None])


def rate_ratio(fs_in: float, fs_out: float):
    """(L, M) with fs_out / fs_in = L / M in lowest terms (both rates integral in Hz)."""
    fr = Fraction(int(round(fs_out)), int(round(fs_in)))
    return fr.numerator, fr.denominator


def lowpass_sos(fs_high: float, fc: float, order: int = 8, rp_db: float = 0.05):
    """P-2 design: Chebyshev I low-pass with passband edge fc at the sampling rate fs_high."""
    return cheby1(order, rp_db, fc, btype="low", fs=fs_high, output="sos")


def filtfilt_zero_state(sos, x):
    """P-2 application: forward pass, then a pass over the reversed output, zero initial state."""
    y = sosfilt(sos, x, axis=0)
    return sosfilt(sos, y[::-1], axis=0)[::-1]


def preprocess(Y, fs_in: float, fs_out: float, order: int = 8, rp_db: float = 0.05):
    """P-1 .. P-3 on a record Y [N][l]. Returns the FP64 record [floor(N L / M)][l]."""
    L, M = rate_ratio(fs_in, fs_out)
    X = detrend(Y)
    N, l = X.shape
    U = np.zeros((N * L, l))
    U[::L] = L * X
    sos = lowpass_sos(fs_in * L, 0.8 * fs_out / 2.0, order, rp_db)
    V = filtfilt_zero_state(sos, U)
    n_out = (N * L) // M
    return np.ascontiguousarray(V[::M][:n_out])
