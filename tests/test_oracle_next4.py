"""Pins of the NEXT-4 oracle (oracle/preprocess.py, oracle/frame.py), -m "not gpu".

Each function is checked against something other than itself: closed forms (the Chebyshev-I
magnitude |H|² = 1/(1 + ε² T_n²(tan(πf/fs)/tan(πf_c/fs))) of the bilinear design, the zero-phase
steady-state response |H(f)|² cos(2πft), the least-squares normal equations), SPEC.md's worked
examples, the paper's printed Rayleigh coefficients and Table 1
(PAPER.md:314, :329-334), and an impulse response computed through a different matrix exponential."""
import os

import numpy as np
import pytest
from scipy.signal import sosfreqz

import oracle
import importlib

pp = importlib.import_module("oracle.preprocess")
fr = importlib.import_module("oracle.frame")

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _table1():
    rows = [r.split() for r in open(os.path.join(GOLD, "table1_10dof.txt")) if r.strip() and r[0] != "#"]
    return np.array([[float(x) for x in r[1:]] for r in rows])


# ------------------------------------------------------------------ P-1 detrend
def test_detrend_pure_linear_trend_is_zero():
    """channel y_h = 3 + 0.5 h -> all-zero output."""
    h = np.arange(5000.0)
    Y = np.stack([3 + 0.5 * h, -2.0 + 1e-3 * h], axis=1)
    assert np.abs(pp.detrend(Y)).max() <= 1e-9


def test_detrend_satisfies_the_normal_equations_and_is_idempotent():
    rng = np.random.default_rng(1)
    N = 7001
    h = np.arange(N, dtype=float)
    Y = rng.standard_normal((N, 4)) + np.sin(h / 10.0)[:, None] + 0.01 * h[:, None]
    Z = pp.detrend(Y)
    # residual orthogonal to 1 and h (least squares)
    assert np.abs(Z.sum(axis=0)).max() <= 1e-8 * N
    assert np.abs((h[:, None] * Z).sum(axis=0)).max() <= 1e-8 * N * N
    # the removed part is exactly a line: second differences vanish
    D = Y - Z
    assert np.abs(np.diff(D, 2, axis=0)).max() <= 1e-10
    np.testing.assert_allclose(pp.detrend(Z), Z, atol=1e-10)


# ------------------------------------------------------------------ P-2 design and zero-phase filter
def _cheb(n, x):
    x = np.asarray(x, dtype=float)
    out = np.empty_like(x)
    a = np.abs(x) <= 1
    out[a] = np.cos(n * np.arccos(x[a]))
    out[~a] = np.cosh(n * np.arccosh(np.abs(x[~a]))) * np.sign(x[~a]) ** n
    return out


@pytest.mark.parametrize("fs,fc", [(200.0, 16.0), (1000.0, 16.0), (125.0, 10.0)])
def test_lowpass_matches_the_chebyshev_closed_form(fs, fc):
    """Bilinear Chebyshev-I: |H(e^{j2πf/fs})|² = 1/(1 + ε² T_8²(tan(πf/fs)/tan(πf_c/fs))),
    ε² = 10^{0.05/10} − 1; order 8 = the paper's 'eighth-order'."""
    sos = pp.lowpass_sos(fs, fc)
    assert sos.shape == (4, 6)
    f = np.linspace(0.0, 0.49 * fs, 400)
    _, H = sosfreqz(sos, worN=f, fs=fs)
    eps2 = 10 ** (0.05 / 10) - 1
    ref = 1.0 / (1.0 + eps2 * _cheb(8, np.tan(np.pi * f / fs) / np.tan(np.pi * fc / fs)) ** 2)
    np.testing.assert_allclose(np.abs(H) ** 2, ref, rtol=1e-9, atol=1e-14)


def test_zero_phase_steady_state_is_the_squared_magnitude():
    """Forward-backward filtering of cos(2πf t): away from both ends the output is
    |H(f)|² cos(2πf t) — no phase shift (SPEC.md:70 'zero-phase application')."""
    fs, fc = 200.0, 16.0
    sos = pp.lowpass_sos(fs, fc)
    t = np.arange(40000) / fs
    for f0 in (2.0, 12.0, 17.0):
        x = np.cos(2 * np.pi * f0 * t)
        y = pp.filtfilt_zero_state(sos, x[:, None])[:, 0]
        _, H = sosfreqz(sos, worN=[f0], fs=fs)
        mid = slice(15000, 25000)
        np.testing.assert_allclose(y[mid], abs(H[0]) ** 2 * x[mid], atol=1e-9)


def test_spec_decimation_examples():
    """2 Hz sine at 200 Hz -> 40 Hz keeps its amplitude within 1 %; 19 Hz (above
    the 16 Hz edge) is attenuated below 5 %; N_out = floor(N fs_out / fs_in)."""
    fs = 200.0
    N = 30000
    t = np.arange(N) / fs
    for f0, lo, hi in ((2.0, 0.99, 1.01), (19.0, 0.0, 0.05)):
        Y = np.sin(2 * np.pi * f0 * t)[:, None]
        Z = oracle.preprocess(Y, fs, 40.0)
        assert Z.shape == (N // 5, 1)
        amp = np.abs(Z[1000:-1000, 0]).max()
        assert lo <= amp <= hi, (f0, amp)


@pytest.mark.parametrize("N", [9999, 10000, 12345])
def test_rational_125_to_40(N):
    """The bridge rate change (125 Hz records, decimation to 40 Hz) is L/M = 8/25:
    N_out = floor(8N/25); a 3 Hz sine comes out sampled at 40 Hz with gain |H(3)|² of the design
    at 1 kHz and no phase shift (closed form), a 30 Hz component is removed."""
    assert pp.rate_ratio(125, 40) == (8, 25)
    t = np.arange(N) / 125.0
    Y = np.stack([np.sin(2 * np.pi * 3 * t) + 0.5 * np.sin(2 * np.pi * 30 * t), 1.0 + 0.001 * np.arange(N)], axis=1)
    Z = oracle.preprocess(Y, 125.0, 40.0)
    assert Z.shape == ((8 * N) // 25, 2)
    _, H = sosfreqz(pp.lowpass_sos(1000.0, 16.0), worN=[0.0, 3.0], fs=1000.0)
    j = np.arange(Z.shape[0])
    mid = slice(800, Z.shape[0] - 800)
    # the detrend also removes the sine's own least-squares line α + β h; a zero-phase filter
    # passes a line with its DC gain |H(0)|² (its symmetric impulse response preserves lines)
    h = np.arange(N, dtype=float)
    s = Y[:, 0]
    beta = ((h - (N - 1) / 2) * s).sum() / ((h - (N - 1) / 2) ** 2).sum()
    alpha = s.mean() - beta * (N - 1) / 2
    ref = abs(H[1]) ** 2 * np.sin(2 * np.pi * 3 * j / 40.0) - abs(H[0]) ** 2 * (alpha + beta * j * 25 / 8)
    np.testing.assert_allclose(Z[mid, 0], ref[mid], atol=1e-6)
    assert np.abs(Z[mid, 1]).max() <= 1e-9            # a pure trend vanishes


# ------------------------------------------------------------------ F-1 .. F-4 frame generator
def test_frame_rayleigh_coefficients_and_table1():
    """PAPER.md:314 + Table 1: a = 0.5815 s^-1, b = 7.781e-5 s;
    the zero-order-hold discrete system's poles, converted by reading A-1, give Table 1."""
    M, K, C, (a, b) = fr.frame_matrices()
    assert abs(a - 0.5815) < 5e-5 and abs(b - 7.781e-5) < 5e-9
    Ad, Bd, Co = fr.discretize(M, K, C, 200.0)
    lam = np.log(np.linalg.eigvals(Ad)) * 200.0
    lam = lam[lam.imag > 0]
    o = np.argsort(np.abs(lam))
    f = np.abs(lam[o]) / (2 * np.pi)
    xi = 100 * -lam[o].real / np.abs(lam[o])
    gold = _table1()
    np.testing.assert_allclose(f, gold[:, 0], atol=5e-4)
    np.testing.assert_allclose(xi, gold[:, 1], atol=5e-4)


def test_frame_zoh_input_matrix_by_quadrature():
    """B_d = ∫_0^Δt e^{A_c s} ds B_c (F-2), checked by composite Simpson quadrature of expm."""
    from scipy.linalg import expm
    M, K, C, _ = fr.frame_matrices(n=3, m=50.0, k=2.0e5, mode_b=3)
    Ad, Bd, Co = fr.discretize(M, K, C, 100.0)
    n = 3
    Mi = np.linalg.inv(M)
    Ac = np.block([[np.zeros((n, n)), np.eye(n)], [-Mi @ K, -Mi @ C]])
    Bc = np.vstack([np.zeros((n, n)), Mi])
    s = np.linspace(0.0, 0.01, 201)
    vals = np.array([expm(Ac * x) @ Bc for x in s])
    w = np.ones_like(s); w[1:-1:2] = 4; w[2:-1:2] = 2
    quad = (w[:, None, None] * vals).sum(axis=0) * (s[1] - s[0]) / 3
    np.testing.assert_allclose(Bd, quad, rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(Ad, expm(Ac * 0.01), rtol=1e-12, atol=1e-15)


def test_frame_recursion_impulse_response():
    """With the draws replaced by one unit force pulse on DOF j at step 0, y_h = C_o e^{A_c (h−1)Δt}
    B_d e_j for h >= 1 — powers of A_d against direct matrix exponentials."""
    from scipy.linalg import expm
    M, K, C, _ = fr.frame_matrices()
    Ad, Bd, Co = fr.discretize(M, K, C, 200.0)
    n = 10
    Mi = np.linalg.inv(M)
    Ac = np.block([[np.zeros((n, n)), np.eye(n)], [-Mi @ K, -Mi @ C]])
    x = Bd[:, 3].copy()
    for h in range(1, 60):
        ref = Co @ expm(Ac * (h - 1) / 200.0) @ Bd[:, 3]
        np.testing.assert_allclose(Co @ x, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())
        x = Ad @ x


def test_frame_simulation_snr_and_spectral_peaks():
    """per-channel empirical SNR within ±0.5 dB of the spec; the PSD of the
    record at SNR 20 dB (summed over the channels) peaks within ±0.2 Hz of the Table 1 frequencies
    of modes 1..8; modes 9 and 10 (68.0, 70.4 Hz, half-power bands 2ξf ≈ 2.4 and 2.5 Hz) overlap
    and merge into one peak between them."""
    from scipy.signal import welch
    M, K, C, _ = fr.frame_matrices()
    Ad, Bd, Co = fr.discretize(M, K, C, 200.0)
    Y, clean = fr.simulate(Ad, Bd, Co, 60000, 2000, 20.0, 0xE3, 1)
    snr = 10 * np.log10((clean ** 2).mean(axis=0) / ((Y - clean) ** 2).mean(axis=0))
    assert np.all(np.abs(snr - 20.0) <= 0.5), snr
    f, P = welch(Y, fs=200.0, nperseg=8192, axis=0)
    P = P.sum(axis=1)
    gold = _table1()[:, 0]
    for f0 in gold[:8]:
        w = (f > f0 - 1.0) & (f < f0 + 1.0)
        fpk = f[w][np.argmax(P[w])]
        assert abs(fpk - f0) <= 0.2 + (f[1] - f[0]), (f0, fpk)
    w = (f > 66.5) & (f < 72.5)
    assert gold[8] - 0.2 <= f[w][np.argmax(P[w])] <= gold[9] + 0.2


def test_frame_draws_are_the_reading_a11_stream():
    """u_h is column h of the A-11 Gaussian sketch (n x (n_burn+N), stream 2 s_id): a one-step
    simulation from x_0 = 0 gives y_1 = C_o B_d u_0."""
    M, K, C, _ = fr.frame_matrices()
    Ad, Bd, Co = fr.discretize(M, K, C, 200.0)
    Y, clean = fr.simulate(Ad, Bd, Co, 2, 0, 20.0, 5, 7)
    u0 = oracle.gaussian_sketch(10, 2, 5, 14)[:, 0]
    np.testing.assert_allclose(clean[0], 0.0)
    np.testing.assert_allclose(clean[1], Co @ Bd @ u0, rtol=1e-12)
