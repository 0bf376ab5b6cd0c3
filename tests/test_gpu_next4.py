"""NEXT-4 GPU parity (-m gpu): ssi_preprocess (detrend + zero-phase Chebyshev-I + L/M
resampling) and ssi_frame_simulate (the 10-DOF shear frame)
against oracle/preprocess.py and oracle/frame.py on the same synthetic inputs.

Tolerances: the GPU runs the IIR recursion in time chunks (two passes and a state scan per
direction), the oracle sequentially; the results agree up to rounding amplified by the filter's
state gain — gated at 1e-9 of each channel's output scale. The frame generator: model matrices
within 1e-12, records within 1e-9 of the channel scale."""
import numpy as np
import pytest
from scipy.signal import sosfreqz

import oracle
from synth.raw import make_raw_record

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2411_05510_b200 import api, build
    build.build()
    return api


def _cheb(n, x):
    x = np.asarray(x, dtype=float)
    out = np.empty_like(x)
    a = np.abs(x) <= 1
    out[a] = np.cos(n * np.arccos(x[a]))
    out[~a] = np.cosh(n * np.arccosh(np.abs(x[~a]))) * np.sign(x[~a]) ** n
    return out


@pytest.mark.parametrize("order,rp,fc,fs", [(8, 0.05, 16.0, 1000.0), (8, 0.05, 16.0, 200.0), (4, 0.5, 10.0, 125.0),
                                            (16, 0.05, 8.0, 100.0), (2, 1.0, 30.0, 100.0)])
def test_lowpass_design_closed_form(api, order, rp, fc, fs):
    """The device design (analog prototype, prewarp, bilinear) against the Chebyshev-I closed form
    and against the oracle's (scipy) design."""
    sos = api.lowpass_design(order, rp, fc, fs).cpu().numpy()
    full = np.hstack([sos[:, :3], np.ones((len(sos), 1)), sos[:, 3:]])
    f = np.linspace(0.0, 0.49 * fs, 500)
    _, H = sosfreqz(full, worN=f, fs=fs)
    eps2 = 10 ** (rp / 10) - 1
    ref = 1.0 / (1.0 + eps2 * _cheb(order, np.tan(np.pi * f / fs) / np.tan(np.pi * fc / fs)) ** 2)
    np.testing.assert_allclose(np.abs(H) ** 2, ref, rtol=1e-9, atol=1e-14)
    _, Ho = sosfreqz(oracle.lowpass_sos(fs, fc, order, rp), worN=f, fs=fs)
    np.testing.assert_allclose(H, Ho, rtol=1e-9, atol=1e-13)


def _check(Z, Zo, tol=1e-9):
    assert Z.shape == Zo.shape
    scale = np.abs(Zo).max(axis=0) + 1e-300
    err = (np.abs(Z - Zo) / scale).max()
    print(f"max error / channel scale {err:.2e}")
    assert err <= tol


@pytest.mark.parametrize("fs_in,fs_out,N,l,dt", [
    (200.0, 40.0, 30000, 10, np.float64),     # the 10-DOF rate, integer decimation by 5
    (125.0, 40.0, 20011, 12, np.float32),     # the bridge rate change 8/25, ragged length
    (125.0, 25.0, 7777, 3, np.float32),       # integer decimation by 5 at the bridge rate
    (100.0, 100.0, 5000, 7, np.float64),      # L = M = 1: detrend + zero-phase low-pass only
    (125.0, 40.0, 50, 2, np.float64),         # shorter than one chunk
])
def test_preprocess_parity(api, fs_in, fs_out, N, l, dt):
    Y, _ = make_raw_record(l=l, fs=fs_in, N=N, seed=int(fs_in + N), dtype=dt)
    Z = api.preprocess(torch.from_numpy(Y).cuda(), fs_in, fs_out)
    torch.cuda.synchronize()
    _check(Z.cpu().numpy(), oracle.preprocess(Y, fs_in, fs_out))


def test_preprocess_fp32_output_and_strided_input(api):
    Y, _ = make_raw_record(l=6, fs=125.0, N=9000, seed=3, dtype=np.float64)
    big = torch.zeros((9000, 9), dtype=torch.float64, device="cuda")
    big[:, :6] = torch.from_numpy(Y).cuda()
    Z = api.preprocess(big[:, :6], 125.0, 40.0, out_dtype=torch.float32)
    Zo = oracle.preprocess(Y, 125.0, 40.0)
    assert Z.dtype == torch.float32
    np.testing.assert_allclose(Z.cpu().numpy(), Zo.astype(np.float32), rtol=0, atol=2e-7 * np.abs(Zo).max())


def test_preprocess_two_hour_bridge_record(api):
    """Full size: 114 channels, 2 h at 125 Hz (900 000 FP32 samples) -> 40 Hz
    (288 000 samples). The oracle runs on a channel sample (channels are independent)."""
    Y, _ = make_raw_record(l=114, fs=125.0, N=900000, seed=482)
    Yd = torch.from_numpy(Y).cuda()
    Z = api.preprocess(Yd, 125.0, 40.0)
    torch.cuda.synchronize()
    assert Z.shape == (288000, 114)
    cols = [0, 57, 113]
    _check(Z.cpu().numpy()[:, cols], oracle.preprocess(Y[:, cols], 125.0, 40.0))


def test_frame_model_matches_oracle(api):
    M, K, C, (a, b) = oracle.frame_matrices()
    Ad_o, Bd_o, Co_o = oracle.discretize(M, K, C, 200.0)
    Ad, Bd, Co, ab = [t.cpu().numpy() for t in api.frame_model(api.Frame(), 200.0)]
    np.testing.assert_allclose(ab, [a, b], rtol=1e-13)
    np.testing.assert_allclose(Ad, Ad_o, rtol=1e-12, atol=1e-13 * np.abs(Ad_o).max())
    np.testing.assert_allclose(Bd, Bd_o, rtol=1e-11, atol=1e-13 * np.abs(Bd_o).max())
    np.testing.assert_allclose(Co, Co_o, rtol=1e-14)


@pytest.mark.parametrize("N,n_burn,snr,seed,sid,frame", [
    (60000, 2000, 20.0, 0xE3, 1, None),                         # the paper's E2/E3 record (5 min at 200 Hz)
    (777, 0, 10.0, 7, 3, None),                                  # short, no burn-in
    (5000, 100, 25.0, 11, 0, dict(n_dof=3, m=50.0, k=2.0e5, mode_b=3)),
])
def test_frame_simulate_matches_oracle(api, N, n_burn, snr, seed, sid, frame):
    fr = api.Frame(**(frame or {}))
    M, K, C, _ = oracle.frame_matrices(fr.n_dof, fr.m, fr.k, fr.xi, fr.mode_a, fr.mode_b)
    Ad, Bd, Co = oracle.discretize(M, K, C, 200.0)
    Yo, clo = oracle.simulate_frame(Ad, Bd, Co, N, n_burn, snr, seed, sid)
    Y, cl = api.frame_simulate(N, 200.0, snr, seed, sid, fr, n_burn=n_burn, with_clean=True)
    torch.cuda.synchronize()
    _check(cl.cpu().numpy(), clo)
    _check(Y.cpu().numpy(), Yo)


def test_raw_record_through_preprocess_and_identification(api):
    """NEXT-4 feeding the hot path: a raw 125 Hz record with trends and out-of-band modes ->
    ssi_preprocess -> 40 Hz -> covariances, structured RSVD, modal sweep. The in-band modes are
    identified (statistical band); the out-of-band ones are gone."""
    from paper_2411_05510_b200 import drivers
    Y, modes = make_raw_record(l=24, fs=125.0, N=450000, seed=9)
    P = drivers.SweepParams(l=24, i=40, n_max=60, p=20, q=2, fs=40.0, seed=1)
    tab, Z = drivers.identify_raw(torch.from_numpy(Y).cuda(), 125.0, 40.0, P, stream_id=1)
    torch.cuda.synchronize()
    n = 2 * len(modes.f)
    o = (n - P.n_min) // P.n_step
    cnt = int(tab.count[o])
    f = tab.f[o, :cnt].cpu().numpy()
    xi = tab.xi[o, :cnt].cpu().numpy()
    for f0 in modes.f:
        j = np.argmin(np.abs(f - f0))
        assert abs(f[j] - f0) / f0 <= 0.01, (f0, f[j])
    assert f.max() < 20.0


@pytest.mark.parametrize("order,rp", [(2, 0.5), (16, 0.05)])
def test_preprocess_other_orders(api, order, rp):
    """Orders at the ends of the supported range (2 and 16 poles) through the same chunked passes."""
    Y, _ = make_raw_record(l=4, fs=125.0, N=12000, seed=order, dtype=np.float64)
    Z = api.preprocess(torch.from_numpy(Y).cuda(), 125.0, 40.0, order=order, rp_db=rp)
    _check(Z.cpu().numpy(), oracle.preprocess(Y, 125.0, 40.0, order=order, rp_db=rp))


def test_preprocess_and_frame_reject_bad_arguments(api):
    """Synchronous checks (ssi.h): odd order, edge at/above Nyquist, no output sample, bad frame."""
    import ctypes as C
    from paper_2411_05510_b200 import _lib
    lib = _lib.get()
    Y = torch.zeros((100, 3), dtype=torch.float32, device="cuda")
    Z = torch.zeros((100, 3), dtype=torch.float32, device="cuda")
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    p = lambda t: C.c_void_p(t.data_ptr())
    call = lambda *a: lib.ssi_preprocess(p(Y), 0, 100, 3, 3, *a, p(Z), 0, 3, p(ws), ws.numel(), None)
    assert call(125.0, 8, 25, 7, 0.05, 16.0) == 1                 # odd order
    assert call(125.0, 8, 25, 8, 0.05, 500.0) == 1                # edge >= L fs / 2
    assert call(125.0, 1, 1000, 8, 0.05, 16.0) == 1               # N L / M < 1
    assert lib.ssi_preprocess(p(Y), 0, 100, 3, 2, 125.0, 8, 25, 8, 0.05, 16.0, p(Z), 0, 3, p(ws), ws.numel(),
                              None) == 2                          # ldY < l
    b = C.c_size_t(0)
    assert lib.ssi_frame_simulate_ws(13, 100, 0, C.byref(b)) == 1  # n_dof > 12
    assert lib.ssi_frame_model(10, 100.0, 5e6, 0.01, 4, 4, 200.0, p(ws), p(ws), p(ws), p(ws), None) == 1  # equal modes
    torch.cuda.synchronize()
    assert torch.all(Z == 0)
