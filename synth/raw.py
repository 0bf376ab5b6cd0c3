"""Seeded raw acceleration records for the NEXT-4 preprocessing tests (input generation only).

A bridge-like raw record before preprocessing (114 channels at 125 Hz, 2-hour files):
the modal model of synth/records.py with `n_in` modes inside the 0.5..15 Hz band the identification
looks at and `n_out` modes above the 16 Hz passband edge (20..55 Hz, which the low-pass must
remove), 5 % measurement noise, plus a per-channel offset and linear trend (which the detrend
must remove). Mode shapes are random unit vectors."""
import numpy as np

from .records import Modes, _simulate


def make_raw_record(l: int = 114, fs: float = 125.0, N: int = 900000, seed: int = 482, n_in: int = 12,
                    n_out: int = 4, dtype=np.float32):
    rng = np.random.default_rng([seed, 0x4E58])
    while True:
        f_in = np.sort(rng.uniform(0.5, 15.0, n_in))
        if np.all(np.diff(f_in) / f_in[1:] >= 0.04):
            break
    f_out = np.sort(rng.uniform(20.0, 55.0, n_out))
    f = np.concatenate([f_in, f_out])
    xi = rng.uniform(0.005, 0.03, n_in + n_out)
    phi = rng.standard_normal((n_in + n_out, l))
    phi /= np.linalg.norm(phi, axis=1, keepdims=True)
    modes = Modes(f, xi, phi, fs)
    y = _simulate(modes, N, 0.05, np.random.default_rng([seed, 0xACC]))
    off = rng.uniform(-0.5, 0.5, l)
    slope = rng.uniform(-1e-5, 1e-5, l)
    y += off[None, :] + slope[None, :] * np.arange(N)[:, None]
    return np.ascontiguousarray(y.astype(dtype)), Modes(f_in, xi[:n_in], phi[:n_in], fs)


def make_bridge_raw(record: int = 0, N: int = 900000, dtype=np.float32):
    """A San-Faustino-shaped raw acquisition: 114 channels, one 2-hour
    file at 125 Hz (900 000 samples), 17 modes between 2.5 and 15 Hz (the paper identifies 17,
    fundamental 2.64 Hz) plus 4 modes above the 16 Hz passband, 5 % noise,
    offsets and linear trends. Synthetic: the bridge data are proprietary."""
    rng = np.random.default_rng([0x5F, 17])
    while True:
        f_in = np.sort(np.r_[2.64, rng.uniform(2.8, 15.0, 16)])
        if np.all(np.diff(f_in) / f_in[1:] >= 0.03):
            break
    f_out = np.sort(rng.uniform(20.0, 55.0, 4))
    f = np.concatenate([f_in, f_out])
    xi = rng.uniform(0.005, 0.03, 21)
    phi = rng.standard_normal((21, 114))
    phi /= np.linalg.norm(phi, axis=1, keepdims=True)
    modes = Modes(f, xi, phi, 125.0)
    y = _simulate(modes, N, 0.05, np.random.default_rng([0x5F, 17, record]))
    off = rng.uniform(-0.5, 0.5, 114)
    slope = rng.uniform(-1e-6, 1e-6, 114)
    y += off[None, :] + slope[None, :] * np.arange(N)[:, None]
    return np.ascontiguousarray(y.astype(dtype)), Modes(f_in, xi[:17], phi[:17], 125.0)
