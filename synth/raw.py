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
