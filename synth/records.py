"""Synthetic output-only records for the five BASELINE.json configurations.

Model (Eq. 5, with the modal form of Eqs. 2-4):
each mode m has continuous pole lambda_m = -xi_m w_m + i w_m sqrt(1 - xi_m^2) (Eq. 3),
discrete pole mu_m = exp(lambda_m dt), and a complex modal coordinate

    z_{m,h+1} = mu_m z_{m,h} + g_m (w1_h + i w2_h),   g_m = sqrt(1 - |mu_m|^2)

(a real 2x2 rotation-contraction block of A with isotropic white input), started from
its stationary law z_{m,0} = a + i b, a, b ~ N(0, 1). The clean output is
s_h = sum_m phi_m Re(z_{m,h}) (C = [phi_m, 0] per block) and the record is
y_h = s_h + v_h with v_h[c] ~ N(0, (0.05 rho_c)^2), rho_c the exact stationary RMS of
channel c ("5% RMS Gaussian measurement noise", BASELINE.json configs).

The generator returns the record and the generating (f, xi, phi); it does not compute
any quantity of the identification method.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np
from scipy.signal import lfilter


@dataclass(frozen=True)
class Config:
    name: str
    l: int                 # channels
    fs: float              # sampling frequency [Hz]
    N: int                 # samples per record
    dtype: str             # "f64" or "f32" storage of the record
    i: int                 # time-lag step (block rows of T); PAPER.md j_b
    n_max: int             # maximum model order
    p: int                 # oversampling
    q: int                 # power iterations
    n_min: int = 2
    n_step: int = 2
    lags: tuple = ()       # lag sweep (c4); empty = single lag i
    n_records: int = 1     # record batch (c5)
    seed: int = 0
    philox_key: int = 0
    noise_rms: float = 0.05

    @property
    def k(self) -> int:
        return self.n_max + self.p

    @property
    def m(self) -> int:
        return self.l * self.i

    @property
    def dt(self) -> float:
        return 1.0 / self.fs

    @property
    def orders(self) -> list:
        return list(range(self.n_min, self.n_max + 1, self.n_step))


CONFIGS = {
    # BASELINE.json configs[0]: 3 modes, l=6, fs=50, N=6000 FP64, i=20, n_max=30, p=10, q=2
    "c1": Config("c1", l=6, fs=50.0, N=6000, dtype="f64", i=20, n_max=30, p=10, q=2,
                 seed=1, philox_key=0x5EED0001),
    # configs[1]: l=48, 10 modes, fs=100, N=180000 FP32, i=60, n_max=100, p=20, q=2
    "c2": Config("c2", l=48, fs=100.0, N=180000, dtype="f32", i=60, n_max=100, p=20, q=2,
                 seed=2, philox_key=0x5EED0002),
    # configs[2] (the metric's workload): l=192, 20 modes, fs=100, N=360000 FP32, i=60,
    # n_max=200, p=20, q=2
    "c3": Config("c3", l=192, fs=100.0, N=360000, dtype="f32", i=60, n_max=200, p=20, q=2,
                 seed=3, philox_key=0x5EED0003),
    # configs[3]: c3 record, lags 20..80 step 4
    "c4": Config("c4", l=192, fs=100.0, N=360000, dtype="f32", i=80, n_max=200, p=20, q=2,
                 lags=tuple(range(20, 81, 4)), seed=3, philox_key=0x5EED0004),
    # configs[4]: 64 records of 30 min, c3 model with +-2% drift, i=50
    "c5": Config("c5", l=192, fs=100.0, N=180000, dtype="f32", i=50, n_max=200, p=20, q=2,
                 n_records=64, seed=5000, philox_key=0x5EED0005),
}


def config(name: str, **overrides) -> Config:
    c = CONFIGS[name]
    if overrides:
        d = dict(c.__dict__)
        d.update(overrides)
        c = Config(**d)
    return c


@dataclass
class Modes:
    f: np.ndarray        # [M] Hz
    xi: np.ndarray       # [M] damping ratio
    phi: np.ndarray      # [M, l] real unit-norm mode shapes
    fs: float

    @property
    def lam(self) -> np.ndarray:
        """Continuous poles, Eq. (3)."""
        w = 2 * np.pi * self.f
        return -self.xi * w + 1j * w * np.sqrt(1 - self.xi ** 2)

    @property
    def mu(self) -> np.ndarray:
        """Discrete poles exp(lambda dt) of Eq. (5)'s A."""
        return np.exp(self.lam / self.fs)


def _unit(v):
    return v / np.linalg.norm(v)


def _bridge_shapes(rng, n_modes: int, stations: int = 64):
    """c3/c4/c5 mode shapes: 64 triaxial stations along a span, channel c = 3 s + a.
    Each mode gets a distinct (half-wave number h in 1..7, dominant axis a*) pair; the
    dominant axis has weight 1 and phase 0, the others weight U[0.05, 0.3] and phase
    U[0, pi]."""
    combos = [(h, a) for h in range(1, 8) for a in range(3)]
    pick = rng.permutation(len(combos))[:n_modes]
    x = (np.arange(stations) + 0.5) / stations
    phi = np.zeros((n_modes, 3 * stations))
    for m, ci in enumerate(pick):
        h, astar = combos[ci]
        for a in range(3):
            if a == astar:
                w, th = 1.0, 0.0
            else:
                w, th = rng.uniform(0.05, 0.3), rng.uniform(0.0, np.pi)
            phi[m, a::3] = w * np.sin(np.pi * h * x + th)
        phi[m] = _unit(phi[m])
    return phi


def make_modes(cfg: Config, record: int = 0) -> Modes:
    """Mode parameters (draw order: frequencies, damping, shapes)."""
    if cfg.name == "c1":
        rng = np.random.default_rng(cfg.seed)
        f = np.array([1.2, 3.5, 7.1])
        xi = np.array([0.01, 0.015, 0.02])
        phi = np.stack([_unit(rng.standard_normal(cfg.l)) for _ in range(3)])
        return Modes(f, xi, phi, cfg.fs)
    if cfg.name == "c2":
        rng = np.random.default_rng(cfg.seed)
        f = np.sort(rng.uniform(0.8, 12.0, 10))
        xi = rng.uniform(0.005, 0.03, 10)
        phi = np.stack([_unit(rng.standard_normal(cfg.l)) for _ in range(10)])
        return Modes(f, xi, phi, cfg.fs)
    # c3 / c4 / c5 share the bridge model drawn from seed 3
    rng = np.random.default_rng(3)
    while True:
        f = np.sort(rng.uniform(0.5, 15.0, 20))
        if np.all(np.diff(f) / f[1:] >= 0.03):
            break
    xi = rng.uniform(0.005, 0.03, 20)
    phi = _bridge_shapes(rng, 20)
    if cfg.name == "c5":
        psi = np.random.default_rng(cfg.seed).uniform(0.0, 2 * np.pi, 20)
        f = f * (1.0 + 0.02 * np.sin(2 * np.pi * record / 64.0 + psi))
    return Modes(f, xi, phi, cfg.fs)


def _simulate(modes: Modes, N: int, noise_rms: float, rng) -> np.ndarray:
    """Record y[N][l] in FP64 (draw order: z0 per mode, innovations mode by mode
    (N-1) x 2, measurement noise N x l)."""
    M, l = modes.phi.shape
    mu = modes.mu
    r = np.abs(mu)
    g = np.sqrt(1.0 - r ** 2)
    z0 = rng.standard_normal((M, 2))
    y = np.zeros((N, l))
    for m in range(M):
        w = rng.standard_normal((N - 1, 2))
        x = g[m] * (w[:, 0] + 1j * w[:, 1])
        zi = np.array([mu[m] * (z0[m, 0] + 1j * z0[m, 1])])
        z = np.empty(N, dtype=np.complex128)
        z[0] = z0[m, 0] + 1j * z0[m, 1]
        z[1:], _ = lfilter([1.0], [1.0, -mu[m]], x, zi=zi)
        y += np.outer(z.real, modes.phi[m])
    rho = np.sqrt((modes.phi ** 2).sum(axis=0))          # exact stationary clean RMS
    y += rng.standard_normal((N, l)) * (noise_rms * rho)
    return y


def make_record(cfg: Config, record: int = 0, N: int | None = None):
    """(Y, modes): Y is [N][l] time-major, float64 for c1 and float32 otherwise."""
    modes = make_modes(cfg, record)
    seed = cfg.seed + record if cfg.name == "c5" else cfg.seed
    # a stream separate from the mode-parameter draws, so realizations are independent
    rng = np.random.default_rng([seed, 0xC0FFEE])
    y = _simulate(modes, N or cfg.N, cfg.noise_rms, rng)
    if cfg.dtype == "f32":
        y = y.astype(np.float32)
    return np.ascontiguousarray(y), modes


def make_batch_record(cfg: Config, record: int, N: int | None = None):
    return make_record(cfg, record, N)


def exact_poles(modes: Modes):
    """Generating (f, xi) sorted by f; used by statistical end-to-end checks (P17)."""
    o = np.argsort(modes.f)
    return modes.f[o], modes.xi[o]
