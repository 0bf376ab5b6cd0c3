"""SSI_COV_INT8X3 (tcgen05 kind::i8, exact int32 slice sums) vs the FP64 oracle (-m gpu).

Contract: relative Frobenius error <= 1e-4 for the split-precision path (north star).
Internal tripwire: <= 1e-7, well above the slicing bound (each sample is represented to
2^-21 of its channel's max), so a descriptor, TMA or accumulator bug cannot hide."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2411_05510_b200 import api, build
    build.build()
    return api


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("N,l,lag_hi", [(5000, 64, 40), (3001, 128, 17), (20000, 192, 119), (700, 64, 33),
                                         (4000, 48, 59), (1000, 16, 3)])
def test_int8x3_random_records(api, N, l, lag_hi):
    rng = np.random.default_rng(N + l)
    Y = (rng.standard_normal((N, l)) * rng.uniform(0.1, 10, l)).astype(np.float32)
    R = api.covariances(torch.from_numpy(Y).cuda(), lag_hi, mode="int8x3", check=True).cpu().numpy()
    Ro = oracle.covariances(Y, lag_hi)
    assert _rel(R, Ro) <= 1e-4            # contract
    # white noise: R_k ~ 1/sqrt(N) of the signal; compare against the diagonal scale
    scale = np.sqrt(np.mean(Y.astype(np.float64) ** 2, axis=0))
    err = np.abs(R - Ro) / np.outer(scale, scale)[None]
    assert err.max() <= 1e-5


def test_int8x3_c3_shaped_record(api):
    """c3 model (l=192, bridge shapes, 5% noise), 40000 samples, all 119 lags."""
    cfg = synth.config("c3")
    Y, _ = synth.make_record(cfg, N=40000)
    R = api.covariances(torch.from_numpy(Y).cuda(), 119, mode="int8x3", check=True).cpu().numpy()
    Ro = oracle.covariances(Y, 119)
    e = _rel(R, Ro)
    assert e <= 1e-4                      # contract
    assert e <= 1e-7                      # internal tripwire
    for k in range(119):
        assert _rel(R[k], Ro[k]) <= 1e-6


def test_int8x3_c2_record(api):
    """c2 (l = 48, N = 180000 FP32): the split path against the FP64 oracle."""
    cfg = synth.config("c2")
    Y, _ = synth.make_record(cfg)
    R = api.covariances(torch.from_numpy(Y).cuda(), 119, mode="int8x3", check=True).cpu().numpy()
    Ro = oracle.covariances(Y, 119)
    assert _rel(R, Ro) <= 1e-7


def test_int8x3_time_shards(api):
    """Raw shard sums add up to the full sums (scales are per whole record)."""
    rng = np.random.default_rng(5)
    Y = rng.standard_normal((9000, 64)).astype(np.float32)
    Yd = torch.from_numpy(Y).cuda()
    tot = 0
    for tb, te in ((0, 3001), (3001, 6007), (6007, 9000)):
        tot = tot + api.covariances(Yd, 50, 1, mode="int8x3", t_begin=tb, t_end=te, normalize=False,
                                    check=True).cpu().numpy()
    full = oracle.covariance_partial_sums(Y, 1, 50)
    # white noise: the sums are O(sqrt(N)); judge the error against the N sigma^2 scale
    # (slicing error ~4e-7 sigma per sample -> ~1e-8 at the max over 2e5 entries)
    assert np.max(np.abs(tot - full)) / 9000.0 <= 5e-8


def test_int8x3_unsupported_width_rejected(api):
    from paper_2411_05510_b200._lib import SSIError
    Y = torch.zeros((100, 40), dtype=torch.float32, device="cuda")
    with pytest.raises(SSIError) as e:
        api.covariances(Y, 5, mode="int8x3")
    assert e.value.code == 3
