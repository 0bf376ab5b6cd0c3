"""Full-size parity in bench.py's launch configuration (-m gpu): spectral covariances (segment
FFTs + cross-spectral FP64 DMMA products; the int8x3 tcgen05 path checked beside them on c3),
FP64 RSVD, per-order eigen-solves, through the same drivers the bench uses, against the FP64
oracle run end to end on the same synthetic records.

Contract (north star): covariances rel. Frobenius <= 1e-4 (split path); leading singular
values <= 1e-5; every oracle-stable pole |df|/f <= 1e-5 and |dxi| <= 1e-4; pole counts and
stable counts equal per (lag, order) cell. Non-stable (spurious) poles are reported."""
import numpy as np
import pytest

import oracle
import synth
from tests.parity import gpu_cells, compare_tables

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2411_05510_b200 import api, drivers, build
    build.build()
    return api, drivers


def _params(drivers, cfg, mode="spectral", i=None):
    return drivers.SweepParams(l=cfg.l, i=i or cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs,
                               n_min=cfg.n_min, n_step=cfg.n_step, seed=cfg.philox_key, cov_mode=mode)


def _check_contract(st, label):
    print(f"{label}: {st['n_poles']} poles, {st['n_stable']} oracle-stable; max df/f stable "
          f"{st['max_df_stable']:.2e} all {st['max_df_all']:.2e}; max dxi stable {st['max_dxi_stable']:.2e} "
          f"all {st['max_dxi_all']:.2e}; count mismatches {st['count_mismatch']}")
    assert st["count_mismatch"] == []
    assert st["n_stable"] > 0
    assert st["max_df_stable"] <= 1e-5
    assert st["max_dxi_stable"] <= 1e-4


def test_c3_record_full_size(mods):
    """The metric's workload: one c3 record (l=192, N=360000, i=60, k=220, q=2, 100 orders)."""
    api, drivers = mods
    cfg = synth.config("c3")
    Y, _ = synth.make_record(cfg)
    P = _params(drivers, cfg)
    eng = drivers.Engine(P, cfg.N)
    Yd = torch.from_numpy(Y).cuda()
    R = eng.covariances(Yd).cpu().numpy()
    tab, (U, S) = eng.decompose(eng.R, cfg.i, stream_id=cfg.i)
    torch.cuda.synchronize()
    for ws in (eng.ws_cov, eng.ws_rsvd, eng.ws_modal):
        assert api.device_status(ws) == 0

    Ro = oracle.covariances(Y, 2 * cfg.i - 1)
    cov_err = np.linalg.norm(R - Ro) / np.linalg.norm(Ro)
    assert cov_err <= 1e-6                                   # contract (FP64 path)
    assert cov_err <= 1e-12                                  # measured 1.6e-14
    R8 = api.covariances(Yd, 2 * cfg.i - 1, mode="int8x3", check=True).cpu().numpy()
    i8_err = np.linalg.norm(R8 - Ro) / np.linalg.norm(Ro)
    print(f"c3: int8x3 covariances rel {i8_err:.2e}")
    assert i8_err <= 1e-8                                    # measured 4e-9
    To = oracle.toeplitz(Ro, cfg.i)
    Uo, So, _ = oracle.rsvd(To, cfg.k, cfg.q, cfg.philox_key, cfg.i, cfg.n_max)
    s_err = np.max(np.abs(S.cpu().numpy()[:cfg.n_max] - So[:cfg.n_max]) / So[:cfg.n_max])
    print(f"c3: cov rel {cov_err:.2e}, leading sigma rel {s_err:.2e}")
    assert s_err <= 1e-5
    cells = oracle.modal_sweep(Uo, So, cfg.l, cfg.i, cfg.orders, cfg.dt)
    crit = oracle.SC_BRIDGE_3D
    flags_o, counts_o = oracle.stab3d([cells], crit, cfg.n_max // 2)
    st = compare_tables(gpu_cells(tab), cells, flags_o[0])
    _check_contract(st, "c3")
    _, counts = api.stab3d([tab], api.Criteria(**crit.__dict__))
    assert np.array_equal(counts.cpu().numpy(), counts_o)


def test_c4_lag_sweep_subset(mods):
    """3D sweep (config c4 record and parameters) over four consecutive lags of its grid:
    covariances once to lag 2 max(i) - 1, per-lag RSVD + modal sweep, 3D flags."""
    api, drivers = mods
    cfg = synth.config("c4")
    lags = [52, 56, 60, 64]
    Y, _ = synth.make_record(cfg)
    P = _params(drivers, cfg, i=max(lags))
    crit = oracle.SC_BRIDGE_3D
    tables, flags, counts = drivers.lag_sweep_3d(torch.from_numpy(Y).cuda(), P, lags,
                                                 api.Criteria(**crit.__dict__))
    Ro = oracle.covariances(Y, 2 * max(lags) - 1)
    cells_o = []
    for i in lags:
        To = oracle.toeplitz(Ro, i)
        Uo, So, _ = oracle.rsvd(To, cfg.k, cfg.q, cfg.philox_key, i, cfg.n_max)
        cells_o.append(oracle.modal_sweep(Uo, So, cfg.l, i, cfg.orders, cfg.dt))
    flags_o, counts_o = oracle.stab3d(cells_o, crit, cfg.n_max // 2)
    for g, i in enumerate(lags):
        _check_contract(compare_tables(gpu_cells(tables[i]), cells_o[g], flags_o[g]), f"c4 lag {i}")
    assert np.array_equal(counts.cpu().numpy(), counts_o)


def test_c5_record_batch_subset(mods):
    """Continuous monitoring (config c5: drifting model, i=50): two records through the
    multi-stream record pipeline, each against the oracle."""
    api, drivers = mods
    cfg = synth.config("c5")
    recs = [synth.make_record(cfg, r)[0] for r in (0, 17)]
    P = _params(drivers, cfg)
    tabs = drivers.record_batch([torch.from_numpy(y).cuda() for y in recs], P, n_streams=2)
    crit = oracle.SC_BRIDGE_3D
    for j, Y in enumerate(recs):
        Ro = oracle.covariances(Y, 2 * cfg.i - 1)
        Uo, So, _ = oracle.rsvd(oracle.toeplitz(Ro, cfg.i), cfg.k, cfg.q, cfg.philox_key, (j << 32) | cfg.i,
                                cfg.n_max)
        cells = oracle.modal_sweep(Uo, So, cfg.l, cfg.i, cfg.orders, cfg.dt)
        flags_o, counts_o = oracle.stab3d([cells], crit, cfg.n_max // 2)
        _check_contract(compare_tables(gpu_cells(tabs[j]), cells, flags_o[0]), f"c5 record {j}")
        _, counts = api.stab3d([tabs[j]], api.Criteria(**crit.__dict__))
        assert np.array_equal(counts.cpu().numpy(), counts_o)


def test_c4_full_lag_sweep(mods):
    """The whole c4 sweep (i = 20..80 step 4, 16 lags up to m = 15360) through drivers.lag_sweep_3d:
    poles at the smallest and largest lag against the oracle, and ssi_stab3d over all 16 GPU
    tables against the oracle's stab3d applied to the same tables."""
    api, drivers = mods
    cfg = synth.config("c4")
    lags = list(cfg.lags)
    Y, _ = synth.make_record(cfg)
    P = _params(drivers, cfg, i=max(lags))
    crit = oracle.SC_BRIDGE_3D
    tables, flags, counts = drivers.lag_sweep_3d(torch.from_numpy(Y).cuda(), P, lags,
                                                 api.Criteria(**crit.__dict__))
    torch.cuda.synchronize()
    Ro = oracle.covariances(Y, 2 * max(lags) - 1)
    for i in (lags[0], lags[-1]):
        To = oracle.toeplitz(Ro, i)
        Uo, So, _ = oracle.rsvd(To, cfg.k, cfg.q, cfg.philox_key, i, cfg.n_max)
        cells = oracle.modal_sweep(Uo, So, cfg.l, i, cfg.orders, cfg.dt)
        flags_o, _ = oracle.stab3d([cells], crit, cfg.n_max // 2)
        _check_contract(compare_tables(gpu_cells(tables[i]), cells, flags_o[0]), f"c4 full sweep, lag {i}")
    gcells = [gpu_cells(tables[i]) for i in lags]
    flags_ref, counts_ref = oracle.stab3d(gcells, crit, cfg.n_max // 2)
    assert np.array_equal(counts.cpu().numpy(), counts_ref)
    assert np.array_equal(flags.cpu().numpy(), flags_ref)


def test_c5_batch_eight_records(mods):
    """Continuous monitoring in bench.py's launch configuration (RecordPipeline, 8 streams,
    records in flight): 8 drifting c5 records; two sampled records against the oracle, and every
    record's table equal to the same record identified alone (stream pipelining changes nothing)."""
    api, drivers = mods
    cfg = synth.config("c5")
    recs = [synth.make_record(cfg, r)[0] for r in range(8)]
    P = _params(drivers, cfg)
    dev = [torch.from_numpy(y).cuda() for y in recs]
    tabs = drivers.record_batch(dev, P, n_streams=8)
    crit = oracle.SC_BRIDGE_3D
    for j in (0, 7):
        Ro = oracle.covariances(recs[j], 2 * cfg.i - 1)
        Uo, So, _ = oracle.rsvd(oracle.toeplitz(Ro, cfg.i), cfg.k, cfg.q, cfg.philox_key, (j << 32) | cfg.i,
                                cfg.n_max)
        cells = oracle.modal_sweep(Uo, So, cfg.l, cfg.i, cfg.orders, cfg.dt)
        flags_o, _ = oracle.stab3d([cells], crit, cfg.n_max // 2)
        _check_contract(compare_tables(gpu_cells(tabs[j]), cells, flags_o[0]), f"c5 batch record {j}")
    eng = drivers.Engine(P, cfg.N)
    for j in range(8):
        alone = eng.identify(dev[j], stream_id=(j << 32) | cfg.i)
        torch.cuda.synchronize()
        for a, b in zip(alone.tensors(), tabs[j].tensors()):
            assert torch.equal(a, b), j          # bit-identical: fixed reduction orders
    # the same batch from pinned host records (RecordPipeline.submit_host: copy stream + input
    # ring) gives bit-identical tables
    host = [torch.from_numpy(y).pin_memory() for y in recs]
    tabs_h = drivers.record_batch(host, P, n_streams=3)
    for j in range(8):
        for a, b in zip(tabs_h[j].tensors(), tabs[j].tensors()):
            assert torch.equal(a, b), ("host record", j)
    # the tail hint (last records' covariances on the high-priority streams) is scheduling only
    for src, ns in ((dev, 8), (host, 3)):
        tabs_t = drivers.record_batch(src, P, n_streams=ns, tail=3)
        for j in range(8):
            for a, b in zip(tabs_t[j].tensors(), tabs[j].tensors()):
                assert torch.equal(a, b), ("tail hint", ns, j)
