"""Multi-GPU host logic on CPU (-m "not gpu"): world-size-2 gloo process groups exercise the
exchange steps of the lag sweep and the record batch without a GPU. The covariance shards
are computed here by the oracle (test infrastructure) standing in for ssi_covariances'
raw-sum mode; the product code under test is drivers.allreduce_sums (the one exchange of
the time-sharded covariances; the 1/(N-k) that follows runs in libssi, ssi_cov_normalize,
covered by the GPU tests), drivers.gather_tables (one packed all_gather) and the
assignment helpers."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2411_05510_b200 import api, drivers


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _record():
    rng = np.random.default_rng(31)
    return rng.standard_normal((2003, 5))


def _cov_rank(rank, world):
    Y = _record()
    tb, te = drivers.time_shards(Y.shape[0], world)[rank]
    S = torch.from_numpy(oracle.covariance_partial_sums(Y, 1, 17, tb, te))
    return drivers.allreduce_sums(S).numpy()


def test_time_sharded_covariance_allreduce_gloo():
    """Lag sweep exchange step: per-rank time shards (halo read by the kernel), one
    all-reduce of raw FP64 sums — equals the full-record raw sums on every rank."""
    out = _spawn(_cov_rank)
    Y = _record()
    ref = oracle.covariance_partial_sums(Y, 1, 17, 0, Y.shape[0])
    for r in (0, 1):
        np.testing.assert_allclose(out[r], ref, rtol=1e-12, atol=1e-12)
    assert np.array_equal(out[0], out[1])          # every rank holds identical sums


def _fake_table(key, n_min=2, n_max=10, l=3):
    t = api.PoleTable.empty(n_min, n_max, 2, l, "cpu")
    for x in t.tensors():
        x.copy_(torch.arange(x.numel(), dtype=x.dtype).reshape(x.shape) * 0 + key)
    return t


def _gather_rank(rank, world):
    lags = list(range(20, 81, 4))
    assign = drivers.lpt_assign(lags, world)
    local = {i: _fake_table(i) for i in assign[rank]}
    tabs = drivers.gather_tables(local, assign, lambda: api.PoleTable.empty(2, 10, 2, 3, "cpu"), rank, world)
    return {i: float(tabs[i].f.mean()) for i in lags}


def test_gather_tables_gloo():
    """Lag sweep / record batch collective: every rank ends with every (lag) table."""
    out = _spawn(_gather_rank)
    lags = list(range(20, 81, 4))
    for r in (0, 1):
        assert sorted(out[r]) == lags
        assert all(out[r][i] == float(i) for i in lags)


def _gather_uneven_rank(rank, world):
    # 3 tables over 2 ranks: rank 0 owns two, rank 1 one (padding of the packed buffer)
    assign = [[0, 2], [1]]
    local = {}
    for key in assign[rank]:
        t = api.PoleTable.empty(2, 8, 2, 3, "cpu")
        g = torch.Generator().manual_seed(key)
        for x in t.tensors():
            x.copy_((torch.rand(x.shape, generator=g, dtype=torch.float64) * 1000).to(x.dtype))
        local[key] = t
    tabs = drivers.gather_tables(local, assign, lambda: api.PoleTable.empty(2, 8, 2, 3, "cpu"), rank, world)
    return {k: [x.numpy().copy() for x in tabs[k].tensors()] for k in (0, 1, 2)}


def test_gather_tables_bytes_exact_gloo():
    """The packed all_gather moves every array of every table bit for bit (int32 counts too)."""
    out = _spawn(_gather_uneven_rank)
    for k in (0, 1, 2):
        for a, b in zip(out[0][k], out[1][k]):
            assert a.dtype == b.dtype and np.array_equal(a, b)
    assert out[0][1][0].dtype == np.int32


def test_pack_unpack_roundtrip():
    t = api.PoleTable.empty(2, 6, 2, 2, "cpu")
    for j, x in enumerate(t.tensors()):
        x.copy_(torch.arange(x.numel()).reshape(x.shape).to(x.dtype) + j)
    buf = drivers.pack_tables([t, t], "cpu")
    u = drivers.unpack_table(buf[: buf.numel() // 2], api.PoleTable.empty(2, 6, 2, 2, "cpu"))
    for a, b in zip(t.tensors(), u.tensors()):
        assert torch.equal(a, b)


def test_assignment_helpers():
    lags = list(range(20, 81, 4))                  # config c4
    for G in (1, 2, 4, 8):
        a = drivers.lpt_assign(lags, G)
        assert sorted(sum(a, [])) == lags
        loads = [sum(i * i for i in x) for x in a]
        assert max(loads) <= max(sum(i * i for i in lags) / G, 80 ** 2) * 1.15 + 1
        sh = drivers.time_shards(360000, G)
        assert sh[0][0] == 0 and sh[-1][1] == 360000
        assert all(sh[j][1] == sh[j + 1][0] for j in range(G - 1))
        rec = drivers.record_assignment(64, G)             # config c5
        assert sorted(sum(rec, [])) == list(range(64)) and len({len(x) for x in rec}) == 1
