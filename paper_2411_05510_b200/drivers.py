"""Drivers over the C ABI: one record (the metric's unit of work), the 3D lag sweep
(§2.3 steps i-ii) and the continuous-monitoring record batch
(PAPER.md:516-518). Buffers and workspaces are allocated once per shape and reused.

Multi-GPU (one process per GPU, torch.distributed over NCCL):
  * record batch: records are independent, assigned round-robin to ranks; no data-path
    collective (weak scaling); pole tables are gathered at the end.
  * lag sweep: the covariance sum is time-sharded across ranks (halo of lag_hi rows
    read by the kernel), partial FP64 sums are all-reduced once, then normalized; lags
    are assigned to ranks by LPT on the i^2 cost model; tables are gathered for stab3d.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import api


@dataclass(frozen=True)
class SweepParams:
    l: int
    i: int
    n_max: int
    p: int
    q: int
    fs: float
    n_min: int = 2
    n_step: int = 2
    seed: int = 0
    cov_mode: str = "fp64"

    @property
    def k(self):
        return self.n_max + self.p

    @property
    def m(self):
        return self.l * self.i

    @property
    def dt(self):
        return 1.0 / self.fs


class Engine:
    """Reusable device buffers for identify(); one Engine per (device, stream) user."""

    def __init__(self, P: SweepParams, N: int, device="cuda", lag_hi: int | None = None):
        self.P = P
        self.N = N
        self.dev = torch.device(device)
        self.lag_hi = lag_hi or 2 * P.i - 1
        d64 = dict(dtype=torch.float64, device=self.dev)
        self.R = torch.empty((self.lag_hi, P.l, P.l), **d64)
        self.T = torch.empty((P.m, P.m), **d64)
        self.U = torch.empty((P.n_max, P.m), **d64).t()          # column-major m x n_max
        self.S = torch.empty(P.k, **d64)
        self.table = api.PoleTable.empty(P.n_min, P.n_max, P.n_step, P.l, self.dev)
        self.ws_cov = api._workspace(api.covariances_ws_bytes(N, P.l, self.lag_hi, 1, P.cov_mode), self.dev)
        self.ws_rsvd = api._workspace(api.rsvd_ws_bytes(P.m, P.k, P.n_max), self.dev)
        self.ws_modal = api._workspace(
            api.modal_sweep_ws_bytes(P.l, P.i, P.n_min, P.n_max, P.n_step), self.dev)

    def covariances(self, Y):
        return api.covariances(Y, self.lag_hi, 1, self.P.cov_mode, out=self.R, ws=self.ws_cov)

    def decompose(self, R, i=None, stream_id=0):
        """Toeplitz + RSVD + modal sweep for time-lag step i from covariances R."""
        P = self.P
        i = i or P.i
        m = P.l * i
        if i == P.i:
            T, U, S = self.T, self.U, self.S
            api.toeplitz(R, i, out=T)
            api.rsvd_into(T, P.k, P.q, P.seed, stream_id, P.n_max, U, S, ws=self.ws_rsvd)
            tab = api.modal_sweep(U, S, P.l, i, P.n_min, P.n_max, P.n_step, P.dt, out=self.table,
                                  ws=self.ws_modal)
            return tab, (U, S)
        T = api.toeplitz(R, i, out=self.T.view(-1)[:m * m].view(m, m))
        U, S = api.rsvd(T, P.k, P.q, P.seed, stream_id, P.n_max, ws=self.ws_rsvd)
        return api.modal_sweep(U, S, P.l, i, P.n_min, P.n_max, P.n_step, P.dt, ws=self.ws_modal), (U, S)

    def identify(self, Y, stream_id=0):
        """A1-A11 for one record (the metric's unit of work)."""
        R = self.covariances(Y)
        tab, _ = self.decompose(R, self.P.i, stream_id)
        return tab


def identify_record(Y: torch.Tensor, P: SweepParams, stream_id: int = 0) -> api.PoleTable:
    return Engine(P, Y.shape[0], Y.device).identify(Y, stream_id)


class RecordPipeline:
    """Continuous-monitoring batch: records go round-robin to n_streams
    engines, each on its own CUDA stream, so one record's latency-bound kernels (Cholesky,
    Jacobi, per-order eigen-solves) overlap the tensor-core work of the next ones.
    submit() returns the engine's pole table, valid once that stream passes the record; an
    engine's table is reused n_streams submissions later."""

    def __init__(self, P: SweepParams, N: int, device="cuda", n_streams: int = 3):
        self.engines = [Engine(P, N, device) for _ in range(n_streams)]
        self.streams = [torch.cuda.Stream(device=device) for _ in range(n_streams)]
        self.j = 0

    def submit(self, Y: torch.Tensor, stream_id: int, events=None):
        e = self.engines[self.j % len(self.engines)]
        st = self.streams[self.j % len(self.streams)]
        self.j += 1
        with torch.cuda.stream(st):
            if events is not None:
                events[0].record(st)
            R = e.covariances(Y)
            if events is not None:
                events[1].record(st)
            tab, _ = e.decompose(R, e.P.i, stream_id)
        return tab, st

    def join(self, stream=None):
        """Make `stream` (default: current) wait for all pipeline streams."""
        cur = stream or torch.cuda.current_stream()
        for st in self.streams:
            cur.wait_stream(st)


# ------------------------------------------------------------------ multi-GPU host logic
def time_shards(N: int, world: int):
    """Contiguous time shards [t_b, t_e) of the covariance sum, one per rank."""
    base, rem = divmod(N, world)
    out, t = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((t, t + n))
        t += n
    return out


def lpt_assign(lags, world: int):
    """Longest-processing-time assignment of lags to ranks (cost ~ i^2: RSVD passes
    scale with m^2 = (l i)^2). Returns a list of lag lists, one per rank."""
    loads = [0.0] * world
    out = [[] for _ in range(world)]
    for lag in sorted(lags, key=lambda x: (-x, x)):
        r = min(range(world), key=lambda j: (loads[j], j))
        out[r].append(lag)
        loads[r] += float(lag) ** 2
    return [sorted(x) for x in out]


def allreduce_covariance_sums(S: torch.Tensor, N: int, lag_lo: int, group=None) -> torch.Tensor:
    """Sum time-sharded raw covariance sums over ranks, then divide by (N - k)
    (reading A-6). S: [L][l][l] FP64 on any backend's device."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(S, op=dist.ReduceOp.SUM, group=group)
    k = torch.arange(lag_lo, lag_lo + S.shape[0], dtype=torch.float64, device=S.device)
    return S / (N - k).view(-1, 1, 1)


def sharded_covariances(Y: torch.Tensor, lag_hi: int, rank: int, world: int, mode="fp64",
                        group=None) -> torch.Tensor:
    """Time-sharded A1 across ranks + one all-reduce (the lag sweep's only exchange)."""
    N = Y.shape[0]
    tb, te = time_shards(N, world)[rank]
    S = api.covariances(Y, lag_hi, 1, mode, t_begin=tb, t_end=te, normalize=False)
    return allreduce_covariance_sums(S, N, 1, group)


def record_assignment(n_records: int, world: int):
    return [list(range(r, n_records, world)) for r in range(world)]


def lag_sweep_3d(Y: torch.Tensor, P: SweepParams, lags, crit: api.Criteria, rank=0, world=1,
                 group=None):
    """3D stabilization diagram: covariances once to lag 2 max(i) - 1
    (time-sharded), RSVD + modal sweep per lag (LPT-sharded), all-gather, stab3d."""
    lag_hi = 2 * max(lags) - 1
    R = sharded_covariances(Y, lag_hi, rank, world, P.cov_mode, group)
    mine = lpt_assign(lags, world)[rank]
    eng = Engine(P, Y.shape[0], Y.device, lag_hi=lag_hi)
    eng.T = torch.empty((P.l * max(lags), P.l * max(lags)), dtype=torch.float64, device=Y.device)
    tables = {}
    for i in mine:
        Pi = SweepParams(**{**P.__dict__, "i": i})
        e2 = Engine.__new__(Engine)
        e2.__dict__.update(eng.__dict__)
        e2.P = Pi
        e2.ws_rsvd = api._workspace(api.rsvd_ws_bytes(Pi.m, Pi.k, Pi.n_max), Y.device)
        e2.ws_modal = api._workspace(api.modal_sweep_ws_bytes(Pi.l, i, Pi.n_min, Pi.n_max, Pi.n_step), Y.device)
        m = Pi.m
        T = api.toeplitz(R, i, out=eng.T.view(-1)[:m * m].view(m, m))
        U, S = api.rsvd(T, Pi.k, Pi.q, Pi.seed, i, Pi.n_max, ws=e2.ws_rsvd)
        tables[i] = api.modal_sweep(U, S, Pi.l, i, Pi.n_min, Pi.n_max, Pi.n_step, Pi.dt, ws=e2.ws_modal)
    tables = gather_tables(tables, lags, rank, world, group)
    flags, counts = api.stab3d([tables[i] for i in sorted(lags)], crit)
    return tables, flags, counts


def gather_tables(local: dict, keys, rank: int, world: int, group=None) -> dict:
    """All-gather of fixed-size pole tables (the sweep's second collective)."""
    if world == 1:
        return local
    import torch.distributed as dist
    owner = {}
    for r, ks in enumerate(lpt_assign(keys, world) if isinstance(keys, list) else keys):
        for k in ks:
            owner[k] = r
    ref = next(iter(local.values())) if local else None
    out = {}
    for k in sorted(owner):
        src = owner[k]
        t = local.get(k) if src == rank else api.PoleTable.empty(
            ref.n_min, ref.n_min + (ref.n_orders - 1) * ref.n_step, ref.n_step, ref.l,
            ref.count.device, ref.cap)
        for x in t.tensors():
            dist.broadcast(x, src=src, group=group)
        out[k] = t
    return out
