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

import math
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
    cov_mode: str = "spectral"
    structured: bool = True     # RSVD through the block structure of T (T never formed)
    rank_rule: bool = False     # k = ceil(kbar(T) % T) per lag instead of n_max + p

    @property
    def k(self):
        return self.k_for(self.i)

    def k_for(self, i: int) -> int:
        """Sketch width at time-lag step i: n_max + p (north star), or the paper's rank rule
        k = ceil(kbar(T) % * T), kbar(T) = max{30 - 0.00156 T; 25} % with T = l i (Eq.
        empirical_formula)."""
        if not self.rank_rule:
            return self.n_max + self.p
        T = self.l * i
        pct = max(30.0 - 0.00156 * T, 25.0)
        return max(self.n_max, min(T, math.ceil(pct * T / 100.0 - 1e-9)))

    @property
    def m(self):
        return self.l * self.i

    @property
    def dt(self):
        return 1.0 / self.fs


def check_status(workspaces, what: str) -> None:
    """Raise if any call that used one of `workspaces` reported a device-side numeric failure
    (the status word accumulates across calls; reading it synchronises the current stream)."""
    for ws in workspaces:
        code = api.device_status(ws)
        if code != 0:
            from . import _lib
            raise _lib.SSIError(what + " (device status)", code)


class Engine:
    """Reusable device buffers for identify(); one Engine per (device, stream) user."""

    def __init__(self, P: SweepParams, N: int, device="cuda", lag_hi: int | None = None):
        self.P = P
        self.N = N
        self.dev = torch.device(device)
        self.lag_hi = lag_hi or 2 * P.i - 1
        d64 = dict(dtype=torch.float64, device=self.dev)
        self.R = torch.empty((self.lag_hi, P.l, P.l), **d64)
        self.T = None if P.structured else torch.empty((P.m, P.m), **d64)
        self.U = torch.empty((P.n_max, P.m), **d64).t()          # column-major m x n_max
        self.S = torch.empty(P.k, **d64)
        self.table = api.PoleTable.empty(P.n_min, P.n_max, P.n_step, P.l, self.dev)
        self.ws_cov = api._workspace(api.covariances_ws_bytes(N, P.l, self.lag_hi, 1, P.cov_mode), self.dev)
        self.ws_rsvd = api._workspace(
            api.rsvd_toeplitz_ws_bytes(P.l, P.i, P.k, P.n_max) if P.structured
            else api.rsvd_ws_bytes(P.m, P.k, P.n_max), self.dev)
        self.ws_modal = api._workspace(
            api.modal_sweep_ws_bytes(P.l, P.i, P.n_min, P.n_max, P.n_step), self.dev)

    def covariances(self, Y):
        return api.covariances(Y, self.lag_hi, 1, self.P.cov_mode, out=self.R, ws=self.ws_cov)

    def decompose(self, R, i=None, stream_id=0):
        """Toeplitz + RSVD + modal sweep for time-lag step i from covariances R."""
        P = self.P
        i = i or P.i
        m = P.l * i
        if P.structured:
            if i == P.i:
                U, S = api.rsvd_toeplitz(R, i, P.k, P.q, P.seed, stream_id, P.n_max, U=self.U, S=self.S,
                                         ws=self.ws_rsvd)
                tab = api.modal_sweep(U, S, P.l, i, P.n_min, P.n_max, P.n_step, P.dt, out=self.table,
                                      ws=self.ws_modal)
            else:
                U, S = api.rsvd_toeplitz(R, i, P.k_for(i), P.q, P.seed, stream_id, P.n_max, ws=self.ws_rsvd)
                tab = api.modal_sweep(U, S, P.l, i, P.n_min, P.n_max, P.n_step, P.dt, ws=self.ws_modal)
            return tab, (U, S)
        if i == P.i:
            T, U, S = self.T, self.U, self.S
            api.toeplitz(R, i, out=T)
            api.rsvd_into(T, P.k, P.q, P.seed, stream_id, P.n_max, U, S, ws=self.ws_rsvd)
            tab = api.modal_sweep(U, S, P.l, i, P.n_min, P.n_max, P.n_step, P.dt, out=self.table,
                                  ws=self.ws_modal)
            return tab, (U, S)
        T = api.toeplitz(R, i, out=self.T.view(-1)[:m * m].view(m, m))
        U, S = api.rsvd(T, P.k_for(i), P.q, P.seed, stream_id, P.n_max, ws=self.ws_rsvd)
        return api.modal_sweep(U, S, P.l, i, P.n_min, P.n_max, P.n_step, P.dt, ws=self.ws_modal), (U, S)

    def workspaces(self):
        return (self.ws_cov, self.ws_rsvd, self.ws_modal)

    def identify(self, Y, stream_id=0, check: bool = True):
        """A1-A11 for one record (the metric's unit of work). check: synchronise and raise if any
        call so far on this engine reported a device-side numeric failure."""
        R = self.covariances(Y)
        tab, _ = self.decompose(R, self.P.i, stream_id)
        if check:
            check_status(self.workspaces(), "identify")
        return tab


def identify_record(Y: torch.Tensor, P: SweepParams, stream_id: int = 0) -> api.PoleTable:
    return Engine(P, Y.shape[0], Y.device).identify(Y, stream_id)


class RecordPipeline:
    """Continuous-monitoring batch: records go round-robin to n_streams
    engines, each on its own CUDA stream, so one record's latency-bound kernels (Cholesky,
    Jacobi, per-order eigen-solves) overlap the tensor-core work of the next ones.
    submit() returns the engine's pole table, valid once that stream passes the record; an
    engine's table is reused n_streams submissions later."""

    def __init__(self, P: SweepParams, N: int, device="cuda", n_streams: int = 3, split_priority: bool = True):
        self.engines = [Engine(P, N, device) for _ in range(n_streams)]
        # the latency-bound chain (RSVD: Cholesky, Jacobi; modal sweep: per-order eigen-solves)
        # runs on high-priority streams so its small launches are scheduled ahead of the wide
        # covariance grids of other records, which run on low-priority streams
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
        self.split = split_priority
        self.streams = [torch.cuda.Stream(device=device, priority=hi if split_priority else 0)
                        for _ in range(n_streams)]
        self.cov_streams = ([torch.cuda.Stream(device=device, priority=lo) for _ in range(n_streams)]
                            if split_priority else self.streams)
        self.j = 0
        self.device = torch.device(device)
        # host records (submit_host): a ring of device input buffers filled on one copy stream
        self._in_bufs, self._in_free, self._hb = [], [], 0
        self.copy_stream = None

    def submit(self, Y: torch.Tensor, stream_id: int, events=None, ready: torch.cuda.Event | None = None,
               tail: bool = False):
        """tail: no record will follow this one soon (the end of a batch). Its covariances then run
        on the engine's high-priority stream: with nothing behind it to fill the gaps, a low-priority
        A1 would only delay the start of this record's latency-bound chain (same kernels, same
        results; scheduling only)."""
        tab, st, _ = self._submit(Y, stream_id, events, ready, tail)
        return tab, st

    def _submit(self, Y, stream_id, events=None, ready=None, tail=False):
        k = self.j % len(self.engines)
        e, st = self.engines[k], self.streams[k]
        cst = st if tail else self.cov_streams[k]
        self.j += 1
        if ready is None:
            st.wait_stream(torch.cuda.current_stream(Y.device))   # Y was produced on the caller's stream
        if cst is not st:
            cst.wait_stream(st)            # the engine's buffers are free (and Y is ready on st)
        if ready is not None:
            cst.wait_event(ready)          # Y arrives from the copy stream
        else:
            Y.record_stream(cst)           # the caching allocator must not reuse Y before A1 read it
        with torch.cuda.stream(cst):
            if events is not None:
                events[0].record(cst)
            R = e.covariances(Y)
            if events is not None:
                events[1].record(cst)
            read = torch.cuda.Event()
            read.record(cst)               # A1 is the only reader of Y
        if cst is not st:
            st.wait_stream(cst)
        with torch.cuda.stream(st):
            tab, _ = e.decompose(R, e.P.i, stream_id)
        return tab, st, read

    def reserve_host_inputs(self, shape, dtype):
        """Allocate submit_host's device input ring (n_streams + 2 records) and copy stream now,
        so that no allocation happens while records stream through."""
        if not self._in_bufs:
            self.copy_stream = torch.cuda.Stream(device=self.device)
            self._in_bufs = [torch.empty(tuple(shape), dtype=dtype, device=self.device)
                             for _ in range(len(self.engines) + 2)]
            self._in_free = [None] * len(self._in_bufs)

    def submit_host(self, Yh: torch.Tensor, stream_id: int, events=None, tail: bool = False):
        """submit() for a record in (pinned) host memory. The host-to-device copy runs on the
        pipeline's copy stream into a ring of n_streams + 2 device buffers, so the copy of the
        next records overlaps the compute of the ones in flight; a buffer is refilled once the
        covariances (A1, its only reader) of its previous record are done. Returns (table,
        stream) like submit()."""
        self.reserve_host_inputs(Yh.shape, Yh.dtype)
        nbuf = len(self._in_bufs)
        b = self._hb % nbuf
        self._hb += 1
        buf = self._in_bufs[b]
        if buf.shape != Yh.shape or buf.dtype != Yh.dtype:
            raise ValueError(f"submit_host: record {tuple(Yh.shape)} {Yh.dtype} differs from the pipeline's "
                             f"{tuple(buf.shape)} {buf.dtype}")
        cs = self.copy_stream
        cs.wait_stream(torch.cuda.current_stream(self.device))    # Yh was produced before this call
        if self._in_free[b] is not None:
            cs.wait_event(self._in_free[b])
        with torch.cuda.stream(cs):
            buf.copy_(Yh, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(cs)
        tab, st, read = self._submit(buf, stream_id, events, ready, tail)
        self._in_free[b] = read
        return tab, st

    def check(self):
        """Raise if any record so far reported a device-side numeric failure (synchronises)."""
        for e in self.engines:
            check_status(e.workspaces(), "RecordPipeline")

    def join(self, stream=None):
        """Make `stream` (default: current) wait for all pipeline streams."""
        cur = stream or torch.cuda.current_stream()
        for st in self.streams:
            cur.wait_stream(st)
        if self.copy_stream is not None:
            cur.wait_stream(self.copy_stream)
        if self.split:
            for st in self.cov_streams:
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


def allreduce_sums(S: torch.Tensor, group=None) -> torch.Tensor:
    """Sum time-sharded raw covariance sums over ranks in place (one all-reduce; the lag sweep's
    only exchange). When the process group's backend cannot reduce device tensors (gloo), the
    sums are staged through host memory. No arithmetic of the method runs here."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return S
    if S.is_cuda and dist.get_backend(group) != "nccl":
        h = S.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        S.copy_(h)
    else:
        dist.all_reduce(S, op=dist.ReduceOp.SUM, group=group)
    return S


def sharded_covariances(Y: torch.Tensor, lag_hi: int, rank: int, world: int, mode="fp64",
                        group=None, out: torch.Tensor | None = None, ws: torch.Tensor | None = None) -> torch.Tensor:
    """Time-sharded A1 across ranks: raw sums over this rank's shard (ssi_covariances, normalize=0),
    one all-reduce, then 1/(N - k) on the device (ssi_cov_normalize)."""
    N = Y.shape[0]
    tb, te = time_shards(N, world)[rank]
    S = api.covariances(Y, lag_hi, 1, mode, t_begin=tb, t_end=te, normalize=False, out=out, ws=ws)
    if world > 1:                      # world = 1 is a local call even inside a process group
        allreduce_sums(S, group)
    return api.cov_normalize(S, N, 1)


def record_assignment(n_records: int, world: int):
    """Records are independent: round-robin over ranks."""
    return [list(range(r, n_records, world)) for r in range(world)]


def _segments(t: api.PoleTable):
    """Byte layout of one pole table in a packed buffer: (tensor, offset, nbytes), 16-byte aligned."""
    out, off = [], 0
    for x in t.tensors():
        nb = x.numel() * x.element_size()
        out.append((x, off, nb))
        off += (nb + 15) // 16 * 16
    return out, off


def pack_tables(tables, device) -> torch.Tensor:
    """Tables -> one contiguous uint8 buffer [len(tables)][table bytes] (byte copies only)."""
    tb = _segments(tables[0])[1] if tables else 0
    buf = torch.zeros(len(tables) * tb, dtype=torch.uint8, device=device)
    for j, t in enumerate(tables):
        for x, off, nb in _segments(t)[0]:
            buf[j * tb + off: j * tb + off + nb].copy_(x.contiguous().view(-1).view(torch.uint8))
    return buf


def unpack_table(buf: torch.Tensor, t: api.PoleTable) -> api.PoleTable:
    for x, off, nb in _segments(t)[0]:
        x.view(-1).view(torch.uint8).copy_(buf[off: off + nb])
    return t


def gather_tables(local: dict, assignment, make_empty, rank: int, world: int, group=None) -> dict:
    """All ranks receive every pole table: table key -> owner from `assignment` (a list of key
    lists, one per rank). Each rank packs its tables into one byte buffer, padded to the largest
    per-rank count, and ONE all_gather exchanges them (the sweep's / batch's last collective;
    ~31 MB per c3-sized table). Over gloo the buffer is staged through host memory.
    make_empty() allocates a table of the common shape."""
    if world == 1:
        return dict(local)
    import torch.distributed as dist
    proto = make_empty()
    tb = _segments(proto)[1]
    cap = max(len(k) for k in assignment)
    dev = proto.count.device
    mine = [local[key] for key in assignment[rank]]
    send = torch.zeros(cap * tb, dtype=torch.uint8, device=dev)
    if mine:
        send[: len(mine) * tb].copy_(pack_tables(mine, dev))
    if dist.get_backend(group) == "nccl":
        recv = torch.empty(world * cap * tb, dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(recv, send, group=group)
    else:
        parts = [torch.empty(cap * tb, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, send.cpu(), group=group)
        recv = torch.cat(parts).to(dev)
    out = {}
    for r, keys in enumerate(assignment):
        for j, key in enumerate(keys):
            if r == rank:
                out[key] = local[key]
            else:
                base = (r * cap + j) * tb
                out[key] = unpack_table(recv[base: base + tb], make_empty())
    return out


def run_lags(R: torch.Tensor, P: SweepParams, mine, n_streams: int = 8):
    """Toeplitz + RSVD + modal sweep for the time-lag steps `mine` from covariances R (lags
    independent: n_streams high-priority CUDA streams, largest lag first, each stream with its
    own workspaces). The streams are returned; the caller joins them. Returns (tables by lag,
    per-stream workspaces, streams)."""
    dev = R.device
    mine = sorted(mine, reverse=True)                    # largest lags first (longest chains)
    ns = min(n_streams, len(mine))                       # 0 when this rank got no lag
    cur = torch.cuda.current_stream(dev)
    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    streams = [torch.cuda.Stream(device=dev, priority=hi) for _ in range(ns)]
    slots = []
    for j in range(ns):
        lag_max = max(mine[j::ns])                       # workspaces sized for the slot's largest lag
        m_max = P.l * lag_max
        k_max = max(P.k_for(i) for i in mine[j::ns])
        if P.structured:
            ws_r = api._workspace(max(api.rsvd_toeplitz_ws_bytes(P.l, i, P.k_for(i), P.n_max) for i in mine[j::ns]), dev)
            tb = None
        else:
            ws_r = api._workspace(api.rsvd_ws_bytes(m_max, k_max, P.n_max), dev)
            tb = torch.empty(m_max * m_max, dtype=torch.float64, device=dev)
        ws_m = api._workspace(max(api.modal_sweep_ws_bytes(P.l, i, P.n_min, P.n_max, P.n_step)
                                  for i in mine[j::ns]), dev)
        slots.append((ws_r, tb, ws_m))
    local = {}
    for n_, i in enumerate(mine):
        j = n_ % ns
        st = streams[j]
        st.wait_stream(cur)                              # R (and the workspaces) are ready
        ws_r, tb, ws_m = slots[j]
        with torch.cuda.stream(st):
            m = P.l * i
            if P.structured:
                U, S = api.rsvd_toeplitz(R, i, P.k_for(i), P.q, P.seed, i, P.n_max, ws=ws_r)
            else:
                T = api.toeplitz(R, i, out=tb[:m * m].view(m, m))
                U, S = api.rsvd(T, P.k_for(i), P.q, P.seed, i, P.n_max, ws=ws_r)
            local[i] = api.modal_sweep(U, S, P.l, i, P.n_min, P.n_max, P.n_step, P.dt, ws=ws_m)
    return local, slots, streams


def lag_sweep_3d(Y: torch.Tensor, P: SweepParams, lags, crit: api.Criteria, rank: int = 0, world: int = 1,
                 group=None, n_streams: int = 8, timing: dict | None = None):
    """3D stabilization diagram (steps i-ii) for the time-lag steps `lags`:
    covariances once up to lag 2 max(i) - 1 (time-sharded over ranks + one all-reduce),
    Toeplitz + RSVD + modal sweep per lag (lags assigned by LPT; on a rank the lags are
    independent and run on `n_streams` CUDA streams, largest first, each stream with its own
    workspaces), all tables gathered, ssi_stab3d over the lag axis.
    timing: optional dict that receives CUDA events recorded on the current stream at the phase
    boundaries ("start", "cov" = covariances + all-reduce + normalisation, "lags", "gather",
    "stab").
    Returns ({i: PoleTable}, flags, stable_count)."""
    lags = sorted(lags)
    lag_hi = 2 * lags[-1] - 1
    dev = Y.device

    def mark(name):
        if timing is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(torch.cuda.current_stream(dev))
            timing[name] = ev

    mark("start")
    ws_c = api._workspace(api.covariances_ws_bytes(Y.shape[0], P.l, lag_hi, 1, P.cov_mode), dev)
    R = sharded_covariances(Y, lag_hi, rank, world, P.cov_mode, group, ws=ws_c)
    mark("cov")
    assign = lpt_assign(lags, world)
    local, slots, streams = run_lags(R, P, assign[rank], n_streams)
    cur = torch.cuda.current_stream(dev)
    for st in streams:
        cur.wait_stream(st)
    mark("lags")
    check_status([ws_c] + [w for sl in slots for w in (sl[0], sl[2])], "lag_sweep_3d")
    tables = gather_tables(local, assign, lambda: api.PoleTable.empty(P.n_min, P.n_max, P.n_step, P.l, dev),
                           rank, world, group)
    mark("gather")
    flags, counts = api.stab3d([tables[i] for i in lags], crit)
    mark("stab")
    return tables, flags, counts


def record_batch(records, P: SweepParams, rank: int = 0, world: int = 1, n_streams: int = 3, group=None,
                 gather: bool = True, tail: int = 0):
    """Continuous monitoring: records (a list of device tensors, or a
    callable j -> device tensor) processed on this rank by a RecordPipeline; tables gathered
    on every rank when `gather`. No data-path collective (records are independent). The last
    `tail` records of this rank are submitted with the pipeline's tail hint (scheduling only)."""
    n = len(records) if not callable(records) else records.n
    assign = record_assignment(n, world)
    fetch = records if callable(records) else (lambda j: records[j])
    first = fetch(assign[rank][0]) if assign[rank] else fetch(0)
    device = first.device if first.is_cuda else torch.device("cuda", torch.cuda.current_device())
    pipe = RecordPipeline(P, first.shape[0], device, n_streams)
    local = {}
    for n_done, j in enumerate(assign[rank]):
        Yj = fetch(j)
        last = n_done >= len(assign[rank]) - tail
        # host records (pinned) stream in through the pipeline's copy stream
        tab, st = (pipe.submit(Yj, (j << 32) | P.i, tail=last) if Yj.is_cuda
                   else pipe.submit_host(Yj, (j << 32) | P.i, tail=last))
        with torch.cuda.stream(st):
            local[j] = api.PoleTable(tab.n_min, tab.n_step, tab.l, tab.cap, *[t.clone() for t in tab.tensors()])
    pipe.join()
    torch.cuda.current_stream().synchronize()
    pipe.check()
    if not gather:
        return local
    return gather_tables(local, assign, lambda: api.PoleTable.empty(P.n_min, P.n_max, P.n_step, P.l, device),
                         rank, world, group)


# ------------------------------------------------------------------ NEXT-2: step iii + tracking
def identify_3d(Y: torch.Tensor, P: SweepParams, lags, crit: api.Criteria, cutoff: float = 0.10,
                min_size: int | None = None, rank: int = 0, world: int = 1, group=None, n_streams: int = 8,
                timing: dict | None = None):
    """The whole 3D-RSVD identification (§2.3 steps i-iii): lag sweep and 3D
    stabilization (lag_sweep_3d), then the two-stage clustering of the stable poles (api.cluster3d;
    every rank clusters the gathered diagram). min_size defaults to 20 % of the diagram's
    (lag, order) cells (the share used in the NEXT-2 tests of the paper's frame).
    Returns (tables, flags, stable_count, Clustering)."""
    lags = sorted(lags)
    tables, flags, counts = lag_sweep_3d(Y, P, lags, crit, rank, world, group, n_streams, timing)
    O = tables[lags[0]].n_orders
    ms = min_size if min_size is not None else max(1, int(0.2 * O * len(lags)))
    cl = api.cluster3d([tables[i] for i in lags], flags, crit, cutoff=cutoff, min_size=ms)
    if timing is not None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream(Y.device))
        timing["cluster"] = ev
    return tables, flags, counts, cl


def session_modes(tab: api.PoleTable, crit: api.Criteria, cutoff: float = 0.10, min_size: int | None = None):
    """Modes of one monitoring session from its (single-lag) stabilization diagram: stab3d with
    one lag (the 2D order-axis criteria), then the two-stage clustering."""
    flags, _ = api.stab3d([tab], crit)
    ms = min_size if min_size is not None else max(1, int(0.2 * tab.n_orders))
    return api.cluster3d([tab], flags, crit, cutoff=cutoff, min_size=ms)


def track_campaign(tables, crit: api.Criteria, max_modes: int = 64, df_max: float = 0.05,
                   macd_max: float = 0.15, cutoff: float = 0.10, min_size: int | None = None, ref=None):
    """Modal tracking over a campaign (§3.2.2; Table 4): every session's modes from
    session_modes(); reference modes = those of the first session unless `ref` = (f, shape) is
    given ("The reference modal properties are those identified ... from the first acquisition
    record", Table 4). Returns (match [S][R], success [R] in %, ref_f, ref_shape)."""
    dev = tables[0].count.device
    sess = [session_modes(t, crit, cutoff, min_size) for t in tables]
    l = tables[0].l
    S = len(sess)
    f = torch.zeros((S, max_modes), dtype=torch.float64, device=dev)
    sh = torch.zeros((S, max_modes, l, 2), dtype=torch.float64, device=dev)
    cnt = torch.zeros(S, dtype=torch.int32, device=dev)
    for s, c in enumerate(sess):
        k = min(c.n_clusters, max_modes)
        f[s, :k] = c.f[:k]
        sh[s, :k] = c.shape[:k]
        cnt[s] = k
    if ref is None:
        k0 = int(cnt[0])
        ref_f, ref_shape = f[0, :k0].contiguous(), sh[0, :k0].contiguous()
    else:
        ref_f, ref_shape = ref
    match, success = api.track(ref_f, ref_shape, f, sh, cnt, df_max, macd_max)
    return match, success, ref_f, ref_shape


def identify_raw(raw: torch.Tensor, fs_in: float, fs_out: float, P: SweepParams, stream_id: int = 0,
                 order: int = 8, rp_db: float = 0.05, engine: Engine | None = None):
    """A raw acquisition file to its pole table (PAPER.md:482 then §2.1): ssi_preprocess (detrend,
    zero-phase Chebyshev-I low-pass, rate change fs_in -> fs_out) into an FP32 record, then A1-A11.
    P.fs must equal fs_out. Returns (table, preprocessed record)."""
    if abs(P.fs - fs_out) > 1e-9 * fs_out:
        raise ValueError("P.fs must be the output rate")
    Y = api.preprocess(raw, fs_in, fs_out, order=order, rp_db=rp_db, out_dtype=torch.float32)
    eng = engine or Engine(P, Y.shape[0], Y.device)
    return eng.identify(Y, stream_id), Y


# ------------------------------------------------------------------ the paper's bridge workload
def bridge_params(i: int = 76) -> SweepParams:
    """The San Faustino settings: 114 channels at 40 Hz, j_b = 76 (T = 8664), orders
    250..400 step 2, Algorithm 1 verbatim (q = 0) with the rank rule (25 % of T, k = 2166)."""
    return SweepParams(l=114, i=i, n_max=400, p=0, q=0, fs=40.0, n_min=250, n_step=2, rank_rule=True)


def bridge_identify_2d(raw: torch.Tensor, P: SweepParams | None = None, min_size: int | None = None):
    """One record, 2D diagram: preprocessing 125 -> 40 Hz, covariances, RSVD,
    modal sweep over orders 250..400, hard + soft criteria along the order axis (2 %, 3 %, 2 %)
    and the two-stage clustering. Returns (table, flags, Clustering)."""
    P = P or bridge_params()
    tab, Y = identify_raw(raw, 125.0, P.fs, P)
    crit = api.CRITERIA_BRIDGE_2D
    flags, _ = api.stab3d([tab], crit)
    ms = min_size if min_size is not None else max(1, int(0.2 * tab.n_orders))
    return tab, flags, api.cluster3d([tab], flags, crit, min_size=ms)


def bridge_identify_3d(raw: torch.Tensor, lags=tuple(range(69, 105, 5)), min_size: int | None = None,
                       timing: dict | None = None):
    """One record, 3D diagram: preprocessing, then 8 time lags j_b = 69..104 (rank
    rule per lag), the 3D soft criteria (2.5 %, 5 %, 3 %) and the two-stage clustering."""
    P = bridge_params(max(lags))
    Y = api.preprocess(raw, 125.0, P.fs, out_dtype=torch.float32)
    return identify_3d(Y, P, lags, api.CRITERIA_BRIDGE_3D, min_size=min_size, timing=timing)
