#!/usr/bin/env python
"""Benchmark of the CoV-SSI + RSVD hot path on B200 (BASELINE.json metric):

  CoV-SSI records/s (cov + Toeplitz + RSVD + modal sweep) at l=192, i=60 (config c3:
  N=360000 FP32 samples, k = n_max + p = 220, q = 2, orders 2..200 step 2), plus the
  roofline fractions of its kernels.

A "step" is one record through A1 (covariances) -> A2 (Toeplitz, applied through its block
structure) -> A3-A8 (RSVD) -> A9-A11 (modal sweep). Records are device-resident (2 distinct
276 MB records rotated per rank, each > the 126 MB L2), 8 in flight. Multi-GPU (torchrun): each
rank processes its own records (weak scaling, no data-path collective); time = max over ranks.

Two more workloads are timed in every run (keys "lag_sweep_c4" and "record_batch_c5"; the
north star's scaling targets), at the launch's N GPUs:
  * c4 — the 3D stabilization sweep on the c3 record, i = 20..80 step 4: time-sharded spectral
    covariances to lag 159 (ssi_covariances, normalize=0) -> one NCCL all_reduce ->
    ssi_cov_normalize -> lags by LPT on 8 high-priority streams per rank -> one packed all_gather
    of the pole tables -> ssi_stab3d (strong scaling: one sweep, fixed work);
  * c5 — the continuous-monitoring batch: 64 records of 180000 samples (i = 50) round-robin over
    the ranks, 8 in flight per rank, then one packed all_gather of the 64 tables (strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c4|c5] [--impl reference]
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CoV-SSI records/sec (cov+RSVD+modal sweep), l=192,i=60; % of B200 roofline"
UNIT = "records/s"
C4_LAGS = tuple(range(20, 81, 4))          # BASELINE.json configs[3]
C5_RECORDS = 64                            # BASELINE.json configs[4]
FP64_ALU_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 148 SMs x 64 FP64 FMA lanes x 2 x 1965 MHz


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=80)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c3", "c4", "c5"],
                    help="headline workload: c3 records (the metric), c4 lag sweeps or c5 record batches")
    ap.add_argument("--cov", default=os.environ.get("SSI_COV_MODE", "spectral"), choices=["fp64", "int8x3", "spectral"])
    ap.add_argument("--explicit-t", action="store_true",
                    help="materialize T (A2) and stream it through the RSVD GEMMs instead of "
                         "applying it through its block structure")
    ap.add_argument("--records", type=int, default=2)
    ap.add_argument("--streams", type=int, default=8, help="records in flight (one engine per stream)")
    ap.add_argument("--tail", type=int, default=0,
                    help="the last TAIL records of the timed batch are submitted with the pipeline's tail hint "
                         "(covariances at high priority: nothing follows them)")
    ap.add_argument("--no-priority", action="store_true",
                    help="one stream per record (no low-priority covariance streams)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-legs", action="store_true", help="skip the c4 / c5 legs")
    return ap.parse_args()


def workload_desc(cfg):
    return (f"{cfg.name}: l={cfg.l}, N={cfg.N} {cfg.dtype.upper()}, fs={cfg.fs:g} Hz, i={cfg.i} "
            f"(T {cfg.m}x{cfg.m}), k={cfg.k} (n_max {cfg.n_max} + p {cfg.p}), q={cfg.q}, "
            f"orders {cfg.n_min}..{cfg.n_max} step {cfg.n_step}")


def cov_flops(cfg):
    L = 2 * cfg.i - 1
    return 2.0 * cfg.l * cfg.l * sum(cfg.N - k for k in range(1, L + 1))


def record_flops(cfg, api):
    """Algorithmic flops of one record through the path as built, by stage:
    A1 spectral: cross-spectral product 6 lp^2 S (F/2+1) + inverse DFT 2 lp^2 L (F+2);
    A4/A6/A7 (2q+2 passes through the block DFT): per pass 2 i (2l)^2 k (block products) +
    2 x 2 l (2i) i k (forward and inverse DFT);  A5/A8: 2q + 4 CholeskyQR passes (one between the power-iteration products,
    two for the last Q and for B^T), each m k^2 (symmetric Gram) + m k^2 (triangular Y L^-T) + k^3/3, U = Q U~
    (2 m k n_max), Jacobi (~9 sweeps x k^2/2 pairs x 6k); A9-A11: CholeskyQR2 of U^up + Q^T U^down
    (~6 m n_max^2) and per order n: Hessenberg (10/3 n^3) with C_n = U[0:l,:n] Q_H (2 l n^2), and
    the Francis QR (~10 n^3) with its l-row Schur vectors (~15 l n^2; LAPACK's 25 n^3 for an
    n-row Z scaled to l rows)."""
    l, i, k, n_max, m, q = cfg.l, cfg.i, cfg.k, cfg.n_max, cfg.m, cfg.q
    f_prod, f_inv = api.cov_spectral_flops(cfg.N, l, 2 * i - 1)
    passes = 2 * q + 2                       # Y = T Omega, 2q power-iteration passes, B^T = T^T Q
    rsvd_passes = passes * (2 * i * (2 * l) ** 2 * k + 2 * 2 * l * (2 * i) * i * k)
    # CholeskyQR passes (Gram m k^2 + triangular Y L^-T m k^2 + Cholesky/inverse k^3/3 each):
    # one per re-orthonormalisation between the power iterations' products (2q when q > 0),
    # two for the Q entering B = Q^T T and two for qr(B^T) (reading A-12)
    npass = 2 * q + 4
    qr = npass * (2.0 * m * k * k + k ** 3 / 3)
    small = 2.0 * m * k * n_max + 9 * (k * k / 2) * 6 * k
    modal = 6.0 * m * n_max ** 2 + sum(10.0 / 3 * n ** 3 + 2.0 * l * n * n + 10.0 * n ** 3 + 15.0 * l * n * n
                                       for n in cfg.orders)
    return {"A1": f_prod + f_inv, "A4_A6_A7": rsvd_passes, "A5_A8": qr + small, "A9_A11": modal}


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4) if r[3 + j].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU oracle (reported baseline)
def cores_used():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class OracleRecord:
    """One record through the UNMODIFIED oracle (oracle/, FP64 numpy/LAPACK), cut into `n`
    pieces that run in order and together are exactly one record: the covariances as time shards
    of the direct sum (oracle.covariance_partial_sums; the last shard divides by N - k), then the
    Toeplitz + RSVD (same Philox sketch), then the literal pinv + eig modal sweep over every
    order, in chunks of orders. Nothing is fitted or extrapolated: timing all n pieces times one
    whole record. The FP32 record is converted to FP64 once, outside the timing."""

    def __init__(self, cfg, Y, n: int):
        import oracle
        self.oracle = oracle
        self.cfg = cfg
        self.Y = np.asarray(Y, dtype=np.float64)
        self.L = 2 * cfg.i - 1
        n = max(3, n)
        n_mod = max(1, n // 5)
        n_cov = n - 1 - n_mod
        N = self.Y.shape[0]
        bounds = np.linspace(0, N, n_cov + 1).round().astype(int)
        self.pieces = [("cov", int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:])]
        self.pieces.append(("rsvd",))
        w = np.cumsum([o ** 3 for o in cfg.orders]).astype(float)    # equal-cost chunks of orders
        cut = np.searchsorted(w, w[-1] * np.arange(1, n_mod) / n_mod)
        chunks = np.split(np.array(cfg.orders), cut)
        self.pieces += [("modal", [int(o) for o in c]) for c in chunks if len(c)]
        self.stage_s = {"cov": 0.0, "toeplitz": 0.0, "rsvd": 0.0, "modal": 0.0}
        self.S = None
        self.cells = []

    def __len__(self):
        return len(self.pieces)

    def run(self, j):
        o, cfg = self.oracle, self.cfg
        pc = self.pieces[j]
        t0 = time.perf_counter()
        if pc[0] == "cov":
            part = o.covariance_partial_sums(self.Y, 1, self.L, pc[1], pc[2])
            self.S = part if self.S is None else self.S + part
            if pc[2] == self.Y.shape[0]:
                N = self.Y.shape[0]
                for k in range(1, self.L + 1):
                    self.S[k - 1] /= (N - k)
            self.stage_s["cov"] += time.perf_counter() - t0
        elif pc[0] == "rsvd":
            T = o.toeplitz(self.S, cfg.i)
            t1 = time.perf_counter()
            self.stage_s["toeplitz"] += t1 - t0
            self.U, self.Sv, _ = o.rsvd(T, cfg.k, cfg.q, cfg.philox_key, cfg.i, cfg.n_max)
            self.stage_s["rsvd"] += time.perf_counter() - t1
        else:
            self.cells += o.modal_sweep(self.U, self.Sv, cfg.l, cfg.i, pc[1], cfg.dt)
            self.stage_s["modal"] += time.perf_counter() - t0
        return time.perf_counter() - t0

    def describe(self):
        n_cov = sum(1 for p in self.pieces if p[0] == "cov")
        n_mod = sum(1 for p in self.pieces if p[0] == "modal")
        return (f"one whole {self.cfg.name} record through the unmodified FP64 oracle, cut into {len(self)} "
                f"pieces run in order: covariances by direct summation over all {self.L} lags in {n_cov} "
                f"time shards, full Toeplitz + RSVD (k={self.cfg.k}, q={self.cfg.q}, same Philox sketch), "
                f"literal pinv+eig modal sweep over all {len(self.cfg.orders)} orders in {n_mod} chunks; "
                f"nothing fitted or extrapolated")


def cpu_extras(cfg, cells):
    """Beside the record: O-5 (one full dgesdd of the Toeplitz, timed at c2 size, 2880^2; the c3
    11520^2 one takes minutes — profiles/), O-8 (oracle stab3d over the record's table), and a
    single-thread direct-sum covariance rate (GFLOP/s)."""
    import oracle
    import synth
    out = {}
    c2 = synth.config("c2")
    Y2, _ = synth.make_record(c2)
    T2 = oracle.toeplitz(oracle.covariances(Y2, 2 * c2.i - 1), c2.i)
    t0 = time.perf_counter()
    oracle.full_svd(T2)
    out["o5_full_svd_c2_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.stab3d([cells], oracle.SC_BRIDGE_3D, cfg.n_max // 2)
    out["o8_stab3d_s"] = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_limits
        Y, _ = synth.make_record(cfg, N=3000)
        Y = np.asarray(Y, dtype=np.float64)
        L = 2 * cfg.i - 1
        with threadpool_limits(limits=1):
            t0 = time.perf_counter()
            oracle.covariance_partial_sums(Y, 1, L)
            dt = time.perf_counter() - t0
        out["cov_gflops_1thread"] = 2.0 * cfg.l ** 2 * sum(Y.shape[0] - k for k in range(1, L + 1)) / dt / 1e9
    except Exception as e:            # threadpoolctl missing: report why
        out["cov_gflops_1thread"] = None
        out["cov_1thread_error"] = str(e)[:100]
    return out


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The oracle as the reference arm (this tier has no reference code; /root/reference is a
    paper): rank 0 only; each of the K timed steps is one piece of ONE whole c3 record (so the K
    steps together are exactly one record, timed piece by piece, nothing extrapolated); the W
    warm-up steps run pieces of a tiny c1 record."""
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = synth.config("c3")
    Y, _ = synth.make_record(cfg)
    c1 = synth.config("c1")
    warm = OracleRecord(c1, synth.make_record(c1)[0], max(args.warmup, 3))
    for j in range(args.warmup):
        warm.run(j % len(warm))
    rec = OracleRecord(cfg, Y, args.steps)
    secs = [rec.run(j) for j in range(len(rec))]
    total = float(np.sum(secs))
    v = 1.0 / total
    steps = len(rec)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_desc(cfg)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores_used(), "cpu_model": cpu_model(),
                             "kind": "oracle", "sample": rec.describe(),
                             "stage_s": {k: round(t, 3) for k, t in rec.stage_s.items()}},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def count_launches(fn):
    """Kernels of libssi launched by fn() (CUPTI through torch.profiler); torch's own kernels
    (the status-word bookkeeping, copies) are excluded."""
    import torch
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ours = [n for n in names if "ssi::" in n and "at::" not in n]
    return len(ours), names


def _max_over_ranks(x, world, dev):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor(x, dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sweep_leg(api, drivers, synth, torch, dist, Y, world, rank, dev, reps=3, warm=2):
    """c4: the whole 3D stabilization sweep (strong scaling over ranks), device time (events on
    the current stream, which every phase joins), max over ranks."""
    cfg = synth.config("c4")
    P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs,
                            n_min=cfg.n_min, n_step=cfg.n_step, seed=cfg.philox_key)
    crit = api.CRITERIA_BRIDGE_3D
    for _ in range(warm):
        drivers.identify_3d(Y, P, C4_LAGS, crit, rank=rank, world=world)
    torch.cuda.synchronize()
    rows = []
    for _ in range(reps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        tm = {}
        tabs, flags, counts, cl = drivers.identify_3d(Y, P, C4_LAGS, crit, rank=rank, world=world, timing=tm)
        torch.cuda.synchronize()
        ph = [tm["start"].elapsed_time(tm["cov"]), tm["cov"].elapsed_time(tm["lags"]),
              tm["lags"].elapsed_time(tm["gather"]), tm["gather"].elapsed_time(tm["stab"]),
              tm["stab"].elapsed_time(tm["cluster"]), tm["start"].elapsed_time(tm["stab"]),
              tm["start"].elapsed_time(tm["cluster"])]
        rows.append(_max_over_ranks(ph, world, dev))
    best = min(rows, key=lambda r: r[-1])
    med = sorted(r[-2] for r in rows)[len(rows) // 2]
    med_all = sorted(r[-1] for r in rows)[len(rows) // 2]
    return {"workload": "c4: c3 record, i = 20..80 step 4 (16 lags, T up to 15360^2), k=220, q=2, orders 2..200",
            "ms_per_sweep": med, "ms_best": best[-2],
            "ms_with_clustering": med_all,
            "phase_ms_best": {"cov_allreduce_normalize": best[0], "lags": best[1], "gather": best[2],
                              "stab3d": best[3], "cluster_stage_I_II": best[4]},
            "sweeps_per_s": 1e3 / med, "n_gpus": world, "reps": reps, "scaling": "strong",
            "stable_poles": int(counts.sum().item()), "retained_poles": cl.n_retained,
            "clusters": cl.n_clusters,
            "lag_assignment": drivers.lpt_assign(list(C4_LAGS), world)}


def _event_ms(torch, fn, reps=3):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def next_legs(api, synth, torch, R_c3, dev):
    """Per-GPU legs of the paper's own settings (one GPU, device time, median of 3):
    * NEXT-1: Algorithm 1 verbatim (q = p = 0) at the paper's rank rule k = ceil(kbar(T) % T)
       on the c3 record: T = 11520, kbar = 25 %, k = 2880 (structured RSVD);
    * NEXT-4: preprocessing of a 2-hour 114-channel 125 Hz acquisition to 40 Hz."""
    from synth.raw import make_raw_record
    cfg = synth.config("c3")
    m = cfg.m
    k = int(-(-max(30.0 - 0.00156 * m, 25.0) * m // 100))
    ws = api._workspace(api.rsvd_toeplitz_ws_bytes(cfg.l, cfg.i, k, cfg.n_max), dev)
    ms_rr = _event_ms(torch, lambda: api.rsvd_toeplitz(R_c3, cfg.i, k, 0, cfg.philox_key, cfg.i, cfg.n_max, ws=ws))
    del ws
    raw, _ = make_raw_record(l=114, fs=125.0, N=900000, seed=482)
    rawd = torch.from_numpy(raw).to(dev)
    wsp = api._workspace(api.preprocess_ws_bytes(900000, 114, 8), dev)
    Z = torch.empty((288000, 114), dtype=torch.float32, device=dev)
    ms_pp = _event_ms(torch, lambda: api.preprocess(rawd, 125.0, 40.0, out=Z, ws=wsp))
    # the paper's own end-to-end bridge workload: one synthetic 2-hour
    # 114-channel 125 Hz acquisition, preprocessing to 40 Hz, 2D (j_b = 76) and 3D (j_b = 69..104)
    from paper_2411_05510_b200 import drivers
    from synth.raw import make_bridge_raw
    braw = torch.from_numpy(make_bridge_raw()[0]).to(dev)
    ms_b2 = _event_ms(torch, lambda: drivers.bridge_identify_2d(braw), reps=1)
    ms_b3 = _event_ms(torch, lambda: drivers.bridge_identify_3d(braw), reps=1)
    bridge = {"workload": "synthetic San-Faustino-shaped acquisition: 114 ch x 900000 FP32 at 125 Hz (2 h) -> 40 Hz; "
                          "Algorithm 1 verbatim at the rank rule (j_b = 76: T = 8664, k = 2166), orders 250..400, "
                          "HC + SC + two-stage clustering",
              "identify_2d_ms": ms_b2, "identify_3d_8_lags_ms": ms_b3,
              "paper_cpu_s": {"rsvd_2d": 204, "rsvd_3d": 512, "svd_2d": 449,
                              "hardware": "i7-8750H (PAPER.md:544), other hardware: context only"}}
    return {"bridge_record": bridge,
            "rank_rule_rsvd_c3": {"workload": f"c3 record, T = {m}, Algorithm 1 verbatim (q = p = 0), k = {k} "
                                              "(kbar(T) = 25 %), T through its block structure",
                                  "ms_per_rsvd": ms_rr},
            "preprocess_bridge_2h": {"workload": "114 ch x 900000 FP32 at 125 Hz -> 288000 at 40 Hz (L/M = 8/25), "
                                                 "detrend + zero-phase 8th-order Chebyshev-I",
                                     "ms": ms_pp, "hours_of_data_per_s": 2.0 / (ms_pp / 1e3)}}


def batch_leg(api, drivers, synth, torch, dist, world, rank, dev, streams):
    """c5: 64 records of 180000 samples over all ranks (strong scaling), 8 in flight per rank,
    one packed all_gather of the 64 tables; device time, max over ranks."""
    cfg = synth.config("c5")
    P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs,
                            n_min=cfg.n_min, n_step=cfg.n_step, seed=cfg.philox_key)
    # two distinct drifted records per rank, device-resident, rotated (each 138 MB > L2)
    Ys = [torch.from_numpy(synth.make_record(cfg, record=2 * rank + j)[0]).to(dev) for j in range(2)]
    recs = [Ys[j % 2] for j in range(C5_RECORDS)]
    drivers.record_batch(recs, P, rank, world, n_streams=streams)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    tabs = drivers.record_batch(recs, P, rank, world, n_streams=streams)
    b.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks([a.elapsed_time(b)], world, dev)[0]
    # monitoring step iii on the gathered tables: per-session two-stage clustering
    # of the 2D diagram and tracking against the first session (every rank holds every table)
    crit = api.CRITERIA_BRIDGE_2D
    c = torch.cuda.Event(enable_timing=True); d = torch.cuda.Event(enable_timing=True)
    c.record()
    match, succ, ref_f, _ = drivers.track_campaign([tabs[j] for j in range(C5_RECORDS)], crit)
    d.record()
    torch.cuda.synchronize()
    track = {"ms": c.elapsed_time(d), "sessions": C5_RECORDS, "reference_modes": int(ref_f.numel()),
             "mean_success_pct": float(succ.mean().item()) if succ.numel() else None,
             "note": "per-session ssi_stab3d + ssi_cluster_stage1/2 (one host read of the retained count "
                     "each) + one ssi_track; 2 distinct records rotated, so success is ~100 % by construction"}
    return {"workload": f"c5: {C5_RECORDS} records x 180000 F32 samples, l=192, i=50, k=220, q=2, orders 2..200 "
                        "(2 distinct drifted records per rank rotated)",
            "ms_per_batch": ms, "records_per_s": C5_RECORDS / (ms / 1e3), "n_gpus": world, "scaling": "strong",
            "records_per_rank": len(drivers.record_assignment(C5_RECORDS, world)[0]),
            "campaign_clustering_tracking": track}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import synth
    from paper_2411_05510_b200 import api, drivers, build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SSI_DIST_BACKEND=gloo: a functional run of the N-rank path with several ranks sharing the
    # GPUs there are (no timing claim; e.g. 2 ranks on one B200); the default is NCCL, one GPU per rank
    backend = os.environ.get("SSI_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()

    cfg = synth.config("c3")
    P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs,
                            n_min=cfg.n_min, n_step=cfg.n_step, seed=cfg.philox_key, cov_mode=args.cov,
                            structured=not args.explicit_t)
    # distinct records per rank (weak scaling): record index = rank * R + j; the c3 record itself
    # (seed cfg.seed) is also the c4 sweep's input on every rank
    host = []
    for j in range(args.records):
        Yh, _ = synth.make_record(synth.config("c3", seed=cfg.seed + 100 * (rank * args.records + j) if j or rank else cfg.seed))
        host.append(Yh)
    Ys = [torch.from_numpy(h).to(dev) for h in host]
    Y_c3 = Ys[0] if rank == 0 else torch.from_numpy(synth.make_record(cfg)[0]).to(dev)
    pipe = drivers.RecordPipeline(P, cfg.N, dev, n_streams=args.streams, split_priority=not args.no_priority)
    eng = pipe.engines[0]
    stream = torch.cuda.current_stream()

    def step(j, ev=None, tail=False):
        tab, _ = pipe.submit(Ys[j % len(Ys)], (j << 32) | cfg.i, ev, tail=tail)
        return tab

    for j in range(args.warmup):
        step(j)
    pipe.join()
    torch.cuda.synchronize()
    pipe.check()
    n_launch, _ = count_launches(lambda: (step(0), pipe.join()))

    # per-stage breakdown (one extra untimed record on one stream, events between stages)
    stage = {}
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    Y = Ys[0]
    evs[0].record(stream); R = eng.covariances(Y); evs[1].record(stream)
    if P.structured:
        evs[2].record(stream)
        U, S = api.rsvd_toeplitz(R, cfg.i, P.k, P.q, P.seed, cfg.i, P.n_max, U=eng.U, S=eng.S, ws=eng.ws_rsvd)
    else:
        T = api.toeplitz(R, cfg.i, out=eng.T); evs[2].record(stream)
        U, S = api.rsvd_into(T, P.k, P.q, P.seed, cfg.i, P.n_max, eng.U, eng.S, ws=eng.ws_rsvd)
    evs[3].record(stream)
    api.modal_sweep(U, S, P.l, cfg.i, P.n_min, P.n_max, P.n_step, P.dt, out=eng.table, ws=eng.ws_modal)
    evs[4].record(stream)
    torch.cuda.synchronize()
    for nm, a, b in (("cov", 0, 1), ("toeplitz", 1, 2), ("rsvd", 2, 3), ("modal", 3, 4)):
        stage[nm] = evs[a].elapsed_time(evs[b])

    # ---------------- timed region (device-resident records)
    cov_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
    clk = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    time.sleep(0.3)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for st in pipe.streams:
        st.wait_stream(stream)
    for j in range(args.steps):
        step(j, cov_ev[j], tail=j >= args.steps - args.tail)
    pipe.join(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    pipe.check()
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end)
    cov_ms = float(np.mean([a.elapsed_time(b) for a, b in cov_ev]))
    ms = _max_over_ranks([ms], world, dev)[0]
    value = world * args.steps / (ms / 1e3)

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        ns = len(pipe.streams)
        pinned = [torch.from_numpy(h).pin_memory() for h in host[:2]]
        pipe.reserve_host_inputs(pinned[0].shape, pinned[0].dtype)
        tab_host = [[torch.empty_like(t, device="cpu").pin_memory() for t in e.table.tensors()]
                    for e in pipe.engines]
        d2h = sum(t.numel() * t.element_size() for t in tab_host[0])
        h2d = pinned[0].numel() * pinned[0].element_size()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        a.record(stream)
        for st in pipe.streams:
            st.wait_stream(stream)
        for j in range(args.steps):
            slot = pipe.j % ns
            # H2D of this step's record inside the timed region, on the pipeline's copy stream
            # (submit_host: a ring of device input buffers, copies overlap the records in flight)
            tab, st = pipe.submit_host(pinned[j % 2], (j << 32) | cfg.i, tail=j >= args.steps - args.tail)
            with torch.cuda.stream(st):
                for hst, d in zip(tab_host[slot], tab.tensors()):      # D2H of the result
                    hst.copy_(d, non_blocking=True)
        pipe.join(stream)
        b.record(stream)
        torch.cuda.synchronize()
        pipe.check()
        ems = _max_over_ranks([a.elapsed_time(b)], world, dev)[0]
        e2e = {"value": world * args.steps / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}

    # ---------------- the c4 sweep and the c5 batch at this N
    legs = {}
    if not args.no_legs or args.workload == "c4":     # --workload c4 / c5 needs its leg
        legs["lag_sweep_c4"] = sweep_leg(api, drivers, synth, torch, dist, Y_c3, world, rank, dev)
    if not args.no_legs or args.workload == "c5":
        legs["record_batch_c5"] = batch_leg(api, drivers, synth, torch, dist, world, rank, dev, args.streams)
    if not args.no_legs and rank == 0:
        legs["paper_settings"] = next_legs(api, synth, torch, eng.R, dev)

    # ---------------- roofline
    # The covariance stage alone (CUDA events around one record's A1 on the current stream) and
    # its dominant kernel, the cross-spectral product, re-run alone on the spectra the call left
    # in the engine's workspace (measurement entry point ssi_cov_spectral_phases).
    iso = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream); eng.covariances(Ys[0]); b.record(stream)
        torch.cuda.synchronize()
        iso.append(a.elapsed_time(b))
    iso_ms = float(np.median(iso))
    extra = json.load(open(os.path.join(ROOT, "profiles", "peaks_extra_r01.json")))
    dgemm = extra["fp64_dgemm_tflops_burst"]
    dgemm_sus = extra["fp64_dgemm_tflops_sustained"]
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    roof = None
    stage_cov = None
    if args.cov == "spectral":
        pt = []
        for _ in range(3):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream); api.cov_spectral_phases(Ys[0], eng.lag_hi, 2, eng.R, eng.ws_cov); b.record(stream)
            torch.cuda.synchronize()
            pt.append(a.elapsed_time(b))
        prod_ms = float(np.median(pt))
        f_main, f_inv = api.cov_spectral_flops(cfg.N, cfg.l, 2 * cfg.i - 1)
        F, S_ = api.cov_spectral_plan(cfg.N, cfg.l, 2 * cfg.i - 1)
        stage_cov = {"stage_ms": iso_ms, "plan": {"F": F, "S": S_}, "stage_flop": f_main + f_inv,
                     "stage_tflops": (f_main + f_inv) / (iso_ms / 1e3) / 1e12,
                     "stage_frac": (f_main + f_inv) / (iso_ms / 1e3) / 1e12 / dgemm,
                     "direct_sum_flop_equiv": cov_flops(cfg)}
        traffic = None
        try:
            sp = os.path.join(ROOT, "profiles", "ncu_summary_r02.json")    # round-2 capture of the current kernel
            nsum = json.load(open(sp if os.path.exists(sp) else os.path.join(ROOT, "profiles", "ncu_summary_r01.json")))
            mb = lambda d: d["value"] * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[d["unit"]]
            traffic = mb(nsum["cross3m_kernel"]["dram__bytes_read.sum"]) + mb(nsum["cross3m_kernel"]["dram__bytes_write.sum"])
        except Exception:
            traffic = None
        achieved = f_main / (prod_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": "cross3m_kernel (A1 cross-spectral product, FP64 DMMA, three real "
                                              "products per complex one)",
                "achieved": achieved, "peak": dgemm, "unit": "TFLOP/s", "frac": achieved / dgemm,
                "traffic": traffic, "peak_source": "measured cuBLAS DGEMM 8192^3 burst on this pool's B200 "
                                                   "(profiles/peaks_extra_r01.json); MEASURED_PEAKS.json has no FP64 entry",
                "kernel_ms": prod_ms, "algorithmic_flop_per_launch": f_main,
                "stage_ms_in_pipeline": cov_ms, "covariance_stage": stage_cov}
    else:
        flops = cov_flops(cfg)
        if args.cov == "fp64":
            peak, work, unit = dgemm, flops, "TFLOP/s"
        else:
            peak, work, unit = 2.0 * peaks.get("bf16_tflops", 1644.3), 8.0 * flops, "TOP/s"
        achieved = work / (iso_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": f"covariance A1 ({args.cov})", "achieved": achieved, "peak": peak,
                "unit": unit, "frac": achieved / peak, "traffic": None, "kernel_ms": iso_ms,
                "algorithmic_flop_per_launch": work}
    # whole record: the path's own algorithmic flops (record_flops) per ms_per_step against the
    # sustained DGEMM peak (every stage is FP64 DMMA or FP64 ALU), and per stage (one record alone)
    rf = record_flops(cfg, api) if args.cov == "spectral" and P.structured else None
    if rf is not None:
        tot = sum(rf.values())
        roof["record"] = {"algorithmic_flop": tot, "flop_by_stage": rf,
                          "achieved_tflops": tot / (ms / args.steps / 1e3) / 1e12 / world,
                          "peak": dgemm_sus, "frac": tot / (ms / args.steps / 1e3) / 1e12 / world / dgemm_sus,
                          "peak_source": "measured cuBLAS DGEMM sustained (profiles/peaks_extra_r01.json)"}
        roof["stage_frac_alone"] = {
            "A1": rf["A1"] / (stage["cov"] / 1e3) / 1e12 / dgemm,
            "A2_A8": (rf["A4_A6_A7"] + rf["A5_A8"]) / (stage["rsvd"] / 1e3) / 1e12 / dgemm,
            "A9_A11": rf["A9_A11"] / (stage["modal"] / 1e3) / 1e12 / FP64_ALU_TFLOPS,
            "note": "one record alone on one stream (no overlap): latency-bound stages read low here; "
                    "the 8-in-flight pipeline overlaps them (the record fraction above)"}
    try:   # SM-time shares of one record's kernels, from the committed ncu pass
        sm = json.load(open(os.path.join(ROOT, "profiles", "smtime_spectral_latest.json")))
        top = sorted(sm["kernels"].items(), key=lambda kv: -kv[1]["share_sm_time"])[:6]
        roof["sm_time_share"] = {"source": sm.get("source", "profiles/smtime_spectral_latest.json"),
                                 "top_kernels": {k.split("(")[0].replace("ssi::<unnamed>::", ""):
                                                 round(v["share_sm_time"], 4) for k, v in top}}
        # the RSVD's tensor-core kernels (every gemm_tall launch of a record: the block-DFT passes
        # of A4/A6/A7, the CholeskyQR Gram and Y L^-T products, the modal sweep's CholeskyQR2 of
        # U^up) by their SM-time: algorithmic flops / GPU-ms equivalent against the DGEMM peak
        if rf is not None:
            l_, i_, k_, nm_, m_, q_ = cfg.l, cfg.i, cfg.k, cfg.n_max, cfg.m, cfg.q
            g_flop = (rf["A4_A6_A7"] + (2 * q_ + 4) * 2.0 * m_ * k_ * k_ + 2 * 2.0 * (m_ - l_) * nm_ * nm_
                      + 2.0 * l_ * l_ * (2 * i_ - 1) * 2 * i_          # block spectrum Z = R W
                      + 2.0 * (m_ - l_) * nm_ * nm_ + 2.0 * m_ * k_ * nm_)   # W = Q^T U_down, U = Q U~
            g_ms = sum(v["gpu_ms_equiv"] for kname, v in sm["kernels"].items() if "gemm_tall_kernel" in kname)
            if g_ms > 0:
                ach = g_flop / (g_ms / 1e3) / 1e12
                roof["rsvd_tensor_kernels"] = {
                    "kernels": "gemm_tall_kernel (all launches of one record)", "algorithmic_flop": g_flop,
                    "gpu_ms_equiv": g_ms, "achieved": ach, "peak": dgemm, "unit": "TFLOP/s",
                    "frac": ach / dgemm, "note": "rate while resident (SM-time from the committed ncu pass)"}
        # the kernel with the largest SM-time share: the per-order Francis QR (A10), one CTA per
        # order, a latency-bound bulge chase; its algorithmic flops (~10 n^3 per order, LAPACK's
        # count for the eigenvalues) over its SM-time, against the FP64 ALU peak
        name, v = top[0]
        if "eig_order_kernel" in name:
            eig_flop = sum(10.0 * n ** 3 for n in cfg.orders)
            ach = eig_flop / (v["gpu_ms_equiv"] / 1e3) / 1e12
            roof["sm_time_dominant"] = {
                "kernel": "eig_order_kernel (A10 per-order Francis QR + Schur vectors + poles)",
                "bound": "latency (one warp's dependent FP64 chain per order)", "share_sm_time": v["share_sm_time"],
                "gpu_ms_equiv": v["gpu_ms_equiv"], "algorithmic_flop": eig_flop, "achieved": ach,
                "peak": FP64_ALU_TFLOPS, "unit": "TFLOP/s", "frac": ach / FP64_ALU_TFLOPS,
                "peak_source": "148 SMs x 64 FP64 FMA lanes x 2 x 1965 MHz (B200_PROFILING.md unit counts)"}
    except Exception:
        pass

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        rec = OracleRecord(cfg, host[0], 1)
        tot = sum(rec.run(j) for j in range(len(rec)))
        cpu = {"value": 1.0 / tot, "unit": UNIT, "cores": cores_used(), "cpu_model": cpu_model(), "kind": "oracle",
               "sample": rec.describe(), "stage_s": {k: round(t, 3) for k, t in rec.stage_s.items()}}
        cpu.update(cpu_extras(cfg, rec.cells))

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_desc(cfg), "cov_mode": args.cov,
                           "records_rotated": len(Ys), "streams": args.streams,
                           "toeplitz": ("explicit T (1.06 GB) streamed by the RSVD GEMMs" if args.explicit_t else
                                        "T applied through its block structure (block DFT, T never formed)"),
                           "l2": "inputs larger than L2 (276 MB FP32 record per step, 2 records rotated)",
                           "parallelism": f"records sharded over {world} GPU(s)"},
                "stage_ms": stage, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": n_launch * args.steps, "clocks": clocks}
        line.update(legs)
        if args.workload != "c3" and legs:
            # headline on another workload (manual runs): its unit of work per second
            if args.workload == "c4":
                lg = legs["lag_sweep_c4"]
                line.update(metric="CoV-SSI 3D lag sweeps/sec (c4)", value=lg["sweeps_per_s"], unit="sweeps/s",
                            ms_per_step=lg["ms_per_sweep"], scaling="strong",
                            config={**line["config"], "workload": lg["workload"]})
            else:
                lg = legs["record_batch_c5"]
                line.update(metric="CoV-SSI records/sec (c5 batch)", value=lg["records_per_s"], unit=UNIT,
                            ms_per_step=lg["ms_per_batch"] / C5_RECORDS, scaling="strong",
                            config={**line["config"], "workload": lg["workload"]})
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
