#!/usr/bin/env python
"""Benchmark of the CoV-SSI + RSVD hot path on B200 (BASELINE.json metric):

  CoV-SSI records/s (cov + Toeplitz + RSVD + modal sweep) at l=192, i=60 (config c3:
  N=360000 FP32 samples, k = n_max + p = 220, q = 2, orders 2..200 step 2), plus the
  dominant kernel's fraction of the B200 roofline.

A "step" is one record through A1 (covariances) -> A2 (Toeplitz) -> A3-A8 (RSVD) ->
A9-A11 (modal sweep). Records are device-resident (4 distinct records rotated, each
276 MB > the 126 MB L2). Multi-GPU (torchrun): each rank processes its own records
(weak scaling, no data-path collective); time = max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--cov fp64|int8x3|spectral] [--impl reference]
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=80)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cov", default=os.environ.get("SSI_COV_MODE", "spectral"), choices=["fp64", "int8x3", "spectral"])
    ap.add_argument("--explicit-t", action="store_true",
                    help="materialize T (A2) and stream it through the RSVD GEMMs instead of "
                         "applying it through its block structure")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--records", type=int, default=2)
    ap.add_argument("--streams", type=int, default=8, help="records in flight (one engine per stream)")
    ap.add_argument("--no-priority", action="store_true",
                    help="one stream per record (no low-priority covariance streams)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def workload_desc(cfg):
    return (f"{cfg.name}: l={cfg.l}, N={cfg.N} {cfg.dtype.upper()}, fs={cfg.fs:g} Hz, i={cfg.i} "
            f"(T {cfg.m}x{cfg.m}), k={cfg.k} (n_max {cfg.n_max} + p {cfg.p}), q={cfg.q}, "
            f"orders {cfg.n_min}..{cfg.n_max} step {cfg.n_step}")


def cov_flops(cfg):
    L = 2 * cfg.i - 1
    return 2.0 * cfg.l * cfg.l * sum(cfg.N - k for k in range(1, L + 1))


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
def oracle_sample(cfg, Y, orders=(100, 200), cov_lags=None, R_full=None):
    """Times the unmodified oracle on one c3 record: the covariances (all 2i-1 lags, or
    `cov_lags` evenly spaced lags scaled to all of them: each lag is one independent matmul of
    the same size), the full Toeplitz, the full RSVD (same Philox sketch), and the literal
    pinv+eig modal identification at the given orders only (per-order cost fitted as
    a + b n^2 and summed over all orders). With cov_lags the Toeplitz / RSVD / modal stages run on
    `R_full` (the record's full covariances, computed once outside the timing).
    Returns (seconds per record, stage seconds, description)."""
    import oracle
    t = {}
    L = 2 * cfg.i - 1
    t0 = time.perf_counter()
    if cov_lags is None:
        R = oracle.covariances(Y, L)
        t["cov"] = time.perf_counter() - t0
    else:
        ks = sorted(set(int(round(x)) for x in np.linspace(1, L, cov_lags)))
        for k in ks:
            oracle.covariances(Y, k, k)
        t["cov"] = (time.perf_counter() - t0) * L / len(ks)
        R = R_full
    t0 = time.perf_counter()
    T = oracle.toeplitz(R, cfg.i)
    t["toeplitz"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    U, S, _ = oracle.rsvd(T, cfg.k, cfg.q, cfg.philox_key, cfg.i, cfg.n_max)
    t["rsvd"] = time.perf_counter() - t0
    per = []
    for n in orders:
        t0 = time.perf_counter()
        oracle.modal_sweep(U, S, cfg.l, cfg.i, [n], cfg.dt)
        per.append((n, time.perf_counter() - t0))
    (n1, a1), (n2, a2) = per[0], per[-1]
    b = (a2 - a1) / (n2 ** 2 - n1 ** 2) if n2 != n1 else 0.0
    a = a1 - b * n1 ** 2
    t["modal"] = sum(max(a + b * n * n, 0.0) for n in cfg.orders)
    total = sum(t.values())
    cov_desc = f"full covariances ({L} lags)" if cov_lags is None else \
        f"covariances timed on {cov_lags} of the {L} lags and scaled to all {L}"
    sample = (f"one {cfg.name} record: {cov_desc}, full Toeplitz, full RSVD "
              f"(k={cfg.k}, q={cfg.q}), modal sweep timed at orders {list(orders)} and fitted a+b*n^2 "
              f"over the {len(cfg.orders)} orders")
    return total, t, sample


def cores_used():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    cfg = synth.config(args.config)
    Y, _ = synth.make_record(cfg)
    for _ in range(max(0, min(args.warmup, 1))):
        oracle_sample(synth.config("c1"), synth.make_record(synth.config("c1"))[0], (10, 20))
    # each step is a bounded sample (about 3 s of CPU work) so K steps finish in minutes
    R_full = oracle.covariances(Y, 2 * cfg.i - 1)
    secs = []
    for _ in range(args.steps):
        tot, _, sample = oracle_sample(cfg, Y, cov_lags=8, R_full=R_full)
        secs.append(tot)
    v = 1.0 / float(np.mean(secs))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_desc(cfg)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores_used(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def count_launches(fn):
    """Kernels of libssi launched by fn() (CUPTI through torch.profiler)."""
    import torch
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ours = [n for n in names if any(s in n for s in ("ssi::", "kernel", "cov_", "splitk", "toeplitz",
                                                     "sketch", "jacobi", "chol", "eig_order", "gemm",
                                                     "stab_", "i8"))
            and "Memset" not in n and "Memcpy" not in n]
    return len(ours), names


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
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()

    cfg = synth.config(args.config)
    P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs,
                            n_min=cfg.n_min, n_step=cfg.n_step, seed=cfg.philox_key, cov_mode=args.cov,
                            structured=not args.explicit_t)
    # distinct records per rank (weak scaling): record index = rank * R + j
    host = []
    for j in range(args.records):
        Yh, _ = synth.make_record(synth.config(args.config, seed=cfg.seed + 100 * (rank * args.records + j) if j or rank else cfg.seed))
        host.append(Yh)
    Ys = [torch.from_numpy(h).to(dev) for h in host]
    pipe = drivers.RecordPipeline(P, cfg.N, dev, n_streams=args.streams, split_priority=not args.no_priority)
    eng = pipe.engines[0]
    stream = torch.cuda.current_stream()

    def step(j, ev=None):
        tab, _ = pipe.submit(Ys[j % len(Ys)], (j << 32) | cfg.i, ev)
        return tab

    for j in range(args.warmup):
        step(j)
    pipe.join()
    torch.cuda.synchronize()
    for e in pipe.engines:
        for ws in (e.ws_cov, e.ws_rsvd, e.ws_modal):
            code = api.device_status(ws)
            if code != 0:
                raise RuntimeError(f"device status {code} after warm-up")
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
        step(j, cov_ev[j])
    pipe.join(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end)
    cov_ms = float(np.mean([a.elapsed_time(b) for a, b in cov_ev]))
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = world * args.steps / (ms / 1e3)

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        ns = len(pipe.streams)
        pinned = [torch.from_numpy(h).pin_memory() for h in host[:2]]
        Ydev = [torch.empty_like(Ys[0]) for _ in range(ns)]
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
            st = pipe.streams[slot]
            with torch.cuda.stream(st):
                Ydev[slot].copy_(pinned[j % 2], non_blocking=True)       # H2D inside the step
            tab, _ = pipe.submit(Ydev[slot], (j << 32) | cfg.i)
            with torch.cuda.stream(st):
                for hst, d in zip(tab_host[slot], tab.tensors()):      # D2H of the result
                    hst.copy_(d, non_blocking=True)
        pipe.join(stream)
        b.record(stream)
        torch.cuda.synchronize()
        ems = a.elapsed_time(b)
        if world > 1:
            tt = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": world * args.steps / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}

    # ---------------- roofline of the dominant tensor-core kernel (covariance contraction)
    # Timed in isolation (the pipelined timed region overlaps streams, so a launch's event
    # span there includes other records' kernels; that span is reported for context).
    iso = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream); eng.covariances(Ys[0]); b.record(stream)
        torch.cuda.synchronize()
        iso.append(a.elapsed_time(b))
    iso_ms = float(np.median(iso))
    prod_ms = None
    if args.cov == "spectral":
        # the dominant kernel alone: the cross-spectral product re-run on the spectra the call
        # above left in the engine's workspace (library measurement hook SSI_SPEC_PHASES=2)
        os.environ["SSI_SPEC_PHASES"] = "2"
        try:
            pt = []
            for _ in range(3):
                a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
                a.record(stream); eng.covariances(Ys[0]); b.record(stream)
                torch.cuda.synchronize()
                pt.append(a.elapsed_time(b))
            prod_ms = float(np.median(pt))
        finally:
            del os.environ["SSI_SPEC_PHASES"]
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    extra = json.load(open(os.path.join(ROOT, "profiles", "peaks_extra_r01.json")))
    flops = cov_flops(cfg)                  # 2 l^2 sum_k (N - k) per record
    traffic = None
    try:
        nsum = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary_r01.json")))
        key = {"int8x3": "cov_i8_kernel", "spectral": "cross3m_kernel"}.get(args.cov)
        if key and key in nsum:
            mb = lambda d: d["value"] * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[d["unit"]]
            traffic = mb(nsum[key]["dram__bytes_read.sum"]) + mb(nsum[key]["dram__bytes_write.sum"])
    except Exception:
        traffic = None
    stage = None
    if args.cov == "spectral":
        # dominant kernel: the cross-spectral product (FP64 DMMA), its algorithmic flops
        # 6 lp^2 S (F/2+1) over its own live duration; the whole covariance stage beside it
        f_main, f_inv = api.cov_spectral_flops(cfg.N, cfg.l, 2 * cfg.i - 1)
        F, S = api.cov_spectral_plan(cfg.N, cfg.l, 2 * cfg.i - 1)
        peak = extra["fp64_dgemm_tflops_burst"]
        peak_src = "measured cuBLAS DGEMM 8192^3 on this pool's B200 (profiles/peaks_extra_r01.json)"
        work, unit = f_main, "TFLOP/s"
        stage = {"stage_ms": iso_ms, "plan": {"F": F, "S": S}, "stage_dmma_flop": f_main + f_inv,
                 "stage_tflops": (f_main + f_inv) / (iso_ms / 1e3) / 1e12,
                 "stage_frac": (f_main + f_inv) / (iso_ms / 1e3) / 1e12 / peak,
                 "direct_sum_flop_equiv": flops}
        iso_k = prod_ms
    elif args.cov == "fp64":
        peak = extra["fp64_dgemm_tflops_burst"]
        peak_src = "measured cuBLAS DGEMM 8192^3 on this pool's B200 (profiles/peaks_extra_r01.json)"
        work, unit = flops, "TFLOP/s"
    else:
        peak = 2.0 * peaks.get("bf16_tflops", 1644.3)
        peak_src = "of measured: 2 x bf16 dense burst (MEASURED_PEAKS.json) = nominal int8:bf16 ratio"
        work, unit = 8.0 * flops, "TOP/s"   # each multiply-add runs as eight int8 slice products
    if args.cov != "spectral":
        iso_k = iso_ms
    achieved = work / (iso_k / 1e3) / 1e12
    share = None
    try:   # the covariance stage's share of one record's SM-time, from the committed ncu pass
        src = {"int8x3": "smtime_r01.json", "spectral": "smtime_spectral_r01.json"}[args.cov]
        sm = json.load(open(os.path.join(ROOT, "profiles", src)))
        a1 = sm["stages"]["A1"]
        top = sorted(sm["kernels"].items(), key=lambda kv: -kv[1]["share_sm_time"])[:6]
        share = {"stage_sm_time_share_of_record": a1["share_sm_time"],
                 "stage_serial_share_of_record": a1["share_serial"],
                 "top_kernels_sm_time_share": {k.split("(")[0].replace("ssi::<unnamed>::", ""):
                                               round(v["share_sm_time"], 4) for k, v in top},
                 "source": f"profiles/{src} (ncu sm__cycles_active.sum over one c3 record)"}
    except Exception:
        share = None
    kname = {"int8x3": "covariance A1 (int8x3: chan_max + slice + tcgen05 contraction + reduce)",
             "fp64": "covariance A1 (fp64 DMMA)",
             "spectral": "cross-spectral product of A1 (cross3m_kernel: FP64 DMMA, three real products per complex one)"}
    roof = {"bound": "tensor", "step_share": share, "kernel": kname[args.cov],
            "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak, "traffic": traffic,
            "peak_source": peak_src, "kernel_ms": iso_k, "stage_ms_in_pipeline": cov_ms,
            "algorithmic_flop_per_launch": work, "covariance_stage": stage}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        tot, parts, sample = oracle_sample(cfg, host[0])
        cpu = {"value": 1.0 / tot, "unit": UNIT, "cores": cores_used(), "kind": "oracle",
               "sample": sample, "stage_s": parts}

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
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
