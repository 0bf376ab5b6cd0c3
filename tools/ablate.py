"""Development probe: pipelined records/s with stages removed (not a bench number).
  python tools/ablate.py [streams]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2411_05510_b200 import api, drivers

cfg = synth.config("c3")
Y, _ = synth.make_record(cfg)
Ys = [torch.from_numpy(Y).cuda(), torch.from_numpy(synth.make_record(synth.config("c3", seed=103))[0]).cuda()]
P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, seed=cfg.philox_key,
                        cov_mode=os.environ.get("SSI_COV_MODE", "spectral"))
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 8
engines = [drivers.Engine(P, cfg.N) for _ in range(ns)]
streams = [torch.cuda.Stream() for _ in range(ns)]


def run(stages, n=48):
    def one(j):
        e, st = engines[j % ns], streams[j % ns]
        with torch.cuda.stream(st):
            if "cov" in stages:
                e.covariances(Ys[j % 2])
            if "rsvd" in stages:
                api.rsvd_toeplitz(e.R, P.i, P.k, P.q, P.seed, P.i, P.n_max, U=e.U, S=e.S, ws=e.ws_rsvd)
            if "modal" in stages:
                api.modal_sweep(e.U, e.S, P.l, P.i, P.n_min, P.n_max, P.n_step, P.dt, out=e.table, ws=e.ws_modal)
    for j in range(ns):
        one(j)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for j in range(n):
        one(j)
    torch.cuda.synchronize()
    return n / (time.perf_counter() - t0)


for stages in (("cov", "rsvd", "modal"), ("cov",), ("rsvd",), ("modal",), ("cov", "rsvd"), ("rsvd", "modal"),
               ("cov", "modal"), ("cov", "rsvd", "modal")):
    r = run(stages)
    print(f"{'+'.join(stages):20s} {r:7.2f} rec/s  {1e3 / r:7.2f} ms/rec")
