import os, sys, time
sys.path.insert(0, "/root/repo")
import torch, synth
from paper_2411_05510_b200 import api, drivers
cfg = synth.config("c4")
lags = list(cfg.lags)
Y = torch.from_numpy(synth.make_record(cfg)[0]).cuda()
for mode in ("spectral", "int8x3"):
    P = drivers.SweepParams(l=cfg.l, i=max(lags), n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, n_min=cfg.n_min,
                            n_step=cfg.n_step, seed=cfg.philox_key, cov_mode=mode)
    crit = api.CRITERIA_BRIDGE_3D
    for rep in range(3):
        torch.cuda.synchronize()
        a, b, c = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        a.record()
        R = drivers.sharded_covariances(Y, 159, 0, 1, mode, None)
        b.record()
        tables, flags, counts = drivers.lag_sweep_3d(Y, P, lags, crit)
        c.record()
        torch.cuda.synchronize()
        print(mode, "cov", round(a.elapsed_time(b), 2), "sweep", round(b.elapsed_time(c), 2), flush=True)
