"""c4 lag sweep (drivers.lag_sweep_3d) with 4 / 8 / 12 / 16 CUDA streams on one GPU (median of 3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2411_05510_b200 import api, drivers

LAGS = tuple(range(20, 81, 4))
cfg = synth.config("c3")
Yd = torch.from_numpy(synth.make_record(cfg)[0]).cuda()
P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, seed=cfg.philox_key)
for ns in (8, 16, 12, 4, 8, 16):
    ts = []
    for rep in range(4):
        tm = {}
        drivers.lag_sweep_3d(Yd, P, LAGS, api.CRITERIA_BRIDGE_3D, n_streams=ns, timing=tm)
        torch.cuda.synchronize()
        ts.append(tm["start"].elapsed_time(tm["stab"]))
    print(ns, "streams:", round(float(np.median(ts[1:])), 1), "ms", [round(t, 1) for t in ts])
