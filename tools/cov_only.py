"""Runs the c3 covariance a few times (profiling target; not a bench number).
    python tools/cov_only.py [config] [mode: int8x3 | spectral | fp64]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2411_05510_b200 import api
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c3")
Y, _ = synth.make_record(cfg)
Yd = torch.from_numpy(Y).cuda()
L = 2 * cfg.i - 1
mode = sys.argv[2] if len(sys.argv) > 2 else "int8x3"
ws = api._workspace(api.covariances_ws_bytes(cfg.N, cfg.l, L, 1, mode), Yd.device)
for _ in range(3):
    R = api.covariances(Yd, L, mode=mode, ws=ws)
torch.cuda.synchronize()
