"""Runs the c3 covariance (int8x3) a few times (profiling target; not a bench number)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2411_05510_b200 import api
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c3")
Y, _ = synth.make_record(cfg)
Yd = torch.from_numpy(Y).cuda()
L = 2 * cfg.i - 1
ws = api._workspace(api.covariances_ws_bytes(cfg.N, cfg.l, L, 1, "int8x3"), Yd.device)
for _ in range(3):
    R = api.covariances(Yd, L, mode="int8x3", ws=ws)
torch.cuda.synchronize()
