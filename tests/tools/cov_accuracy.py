"""Measured covariance error of the int8x3 split path vs the FP64 oracle on a full config record."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle, synth
from paper_2411_05510_b200 import api
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c3")
Y, _ = synth.make_record(cfg)
L = 2 * cfg.i - 1
Yd = torch.from_numpy(Y).cuda()
R8 = api.covariances(Yd, L, mode="int8x3", check=True).cpu().numpy()
R64 = api.covariances(Yd, L, mode="fp64", check=True).cpu().numpy()
t0 = time.time(); Ro = oracle.covariances(Y, L); t = time.time() - t0
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
print(f"{cfg.name}: int8x3 rel {rel(R8, Ro):.3e}  fp64 rel {rel(R64, Ro):.3e}  max per-lag int8 {max(rel(R8[k], Ro[k]) for k in range(L)):.3e}  oracle {t:.1f}s")
