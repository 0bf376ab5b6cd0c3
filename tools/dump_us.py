"""Dumps U, S of one c3 record (covariances -> structured RSVD) to gpurun_out/c3_us.npz: the input
of tools/aed_model.py (development probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2411_05510_b200 import api
cfg = synth.config("c3")
Y, _ = synth.make_record(cfg)
Yd = torch.from_numpy(Y).cuda()
R = api.covariances(Yd, 2 * cfg.i - 1, mode="spectral")
U, S = api.rsvd_toeplitz(R, cfg.i, cfg.n_max + cfg.p, cfg.q, cfg.philox_key, 0, cfg.n_max, check=True)
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/c3_us.npz", U=U.cpu().numpy(), S=S.cpu().numpy())
print(U.shape, S[:5])
