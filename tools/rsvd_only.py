"""Runs one c3 structured RSVD (profiling target; not a bench number)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2411_05510_b200 import api, drivers
cfg = synth.config("c3")
Y, _ = synth.make_record(cfg)
P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, seed=cfg.philox_key,
                        cov_mode="int8x3")
eng = drivers.Engine(P, cfg.N)
R = eng.covariances(torch.from_numpy(Y).cuda())
for _ in range(2):
    api.rsvd_toeplitz(R, P.i, P.k, P.q, P.seed, P.i, P.n_max, U=eng.U, S=eng.S, ws=eng.ws_rsvd)
torch.cuda.synchronize()
