"""Dumps U, S of one structured RSVD on the c2 and c3 records (for bit-for-bit A/B of build
variants, e.g. the Jacobi kernels). Usage: dump_rsvd.py out_prefix"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2411_05510_b200 import api, drivers

for name in ("c2", "c3"):
    cfg = synth.config(name)
    Y, _ = synth.make_record(cfg)
    P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, seed=cfg.philox_key)
    eng = drivers.Engine(P, cfg.N)
    R = eng.covariances(torch.from_numpy(Y).cuda())
    U, S = api.rsvd_toeplitz(R, P.i, P.k, P.q, P.seed, P.i, P.n_max, ws=eng.ws_rsvd)
    torch.cuda.synchronize()
    np.save(f"{sys.argv[1]}_{name}_U.npy", U.cpu().numpy())
    np.save(f"{sys.argv[1]}_{name}_S.npy", S.cpu().numpy())
