"""One warm c3 record (covariances -> structured RSVD -> modal sweep) on one stream: the ncu
target for the per-kernel SM-time table (tools/smtime.py). Usage: record_profile.py [cov_mode]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2411_05510_b200 import drivers

mode = sys.argv[1] if len(sys.argv) > 1 else "spectral"
cfg = synth.config("c3")
Y, _ = synth.make_record(cfg)
Yd = torch.from_numpy(Y).cuda()
P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, seed=cfg.philox_key,
                        cov_mode=mode)
eng = drivers.Engine(P, cfg.N)
eng.identify(Yd, cfg.i)
torch.cuda.synchronize()
