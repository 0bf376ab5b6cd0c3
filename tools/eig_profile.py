"""Per-order phase clocks of eig_order_kernel on one c3 record (development probe; the
kernel prints when SSI_EIG_PROFILE=2)."""
import os, sys
os.environ.setdefault("SSI_EIG_PROFILE", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2411_05510_b200 import drivers

cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c3")
Y, _ = synth.make_record(cfg)
Yd = torch.from_numpy(Y).cuda()
P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, seed=cfg.philox_key,
                        cov_mode="int8x3")
eng = drivers.Engine(P, cfg.N)
eng.identify(Yd, cfg.i)
torch.cuda.synchronize()
