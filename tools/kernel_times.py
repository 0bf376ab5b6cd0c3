"""Per-kernel device times for one c3 record (CUPTI via torch.profiler; not a bench number)."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import synth
from paper_2411_05510_b200 import drivers

cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c3")
mode = sys.argv[2] if len(sys.argv) > 2 else "fp64"
Y, _ = synth.make_record(cfg)
Yd = torch.from_numpy(Y).cuda()
P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, seed=cfg.philox_key, cov_mode=mode)
eng = drivers.Engine(P, cfg.N)
for _ in range(2):
    eng.identify(Yd, cfg.i)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.identify(Yd, cfg.i)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name[:90]][0] += 1
        agg[e.name[:90]][1] += e.device_time_total / 1e3
tot = sum(v[1] for v in agg.values())
print(f"total kernel time {tot:.2f} ms")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v:9.3f} ms {c:4d}x  {100 * v / tot:5.1f}%  {n}")
