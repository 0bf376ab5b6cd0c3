"""Per-kernel device times of the NEXT-2 clustering on the c4 diagram (CUPTI via torch.profiler;
not a bench number): drivers.lag_sweep_3d once, then api.cluster3d profiled."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import synth
from paper_2411_05510_b200 import api, drivers

cfg = synth.config("c4")
Y, _ = synth.make_record(cfg)
Yd = torch.from_numpy(Y).cuda()
P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, seed=cfg.philox_key)
crit = api.CRITERIA_BRIDGE_3D
lags = list(cfg.lags)
tabs, flags, counts = drivers.lag_sweep_3d(Yd, P, lags, crit)
T = [tabs[i] for i in lags]
ms = int(0.2 * len(cfg.orders) * len(lags))
for _ in range(2):
    cl = api.cluster3d(T, flags, crit, min_size=ms)
torch.cuda.synchronize()
t0 = time.perf_counter()
cl = api.cluster3d(T, flags, crit, min_size=ms)
torch.cuda.synchronize()
print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms; stable {cl.n_stable} retained {cl.n_retained} "
      f"components {cl.n_components} merges {cl.n_merges} clusters {cl.n_clusters} fcm iters {cl.fcm_iters}")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    api.cluster3d(T, flags, crit, min_size=ms)
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
