"""Per-kernel device times of the c3 covariance call (CUPTI via torch.profiler), averaged over
20 calls; for kernel A/B experiments (not a bench number).
    python tools/cov_time.py [config] [mode]"""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import synth
from paper_2411_05510_b200 import api

cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c3")
mode = sys.argv[2] if len(sys.argv) > 2 else "spectral"
Y, _ = synth.make_record(cfg)
Yd = torch.from_numpy(Y).cuda()
L = 2 * cfg.i - 1
ws = api._workspace(api.covariances_ws_bytes(cfg.N, cfg.l, L, 1, mode), Yd.device)
for _ in range(3):
    api.covariances(Yd, L, mode=mode, ws=ws)
torch.cuda.synchronize()
REP = 20
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
    for _ in range(REP):
        api.covariances(Yd, L, mode=mode, ws=ws)
    torch.cuda.synchronize()
agg = collections.defaultdict(float)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name[:60]] += e.device_time_total / 1e3 / REP
print(" ".join(os.environ.get("SSI_NVCC_EXTRA", "default").split()), f"total {sum(agg.values()):.3f} ms",
      "; ".join(f"{n.split('::')[-1][:24]} {v:.3f}" for n, v in sorted(agg.items(), key=lambda x: -x[1])[:4]))
