"""Device time of Algorithm 1 verbatim (q = 0) at the paper's rank rule k = ceil(kbar(T) % T)
(PAPER.md:367-371): c2 (T = 2880, k = 735) and c3 (T = 11520, k = 2880), structured RSVD through
ssi_rsvd_toeplitz, CUDA events after warm-up, plus the per-kernel split (CUPTI)."""
import collections, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import synth
from paper_2411_05510_b200 import api

out = {}
for name in ("c2", "c3"):
    cfg = synth.config(name)
    Y, _ = synth.make_record(cfg)
    m = cfg.m
    k = -(-max(30.0 - 0.00156 * m, 25.0) * m // 100)
    k = int(k)
    R = api.covariances(torch.from_numpy(Y).cuda(), 2 * cfg.i - 1, 1, "spectral")
    ws = api._workspace(api.rsvd_toeplitz_ws_bytes(cfg.l, cfg.i, k, cfg.n_max), "cuda")
    run = lambda: api.rsvd_toeplitz(R, cfg.i, k, 0, cfg.philox_key, cfg.i, cfg.n_max, ws=ws)
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run()
        torch.cuda.synchronize()
    agg = collections.defaultdict(float)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            agg[e.name.replace("(anonymous namespace)::", "").split("(")[0][:70]] += e.device_time_total / 1e3
    top = dict(sorted(agg.items(), key=lambda x: -x[1])[:8])
    out[name] = {"T": m, "k": k, "q": 0, "ms": sorted(ts)[1], "kernel_ms_top": top}
print(json.dumps(out, indent=1))
