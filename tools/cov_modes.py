"""Times ssi_covariances per mode on a config's record (CUDA events, warm) and compares the
modes with each other at full size: a development probe, not a bench number."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2411_05510_b200 import api

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["int8x3", "spectral"]
cfg = synth.config(name)
Y, _ = synth.make_record(cfg)
Yd = torch.from_numpy(Y).cuda()
L = 2 * cfg.i - 1
out = {}
Rs = {}
for mode in modes:
    ws = api._workspace(api.covariances_ws_bytes(cfg.N, cfg.l, L, 1, mode), Yd.device)
    R = api.covariances(Yd, L, mode=mode, ws=ws, check=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        api.covariances(Yd, L, mode=mode, ws=ws, out=R)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    Rs[mode] = R.cpu().numpy()
    out[mode] = {"ms": sorted(ts), "ws_GB": ws.numel() / 1e9}
ref = Rs.get("fp64", Rs.get("spectral"))
for mode in modes:
    d = Rs[mode] - ref
    out[mode]["rel_vs_" + ("fp64" if "fp64" in Rs else "spectral")] = float(np.linalg.norm(d) / np.linalg.norm(ref))
print(json.dumps(out, indent=1))
