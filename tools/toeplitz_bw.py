"""Achieved HBM bandwidth of the explicit block-Toeplitz assembly (A2, ssi_toeplitz) at c3 and c4's
largest lag: bytes written (m^2 * 8) + R read, over CUDA-event time (warm, median of 5). The
timed RSVD path never forms T; this measures the explicit-T variant's assembly kernel."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_05510_b200 import api

out = {}
for name, l, i in (("c3", 192, 60), ("c4_i80", 192, 80)):
    R = torch.randn((2 * i - 1, l, l), dtype=torch.float64, device="cuda")
    m = l * i
    T = torch.empty((m, m), dtype=torch.float64, device="cuda")
    api.toeplitz(R, i, out=T)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); api.toeplitz(R, i, out=T); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[2]
    byt = m * m * 8 + R.numel() * 8
    out[name] = {"m": m, "ms": ms, "bytes": byt, "GBps": byt / (ms / 1e3) / 1e9}
print(json.dumps(out))
