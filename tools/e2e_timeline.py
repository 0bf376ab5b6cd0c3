"""Timeline of the bench's end-to-end loop at the driver's 20 steps (CUDA events): when each
record's H2D copy, covariances and table are done, relative to the start (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2411_05510_b200 import drivers

cfg = synth.config("c3")
P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, seed=cfg.philox_key)
host = [synth.make_record(synth.config("c3", seed=cfg.seed + 100 * j))[0] for j in range(2)]
pinned = [torch.from_numpy(h).pin_memory() for h in host]
pipe = drivers.RecordPipeline(P, cfg.N, "cuda", n_streams=8)
pipe.reserve_host_inputs(pinned[0].shape, pinned[0].dtype)
tab_host = [[torch.empty_like(t, device="cpu").pin_memory() for t in e.table.tensors()] for e in pipe.engines]
cur = torch.cuda.current_stream()
for j in range(5):                                      # warm-up
    pipe.submit_host(pinned[j % 2], (j << 32) | cfg.i)
pipe.join(); torch.cuda.synchronize()
for K in (20, 20):
    a = torch.cuda.Event(enable_timing=True); a.record(cur)
    for st in pipe.streams:
        st.wait_stream(cur)
    marks = []
    for j in range(K):
        slot = pipe.j % 8
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        tab, st = pipe.submit_host(pinned[j % 2], (j << 32) | cfg.i, events=ev)
        cpy = torch.cuda.Event(enable_timing=True); cpy.record(pipe.copy_stream)
        with torch.cuda.stream(st):
            for hst, d in zip(tab_host[slot], tab.tensors()):
                hst.copy_(d, non_blocking=True)
            done = torch.cuda.Event(enable_timing=True); done.record(st)
        marks.append((cpy, ev[0], ev[1], done))
    pipe.join(cur)
    b = torch.cuda.Event(enable_timing=True); b.record(cur)
    torch.cuda.synchronize()
    print(f"K={K}: total {a.elapsed_time(b):.1f} ms = {K / a.elapsed_time(b) * 1e3:.1f} records/s")
    for j, (c, e0, e1, d) in enumerate(marks):
        print(f"  rec {j:2d}: copy done {a.elapsed_time(c):6.1f}  cov {a.elapsed_time(e0):6.1f}-{a.elapsed_time(e1):6.1f}  table on host {a.elapsed_time(d):6.1f}")
