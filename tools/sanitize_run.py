"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

c1 and c2 records go through Engine.identify (A1-A11, one stream) and through a 3-stream
RecordPipeline (the bench's overlap pattern, with the low-priority covariance streams), then one
two-lag stab3d. The c2 record is cut to N = 40000 samples so the run stays within minutes under
the sanitizer's ~100x slowdown. Exits non-zero if any device status word is set.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_05510_b200 import api, drivers  # noqa: E402
from synth import records  # noqa: E402


def params(cfg, **kw):
    return drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs,
                               n_min=cfg.n_min, n_step=cfg.n_step, seed=7, **kw)


def main():
    dev = torch.device("cuda:0")
    cases = (("c1", None), ("c2", 40000))
    if len(sys.argv) > 1:
        cases = tuple(c for c in cases if c[0] in sys.argv[1:])
    for name, N in cases:
        cfg = records.config(name)
        Y = torch.from_numpy(records.make_record(cfg, 0, N=N)[0]).to(dev)
        for structured in (True, False):
            P = params(cfg, structured=structured)
            eng = drivers.Engine(P, Y.shape[0], dev)
            tab = eng.identify(Y, stream_id=1, check=True)
            print(name, "structured" if structured else "explicit", "poles", int(tab.count.clamp(min=0).sum()))
        P = params(cfg)
        pipe = drivers.RecordPipeline(P, Y.shape[0], dev, n_streams=3)
        for j in range(4):
            pipe.submit(Y, j)
        pipe.join()
        torch.cuda.synchronize()
        pipe.check()
        tables, flags, counts = drivers.lag_sweep_3d(Y, P, [cfg.i - 2, cfg.i], api.CRITERIA_10DOF_3D, n_streams=2)
        torch.cuda.synchronize()
        print(name, "pipeline + 2-lag sweep ok; stable", int(counts.sum()))
    print("SANITIZE_RUN_OK")


if __name__ == "__main__":
    main()
