"""Single-GPU timings of the two repetition workloads (not bench.py's metric):
  c4: the full 3D lag sweep (i = 20..80 step 4, covariances once to lag 159, 16 structured RSVDs +
      modal sweeps, stab3d) -- wall time on the device (CUDA events), after one warm-up sweep;
  c5: continuous monitoring, records/s of the RecordPipeline (8 in flight) over 32 records
      (8 distinct drifting c5 records rotated, device-resident).
Prints one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2411_05510_b200 import api, drivers

out = {}
# ---- c4
cfg = synth.config("c4")
lags = list(cfg.lags)
Y = torch.from_numpy(synth.make_record(cfg)[0]).cuda()
P = drivers.SweepParams(l=cfg.l, i=max(lags), n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, n_min=cfg.n_min,
                        n_step=cfg.n_step, seed=cfg.philox_key, cov_mode=os.environ.get("SSI_COV_MODE", "spectral"))
crit = api.CRITERIA_BRIDGE_3D
drivers.lag_sweep_3d(Y, P, lags, crit)
torch.cuda.synchronize()
ts = []
for _ in range(7):   # median of 7 after a warm-up (stream interleaving of 16 lags varies run to run)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tables, flags, counts = drivers.lag_sweep_3d(Y, P, lags, crit)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
out["c4_sweep_ms"] = sorted(ts)[3]
out["c4_sweep_ms_min"] = min(ts)
out["c4_sweep_ms_all"] = ts
out["c4_lags"] = len(lags)
out["c4_stable_poles"] = int(counts.sum().item())
del Y
# ---- c5
cfg = synth.config("c5")
recs = [torch.from_numpy(synth.make_record(cfg, r)[0]).cuda() for r in range(8)]
P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, n_min=cfg.n_min,
                        n_step=cfg.n_step, seed=cfg.philox_key, cov_mode=os.environ.get("SSI_COV_MODE", "spectral"))
pipe = drivers.RecordPipeline(P, cfg.N, "cuda", n_streams=8)
for j in range(8):
    pipe.submit(recs[j], (j << 32) | cfg.i)
pipe.join()
torch.cuda.synchronize()
n = 32
a.record()
for st in pipe.streams:
    st.wait_stream(torch.cuda.current_stream())
for j in range(n):
    pipe.submit(recs[j % 8], (j << 32) | cfg.i)
pipe.join()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b)
out["c5_records_per_s"] = n / (ms / 1e3)
out["c5_ms_per_record"] = ms / n
out["gpu"] = torch.cuda.get_device_name()
out["cov_mode"] = P.cov_mode
print(json.dumps(out))
