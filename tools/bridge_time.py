"""The paper's own end-to-end workload at its own sizes (PAPER.md:518,
:541-544): one synthetic 2-hour San-Faustino-shaped acquisition (114 channels, 125 Hz) through
preprocessing, covariances, RSVD at the rank rule (q = 0), the modal sweep over orders 250..400,
stability criteria and the two-stage clustering — the 2D diagram at j_b = 76 (paper: ~204 s per
record on an i7-8750H) and the 3D diagram over j_b = 69..104 (paper: ~512 s). Device time,
CUDA events, after one warm-up; prints JSON."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth.raw import make_bridge_raw
from paper_2411_05510_b200 import api, drivers

raw, modes = make_bridge_raw()
rawd = torch.from_numpy(raw).cuda()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out = fn(); b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b), out


ms2, (tab, flags, cl) = timed(lambda: drivers.bridge_identify_2d(rawd))
f2 = cl.f.cpu().numpy()
tm = {}
ms3, (tabs, flags3, counts3, cl3) = timed(lambda: drivers.bridge_identify_3d(rawd, timing=tm))
f3 = cl3.f.cpu().numpy()
hit = lambda reps: int(sum(1 for f in modes.f if len(reps) and min(abs(reps - f) / f) < 0.01))
out = {"workload": "114 ch x 900000 FP32 at 125 Hz (2 h) -> 40 Hz; j_b = 76 (T = 8664, k = 2166, q = 0), orders 250..400",
       "identify_2d_ms": ms2, "paper_2d_rsvd_s": 204, "clusters_2d": int(cl.n_clusters), "modes_found_2d": hit(f2),
       "identify_3d_ms": ms3, "paper_3d_rsvd_s": 512, "clusters_3d": int(cl3.n_clusters), "modes_found_3d": hit(f3),
       "phases_3d_ms": {k: tm["start"].elapsed_time(v) for k, v in tm.items() if k != "start"},
       "stable_poles_3d": int(counts3.sum().item()), "retained_3d": int(cl3.n_retained), "true_modes": len(modes.f)}
print(json.dumps(out, indent=1))
