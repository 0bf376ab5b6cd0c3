"""Device time of the NEXT-4 entry points (CUDA events on the launching stream, after warm-up):
ssi_preprocess on a 2-hour 114-channel 125 Hz record -> 40 Hz, and
ssi_frame_simulate of the paper's 5-minute 200 Hz 10-DOF record."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth.raw import make_raw_record
from paper_2411_05510_b200 import api


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


out = {}
Y, _ = make_raw_record(l=114, fs=125.0, N=900000, seed=482)
Yd = torch.from_numpy(Y).cuda()
N, l = Yd.shape
ws = api._workspace(api.preprocess_ws_bytes(N, l, 8), "cuda")
Z = torch.empty((288000, 114), dtype=torch.float32, device="cuda")
ms = timed(lambda: api.preprocess(Yd, 125.0, 40.0, out=Z, ws=ws))
# algorithmic work: 2 passes x (N L l samples) x 4 biquads x 5 FMA (forward + backward), the
# chunked scheme runs each recursion twice (pass A + pass B)
samples = N * 8 * l
out["preprocess_2h_bridge"] = {"ms": ms, "record": "114 ch x 900000 FP32 @125 Hz -> 288000 @40 Hz (L/M = 8/25)",
                               "hours_of_data_per_s": 2.0 / (ms / 1e3), "high_rate_samples": samples,
                               "hbm_bytes_min": N * l * 4 + 3 * samples * 8 + 288000 * l * 4,
                               "GBps_vs_min_traffic": (N * l * 4 + 3 * samples * 8 + 288000 * l * 4) / (ms * 1e6)}
Z2 = torch.empty((60000, 114), dtype=torch.float32, device="cuda")
ws2 = api._workspace(api.preprocess_ws_bytes(300000, l, 1), "cuda")
Y2 = Yd[:300000]
out["preprocess_integer_q5"] = {"ms": timed(lambda: api.preprocess(Y2, 200.0, 40.0, out=Z2, ws=ws2)),
                                "record": "114 ch x 300000 @200 Hz -> 60000 @40 Hz (q = 5)"}
out["frame_simulate_10dof"] = {"ms": timed(lambda: api.frame_simulate(60000, 200.0, 20.0, 0xE3, 1)),
                               "record": "10-DOF, 60000 + 2000 burn-in samples @200 Hz, SNR 20 dB"}
print(json.dumps(out, indent=1))
