"""Per-rank work of the c4 3D lag sweep at N = 1, 2, 4, 8 ranks, measured on ONE B200 (gpurun
gives one GPU): for each rank of an N-rank run, the rank's own part of drivers.lag_sweep_3d —
its time shard of the spectral covariance sums (ssi_covariances, normalize = 0) and its LPT
share of the lags (drivers.run_lags, 8 streams) — is run alone on the device and timed with CUDA
events (median of 3). The slowest rank bounds the N-rank sweep; the collectives (one all-reduce
of the FP64 sums, one all_gather of the pole tables) are NOT measured here and are listed with
their byte counts only. A projection from measured per-rank work, not a multi-GPU measurement.
    python tools/sweep_projection.py [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2411_05510_b200 import api, drivers

LAGS = tuple(range(20, 81, 4))
cfg = synth.config("c3")
Y, _ = synth.make_record(cfg)
Yd = torch.from_numpy(Y).cuda()
P = drivers.SweepParams(l=cfg.l, i=cfg.i, n_max=cfg.n_max, p=cfg.p, q=cfg.q, fs=cfg.fs, seed=cfg.philox_key)
lag_hi = 2 * max(LAGS) - 1
N = Y.shape[0]
ws_c = api._workspace(api.covariances_ws_bytes(N, P.l, lag_hi, 1, P.cov_mode), Yd.device)
R = api.covariances(Yd, lag_hi, 1, P.cov_mode, ws=ws_c)
Rraw = torch.empty_like(R)
cur = torch.cuda.current_stream()


def rank_work(W, r):
    tb, te = drivers.time_shards(N, W)[r]
    mine = drivers.lpt_assign(list(LAGS), W)[r]
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    e[0].record(cur)
    api.covariances(Yd, lag_hi, 1, P.cov_mode, t_begin=tb, t_end=te, normalize=False, out=Rraw, ws=ws_c)
    e[1].record(cur)
    keep = None
    if mine:
        keep = drivers.run_lags(R, P, mine, 8)
        for st in keep[2]:
            cur.wait_stream(st)
    e[2].record(cur)
    torch.cuda.synchronize()
    del keep                                             # workspaces freed after the streams finished
    return e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), mine


for _ in range(2):
    rank_work(1, 0)                                      # warm-up (workspaces, first launches)
# the whole single-GPU sweep through the product driver, for comparison with rank_work(1, 0)
crit = api.CRITERIA_BRIDGE_3D
full = []
for _ in range(3):
    tm = {}
    drivers.lag_sweep_3d(Yd, P, LAGS, crit, timing=tm)
    torch.cuda.synchronize()
    full.append(tm["start"].elapsed_time(tm["stab"]))
print("lag_sweep_3d (1 GPU):", [round(x, 1) for x in full])
out = {"how": __doc__.split("\n    python")[0], "workload": "c4: c3 record, i = 20..80 step 4 (16 lags)",
       "table_bytes": None, "by_world": {}, "lag_sweep_3d_1gpu_ms": full}
tab_bytes = sum(t.numel() * t.element_size() for t in api.PoleTable.empty(P.n_min, P.n_max, P.n_step, P.l, "cuda").tensors())
out["table_bytes"] = tab_bytes
for W in (1, 2, 4, 8):
    ranks = []
    for r in range(W):
        reps = [rank_work(W, r) for _ in range(3)]
        print(W, r, [round(x[0] + x[1], 1) for x in reps])
        cov = float(np.median([x[0] for x in reps]))
        lag = float(np.median([x[1] for x in reps]))
        ranks.append({"rank": r, "lags": reps[0][2], "cov_shard_ms": cov, "lags_ms": lag, "total_ms": cov + lag})
    slow = max(ranks, key=lambda d: d["total_ms"])
    out["by_world"][W] = {"ranks": ranks, "slowest_rank_ms": slow["total_ms"],
                          "collectives_not_timed": {"all_reduce_bytes": int(R.numel() * 8),
                                                    "all_gather_bytes": int(tab_bytes * len(LAGS))}}
    print(W, "ranks: slowest", round(slow["total_ms"], 2), "ms", [round(d["total_ms"], 1) for d in ranks])
base = out["by_world"][1]["slowest_rank_ms"]
for W, d in out["by_world"].items():
    d["projected_speedup_excl_collectives"] = base / d["slowest_rank_ms"]
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep_projection.json", "w"), indent=1)
