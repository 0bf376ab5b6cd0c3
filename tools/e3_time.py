"""Times the E3 workload (10-DOF shear frame, j_b = 189, T = 1890, k = 512,
q = p = 0, orders 2..30) on one GPU: each stage and the whole chain, record resident in HBM,
CUDA events, median of 7 after warm-up. Prints one JSON object (evidence; not the bench line)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from synth.records import _simulate
from tests.analytic import shear_frame_modes
from paper_2411_05510_b200 import api

FS, N, L, I, K, SEED, NMAX = 200.0, 60000, 10, 189, 512, 0xE3, 30
Y = torch.from_numpy(_simulate(shear_frame_modes(FS), N, 0.1, np.random.default_rng([27, 0xE3]))).cuda()


def timed(fn, reps=7):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


R = api.covariances(Y, 2 * I - 1, 1, "spectral")
T = api.toeplitz(R, I)
U, S = api.rsvd_toeplitz(R, I, K, 0, SEED, I, NMAX)
out = {
    "workload": "E3: 10-DOF shear frame, fs 200 Hz, 5 min, SNR 20 dB, j_b 189 (T = 1890), k = 512, q = p = 0, orders 2..30",
    "ms": {
        "covariances_spectral": timed(lambda: api.covariances(Y, 2 * I - 1, 1, "spectral", out=R)),
        "toeplitz": timed(lambda: api.toeplitz(R, I, out=T)),
        "rsvd_explicit_T": timed(lambda: api.rsvd(T, K, 0, SEED, I, NMAX)),
        "rsvd_structured": timed(lambda: api.rsvd_toeplitz(R, I, K, 0, SEED, I, NMAX)),
        "modal_sweep": timed(lambda: api.modal_sweep(U, S, L, I, 2, NMAX, 2, 1.0 / FS)),
    },
}


def chain():
    R2 = api.covariances(Y, 2 * I - 1, 1, "spectral")
    U2, S2 = api.rsvd_toeplitz(R2, I, K, 0, SEED, I, NMAX)
    api.modal_sweep(U2, S2, L, I, 2, NMAX, 2, 1.0 / FS)


out["ms"]["whole_chain_structured"] = timed(chain)
out["paper_context"] = "PAPER.md:386-391 (CPU, MATLAB): full SVD 1.77 s, RSVD 0.32 s for this decomposition"
print(json.dumps(out))
