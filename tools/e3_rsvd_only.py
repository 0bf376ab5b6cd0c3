"""One E3 structured RSVD (k = 512, q = 0) after one warm-up call (profiling target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from synth.records import _simulate
from tests.analytic import shear_frame_modes
from paper_2411_05510_b200 import api
Y = torch.from_numpy(_simulate(shear_frame_modes(200.0), 60000, 0.1, np.random.default_rng([27, 0xE3]))).cuda()
R = api.covariances(Y, 377, 1, "spectral")
for _ in range(2):
    api.rsvd_toeplitz(R, 189, 512, 0, 0xE3, 189, 30)
torch.cuda.synchronize()
