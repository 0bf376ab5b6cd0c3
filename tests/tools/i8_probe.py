import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2411_05510_b200 import api
import oracle
N, l, L = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(0)
Y = rng.standard_normal((N, l)).astype(np.float32)
try:
    R = api.covariances(torch.from_numpy(Y).cuda(), L, mode="int8x3", check=True).cpu().numpy()
    Ro = oracle.covariances(Y, L)
    print("dbg", os.environ.get("SSI_I8_DEBUG"), "rel err", np.linalg.norm(R - Ro) / np.linalg.norm(Ro), "R00", R[0,0,:3], Ro[0,0,:3])
except Exception as e:
    print("dbg", os.environ.get("SSI_I8_DEBUG"), "FAIL", str(e)[:200])
