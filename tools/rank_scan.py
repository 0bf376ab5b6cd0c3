"""The paper's rank study (§3.1.2, Fig. 3) on the GPU: for the 10-DOF shear frame
(ssi_frame_simulate, 5 min at 200 Hz) at SNR 10/15/20/25 dB and time-lag steps j_b (T = 10 j_b),
find the minimum percentage rank kbar at which the RSVD-CoV-SSI stabilization diagram (Algorithm 1
verbatim, q = p = 0) reproduces the classical CoV-SSI one (the full SVD of T: the same path with
k = T), and compare kbar(T) with Eq. (empirical_formula) max{30 - 0.00156 T; 25} %.

Settings as printed: model orders 10..100 step 2; HC xi <= 10 %, MPC > 60 %,
MPD < 50 %; SC along the order axis 2 %, 2 %, 5 %; matching tolerances 1 % (f), 1 % (xi), 2 %
(1 - MAC). Reading R-1: "the modal characteristics converge" = the modes identified
from the two diagrams (the stable poles of each, clustered by the same two-stage clustering,
ssi_cluster_stage1/2; a mode = a cluster present at >= MIN_SIZE of the model orders, its
medoid's f, xi and shape) match one to one within those tolerances; kbar = the smallest rank
(1 % steps) from which every larger rank of the scan matches. T is limited to 4096 here (k = T for the reference SVD:
the block Jacobi's limit), i.e. j_b = 100..400. Prints JSON.

    python tools/rank_scan.py [jb ...]"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2411_05510_b200 import api

FS, N, L = 200.0, 60000, 10
ORDERS = (10, 100, 2)
CRIT = api.Criteria(alpha_f=0.02, alpha_xi=0.02, alpha_mac=0.05)
TOL = (0.01, 0.01, 0.02)
JBS = [int(a) for a in sys.argv[1:]] or [100, 150, 200, 250, 300, 350, 400]


MIN_SIZE = 10   # of the 46 orders 10..100


def modes(U, S, i):
    tab = api.modal_sweep(U, S, L, i, *ORDERS, 1.0 / FS)
    flags, _ = api.stab3d([tab], CRIT)
    c = api.cluster3d([tab], flags, CRIT)
    keep = (c.size >= MIN_SIZE).cpu().numpy()
    f, xi = c.f.cpu().numpy()[keep], c.xi.cpu().numpy()[keep]
    sh = c.shape.cpu().numpy()[keep]
    return f, xi, sh[..., 0] + 1j * sh[..., 1], int(c.n_stable), c.size.cpu().numpy()[keep]


def representatives(m):
    """The identified modes: clusters of size >= MIN_SIZE grouped by frequency (a new group when
    the next frequency is more than 2 % above the previous), the largest cluster of each group."""
    f, size = m[0], m[4]
    order = np.argsort(f)
    groups, cur = [], []
    for j in order:
        if cur and f[j] > f[cur[-1]] * 1.02:
            groups.append(cur)
            cur = []
        cur.append(j)
    if cur:
        groups.append(cur)
    return [max(g, key=lambda j: (size[j], -j)) for g in groups]


def worst(ref, got):
    """Per identified mode of ref, the closest mode of got by d = df + dxi + (1 - MAC); returns
    the worst (df, dxi, 1 - MAC) over ref's modes and the mode counts."""
    ra, ga = representatives(ref), representatives(got)
    w = np.zeros(3)
    for j in ra:
        fb, xb, sb = got[0][ga], got[1][ga], got[2][ga]
        df = np.abs(fb - ref[0][j]) / np.maximum(fb, ref[0][j])
        dx = np.abs(xb - ref[1][j]) / np.maximum(xb, ref[1][j])
        mac = np.abs(sb.conj() @ ref[2][j]) ** 2 / (np.sum(np.abs(sb) ** 2, axis=1) * np.sum(np.abs(ref[2][j]) ** 2))
        q = int(np.argmin(df + dx + (1 - mac)))
        w = np.maximum(w, [df[q], dx[q], 1 - mac[q]])
    return w, len(ra), len(ga)


def matches(ref, got):
    w, nr, ng = worst(ref, got)
    return nr == ng and bool(np.all(w <= TOL)), w


rows = []
for snr in (10.0, 15.0, 20.0, 25.0):
    Y = api.frame_simulate(N, FS, snr, seed=0xF163, stream_id=int(snr), dtype=torch.float32)
    R = api.covariances(Y, 2 * max(JBS) - 1, 1, "spectral", check=True)
    for jb in JBS:
        T = L * jb
        U, S = api.rsvd_toeplitz(R, jb, T, 0, 0x5EED, jb, ORDERS[1], check=True)     # full SVD (k = T)
        ref = modes(U, S, jb)
        ok, worst_at = {}, {}
        pct = 2
        while pct <= 60:
            k = max(ORDERS[1], math.ceil(pct * T / 100))
            Ur, Sr = api.rsvd_toeplitz(R, jb, k, 0, 0x5EED, jb, ORDERS[1], check=True)
            ok[pct], w = matches(ref, modes(Ur, Sr, jb))
            worst_at[pct] = [round(float(x), 4) for x in w]
            # stop once a run of 5 consecutive ranks matches
            if pct >= 6 and all(ok.get(pct - d, False) for d in range(5)):
                break
            pct += 1
        kbar = None
        for p in sorted(ok):
            if all(ok[q] for q in ok if q >= p):
                kbar = p
                break
        rows.append({"snr_db": snr, "jb": jb, "T": T, "kbar_pct": kbar,
                     "rule_pct": max(30.0 - 0.00156 * T, 25.0),
                     "modes_svd": len(representatives(ref)),
                     "f_svd": [round(float(ref[0][j]), 3) for j in representatives(ref)],
                     "worst_df_dxi_dmac": {p: worst_at[p] for p in (10, 20, 25, 30, 40) if p in worst_at},
                     "stable_poles_svd": ref[3], "matched": sorted(p for p in ok if ok[p])})
        print(json.dumps(rows[-1]), flush=True)
print(json.dumps({"rank_scan": rows}))
