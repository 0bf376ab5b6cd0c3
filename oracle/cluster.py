"""Two-stage 3D clustering of the stable poles (§2.3 step iii; PAPER.md:402-415,
§3.1.3; §3.2.2). TEST INFRASTRUCTURE (see oracle/__init__.py).

PAPER.md:293: "A two-stage clustering approach is adopted ... a fuzzy C-means clustering
algorithm is followed by a hierarchical clustering one ... the previously identified stable
poles are collected and divided into two clusters (possibly physical and certainly unphysical)
based on a comprehensive evaluation of their stability (along the time lag and model order
axes) in terms of frequency, damping ratio, MAC, MPC, and MPD values. Only the resulting cluster
of possibly physical poles are retained for Stage II. This stage involves a hierarchical
clustering algorithm that constructs a hierarchical Π-shaped dendrogram based on a distance
metric defined as the sum of the relative differences of the retained poles in terms of
frequencies, damping and MAC. Finally, the physical modes ... can be identified by imposing a
threshold for the distance metric and a minimum cluster size."
PAPER.md:405 defines d_f^{ij} = |f_i − f_j| / max(f_i, f_j), d_ξ^{ij} likewise; PAPER.md:415:
"fuzzy membership grade P ... possibly physical poles if P ≥ 0.5"; the physical cluster's
centroid "is positioned very close to the origin".

Readings (C-1 .. C-5; SPEC.md:445-483 for the shapes of the operations):
  C-1 Stage-I features of a pole flagged stable by stab3d (flag 2): its best neighbour is the
      kept predecessor — order axis (g, o−1) first, then lag axis (g−1, o), slots ascending —
      that meets all three soft criteria and minimises d_f + d_ξ + (1 − MAC) (first one kept on
      ties); x = (d_f, d_ξ, 1 − MAC, 1 − MPC, MPD) with MPC and MPD of the pole itself.
  C-2 Fuzzy C-means: c = 2, fuzzifier m = 2, Euclidean distance, centroids initialised at the
      feature-wise minimum and maximum of the points (deterministic), then alternate
      memberships u_ij = 1 / Σ_k (d_ij² / d_ik²)^{1/(m−1)} (a point at distance 0 from a centroid
      takes membership 1 there, 0 elsewhere, the first such centroid on ties) and centroids
      v_j = Σ_i u_ij^m x_i / Σ_i u_ij^m until the largest centroid coordinate moves < tol = 1e−10
      (or 1000 iterations); memberships are then recomputed from the final centroids.
  C-3 The physical cluster is the one whose centroid has the smaller Euclidean norm; a pole is
      retained iff its membership there is ≥ 0.5.
  C-4 Stage II: d(i, j) = d_f + d_ξ + (1 − MAC) between retained poles, average linkage
      (UPGMA), flat clusters = merges at height ≤ cutoff; clusters smaller than min_size are
      dropped; representative f and ξ = lower median of the members, shape = the medoid member
      (least summed distance to the other members, lowest index on ties); clusters ordered by
      representative f, then by their smallest member index.
"""
import numpy as np
from scipy.cluster.hierarchy import linkage, fcluster
from scipy.spatial.distance import squareform

from .indicators import mac
from .stab import _hard_ok


def _sc(p, q, crit):
    df = abs(p.f - q.f) / max(p.f, q.f)
    dxi = abs(p.xi - q.xi) / max(p.xi, q.xi)
    dm = 1.0 - mac(p.shape, q.shape)
    return df, dxi, dm, (df <= crit.alpha_f and dxi <= crit.alpha_xi and dm <= crit.alpha_mac)


def stable_pole_features(tables, flags, crit):
    """tables[g][o] = OrderCell (lags increasing, orders increasing), flags [G][O][cap] from
    stab3d. Returns (idx [n][3] of (g, o, s) in lexicographic order, X [n][5]) — reading C-1."""
    G, O = len(tables), len(tables[0])
    idx, X = [], []
    for g in range(G):
        for o in range(O):
            for s, p in enumerate(tables[g][o].poles):
                if flags[g][o][s] != 2:
                    continue
                best = None
                for gg, oo in ((g, o - 1), (g - 1, o)):
                    if gg < 0 or oo < 0:
                        continue
                    for q in tables[gg][oo].poles:
                        if not _hard_ok(q, crit):
                            continue
                        df, dxi, dm, ok = _sc(p, q, crit)
                        if ok and (best is None or df + dxi + dm < best[0]):
                            best = (df + dxi + dm, df, dxi, dm)
                assert best is not None, "a stable pole has an SC neighbour by definition"
                idx.append((g, o, s))
                X.append([best[1], best[2], best[3], 1.0 - p.mpc, p.mpd])
    return np.array(idx, dtype=np.int64).reshape(-1, 3), np.array(X, dtype=np.float64).reshape(-1, 5)


def fcm_memberships(X, V, m: float = 2.0):
    """u_ij = 1 / Σ_k (d_ij² / d_ik²)^{1/(m−1)}; a zero distance takes the whole membership."""
    D2 = ((X[:, None, :] - V[None, :, :]) ** 2).sum(axis=2)
    U = np.zeros_like(D2)
    for i in range(X.shape[0]):
        z = np.flatnonzero(D2[i] == 0.0)
        if z.size:
            U[i, z[0]] = 1.0
        else:
            U[i] = 1.0 / ((D2[i][:, None] / D2[i][None, :]) ** (1.0 / (m - 1.0))).sum(axis=1)
    return U


def fuzzy_cmeans(X, c: int = 2, m: float = 2.0, tol: float = 1e-10, max_iter: int = 1000):
    """Reading C-2. Returns (U [n][c], V [c][d], iterations)."""
    X = np.asarray(X, dtype=np.float64)
    lo, hi = X.min(axis=0), X.max(axis=0)
    V = np.array([lo + (hi - lo) * (j / (c - 1)) for j in range(c)])
    it = 0
    for it in range(1, max_iter + 1):
        W = fcm_memberships(X, V, m) ** m
        Vn = (W.T @ X) / W.sum(axis=0)[:, None]
        delta = np.abs(Vn - V).max()
        V = Vn
        if delta < tol:
            break
    return fcm_memberships(X, V, m), V, it


def select_physical(U, V):
    """Reading C-3: (index of the physical cluster, boolean mask of retained poles)."""
    j = int(np.argmin(np.linalg.norm(V, axis=1)))
    return j, U[:, j] >= 0.5


def pole_distances(f, xi, shapes):
    """d(i, j) = d_f + d_ξ + (1 − MAC) between poles; shapes [n][l] complex."""
    f = np.asarray(f, dtype=np.float64)
    xi = np.asarray(xi, dtype=np.float64)
    S = np.asarray(shapes, dtype=np.complex128)
    nrm = np.einsum("ij,ij->i", S.conj(), S).real
    M = np.abs(S.conj() @ S.T) ** 2 / np.outer(nrm, nrm)
    D = (np.abs(f[:, None] - f[None, :]) / np.maximum(f[:, None], f[None, :])
         + np.abs(xi[:, None] - xi[None, :]) / np.maximum(xi[:, None], xi[None, :])
         + (1.0 - M))
    np.fill_diagonal(D, 0.0)
    return D


def hierarchical_clusters(D, f, xi, cutoff: float, min_size: int):
    """Reading C-4 on a distance matrix D (library primitive: scipy's average linkage).
    Returns (labels [n] in 0..K-1 or -1, list of dicts {f, xi, medoid, size, members})."""
    n = D.shape[0]
    if n == 1:
        raw = np.array([1])
    else:
        Z = linkage(squareform(D, checks=False), method="average")
        raw = fcluster(Z, t=cutoff, criterion="distance")
    groups = {}
    for i, r in enumerate(raw):
        groups.setdefault(int(r), []).append(i)
    clusters = []
    for mem in groups.values():
        if len(mem) < min_size:
            continue
        mem = sorted(mem)
        fs = np.sort(np.asarray(f)[mem])
        xs = np.sort(np.asarray(xi)[mem])
        sums = D[np.ix_(mem, mem)].sum(axis=1)
        medoid = mem[int(np.argmin(sums))]
        clusters.append(dict(f=float(fs[(len(mem) - 1) // 2]), xi=float(xs[(len(mem) - 1) // 2]),
                             medoid=medoid, size=len(mem), members=mem))
    clusters.sort(key=lambda c: (c["f"], c["members"][0]))
    labels = -np.ones(n, dtype=np.int64)
    for k, c in enumerate(clusters):
        labels[c["members"]] = k
    return labels, clusters


def cluster_3d(tables, flags, crit, cutoff: float = 0.10, min_size: int = 1):
    """Stage I + stage II on a 3D grid (readings C-1 .. C-4). Returns a dict with the stable-pole
    index list, features, memberships, centroids, the physical cluster, the retained mask and the
    stage-II labels (over the retained poles) and clusters."""
    idx, X = stable_pole_features(tables, flags, crit)
    U, V, it = fuzzy_cmeans(X)
    phys, keep = select_physical(U, V)
    r = idx[keep]
    poles = [tables[g][o].poles[s] for g, o, s in r]
    f = np.array([p.f for p in poles])
    xi = np.array([p.xi for p in poles])
    sh = np.array([p.shape for p in poles]).reshape(len(poles), -1)
    D = pole_distances(f, xi, sh) if len(poles) else np.zeros((0, 0))
    labels, clusters = hierarchical_clusters(D, f, xi, cutoff, min_size) if len(poles) else (np.zeros(0, int), [])
    return dict(idx=idx, X=X, U=U, V=V, iters=it, phys=phys, keep=keep, retained=r, labels=labels,
                clusters=clusters, f=f, xi=xi, shapes=sh)
