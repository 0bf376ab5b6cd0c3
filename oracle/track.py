"""Modal tracking over a monitoring campaign (§3.2.2; Table 4 at PAPER.md:555-585).
TEST INFRASTRUCTURE (see oracle/__init__.py).

PAPER.md:544: "the modes derived from the 3D stabilization diagram were used to perform the
tracking over the reference period. The main tracking parameters used in the analysis consider
the maximum relative differences in terms of frequencies and MACs equal to 5% and 15%";
Table 4: "success ratios ... defined as the ratio between the number of sets of time histories
in which each mode was identified and the total number of time histories", "The reference
modal properties are those identified by 3D-RSVD from the first acquisition record".

Reading C-5: a session mode c is a candidate for reference
mode r iff d_f = |f_c − f_r| / max(f_c, f_r) ≤ df_max and 1 − MAC(φ_c, φ_r) ≤ macd_max (the
printed "MACs equal to 15%" read as a bound on 1 − MAC); candidates are assigned one-to-one by
ascending score d_f + (1 − MAC), ties to the lower reference index, then the lower candidate
index (greedy); success ratio = 100 × matched sessions / sessions.
"""
import numpy as np

from .indicators import mac


def track_session(ref_f, ref_shapes, f, shapes, df_max: float = 0.05, macd_max: float = 0.15):
    """match[r] = index of the session mode assigned to reference mode r, or -1."""
    pairs = []
    for r in range(len(ref_f)):
        for c in range(len(f)):
            df = abs(f[c] - ref_f[r]) / max(f[c], ref_f[r])
            dm = 1.0 - mac(shapes[c], ref_shapes[r])
            if df <= df_max and dm <= macd_max:
                pairs.append((df + dm, r, c))
    pairs.sort()
    match = -np.ones(len(ref_f), dtype=np.int64)
    used = set()
    for _, r, c in pairs:
        if match[r] < 0 and c not in used:
            match[r] = c
            used.add(c)
    return match


def success_ratio(matches):
    """matches [sessions][n_ref] (-1 = miss) -> per reference mode percentage."""
    m = np.asarray(matches)
    return 100.0 * (m >= 0).sum(axis=0) / m.shape[0]
