"""Numpy model of the per-order Francis QR (4 shifts per sweep from the trailing 4 x 4 block, dlahqr
deflation test) with and without dlaqr3-style aggressive early deflation (window Schur form, spike
test with reordering, shifts from the undeflated window eigenvalues), on A_n of a c3 record
(tools/dump_us.py). Counts sweeps, bulge steps and AED windows; DESIGN.md quotes the n = 200 run.
    python tools/aed_model.py [n] [nw ...]"""
import numpy as np, scipy.linalg as sl, sys
from scipy.linalg import lapack
d = np.load(__import__('os').path.join(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))), 'gpurun_out', 'c3_us.npz')); U, S = d['U'], d['S']
l, i = 192, 60
def Amat(n):
    O = U[:, :n] * np.sqrt(S[:n]); Ot, Ob = O[: l*(i-1)], O[l:]
    return np.linalg.lstsq(Ot, Ob, rcond=None)[0]
ulp = np.finfo(float).eps; smin = np.finfo(float).tiny / ulp

def refl(x):
    a = x[0]; s = np.dot(x[1:], x[1:])
    if s == 0: return None
    nrm = np.sqrt(a*a + s); beta = -np.copysign(nrm, a)
    v = x.copy(); v[0] = a - beta; tau = 2.0 / np.dot(v, v)
    return v, tau

def sweep(H, lo, hi, shifts, Z=None):
    # multishift bulge from shifts (list of complex, conj pairs/real pairs); one bulge
    ns = len(shifts); m = ns + 1
    x = np.zeros(hi - lo + 1); x[0] = 1
    Hs = H[lo:hi+1, lo:hi+1]
    w = np.zeros(hi-lo+1); w[0] = 1.0
    k = 0
    while k < ns:
        a, b = shifts[k], shifts[k+1]
        t = (a + b).real; dd = (a * b).real
        w = Hs @ (Hs @ w) - t * (Hs @ w) + dd * w
        w /= np.abs(w).sum()
        k += 2
    steps = 0
    n = H.shape[0]
    for kk in range(lo - 1, hi - 1):
        nr = min(m, hi - kk)
        if kk == lo - 1: xv = w[:nr].copy()
        else: xv = H[kk+1:kk+1+nr, kk].copy()
        r = refl(xv)
        steps += 1
        if r is None: continue
        v, tau = r
        rows = slice(kk+1, kk+1+nr)
        c0 = max(kk, 0)
        H[rows, c0:] -= tau * np.outer(v, v @ H[rows, c0:])
        rmax = min(kk + 1 + nr + 1, hi + 1)
        H[:rmax, rows] -= tau * np.outer(H[:rmax, rows] @ v, v)
        if kk >= lo: H[kk+2:kk+1+nr, kk] = 0.0
    return steps

def small_tst(H, ll):
    h = abs(H[ll, ll-1])
    if h <= smin: return True
    tst = abs(H[ll-1, ll-1]) + abs(H[ll, ll])
    return h <= ulp * tst

def qr(H0, nsh=4, aed_nw=0, verbose=False):
    H = H0.copy(); n = H.shape[0]; hi = n - 1; sweeps = 0; steps = 0; its = 0
    aed_calls = 0; aed_defl = 0; aed_cost = 0
    while hi >= 0:
        lo = 0
        for ll in range(hi, 0, -1):
            if small_tst(H, ll): lo = ll; break
        if lo > 0: H[lo, lo-1] = 0
        if lo == hi: hi -= 1; its = 0; continue
        if lo == hi - 1: hi -= 2; its = 0; continue
        shifts = None
        if aed_nw and hi - lo + 1 > aed_nw + 4:
            nw = aed_nw; kt = hi - nw + 1
            s = H[kt, kt-1]
            T, V = sl.schur(H[kt:hi+1, kt:hi+1], output='real')
            aed_calls += 1; aed_cost += 2.5 * nw * nw / 2    # small-QR steps estimate
            spike = s * V[0, :].copy()
            # deflation check with reordering (LAPACK dlaqr3 style)
            ns_ = nw; ilst = 0  # undeflated count moves to top
            nd = 0
            j = nw - 1
            Tm, Vm, sp = T, V, spike
            while j >= ilst:
                bs = 2 if (j > 0 and Tm[j, j-1] != 0) else 1
                if bs == 1:
                    foo = abs(Tm[j, j]) or abs(s)
                    ok = abs(s * Vm[0, j]) <= max(smin, ulp * foo)
                else:
                    foo = abs(Tm[j, j]) + np.sqrt(abs(Tm[j, j-1])) * np.sqrt(abs(Tm[j-1, j]))
                    foo = foo or abs(s)
                    ok = max(abs(s * Vm[0, j]), abs(s * Vm[0, j-1])) <= max(smin, ulp * foo)
                if ok:
                    nd += bs; j -= bs
                else:
                    # move block j to position ilst
                    src = j - bs + 1
                    Tm, Vm, info = lapack.dtrexc(Tm, Vm, src + 1, ilst + 1)
                    ilst += bs
            if nd > 0:
                # apply V to H window and outside, set spike, restore Hessenberg of undeflated part
                W = Vm
                H[kt:hi+1, kt:] = W.T @ H[kt:hi+1, kt:]
                H[:hi+1, kt:hi+1] = H[:hi+1, kt:hi+1] @ W
                H[kt:hi+1, kt-1] = s * W[0, :]
                H[kt+nw-nd:hi+1, kt-1] = 0.0
                # restore Hessenberg on rows/cols kt-1.. kt+nw-nd-1 (undeflated part)
                nu = nw - nd
                if nu > 1:
                    blk = H[kt-1:kt+nu, kt-1:kt+nu]
                    # reduce column 0 spike + rest to Hessenberg using householder on full window-later
                    Hq, Q = sl.hessenberg(H[kt:kt+nu, kt:kt+nu] , calc_q=True)
                    # proper: need reduction of [spike T] ; approximate with orthogonal Q making spike e1
                    v = H[kt:kt+nu, kt-1].copy()
                    r = refl(v)
                    if r is not None:
                        vv, tau = r
                        P = np.eye(nu) - tau * np.outer(vv, vv)
                        H[kt:kt+nu, kt-1:] = P @ H[kt:kt+nu, kt-1:]
                        H[:hi+1, kt:kt+nu] = H[:hi+1, kt:kt+nu] @ P
                    Hh, Q = sl.hessenberg(H[kt:kt+nu, kt:kt+nu], calc_q=True)
                    H[kt:kt+nu, kt:] = Q.T @ H[kt:kt+nu, kt:]
                    H[:hi+1, kt:kt+nu] = H[:hi+1, kt:kt+nu] @ Q
                    H[kt+1:kt+nu, kt-1] = 0.0
                    H[np.tril_indices(n, -2)] = 0.0
                aed_defl += nd
                hi -= nd
                its = 0
                continue_sweep = True
            # shifts from undeflated window eigenvalues (bottom nsh)
            ev = np.linalg.eigvals(Tm[:nw-nd, :nw-nd]) if nw - nd > 0 else []
            if len(ev) >= nsh:
                # take the nsh eigenvalues at the bottom of Schur order
                evb = []
                jj = nw - nd - 1
                while len(evb) < nsh and jj >= 0:
                    if jj > 0 and Tm[jj, jj-1] != 0:
                        e = np.linalg.eigvals(Tm[jj-1:jj+1, jj-1:jj+1]); evb += list(e); jj -= 2
                    else: evb.append(Tm[jj, jj]); jj -= 1
                shifts = evb[:nsh]
            if nd > 0: continue
        its += 1
        if its in (10, 20) or hi - lo + 1 < nsh + 2 or shifts is None:
            blk = H[hi-nsh+1:hi+1, hi-nsh+1:hi+1] if hi - lo + 1 >= nsh + 2 else H[hi-1:hi+1, hi-1:hi+1]
            ev = np.linalg.eigvals(blk)
            shifts = list(ev)
        # pair shifts: conj pairs or two reals
        cs = [e for e in shifts if e.imag > 0] if np.iscomplexobj(shifts) else []
        sh = []
        re_ = sorted([e.real for e in shifts if abs(np.imag(e)) == 0])
        for e in shifts:
            if np.imag(e) > 0: sh += [e, np.conj(e)]
        for q in range(0, len(re_) - 1, 2): sh += [re_[q], re_[q+1]]
        if len(sh) == 0: sh = list(shifts[:2])
        steps += sweep(H, lo, hi, sh)
        sweeps += 1
    return sweeps, steps, aed_calls, aed_defl, aed_cost

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
A = Amat(n)
H = sl.hessenberg(A)
ev_ref = np.sort_complex(np.linalg.eigvals(A))
for nw in [0] + [int(x) for x in sys.argv[2:]]:
    sw, st, ac, ad, acost = qr(H, 4, nw)
    print(f"n={n} nw={nw}: sweeps {sw} steps {st} aed calls {ac} deflated {ad} small-QR steps est {acost:.0f}")
