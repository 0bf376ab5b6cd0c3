"""Gaussian sketch Ω of Eq. (14) (§2.2; Algorithm 1 line 1).

PAPER.md:227: "this work adopts a matrix with normally distributed random entries".
The generator is unstated; reading A-11 fixes a counter-based one so the
GPU and the oracle draw the same Ω:

  * Philox4x32-10 (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3"):
    round  (c0,c1,c2,c3) -> (hi(M1·c2) ^ c1 ^ k0, lo(M1·c2), hi(M0·c0) ^ c3 ^ k1, lo(M0·c0))
    with M0 = 0xD2511F53, M1 = 0xCD9E8D57; key bump k0 += 0x9E3779B9, k1 += 0xBB67AE85
    between the 10 rounds.
  * Ω is m×k column-major; element e = col·m + row; pair p = e // 2 uses
    counter = (p_lo, p_hi, stream_lo, stream_hi), key = (seed_lo, seed_hi).
  * u1 = ((w0 | w1<<32) >> 11) + 0.5)·2^-53, u2 likewise from (w2, w3), both in (0, 1).
  * Box–Muller: Ω[2p] = sqrt(−2 ln u1) cos(2π u2), Ω[2p+1] = sqrt(−2 ln u1) sin(2π u2).
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint32(0x9E3779B9)
W1 = np.uint32(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """ctr: uint32 array [..., 4]; key: uint32 array [..., 2] (broadcast). Returns the
    four output words [..., 4] as uint32."""
    ctr = np.asarray(ctr, dtype=np.uint32)
    key = np.asarray(key, dtype=np.uint32)
    c0, c1, c2, c3 = (ctr[..., j].astype(np.uint64) for j in range(4))
    k0 = np.broadcast_to(key[..., 0], ctr.shape[:-1]).astype(np.uint64)
    k1 = np.broadcast_to(key[..., 1], ctr.shape[:-1]).astype(np.uint64)
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + np.uint64(W0)) & MASK   # wraps mod 2^32
            k1 = (k1 + np.uint64(W1)) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0,
                          lo1,
                          hi0 ^ c3 ^ k1,
                          lo0)
    return np.stack([c0, c1, c2, c3], axis=-1).astype(np.uint32)


def philox_words(pairs, seed: int, stream_id: int):
    """Words for pair indices `pairs` (int array) under (seed, stream_id), reading A-11."""
    pairs = np.asarray(pairs, dtype=np.uint64)
    ctr = np.empty(pairs.shape + (4,), dtype=np.uint32)
    ctr[..., 0] = (pairs & MASK).astype(np.uint32)
    ctr[..., 1] = (pairs >> np.uint64(32)).astype(np.uint32)
    ctr[..., 2] = np.uint32(stream_id & 0xFFFFFFFF)
    ctr[..., 3] = np.uint32((stream_id >> 32) & 0xFFFFFFFF)
    key = np.array([seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF], dtype=np.uint32)
    return philox4x32_10(ctr, key)


def uniforms_from_words(w):
    """(u1, u2) in (0,1) from words [...,4] (reading A-11): 53-bit mantissas, +0.5 offset."""
    w = w.astype(np.uint64)
    a = (w[..., 0] | (w[..., 1] << np.uint64(32))) >> np.uint64(11)
    b = (w[..., 2] | (w[..., 3] << np.uint64(32))) >> np.uint64(11)
    scale = 2.0 ** -53
    return (a.astype(np.float64) + 0.5) * scale, (b.astype(np.float64) + 0.5) * scale


def gaussian_sketch(m: int, k: int, seed: int, stream_id: int) -> np.ndarray:
    """Ω ∈ R^{m×k} (column-major element order), i.i.d. N(0,1)."""
    n = m * k
    pairs = np.arange((n + 1) // 2, dtype=np.uint64)
    u1, u2 = uniforms_from_words(philox_words(pairs, seed, stream_id))
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * pairs.size)
    z[0::2] = r * np.cos(2.0 * np.pi * u2)
    z[1::2] = r * np.sin(2.0 * np.pi * u2)
    return z[:n].reshape(k, m).T.copy()     # column-major element order → [m][k]
