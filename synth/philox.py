"""Counter-based Philox4x32-10 (Salmon et al., SC'11), vectorised in numpy.

Used to synthesise the C5 matrix (100000 x 200000, 160 GB)
identically on the host (here, for sampled checks) and on the device
(synth/csrc/gen.cu, for the data itself).  Element (i, j) of matrix `mat`
with seed `seed` comes from counter (i >> 1, j, mat, 0), key (seed lo, seed
hi): words (x0, x1) give row 2p, (x2, x3) row 2p+1, as the 64-bit integer
(x_hi << 32 | x_lo) >> 11 scaled by 2^-53 (a uniform in [0, 1)).
No method arithmetic lives here.
"""
from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & MASK for v in (c0, c1, c2, c3))
    k0 = np.uint64(k0) & MASK
    k1 = np.uint64(k1) & MASK
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK, lo1, (hi0 ^ c3 ^ k1) & MASK, lo0
    return c0, c1, c2, c3


def uniform_block(rows, cols, seed: int, mat: int = 0):
    """Uniforms u[i, j] for the given row / column index arrays (outer product)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    R, Cc = np.meshgrid(rows, cols, indexing="ij")
    p = (R >> 1).astype(np.uint64)
    x0, x1, x2, x3 = philox4x32_10(p, Cc.astype(np.uint64), np.uint64(mat), np.uint64(0),
                                   seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    even = (x1 << np.uint64(32)) | x0
    odd = (x3 << np.uint64(32)) | x2
    bits = np.where((R & 1) == 0, even, odd) >> np.uint64(11)
    return bits.astype(np.float64) * (2.0 ** -53)


def centered_block(rows, cols, m: int, seed: int, mat: int = 0):
    """C5 entries A_ij = (u_ij - 1/2) * sqrt(12/m) (exact subtraction, one rounded multiply)."""
    scale = np.sqrt(12.0 / m)
    return (uniform_block(rows, cols, seed, mat) - 0.5) * scale
