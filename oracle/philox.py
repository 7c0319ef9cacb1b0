"""Philox4x32-10 counter-based generator and the Gaussian start blocks.

ORACLE / TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:406 (Sec. 4): start vectors are drawn with cuRAND from "a random
Poisson distribution with zero mean and deviation of 1"; a Poisson law cannot
have zero mean, so we read it as the standard normal N(0,1) of Halko et al.
[11] (reading R9).  The generator is Philox4x32-10
(Salmon et al., Random123; the cuRAND Philox round function):

  round:  (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2
          c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
  key bump between rounds: k0 += W0, k1 += W1 (mod 2^32); 10 rounds.

Element (i, j) of a q x w block, draw t, seed s:
  key = (lo32(s), hi32(s));  e = i + j*q;  ctr = (lo32(e), hi32(e), lo32(t), hi32(t))
  a = ((x1<<32)|x0) >> 11 ; c = ((x3<<32)|x2) >> 11
  u1 = (a+1) 2^-53 in (0,1] ; u2 = c 2^-53 in [0,1)
  z = sqrt(-2 ln u1) cos(2 pi u2)          (Box-Muller, first output only)
The index is global and column-major, so a block is independent of any row
partition of it.
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """Vectorised Philox4x32-10.  ctr: 4 uint32-valued arrays (broadcastable),
    key: 2 python ints or arrays.  Returns 4 uint64 arrays holding uint32."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & MASK for c in ctr)
    k0 = np.asarray(key[0], dtype=np.uint64) & MASK
    k1 = np.asarray(key[1], dtype=np.uint64) & MASK
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + np.uint64(W0)) & MASK
            k1 = (k1 + np.uint64(W1)) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def gaussian_from_words(x0, x1, x2, x3):
    """Box-Muller on the two 53-bit uniforms built from one Philox output."""
    a = ((x1 << np.uint64(32)) | x0) >> np.uint64(11)
    c = ((x3 << np.uint64(32)) | x2) >> np.uint64(11)
    u1 = (a.astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = c.astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def gaussian_block(q: int, w: int, seed: int, draw: int = 0,
                   row0: int = 0, q_total: int | None = None) -> np.ndarray:
    """G(q, w, draw): rows row0..row0+q-1 of the q_total x w Gaussian block,
    returned row-major (q x w) float64."""
    if q_total is None:
        q_total = q
    i = np.arange(row0, row0 + q, dtype=np.uint64)[:, None]
    j = np.arange(w, dtype=np.uint64)[None, :]
    e = i + j * np.uint64(q_total)
    t = np.uint64(draw)
    key = (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    x = philox4x32_10((e & MASK, e >> np.uint64(32), t & MASK, t >> np.uint64(32)), key)
    return gaussian_from_words(*x)
