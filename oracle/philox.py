"""Philox4x32-10 counter-based RNG (Salmon et al., SC'11) — TEST INFRASTRUCTURE ONLY.

Written independently of the CUDA side (which has its own device
implementation); both sides implement the same published generator so that
the k-means draws (reading R16) agree without sharing code.  Pinned by the
Random123 known-answer vectors in tests/test_oracle_kmeans.py.

Uniform double from one Philox output block x = (x0, x1, x2, x3):
    u = ((x0 >> 5) * 2^26 + (x1 >> 6)) / 2^53   in [0, 1).
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """ctr: (..., 4) uint32-valued, key: (..., 2).  Returns (..., 4) uint64 holding uint32."""
    c = [np.asarray(ctr[..., i], dtype=np.uint64) & MASK for i in range(4)]
    k0 = np.asarray(key[..., 0], dtype=np.uint64) & MASK
    k1 = np.asarray(key[..., 1], dtype=np.uint64) & MASK
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return np.stack(c, axis=-1)


def uniform(seed: int, c0, c1, c2: int, c3: int = 0) -> np.ndarray:
    """u(seed; counter = (c0, c1, c2, c3)) in [0,1); c0/c1 may be arrays."""
    c0 = np.asarray(c0, dtype=np.uint64)
    c1 = np.broadcast_to(np.asarray(c1, dtype=np.uint64), c0.shape)
    ctr = np.stack([c0, c1, np.full(c0.shape, c2, np.uint64), np.full(c0.shape, c3, np.uint64)], -1)
    key = np.broadcast_to(np.array([seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF], np.uint64),
                          c0.shape + (2,))
    x = philox4x32_10(ctr, key)
    return ((x[..., 0] >> np.uint64(5)).astype(np.float64) * 67108864.0
            + (x[..., 1] >> np.uint64(6)).astype(np.float64)) / 9007199254740992.0
