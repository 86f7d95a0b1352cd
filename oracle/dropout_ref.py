"""CPU restatement of the attention-dropout keep mask -- TEST INFRASTRUCTURE ONLY.

Philox4x32-10 (Salmon, Moraes, Dror, Shaw: "Parallel random numbers: as easy as 1, 2, 3",
SC'11 -- the Random123 round function and Weyl key schedule), in numpy uint32 arithmetic,
pinned by the Random123 known-answer vectors in tests/test_oracle.py.  The reference
repository has no dropout (it models activation memory only); this restates the
definition csrc/dropout.cuh implements so the runtime's dropout can be checked against the
model oracle:

  element (query i, key j) of sample bg, head hg:
    counter = (j // 4, i, bg * H_total + hg, offset), key = (seed & 0xffffffff, seed >> 32)
    u = philox4x32_10(counter, key)[j % 4];   kept iff u >= floor(p * 2^32)
"""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """ctr: uint32 array [..., 4]; key: (k0, k1) uint32 -> uint32 [..., 4]."""
    c = [np.asarray(ctr[..., n], dtype=np.uint64) for n in range(4)]
    k0, k1 = np.uint32(key[0]), np.uint32(key[1])
    for r in range(10):
        if r:
            k0 = np.uint32((int(k0) + int(W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(W1)) & 0xFFFFFFFF)
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return np.stack([x.astype(np.uint32) for x in c], axis=-1)


def threshold(p: float) -> int:
    t = int(p * 4294967296.0)
    return max(1, min(t, 0xFFFFFFFF)) if p > 0 else 0


def keep_mask(B: int, S: int, H: int, p: float, seed: int, offset: int, *, b0: int = 0,
              h0: int = 0, H_total: int | None = None) -> np.ndarray:
    """bool [B, H, S, S]: True where attention probability (b, h, i, j) is kept."""
    H_total = H if H_total is None else H_total
    if p <= 0:
        return np.ones((B, H, S, S), dtype=bool)
    G = (S + 3) // 4
    b = np.arange(B, dtype=np.uint64)[:, None, None, None]
    h = np.arange(H, dtype=np.uint64)[None, :, None, None]
    i = np.arange(S, dtype=np.uint64)[None, None, :, None]
    g = np.arange(G, dtype=np.uint64)[None, None, None, :]
    bh = (b + np.uint64(b0)) * np.uint64(H_total) + np.uint64(h0) + h
    shape = (B, H, S, G)
    ctr = np.stack([np.broadcast_to(g, shape), np.broadcast_to(i, shape),
                    np.broadcast_to(bh, shape),
                    np.full(shape, offset & 0xFFFFFFFF, dtype=np.uint64)], axis=-1)
    key = (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    u = philox4x32_10(ctr.astype(np.uint32), key).reshape(B, H, S, G * 4)[..., :S]
    return u >= np.uint32(threshold(p))
