"""Deterministic hub-heavy test graph (pure numpy, no reference import).

Used by ``make_golden.py`` (which feeds its edge list to the reference's
``make_dataset``) and by the tests (which rebuild the same CSR without the
reference).  Destinations 0..3 have in-degrees 70,000 / 40,000 / 300 / 129,
so the importance score's row sums cover every branch of numpy's pairwise
summation (< 8, <= 128, recursive halves, and rows past 32,768 terms); the
sources' own in-degrees vary so the summation order is visible in the bits.
"""

from __future__ import annotations

import numpy as np

N = 80_000
HUBS = (70_000, 40_000, 300, 129, 7, 1)


def edges() -> np.ndarray:
    rng = np.random.default_rng(1234)
    parts = []
    for h, deg in enumerate(HUBS):
        src = rng.choice(np.arange(len(HUBS), N), size=deg, replace=False)
        parts.append(np.stack([src, np.full(deg, h)], axis=1))
    # background: every non-hub node gets 0..12 in-edges from random nodes
    dst_deg = rng.integers(0, 13, size=N - len(HUBS))
    dst = np.repeat(np.arange(len(HUBS), N), dst_deg)
    src = rng.integers(0, N, size=dst.size)
    parts.append(np.stack([src, dst], axis=1))
    return np.concatenate(parts).astype(np.int64)


def csr() -> tuple[np.ndarray, np.ndarray]:
    """Same CSR as the reference's build_csr (graphstore.py:69-88): by dst, sources ascending."""
    e = edges()
    order = np.lexsort((e[:, 0], e[:, 1]))
    counts = np.bincount(e[order, 1], minlength=N)
    off = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return off, e[order, 0].copy()


def features(F: int = 4) -> np.ndarray:
    return np.random.default_rng(99).standard_normal((N, F)).astype(np.float32)


def request(B: int = 4, F: int = 4) -> tuple[np.ndarray, np.ndarray]:
    """Query q attaches to hub q (both directions) and to 40 random training nodes."""
    rng = np.random.default_rng(77)
    pairs = []
    for q in range(B):
        ts = [q % len(HUBS)] + list(rng.choice(N, size=40, replace=False))
        for t in ts:
            pairs.append((N + q, int(t)))
            pairs.append((int(t), N + q))
    return np.array(pairs, dtype=np.int64), rng.standard_normal((B, F)).astype(np.float32)
