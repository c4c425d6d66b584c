"""Oracle: numpy's per-destination neighbour sampling, restated (pure Python ints).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.

``build_sampled`` (compgraph.py:248-284) keeps, for every destination v of
block l whose serving in-sources outnumber the fanout f, the sources at

    np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(l, v)))
        .choice(len(nbrs), size=f, replace=False)

sorted ascending.  The randomness is numpy's (pinned only as ``numpy>=1.24``,
pkg/pyproject.toml:11; this container has numpy 2.3).  Its published
algorithms, restated here because the CUDA path re-implements them per
destination thread (``k_sample_spans`` in ob_build.cu):

* ``SeedSequence`` (numpy/random/bit_generator.pyx): the entropy and spawn
  key become uint32 words (little-endian limbs, 0 -> [0]); with a spawn key
  the entropy is zero-padded to the pool size 4; a 4-word pool is filled by
  ``hashmix`` (INIT_A / MULT_A), cross-mixed, the remaining words are folded
  in with ``mix``; ``generate_state(4, uint64)`` draws 8 words with
  INIT_B / MULT_B and pairs them little-endian.
* ``PCG64`` (numpy/random/src/pcg64): 128-bit LCG, multiplier
  0x2360ED051FC65DA44385DF649FCCF645, seeded from state words (s_hi, s_lo,
  i_hi, i_lo) by ``pcg_setseq_128_srandom_r``; XSL-RR output; 32-bit draws
  split one 64-bit output low half first.
* ``Generator.choice(n, size, replace=False)`` without p: Floyd's algorithm
  (j = n-size .. n-1, t = bounded(0, j) by Lemire's 32-bit method; keep t
  unless already chosen, else j), valid when n <= 10000 or size <= n // 50
  (the tail-shuffle branch is never reached for size <= 200, the device cap).
  The final shuffle does not change the set, which is all build_sampled uses.
"""

from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF
M64 = (1 << 64) - 1
M128 = (1 << 128) - 1
INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
MIX_L, MIX_R = 0xCA01F9DD, 0x4973F715
PCG_MULT = (2549297995355413924 << 64) + 4865540595714422341
MAX_FANOUT = 200


def _words(n: int) -> list[int]:
    if n == 0:
        return [0]
    out = []
    while n > 0:
        out.append(n & M32)
        n >>= 32
    return out


def seed_state(entropy: int, spawn_key: tuple) -> list[int]:
    """SeedSequence(entropy, spawn_key).generate_state(4, np.uint64)."""
    run = _words(int(entropy))
    spawn = [w for k in spawn_key for w in _words(int(k))]
    if spawn and len(run) < 4:
        run = run + [0] * (4 - len(run))
    ent = run + spawn
    hc = [INIT_A]

    def hashmix(v):
        v ^= hc[0]
        hc[0] = (hc[0] * MULT_A) & M32
        v = (v * hc[0]) & M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (MIX_L * x - MIX_R * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    hb, out = INIT_B, []
    for i in range(8):
        v = pool[i % 4] ^ hb
        hb = (hb * MULT_B) & M32
        v = (v * hb) & M32
        out.append(v ^ (v >> 16))
    return [out[2 * i] | (out[2 * i + 1] << 32) for i in range(4)]


class Pcg64:
    """numpy's PCG64 bit generator (XSL-RR 128/64) with its 32-bit draw buffer."""

    def __init__(self, st: list[int]):
        seed = (st[0] << 64) | st[1]
        inc = (st[2] << 64) | st[3]
        self.inc = ((inc << 1) | 1) & M128
        self.state = 0
        self._step()
        self.state = (self.state + seed) & M128
        self._step()
        self.has32, self.buf32 = False, 0

    def _step(self):
        self.state = (self.state * PCG_MULT + self.inc) & M128

    def next64(self) -> int:
        self._step()
        hi, lo = self.state >> 64, self.state & M64
        rot, x = hi >> 58, hi ^ lo
        return ((x >> rot) | (x << ((64 - rot) & 63))) & M64

    def next32(self) -> int:
        if self.has32:
            self.has32 = False
            return self.buf32
        n = self.next64()
        self.has32, self.buf32 = True, n >> 32
        return n & M32

    def bounded32(self, rng: int) -> int:
        """random_bounded_uint64(0, rng) for 0 < rng < 2^32-1: Lemire's method."""
        ex = rng + 1
        m = self.next32() * ex
        left = m & M32
        if left < ex:
            thr = (M32 - rng) % ex
            while left < thr:
                m = self.next32() * ex
                left = m & M32
        return m >> 32


def choice_set(n: int, size: int, seed: int, layer: int, v: int) -> list[int]:
    """sorted(default_rng(SeedSequence(seed, (layer, v))).choice(n, size, replace=False))."""
    if size > MAX_FANOUT:
        raise ValueError("fanout above the device cap")
    g = Pcg64(seed_state(seed, (layer, v)))
    chosen: list[int] = []
    for j in range(n - size, n):
        t = g.bounded32(j) if j > 0 else 0
        chosen.append(j if t in chosen else t)
    return sorted(chosen)


def numpy_choice_set(n: int, size: int, seed: int, layer: int, v: int) -> np.ndarray:
    """The reference's own call (compgraph.py:272-273), for pinning the restatement."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(layer, int(v))))
    return np.sort(rng.choice(n, size=size, replace=False))


# ---------------------------------------------------------------------------
# RANDOM selection policy (policy.py:122-124): default_rng(tie_seed).permutation(|R|)
# ---------------------------------------------------------------------------


def random_interval(g: Pcg64, mx: int) -> int:
    """numpy's random_interval (distributions.c): masked rejection on 32-bit draws (mx < 2^32)."""
    if mx == 0:
        return 0
    mask = mx
    for s in (1, 2, 4, 8, 16):
        mask |= mask >> s
    while True:
        v = g.next32() & mask
        if v <= mx:
            return v


def permutation_prefix(m: int, budget: int, seed: int) -> list[int]:
    """default_rng(seed).permutation(m)[:budget]: numpy's Fisher-Yates shuffle of arange(m)
    (Generator.shuffle: for i = m-1 .. 1, j = random_interval(i), swap a[i], a[j])."""
    g = Pcg64(seed_state(seed, ()))
    a = list(range(m))
    for i in range(m - 1, 0, -1):
        j = random_interval(g, i)
        a[i], a[j] = a[j], a[i]
    return a[:budget]


def swap_draws(m: int, seed: int) -> list[int]:
    """j_i for i = 1 .. m-1 (index i), the draws the shuffle makes (drawn for i = m-1 first)."""
    g = Pcg64(seed_state(seed, ()))
    j = [0] * max(m, 1)
    for i in range(m - 1, 0, -1):
        j[i] = random_interval(g, i)
    return j


def permutation_prefix_traced(m: int, budget: int, seed: int) -> list[int]:
    """The same prefix without performing the swaps -- the order the CUDA path evaluates it in.

    The shuffle applies transpositions t_i = (i, j_i) for i = m-1 down to 1, so the final array
    is a[p] = t_1(t_2(... t_{m-1}(p) ...)) read right to left as "apply t_{m-1} last":
    a[p] = (t_{m-1} o ... o t_1)(p).  Tracing p forward through i = 1 .. m-1: nothing moves it
    before step p (j_i <= i < p); at step p it becomes j_p; afterwards it moves only when a
    later step draws exactly its current value x, and then to that step's index.  So a[p] is
    found by hopping to the first later step whose draw equals the current value.
    """
    j = swap_draws(m, seed)
    occ: dict[int, list[int]] = {}
    for i in range(1, m):
        occ.setdefault(j[i], []).append(i)  # ascending steps per drawn value
    out = []
    for p in range(budget):
        x, s = (j[p], p) if p > 0 else (0, 0)
        while True:
            nxt = [i for i in occ.get(x, []) if i > s]
            if not nxt:
                break
            x = s = nxt[0]
        out.append(x)
    return out
