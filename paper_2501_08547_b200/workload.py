"""Synthetic graphs and serving requests (input synthesis, not the hot path).

``gen_powerlaw_graph`` / ``split_holdout`` / ``make_request`` reproduce the
reference generator (``gnnserve/workload.py:47-168``) draw for draw on the
same numpy ``default_rng`` streams, so the graphs, hold-out pools and
requests are bit-identical to the reference's for the same seeds
(``tests/test_workload.py`` pins this against golden hashes).  The only
change is speed: CSR construction sorts one combined key instead of a
two-key lexsort, and the hold-out split reuses the already-sorted CSR order.

For graphs too large for the host, the engine
generates the graph on the device from a ``graphstore.SyntheticGraph``
descriptor (``ob_generate_graph``: same degree law, Zipf-rank sampling, *not*
the numpy stream); ``make_request_synthetic`` draws query batches against such
a graph from the same law on the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .compgraph import ServingRequest
from .graphstore import GraphDataset, export_edges


@dataclass
class HoldoutPool:
    ids: np.ndarray
    removed: np.ndarray
    features: np.ndarray
    incident_edges: np.ndarray


def _degree_sequence(rng: np.random.Generator, n: int, avg: float, exponent: float, dmax: int) -> np.ndarray:
    """Power-law degrees with an exact total (workload.py:119-143), same draws."""
    target = int(round(n * avg))
    if target > n * dmax:
        raise ValueError("average degree infeasible for the degree cap")
    pmf = np.arange(1, dmax + 1, dtype=np.float64) ** (-exponent)
    cdf = np.cumsum(pmf / pmf.sum())
    raw = np.searchsorted(cdf, rng.random(n)) + 1
    deg = np.clip(np.round(raw * (avg / raw.mean())), 1, dmax).astype(np.int64)
    for _ in range(1000):
        diff = target - int(deg.sum())
        if diff == 0:
            return deg
        pick = rng.integers(0, n, size=abs(diff))
        if diff > 0:
            pick = pick[deg[pick] < dmax]
            np.add.at(deg, pick, 1)
        else:
            pick = pick[deg[pick] > 1]
            np.add.at(deg, pick, -1)
        np.clip(deg, 1, dmax, out=deg)
    raise ValueError("could not realize the requested degree sequence")


def _csr_from_edges(src: np.ndarray, dst: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray]:
    key = np.sort(dst * np.int64(n) + src)
    d = key // n
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(d, minlength=n), out=offsets[1:])
    return offsets, key - d * n


def gen_powerlaw_graph(n: int, avg_degree: float, exponent: float, feature_dim: int, seed: int) -> GraphDataset:
    """Configuration-model graph (workload.py:146-168)."""
    if n < 2:
        raise ValueError("need at least two nodes")
    if avg_degree < 1:
        raise ValueError("average degree must be >= 1")
    rng = np.random.default_rng(seed)
    out_deg = _degree_sequence(rng, n, avg_degree, exponent, n - 1)
    in_deg = _degree_sequence(rng, n, avg_degree, exponent, n - 1)
    src = np.repeat(np.arange(n, dtype=np.int64), out_deg)
    dst = np.repeat(np.arange(n, dtype=np.int64), in_deg)
    rng.shuffle(src)
    rng.shuffle(dst)
    features = rng.standard_normal((n, feature_dim)).astype(np.float32)
    perm = rng.permutation(n)
    split = int(0.8 * n)
    train = np.zeros(n, dtype=bool)
    test = np.zeros(n, dtype=bool)
    train[perm[:split]] = True
    test[perm[split:]] = True
    offsets, nbrs = _csr_from_edges(src, dst, n)
    del src, dst
    return GraphDataset(n, offsets, nbrs, features, train, test)


def split_holdout(dataset: GraphDataset, fraction: float, seed: int) -> tuple[GraphDataset, HoldoutPool]:
    """Hold out test nodes and every edge touching them (workload.py:47-75)."""
    test_ids = np.flatnonzero(dataset.test_mask)
    if not test_ids.size:
        raise ValueError("dataset has no test nodes")
    count = min(len(test_ids), max(1, int(round(fraction * len(test_ids)))))
    rng = np.random.default_rng(seed)
    held = np.sort(rng.choice(test_ids, size=count, replace=False)).astype(np.int64)
    removed = np.zeros(dataset.num_nodes, dtype=bool)
    removed[held] = True
    edges = export_edges(dataset)
    incident = removed[edges[:, 0]] | removed[edges[:, 1]]
    keep = edges[~incident]  # CSR order is (dst, src) sorted: filtering keeps it sorted
    offsets = np.zeros(dataset.num_nodes + 1, dtype=np.int64)
    np.cumsum(np.bincount(keep[:, 1], minlength=dataset.num_nodes), out=offsets[1:])
    serving = GraphDataset(dataset.num_nodes, offsets, np.ascontiguousarray(keep[:, 0]), dataset.features,
                           dataset.train_mask & ~removed, dataset.test_mask & ~removed)
    pool = HoldoutPool(held, removed, dataset.features[held], edges[incident])
    return serving, pool


def make_request(pool: HoldoutPool, serving_graph: GraphDataset, batch_size: int, seed: int,
                 include_query_query: bool = False) -> ServingRequest:
    """Re-attach a random batch of held-out nodes as queries, both directions (workload.py:78-116)."""
    if batch_size > len(pool.ids):
        raise ValueError("batch size exceeds holdout pool")
    rng = np.random.default_rng(seed)
    selected = np.sort(rng.choice(pool.ids, size=batch_size, replace=False)).astype(np.int64)
    base = serving_graph.num_nodes
    qid = np.full(base, -1, dtype=np.int64)
    qid[selected] = base + np.arange(batch_size)
    a, b = pool.incident_edges[:, 0], pool.incident_edges[:, 1]
    aq, bq = qid[a] >= 0, qid[b] >= 0
    keep = ~((pool.removed[a] & ~aq) | (pool.removed[b] & ~bq))
    if not include_query_query:
        keep &= ~(aq & bq)
    a, b = a[keep], b[keep]
    s = np.where(qid[a] >= 0, qid[a], a)
    d = np.where(qid[b] >= 0, qid[b], b)
    edges = np.concatenate([np.stack([s, d], axis=1), np.stack([d, s], axis=1)])
    return ServingRequest(base, batch_size, pool.features[np.searchsorted(pool.ids, selected)], edges)


def _zipf_norm(n: int, s: float) -> float:
    """sum_{r=1..n} r^-s in float64 (chunked), the generator's normaliser."""
    tot = 0.0
    step = 1 << 24
    for a in range(1, n + 1, step):
        r = np.arange(a, min(n, a + step - 1) + 1, dtype=np.float64)
        tot += float(np.sum(r ** -s))
    return tot


def make_request_synthetic(num_nodes: int, avg_degree: float, exponent: float, feature_dim: int,
                           batch_size: int, seed: int) -> ServingRequest:
    """A query batch against a device-generated graph (ob_generate_graph's law).

    Each query is a new node (ids N..N+B-1, like a re-attached hold-out node in
    make_request, workload.py:78-116) whose degree is drawn from the in-degree
    law and whose neighbours are drawn by popularity rank; every incident edge
    is added in both directions, as the reference does.
    """
    n = int(num_nodes)
    s = 1.0 / (exponent - 1.0)
    c1 = (n + 1.0) ** (1.0 - s) - 1.0
    E = avg_degree * n
    H = _zipf_norm(n, s)
    rng = np.random.default_rng(seed)
    # incident edges of a held-out node: one in-degree and one out-degree draw
    r = rng.integers(0, n, size=(2, batch_size)).astype(np.float64)
    deg = np.clip(np.floor(E * (r + 1.0) ** -s / H + 0.5), 1, n - 1).astype(np.int64).sum(axis=0)
    q = np.repeat(np.arange(batch_size, dtype=np.int64), deg) + n
    x = rng.random(int(deg.sum()))
    u = np.clip(np.floor((1.0 + x * c1) ** (1.0 / (1.0 - s))).astype(np.int64) - 1, 0, n - 1)
    edges = np.concatenate([np.stack([u, q], axis=1), np.stack([q, u], axis=1)])
    feats = rng.standard_normal((batch_size, feature_dim)).astype(np.float32)
    return ServingRequest(n, batch_size, feats, edges)
