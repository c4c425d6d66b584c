"""Oracle: SRPE selection, computation-graph builders, partitioning (numpy).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Every function
restates one reference routine; the citation is in its docstring
(paths relative to ``/root/reference/pkg/src/gnnserve``).

Conventions shared with the CUDA path:

* ids are int64; queries are numbered ``num_base .. num_base+B-1`` and
  therefore sort after every training id, so "training ids ascending, then
  query ids ascending" (compgraph.py:174-177) is plain ascending order.
* a block's edges are ordered by (dst local index, src local index)
  (compgraph.py:197-201).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BIND_FEATURE = 0  # compgraph.py:28-30
BIND_PE = 1
BIND_COMPUTED = 2

_I64 = np.int64


@dataclass
class Block:
    """One layer's computation block (compgraph.py:33-57)."""

    src_ids: np.ndarray
    dst_ids: np.ndarray
    edge_src: np.ndarray
    edge_dst: np.ndarray
    bind_kind: np.ndarray
    bind_pe_layer: np.ndarray
    src_degree: np.ndarray
    dst_self_src: np.ndarray | None

    @property
    def num_edges(self) -> int:
        return int(self.edge_src.shape[0])

    def dst_ptr(self) -> np.ndarray:
        ptr = np.zeros(len(self.dst_ids) + 1, dtype=_I64)
        np.cumsum(np.bincount(self.edge_dst, minlength=len(self.dst_ids)), out=ptr[1:])
        return ptr


# ---------------------------------------------------------------------------
# request helpers
# ---------------------------------------------------------------------------


def query_in_degrees(edges: np.ndarray, num_base: int, num_queries: int) -> np.ndarray:
    """compgraph.py:99-105 -- request in-degree of each query."""
    d = edges[:, 1]
    return np.bincount(d[d >= num_base] - num_base, minlength=num_queries).astype(_I64)


class RequestIndex:
    """Request edges grouped by destination, sources ascending (compgraph.py:155-171)."""

    def __init__(self, edges: np.ndarray):
        edges = np.asarray(edges, dtype=_I64).reshape(-1, 2)
        order = np.lexsort((edges[:, 0], edges[:, 1]))
        self.src = edges[order, 0]
        self.dst = edges[order, 1]

    def spans(self, ids: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        lo = np.searchsorted(self.dst, ids, side="left")
        hi = np.searchsorted(self.dst, ids, side="right")
        return lo.astype(_I64), (hi - lo).astype(_I64)


def _segment_positions(starts: np.ndarray, lens: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(flat source index, owning segment) for the concatenation of segments."""
    seg = np.repeat(np.arange(len(lens), dtype=_I64), lens)
    first = np.cumsum(lens) - lens
    pos = np.arange(int(lens.sum()), dtype=_I64) - first[seg] + starts[seg]
    return pos, seg


def _concat_per_dst(parts: list[tuple[np.ndarray, np.ndarray, np.ndarray]], num_dst: int):
    """Per destination, concatenate several (values, starts, lens) segment lists in order.

    Returns (flat values, per-destination counts).
    """
    total = np.zeros(num_dst, dtype=_I64)
    for _, _, lens in parts:
        total += lens
    ptr = np.zeros(num_dst + 1, dtype=_I64)
    np.cumsum(total, out=ptr[1:])
    flat = np.empty(int(ptr[-1]), dtype=_I64)
    shift = ptr[:-1].copy()
    for values, starts, lens in parts:
        pos, seg = _segment_positions(starts, lens)
        local = np.arange(len(pos), dtype=_I64) - (np.cumsum(lens) - lens)[seg]
        flat[shift[seg] + local] = values[pos]
        shift += lens
    return flat, total


def _src_degree(ids: np.ndarray, num_base: int, train_deg: np.ndarray, q_deg: np.ndarray) -> np.ndarray:
    """DegreeView.source_degree (compgraph.py:145-152)."""
    out = np.zeros(len(ids), dtype=_I64)
    q = ids >= num_base
    out[q] = q_deg[ids[q] - num_base]
    out[~q] = train_deg[ids[~q]]
    return out


def _reuse_binding(src_ids: np.ndarray, num_base: int, targets: np.ndarray, layer: int):
    """_reuse_bind_fn (compgraph.py:287-305)."""
    n = len(src_ids)
    if layer == 1:
        return np.zeros(n, dtype=np.uint8), np.zeros(n, dtype=np.int32)
    fresh = (src_ids >= num_base) | np.isin(src_ids, targets)
    kind = np.where(fresh, BIND_COMPUTED, BIND_PE).astype(np.uint8)
    pe_layer = np.where(fresh, 0, layer - 1).astype(np.int32)
    return kind, pe_layer


def _uniform_binding(src_ids: np.ndarray, layer: int):
    """build_full_k_hop's bind_fn (compgraph.py:234-241)."""
    n = len(src_ids)
    kind = BIND_COMPUTED if layer > 1 else BIND_FEATURE
    return np.full(n, kind, dtype=np.uint8), np.zeros(n, dtype=np.int32)


def _assemble(dst_ids, flat, counts, num_base, binding, train_deg, q_deg, include_self=True) -> Block:
    """_make_block (compgraph.py:180-213): dedup/relabel, (dst, src) edge order."""
    dst_ids = np.asarray(dst_ids, dtype=_I64)
    pool = np.concatenate([dst_ids, flat]) if include_self else flat
    src_ids = np.unique(pool).astype(_I64)
    edge_src = np.searchsorted(src_ids, flat).astype(_I64)
    edge_dst = np.repeat(np.arange(len(dst_ids), dtype=_I64), counts)
    order = np.lexsort((edge_src, edge_dst))
    kind, pe_layer = binding(src_ids)
    return Block(
        src_ids=src_ids,
        dst_ids=dst_ids,
        edge_src=edge_src[order],
        edge_dst=edge_dst[order],
        bind_kind=kind,
        bind_pe_layer=pe_layer,
        src_degree=_src_degree(src_ids, num_base, train_deg, q_deg),
        dst_self_src=np.searchsorted(src_ids, dst_ids).astype(_I64) if include_self else None,
    )


def _serving_sources(dst_ids, num_base, offsets, nbrs, ridx: RequestIndex):
    """_serving_in_sources for a list of destinations (compgraph.py:216-221).

    Training v: CSR in-neighbours of v followed by request sources into v;
    query v: request sources only.
    """
    dst_ids = np.asarray(dst_ids, dtype=_I64)
    train = dst_ids < num_base
    c_start = np.zeros(len(dst_ids), dtype=_I64)
    c_len = np.zeros(len(dst_ids), dtype=_I64)
    c_start[train] = offsets[dst_ids[train]]
    c_len[train] = offsets[dst_ids[train] + 1] - offsets[dst_ids[train]]
    r_start, r_len = ridx.spans(dst_ids)
    return _concat_per_dst([(nbrs, c_start, c_len), (ridx.src, r_start, r_len)], len(dst_ids))


# ---------------------------------------------------------------------------
# SRPE selection
# ---------------------------------------------------------------------------


def candidates(edges: np.ndarray, num_base: int, train_deg: np.ndarray):
    """candidate_arrays + find_candidates (compgraph.py:108-121, policy.py:64-67).

    Returns (ids ascending, nq = #request edges into id, total = in-degree + nq).
    """
    edges = np.asarray(edges, dtype=_I64).reshape(-1, 2)
    s, d = edges[:, 0], edges[:, 1]
    ids = np.unique(np.concatenate([s[s < num_base], d[d < num_base]])).astype(_I64)
    into = d[d < num_base]
    nq = np.bincount(np.searchsorted(ids, into), minlength=len(ids)).astype(_I64)
    total = (train_deg[ids] + nq).astype(_I64)
    return ids, nq, total


def ratio_scores(nq: np.ndarray, total: np.ndarray) -> np.ndarray:
    """score_query_edge_ratio (policy.py:77-81): IEEE fp64 nq / total."""
    if np.any(total <= 0):
        raise ValueError("candidate with zero total degree")
    return nq.astype(np.float64) / total.astype(np.float64)


def _is_terms(srcs: np.ndarray, train_deg: np.ndarray) -> np.ndarray:
    nd = train_deg[srcs].astype(np.float64)
    return np.where(nd > 0, 1.0 / np.maximum(nd, 1.0), 0.0)


def importance_scores(ids: np.ndarray, offsets: np.ndarray, nbrs: np.ndarray, train_deg: np.ndarray) -> np.ndarray:
    """score_importance (policy.py:84-95): (1/deg v) * sum_{u in N(v)} 1/deg u, fp64.

    The row sum is numpy's pairwise ``np.sum`` over the CSR row in order (the
    exact association the CUDA path reproduces); zero-in-degree rows score 0.
    """
    out = np.zeros(len(ids), dtype=np.float64)
    deg = np.asarray(train_deg)
    for i, v in enumerate(np.asarray(ids, dtype=_I64)):
        d = float(deg[v])
        if d <= 0:
            continue
        out[i] = np.sum(_is_terms(nbrs[offsets[v]:offsets[v + 1]], deg)) / d
    return out


def importance_partial_sums(ids: np.ndarray, part_offsets: np.ndarray, part_srcs: np.ndarray,
                            train_deg: np.ndarray) -> np.ndarray:
    """importance_partial_sums (policy.py:98-107): one partition's share of each numerator."""
    out = np.zeros(len(ids), dtype=np.float64)
    for i, v in enumerate(np.asarray(ids, dtype=_I64)):
        srcs = part_srcs[part_offsets[v]:part_offsets[v + 1]]
        if srcs.size:
            out[i] = np.sum(_is_terms(srcs, train_deg))
    return out


def importance_scores_distributed(ids: np.ndarray, partials: list, train_deg: np.ndarray) -> np.ndarray:
    """select_targets_distributed's IS branch (runtime.py:168-175): partials summed in rank order."""
    sums = np.zeros(len(ids), dtype=np.float64)
    for p in partials:
        sums += p
    deg = np.asarray(train_deg)[np.asarray(ids, dtype=_I64)].astype(np.float64)
    return np.where(deg > 0, sums / np.maximum(deg, 1.0), 0.0)


def select_random(ids: np.ndarray, gamma: float, seed: int) -> np.ndarray:
    """select_targets with policy RANDOM (policy.py:118-135): the first floor(gamma*|R|) of
    default_rng(seed).permutation(|R|), sorted; the permutation restated in oracle/sampling.py."""
    from .sampling import permutation_prefix

    if not 0.0 <= gamma <= 1.0:
        raise ValueError("gamma must lie in [0, 1]")
    budget = int(np.floor(float(gamma) * len(ids)))
    order = np.asarray(permutation_prefix(len(ids), budget, int(seed)), dtype=_I64)
    return np.sort(np.asarray(ids, dtype=_I64)[order]).astype(_I64)


def select_top(ids: np.ndarray, scores: np.ndarray, gamma: float) -> np.ndarray:
    """select_targets (policy.py:110-135): top floor(gamma*|R|), score desc, id asc."""
    if not 0.0 <= gamma <= 1.0:
        raise ValueError("gamma must lie in [0, 1]")
    budget = int(np.floor(float(gamma) * len(ids)))
    order = np.lexsort((ids, -np.asarray(scores, dtype=np.float64)))
    return np.sort(ids[order[:budget]]).astype(_I64)


# ---------------------------------------------------------------------------
# builders
# ---------------------------------------------------------------------------


def build_srpe(num_base, num_queries, offsets, nbrs, edges, targets, k, pe_layers: int) -> list[Block]:
    """build_srpe (compgraph.py:308-345); returns blocks[0..k-1]."""
    if k < 2:
        raise ValueError("reuse graphs need k >= 2")
    if pe_layers < k - 1:
        raise ValueError(f"stored embeddings missing for layers 1..{k - 1}")
    edges = np.asarray(edges, dtype=_I64).reshape(-1, 2)
    train_deg = np.diff(offsets).astype(_I64)
    targets = np.unique(np.asarray(targets, dtype=_I64))
    cand, _, _ = candidates(edges, num_base, train_deg)
    if targets.size and not np.all(np.isin(targets, cand)):
        raise ValueError("targets not candidates")
    q_deg = query_in_degrees(edges, num_base, num_queries)
    ridx = RequestIndex(edges)
    queries = np.arange(num_base, num_base + num_queries, dtype=_I64)

    blocks: list[Block] = [None] * k  # type: ignore[list-item]
    r_start, r_len = ridx.spans(queries)
    flat, cnt = _concat_per_dst([(ridx.src, r_start, r_len)], len(queries))
    blocks[k - 1] = _assemble(
        queries, flat, cnt, num_base,
        lambda s: _reuse_binding(s, num_base, targets, k), train_deg, q_deg,
    )
    mid = np.unique(np.concatenate([queries, targets]))
    flat, cnt = _serving_sources(mid, num_base, offsets, nbrs, ridx)
    for l in range(k - 1, 0, -1):
        blocks[l - 1] = _assemble(
            mid, flat, cnt, num_base,
            lambda s, _l=l: _reuse_binding(s, num_base, targets, _l), train_deg, q_deg,
        )
    return blocks


def build_sampled(num_base, num_queries, offsets, nbrs, edges, fanouts, seed) -> list[Block]:
    """build_sampled (compgraph.py:248-284): build_full_k_hop with fanout-capped source lists.

    Block l keeps at most fanouts[l-1] of each destination's serving in-sources,
    chosen by numpy's SeedSequence(seed, (l, v)) stream (oracle/sampling.py).
    """
    fanouts = [int(f) for f in fanouts]
    if any(f < 1 for f in fanouts):
        raise ValueError("fanouts must be >= 1")
    k = len(fanouts)
    edges = np.asarray(edges, dtype=_I64).reshape(-1, 2)
    train_deg = np.diff(offsets).astype(_I64)
    q_deg = query_in_degrees(edges, num_base, num_queries)
    ridx = RequestIndex(edges)
    dst = np.arange(num_base, num_base + num_queries, dtype=_I64)
    blocks: list[Block] = [None] * k  # type: ignore[list-item]
    for l in range(k, 0, -1):
        fan = fanouts[l - 1]
        flat, cnt = _serving_sources(dst, num_base, offsets, nbrs, ridx)
        ptr = np.zeros(len(dst) + 1, dtype=_I64)
        np.cumsum(cnt, out=ptr[1:])
        parts, counts = [], []
        for i, v in enumerate(dst):
            row = flat[ptr[i]:ptr[i + 1]]
            if len(row) > fan:
                rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(l, int(v))))
                row = np.sort(row[rng.choice(len(row), size=fan, replace=False)])
            parts.append(row)
            counts.append(len(row))
        flat = np.concatenate(parts) if parts else np.empty(0, dtype=_I64)
        blocks[l - 1] = _assemble(
            dst, flat, np.asarray(counts, dtype=_I64), num_base, lambda s, _l=l: _uniform_binding(s, _l),
            train_deg, q_deg,
        )
        dst = blocks[l - 1].src_ids
    return blocks


def build_full(num_base, num_queries, offsets, nbrs, edges, k) -> list[Block]:
    """build_full_k_hop (compgraph.py:224-245)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    edges = np.asarray(edges, dtype=_I64).reshape(-1, 2)
    train_deg = np.diff(offsets).astype(_I64)
    q_deg = query_in_degrees(edges, num_base, num_queries)
    ridx = RequestIndex(edges)
    dst = np.arange(num_base, num_base + num_queries, dtype=_I64)
    blocks: list[Block] = [None] * k  # type: ignore[list-item]
    for l in range(k, 0, -1):
        flat, cnt = _serving_sources(dst, num_base, offsets, nbrs, ridx)
        blocks[l - 1] = _assemble(
            dst, flat, cnt, num_base, lambda s, _l=l: _uniform_binding(s, _l), train_deg, q_deg
        )
        dst = blocks[l - 1].src_ids
    return blocks


def fetch_bytes(blocks: list[Block], num_base: int, feature_dim: int, pe_dims: list[int]) -> int:
    """graph_fetch_bytes without a cache (runtime.py:105-120)."""
    total = 0
    for b in blocks:
        total += 16 * b.num_edges
        total += 4 * feature_dim * int(np.sum((b.bind_kind == BIND_FEATURE) & (b.src_ids < num_base)))
        pe = b.bind_kind == BIND_PE
        for layer in np.unique(b.bind_pe_layer[pe]):
            total += 4 * pe_dims[int(layer) - 1] * int(np.sum(pe & (b.bind_pe_layer == layer)))
    return total


# ---------------------------------------------------------------------------
# partitioning (CGP)
# ---------------------------------------------------------------------------

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (graphstore.py:25-30), uint64 wraparound."""
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def owner_hash(num_nodes: int, num_parts: int, seed: int) -> np.ndarray:
    """partition_random_hash's owner map (graphstore.py:33-37,230)."""
    key = _mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    h = _mix64(np.arange(num_nodes, dtype=np.uint64) ^ key)
    return (h % np.uint64(num_parts)).astype(_I64)


@dataclass
class Shard:
    """One partition's store (graphstore.py:183-216)."""

    index: int
    owned: np.ndarray
    offsets: np.ndarray  # source-split CSR over every destination
    srcs: np.ndarray


def partition_graph(offsets, nbrs, num_nodes, num_parts, seed, owner=None):
    """partition_random_hash (graphstore.py:219-263): edges live at their source's owner."""
    if num_parts < 1:
        raise ValueError("num_partitions must be >= 1")
    if owner is None:
        owner = owner_hash(num_nodes, num_parts, seed)
    deg = np.diff(offsets)
    dst = np.repeat(np.arange(num_nodes, dtype=_I64), deg)
    shards = []
    for p in range(num_parts):
        keep = owner[nbrs] == p
        s, d = nbrs[keep], dst[keep]
        order = np.lexsort((s, d))
        s, d = s[order], d[order]
        off = np.zeros(num_nodes + 1, dtype=_I64)
        np.cumsum(np.bincount(d, minlength=num_nodes), out=off[1:])
        shards.append(Shard(p, np.flatnonzero(owner == p).astype(_I64), off, s.astype(_I64)))
    return owner, shards


def query_owner(ids: np.ndarray, num_base: int, num_parts: int) -> np.ndarray:
    """compgraph.py:362-364 -- round robin by query id."""
    return ((np.asarray(ids, dtype=_I64) - num_base) % num_parts).astype(_I64)


def split_request(edges, num_base, owner, num_parts):
    """partition_request (compgraph.py:367-392): each edge goes to its source's owner."""
    edges = np.asarray(edges, dtype=_I64).reshape(-1, 2)
    s = edges[:, 0]
    eo = np.where(s >= num_base, (s - num_base) % num_parts, owner[np.minimum(s, num_base - 1)])
    return [edges[eo == p] for p in range(num_parts)]


def build_partitioned_shard(
    num_base, num_queries, shard: Shard, owner, num_parts, edges_p, q_deg, train_deg, targets, k
) -> list[Block]:
    """build_partitioned (compgraph.py:395-459): local sources only, no self rows."""
    if k < 2:
        raise ValueError("reuse graphs need k >= 2")
    p = shard.index
    targets = np.unique(np.asarray(targets, dtype=_I64))
    queries = np.arange(num_base, num_base + num_queries, dtype=_I64)
    ridx = RequestIndex(edges_p)

    def check_local(src_ids):
        q = src_ids >= num_base
        if np.any((src_ids[q] - num_base) % num_parts != p):
            raise ValueError(f"query source not assigned to partition {p}")
        if np.any(owner[src_ids[~q]] != p):
            raise ValueError(f"source not owned by partition {p}")

    blocks: list[Block] = [None] * k  # type: ignore[list-item]
    r_start, r_len = ridx.spans(queries)
    flat, cnt = _concat_per_dst([(ridx.src, r_start, r_len)], num_queries)
    blk = _assemble(queries, flat, cnt, num_base,
                    lambda s: _reuse_binding(s, num_base, targets, k), train_deg, q_deg,
                    include_self=False)
    check_local(blk.src_ids)
    blocks[k - 1] = blk

    mid = np.unique(np.concatenate([queries, targets]))
    train = mid < num_base
    c_start = np.zeros(len(mid), dtype=_I64)
    c_len = np.zeros(len(mid), dtype=_I64)
    c_start[train] = shard.offsets[mid[train]]
    c_len[train] = shard.offsets[mid[train] + 1] - shard.offsets[mid[train]]
    r_start, r_len = ridx.spans(mid)
    flat, cnt = _concat_per_dst([(shard.srcs, c_start, c_len), (ridx.src, r_start, r_len)], len(mid))
    for l in range(k - 1, 0, -1):
        blk = _assemble(mid, flat, cnt, num_base,
                        lambda s, _l=l: _reuse_binding(s, num_base, targets, _l), train_deg, q_deg,
                        include_self=False)
        check_local(blk.src_ids)
        blocks[l - 1] = blk
    return blocks
