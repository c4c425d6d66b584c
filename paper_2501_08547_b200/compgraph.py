"""Serving request and computation-block views (host side).

``ServingRequest`` mirrors ``gnnserve/compgraph.py:73-105`` including its
validation, so malformed requests fail at construction exactly as in the
reference.  ``ComputationBlock`` / ``ComputationGraph`` here are read-only
host copies of the blocks the GPU built for the last request
(``ServingEngine.last_graph()``), laid out like the reference's
(compgraph.py:33-70) for bit-exact parity checks.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

BIND_FEATURE = 0
BIND_PE = 1
BIND_COMPUTED = 2


@dataclass
class ComputationBlock:
    src_ids: np.ndarray
    dst_ids: np.ndarray
    edge_src: np.ndarray
    edge_dst: np.ndarray
    bind_kind: np.ndarray
    bind_pe_layer: np.ndarray
    src_degree: np.ndarray
    dst_self_src: np.ndarray | None = None

    @property
    def num_src(self) -> int:
        return len(self.src_ids)

    @property
    def num_dst(self) -> int:
        return len(self.dst_ids)

    @property
    def num_edges(self) -> int:
        return len(self.edge_src)

    def in_edge_counts(self) -> np.ndarray:
        return np.bincount(self.edge_dst, minlength=self.num_dst)


@dataclass
class ComputationGraph:
    blocks: list
    query_ids: np.ndarray
    strategy: str
    num_base: int
    targets: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))

    @property
    def k(self) -> int:
        return len(self.blocks)


@dataclass
class ServingRequest:
    """Query nodes, their features and query<->graph edges (compgraph.py:73-105)."""

    num_base: int
    num_queries: int
    query_features: np.ndarray
    edges: np.ndarray

    def __post_init__(self):
        self.query_features = np.ascontiguousarray(self.query_features, dtype=np.float32)
        # int64 like the reference; int32 pairs are kept as given (the engine ships them as
        # 8 bytes per edge and widens on the device)
        e = np.asarray(self.edges)
        self.edges = np.ascontiguousarray(e.reshape(-1, 2) if e.dtype == np.int32 else e.astype(np.int64).reshape(-1, 2))
        if not np.all(np.isfinite(self.query_features)):
            raise ValueError("query features must be finite")
        hi = self.num_base + self.num_queries
        if self.edges.size:
            if self.edges.min() < 0 or self.edges.max() >= hi:
                raise ValueError("request edge endpoint out of range")
            if not np.all((self.edges >= self.num_base).any(axis=1)):
                raise ValueError("every request edge needs a query endpoint")

    @property
    def query_ids(self) -> np.ndarray:
        return np.arange(self.num_base, self.num_base + self.num_queries, dtype=np.int64)

    def query_in_degrees(self) -> np.ndarray:
        if not self.edges.size:
            return np.zeros(self.num_queries, dtype=np.int64)
        d = self.edges[:, 1]
        return np.bincount(d[d >= self.num_base] - self.num_base, minlength=self.num_queries).astype(np.int64)


def query_owner(query_ids, num_base: int, num_partitions: int) -> np.ndarray:
    """Round-robin query placement (compgraph.py:362-364)."""
    return ((np.asarray(query_ids, dtype=np.int64) - num_base) % num_partitions).astype(np.int64)


# request directory (compgraph.py:467-500): header, query_features.bin (f32), query_edges.bin (u64 pairs)


def save_request(request: ServingRequest, path: str, k: int) -> None:
    os.makedirs(path, exist_ok=True)
    with open(os.path.join(path, "header"), "w") as f:
        f.write(f"B={request.num_queries}\nF={request.query_features.shape[1]}\nk={k}\n")
    request.query_features.astype("<f4").tofile(os.path.join(path, "query_features.bin"))
    request.edges.astype("<u8").tofile(os.path.join(path, "query_edges.bin"))


def load_request(path: str, num_base: int) -> tuple[ServingRequest, int]:
    with open(os.path.join(path, "header")) as f:
        h = {k: int(v) for k, v in (line.strip().split("=", 1) for line in f if line.strip())}
    q = np.fromfile(os.path.join(path, "query_features.bin"), dtype="<f4").reshape(h["B"], h["F"])
    e = np.fromfile(os.path.join(path, "query_edges.bin"), dtype="<u8").astype(np.int64).reshape(-1, 2)
    return ServingRequest(num_base, h["B"], q, e), h["k"]
