"""Graph dataset, stored-embedding store and dataset-directory IO (host side).

Mirrors the reference's data-plane types (``gnnserve/graphstore.py``) so a
``gnnserve`` user can switch imports: ``GraphDataset`` (in-CSR, sources
ascending per destination, duplicates kept), ``build_csr`` /
``make_dataset``, ``PeStore`` and the on-disk format.  These are load-time
containers; the serving engine copies them into HBM once
(``ServingEngine.__init__``) and never touches them per request.

``precompute_embeddings`` runs on the GPU (``ob_precompute_pe``), replacing
the reference's float64 CPU pass (graphstore.py:330-365), which is infeasible
beyond desk-scale graphs.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


@dataclass
class GraphDataset:
    """Whole-graph view (graphstore.py:40-66)."""

    num_nodes: int
    in_offsets: np.ndarray
    in_neighbors: np.ndarray
    features: np.ndarray
    train_mask: np.ndarray
    test_mask: np.ndarray

    @property
    def feature_dim(self) -> int:
        return int(self.features.shape[1])

    @property
    def num_edges(self) -> int:
        return int(self.in_neighbors.shape[0])

    def in_degrees(self) -> np.ndarray:
        return np.diff(self.in_offsets)

    def out_degrees(self) -> np.ndarray:
        return np.bincount(self.in_neighbors, minlength=self.num_nodes).astype(np.int64)

    def in_neighbors_of(self, v: int) -> np.ndarray:
        return self.in_neighbors[self.in_offsets[v]:self.in_offsets[v + 1]]


def build_csr(edges, num_nodes: int) -> tuple[np.ndarray, np.ndarray]:
    """Group (src, dst) by destination, sources ascending; duplicates kept (graphstore.py:69-88).

    Sorting one combined key ``dst * N + src`` is equivalent to the
    reference's two-key lexsort (equal keys are identical pairs) and is much
    faster on large graphs.
    """
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if edges.size and (edges.min() < 0 or edges.max() >= num_nodes):
        raise ValueError("edge endpoint out of range")
    key = np.sort(edges[:, 1] * np.int64(num_nodes) + edges[:, 0]) if edges.size else np.empty(0, np.int64)
    dst = key // num_nodes
    src = key - dst * num_nodes
    offsets = np.zeros(num_nodes + 1, dtype=np.int64)
    np.cumsum(np.bincount(dst, minlength=num_nodes), out=offsets[1:])
    return offsets, src


def make_dataset(edges, num_nodes: int, features, train_mask=None, test_mask=None) -> GraphDataset:
    """graphstore.py:91-112."""
    offsets, neighbors = build_csr(edges, num_nodes)
    features = np.asarray(features, dtype=np.float32)
    if features.shape[0] != num_nodes:
        raise ValueError("feature row count must equal num_nodes")
    if train_mask is None:
        train_mask = np.ones(num_nodes, dtype=bool)
    if test_mask is None:
        test_mask = np.zeros(num_nodes, dtype=bool)
    return GraphDataset(num_nodes, offsets, neighbors, features,
                        np.asarray(train_mask, dtype=bool), np.asarray(test_mask, dtype=bool))


def export_edges(dataset: GraphDataset) -> np.ndarray:
    """(src, dst) rows in CSR order (graphstore.py:115-119)."""
    dst = np.repeat(np.arange(dataset.num_nodes, dtype=np.int64), dataset.in_degrees())
    return np.stack([dataset.in_neighbors, dst], axis=1)


@dataclass
class SyntheticGraph:
    """A power-law graph generated on the device.

    Same degree law as ``workload.gen_powerlaw_graph`` (workload.py:119-168) but
    drawn by ``ob_generate_graph`` on the GPU, so papers-scale graphs never exist
    on the host; it is *not* the reference's numpy stream.  Under NCCL-mode CGP
    each rank generates only its own share (source-split CSR + owned rows).
    """

    num_nodes: int
    avg_degree: float
    exponent: float
    feature_dim: int
    seed: int = 1


@dataclass
class SyntheticPe:
    """N(0, 1) stored embeddings generated on the device for layers 1..k-1 (bench inputs only:
    the serving kernels are data-independent; parity uses precomputed PEs)."""

    dims: list
    seed: int = 2

    @property
    def num_layers(self) -> int:
        return len(self.dims)


class PeStore:
    """Per-layer stored embeddings for layers 1..k-1 (graphstore.py:122-171)."""

    def __init__(self, layers, node_ids=None, num_nodes=None):
        self.layers = [np.asarray(m, dtype=np.float32) for m in layers]
        self.node_ids = None if node_ids is None else np.asarray(node_ids, dtype=np.int64)
        self._pos = None
        if self.node_ids is not None:
            if num_nodes is None:
                raise ValueError("num_nodes required for a restricted store")
            pos = np.full(num_nodes, -1, dtype=np.int64)
            pos[self.node_ids] = np.arange(len(self.node_ids))
            self._pos = pos

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    def dim(self, layer: int) -> int:
        return int(self.layers[layer - 1].shape[1])

    def rows(self, layer: int, ids) -> np.ndarray:
        if layer < 1 or layer > self.num_layers:
            raise ValueError(f"no stored embeddings for layer {layer}")
        ids = np.asarray(ids, dtype=np.int64)
        if self._pos is None:
            return self.layers[layer - 1][ids]
        r = self._pos[ids]
        if r.size and r.min() < 0:
            raise KeyError(f"embedding rows not stored locally: {ids[r < 0][:5].tolist()}")
        return self.layers[layer - 1][r]

    def row(self, layer: int, node: int) -> np.ndarray:
        return self.rows(layer, np.asarray([node]))[0]

    def restrict(self, node_ids, num_nodes: int) -> "PeStore":
        node_ids = np.asarray(node_ids, dtype=np.int64)
        return PeStore([m[node_ids] for m in self.layers], node_ids=node_ids, num_nodes=num_nodes)


def precompute_embeddings(dataset: GraphDataset, model, weights, device: int = 0) -> PeStore:
    """Stored layer embeddings 1..k-1 computed on the GPU (graphstore.py:330-365)."""
    from .runtime import ServeConfig, ServingEngine

    if model.k < 2:
        raise ValueError("stored embeddings need a model with k >= 2 layers")
    eng = ServingEngine(dataset, None, model, weights, ServeConfig(strategy="full", device=device))
    try:
        eng.precompute_pe()
        return PeStore([eng.read_pe(l) for l in range(1, model.k)])
    finally:
        eng.close()


# ---------------------------------------------------------------------------
# dataset directory (graphstore.py:368-446): meta, offsets.bin, neighbors.bin
# (u64), features.bin (f32), train/test_mask.bin (u8), pe_l{l}.bin (f32)
# ---------------------------------------------------------------------------


def save_dataset(dataset: GraphDataset, path: str, pe: PeStore | None = None) -> None:
    os.makedirs(path, exist_ok=True)
    hidden = [] if pe is None else [pe.dim(l) for l in range(1, pe.num_layers + 1)]
    meta = dict(num_nodes=dataset.num_nodes, num_edges=dataset.num_edges, feature_dim=dataset.feature_dim,
                num_layers_pe=0 if pe is None else pe.num_layers, hidden_dims=",".join(map(str, hidden)))
    with open(os.path.join(path, "meta"), "w") as f:
        f.writelines(f"{k}={v}\n" for k, v in meta.items())
    dataset.in_offsets.astype("<u8").tofile(os.path.join(path, "offsets.bin"))
    dataset.in_neighbors.astype("<u8").tofile(os.path.join(path, "neighbors.bin"))
    dataset.features.astype("<f4").tofile(os.path.join(path, "features.bin"))
    dataset.train_mask.astype(np.uint8).tofile(os.path.join(path, "train_mask.bin"))
    dataset.test_mask.astype(np.uint8).tofile(os.path.join(path, "test_mask.bin"))
    if pe is not None:
        if pe.node_ids is not None:
            raise ValueError("only whole-graph stores are saved to dataset dirs")
        for l in range(1, pe.num_layers + 1):
            pe.layers[l - 1].astype("<f4").tofile(os.path.join(path, f"pe_l{l}.bin"))


def read_meta(path: str) -> dict:
    with open(os.path.join(path, "meta")) as f:
        return dict(line.strip().split("=", 1) for line in f if line.strip())


def load_dataset(path: str) -> tuple[GraphDataset, PeStore | None]:
    meta = read_meta(path)
    n, m, fdim = int(meta["num_nodes"]), int(meta["num_edges"]), int(meta["feature_dim"])
    off = np.fromfile(os.path.join(path, "offsets.bin"), dtype="<u8").astype(np.int64)
    nb = np.fromfile(os.path.join(path, "neighbors.bin"), dtype="<u8").astype(np.int64)
    if off.shape[0] != n + 1 or nb.shape[0] != m:
        raise ValueError("dataset files inconsistent with meta")
    feats = np.fromfile(os.path.join(path, "features.bin"), dtype="<f4").reshape(n, fdim)
    tr = np.fromfile(os.path.join(path, "train_mask.bin"), dtype=np.uint8).astype(bool)
    te = np.fromfile(os.path.join(path, "test_mask.bin"), dtype=np.uint8).astype(bool)
    ds = GraphDataset(n, off, nb, feats, tr, te)
    npe = int(meta.get("num_layers_pe", "0"))
    pe = None
    if npe:
        dims = [int(x) for x in meta["hidden_dims"].split(",") if x]
        pe = PeStore([np.fromfile(os.path.join(path, f"pe_l{l}.bin"), dtype="<f4").reshape(n, dims[l - 1])
                      for l in range(1, npe + 1)])
    return ds, pe
