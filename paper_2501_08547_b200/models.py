"""Model specification and weights (host side), mirroring ``gnnserve/models.py``.

Layer semantics run on the GPU (``csrc/ob_layers.cu``); this module holds
the types the serving API takes -- ``LayerSpec``, ``ModelSpec``,
``Weights`` -- plus the reference's seeded initialiser and ``weights.bin``
format, so models move between the two implementations unchanged.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np

GCN = "gcn"
SAGE_MEAN = "sage_mean"
SAGE_MAX = "sage_max"
GAT = "gat"
POWER_MEAN = "power_mean"
MOMENTS = "moments"

KIND_TAGS = {GCN: 0, SAGE_MEAN: 1, GAT: 2, POWER_MEAN: 3, MOMENTS: 4, SAGE_MAX: 5}  # models.py:36
_TAG_KINDS = {v: k for k, v in KIND_TAGS.items()}
MERGE_OF_KIND = {GCN: "sum", SAGE_MEAN: "mean", SAGE_MAX: "max", POWER_MEAN: "powmean",
                 MOMENTS: "moments", GAT: "softmax"}


@dataclass
class LayerSpec:
    """models.py:49-70."""

    kind: str
    in_dim: int
    out_dim: int
    p: float = 0.0
    n: int = 0
    num_heads: int = 1

    def __post_init__(self):
        if self.kind not in KIND_TAGS:
            raise ValueError(f"unknown layer kind {self.kind!r}")
        if self.kind == POWER_MEAN and self.p == 0.0:
            raise ValueError("power_mean needs p != 0")
        if self.kind == MOMENTS and self.n < 2:
            raise ValueError("moments needs n >= 2")
        if self.num_heads != 1:
            raise ValueError("only single-head attention is supported")

    @property
    def merge_kind(self) -> str:
        return MERGE_OF_KIND[self.kind]


@dataclass
class ModelSpec:
    """models.py:73-87."""

    layers: list

    def __post_init__(self):
        if not self.layers:
            raise ValueError("model needs at least one layer")
        for a, b in zip(self.layers, self.layers[1:]):
            if a.out_dim != b.in_dim:
                raise ValueError("adjacent layer dimensions do not chain")

    @property
    def k(self) -> int:
        return len(self.layers)


def make_model(kind: str, k: int, in_dim: int, hidden: int, p: float = 2.0, n: int = 2) -> ModelSpec:
    """Uniform-width model of one kind (models.py:90-104)."""
    return ModelSpec([
        LayerSpec(kind, in_dim if l == 0 else hidden, hidden,
                  p=p if kind == POWER_MEAN else 0.0, n=n if kind == MOMENTS else 0)
        for l in range(k)
    ])


@dataclass
class Weights:
    layers: list = field(default_factory=list)


def weight_matrix_names(kind: str) -> list[str]:
    """Matrix order per kind (models.py:111-118); also the C ABI's mats order."""
    if kind == GCN:
        return ["w"]
    if kind in (SAGE_MEAN, SAGE_MAX):
        return ["w_self", "w_neigh"]
    if kind == GAT:
        return ["w", "a_src", "a_dst"]
    return ["w_self", "w"]


def init_weights(model: ModelSpec, seed: int) -> Weights:
    """uniform(+-1/sqrt(in_dim)) per matrix in declaration order (models.py:121-133, densemath.py:64-68)."""
    rng = np.random.default_rng(seed)
    out = Weights()
    for spec in model.layers:
        bound = 1.0 / math.sqrt(spec.in_dim)
        mats = {}
        for name in weight_matrix_names(spec.kind):
            shape = (spec.out_dim,) if name in ("a_src", "a_dst") else (spec.in_dim, spec.out_dim)
            # a_src / a_dst use rows = out_dim in the reference's init_uniform
            b = 1.0 / math.sqrt(spec.out_dim) if name in ("a_src", "a_dst") else bound
            mats[name] = rng.uniform(-b, b, size=shape).astype(np.float32)
        out.layers.append(mats)
    return out


def save_weights(model: ModelSpec, weights: Weights, path: str) -> None:
    """weights.bin (models.py:303-318)."""
    with open(path, "wb") as f:
        f.write(struct.pack("<I", model.k))
        for spec in model.layers:
            param = spec.p if spec.kind == POWER_MEAN else float(spec.n)
            f.write(struct.pack("<IIIf", KIND_TAGS[spec.kind], spec.in_dim, spec.out_dim, param))
        for spec, mats in zip(model.layers, weights.layers):
            for name in weight_matrix_names(spec.kind):
                f.write(np.asarray(mats[name], dtype="<f4").tobytes())


def load_weights(path: str) -> tuple[ModelSpec, Weights]:
    """models.py:321-351."""
    with open(path, "rb") as f:
        (k,) = struct.unpack("<I", f.read(4))
        specs = []
        for _ in range(k):
            tag, i, o, param = struct.unpack("<IIIf", f.read(16))
            kind = _TAG_KINDS[tag]
            specs.append(LayerSpec(kind, i, o, p=param if kind == POWER_MEAN else 0.0,
                                   n=int(param) if kind == MOMENTS else 0))
        model = ModelSpec(specs)
        w = Weights()
        for spec in specs:
            mats = {}
            for name in weight_matrix_names(spec.kind):
                shape = (spec.out_dim,) if name in ("a_src", "a_dst") else (spec.in_dim, spec.out_dim)
                cnt = int(np.prod(shape))
                mats[name] = np.frombuffer(f.read(4 * cnt), dtype="<f4").reshape(shape).copy()
            w.layers.append(mats)
    return model, w
