"""Shared test setup: repo root on sys.path, the ``gpu`` marker, golden loaders."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

KINDS = [("gcn", {}), ("sage_mean", {}), ("sage_max", {}), ("power_mean", {"p": 2.0}),
         ("moments", {"n": 3}), ("gat", {})]
SMALL_CASES = ["demo", "small_s3", "small_s50", "small_s60"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libomega_b200.so")


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def golden_weights(g: dict, prefix: str, kind: str, k: int) -> list[dict]:
    from oracle.layers import WEIGHT_NAMES

    return [{n: g[f"{prefix}.l{l}.{n}"] for n in WEIGHT_NAMES[kind]} for l in range(1, k + 1)]


def golden_layers(kind: str, kw: dict, k: int, F: int, H: int = 6) -> list[dict]:
    return [dict(kind=kind, in_dim=F if l == 0 else H, out_dim=H, p=kw.get("p", 0.0), n=kw.get("n", 0))
            for l in range(k)]


BLOCK_FIELDS = ("src_ids", "dst_ids", "edge_src", "edge_dst", "bind_kind", "bind_pe_layer", "src_degree",
                "dst_self_src")


def assert_block_equal(got, g: dict, prefix: str, fields=BLOCK_FIELDS):
    for f in fields:
        key = f"{prefix}.{f}"
        v = getattr(got, f)
        if key not in g:
            assert v is None or f == "dst_self_src", key
            continue
        exp = g[key]
        assert v is not None, key
        assert np.array_equal(np.asarray(v).astype(np.int64), exp.astype(np.int64)), key


@pytest.fixture(scope="session")
def goldens() -> dict:
    return {n: load_golden(n) for n in SMALL_CASES}
