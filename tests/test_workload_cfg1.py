"""Input synthesis reproduces the reference's graphs; the oracle reproduces config 1.

Config 1 (BASELINE.json configs[0]: GCN k=2, 100K nodes, F=64, B=256,
gamma=0.1) is regenerated with the package's generator and checked against
hashes of the reference's own arrays (tests/golden/cfg1.npz), then the
oracle's selection/structure/embeddings are checked against the reference's.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import load_golden
from oracle import layers as OL
from oracle import structure as OS
from paper_2501_08547_b200 import models, workload


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def cfg1():
    full = workload.gen_powerlaw_graph(100_000, 20.0, 2.1, 64, seed=1)
    serving, pool = workload.split_holdout(full, 0.25, seed=1)
    req = workload.make_request(pool, serving, 256, seed=3)
    model = models.make_model("gcn", 2, 64, 64)
    w = models.init_weights(model, 2)
    return serving, pool, req, model, w


def test_generator_bit_identical(cfg1):
    serving, pool, req, model, w = cfg1
    g = load_golden("cfg1")
    assert sha(serving.in_offsets, serving.in_neighbors, serving.features) == str(g["graph_sha"])
    assert sha(pool.ids, pool.incident_edges) == str(g["pool_sha"])
    assert sha(req.edges, req.query_features) == str(g["request_sha"])
    assert sha(w.layers[0]["w"], w.layers[1]["w"]) == str(g["weights_sha"])


def test_oracle_cfg1(cfg1):
    serving, pool, req, model, w = cfg1
    g = load_golden("cfg1")
    N = serving.num_nodes
    layers = [dict(kind="gcn", in_dim=64, out_dim=64)] * 2
    ws = w.layers
    pe = OL.precompute(layers, ws, serving.in_offsets, serving.in_neighbors, serving.features)
    assert OL.max_rel_err(pe[0][::97], g["pe_l1"]) <= 1e-5
    r = OL.serve("srpe", layers, ws, N, 256, serving.in_offsets, serving.in_neighbors, serving.features,
                 req.query_features, req.edges, pe_layers=pe, gamma=0.1)
    plan = r["plan"]
    assert len(plan["ids"]) == int(g["cand.n"])
    assert sha(plan["ids"], plan["scores"]) == str(g["cand_sha"])
    assert np.array_equal(plan["targets"], g["targets"])
    for l, b in enumerate(r["blocks"], start=1):
        fields = ("src_ids", "dst_ids", "edge_src", "edge_dst", "bind_kind", "bind_pe_layer", "src_degree",
                  "dst_self_src")
        assert sha(*[np.asarray(getattr(b, f), dtype=np.int64) for f in fields]) == str(g[f"b{l}.sha"])
    assert r["fetch_bytes"] == int(g["fetch_bytes"])
    assert OL.max_rel_err(r["emb"], g["emb"]) <= 1e-5


def test_models_init_matches_reference_layout():
    m = models.make_model("gat", 2, 5, 4)
    w = models.init_weights(m, 0)
    assert w.layers[0]["w"].shape == (5, 4) and w.layers[0]["a_src"].shape == (4,)
    assert np.all(np.abs(w.layers[0]["a_src"]) <= 0.5)
