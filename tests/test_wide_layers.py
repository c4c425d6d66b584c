"""Layers wider than one TMEM accumulator (H > 256, e.g. the Yelp/Amazon-shaped H = 512 of
BASELINE configs[4]): the GEMM runs as <= 256-column weight slabs.  CUDA path vs the oracle."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def graph():
    from paper_2501_08547_b200 import workload

    full = workload.gen_powerlaw_graph(4000, 14.0, 2.1, 40, seed=8)
    serving, pool = workload.split_holdout(full, 0.25, seed=8)
    req = workload.make_request(pool, serving, 24, seed=9)
    return serving, req


@pytest.mark.parametrize("kind,kw", [("gcn", {}), ("sage_mean", {}), ("gat", {}), ("sage_max", {}),
                                     ("power_mean", {"p": 2.0})])
@pytest.mark.parametrize("H", [300, 512])
@pytest.mark.parametrize("strategy", ["full", "srpe"])
def test_wide_hidden(graph, kind, kw, H, strategy):
    from oracle import layers as OL
    from paper_2501_08547_b200 import graphstore, models, runtime

    serving, req = graph
    k = 3
    model = models.make_model(kind, k, serving.feature_dim, H, **kw)
    w = models.init_weights(model, 4)
    layers = [dict(kind=s.kind, in_dim=s.in_dim, out_dim=s.out_dim, p=kw.get("p", 0.0), n=0) for s in model.layers]
    pe = None
    if strategy == "srpe":
        pe = graphstore.PeStore(OL.precompute(layers, w.layers, serving.in_offsets, serving.in_neighbors,
                                              serving.features))
    eng = runtime.ServingEngine(serving, pe, model, w, runtime.ServeConfig(strategy=strategy, gamma=0.2))
    emb, _ = eng.serve(req)
    ref = OL.serve(strategy, layers, w.layers, serving.num_nodes, req.num_queries, serving.in_offsets,
                   serving.in_neighbors, serving.features, req.query_features, req.edges,
                   pe_layers=pe.layers if pe else None, gamma=0.2)
    assert emb.shape == (req.num_queries, H)
    assert OL.max_rel_err(emb, ref["emb"]) <= TOL
    eng.close()


def test_wide_precompute(graph):
    """GPU PE precompute (full-graph layers) at H = 512 vs the oracle."""
    from oracle import layers as OL
    from paper_2501_08547_b200 import graphstore, models

    serving, _ = graph
    model = models.make_model("sage_mean", 3, serving.feature_dim, 512)
    w = models.init_weights(model, 6)
    pe = graphstore.precompute_embeddings(serving, model, w)
    layers = [dict(kind=s.kind, in_dim=s.in_dim, out_dim=s.out_dim) for s in model.layers]
    ref = OL.precompute(layers, w.layers, serving.in_offsets, serving.in_neighbors, serving.features)
    for a, r in zip(pe.layers, ref):
        assert OL.max_rel_err(a, r) <= TOL
