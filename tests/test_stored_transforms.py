"""Stored transforms and stored aggregates.

Stored transforms: x_v W precomputed for every training node whose layer input is static
(features at layer 1, stored embeddings above) replace the per-request GEMM over those sources;
only queries and recomputed rows are transformed per request.  Results must equal the
per-request path bit for bit (same GEMM kernel per row) and the oracle within 1e-4."""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def graph():
    from paper_2501_08547_b200 import workload

    full = workload.gen_powerlaw_graph(5000, 14.0, 2.1, 48, seed=12)
    serving, pool = workload.split_holdout(full, 0.25, seed=12)
    reqs = [workload.make_request(pool, serving, 32, seed=s) for s in (1, 2)]
    return serving, reqs


def _serve(serving, reqs, model, w, pe, strategy, no_transforms=False, no_aggregates=False):
    from paper_2501_08547_b200 import runtime

    keys = {"OB_NO_STORED_TRANSFORMS": no_transforms, "OB_NO_STORED_AGGREGATES": no_aggregates}
    old = {k: os.environ.get(k) for k in keys}
    for k, v in keys.items():
        os.environ[k] = "1" if v else "0"
    try:
        cfg = runtime.ServeConfig(strategy=strategy, gamma=0.3, fanouts=(6, 4, 3) if strategy == "sampled" else None)
        eng = runtime.ServingEngine(serving, pe, model, w, cfg)
        out = [eng.serve(r)[0] for r in reqs]
        eng.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return out


@pytest.mark.parametrize("kind", ["gat", "sage_mean", "gcn"])
@pytest.mark.parametrize("strategy", ["srpe", "full", "sampled"])
def test_stored_transforms_bitwise(graph, kind, strategy):
    from oracle import layers as OL
    from paper_2501_08547_b200 import graphstore, models

    serving, reqs = graph
    model = models.make_model(kind, 3, serving.feature_dim, 16)  # F=48 > 16: transform-first at layer 1
    w = models.init_weights(model, 3)
    layers = [dict(kind=s.kind, in_dim=s.in_dim, out_dim=s.out_dim) for s in model.layers]
    pe = graphstore.PeStore(OL.precompute(layers, w.layers, serving.in_offsets, serving.in_neighbors,
                                          serving.features)) if strategy == "srpe" else None
    a = _serve(serving, reqs, model, w, pe, strategy)  # stored transforms + stored aggregates
    b = _serve(serving, reqs, model, w, pe, strategy, no_aggregates=True)  # stored transforms only
    c = _serve(serving, reqs, model, w, pe, strategy, no_transforms=True, no_aggregates=True)
    for x, y, z in zip(a, b, c):
        assert np.array_equal(y, z)  # same GEMM per row: bitwise
        assert OL.max_rel_err(x, z) <= 1e-5  # layer-1 sums re-associated (static CSR part + request span)
    if strategy != "sampled":
        r = reqs[0]
        ref = OL.serve(strategy, layers, w.layers, serving.num_nodes, r.num_queries, serving.in_offsets,
                       serving.in_neighbors, serving.features, r.query_features, r.edges,
                       pe_layers=pe.layers if pe else None, gamma=0.3)
        assert OL.max_rel_err(a[0], ref["emb"]) <= 1e-4


def _serve_env(serving, reqs, model, w, pe, env, lanes=1):
    from paper_2501_08547_b200 import runtime

    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        eng = runtime.ServingEngine(serving, pe, model, w, runtime.ServeConfig(strategy="srpe", gamma=0.3))
        if lanes > 1:
            eng.set_lanes(lanes)
            out = [o for o, _ in eng.serve_stream(reqs, depth=4)]
        else:
            out = [eng.serve(r)[0] for r in reqs]
        eng.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return out


@pytest.mark.parametrize("kind", ["sage_mean", "gcn"])
@pytest.mark.parametrize("k,hidden", [(3, 16), (4, 16), (3, 48)])
@pytest.mark.parametrize("lanes", [1, 2])
def test_delta_aggregates(graph, kind, k, hidden, lanes):
    """Mid-block layers >= 2 of sum kinds: static CSR-part sums of the stored rows plus (h - PE) delta
    rows of the recomputed sources, against the full gather (OB_NO_DELTA_AGGREGATES=1) and the oracle."""
    from oracle import layers as OL
    from paper_2501_08547_b200 import graphstore, models

    serving, reqs = graph
    model = models.make_model(kind, k, serving.feature_dim, hidden)
    w = models.init_weights(model, 4)
    layers = [dict(kind=s.kind, in_dim=s.in_dim, out_dim=s.out_dim) for s in model.layers]
    pe = graphstore.PeStore(OL.precompute(layers, w.layers, serving.in_offsets, serving.in_neighbors,
                                          serving.features))
    a = _serve_env(serving, reqs, model, w, pe, {"OB_NO_DELTA_AGGREGATES": "0"}, lanes)
    b = _serve_env(serving, reqs, model, w, pe, {"OB_NO_DELTA_AGGREGATES": "1"}, lanes)
    for i, r in enumerate(reqs):
        assert OL.max_rel_err(a[i], b[i]) <= 1e-5
        ref = OL.serve("srpe", layers, w.layers, serving.num_nodes, r.num_queries, serving.in_offsets,
                       serving.in_neighbors, serving.features, r.query_features, r.edges, pe_layers=pe.layers,
                       gamma=0.3)
        assert OL.max_rel_err(a[i], ref["emb"]) <= 1e-4
