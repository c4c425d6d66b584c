"""Drop-in boundary: the reference's own objects through the B200 engine -- needs a B200.

The reference package (``gnnserve``, installed unmodified into the git-ignored
``baseline/_ref`` by ``pip install --no-deps --target baseline/_ref``, DESIGN.md
"Reference arm") builds the dataset, stored embeddings, model, weights, config
and request exactly as a reference user would (``gnnserve/workload.py``,
``graphstore.precompute_embeddings``, ``models.make_model/init_weights``,
``runtime.ServeConfig``).  Those objects go unchanged into
``paper_2501_08547_b200.runtime.ServingEngine`` and the result is compared with
``gnnserve.runtime.ServingEngine.serve`` (runtime.py:258-358) on the same
request: targets and fetch bytes exactly, embeddings within 1e-4.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-4
REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def gn():
    if not os.path.isdir(os.path.join(REF, "gnnserve")):
        pytest.skip("reference not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import gnnserve.compgraph
    import gnnserve.graphstore
    import gnnserve.models
    import gnnserve.runtime
    import gnnserve.workload

    return gnnserve


@pytest.fixture(scope="module")
def workload(gn):
    """A config-1-shaped workload (smaller graph so the reference's generator stays quick)."""
    W, G = gn.workload, gn.graphstore
    full = W.gen_powerlaw_graph(20_000, 20.0, 2.1, 32, seed=1)
    serving, pool = W.split_holdout(full, 0.25, seed=1)
    reqs = [W.make_request(pool, serving, 64, seed=3 + i) for i in range(2)]
    return serving, reqs


def _rel(a, r):
    from oracle.layers import max_rel_err

    return max_rel_err(a, r)


@pytest.mark.parametrize("kind,k", [("gcn", 2), ("sage_mean", 3), ("gat", 3)])
@pytest.mark.parametrize("strategy,gamma", [("srpe", 0.1), ("srpe", 0.5), ("full", 0.0)])
def test_reference_objects_unchanged(gn, workload, kind, k, strategy, gamma):
    from paper_2501_08547_b200 import runtime as ours

    serving, reqs = workload
    M, G, R = gn.models, gn.graphstore, gn.runtime
    model = M.make_model(kind, k, serving.feature_dim, 16)
    w = M.init_weights(model, 2)
    pe = G.precompute_embeddings(serving, model, w) if strategy == "srpe" else None
    cfg = R.ServeConfig(strategy=strategy, gamma=gamma)  # the reference's config class
    ref = R.ServingEngine(serving, pe, model, w, cfg)
    eng = ours.ServingEngine(serving, pe, model, w, cfg)
    try:
        for req in reqs:  # gnnserve.compgraph.ServingRequest objects
            assert type(req).__module__ == "gnnserve.compgraph"
            r_emb, r_bd = ref.serve(req)
            emb, bd = eng.serve(req)
            assert emb.shape == r_emb.shape and emb.dtype == np.float32
            assert _rel(emb, r_emb) <= TOL
            assert bd.fetch_bytes == r_bd.fetch_bytes
            if strategy == "srpe":
                plan = ref._centralized_plan(req)
                assert np.array_equal(eng.last_plan()["targets"], plan.targets)
    finally:
        eng.close()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_reference_objects_cgp(gn, workload, P):
    """srpe-cgp with P partitions (single-process emulation) against the reference's simulated ranks."""
    from paper_2501_08547_b200 import runtime as ours

    serving, reqs = workload
    M, G, R = gn.models, gn.graphstore, gn.runtime
    model = M.make_model("sage_mean", 3, serving.feature_dim, 16)
    w = M.init_weights(model, 2)
    pe = G.precompute_embeddings(serving, model, w)
    cfg = R.ServeConfig(strategy="srpe-cgp", gamma=0.1, num_partitions=P, seed=0)
    ref = R.ServingEngine(serving, pe, model, w, cfg)
    eng = ours.ServingEngine(serving, pe, model, w, cfg)
    try:
        r_emb, r_bd = ref.serve(reqs[0])
        emb, bd = eng.serve(reqs[0])
        assert _rel(emb, r_emb) <= TOL
        assert bd.fetch_bytes == r_bd.fetch_bytes
        assert np.array_equal(eng.partition_owner(), ref.pmap.owner)
    finally:
        eng.close()


def test_reference_request_errors(gn, workload):
    """The reference's request validation and the engine's agree on a bad request (ValueError)."""
    from paper_2501_08547_b200 import runtime as ours

    serving, reqs = workload
    M, G, R = gn.models, gn.graphstore, gn.runtime
    model = M.make_model("gcn", 2, serving.feature_dim, 16)
    w = M.init_weights(model, 2)
    pe = G.precompute_embeddings(serving, model, w)
    eng = ours.ServingEngine(serving, pe, model, w, R.ServeConfig(strategy="srpe", gamma=0.1))
    try:
        bad = reqs[0]
        bad = type(bad).__new__(type(bad))  # bypass the reference's own __post_init__ check
        bad.num_base, bad.num_queries = reqs[0].num_base, reqs[0].num_queries
        bad.query_features = reqs[0].query_features
        e = reqs[0].edges.copy()
        e[0] = (0, 1)  # no query endpoint
        bad.edges = e
        with pytest.raises(ValueError):
            eng.serve(bad)
        emb, _ = eng.serve(reqs[0])  # the engine keeps serving after a rejected request
        assert np.all(np.isfinite(emb))
    finally:
        eng.close()
