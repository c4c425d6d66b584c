"""Pipelined host path (ob_serve_submit / ob_serve_wait via ServingEngine.serve_stream):
every result equals the synchronous serve() of the same request, bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    from paper_2501_08547_b200 import graphstore, models, workload

    full = workload.gen_powerlaw_graph(6000, 12.0, 2.1, 24, seed=4)
    serving, pool = workload.split_holdout(full, 0.25, seed=4)
    model = models.make_model("sage_mean", 3, 24, 16)
    w = models.init_weights(model, 2)
    pe = graphstore.precompute_embeddings(serving, model, w)
    reqs = [workload.make_request(pool, serving, b, seed=s) for s, b in zip(range(9), (32, 32, 8, 64, 32, 16, 32, 1, 48))]
    return serving, model, w, pe, reqs


@pytest.mark.parametrize("strategy", ["srpe", "full"])
def test_stream_equals_serve(setup, strategy):
    from paper_2501_08547_b200 import runtime

    serving, model, w, pe, reqs = setup
    eng = runtime.ServingEngine(serving, pe, model, w, runtime.ServeConfig(strategy=strategy, gamma=0.2))
    ref = [eng.serve(r) for r in reqs]
    got = list(eng.serve_stream(reqs))
    assert len(got) == len(reqs)
    for (a, ba), (b, bb) in zip(got, ref):
        assert np.array_equal(a, b)
        assert ba.fetch_bytes == bb.fetch_bytes
    # interleaving with the synchronous path keeps working
    again = list(eng.serve_stream(reqs[:3]))
    assert all(np.array_equal(a, b[0]) for (a, _), b in zip(again, ref[:3]))
    eng.close()


def test_stream_error_is_raised_in_order_and_engine_recovers(setup):
    from paper_2501_08547_b200 import runtime
    from paper_2501_08547_b200.compgraph import ServingRequest

    serving, model, w, pe, reqs = setup
    eng = runtime.ServingEngine(serving, pe, model, w, runtime.ServeConfig(strategy="srpe", gamma=0.2))
    bad = ServingRequest.__new__(ServingRequest)  # skip host validation: the device check must catch it
    bad.num_base, bad.num_queries = reqs[0].num_base, reqs[0].num_queries
    bad.query_features = reqs[0].query_features
    e = reqs[0].edges.copy()
    e[0, 0] = serving.num_nodes + 10_000  # out of range
    bad.edges = e
    out = []
    with pytest.raises(ValueError):
        for r in eng.serve_stream([reqs[0], bad, reqs[1]]):
            out.append(r)
    assert len(out) == 1 and np.array_equal(out[0][0], eng.serve(reqs[0])[0])
    emb, _ = eng.serve(reqs[1])
    got = [r[0] for r in eng.serve_stream([reqs[1]])]
    assert np.array_equal(got[0], emb)
    eng.close()


@pytest.mark.parametrize("strategy", ["srpe", "full"])
def test_two_lanes_equal_serve(setup, strategy):
    """Two request lanes (two workspaces on two streams, requests in flight together) change nothing."""
    from paper_2501_08547_b200 import runtime

    serving, model, w, pe, reqs = setup
    eng = runtime.ServingEngine(serving, pe, model, w, runtime.ServeConfig(strategy=strategy, gamma=0.2))
    ref = [eng.serve(r) for r in reqs]
    plan_ref = eng.last_plan() if strategy == "srpe" else None
    for lanes, depth in ((2, 2), (3, 4), (4, 4)):
        eng.set_lanes(lanes)
        got = list(eng.serve_stream(reqs, depth=depth))
        for (a, ba), (b, bb) in zip(got, ref):
            assert np.array_equal(a, b)
            assert ba.fetch_bytes == bb.fetch_bytes
    if strategy == "srpe":  # parity hooks read the lane that served the last request
        assert np.array_equal(eng.last_plan()["targets"], plan_ref["targets"])
    eng.set_lanes(1)
    assert np.array_equal(eng.serve(reqs[2])[0], ref[2][0])
    eng.close()


def test_lanes_under_cgp_emulation(setup):
    """All P partitions on one device (no NCCL): lanes swap the CGP request state too."""
    from paper_2501_08547_b200 import runtime

    serving, model, w, pe, reqs = setup
    eng = runtime.ServingEngine(serving, pe, model, w,
                                runtime.ServeConfig(strategy="srpe-cgp", gamma=0.2, num_partitions=3, seed=5))
    ref = [eng.serve(r)[0] for r in reqs]
    eng.set_lanes(3)
    got = [x[0] for x in eng.serve_stream(reqs, depth=4)]
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))
    eng.close()


def test_lane_api_errors(setup):
    import ctypes as C

    from paper_2501_08547_b200 import _native as nat
    from paper_2501_08547_b200 import runtime

    serving, model, w, pe, reqs = setup
    eng = runtime.ServingEngine(serving, pe, model, w, runtime.ServeConfig(strategy="srpe", gamma=0.2))
    with pytest.raises(ValueError):
        eng.set_lanes(0)
    with pytest.raises(ValueError):
        eng.set_lanes(9)
    eng.set_lanes(2)
    with pytest.raises(RuntimeError):  # profiling needs one lane
        nat.check(nat.lib.ob_profile(eng._h, 1))
    it = eng.serve_stream(reqs, depth=2)
    next(it)  # one request retired, one still in flight
    with pytest.raises(RuntimeError):
        eng.set_lanes(1)
    rest = list(it)
    assert len(rest) == len(reqs) - 1
    eng.set_lanes(1)
    nat.check(nat.lib.ob_profile(eng._h, 1))
    nat.check(nat.lib.ob_profile(eng._h, 0))
    _ = C
    eng.close()


def test_source_range_passes_match_oracle():
    """Lanes on + a source-row set above 64 MB: the sum gathers run as source-range passes."""
    from oracle import layers as OL
    from paper_2501_08547_b200 import graphstore, models, runtime, workload

    full = workload.gen_powerlaw_graph(200_000, 12.0, 2.1, 16, seed=21)
    serving, pool = workload.split_holdout(full, 0.25, seed=21)
    model = models.make_model("sage_mean", 3, 16, 128)  # 512-byte rows: 200K rows exceed 64 MB
    w = models.init_weights(model, 3)
    layers = [dict(kind=s.kind, in_dim=s.in_dim, out_dim=s.out_dim) for s in model.layers]
    pe = graphstore.precompute_embeddings(serving, model, w)
    reqs = [workload.make_request(pool, serving, 64, seed=s) for s in (1, 2, 3)]
    eng = runtime.ServingEngine(serving, pe, model, w, runtime.ServeConfig(strategy="srpe", gamma=0.3))
    one = [eng.serve(r)[0] for r in reqs]
    eng.set_lanes(2)
    two = [x[0] for x in eng.serve_stream(reqs, depth=2)]
    for r, a, b in zip(reqs, one, two):
        ref = OL.serve("srpe", layers, w.layers, serving.num_nodes, r.num_queries, serving.in_offsets,
                       serving.in_neighbors, serving.features, r.query_features, r.edges, pe_layers=pe.layers,
                       gamma=0.3)
        assert OL.max_rel_err(a, ref["emb"]) <= 1e-4
        assert OL.max_rel_err(b, ref["emb"]) <= 1e-4
        assert OL.max_rel_err(a, b) <= 1e-5
    eng.close()


@pytest.mark.parametrize("lanes", [1, 3])
def test_int32_edges_equal_int64(setup, lanes):
    """int32 (src, dst) host edges (ob_serve_i32 / ob_serve_submit_i32, widened on the device) give the
    int64 path's rows bit for bit, and half its request edge bytes."""
    from paper_2501_08547_b200 import runtime
    from paper_2501_08547_b200.compgraph import ServingRequest

    serving, model, w, pe, reqs = setup
    eng = runtime.ServingEngine(serving, pe, model, w, runtime.ServeConfig(strategy="srpe", gamma=0.2))
    eng.set_lanes(lanes)
    r32 = [ServingRequest(r.num_base, r.num_queries, r.query_features, r.edges.astype(np.int32)) for r in reqs]
    assert all(r.edges.dtype == np.int32 for r in r32)
    ref = [eng.serve(r) for r in reqs]
    got = [eng.serve(r) for r in r32]
    for (a, ba), (b, bb) in zip(got, ref):
        assert np.array_equal(a, b)
        assert ba.fetch_bytes == bb.fetch_bytes
    assert eng.last_breakdown.h2d_bytes == 8 * reqs[-1].edges.shape[0] + 4 * reqs[-1].query_features.size
    stream = list(eng.serve_stream(r32 + reqs, depth=4))
    for i, (a, _) in enumerate(stream):
        assert np.array_equal(a, ref[i % len(reqs)][0])
    eng.close()
