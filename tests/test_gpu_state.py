"""Engine state changes between requests -- needs a B200.

A serve captures a CUDA graph of the whole request and builds stored tables
(transforms, layer-1 aggregates) from the weights and stored embeddings.
Replacing either (``reload``: ob_load_model / ob_load_pe, ``precompute_pe``)
must drop those graphs and tables on every request lane, so the next serve
equals a freshly built engine's result bit for bit (graphs replayed
against freed tables).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wl():
    from paper_2501_08547_b200 import workload

    full = workload.gen_powerlaw_graph(6000, 15.0, 2.1, 24, seed=11)
    serving, pool = workload.split_holdout(full, 0.25, seed=11)
    reqs = [workload.make_request(pool, serving, 48, seed=12 + i) for i in range(2)]
    return serving, reqs


def _fresh(serving, pe, model, w, strategy="srpe", gamma=0.3):
    from paper_2501_08547_b200 import runtime

    return runtime.ServingEngine(serving, pe, model, w, runtime.ServeConfig(strategy=strategy, gamma=gamma))


@pytest.mark.parametrize("kind", ["sage_mean", "gcn", "gat"])
@pytest.mark.parametrize("lanes", [1, 3])
def test_reload_weights_and_pe(wl, kind, lanes):
    from paper_2501_08547_b200 import graphstore, models

    serving, reqs = wl
    model = models.make_model(kind, 3, 24, 16)
    w1, w2 = models.init_weights(model, 1), models.init_weights(model, 2)
    rng = np.random.default_rng(3)
    pe1 = graphstore.PeStore([rng.standard_normal((serving.num_nodes, 16)).astype(np.float32) for _ in range(2)])
    pe2 = graphstore.PeStore([rng.standard_normal((serving.num_nodes, 16)).astype(np.float32) for _ in range(2)])
    eng = _fresh(serving, pe1, model, w1)
    eng.set_lanes(lanes)
    for _ in eng.serve_stream(reqs * 2 * lanes, depth=4):  # graphs captured on every lane
        pass
    eng.reload(model, w2)
    got = [eng.serve(r)[0] for r in reqs]
    ref = _fresh(serving, pe1, model, w2)
    exp = [ref.serve(r)[0] for r in reqs]
    for a, b in zip(got, exp):
        assert np.array_equal(a, b)
    eng.reload(pe=pe2)
    got = [emb for emb, _ in eng.serve_stream(reqs * lanes, depth=4)]
    ref.close()
    ref = _fresh(serving, pe2, model, w2)
    exp = [ref.serve(r)[0] for r in reqs]
    for i, a in enumerate(got):
        assert np.array_equal(a, exp[i % len(reqs)])
    ref.close()
    eng.close()


def test_precompute_after_serving(wl):
    from paper_2501_08547_b200 import models

    serving, reqs = wl
    model = models.make_model("sage_mean", 3, 24, 16)
    w1, w2 = models.init_weights(model, 1), models.init_weights(model, 2)
    eng = _fresh(serving, None, model, w1)
    eng.precompute_pe()
    eng.serve(reqs[0])
    eng.reload(model, w2)
    eng.precompute_pe()  # replaces the stored layers (the old ones are freed)
    got = eng.serve(reqs[0])[0]
    ref = _fresh(serving, None, model, w2)
    ref.precompute_pe()
    assert np.array_equal(got, ref.serve(reqs[0])[0])
    ref.close()
    eng.close()


def test_pageable_stream_outputs(wl):
    """serve_stream with pageable numpy outputs (staged through pinned slots) equals serve()."""
    from paper_2501_08547_b200 import models

    serving, reqs = wl
    model = models.make_model("gcn", 2, 24, 16)
    eng = _fresh(serving, None, model, models.init_weights(model, 1), strategy="full")
    exp = [eng.serve(r)[0] for r in reqs]
    got = [emb for emb, _ in eng.serve_stream(reqs * 3, depth=4)]
    for i, a in enumerate(got):
        assert np.array_equal(a, exp[i % 2])
    eng.close()
