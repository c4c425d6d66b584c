"""Sampled strategy (compgraph.py:248-284): oracle vs the reference (CPU) and the CUDA path (GPU).

Every destination's kept sources come from numpy's
SeedSequence(seed, (layer, v)) -> PCG64 -> choice(replace=False) stream; the
CUDA path re-implements that stream per destination, so blocks are compared
bit for bit and embeddings within 1e-4.  Fixtures: tests/golden/sampled.npz
(tests/golden/make_golden.py ``sampled``).
"""

from __future__ import annotations

import sys

import numpy as np
import pytest

from conftest import GOLDEN, assert_block_equal, golden_layers, golden_weights, load_golden

sys.path.insert(0, GOLDEN)
import hubgraph  # noqa: E402

from oracle import layers as OL  # noqa: E402
from oracle import sampling as OSM  # noqa: E402
from oracle import structure as OS  # noqa: E402

RUNS = [((3, 2), 0), ((1, 4), 7), ((4, 3, 2), 0), ((5, 1, 3), 12345678901)]
CASES = [("s3", "small_s3"), ("s50", "small_s50"), ("s60", "small_s60")]
KINDS = [("sage_mean", {}), ("gcn", {}), ("gat", {})]
HUB_RUNS = [((25, 10), 3), ((150, 200), 99)]
TOL = 1e-4
FIELDS = ("src_ids", "dst_ids", "edge_src", "edge_dst", "bind_kind", "src_degree", "dst_self_src")


@pytest.fixture(scope="module")
def gs():
    return load_golden("sampled")


def _run(tag, fan, seed):
    return f"{tag}.f{''.join(map(str, fan))}.seed{seed}"


def test_restated_stream_matches_numpy():
    """SeedSequence + PCG64 + Floyd restated in Python == numpy's own choice (incl. 2-word seeds, big n)."""
    rng = np.random.default_rng(5)
    for t in range(300):
        seed = int(rng.integers(0, 2 ** 40)) if t % 3 == 0 else int(rng.integers(0, 100))
        layer, v = int(rng.integers(1, 4)), int(rng.integers(0, 2 ** 31 - 1))
        n = int(rng.integers(2, 3000)) if t % 5 else int(rng.integers(10_000, 200_000))
        size = int(rng.integers(1, min(n, 200)))
        assert OSM.choice_set(n, size, seed, layer, v) == OSM.numpy_choice_set(n, size, seed, layer, v).tolist()


@pytest.mark.parametrize("tag,name", CASES)
@pytest.mark.parametrize("fan,seed", RUNS)
def test_oracle_sampled_blocks(gs, tag, name, fan, seed):
    g = load_golden(name)
    blocks = OS.build_sampled(int(g["N"]), int(g["B"]), g["offsets"], g["nbrs"], g["edges"], fan, seed)
    for l, b in enumerate(blocks, start=1):
        assert_block_equal(b, gs, f"{_run(tag, fan, seed)}.b{l}", FIELDS)


@pytest.mark.parametrize("tag,name", CASES)
@pytest.mark.parametrize("fan,seed", RUNS)
@pytest.mark.parametrize("kind,kw", KINDS)
def test_oracle_sampled_embeddings(gs, tag, name, fan, seed, kind, kw):
    g = load_golden(name)
    k = len(fan)
    F = g["feats"].shape[1]
    res = OL.serve("sampled", golden_layers(kind, kw, k, F), golden_weights(g, f"w.{kind}.k{k}", kind, k),
                   int(g["N"]), int(g["B"]), g["offsets"], g["nbrs"], g["feats"], g["qfeat"], g["edges"],
                   fanouts=fan, seed=seed)
    assert OL.max_rel_err(res["emb"], gs[f"{_run(tag, fan, seed)}.{kind}.emb"]) <= 1e-5
    assert res["fetch_bytes"] == int(gs[f"{_run(tag, fan, seed)}.{kind}.fetch"])


@pytest.mark.parametrize("fan,seed", HUB_RUNS)
def test_oracle_sampled_hub(gs, fan, seed):
    off, nb = hubgraph.csr()
    e, qf = hubgraph.request()
    blocks = OS.build_sampled(hubgraph.N, len(qf), off, nb, e, fan, seed)
    for l, b in enumerate(blocks, start=1):
        assert_block_equal(b, gs, f"hub.f{fan[0]}_{fan[1]}.seed{seed}.b{l}", FIELDS)


# ---------------------------------------------------------------------------
# CUDA path
# ---------------------------------------------------------------------------


def _engine(g, kind, kw, fan, seed):
    from paper_2501_08547_b200 import graphstore, models, runtime

    N, F, k = int(g["N"]), g["feats"].shape[1], len(fan)
    ds = graphstore.GraphDataset(N, g["offsets"], g["nbrs"], g["feats"], np.ones(N, bool), np.zeros(N, bool))
    model = models.make_model(kind, k, F, 6, **kw)
    w = models.Weights(golden_weights(g, f"w.{kind}.k{k}", kind, k))
    return runtime.ServingEngine(ds, None, model, w, runtime.ServeConfig(strategy="sampled", fanouts=fan, seed=seed))


@pytest.mark.gpu
@pytest.mark.parametrize("tag,name", CASES)
@pytest.mark.parametrize("fan,seed", RUNS)
@pytest.mark.parametrize("kind,kw", KINDS)
def test_gpu_sampled(gs, tag, name, fan, seed, kind, kw):
    from paper_2501_08547_b200.compgraph import ServingRequest

    g = load_golden(name)
    eng = _engine(g, kind, kw, fan, seed)
    emb, bd = eng.serve(ServingRequest(int(g["N"]), int(g["B"]), g["qfeat"], g["edges"]))
    run = _run(tag, fan, seed)
    assert OL.max_rel_err(emb, gs[f"{run}.{kind}.emb"]) <= TOL
    assert bd.fetch_bytes == int(gs[f"{run}.{kind}.fetch"])
    for l in range(1, len(fan) + 1):
        assert_block_equal(eng.last_block(l), gs, f"{run}.b{l}", FIELDS)
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("fan,seed", HUB_RUNS)
def test_gpu_sampled_hub(gs, fan, seed):
    """Rows of up to 70,000 sources sampled down to 10..200 (Floyd draws up to j = 69,999)."""
    from paper_2501_08547_b200 import graphstore, models, runtime
    from paper_2501_08547_b200.compgraph import ServingRequest

    off, nb = hubgraph.csr()
    N = hubgraph.N
    ds = graphstore.GraphDataset(N, off, nb, hubgraph.features(), np.ones(N, bool), np.zeros(N, bool))
    model = models.make_model("sage_mean", 2, 4, 4)
    w = models.init_weights(model, 3)
    eng = runtime.ServingEngine(ds, None, model, w, runtime.ServeConfig(strategy="sampled", fanouts=fan, seed=seed))
    e, qf = hubgraph.request()
    emb, _ = eng.serve(ServingRequest(N, len(qf), qf, e))
    for l in (1, 2):
        assert_block_equal(eng.last_block(l), gs, f"hub.f{fan[0]}_{fan[1]}.seed{seed}.b{l}", FIELDS)
    eng.close()


@pytest.mark.gpu
def test_gpu_sampled_config_errors():
    from paper_2501_08547_b200 import graphstore, models, runtime

    g = load_golden("small_s3")
    with pytest.raises(ValueError):
        _engine(g, "sage_mean", {}, (3, 0), 0)  # fanouts must be >= 1 (compgraph.py:256-257)
    with pytest.raises(ValueError):
        runtime.ServeConfig(strategy="sampled")  # needs fanouts (runtime.py:76-77)
    N, F = int(g["N"]), g["feats"].shape[1]
    ds = graphstore.GraphDataset(N, g["offsets"], g["nbrs"], g["feats"], np.ones(N, bool), np.zeros(N, bool))
    model = models.make_model("sage_mean", 2, F, 6)
    w = models.init_weights(model, 1)
    with pytest.raises(ValueError):  # one fanout per layer (forward_full's depth check, models.py:290-292)
        runtime.ServingEngine(ds, None, model, w, runtime.ServeConfig(strategy="sampled", fanouts=(3, 2, 2)))
