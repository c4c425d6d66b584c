"""Importance (IS) policy: oracle vs the reference's golden vectors (CPU) and the CUDA path (GPU).

Reference: score_importance (policy.py:84-95), importance_partial_sums
(policy.py:98-107), the distributed IS branch of select_targets_distributed
(runtime.py:168-175).  Scores are fp64 and compared bit for bit: the row
sums must follow numpy's pairwise association exactly.  Fixtures:
tests/golden/policy_is.npz (tests/golden/make_golden.py ``is``).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

sys.path.insert(0, GOLDEN)
import hubgraph  # noqa: E402

from oracle import structure as OS  # noqa: E402

TAGS = ["demo", "s3", "s50", "s60"]
GAMMAS = [0.0, 0.1, 0.25, 0.29, 0.5, 0.57, 0.75, 1.0]
TOL = 1e-4


@pytest.fixture(scope="module")
def gis():
    return load_golden("policy_is")


@pytest.fixture(scope="module")
def graphs():
    """tag -> (offsets, nbrs, feats) of the serving graph the fixture was made on."""
    out = {}
    for tag, name in (("demo", "demo"), ("s3", "small_s3"), ("s50", "small_s50"), ("s60", "small_s60")):
        g = load_golden(name)
        out[tag] = (g["offsets"], g["nbrs"], g["feats"])
    off, nb = hubgraph.csr()
    out["hub"] = (off, nb, hubgraph.features())
    return out


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("tag", TAGS + ["hub"])
def test_oracle_importance_scores(gis, graphs, tag):
    off, nb, _ = graphs[tag]
    N = int(gis[f"{tag}.N"])
    deg = np.diff(off)
    ids, _, _ = OS.candidates(gis[f"{tag}.edges"], N, deg)
    assert np.array_equal(ids, gis[f"{tag}.cand.ids"])
    sc = OS.importance_scores(ids, off, nb, deg)
    assert np.array_equal(_bits(sc), _bits(gis[f"{tag}.scores"]))
    for g in GAMMAS:
        assert np.array_equal(OS.select_top(ids, sc, g), gis[f"{tag}.targets.g{g}"])


@pytest.mark.parametrize("tag", TAGS + ["hub"])
@pytest.mark.parametrize("P", [2, 3])
def test_oracle_importance_partials(gis, graphs, tag, P):
    off, nb, _ = graphs[tag]
    N = int(gis[f"{tag}.N"])
    deg = np.diff(off)
    ids = gis[f"{tag}.cand.ids"]
    _, shards = OS.partition_graph(off, nb, N, P, 11)
    partials = []
    for r in range(P):
        p = OS.importance_partial_sums(ids, shards[r].offsets, shards[r].srcs, deg)
        assert np.array_equal(_bits(p), _bits(gis[f"{tag}.P{P}.partial{r}"]))
        partials.append(p)
    sc = OS.importance_scores_distributed(ids, partials, deg)
    if f"{tag}.P{P}.targets" in gis:
        assert np.array_equal(OS.select_top(ids, sc, 0.5), gis[f"{tag}.P{P}.targets"])


def test_hub_rows_need_pairwise_order(graphs):
    """The fixture discriminates: a sequential row sum gives different bits on the hubs."""
    off, nb, _ = graphs["hub"]
    deg = np.diff(off)
    t = OS._is_terms(nb[off[0]:off[1]], deg)
    seq = 0.0
    for x in t:
        seq += x
    assert seq != np.sum(t)


# ---------------------------------------------------------------------------
# CUDA path
# ---------------------------------------------------------------------------


def _dataset(graphs, tag):
    from paper_2501_08547_b200 import graphstore

    off, nb, feats = graphs[tag]
    N = len(off) - 1
    return graphstore.GraphDataset(N, off, nb, feats, np.ones(N, bool), np.zeros(N, bool))


def _request(gis, tag):
    from paper_2501_08547_b200.compgraph import ServingRequest

    q = gis[f"{tag}.qfeat"]
    return ServingRequest(int(gis[f"{tag}.N"]), len(q), q, gis[f"{tag}.edges"])


def _model(gis, tag, F):
    from conftest import golden_weights
    from paper_2501_08547_b200 import graphstore, models

    model = models.make_model("sage_mean", 3, F, 6)
    w = models.Weights(golden_weights(gis, f"{tag}.w", "sage_mean", 3))
    pe = graphstore.PeStore([gis[f"{tag}.pe.l{l}"] for l in (1, 2)])
    return model, w, pe


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_gpu_srpe_is(gis, graphs, tag):
    from oracle.layers import max_rel_err
    from paper_2501_08547_b200 import runtime

    ds = _dataset(graphs, tag)
    model, w, pe = _model(gis, tag, ds.features.shape[1])
    eng = runtime.ServingEngine(ds, pe, model, w, runtime.ServeConfig(strategy="srpe", gamma=0.5, policy="is"))
    emb, _ = eng.serve(_request(gis, tag))
    plan = eng.last_plan()
    assert np.array_equal(plan["ids"], gis[f"{tag}.cand.ids"])
    assert np.array_equal(_bits(plan["scores"]), _bits(gis[f"{tag}.scores"]))
    assert np.array_equal(plan["targets"], gis[f"{tag}.targets.g0.5"])
    assert max_rel_err(emb, gis[f"{tag}.srpe.emb"]) <= TOL
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("gamma", GAMMAS)
def test_gpu_hub_is_scores(gis, graphs, gamma):
    """Rows of 70,000 / 40,000 / 300 / 129 / 7 / 1 terms: every branch of the pairwise sum."""
    from paper_2501_08547_b200 import graphstore, models, runtime

    ds = _dataset(graphs, "hub")
    model = models.make_model("sage_mean", 2, 4, 4)
    w = models.init_weights(model, 3)
    pe = graphstore.PeStore([np.zeros((ds.num_nodes, 4), np.float32)])
    eng = runtime.ServingEngine(ds, pe, model, w, runtime.ServeConfig(strategy="srpe", gamma=gamma, policy="is"))
    eng.serve(_request(gis, "hub"))
    plan = eng.last_plan()
    assert np.array_equal(plan["ids"], gis["hub.cand.ids"])
    assert np.array_equal(_bits(plan["scores"]), _bits(gis["hub.scores"]))
    assert np.array_equal(plan["targets"], gis[f"hub.targets.g{gamma}"])
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("P", [2, 3])
def test_gpu_cgp_is(gis, graphs, tag, P):
    """CGP emulation: rank-ordered partial sums give the reference's distributed plan."""
    from oracle.layers import max_rel_err
    from paper_2501_08547_b200 import runtime

    ds = _dataset(graphs, tag)
    model, w, pe = _model(gis, tag, ds.features.shape[1])
    cfg = runtime.ServeConfig(strategy="srpe-cgp", gamma=0.5, num_partitions=P, seed=11, policy="is")
    eng = runtime.ServingEngine(ds, pe, model, w, cfg)
    emb, _ = eng.serve(_request(gis, tag))
    plan = eng.last_plan()
    deg = np.diff(graphs[tag][0])
    exp = OS.importance_scores_distributed(gis[f"{tag}.cand.ids"],
                                           [gis[f"{tag}.P{P}.partial{r}"] for r in range(P)], deg)
    assert np.array_equal(_bits(plan["scores"]), _bits(exp))
    assert np.array_equal(plan["targets"], gis[f"{tag}.P{P}.targets"])
    assert max_rel_err(emb, gis[f"{tag}.P{P}.emb"]) <= TOL
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3])
def test_gpu_cgp_is_hub_scores(gis, graphs, P):
    from paper_2501_08547_b200 import graphstore, models, runtime

    ds = _dataset(graphs, "hub")
    model = models.make_model("sage_mean", 2, 4, 4)
    w = models.init_weights(model, 3)
    pe = graphstore.PeStore([np.zeros((ds.num_nodes, 4), np.float32)])
    cfg = runtime.ServeConfig(strategy="srpe-cgp", gamma=0.5, num_partitions=P, seed=11, policy="is")
    eng = runtime.ServingEngine(ds, pe, model, w, cfg)
    eng.serve(_request(gis, "hub"))
    plan = eng.last_plan()
    deg = np.diff(graphs["hub"][0])
    exp = OS.importance_scores_distributed(gis["hub.cand.ids"],
                                           [gis[f"hub.P{P}.partial{r}"] for r in range(P)], deg)
    assert np.array_equal(_bits(plan["scores"]), _bits(exp))
    assert np.array_equal(plan["targets"], OS.select_top(gis["hub.cand.ids"], exp, 0.5))
    eng.close()


def test_policy_validation_on_host():
    """Unknown policies fail on the host side before touching the device (ServeConfig mirrors runtime.py:74-82)."""
    from paper_2501_08547_b200 import _native as nat

    assert nat.POLICY == {"ratio": 0, "is": 1, "random": 2}
    _ = os
