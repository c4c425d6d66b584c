"""Pin the CPU oracle to golden vectors produced by the real reference.

The fixtures under tests/golden/ come from running ``gnnserve`` itself
(tests/golden/make_golden.py).  Everything integer (candidates, scores,
targets, block arrays, partition owners, shards, fetch bytes) must match
bit-for-bit; embeddings within max|a-r|/max|r| <= 1e-5 (both sides
accumulate in float64; only summation order differs).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import KINDS, SMALL_CASES, assert_block_equal, golden_layers, golden_weights, load_golden
from oracle import layers as OL
from oracle import structure as OS

TOL = 1e-5


def _case(g):
    N, B = int(g["N"]), int(g["B"])
    return N, B, g["offsets"], g["nbrs"], g["feats"], g["edges"], g["qfeat"]


@pytest.mark.parametrize("name", SMALL_CASES)
def test_candidates_scores_targets(goldens, name):
    g = goldens[name]
    N, B, off, nb, feats, edges, q = _case(g)
    ids, nq, total = OS.candidates(edges, N, np.diff(off))
    assert np.array_equal(ids, g["cand.ids"])
    assert np.array_equal(nq, g["cand.nq"])
    assert np.array_equal(total, g["cand.total"])
    sc = OS.ratio_scores(nq, total)
    assert np.array_equal(sc.view(np.uint64), g["cand.scores"].view(np.uint64))
    for gamma in (0.0, 0.1, 0.25, 0.29, 0.5, 0.57, 0.75, 1.0):
        assert np.array_equal(OS.select_top(ids, sc, gamma), g[f"targets.g{gamma}"]), gamma


def test_demo_known_answers(goldens):
    # pkg/tests/test_policy.py:20-75
    g = goldens["demo"]
    N, B, off, nb, feats, edges, q = _case(g)
    ids, nq, total = OS.candidates(edges, N, np.diff(off))
    assert ids.tolist() == [2, 3, 4, 7]
    assert dict(zip(ids.tolist(), nq.tolist())) == {2: 2, 3: 1, 4: 1, 7: 1}
    assert dict(zip(ids.tolist(), total.tolist())) == {2: 4, 3: 4, 4: 3, 7: 2}
    sc = OS.ratio_scores(nq, total)
    assert sc.tolist() == [0.5, 0.25, 1 / 3, 0.5]
    assert OS.select_top(ids, sc, 0.5).tolist() == [2, 7]
    with pytest.raises(ValueError):
        OS.select_top(ids, sc, 1.5)


@pytest.mark.parametrize("name", SMALL_CASES)
@pytest.mark.parametrize("k", [2, 3])
def test_blocks_exact(goldens, name, k):
    g = goldens[name]
    N, B, off, nb, feats, edges, q = _case(g)
    blocks = OS.build_full(N, B, off, nb, edges, k)
    for l, b in enumerate(blocks, start=1):
        assert_block_equal(b, g, f"full.sage_mean.k{k}.b{l}")
    if not bool(g["cand.scorable"]):
        return
    for gamma in (0.0, 0.5, 1.0):
        tg = g[f"targets.g{gamma}"]
        blocks = OS.build_srpe(N, B, off, nb, edges, tg, k, k - 1)
        for l, b in enumerate(blocks, start=1):
            assert_block_equal(b, g, f"srpe.sage_mean.k{k}.g{gamma}.b{l}")
        assert OS.fetch_bytes(blocks, N, feats.shape[1], [6] * (k - 1)) == int(g[f"srpe.sage_mean.k{k}.g{gamma}.fetch"])
    full = OS.build_full(N, B, off, nb, edges, k)
    assert OS.fetch_bytes(full, N, feats.shape[1], []) == int(g[f"full.sage_mean.k{k}.fetch"])


@pytest.mark.parametrize("name", SMALL_CASES)
@pytest.mark.parametrize("kind,kw", KINDS)
@pytest.mark.parametrize("k", [2, 3])
def test_embeddings(goldens, name, kind, kw, k):
    g = goldens[name]
    N, B, off, nb, feats, edges, q = _case(g)
    tag = f"{kind}.k{k}"
    layers = golden_layers(kind, kw, k, feats.shape[1])
    w = golden_weights(g, f"w.{tag}", kind, k)
    pe = OL.precompute(layers, w, off, nb, feats)
    for l in range(1, k):
        assert OL.max_rel_err(pe[l - 1], g[f"pe.{tag}.l{l}"]) <= TOL
    full = OL.serve("full", layers, w, N, B, off, nb, feats, q, edges)
    assert OL.max_rel_err(full["emb"], g[f"full.{tag}.emb"]) <= TOL
    if not bool(g["cand.scorable"]):
        return
    gpe = [g[f"pe.{tag}.l{l}"] for l in range(1, k)]
    for gamma in (0.0, 0.5, 1.0):
        r = OL.serve("srpe", layers, w, N, B, off, nb, feats, q, edges, pe_layers=gpe, gamma=gamma)
        assert OL.max_rel_err(r["emb"], g[f"srpe.{tag}.g{gamma}.emb"]) <= TOL, gamma
        assert r["fetch_bytes"] == int(g[f"srpe.{tag}.g{gamma}.fetch"])


@pytest.mark.parametrize("name", SMALL_CASES)
@pytest.mark.parametrize("P", [2, 3])
def test_cgp_partitions_and_shards(goldens, name, P):
    g = goldens[name]
    N, B, off, nb, feats, edges, q = _case(g)
    owner, shards = OS.partition_graph(off, nb, N, P, 11)
    assert np.array_equal(owner, g[f"cgp.P{P}.owner"])
    parts = OS.split_request(edges, N, owner, P)
    deg = np.diff(off)
    qdeg = OS.query_in_degrees(edges, N, B)
    tg = g["targets.g0.5"]
    for r in range(P):
        assert np.array_equal(shards[r].offsets, g[f"cgp.P{P}.r{r}.part_offsets"])
        assert np.array_equal(shards[r].srcs, g[f"cgp.P{P}.r{r}.part_srcs"])
        pe_sorted = np.lexsort((parts[r][:, 1], parts[r][:, 0]))
        exp = g[f"cgp.P{P}.r{r}.edges"]
        assert np.array_equal(parts[r][pe_sorted], exp[np.lexsort((exp[:, 1], exp[:, 0]))])
        for k in (2, 3):
            blocks = OS.build_partitioned_shard(N, B, shards[r], owner, P, parts[r], qdeg, deg, tg, k)
            for l, b in enumerate(blocks, start=1):
                assert_block_equal(b, g, f"cgp.sage_mean.k{k}.P{P}.r{r}.b{l}")


@pytest.mark.parametrize("name", SMALL_CASES)
@pytest.mark.parametrize("kind,kw", KINDS)
@pytest.mark.parametrize("P", [2, 3])
def test_cgp_embeddings(goldens, name, kind, kw, P):
    g = goldens[name]
    N, B, off, nb, feats, edges, q = _case(g)
    for k in (2, 3):
        tag = f"{kind}.k{k}"
        layers = golden_layers(kind, kw, k, feats.shape[1])
        w = golden_weights(g, f"w.{tag}", kind, k)
        gpe = [g[f"pe.{tag}.l{l}"] for l in range(1, k)]
        r = OL.cgp_serve(layers, w, N, B, off, nb, feats, q, edges, gpe, 0.5, P, 11)
        assert OL.max_rel_err(r["emb"], g[f"cgp.{tag}.P{P}.emb"]) <= TOL


def test_edge_cases():
    g = load_golden("edge_cases")
    off, nb, feats = g["offsets"], g["nbrs"], g["feats"]
    N = len(off) - 1
    layers = golden_layers("sage_mean", {}, 2, 2, 3)
    w = golden_weights(g, "w", "sage_mean", 2)
    for name in ("empty", "outonly", "dups", "qq"):
        edges = g[f"{name}.edges"].reshape(-1, 2)
        ids, nq, total = OS.candidates(edges, N, np.diff(off))
        assert np.array_equal(ids, g[f"{name}.cand.ids"])
        assert np.array_equal(nq, g[f"{name}.cand.nq"])
        assert np.array_equal(total, g[f"{name}.cand.total"])
        if bool(g[f"{name}.scorable"]):
            assert np.array_equal(OS.select_top(ids, OS.ratio_scores(nq, total), 0.5), g[f"{name}.targets.g0.5"])
        else:
            with pytest.raises(ValueError):
                OS.ratio_scores(nq, total)
        q = np.ones((2, 2), dtype=np.float32)
        r = OL.serve("full", layers, w, N, 2, off, nb, feats, q, edges)
        assert OL.max_rel_err(r["emb"], g[f"{name}.full.emb"]) <= TOL
        for l, b in enumerate(r["blocks"], start=1):
            assert_block_equal(b, g, f"{name}.full.b{l}")
