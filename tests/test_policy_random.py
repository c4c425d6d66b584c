"""RANDOM policy (policy.py:118-135): targets = sort(ids[default_rng(tie_seed).permutation(|R|)[:budget]]).

The permutation is numpy's (the reference's third-party dependency, numpy 2.3 in this image):
Generator.shuffle's Fisher-Yates over arange(|R|) with random_interval's masked rejection on
PCG64's buffered 32-bit draws.  ``oracle/sampling.py`` restates it (directly and in the traced
form the CUDA path evaluates); both are checked against numpy itself here, and the oracle and
the device against golden targets / embeddings produced by the real reference
(``tests/golden/policy_random.npz``, ``make_golden.py random``).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden

SEEDS = (0, 1, 7, (1 << 40) + 3)
GAMMAS = (0.1, 0.5, 1.0)
CASES = ("s3", "s50", "s60", "s7")


@pytest.fixture(scope="module")
def golden():
    return load_golden("policy_random")


@pytest.mark.parametrize("seed", SEEDS + (12345,))
def test_permutation_restatement_equals_numpy(seed):
    from oracle.sampling import permutation_prefix, permutation_prefix_traced

    for m in (0, 1, 2, 3, 5, 31, 32, 33, 100, 1000, 4097):
        b = m // 3 + 1 if m else 0
        ref = np.random.default_rng(seed).permutation(m)[:b].tolist()
        assert permutation_prefix(m, b, seed) == ref, m
        assert permutation_prefix_traced(m, b, seed) == ref, m


@pytest.mark.parametrize("case", CASES)
def test_oracle_targets_vs_reference(golden, case):
    from oracle.structure import select_random

    ids = golden[f"{case}.cand"]
    for tie in SEEDS:
        for g in GAMMAS:
            assert np.array_equal(select_random(ids, g, tie), golden[f"{case}.t{tie}.g{g}.targets"]), (tie, g)


def _engine(golden, case, tie, gamma, strategy="srpe", P=1):
    from oracle.layers import WEIGHT_NAMES
    from paper_2501_08547_b200 import graphstore, models, runtime

    g = golden
    N, F = int(g[f"{case}.N"]), g[f"{case}.feats"].shape[1]
    ds = graphstore.GraphDataset(N, g[f"{case}.offsets"], g[f"{case}.nbrs"], g[f"{case}.feats"], np.ones(N, bool),
                                 np.zeros(N, bool))
    model = models.make_model("sage_mean", 3, F, 6)
    if f"{case}.w.l1.w_self" in g:
        w = models.Weights([{n: g[f"{case}.w.l{l}.{n}"] for n in WEIGHT_NAMES["sage_mean"]} for l in (1, 2, 3)])
        pe = graphstore.PeStore([g[f"{case}.pe.l{l}"] for l in (1, 2)])
    else:
        w = models.init_weights(model, 4)
        pe = graphstore.PeStore([np.zeros((N, 6), np.float32)] * 2)
    cfg = runtime.ServeConfig(strategy=strategy, gamma=gamma, policy="random", seed=tie, num_partitions=P)
    return runtime.ServingEngine(ds, pe, model, w, cfg)


def _request(golden, case):
    from paper_2501_08547_b200.compgraph import ServingRequest

    g = golden
    return ServingRequest(int(g[f"{case}.N"]), int(g[f"{case}.B"]), g[f"{case}.qfeat"], g[f"{case}.edges"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("tie", SEEDS)
def test_device_targets_vs_reference(golden, case, tie):
    for g in GAMMAS:
        eng = _engine(golden, case, tie, g)
        eng.serve(_request(golden, case))
        plan = eng.last_plan()
        assert np.array_equal(plan["ids"], golden[f"{case}.cand"])
        assert np.all(plan["scores"] == 0.0)
        assert np.array_equal(plan["targets"], golden[f"{case}.t{tie}.g{g}.targets"]), g
        eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["s3", "s50", "s60"])
@pytest.mark.parametrize("P", [1, 2])
def test_device_embeddings_vs_reference(golden, case, P):
    """srpe served with policy="random", seed=7, gamma=0.5 (and its srpe-cgp form) against the reference."""
    from oracle.layers import max_rel_err

    eng = _engine(golden, case, 7, 0.5, "srpe" if P == 1 else "srpe-cgp", P)
    emb, bd = eng.serve(_request(golden, case))
    assert max_rel_err(emb, golden[f"{case}.emb"]) <= 1e-4
    if P == 1:
        assert bd.fetch_bytes == int(golden[f"{case}.fetch"])
    assert np.array_equal(eng.last_plan()["targets"], golden[f"{case}.t7.g0.5.targets"])
    eng.close()
