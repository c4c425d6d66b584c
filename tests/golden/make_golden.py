"""Generate golden vectors by running the REAL reference (gnnserve) in this container.

Usage (from the repo root, in the build container where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small ``.npz`` fixtures next to this script.  They pin the oracle
(tests/test_oracle_golden.py) and, transitively, the CUDA path.  Nothing at
test/bench time reads /root/reference: the fixtures are committed.

Cases:
  demo      -- the reference suite's 8-node Fig. 1 graph + two-query request
               (pkg/tests/conftest.py:8-36), every kind, k in {2,3}
  small_*   -- small_workload graphs (pkg/tests/conftest.py:45-48), every
               kind, srpe/full, gamma sweep, CGP shards for P in {2,3}
  cfg1      -- BASELINE config 1 (100K nodes, GCN k=2, B=256, gamma=0.1):
               hashes of the generated graph/request, the selected targets,
               block hashes, embeddings, fetch bytes
  sampled   -- the sampled strategy (compgraph.py:248-284): blocks and
               embeddings for several fanouts and seeds (incl. a seed above
               2^32), small_workload graphs and the hub graph
  policy_random -- the RANDOM policy (policy.py:122-124, default_rng(tie_seed)
               .permutation): candidates and targets for several seeds and gammas,
               incl. a 20K-candidate request; srpe embeddings served with it
  policy_is -- the importance (IS) policy: centralized scores/targets
               (policy.py:84-95), per-rank partial sums and the distributed
               plan (policy.py:98-107, runtime.py:168-175) for P in {2,3}, and
               srpe / srpe-cgp embeddings served with policy="is", on the demo,
               small_workload graphs and a hub-heavy graph (hubgraph.py)
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

from gnnserve import models, policy, workload
from gnnserve.cgpexec import execute_model
from gnnserve.collectives import make_sim_worlds, run_ranks
from gnnserve.compgraph import (ServingRequest, build_full_k_hop, build_partitioned, build_sampled, build_srpe,
                                partition_request)
from gnnserve.graphstore import make_dataset, partition_random_hash, precompute_embeddings, scatter_pe
from gnnserve.models import forward_full, init_weights, make_model
from gnnserve.runtime import ServeConfig, ServingEngine, graph_fetch_bytes, run_cgp_request

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import hubgraph  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DEMO_EDGES = [(1, 0), (2, 0), (3, 0), (1, 2), (4, 2), (0, 3), (5, 3), (7, 3), (6, 7), (5, 4), (6, 4)]
KINDS = [("gcn", {}), ("sage_mean", {}), ("sage_max", {}), ("power_mean", {"p": 2.0}),
         ("moments", {"n": 3}), ("gat", {})]
GAMMAS = [0.0, 0.1, 0.25, 0.29, 0.5, 0.57, 0.75, 1.0]
BLOCK_FIELDS = ("src_ids", "dst_ids", "edge_src", "edge_dst", "bind_kind", "bind_pe_layer", "src_degree",
                "dst_self_src")


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def put_blocks(out: dict, prefix: str, graph) -> None:
    for l, b in enumerate(graph.blocks, start=1):
        for f in BLOCK_FIELDS:
            v = getattr(b, f)
            if v is not None:
                out[f"{prefix}.b{l}.{f}"] = np.asarray(v)


def put_weights(out: dict, prefix: str, model, w) -> None:
    for l, (spec, mats) in enumerate(zip(model.layers, w.layers), start=1):
        for name, m in mats.items():
            out[f"{prefix}.l{l}.{name}"] = m


def case(name: str, serving, request, extra_cgp: bool) -> None:
    out: dict = {}
    out["N"] = np.int64(serving.num_nodes)
    out["B"] = np.int64(request.num_queries)
    out["offsets"] = serving.in_offsets
    out["nbrs"] = serving.in_neighbors
    out["feats"] = serving.features
    out["edges"] = request.edges
    out["qfeat"] = request.query_features
    cand = policy.find_candidates(request, serving)
    out["cand.ids"] = cand.ids
    out["cand.nq"] = cand.query_edge_counts
    out["cand.total"] = cand.total_degrees
    ok = bool(np.all(cand.total_degrees > 0))
    out["cand.scorable"] = np.bool_(ok)
    if ok:
        scores = policy.score_query_edge_ratio(cand)
        out["cand.scores"] = scores
        for g in GAMMAS:
            out[f"targets.g{g}"] = policy.select_targets(cand, scores, g, "ratio").targets
    F = serving.feature_dim
    for kind, kw in KINDS:
        for k in (2, 3):
            tag = f"{kind}.k{k}"
            model = make_model(kind, k, F, 6, **kw)
            w = init_weights(model, 7 + k)
            put_weights(out, f"w.{tag}", model, w)
            pe = precompute_embeddings(serving, model, w)
            for l in range(1, k):
                out[f"pe.{tag}.l{l}"] = pe.layers[l - 1]
            full = build_full_k_hop(request, serving, k)
            out[f"full.{tag}.emb"] = forward_full(model, full, w, serving.features, request.query_features, None)
            if kind == "sage_mean":
                put_blocks(out, f"full.{tag}", full)
                out[f"full.{tag}.fetch"] = np.int64(graph_fetch_bytes(full, F, None, None))
            if not ok:
                continue
            for g in (0.0, 0.5, 1.0):
                eng = ServingEngine(serving, pe, model, w, ServeConfig(strategy="srpe", gamma=g))
                emb, bd = eng.serve(request)
                out[f"srpe.{tag}.g{g}.emb"] = emb
                out[f"srpe.{tag}.g{g}.fetch"] = np.int64(bd.fetch_bytes)
                if kind == "sage_mean":
                    plan = eng._centralized_plan(request)
                    put_blocks(out, f"srpe.{tag}.g{g}", build_srpe(request, serving, pe, k, plan))
            if extra_cgp:
                for P in (2, 3):
                    eng = ServingEngine(serving, pe, model, w,
                                        ServeConfig(strategy="srpe-cgp", gamma=0.5, num_partitions=P, seed=11))
                    emb, _ = eng.serve(request)
                    out[f"cgp.{tag}.P{P}.emb"] = emb
                    if kind == "sage_mean":
                        out[f"cgp.P{P}.owner"] = eng.pmap.owner
                        preqs = partition_request(request, eng.pmap, P)
                        plan = eng._centralized_plan(request)
                        for r in range(P):
                            shard = build_partitioned(preqs[r], eng.parts[r], plan.targets, k)
                            put_blocks(out, f"cgp.{tag}.P{P}.r{r}", shard)
                            out[f"cgp.P{P}.r{r}.edges"] = preqs[r].edges
                            out[f"cgp.P{P}.r{r}.part_offsets"] = eng.parts[r].edge_offsets
                            out[f"cgp.P{P}.r{r}.part_srcs"] = eng.parts[r].edge_srcs
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, len(out), "arrays")


def demo():
    rng = np.random.default_rng(0)
    ds = make_dataset(DEMO_EDGES, 8, rng.standard_normal((8, 4)).astype(np.float32))
    rng = np.random.default_rng(1)
    pairs = [(8, 2), (8, 3), (9, 2), (9, 4), (9, 7)]
    edges = [(q, t) for q, t in pairs] + [(t, q) for q, t in pairs]
    req = ServingRequest(8, 2, rng.standard_normal((2, 4)).astype(np.float32), np.array(edges))
    case("demo", ds, req, extra_cgp=True)


def small(seed: int, n: int, avg: float, F: int, batch: int, req_seed: int):
    full = workload.gen_powerlaw_graph(n, avg, 2.1, F, seed=seed)
    serving, pool = workload.split_holdout(full, 0.25, seed=seed)
    req = workload.make_request(pool, serving, batch, seed=req_seed)
    case(f"small_s{seed}", serving, req, extra_cgp=True)


def edge_cases():
    """Reference edge cases: empty request, unscorable candidate, isolated query, duplicates."""
    out: dict = {}
    ds = make_dataset([(1, 0), (1, 0), (2, 0), (0, 1)], 4, np.arange(8, dtype=np.float32).reshape(4, 2))
    reqs = {
        "empty": np.empty((0, 2), dtype=np.int64),
        "outonly": np.array([(3, 4)]),          # 3 has zero in-degree and only an outgoing edge
        "dups": np.array([(4, 0), (4, 0), (0, 4), (1, 4), (4, 1)]),
        "qq": np.array([(4, 5), (5, 4), (0, 5)]),
    }
    for name, e in reqs.items():
        req = ServingRequest(4, 2, np.ones((2, 2), dtype=np.float32), e)
        cand = policy.find_candidates(req, ds)
        out[f"{name}.edges"] = req.edges
        out[f"{name}.cand.ids"] = cand.ids
        out[f"{name}.cand.nq"] = cand.query_edge_counts
        out[f"{name}.cand.total"] = cand.total_degrees
        try:
            sc = policy.score_query_edge_ratio(cand)
            out[f"{name}.targets.g0.5"] = policy.select_targets(cand, sc, 0.5, "ratio").targets
            out[f"{name}.scorable"] = np.bool_(True)
        except ValueError:
            out[f"{name}.scorable"] = np.bool_(False)
        model = make_model("sage_mean", 2, 2, 3)
        w = init_weights(model, 1)
        full = build_full_k_hop(req, ds, 2)
        out[f"{name}.full.emb"] = forward_full(model, full, w, ds.features, req.query_features, None)
        put_blocks(out, f"{name}.full", full)
    out["offsets"] = ds.in_offsets
    out["nbrs"] = ds.in_neighbors
    out["feats"] = ds.features
    put_weights(out, "w", model, w)
    np.savez_compressed(os.path.join(HERE, "edge_cases.npz"), **out)
    print("edge_cases", len(out), "arrays")


def cfg1():
    """BASELINE config 1: hashes + targets + embeddings (inputs are regenerated, not stored)."""
    full = workload.gen_powerlaw_graph(100_000, 20.0, 2.1, 64, seed=1)
    serving, pool = workload.split_holdout(full, 0.25, seed=1)
    req = workload.make_request(pool, serving, 256, seed=3)
    model = make_model("gcn", 2, 64, 64)
    w = init_weights(model, 2)
    pe = precompute_embeddings(serving, model, w)
    eng = ServingEngine(serving, pe, model, w, ServeConfig(strategy="srpe", gamma=0.1))
    emb, bd = eng.serve(req)
    plan = eng._centralized_plan(req)
    graph = build_srpe(req, serving, pe, 2, plan)
    out = {
        "graph_sha": np.array(sha(serving.in_offsets, serving.in_neighbors, serving.features)),
        "pool_sha": np.array(sha(pool.ids, pool.incident_edges)),
        "request_sha": np.array(sha(req.edges, req.query_features)),
        "weights_sha": np.array(sha(w.layers[0]["w"], w.layers[1]["w"])),
        "pe_l1": pe.layers[0][::97].copy(),  # every 97th row as a spot check
        "cand.n": np.int64(len(plan.candidate_ids)),
        "cand_sha": np.array(sha(plan.candidate_ids, plan.scores)),
        "targets": plan.targets,
        "emb": emb,
        "fetch_bytes": np.int64(bd.fetch_bytes),
    }
    for l, b in enumerate(graph.blocks, start=1):
        out[f"b{l}.sha"] = np.array(sha(*[np.asarray(getattr(b, f), dtype=np.int64) for f in BLOCK_FIELDS]))
        out[f"b{l}.counts"] = np.array([b.num_src, b.num_dst, b.num_edges], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **out)
    print("cfg1", len(out), "arrays", "targets", len(plan.targets))


def _is_case(out: dict, tag: str, serving, request, F: int, with_emb: bool) -> None:
    out[f"{tag}.N"] = np.int64(serving.num_nodes)
    out[f"{tag}.edges"] = request.edges
    out[f"{tag}.qfeat"] = request.query_features
    cand = policy.find_candidates(request, serving)
    scores = policy.score_importance(cand, serving)
    out[f"{tag}.cand.ids"] = cand.ids
    out[f"{tag}.scores"] = scores
    for g in GAMMAS:
        out[f"{tag}.targets.g{g}"] = policy.select_targets(cand, scores, g, "is").targets
    model = make_model("sage_mean", 3, F, 6)
    w = init_weights(model, 21)
    pe = precompute_embeddings(serving, model, w) if with_emb else None
    if with_emb:
        put_weights(out, f"{tag}.w", model, w)
        for l in range(1, 3):
            out[f"{tag}.pe.l{l}"] = pe.layers[l - 1]
        eng = ServingEngine(serving, pe, model, w, ServeConfig(strategy="srpe", gamma=0.5, policy="is"))
        out[f"{tag}.srpe.emb"], _ = eng.serve(request)
    for P in (2, 3):
        pmap, parts = partition_random_hash(serving, P, 11)
        partials = [policy.importance_partial_sums(cand.ids, parts[r]) for r in range(P)]
        for r in range(P):
            out[f"{tag}.P{P}.partial{r}"] = partials[r]
        if not with_emb:
            continue
        eng = ServingEngine(serving, pe, model, w,
                            ServeConfig(strategy="srpe-cgp", gamma=0.5, num_partitions=P, seed=11, policy="is"))
        preqs = partition_request(request, eng.pmap, P)
        args = [(eng.parts[r], preqs[r], model, w, 0.5, "is", 11, None) for r in range(P)]
        res = run_ranks(make_sim_worlds(P), run_cgp_request, args)
        out[f"{tag}.P{P}.targets"] = res[0][1]["targets"]
        out[f"{tag}.P{P}.emb"] = res[0][0]
        emb2, _ = eng.serve(request)
        assert np.array_equal(emb2, res[0][0])


SAMPLED_RUNS = [((3, 2), 0), ((1, 4), 7), ((4, 3, 2), 0), ((5, 1, 3), 12345678901)]


def sampled():
    out: dict = {}
    for seed, n, avg, F, batch, rs in ((3, 300, 8.0, 10, 5, 9), (50, 200, 10.0, 6, 8, 51), (60, 300, 8.0, 10, 6, 5)):
        full = workload.gen_powerlaw_graph(n, avg, 2.1, F, seed=seed)
        serving, pool = workload.split_holdout(full, 0.25, seed=seed)
        req = workload.make_request(pool, serving, batch, seed=rs)
        tag = f"s{seed}"
        for fan, sd in SAMPLED_RUNS:
            k = len(fan)
            run = f"{tag}.f{''.join(map(str, fan))}.seed{sd}"
            put_blocks(out, run, build_sampled(req, serving, fan, sd))
            for kind, kw in (("sage_mean", {}), ("gcn", {}), ("gat", {})):
                model = make_model(kind, k, F, 6, **kw)
                w = init_weights(model, 7 + k)  # the small_* fixtures' weights (case())
                eng = ServingEngine(serving, None, model, w, ServeConfig(strategy="sampled", fanouts=fan, seed=sd))
                out[f"{run}.{kind}.emb"], bd = eng.serve(req)
                out[f"{run}.{kind}.fetch"] = np.int64(bd.fetch_bytes)
    hub = make_dataset(hubgraph.edges(), hubgraph.N, hubgraph.features())
    e, qf = hubgraph.request()
    req = ServingRequest(hubgraph.N, len(qf), qf, e)
    for fan, sd in (((25, 10), 3), ((150, 200), 99)):
        put_blocks(out, f"hub.f{fan[0]}_{fan[1]}.seed{sd}", build_sampled(req, hub, fan, sd))
    np.savez_compressed(os.path.join(HERE, "sampled.npz"), **out)
    print("sampled", len(out), "arrays")


def policy_is():
    out: dict = {}
    rng = np.random.default_rng(0)
    ds = make_dataset(DEMO_EDGES, 8, rng.standard_normal((8, 4)).astype(np.float32))
    rng = np.random.default_rng(1)
    pairs = [(8, 2), (8, 3), (9, 2), (9, 4), (9, 7)]
    edges = [(q, t) for q, t in pairs] + [(t, q) for q, t in pairs]
    req = ServingRequest(8, 2, rng.standard_normal((2, 4)).astype(np.float32), np.array(edges))
    _is_case(out, "demo", ds, req, 4, True)
    for seed, n, avg, F, batch, rs in ((3, 300, 8.0, 10, 5, 9), (50, 200, 10.0, 6, 8, 51), (60, 300, 8.0, 10, 6, 5)):
        full = workload.gen_powerlaw_graph(n, avg, 2.1, F, seed=seed)
        serving, pool = workload.split_holdout(full, 0.25, seed=seed)
        req = workload.make_request(pool, serving, batch, seed=rs)
        _is_case(out, f"s{seed}", serving, req, F, True)
    hub = make_dataset(hubgraph.edges(), hubgraph.N, hubgraph.features())
    off, nb = hubgraph.csr()
    assert np.array_equal(hub.in_offsets, off) and np.array_equal(hub.in_neighbors, nb)
    e, qf = hubgraph.request()
    _is_case(out, "hub", hub, ServingRequest(hubgraph.N, len(qf), qf, e), 4, False)
    np.savez_compressed(os.path.join(HERE, "policy_is.npz"), **out)
    print("policy_is", len(out), "arrays")


def policy_random():
    out: dict = {}
    cases = [(3, 300, 8.0, 10, 5, 9), (50, 200, 10.0, 6, 8, 51), (60, 300, 8.0, 10, 6, 5), (7, 40000, 12.0, 8, 512, 3)]
    for seed, n, avg, F, batch, rs in cases:
        full = workload.gen_powerlaw_graph(n, avg, 2.1, F, seed=seed)
        serving, pool = workload.split_holdout(full, 0.25, seed=seed)
        req = workload.make_request(pool, serving, batch, seed=rs)
        tag = f"s{seed}"
        out[f"{tag}.offsets"] = serving.in_offsets
        out[f"{tag}.nbrs"] = serving.in_neighbors
        out[f"{tag}.feats"] = serving.features
        out[f"{tag}.N"] = np.int64(serving.num_nodes)
        out[f"{tag}.B"] = np.int64(batch)
        out[f"{tag}.qfeat"] = req.query_features
        out[f"{tag}.edges"] = req.edges
        cand = policy.find_candidates(req, serving)
        out[f"{tag}.cand"] = cand.ids
        for tie in (0, 1, 7, (1 << 40) + 3):
            for g in (0.1, 0.5, 1.0):
                plan = policy.select_targets(cand, np.zeros(len(cand)), g, policy.POLICY_RANDOM, tie_seed=tie)
                out[f"{tag}.t{tie}.g{g}.targets"] = plan.targets
        if n <= 300:  # srpe served with the random policy (sage_mean k=3)
            model = make_model("sage_mean", 3, F, 6)
            w = init_weights(model, 4)
            pe = precompute_embeddings(serving, model, w)
            for li, lw in enumerate(w.layers, start=1):
                for nm, m in lw.items():
                    out[f"{tag}.w.l{li}.{nm}"] = m
            for l in range(1, 3):
                out[f"{tag}.pe.l{l}"] = pe.layers[l - 1]
            eng = ServingEngine(serving, pe, model, w, ServeConfig(strategy="srpe", gamma=0.5, policy="random", seed=7))
            emb, bd = eng.serve(req)
            out[f"{tag}.emb"] = emb
            out[f"{tag}.fetch"] = np.int64(bd.fetch_bytes)
    np.savez_compressed(os.path.join(HERE, "policy_random.npz"), **out)
    print("policy_random", len(out), "arrays")


if __name__ == "__main__":
    which = sys.argv[1:] or ["demo", "small", "edge", "cfg1", "is", "sampled", "random"]
    if "random" in which:
        policy_random()
    if "sampled" in which:
        sampled()
    if "is" in which:
        policy_is()
    if "demo" in which:
        demo()
    if "small" in which:
        small(3, 300, 8.0, 10, 5, 9)
        small(50, 200, 10.0, 6, 8, 51)
        small(60, 300, 8.0, 10, 6, 5)
    if "edge" in which:
        edge_cases()
    if "cfg1" in which:
        cfg1()
