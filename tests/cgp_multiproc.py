"""One-process-per-GPU CGP check (launched by torchrun; used by test_gpu_cgp_multi).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 tests/cgp_multiproc.py

Every rank serves the same requests through an NCCL-connected engine; rank 0
compares the result with the reference's CGP embeddings (golden) and with the
single-process emulation, and prints one JSON line.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    from conftest import KINDS, golden_weights, load_golden
    from oracle.layers import max_rel_err
    from paper_2501_08547_b200 import graphstore, models, runtime
    from paper_2501_08547_b200.compgraph import ServingRequest

    results = []
    for name in ("small_s3", "small_s50", "small_s60"):
        g = load_golden(name)
        N, F = int(g["N"]), g["feats"].shape[1]
        ds = graphstore.GraphDataset(N, g["offsets"], g["nbrs"], g["feats"], np.ones(N, bool), np.zeros(N, bool))
        req = ServingRequest(N, int(g["B"]), g["qfeat"], g["edges"])
        for kind, kw in KINDS:
            for k in (2, 3):
                model = models.make_model(kind, k, F, 6, **kw)
                w = models.Weights(golden_weights(g, f"w.{kind}.k{k}", kind, k))
                pe = graphstore.PeStore([g[f"pe.{kind}.k{k}.l{l}"] for l in range(1, k)])
                cfg = runtime.ServeConfig(strategy="srpe-cgp", gamma=0.5, num_partitions=P, seed=11, device=local)
                eng = runtime.distributed_engine(ds, pe, model, w, cfg)
                emb, bd = eng.serve(req)
                # this rank's shard equals the emulation's shard for the same rank
                emu = runtime.ServingEngine(ds, pe, model, w, cfg)
                emb_emu, _ = emu.serve(req)
                same_shard = all(
                    np.array_equal(eng.last_block(l, partition=rank).edge_src,
                                   emu.last_block(l, partition=rank).edge_src)
                    for l in range(1, k + 1))
                if rank == 0:
                    key = f"cgp.{kind}.k{k}.P{P}.emb"
                    ref = g[key] if key in g else emb_emu
                    results.append(dict(case=name, kind=kind, k=k, err_ref=max_rel_err(emb, ref),
                                        err_emu=max_rel_err(emb, emb_emu), shard=bool(same_shard),
                                        coll_bytes=int(bd.collective_bytes)))
                eng.close()
                emu.close()
    # importance policy: per-rank numerators exchanged and summed in rank order
    # (runtime.py:168-175) must give the reference's distributed plan
    gis = load_golden("policy_is")
    for tag, name in (("s3", "small_s3"), ("s50", "small_s50"), ("s60", "small_s60")):
        g = load_golden(name)
        N, F = int(g["N"]), g["feats"].shape[1]
        ds = graphstore.GraphDataset(N, g["offsets"], g["nbrs"], g["feats"], np.ones(N, bool), np.zeros(N, bool))
        q = gis[f"{tag}.qfeat"]
        req = ServingRequest(N, len(q), q, gis[f"{tag}.edges"])
        model = models.make_model("sage_mean", 3, F, 6)
        w = models.Weights(golden_weights(gis, f"{tag}.w", "sage_mean", 3))
        pe = graphstore.PeStore([gis[f"{tag}.pe.l{l}"] for l in (1, 2)])
        cfg = runtime.ServeConfig(strategy="srpe-cgp", gamma=0.5, num_partitions=P, seed=11, device=local,
                                  policy="is")
        eng = runtime.distributed_engine(ds, pe, model, w, cfg)
        emb, bd = eng.serve(req)
        plan = eng.last_plan()
        if rank == 0:
            key = f"{tag}.P{P}.emb"
            ok_t = f"{tag}.P{P}.targets" not in gis or np.array_equal(plan["targets"], gis[f"{tag}.P{P}.targets"])
            results.append(dict(case=f"is.{tag}", kind="sage_mean", k=3,
                                err_ref=max_rel_err(emb, gis[key]) if key in gis else 0.0,
                                err_emu=0.0, shard=bool(ok_t), coll_bytes=int(bd.collective_bytes)))
        eng.close()
    # device-generated graph with partitioned storage: each rank holds only its
    # owned rows and source-split CSR; the single-process emulation holds all
    from paper_2501_08547_b200 import workload

    gds = graphstore.SyntheticGraph(20000, 10.0, 2.1, 32, seed=3)
    for kind, kw in (("sage_mean", {}), ("gat", {}), ("gcn", {})):
        model = models.make_model(kind, 3, 32, 16, **kw)
        w = models.init_weights(model, 5)
        spe = graphstore.SyntheticPe([16, 16], seed=7)
        cfg = runtime.ServeConfig(strategy="srpe-cgp", gamma=0.2, num_partitions=P, seed=11, device=local)
        eng = runtime.distributed_engine(gds, spe, model, w, cfg)
        emu = runtime.ServingEngine(gds, spe, model, w, cfg)
        info = eng.graph_info()
        rows = torch.tensor([info["local_rows"], info["local_edges"]], dtype=torch.int64)
        dist.all_reduce(rows)
        reqs_l = []
        for seed in (1, 2):
            req = workload.make_request_synthetic(gds.num_nodes, gds.avg_degree, gds.exponent, 32, 256, seed)
            reqs_l.append(req)
            emb, bd = eng.serve(req)
            emb_emu, _ = emu.serve(req)
            if rank == 0:
                results.append(dict(case=f"generated.s{seed}", kind=kind, k=3, err_ref=max_rel_err(emb, emb_emu),
                                    err_emu=max_rel_err(emb, emb_emu), shard=True,
                                    partitioned=bool(info["local_rows"] < gds.num_nodes
                                                     and int(rows[0]) == gds.num_nodes
                                                     and int(rows[1]) == info["num_edges"]),
                                    coll_bytes=int(bd.collective_bytes)))
        if kind == "sage_mean":  # request lanes: each lane has its own NVLink exchange
            one = [eng.serve(r)[0] for r in reqs_l * 2]
            eng.set_lanes(2)
            two = [x[0] for x in eng.serve_stream(reqs_l * 2, depth=4)]
            eng.set_lanes(1)
            if rank == 0:
                results.append(dict(case="lanes", kind=kind, k=3, err_ref=0.0 if all(
                    np.array_equal(a, b) for a, b in zip(one, two)) else 1.0, err_emu=0.0, shard=True,
                    coll_bytes=0))
        eng.close()
        emu.close()
    # a peer that stops serving: the waiting rank times out (OB_CGP_TIMEOUT_MS), raises
    # TransportError and poisons the peer's flags, so the late rank fails too instead of
    # reading regions that were overwritten; afterwards both engines refuse requests
    from paper_2501_08547_b200._native import TransportError

    os.environ["OB_CGP_TIMEOUT_MS"] = "300"
    g = load_golden("small_s3")
    N, F = int(g["N"]), g["feats"].shape[1]
    ds = graphstore.GraphDataset(N, g["offsets"], g["nbrs"], g["feats"], np.ones(N, bool), np.zeros(N, bool))
    req = ServingRequest(N, int(g["B"]), g["qfeat"], g["edges"])
    model = models.make_model("sage_mean", 3, F, 6)
    w = models.Weights(golden_weights(g, "w.sage_mean.k3", "sage_mean", 3))
    pe = graphstore.PeStore([g[f"pe.sage_mean.k3.l{l}"] for l in (1, 2)])
    cfg = runtime.ServeConfig(strategy="srpe-cgp", gamma=0.5, num_partitions=P, seed=11, device=local)
    eng = runtime.distributed_engine(ds, pe, model, w, cfg)
    eng.serve(req)  # both ranks in step
    outcome = []

    def attempt():
        try:
            eng.serve(req)
            return "ok"
        except TransportError:
            return "transport"

    if rank == 0:
        outcome.append(attempt())  # rank 1 is not serving this one: timeout
    dist.barrier()
    if rank != 0:
        outcome.append(attempt())  # behind by one request, flags poisoned by rank 0
    dist.barrier()
    outcome.append(attempt())  # both engines refuse further requests
    eng.close()
    os.environ.pop("OB_CGP_TIMEOUT_MS", None)
    got = [None] * P
    dist.all_gather_object(got, outcome)
    if rank == 0:
        results.append(dict(case="peer_timeout", kind="sage_mean", k=3,
                            err_ref=0.0 if all(o == ["transport", "transport"] for o in got) else 1.0,
                            err_emu=0.0, shard=True, coll_bytes=0, outcome=got))
    if rank == 0:
        worst = max(r["err_ref"] for r in results)
        ok = worst <= 1e-4 and all(r["shard"] for r in results) and all(
            r.get("partitioned", True) for r in results)
        print(json.dumps(dict(ok=ok, P=P, cases=len(results), worst_err=worst, results=results[:4] + results[-1:])))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
