"""Serving benchmark: p50/p99 query-batch latency and queries/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

Workload (BASELINE.json configs[1], the largest single-GPU config): 3-layer
GraphSAGE-mean on the Reddit-shaped synthetic graph (233K nodes, 103.6M
edges after the 25% test hold-out, 602-d features, hidden 128), B = 1024
query batches, SRPE ratio policy gamma = 0.1.  The graph, hold-out pool,
requests and weights are the reference generator's own (bit-identical numpy
streams, seeds from SURVEY.md 8(d)); PE comes from the GPU precompute.

One step = one query batch through ServingEngine: selection, graph
construction and all three layers.  ``value`` times the device path with the
request already in HBM (every request replays the one CUDA graph captured for
the reserved request shape); ``e2e`` times the public host-pointer API (pinned
request H2D + D2H of the B x 128 rows inside the region).  L2 is flushed
(512 MB write) before every timed step.  A second, eager pass over the same
requests with per-kernel CUDA events gives the roofline and kernel split.

Under torchrun (N > 1) the default is independent replicas: every rank holds
the whole graph and serves its own request stream (query batches are
independent units, no data-path collective; weak scaling, time = max over
ranks).  ``--parallel cgp`` runs computation-graph parallelism instead: the
graph is hash-partitioned over a group of ``--cgp-size`` GPUs, every rank
aggregates the part of each batch whose sources it owns and partials meet at
the owners over NVLink (peer-mapped exchange buffers); N / size groups serve
independent request streams side by side -- DESIGN.md "Multi-GPU".  The
papers-shaped ``--config cfg4`` (111M nodes, 1.6B edges, generated on the
GPUs) runs only this way, with groups of 2 by default.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

# before any CUDA context: 32 hardware work queues for the engine's per-lane streams
# (paper_2501_08547_b200/__init__.py sets the same default)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, avg_degree, F, kind, k, hidden, B, gamma, description)
    "cfg1": (100_000, 20.0, 64, "gcn", 2, 64, 256, 0.1,
             "2-layer GCN, 100K-node/2M-edge power-law graph, F=64, B=256, SRPE ratio 0.1"),
    "cfg2": (233_000, 493.0, 602, "sage_mean", 3, 128, 1024, 0.1,
             "3-layer GraphSAGE-mean, Reddit-shaped 233K nodes / 103.6M edges, F=602, H=128, B=1024, SRPE ratio 0.1"),
    "cfg3": (2_400_000, 26.0, 100, "gat", 3, 128, 1024, 0.1,
             "3-layer GAT, ogbn-products-shaped 2.4M nodes / 55.9M edges, F=100, H=128, B=1024, SRPE ratio 0.1"),
    # BASELINE configs[3]: generated on the GPUs (ob_generate_graph), partitioned by CGP; N >= 2 only
    "cfg4": (111_059_956, 14.55, 128, "sage_mean", 3, 128, 1024, 0.1,
             "3-layer GraphSAGE-mean, ogbn-papers100M-shaped 111M nodes / ~1.6B edges generated on the GPUs, "
             "F=128, H=128, B=1024, SRPE ratio 0.1, CGP-partitioned"),
    # BASELINE configs[4] (gamma from PAPER.md:560-561): Yelp / Amazon shapes, H = 512;
    # run with --strategy full | srpe | sampled (and --parallel cgp at N > 1) for the ablation
    "cfg5-yelp-gcn": (717_000, 19.5, 300, "gcn", 2, 512, 1024, 0.20,
                      "2-layer GCN, Yelp-shaped 717K nodes / ~14M edges, F=300, H=512, B=1024, SRPE ratio 0.2"),
    "cfg5-yelp-gat": (717_000, 19.5, 300, "gat", 3, 512, 1024, 0.07,
                      "3-layer GAT, Yelp-shaped 717K nodes / ~14M edges, F=300, H=512, B=1024, SRPE ratio 0.07"),
    "cfg5-amazon-gcn": (1_600_000, 165.0, 200, "gcn", 2, 512, 1024, 0.03,
                        "2-layer GCN, Amazon-shaped 1.6M nodes / ~264M edges, F=200, H=512, B=1024, SRPE ratio 0.03"),
    "cfg5-amazon-gat": (1_600_000, 165.0, 200, "gat", 3, 512, 1024, 0.01,
                        "3-layer GAT, Amazon-shaped 1.6M nodes / ~264M edges, F=200, H=512, B=1024, SRPE ratio 0.01"),
}
SYNTHETIC = {"cfg4"}  # device-generated graph + synthetic stored embeddings (never on the host)
METRIC = "queries/s (B-query batches, p50/p99 batch latency in ms alongside)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def make_inputs(cfg, rank, world, n_req, seed_base=3, same_requests=False, stream_id=None):
    """Reference-generator graph + requests; rank 0 builds, others map the same files."""
    from paper_2501_08547_b200 import workload
    from paper_2501_08547_b200.graphstore import GraphDataset

    n, avg, F, kind, k, H, B, gamma, _ = CONFIGS[cfg]
    shm = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
    path = os.path.join(shm, f"omega_bench_{cfg}")
    t0 = time.time()
    if rank == 0 or world == 1:
        full = workload.gen_powerlaw_graph(n, avg, 2.1, F, seed=1)
        serving, pool = workload.split_holdout(full, 0.25, seed=1)
        del full
        if world > 1:
            np.savez(path, off=serving.in_offsets, nb=serving.in_neighbors, feats=serving.features,
                     ids=pool.ids, inc=pool.incident_edges)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        if rank != 0:
            z = np.load(path + ".npz", mmap_mode="r")
            serving = GraphDataset(n, z["off"], z["nb"], z["feats"], np.ones(n, bool), np.zeros(n, bool))
            removed = np.zeros(n, bool)
            removed[z["ids"]] = True
            pool = workload.HoldoutPool(z["ids"], removed, serving.features[z["ids"]], z["inc"])
    log(f"[bench] rank {rank}: graph ready in {time.time() - t0:.1f}s (E={serving.num_edges})")
    rs = (stream_id or 0) if same_requests else rank  # CGP: a group's ranks serve the same request stream
    reqs = [workload.make_request(pool, serving, B, seed=seed_base + 1000 * rs + i) for i in range(n_req)]
    return serving, pool, reqs


class Clocks:
    """NVML sampler (every 2 ms) running during the timed region: SM clock and throttle reasons."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown"}

    def __init__(self, device):
        import threading

        self.samples, self.reasons, self.max_mhz = [], set(), 0
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device]) if vis and vis.split(",")[device].isdigit() else device
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, nm in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        if self.h is None:
            return None
        self._stop.set()
        self.t.join()
        if not self.samples:
            return None
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


class NvlinkCounter:
    """NVML NVLink data counters of this rank's GPU (cumulative KiB, all links): bytes sent and received
    between two reads, so the exchange's real NVLink traffic can sit next to its computed bytes."""

    TX, RX = 138, 139  # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX

    def __init__(self, device):
        self.h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device]) if vis and vis.split(",")[device].isdigit() else device
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.links = [l for l in range(18) if self._link_ok(l)]
        except Exception:
            self.h = None

    def _link_ok(self, l):
        try:
            return self.nv.nvmlDeviceGetNvLinkState(self.h, l) == 1
        except Exception:
            return False

    def read(self):
        if self.h is None or not self.links:
            return None
        ids = [(f, l) for l in self.links for f in (self.TX, self.RX)]
        try:
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, ids)
        except Exception:
            return None
        if not any(v.nvmlReturn == 0 for v in vals):
            return None  # NOT_SUPPORTED on these boxes (profiles/r02/n2/nvml_nvlink_probe.txt)
        tx = sum(int(v.value.ullVal) for v, (f, _) in zip(vals, ids) if f == self.TX and v.nvmlReturn == 0)
        rx = sum(int(v.value.ullVal) for v, (f, _) in zip(vals, ids) if f == self.RX and v.nvmlReturn == 0)
        return tx * 1024, rx * 1024


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def ncu_traffic(cfg, key="dram_bytes_per_launch"):
    """dram bytes per launch (averaged over one request's launches, like roofline.achieved) of the
    aggregation kernel from the committed ncu capture of this config, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_agg_traffic.json")) as f:
            return json.load(f).get(cfg, {}).get(key)
    except Exception:
        return None


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def ref_gnnserve():
    """The unmodified reference package (pip-installed into baseline/_ref), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "gnnserve")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import gnnserve.graphstore
    import gnnserve.models
    import gnnserve.runtime
    import gnnserve.compgraph

    return gnnserve


def ref_sample(gn, serving, pe_layers, pool, cfg, budget_s=12.0, batch=16, max_requests=None, seed=777):
    """The reference's own ServingEngine.serve (gnnserve, runtime.py:308-335) on bounded sub-batches of
    the same workload: same graph, stored embeddings and weights (init_weights(seed=2), the reference's
    own), requests drawn from the same hold-out pool by make_request."""
    from paper_2501_08547_b200 import workload

    n, avg, F, kind, k, H, B, gamma, _ = CONFIGS[cfg]
    G, M, R, CG = gn.graphstore, gn.models, gn.runtime, gn.compgraph
    ds = G.GraphDataset(serving.num_nodes, serving.in_offsets, serving.in_neighbors, serving.features,
                        np.ones(serving.num_nodes, bool), np.zeros(serving.num_nodes, bool))
    model = M.make_model(kind, k, F, H)
    eng = R.ServingEngine(ds, G.PeStore(pe_layers), model, M.init_weights(model, 2),
                          R.ServeConfig(strategy="srpe", gamma=gamma))
    done, t_all, lat = 0, 0.0, []
    while True:
        r = workload.make_request(pool, serving, batch, seed=seed + done)
        req = CG.ServingRequest(r.num_base, r.num_queries, r.query_features, r.edges)
        t0 = time.perf_counter()
        eng.serve(req)
        dt = time.perf_counter() - t0
        lat.append(dt * 1e3)
        t_all += dt
        done += 1
        if t_all >= budget_s or (max_requests and done >= max_requests):
            break
    return batch * done / t_all, done, lat


def port_sample(serving, pe_layers, model, weights, pool, cfg, budget_s=12.0, batch=16, seed=777):
    """The oracle (numpy/scipy port of the reference) on bounded sub-batches of the same workload."""
    from oracle import layers as OL
    from paper_2501_08547_b200 import workload

    n, avg, F, kind, k, H, B, gamma, _ = CONFIGS[cfg]
    specs = [dict(kind=s.kind, in_dim=s.in_dim, out_dim=s.out_dim, p=s.p, n=s.n) for s in model.layers]
    done, q, t_all, lat = 0, 0, 0.0, []
    while True:
        req = workload.make_request(pool, serving, batch, seed=seed + done)
        t0 = time.perf_counter()
        OL.serve("srpe", specs, weights.layers, serving.num_nodes, batch, serving.in_offsets, serving.in_neighbors,
                 serving.features, req.query_features, req.edges, pe_layers=pe_layers, gamma=gamma)
        dt = time.perf_counter() - t0
        lat.append(dt * 1e3)
        t_all += dt
        q += batch
        done += 1
        if t_all >= budget_s:
            break
    return q / t_all, done, lat


def parity_check(eng, serving, pe_layers, model, weights, req, gamma, k):
    """One of the timed B-query requests through the public host API, checked against the oracle:
    plan (ids, nq, totals, fp64 score bits, targets), every block array and the fetch bytes bit-exact,
    embeddings by max|a-r|/max|r| (north_star bar 1e-4).  The oracle's wall time is the port's
    full-batch CPU time (same request, same config)."""
    from oracle import layers as OL

    specs = [dict(kind=s.kind, in_dim=s.in_dim, out_dim=s.out_dim, p=s.p, n=s.n) for s in model.layers]
    emb, bd = eng.serve(req)
    t0 = time.perf_counter()
    ref = OL.serve("srpe", specs, weights.layers, serving.num_nodes, req.num_queries, serving.in_offsets,
                   serving.in_neighbors, serving.features, req.query_features, req.edges, pe_layers=pe_layers,
                   gamma=gamma)
    t_port = time.perf_counter() - t0
    plan, rp = eng.last_plan(), ref["plan"]
    eq = all(np.array_equal(plan[f], rp[f]) for f in ("ids", "nq", "total", "targets"))
    eq = eq and np.array_equal(plan["scores"].view(np.uint64), rp["scores"].view(np.uint64))
    fields = ("src_ids", "dst_ids", "edge_src", "edge_dst", "bind_kind", "bind_pe_layer", "src_degree",
              "dst_self_src")
    for l in range(1, k + 1):
        got, exp = eng.last_block(l), ref["blocks"][l - 1]
        for f in fields:
            eq = eq and np.array_equal(np.asarray(getattr(got, f)).astype(np.int64),
                                       np.asarray(getattr(exp, f)).astype(np.int64))
    eq = eq and int(bd.fetch_bytes) == int(ref["fetch_bytes"])
    err = OL.max_rel_err(emb, ref["emb"])
    return {"request": "the first timed request (B=%d, m=%d)" % (req.num_queries, req.edges.shape[0]),
            "structure_equal": bool(eq), "max_rel_err": float(err), "tolerance": 1e-4,
            "checked": "candidates/nq/totals/score bits/targets, all 8 arrays of every block, fetch bytes; "
                       "embeddings vs oracle (numpy/scipy fp64 restatement of gnnserve)"}, t_port


def run_reference(args):
    """--impl reference: the reference's own CPU path (gnnserve from baseline/_ref; the oracle port when
    it is not installed), rank 0 only, all host cores numpy uses."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2501_08547_b200 import models

    cfg = args.config
    n, avg, F, kind, k, H, B, gamma, desc = CONFIGS[cfg]
    if cfg in SYNTHETIC:
        print(json.dumps({"impl": "reference", "unavailable": f"{cfg}: the ~1.6B-edge graph exists only on the GPUs "
                                                             "(generated per rank); the CPU reference cannot hold it"}))
        return
    serving, pool, _ = make_inputs(cfg, 0, 1, 0)
    model = models.make_model(kind, k, F, H)
    w = models.init_weights(model, 2)
    rng = np.random.default_rng(9)
    # stored embeddings: value-independent for timing (the reference's precompute would need E x F float64
    # temporaries), so fabricated N(0, 0.01) rows of the right shape
    pe = [rng.standard_normal((serving.num_nodes, H)).astype(np.float32) * 0.1 for _ in range(k - 1)]
    batch = args.ref_batch
    gn = ref_gnnserve()
    if gn is not None:
        kind_ = "reference"
        what = "gnnserve.runtime.ServingEngine.serve (the unmodified reference, baseline/_ref)"
        one = lambda i: ref_sample(gn, serving, pe, pool, cfg, budget_s=0.0, batch=batch, seed=777 + 100 * i)
    else:
        kind_ = "port"
        what = "numpy/scipy port of the reference (oracle/); baseline/_ref not installed"
        one = lambda i: port_sample(serving, pe, model, w, pool, cfg, budget_s=0.0, batch=batch, seed=777 + 100 * i)
    for i in range(min(args.warmup, 1)):
        one(1000 + i)
    lat = []
    t_total, q_total = 0.0, 0
    for i in range(args.steps):
        v, nr, l = one(i)
        lat += l
        t_total += sum(l) / 1e3
        q_total += batch * nr
    value = q_total / t_total
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_total * 1e3 / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "sample_batch": batch, "policy": "ratio", "gamma": gamma},
        "p50_ms": float(np.percentile(lat, 50)), "p99_ms": float(np.percentile(lat, 99)),
        "cpu_baseline": {"value": round(value, 3), "unit": "queries/s", "cores": os.cpu_count(), "kind": kind_,
                         "sample": f"{args.steps} requests of {batch} queries each (bounded sub-batches of the "
                                   f"{cfg} workload, same graph and weights, fabricated stored rows); {what}; "
                                   f"numpy free to use every host core"},
        "e2e": {"value": round(value, 3), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--gamma", type=float, default=None)
    ap.add_argument("--strategy", default="srpe", choices=["srpe", "full", "sampled"],
                    help="single-GPU / replica strategy (CGP runs srpe-cgp); config 5's ablation axis")
    ap.add_argument("--policy", default="ratio", choices=["ratio", "is", "random"],
                    help="SRPE scoring policy (policy.py:29-32)")
    ap.add_argument("--lanes", type=int, default=4,
                    help="request lanes for the throughput pass (1 = one request at a time)")
    ap.add_argument("--fanouts", default="15,10,5",
                    help="sampled strategy: comma-separated fanouts, outermost hop first (trimmed to k)")
    ap.add_argument("--ref-batch", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--parallel", default=None, choices=["cgp", "replicas"],
                    help="N > 1: independent replicas (default) or computation-graph parallelism")
    ap.add_argument("--cgp-size", type=int, default=None,
                    help="GPUs per CGP group (default: all for cfg1-3, 2 for cfg4); N / size groups serve "
                         "independent request streams")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2501_08547_b200 import models, runtime

    cfg = args.config
    n, avg, F, kind, k, H, B, gamma, desc = CONFIGS[cfg]
    if args.gamma is not None:
        gamma = args.gamma
    strategy = args.strategy
    fanouts = tuple(int(f) for f in args.fanouts.split(","))[-k:] if strategy == "sampled" else None
    nreq = args.warmup + args.steps
    synthetic = cfg in SYNTHETIC
    mode = args.parallel or ("cgp" if synthetic and world > 1 else ("replicas" if world > 1 else "single"))
    cgp = mode == "cgp" and world > 1
    if synthetic and not cgp:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "unavailable": f"{cfg} needs --parallel cgp on >= 2 GPUs "
                                                               "(one B200 cannot hold its graph + stored rows)"}))
        return
    P = (args.cgp_size or (2 if synthetic else world)) if cgp else 1
    if cgp and (P < 2 or world % P):
        raise SystemExit(f"--cgp-size {P} must be >= 2 and divide the world size {world}")
    groups = world // P if cgp else world
    my_group = rank // P if cgp else rank
    pg = None
    if cgp and groups > 1:  # every rank creates every group, then keeps its own
        import torch.distributed as dist

        pgs = [dist.new_group(list(range(g * P, (g + 1) * P))) for g in range(groups)]
        pg = pgs[my_group]
    if synthetic:
        from paper_2501_08547_b200 import graphstore, workload

        serving = graphstore.SyntheticGraph(n, avg, 2.1, F, seed=1)
        pool = None
        reqs = [workload.make_request_synthetic(n, avg, 2.1, F, B, seed=3 + 1000 * my_group + i) for i in range(nreq)]
        pe_src = graphstore.SyntheticPe([H] * (k - 1), seed=2)
    else:
        serving, pool, reqs = make_inputs(cfg, rank, world, nreq, same_requests=cgp, stream_id=my_group)
        pe_src = None
    model = models.make_model(kind, k, F, H)
    w = models.init_weights(model, 2)
    stream = torch.cuda.Stream(device=local)
    t0 = time.time()
    if cgp:
        scfg = runtime.ServeConfig(strategy="srpe-cgp", gamma=gamma, num_partitions=P, seed=0, device=local,
                                   policy=args.policy)
        eng = runtime.distributed_engine(serving, pe_src, model, w, scfg, stream=stream.cuda_stream, group=pg)
    else:
        scfg = runtime.ServeConfig(strategy=strategy, gamma=gamma, device=local, fanouts=fanouts,
                                   policy=args.policy)
        eng = runtime.ServingEngine(serving, pe_src, model, w, scfg, stream=stream.cuda_stream)
    if not synthetic and (cgp or strategy == "srpe"):
        eng.precompute_pe()
    info = eng.graph_info()
    log(f"[bench] rank {rank}: engine loaded in {time.time() - t0:.1f}s ({info})")
    lib = eng._lib
    ms = np.array([r.edges.shape[0] for r in reqs])
    from paper_2501_08547_b200 import _native as nat

    # plan requests at the p90 edge count (one captured graph serves them); larger ones take
    # their own bucket's graph, captured during warm-up below
    nat.check(lib.ob_reserve(eng._h, B, int(np.percentile(ms, 90))))
    above = sorted(set(int(np.argmax(ms == v)) for v in np.unique(ms) if v > np.percentile(ms, 90)),
                   key=lambda i: -ms[i])
    dev = torch.device("cuda", local)
    d_edges = [torch.from_numpy(r.edges).to(dev) for r in reqs]
    d_q = [torch.from_numpy(r.query_features).to(dev) for r in reqs]
    d_out = torch.empty((B, H), dtype=torch.float32, device=dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def step(i):
        eng.serve_device(B, d_q[i].data_ptr(), d_edges[i].shape[0], d_edges[i].data_ptr(), d_out.data_ptr())

    with torch.cuda.stream(stream):
        for i in above:  # largest first: the arena reaches its final size before any capture we keep
            step(i)  # capture the graphs of the above-bound buckets outside the timed region
        for i in range(args.warmup):
            step(i)
    stream.synchronize()
    # correctness guard on a warm request: errors surface here, not silently
    bd0 = eng.serve_device(B, d_q[0].data_ptr(), d_edges[0].shape[0], d_edges[0].data_ptr(), d_out.data_ptr(),
                           sync=True)

    def timed_pass(profile):
        """K requests, L2 flushed before each, device events around each request."""
        if profile:
            nat.check(lib.ob_profile(eng._h, 1))
        ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        l0 = eng.launch_count()
        clocks = Clocks(local)
        with torch.cuda.stream(stream):
            for j in range(args.steps):
                flush.fill_(j & 0xFF)  # evict L2 (512 MB > 126 MB) outside the timed events
                ev_s[j].record(stream)
                step(args.warmup + j)
                ev_e[j].record(stream)
        stream.synchronize()
        torch.cuda.synchronize()
        clk_ = clocks.stop()
        if world > 1:
            torch.distributed.barrier()
        lat_ = np.array([ev_s[j].elapsed_time(ev_e[j]) for j in range(args.steps)])
        return lat_, eng.launch_count() - l0, clk_

    # headline: every request replays the one captured graph (ob_reserve planned the shape)
    lat, launches, clk = timed_pass(profile=False)
    total_ms = float(lat.sum())
    # roofline: the same requests again, launched eagerly with per-kernel events
    lat_eager, _, _ = timed_pass(profile=True)
    agg = _read_prof(lib, eng, nat, 0)
    gemm = _read_prof(lib, eng, nat, 1)
    fin = _read_prof(lib, eng, nat, 2)
    reqp = _read_prof(lib, eng, nat, 6)  # minus the profiler's own row-count kernels (class 9)
    prof_count_ms = _read_prof(lib, eng, nat, 9)["ms"]
    st = {name: _read_prof(lib, eng, nat, cls) for name, cls in
          (("select", 4), ("request_csr", 7), ("build", 3), ("resolve", 5), ("collectives", 8))}
    nat.check(lib.ob_profile(eng._h, 0))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    served = groups * B  # CGP: the P ranks of a group serve one batch together
    value_single = served * args.steps / (total_ms / 1e3)
    value, lanes_ms, launches_lanes, clk_lanes = value_single, None, None, None
    nvl_measured = None
    lanes = 1 if args.lanes < 2 else args.lanes
    if lanes > 1:
        # throughput with two request lanes: consecutive requests alternate between two request
        # workspaces on two streams, so one's graph construction overlaps the other's gathers.
        # No L2 flush inside this pass (it would serialise the lanes): each request gathers
        # > 0.5 GB of rows, far more than the 126 MB L2.
        eng.set_lanes(lanes)
        with torch.cuda.stream(stream):
            for i in above + list(range(args.warmup)):  # every shape's graph on every lane, outside the region
                for _ in range(lanes):
                    step(i)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        nvl = NvlinkCounter(local) if cgp else None
        nvl0 = nvl.read() if nvl else None
        clocks = Clocks(local)
        l0 = eng.launch_count()
        with torch.cuda.stream(stream):
            a.record(stream)
            nat.check(lib.ob_lanes_fork(eng._h))
            for j in range(args.steps):
                step(args.warmup + j)
            nat.check(lib.ob_lanes_join(eng._h))
            b.record(stream)
        torch.cuda.synchronize()
        clk_lanes = clocks.stop()
        nvl1 = nvl.read() if nvl else None
        ok_nvl = torch.tensor([1 if (nvl0 is not None and nvl1 is not None) else 0], device=dev)
        if world > 1:
            torch.distributed.all_reduce(ok_nvl, op=torch.distributed.ReduceOp.MIN)  # every rank or none
        if int(ok_nvl.item()):
            t = torch.tensor([float(nvl1[0] - nvl0[0]), float(nvl1[1] - nvl0[1])], device=dev)
            torch.distributed.all_reduce(t)  # every rank's counters
            nvl_measured = {"tx_bytes": int(t[0].item()), "rx_bytes": int(t[1].item()), "steps": args.steps,
                            "per_step_bytes": int(t[1].item() / args.steps / max(groups, 1)),
                            "source": "NVML NVLink data counters (all links, all ranks) around the throughput pass"}
        launches_lanes = eng.launch_count() - l0
        lanes_ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([lanes_ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            lanes_ms = float(t.item())
        value = served * args.steps / (lanes_ms / 1e3)

    # end to end through the public host-pointer API (pinned buffers, H2D + D2H inside the region).
    # Request edges cross PCIe as int32 (src, dst) pairs (ob_serve_i32 / ob_serve_submit_i32: N + B < 2^31,
    # widened on the device), the int64 path of the reference's own array type is measured beside it.
    e2e = None
    if not args.no_e2e:
        import ctypes as C

        pin_e64 = [torch.from_numpy(r.edges).pin_memory() for r in reqs]
        pin_e32 = [torch.from_numpy(r.edges.astype(np.int32)).pin_memory() for r in reqs]
        pin_q = [torch.from_numpy(r.query_features).pin_memory() for r in reqs]
        out_h = torch.empty((B, H), dtype=torch.float32).pin_memory()
        depth = 4 if lanes > 1 else 2  # requests in flight on the pipelined path
        outs_p = [torch.empty((B, H), dtype=torch.float32).pin_memory() for _ in range(depth)]

        def e2e_pass(i32):
            serve_fn = lib.ob_serve_i32 if i32 else lib.ob_serve
            submit_fn = lib.ob_serve_submit_i32 if i32 else lib.ob_serve_submit
            pin_e = pin_e32 if i32 else pin_e64
            e2e_ms, h2d, d2h = [], 0, 0
            bd = nat.ObBreakdown()  # host-path calls capture their own graphs (output buffer differs)
            for i in above + [0]:
                nat.check(serve_fn(eng._h, B, C.c_void_p(pin_q[i].data_ptr()), pin_e[i].shape[0],
                                   C.c_void_p(pin_e[i].data_ptr()), C.c_void_p(out_h.data_ptr()), C.byref(bd)))
            for j in range(args.steps):
                i = args.warmup + j
                flush.fill_(j & 0xFF)
                torch.cuda.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                bd = nat.ObBreakdown()
                nat.check(serve_fn(eng._h, B, C.c_void_p(pin_q[i].data_ptr()), pin_e[i].shape[0],
                                   C.c_void_p(pin_e[i].data_ptr()), C.c_void_p(out_h.data_ptr()), C.byref(bd)))
                b.record(stream)
                b.synchronize()
                e2e_ms.append(a.elapsed_time(b))
                h2d += bd.h2d_bytes
                d2h += bd.d2h_bytes
            et = float(np.sum(e2e_ms))

            # pipelined: the same requests through submit / wait (depth in flight), so request t+1's
            # inputs cross PCIe and t-1's rows return while t runs; every step still copies its inputs
            # H2D from pinned memory and its rows D2H inside the timed region
            def submit(i, slot):
                t = C.c_int64()
                nat.check(submit_fn(eng._h, B, C.c_void_p(pin_q[i].data_ptr()), pin_e[i].shape[0],
                                    C.c_void_p(pin_e[i].data_ptr()), C.c_void_p(outs_p[slot].data_ptr()),
                                    C.byref(t)))
                return t.value

            def wait(t):
                bdw = nat.ObBreakdown()
                nat.check(lib.ob_serve_wait(eng._h, t, C.byref(bdw)))
                return bdw

            for i in above + [0]:  # every slot's (lane's) graph captured before timing
                for sl in range(4):
                    wait(submit(i, sl % depth))
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            t_sub, t_done, pend = {}, {}, []
            p0 = time.perf_counter()
            for j in range(args.steps):
                if len(pend) == depth:
                    tk, jj = pend.pop(0)
                    wait(tk)
                    t_done[jj] = time.perf_counter()
                t_sub[j] = time.perf_counter()
                pend.append((submit(args.warmup + j, j % depth), j))
            for tk, jj in pend:
                wait(tk)
                t_done[jj] = time.perf_counter()
            pt = (time.perf_counter() - p0) * 1e3
            if world > 1:
                t = torch.tensor([pt, et], device=dev)
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                pt, et = float(t[0].item()), float(t[1].item())
            plat = [(t_done[j] - t_sub[j]) * 1e3 for j in range(args.steps)]
            return {"value": round(served * args.steps / (pt / 1e3), 3), "unit": "queries/s",
                    "h2d_bytes_per_step": int(h2d // args.steps), "d2h_bytes_per_step": int(d2h // args.steps),
                    "p50_ms": float(np.percentile(plat, 50)), "p99_ms": float(np.percentile(plat, 99)),
                    "sync": {"value": round(served * args.steps / (et / 1e3), 3), "unit": "queries/s",
                             "mode": "one synchronous call per step (H2D, request, D2H, synchronise), CUDA events, "
                                     "L2 flushed before each step",
                             "p50_ms": float(np.percentile(e2e_ms, 50)), "p99_ms": float(np.percentile(e2e_ms, 99))}}

        e2e = e2e_pass(True)
        e2e["mode"] = (f"pipelined host API (ob_serve_submit_i32/ob_serve_wait, {depth} requests in flight over "
                       f"{lanes} request lane(s), pinned host buffers, request edges as int32 pairs); wall clock over "
                       "the K steps; no L2 flush (each request gathers > 0.5 GB)")
        e2e["int64_edges"] = e2e_pass(False)
        e2e["int64_edges"]["mode"] = "the same with int64 edge pairs (ob_serve_submit / ob_serve), 16 bytes per edge"

    cpu = None
    parity = None
    if synthetic:
        cpu = {"value": None, "unit": "queries/s", "cores": 0, "kind": "port",
               "sample": f"none: the {cfg} graph exists only on the GPUs; see the cfg2 line for the CPU baseline"}
    elif rank == 0 and world == 1 and not args.no_cpu and strategy == "srpe" and args.policy == "ratio":
        pe_host = [eng.read_pe(l) for l in range(1, k)]
        # served with the throughput configuration still set (request lanes, source-range passes)
        parity, t_port = parity_check(eng, serving, pe_host, model, w, reqs[args.warmup], gamma, k)
        gn = ref_gnnserve()
        port = {"value": round(B / t_port, 3), "unit": "queries/s", "cores": 1,
                "sample": f"1 request of {B} queries (the parity request above: the bench config itself)"}
        if gn is not None:
            qps, nr, cl = ref_sample(gn, serving, pe_host, pool, cfg, budget_s=12.0, batch=args.ref_batch)
            cpu = {"value": round(qps, 3), "unit": "queries/s", "cores": 1, "kind": "reference",
                   "sample": f"{nr} requests of {args.ref_batch} queries (bounded sub-batches of the {cfg} workload, "
                             f"same graph/stored rows/weights); gnnserve.runtime.ServingEngine.serve, the unmodified "
                             f"reference from baseline/_ref; its hot loops (np.add.at, Python loops) are single-core",
                   "port_full_batch": port}
        else:
            cpu = dict(port, kind="port")
            cpu["sample"] += "; numpy/scipy port of the reference (oracle/), baseline/_ref not installed"

    hbm, tf, which = peaks()
    agg_gbs = agg["bytes"] / (agg["ms"] / 1e3) / 1e9 if agg["ms"] > 0 else 0.0
    roof = {"bound": "hbm", "kernel": "k_agg (edge-chunk gather + segment reduce)",
            "achieved": round(agg_gbs, 1), "peak": hbm, "unit": "GB/s", "frac": round(agg_gbs / hbm, 4),
            "peak_source": which, "traffic": ncu_traffic(cfg),
            "traffic_live": ncu_traffic(cfg, "dram_bytes_per_launch_live"),
            "alg_bytes_per_launch": round(agg["bytes"] / max(agg["n"], 1)),
            "launches": agg["n"], "avg_launch_us": round(agg["ms"] * 1e3 / max(agg["n"], 1), 2),
            "gathered_row_gbs": round(agg["flops"] / (agg["ms"] / 1e3) / 1e9, 1) if agg["ms"] > 0 else None,
            "gather_ceiling_gbs": 15200.0,  # measured random 512-B row gather, L2-sized table (profiles/r01_gather_ceiling.md)
            "note": "k_agg is bound by the per-SM L2->SM return path, not HBM: rows are re-read once per "
                    "edge, ~70-80 % from L2 and ~30 % from L1 (gathered_row_gbs = the row bytes the launches "
                    "loaded, against the measured 15.2 TB/s random-row gather ceiling from L2; L1 hits lift it "
                    "above). traffic = cold ncu --set full DRAM bytes per launch, traffic_live = the same "
                    "without cache flushes between kernels. achieved counts algorithmic "
                    "bytes (each distinct row once): every launch its edge list, the distinct rows it loaded "
                    "and its partials -- the layer-1 launch (stored aggregates) the request-span sources' "
                    "rows, the layer-2 launch (delta aggregates) the delta rows of recomputed CSR sources "
                    "and the request-span sources' rows (distinct rows counted on the device by the "
                    "profiler's k_prof_rows, outside the timed events), the query-block launch every source "
                    "row",
            "share_of_step": round(agg["ms"] / max(reqp["ms"], 1e-9), 3)}
    # the whole request against HBM, with SURVEY.md 8(d)'s per-unit figure: bytes(G) =
    # graph_fetch_bytes(G) + sum_l 4 H_l D_l + 4 F B + 16 m per query batch, over the per-request
    # time of the throughput pass (lanes) -- the bytes the reference's path would move
    try:
        import ctypes as C

        outs_b = 0
        for l in range(1, k + 1):
            ns, nd, ne = C.c_int64(), C.c_int64(), C.c_int64()
            nat.check(lib.ob_last_block_sizes(eng._h, 0, l, C.byref(ns), C.byref(nd), C.byref(ne)))
            outs_b += 4 * model.layers[l - 1].out_dim * nd.value
        req0 = reqs[0]
        bytes_g = int(bd0.fetch_bytes) + outs_b + 4 * F * B + 16 * int(req0.edges.shape[0])
        # each GPU (a CGP group: P GPUs sharing one request) serves `steps` requests in the pass
        ms_req = (lanes_ms if lanes_ms is not None else total_ms) / args.steps
        gbs = bytes_g / (P if cgp else 1) / (ms_req / 1e3) / 1e9
        roof["request"] = {"bytes_per_request": bytes_g, "ms_per_request": round(ms_req, 4),
                           "achieved": round(gbs, 1), "frac": round(gbs / hbm, 4), "unit": "GB/s per GPU",
                           "definition": "SURVEY.md 8(d) bytes(G) of one request (divided over the P GPUs of a CGP "
                                         "group) over the throughput pass's time per request: every request stage, "
                                         "not one kernel"}
    except Exception as ex:  # pragma: no cover - reporting only
        roof["request"] = {"error": str(ex)[:200]}
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round((lanes_ms if lanes_ms is not None else total_ms) / args.steps, 4),
        "value_one_request_at_a_time": round(value_single, 3),
        "p50_ms": round(float(np.percentile(lat, 50)), 4), "p99_ms": round(float(np.percentile(lat, 99)), 4),
        "higher_is_better": True, "scaling": "strong" if (cgp and groups == 1) else "weak", "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": desc, "batch": B, "policy": args.policy, "gamma": gamma,
                   "strategy": "srpe-cgp" if cgp else strategy,
                   **({"fanouts": list(fanouts)} if fanouts else {}),
                   "parallelism": (f"cgp x{P} (NVLink exchange) x {groups} group(s)" if cgp else
                                   (f"replicas x{world}" if world > 1 else "single")),
                   "l2": ("latency pass (p50/p99): L2 flushed (512 MB write) before every step; throughput pass "
                          "(value) with request lanes: no flush, each request gathers > 0.5 GB (> L2)"),
                   "lanes": lanes,
                   "inputs": ("device generator (ob_generate_graph: the reference degree law, not its numpy "
                              "stream), synthetic N(0,1) stored embeddings, host-drawn request batches")
                   if synthetic else "reference generator (bit-identical numpy streams), PE from GPU precompute",
                   "graph": info},
        "roofline": roof,
        "eager_ms_per_step": round(float(lat_eager.mean()) - prof_count_ms / args.steps, 4),
        "kernels_ms_per_step": {"agg": round(agg["ms"] / args.steps, 4), "gemm": round(gemm["ms"] / args.steps, 4),
                                "finalize": round(fin["ms"] / args.steps, 4),
                                **{name: round(st[name]["ms"] / args.steps, 4) for name in st}},
        "gemm_tflops": round(gemm["flops"] / (gemm["ms"] / 1e3) / 1e12, 2) if gemm["ms"] > 0 and gemm["flops"] > 0
        else None,  # 2 M K N per launch whose M is a block counter (listed-row GEMMs count no flops: a lower bound)
        "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "clocks": clk_lanes or clk,
        "gpu_launches": int(launches_lanes if launches_lanes is not None else launches),
        "request": {"edges": int(reqs[0].edges.shape[0]), "candidates": int(bd0.num_candidates),
                    "targets": int(bd0.num_targets), "fetch_bytes": int(bd0.fetch_bytes),
                    "nvlink_bytes_per_step": int(bd0.collective_bytes) if cgp else 0,
                    **({"allgather_rows_bytes": int(bd0.allgather_bytes),
                        "nvlink_note": "per request of one CGP group, all ranks: the exchange's bytes from the "
                                       "request's actual destination counts; allgather_rows_bytes = the all-gather-"
                                       "of-source-rows alternative sum_l (P-1) S_l row_bytes_l",
                        "nvlink_measured": nvl_measured or "unavailable: NVML NVLink throughput counters return "
                                                           "NOT_SUPPORTED here"} if cgp else {})},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def _read_prof(lib, eng, nat, cls):
    import ctypes as C

    ms, n, by, fl = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
    nat.check(lib.ob_profile_read(eng._h, cls, C.byref(ms), C.byref(n), C.byref(by), C.byref(fl)))
    return {"ms": ms.value, "n": n.value, "bytes": by.value, "flops": fl.value}


if __name__ == "__main__":
    main()
