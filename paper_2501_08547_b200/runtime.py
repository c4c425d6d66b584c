"""Serving API: ``ServeConfig``, ``LatencyBreakdown``, ``ServingEngine``.

Drop-in for ``gnnserve/runtime.py:62-358``: same constructor, same
``serve(request) -> (emb[B, H_k] float32, LatencyBreakdown)`` contract, same
exception types.  Construction copies the dataset, stored embeddings and
weights into HBM once; ``serve`` ships only the request (edges + query
features) to the device and reads back the B x H_k rows.  Selection,
computation-graph construction and layer execution all run as sm_100a
kernels in ``libomega_b200.so`` (``_native``); there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .compgraph import ComputationBlock, ComputationGraph, ServingRequest
from .graphstore import GraphDataset, PeStore, SyntheticGraph, SyntheticPe
from .models import ModelSpec, Weights, weight_matrix_names

STRATEGIES = ("full", "sampled", "srpe", "srpe-cgp")
EDGE_BYTES = 16

METRICS_HEADER = (
    "request_id,strategy,batch,partitions,fetch_ms,transfer_ms,compute_ms,"
    "fetch_bytes,collective_bytes,total_ms"
)


@dataclass
class ServeConfig:
    """runtime.py:62-82 (plus the CUDA device ordinal)."""

    strategy: str = "full"
    fanouts: tuple | None = None
    gamma: float = 0.0
    policy: str = "ratio"
    num_partitions: int = 1
    cache_bytes: int = 0
    transport: str = "sim"
    bandwidth_bytes_per_s: float = 12e9
    seed: int = 0
    device: int = 0

    def __post_init__(self):
        if self.strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {self.strategy!r}")
        if self.strategy == "sampled" and not self.fanouts:
            raise ValueError("sampled strategy needs fanouts")
        if not 0.0 <= self.gamma <= 1.0:
            raise ValueError("gamma must lie in [0, 1]")
        if self.strategy == "srpe-cgp" and self.policy == "oracle":
            raise ValueError("oracle policy needs full embeddings; not available under cgp")


@dataclass
class LatencyBreakdown:
    """runtime.py:85-95; fetch/compute are device times of the request's stages."""

    fetch_ms: float = 0.0
    transfer_ms: float = 0.0
    compute_ms: float = 0.0
    collective_bytes: int = 0
    fetch_bytes: int = 0

    @property
    def total_ms(self) -> float:
        return self.fetch_ms + self.transfer_ms + self.compute_ms


def metrics_line(request_id, strategy, batch, partitions, bd: LatencyBreakdown) -> str:
    return (f"{request_id},{strategy},{batch},{partitions},{bd.fetch_ms:.3f},{bd.transfer_ms:.3f},"
            f"{bd.compute_ms:.3f},{bd.fetch_bytes},{bd.collective_bytes},{bd.total_ms:.3f}")


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for a one-process-per-GPU CGP group (call on rank 0, broadcast)."""
    buf = C.create_string_buffer(128)
    nat.check(nat.lib.ob_nccl_unique_id(buf))
    return buf.raw


def broadcast_nccl_id(make_id=nccl_unique_id, group=None) -> bytes:
    """The group's rank 0 draws the NCCL id and every rank of the torch.distributed group gets it.

    The bootstrap is plumbing only (the World of collectives.py:94-137); all
    data-path collectives run inside libomega_b200 on the engine's stream.
    """
    import torch.distributed as dist

    obj = [make_id() if dist.get_rank(group) == 0 else None]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    return bytes(obj[0])


def distributed_engine(dataset, pe, model, weights, config: ServeConfig, stream: int = 0,
                       group=None) -> "ServingEngine":
    """One CGP rank per process/GPU: rank and P from the torch.distributed group (default: the world).

    Several groups can serve side by side (data parallel over CGP groups): each
    group partitions its own copy of the graph over its P GPUs and has its own
    NCCL communicator and NVLink exchange.
    """
    import torch.distributed as dist

    size = dist.get_world_size(group)
    if config.strategy != "srpe-cgp" or config.num_partitions != size:
        raise ValueError("distributed_engine needs strategy='srpe-cgp' with num_partitions == group size")
    nid = broadcast_nccl_id(group=group)
    return ServingEngine(dataset, pe, model, weights, config, stream=stream, nccl_id=nid,
                         rank=dist.get_rank(group))


class ServingEngine:
    """Loaded dataset, stored embeddings and weights, resident on one B200."""

    def __init__(self, dataset: GraphDataset, pe: PeStore | None, model: ModelSpec, weights: Weights,
                 config: ServeConfig, stream: int = 0, nccl_id: bytes | None = None, rank: int = 0):
        """runtime.py:258-288.  The arguments are duck-typed: the reference's own ``GraphDataset``,
        ``PeStore``, ``ModelSpec``, ``Weights`` and ``ServeConfig`` objects are accepted unchanged
        (tests/test_gpu_dropin.py), as are this package's mirrors of them."""
        if config.strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {config.strategy!r}")
        if config.strategy == "sampled":  # build_sampled (compgraph.py:248-284)
            fan = [int(f) for f in config.fanouts]
            if any(f < 1 for f in fan):
                raise ValueError("fanouts must be >= 1")
            if len(fan) != model.k:
                raise ValueError("model depth does not match the computation graph")
            if max(fan) > nat.MAX_FANOUT:
                raise ValueError(f"fanouts above {nat.MAX_FANOUT} are not supported on the device")
        if config.policy not in nat.POLICY:
            raise ValueError(f"policy {config.policy!r} is not on the device path (ratio, is, random)")
        if getattr(config, "cache_bytes", 0):
            raise ValueError("feature caches are subsumed by HBM residency; use cache_bytes=0")
        self.dataset = dataset
        self.pe = pe
        self.model = model
        self.weights = weights
        self.config = config
        device = int(getattr(config, "device", 0))  # gnnserve's own ServeConfig has no device field
        cfg = nat.ObConfig(device=device, strategy=nat.STRATEGY[config.strategy], gamma=float(config.gamma),
                           policy=nat.POLICY[config.policy], num_partitions=int(config.num_partitions),
                           rank=int(rank), seed=int(config.seed) & 0xFFFFFFFFFFFFFFFF, stream=int(stream),
                           nccl_id=None)
        if config.strategy == "sampled":
            if len(config.fanouts) > nat.MAX_LAYERS:
                raise ValueError(f"at most {nat.MAX_LAYERS} layers")
            cfg.num_fanouts = len(config.fanouts)
            for i, f in enumerate(config.fanouts):
                cfg.fanouts[i] = int(f)
        self._id_buf = None
        if nccl_id is not None:
            self._id_buf = C.create_string_buffer(bytes(nccl_id), 128)
            cfg.nccl_id = C.cast(self._id_buf, C.c_void_p)
        h = C.c_void_p()
        nat.check(nat.lib.ob_engine_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._lib = nat.lib
        try:
            self._load(dataset, pe, model, weights)
        except BaseException:
            self.close()
            raise

    # -- loading ---------------------------------------------------------------
    def _load(self, ds, pe, model, weights):
        if isinstance(ds, SyntheticGraph):
            nat.check(self._lib.ob_generate_graph(self._h, int(ds.num_nodes), float(ds.avg_degree),
                                                  float(ds.exponent), int(ds.feature_dim),
                                                  int(ds.seed) & 0xFFFFFFFFFFFFFFFF))
        else:
            off = np.ascontiguousarray(ds.in_offsets, dtype=np.int64)
            nb = np.ascontiguousarray(ds.in_neighbors, dtype=np.int64)
            feats = _f32(ds.features)
            nat.check(self._lib.ob_load_graph(self._h, int(ds.num_nodes), nat.ptr(off), nat.ptr(nb),
                                              int(nb.shape[0]), nat.ptr(feats), int(feats.shape[1])))
        self._load_model(model, weights)
        self._load_pe(pe)

    def _load_model(self, model, weights):
        layers = (nat.ObLayer * model.k)()
        mats = []
        for i, spec in enumerate(model.layers):
            layers[i] = nat.ObLayer(nat.KIND_TAGS[spec.kind], spec.in_dim, spec.out_dim, float(spec.p), int(spec.n))
            for name in weight_matrix_names(spec.kind):
                mats.append(_f32(weights.layers[i][name]))
        arr = (C.c_void_p * len(mats))(*[m.ctypes.data for m in mats])
        nat.check(self._lib.ob_load_model(self._h, model.k, layers, arr))

    def _load_pe(self, pe):
        if isinstance(pe, SyntheticPe):
            for l, dim in enumerate(pe.dims, start=1):
                nat.check(self._lib.ob_generate_pe(self._h, l, int(dim), int(pe.seed) + l))
        elif pe is not None:
            if getattr(pe, "node_ids", None) is not None:
                raise ValueError("the engine needs a whole-graph stored-embedding store")
            for l in range(1, pe.num_layers + 1):
                rows = _f32(pe.layers[l - 1])
                nat.check(self._lib.ob_load_pe(self._h, l, nat.ptr(rows), int(rows.shape[0]), int(rows.shape[1])))

    def reload(self, model=None, weights=None, pe=None) -> None:
        """Replace the weights (model + weights) and/or the stored embeddings in place.

        Captured request graphs and the derived stored tables are dropped (after every in-flight
        request finished) and rebuilt on the next request, so later serves equal a fresh engine's.
        """
        if (model is None) != (weights is None):
            raise ValueError("reload the model and its weights together")
        if model is not None:
            self._load_model(model, weights)
            self.model, self.weights = model, weights
        if pe is not None:
            self._load_pe(pe)
            self.pe = pe

    def precompute_pe(self) -> None:
        """GPU precompute_embeddings into HBM (graphstore.py:330-365)."""
        nat.check(self._lib.ob_precompute_pe(self._h))

    def read_pe(self, layer: int) -> np.ndarray:
        dim = self.model.layers[layer - 1].out_dim
        out = np.empty((self.dataset.num_nodes, dim), dtype=np.float32)
        nat.check(self._lib.ob_read_pe(self._h, layer, nat.ptr(out)))
        return out

    # -- serving ---------------------------------------------------------------
    def _request_arrays(self, request: ServingRequest):
        if request.num_base != self.dataset.num_nodes:
            raise ValueError("request numbered against a different dataset")
        if self.config.strategy not in ("full", "sampled") and self.model.k < 2:
            raise ValueError("reuse graphs need k >= 2")
        B = int(request.num_queries)
        q = _f32(request.query_features)
        if q.shape != (B, self.dataset.feature_dim):
            raise ValueError("query features must be B x F")
        e = np.asarray(request.edges)
        e = np.ascontiguousarray(e if e.dtype == np.int32 else e.astype(np.int64, copy=False)).reshape(-1, 2)
        out = np.empty((B, self.model.layers[-1].out_dim), dtype=np.float32)
        return B, q, e, out

    def serve(self, request: ServingRequest) -> tuple[np.ndarray, LatencyBreakdown]:
        """runtime.py:308-358."""
        B, q, e, out = self._request_arrays(request)
        bd = nat.ObBreakdown()
        fn = self._lib.ob_serve_i32 if e.dtype == np.int32 else self._lib.ob_serve  # int32 pairs: half the PCIe bytes
        nat.check(fn(self._h, B, nat.ptr(q), int(e.shape[0]), nat.ptr(e), nat.ptr(out), C.byref(bd)))
        return out, self._breakdown(bd)

    def serve_stream(self, requests, depth: int = 2):
        """Pipelined serving over an iterable of requests: yields (emb, LatencyBreakdown) in order.

        Request t+1's inputs cross PCIe and request t-1's rows come back while
        request t runs on the device (ob_serve_submit / ob_serve_wait; up to
        ``depth`` <= 4 requests in flight, spread over the request lanes).  Each result equals ``serve(request)``'s; ``compute_ms``
        is the request's device time.
        """
        pending = []  # (ticket, out, keep-alive arrays)
        it = iter(requests)
        done = False
        try:
            while True:
                while not done and len(pending) < max(1, min(int(depth), 4)):
                    try:
                        req = next(it)
                    except StopIteration:
                        done = True
                        break
                    B, q, e, out = self._request_arrays(req)
                    t = C.c_int64()
                    fn = self._lib.ob_serve_submit_i32 if e.dtype == np.int32 else self._lib.ob_serve_submit
                    nat.check(fn(self._h, B, nat.ptr(q), int(e.shape[0]), nat.ptr(e), nat.ptr(out), C.byref(t)))
                    pending.append((t.value, out, (q, e)))
                if not pending:
                    return
                t, out, keep = pending[0]
                bd = nat.ObBreakdown()
                st = self._lib.ob_serve_wait(self._h, t, C.byref(bd))
                pending.pop(0)
                nat.check(st)
                yield out, self._breakdown(bd)
        finally:  # an error or an abandoned stream: retire what is still in flight
            for t, _, _ in pending:
                self._lib.ob_serve_wait(self._h, t, None)

    def _breakdown(self, bd) -> LatencyBreakdown:
        self.last_breakdown = bd
        parts = self.config.num_partitions if self.config.strategy == "srpe-cgp" else 1
        lb = LatencyBreakdown(
            fetch_ms=bd.fetch_ms,
            transfer_ms=bd.fetch_bytes / parts / self.config.bandwidth_bytes_per_s * 1e3,
            compute_ms=bd.compute_ms,
            collective_bytes=int(bd.collective_bytes),
            fetch_bytes=int(bd.fetch_bytes),
        )
        return lb

    def serve_device(self, num_queries: int, d_query_features: int, num_edges: int, d_edges: int, d_out: int,
                     sync: bool = False):
        """Request already in HBM (device pointers as ints); enqueue only unless sync."""
        bd = nat.ObBreakdown() if sync else None
        nat.check(self._lib.ob_serve_device(self._h, int(num_queries), C.c_void_p(d_query_features),
                                            int(num_edges), C.c_void_p(d_edges), C.c_void_p(d_out),
                                            C.byref(bd) if bd is not None else None))
        return bd

    # -- parity hooks ------------------------------------------------------------
    def last_plan(self) -> dict:
        nc, nt = C.c_int64(), C.c_int64()
        nat.check(self._lib.ob_last_plan(self._h, C.byref(nc), C.byref(nt), None, None, None, None, None))
        ids = np.empty(nc.value, np.int64)
        nq = np.empty(nc.value, np.int64)
        tot = np.empty(nc.value, np.int64)
        sc = np.empty(nc.value, np.float64)
        tg = np.empty(nt.value, np.int64)
        nat.check(self._lib.ob_last_plan(self._h, C.byref(nc), C.byref(nt), nat.ptr(ids), nat.ptr(nq),
                                         nat.ptr(tot), nat.ptr(sc), nat.ptr(tg)))
        return dict(ids=ids, nq=nq, total=tot, scores=sc, targets=tg)

    def last_block(self, layer: int, partition: int = 0) -> ComputationBlock:
        ns, nd, ne = C.c_int64(), C.c_int64(), C.c_int64()
        nat.check(self._lib.ob_last_block_sizes(self._h, partition, layer, C.byref(ns), C.byref(nd), C.byref(ne)))
        S, D, E = ns.value, nd.value, ne.value
        b = ComputationBlock(
            src_ids=np.empty(S, np.int64), dst_ids=np.empty(D, np.int64), edge_src=np.empty(E, np.int64),
            edge_dst=np.empty(E, np.int64), bind_kind=np.empty(S, np.uint8), bind_pe_layer=np.empty(S, np.int32),
            src_degree=np.empty(S, np.int64), dst_self_src=np.empty(D, np.int64),
        )
        nat.check(self._lib.ob_last_block(self._h, partition, layer, nat.ptr(b.src_ids), nat.ptr(b.dst_ids),
                                          nat.ptr(b.edge_src), nat.ptr(b.edge_dst), nat.ptr(b.bind_kind),
                                          nat.ptr(b.bind_pe_layer), nat.ptr(b.src_degree),
                                          nat.ptr(b.dst_self_src)))
        if self.config.strategy == "srpe-cgp":
            b.dst_self_src = None
        return b

    def last_graph(self, partition: int = 0) -> ComputationGraph:
        blocks = [self.last_block(l, partition) for l in range(1, self.model.k + 1)]
        n = self.dataset.num_nodes
        tg = (self.last_plan()["targets"] if self.config.strategy not in ("full", "sampled")
              else np.empty(0, np.int64))
        B = int(np.sum(blocks[-1].dst_ids >= n))
        return ComputationGraph(blocks, np.arange(n, n + B, dtype=np.int64), self.config.strategy, n, tg)

    def partition_owner(self) -> np.ndarray:
        """PartitionMap.owner of a CGP engine (graphstore.py:177-181)."""
        out = np.empty(self.dataset.num_nodes, np.int64)
        nat.check(self._lib.ob_partition_owner(self._h, nat.ptr(out)))
        return out

    def graph_info(self) -> dict:
        """Global nodes/edges and the rows/edges this engine holds (partitioned under NCCL CGP)."""
        v = [C.c_int64() for _ in range(4)]
        nat.check(self._lib.ob_graph_info(self._h, *[C.byref(x) for x in v]))
        return dict(num_nodes=v[0].value, num_edges=v[1].value, local_rows=v[2].value, local_edges=v[3].value)

    def graph_csr(self, partition: int = -1) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(offsets, neighbours, in-degrees) of the held in-CSR or of one partition's source-split CSR."""
        info = self.graph_info()
        n = info["num_nodes"]
        if partition < 0:
            ne = info["num_edges"]
        else:
            off = np.empty(n + 1, np.int64)
            nat.check(self._lib.ob_graph_csr(self._h, partition, nat.ptr(off), None, None))
            ne = int(off[-1])
        off = np.empty(n + 1, np.int64)
        nb = np.empty(ne, np.int64)
        deg = np.empty(n, np.int32)
        nat.check(self._lib.ob_graph_csr(self._h, partition, nat.ptr(off), nat.ptr(nb), nat.ptr(deg)))
        return off, nb, deg

    def read_rows(self, table: int, ids) -> np.ndarray:
        """Rows of the feature table (0) or stored layer ``table`` for global ids held here."""
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        w = self.dataset.feature_dim if table == 0 else self.model.layers[table - 1].out_dim
        out = np.empty((len(ids), w), np.float32)
        nat.check(self._lib.ob_read_rows(self._h, table, len(ids), nat.ptr(ids), nat.ptr(out)))
        return out

    def launch_count(self) -> int:
        return int(self._lib.ob_launch_count(self._h))

    def set_lanes(self, n: int) -> None:
        """Request lanes (1..8): requests in flight on separate workspaces and streams (serve_stream / serve_device)."""
        nat.check(self._lib.ob_set_lanes(self._h, int(n)))

    def set_graphs(self, enable: bool) -> None:
        """Replay captured per-shape CUDA graphs (default) or launch every stage eagerly."""
        nat.check(self._lib.ob_set_graphs(self._h, int(bool(enable))))

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.ob_engine_destroy(h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Poisson throughput harness (runtime.py:476-534)
# ---------------------------------------------------------------------------


def poisson_interarrivals(rate_per_s: float, count: int, seed: int) -> np.ndarray:
    """runtime.py:476-480: exponential gaps from numpy's default_rng(seed)."""
    if rate_per_s <= 0:
        raise ValueError("rate must be positive")
    rng = np.random.default_rng(seed)
    return rng.exponential(1.0 / rate_per_s, size=count)


@dataclass
class ThroughputReport:
    """runtime.py:483-490."""

    offered_rate: float
    achieved_rate: float
    completed: int
    p50_ms: float
    p95_ms: float
    p99_ms: float


def throughput_benchmark(serve_fn, request_factory, rate_per_s: float, duration_s: float, seed: int,
                         service_time_fn=None) -> ThroughputReport:
    """FIFO single-server queue in virtual time with measured service times (runtime.py:493-534).

    Arrivals follow the reference's exponential gaps (same numpy stream, so the
    same arrival times for a seed); each admitted request is served for real
    and its completion placed on the virtual timeline; latency = completion -
    arrival.  Service time is the wall clock around ``serve_fn`` (a serve is
    synchronous: it returns host arrays), or ``service_time_fn(result)``
    seconds when given -- e.g. the device-measured time of the request
    (``lambda r: r[1].compute_ms / 1e3 + ...``).
    """
    import time

    if rate_per_s <= 0:
        raise ValueError("rate must be positive")
    rng = np.random.default_rng(seed)
    arrivals = []
    t = 0.0
    while True:
        t += rng.exponential(1.0 / rate_per_s)
        if t >= duration_s:
            break
        arrivals.append(t)
    free_at = 0.0
    latencies = []
    completed = 0
    for i, arr in enumerate(arrivals):
        start = max(arr, free_at)
        if start >= duration_s:
            break
        t0 = time.perf_counter()
        res = serve_fn(request_factory(i))
        service = time.perf_counter() - t0 if service_time_fn is None else float(service_time_fn(res))
        completion = start + service
        free_at = completion
        if completion <= duration_s:
            completed += 1
            latencies.append((completion - arr) * 1e3)
    if latencies:
        p50, p95, p99 = np.percentile(latencies, [50, 95, 99])
    else:
        p50 = p95 = p99 = 0.0
    return ThroughputReport(offered_rate=rate_per_s, achieved_rate=completed / duration_s, completed=completed,
                            p50_ms=float(p50), p95_ms=float(p95), p99_ms=float(p99))
