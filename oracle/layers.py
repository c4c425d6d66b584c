"""Oracle: per-layer GNN math, chained forward, PE precompute, CGP execution.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Accumulation is
float64 and layer outputs are float32, as in the reference
(``models.py:149-228``, ``cgpexec.py:111-240``).  Segment reductions use
CSR sparse products (scipy) over edges sorted by destination; the order of
additions inside one destination therefore differs from ``np.add.at`` by
float64 rounding only.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from . import structure as st

KINDS = ("gcn", "sage_mean", "sage_max", "power_mean", "moments", "gat")
WEIGHT_NAMES = {  # models.py:111-118
    "gcn": ("w",),
    "sage_mean": ("w_self", "w_neigh"),
    "sage_max": ("w_self", "w_neigh"),
    "gat": ("w", "a_src", "a_dst"),
    "power_mean": ("w_self", "w"),
    "moments": ("w_self", "w"),
}


def _f64(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64)


def _relu(x):
    return np.maximum(x, 0.0)


def _softplus(x):
    return np.logaddexp(0.0, x)  # densemath.py:32-34


def _signed_root(x, n):
    """densemath.py:37-41."""
    if n % 2 == 1:
        return np.sign(x) * np.abs(x) ** (1.0 / n)
    return np.maximum(x, 0.0) ** (1.0 / n)


def _spmm(ptr, esrc, weights, x, num_src):
    """Per-destination weighted sums sum_e w_e * x[esrc_e] (float64)."""
    nd = len(ptr) - 1
    if weights is None:
        weights = np.ones(len(esrc))
    a = sp.csr_matrix((_f64(weights), np.asarray(esrc, dtype=np.int64), np.asarray(ptr, dtype=np.int64)),
                      shape=(nd, num_src))
    return np.asarray(a @ x)


def _seg_max(values, ptr, fill):
    nd = len(ptr) - 1
    out = np.full((nd,) + values.shape[1:], fill, dtype=np.float64)
    nz = ptr[1:] > ptr[:-1]
    if values.shape[0] and nz.any():
        out[nz] = np.maximum.reduceat(values, ptr[:-1][nz], axis=0)
    return out


def _attr(spec, name, default=None):
    if isinstance(spec, dict):
        return spec.get(name, default)
    return getattr(spec, name, default)


def aggregate(spec, ptr, esrc, src_degree, x, hv, w):
    """Per-kind aggregation over one block (models.py:172-211).  Returns (agg, counts)."""
    kind = _attr(spec, "kind")
    x = _f64(x)
    nd = len(ptr) - 1
    counts = np.diff(ptr).astype(np.int64)
    nz = counts > 0
    S = x.shape[0]
    if kind == "gcn":
        scale = 1.0 / np.sqrt(_f64(src_degree) + 1.0)
        return _spmm(ptr, esrc, scale[esrc], x, S), counts
    if kind == "sage_mean":
        s = _spmm(ptr, esrc, None, x, S)
        agg = np.zeros_like(s)
        agg[nz] = s[nz] / counts[nz, None]
        return agg, counts
    if kind == "sage_max":
        mx = _seg_max(x[esrc], ptr, -np.inf)
        mx[~nz] = 0.0
        return mx, counts
    if kind == "power_mean":
        p = float(_attr(spec, "p"))
        s = _spmm(ptr, esrc, None, _softplus(x) ** p, S)
        agg = np.zeros_like(s)
        agg[nz] = (s[nz] / counts[nz, None]) ** (1.0 / p)
        return agg, counts
    if kind == "moments":
        n = int(_attr(spec, "n"))
        s = _spmm(ptr, esrc, None, x, S)
        mean = np.zeros_like(s)
        mean[nz] = s[nz] / counts[nz, None]
        edst = np.repeat(np.arange(nd), counts)
        cm_sum = np.zeros_like(s)
        if len(esrc):
            centered = (x[esrc] - mean[edst]) ** n
            cm_sum[nz] = np.add.reduceat(centered, ptr[:-1][nz], axis=0)
        cm = np.zeros_like(s)
        cm[nz] = cm_sum[nz] / counts[nz, None]
        return _signed_root(cm, n), counts
    if kind == "gat":
        wm = _f64(w["w"])
        z = x @ wm
        s_src = z @ _f64(w["a_src"])
        s_dst = (_f64(hv) @ wm) @ _f64(w["a_dst"])
        edst = np.repeat(np.arange(nd), counts)
        logit = s_src[esrc] + s_dst[edst]
        logit = np.where(logit >= 0.0, logit, 0.2 * logit)
        mx = _seg_max(logit, ptr, -np.inf)
        e = np.exp(logit - mx[edst]) if len(esrc) else logit
        den = _spmm(ptr, np.arange(len(esrc)), e, np.ones((len(esrc), 1)), len(esrc))[:, 0] if len(esrc) else np.zeros(nd)
        num = _spmm(ptr, esrc, e, z, S)
        agg = np.zeros_like(num)
        live = den > 0
        agg[live] = num[live] / den[live, None]
        return agg, counts
    raise ValueError(f"unknown layer kind {kind!r}")


def update(spec, hv, agg, counts, w) -> np.ndarray:
    """apply_update (models.py:214-228); ReLU at every layer, float32 out."""
    kind = _attr(spec, "kind")
    if kind == "gcn":
        out = _relu((agg / np.sqrt(_f64(counts) + 1.0)[:, None]) @ _f64(w["w"]))
    elif kind in ("sage_mean", "sage_max"):
        out = _relu(_f64(hv) @ _f64(w["w_self"]) + agg @ _f64(w["w_neigh"]))
    elif kind in ("power_mean", "moments"):
        out = _relu(_f64(hv) @ _f64(w["w_self"]) + agg @ _f64(w["w"]))
    elif kind == "gat":
        out = _relu(agg)
    else:
        raise ValueError(f"unknown layer kind {kind!r}")
    return out.astype(np.float32)


def layer_apply(spec, ptr, esrc, src_degree, x, hv, w) -> np.ndarray:
    """layer_forward (models.py:149-169)."""
    agg, counts = aggregate(spec, ptr, esrc, src_degree, x, hv, w)
    return update(spec, hv, agg, counts, w)


def _lookup(sorted_ids: np.ndarray, ids: np.ndarray) -> np.ndarray:
    pos = np.searchsorted(sorted_ids, ids)
    if ids.size and (np.any(pos >= len(sorted_ids)) or np.any(sorted_ids[np.minimum(pos, len(sorted_ids) - 1)] != ids)):
        raise KeyError("row not available")
    return pos


def resolve_inputs(block: st.Block, num_base, feats, qfeat, pe_layers, prev_out, prev_ids, in_dim):
    """resolve_block_inputs (models.py:231-267)."""
    X = np.empty((len(block.src_ids), in_dim), dtype=np.float32)
    g = block.src_ids
    k = block.bind_kind
    ft = (k == st.BIND_FEATURE) & (g < num_base)
    fq = (k == st.BIND_FEATURE) & (g >= num_base)
    if ft.any():
        X[ft] = feats[g[ft]]
    if fq.any():
        X[fq] = qfeat[g[fq] - num_base]
    pe = k == st.BIND_PE
    for layer in np.unique(block.bind_pe_layer[pe]):
        sel = pe & (block.bind_pe_layer == layer)
        X[sel] = pe_layers[int(layer) - 1][g[sel]]
    comp = k == st.BIND_COMPUTED
    if comp.any():
        order = np.argsort(prev_ids, kind="stable")
        X[comp] = prev_out[order[_lookup(prev_ids[order], g[comp])]]
    return X


def forward(layers, weights, blocks, num_base, feats, qfeat, pe_layers):
    """forward_all_blocks + forward_full (models.py:270-300): returns (per-layer outs, query rows)."""
    prev_out = prev_ids = None
    outs = []
    for l, (spec, blk) in enumerate(zip(layers, blocks), start=1):
        X = resolve_inputs(blk, num_base, feats, qfeat, pe_layers, prev_out, prev_ids, _attr(spec, "in_dim"))
        hv = X[blk.dst_self_src]
        out = layer_apply(spec, blk.dst_ptr(), blk.edge_src, blk.src_degree, X, hv, weights[l - 1])
        outs.append(out)
        prev_out, prev_ids = out, blk.dst_ids
    last = blocks[-1]
    B = int(np.sum(last.dst_ids >= num_base))
    q = np.arange(num_base, num_base + B, dtype=np.int64)
    rows = _lookup(last.dst_ids, q) if not np.array_equal(last.dst_ids, q) else np.arange(B)
    return outs, outs[-1][rows]


def precompute(layers, weights, offsets, nbrs, feats):
    """precompute_embeddings (graphstore.py:330-365): PE layers 1..k-1 over the whole graph."""
    if len(layers) < 2:
        raise ValueError("stored embeddings need a model with k >= 2 layers")
    deg = np.diff(offsets).astype(np.int64)
    h = np.asarray(feats, dtype=np.float32)
    out = []
    for l in range(1, len(layers)):
        h = layer_apply(layers[l - 1], offsets, nbrs, deg, h, h, weights[l - 1])
        out.append(h)
    return out


def serve(strategy, layers, weights, num_base, num_queries, offsets, nbrs, feats, qfeat, edges,
          pe_layers=None, gamma=0.0, fanouts=None, seed=0, policy="ratio"):
    """ServingEngine.serve for the centralized strategies (runtime.py:290-335).

    Returns a dict with the plan, the blocks, the query embeddings and the
    fetch bytes.
    """
    k = len(layers)
    deg = np.diff(offsets).astype(np.int64)
    plan = None
    if strategy == "full":
        blocks = st.build_full(num_base, num_queries, offsets, nbrs, edges, k)
    elif strategy == "sampled":
        if fanouts is None or len(fanouts) != k:
            raise ValueError("sampled strategy needs one fanout per layer")
        blocks = st.build_sampled(num_base, num_queries, offsets, nbrs, edges, fanouts, seed)
    elif strategy == "srpe":
        if pe_layers is None:
            raise ValueError("reuse strategy needs stored embeddings")
        ids, nq, total = st.candidates(edges, num_base, deg)
        if policy == "random":  # runtime.py:182-183, policy.py:122-124
            scores = np.zeros(len(ids))
            targets = st.select_random(ids, gamma, seed)
        else:
            scores = st.ratio_scores(nq, total)
            targets = st.select_top(ids, scores, gamma)
        plan = dict(ids=ids, nq=nq, total=total, scores=scores, targets=targets)
        blocks = st.build_srpe(num_base, num_queries, offsets, nbrs, edges, targets, k, len(pe_layers))
    else:
        raise ValueError(f"unknown strategy {strategy!r}")
    outs, emb = forward(layers, weights, blocks, num_base, feats, qfeat, pe_layers)
    pe_dims = [p.shape[1] for p in (pe_layers or [])]
    fb = st.fetch_bytes(blocks, num_base, feats.shape[1], pe_dims)
    return dict(plan=plan, blocks=blocks, outs=outs, emb=emb, fetch_bytes=fb)


# ---------------------------------------------------------------------------
# CGP: local partials -> rank-ordered merge -> owner update (cgpexec.py)
# ---------------------------------------------------------------------------


def _payloads(spec, blk, x, w, dst_prev_table=None, means_table=None, phase=None):
    """_local_payloads (cgpexec.py:111-164): (counts, payload[nd, w]) in float64."""
    kind = _attr(spec, "kind")
    ptr = blk.dst_ptr()
    esrc = blk.edge_src
    counts = np.diff(ptr).astype(np.int64)
    x = _f64(x)
    S = x.shape[0]
    if kind == "gcn":
        return counts, _spmm(ptr, esrc, (1.0 / np.sqrt(_f64(blk.src_degree) + 1.0))[esrc], x, S)
    if kind == "sage_mean" or (kind == "moments" and phase == 1):
        return counts, _spmm(ptr, esrc, None, x, S)
    if kind == "sage_max":
        return counts, _seg_max(x[esrc], ptr, -np.inf)
    if kind == "power_mean":
        return counts, _spmm(ptr, esrc, None, _softplus(x) ** float(_attr(spec, "p")), S)
    if kind == "moments":
        n = int(_attr(spec, "n"))
        edst = np.repeat(np.arange(len(counts)), counts)
        pay = np.zeros((len(counts), x.shape[1]))
        nz = counts > 0
        if len(esrc):
            pay[nz] = np.add.reduceat((x[esrc] - means_table[edst]) ** n, ptr[:-1][nz], axis=0)
        return counts, pay
    if kind == "gat":
        wm = _f64(w["w"])
        z = x @ wm
        s_src = z @ _f64(w["a_src"])
        s_dst = (_f64(dst_prev_table) @ wm) @ _f64(w["a_dst"])
        edst = np.repeat(np.arange(len(counts)), counts)
        logit = s_src[esrc] + s_dst[edst]
        logit = np.where(logit >= 0.0, logit, 0.2 * logit)
        mx = _seg_max(logit, ptr, -np.inf)
        safe = np.where(np.isfinite(mx), mx, 0.0)
        e = np.exp(logit - safe[edst])
        den = np.zeros(len(counts))
        nz = counts > 0
        if len(esrc):
            den[nz] = np.add.reduceat(e, ptr[:-1][nz])
        num = _spmm(ptr, esrc, e, z, S)
        return counts, np.concatenate([mx[:, None], den[:, None], num], axis=1)
    raise ValueError(f"unknown layer kind {kind!r}")


def merge(kind, pays, cnts, p=0.0, n=0):
    """_merge_arrays (cgpexec.py:189-240); pays [R, nd, w], cnts [R, nd], rank order."""
    total = cnts.sum(axis=0)
    nz = total > 0
    if kind == "sum":
        return pays.sum(axis=0), total
    if kind in ("mean", "moments_p1", "powmean", "moments_p2"):
        s = pays.sum(axis=0)
        out = np.zeros_like(s)
        out[nz] = s[nz] / total[nz, None]
        if kind == "powmean":
            out[nz] = out[nz] ** (1.0 / p)
        if kind == "moments_p2":
            out = _signed_root(out, n)
        return out, total
    if kind == "max":
        mx = np.where((cnts > 0)[:, :, None], pays, -np.inf).max(axis=0)
        mx[~nz] = 0.0
        return mx, total
    if kind == "softmax":
        mx, es, ws = pays[:, :, 0], pays[:, :, 1], pays[:, :, 2:]
        live = es > 0.0
        m_star = np.where(live, mx, -np.inf).max(axis=0)
        m_star = np.where(np.isfinite(m_star), m_star, 0.0)
        scale = np.where(live, np.exp(np.where(live, mx, 0.0) - m_star[None, :]), 0.0)
        den = (es * scale).sum(axis=0)
        num = (ws * scale[:, :, None]).sum(axis=0)
        out = np.zeros_like(num)
        ok = den > 0
        out[ok] = num[ok] / den[ok, None]
        return out, total
    raise ValueError(f"unknown merge kind {kind!r}")


_MERGE = {"gcn": "sum", "sage_mean": "mean", "sage_max": "max", "power_mean": "powmean"}


def cgp_serve(layers, weights, num_base, num_queries, offsets, nbrs, feats, qfeat, edges, pe_layers,
              gamma, num_parts, seed, owner=None):
    """run_cgp_request over all ranks in-process (runtime.py:151-221, cgpexec.py:373-439).

    Returns dict(targets, shards=[per-rank blocks], emb).
    """
    k = len(layers)
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    deg = np.diff(offsets).astype(np.int64)
    owner, shards = st.partition_graph(offsets, nbrs, num_base, num_parts, seed, owner=owner)
    ids, nq, total = st.candidates(edges, num_base, deg)  # == union of per-rank stats
    targets = st.select_top(ids, st.ratio_scores(nq, total), gamma)
    q_deg = st.query_in_degrees(edges, num_base, num_queries)
    parts = st.split_request(edges, num_base, owner, num_parts)
    sh_blocks = [
        st.build_partitioned_shard(num_base, num_queries, shards[r], owner, num_parts, parts[r], q_deg, deg,
                                   targets, k)
        for r in range(num_parts)
    ]

    def owner_of(g):
        return np.where(g >= num_base, (g - num_base) % num_parts, owner[np.minimum(g, num_base - 1)])

    state = [dict() for _ in range(num_parts)]  # rank -> {global id: row}
    for l in range(1, k + 1):
        spec = layers[l - 1]
        w = weights[l - 1]
        kind = _attr(spec, "kind")
        in_dim = _attr(spec, "in_dim")
        dst = sh_blocks[0][l - 1].dst_ids
        down = owner_of(dst)

        def h_prev_rows(ids):
            rows = np.empty((len(ids), in_dim), dtype=np.float32)
            for i, g in enumerate(ids):
                g = int(g)
                if l == 1:
                    rows[i] = qfeat[g - num_base] if g >= num_base else feats[g]
                else:
                    rows[i] = state[int(owner_of(np.array([g]))[0])][g]
            return rows

        xs = []
        for r in range(num_parts):
            blk = sh_blocks[r][l - 1]
            X = np.empty((len(blk.src_ids), in_dim), dtype=np.float32)
            for i, (g, bk, pl) in enumerate(zip(blk.src_ids, blk.bind_kind, blk.bind_pe_layer)):
                g = int(g)
                if bk == st.BIND_FEATURE:
                    X[i] = qfeat[g - num_base] if g >= num_base else feats[g]
                elif bk == st.BIND_PE:
                    X[i] = pe_layers[int(pl) - 1][g]
                else:
                    X[i] = state[r][g]
            xs.append(X)
        table = h_prev_rows(dst)  # all-gathered destination rows (GAT / moments)
        if kind == "moments":
            pc = [_payloads(spec, sh_blocks[r][l - 1], xs[r], w, phase=1) for r in range(num_parts)]
            means, _ = merge("moments_p1", np.stack([p[1] for p in pc]), np.stack([p[0] for p in pc]))
            pc = [_payloads(spec, sh_blocks[r][l - 1], xs[r], w, means_table=means, phase=2)
                  for r in range(num_parts)]
            agg, tot = merge("moments_p2", np.stack([p[1] for p in pc]), np.stack([p[0] for p in pc]),
                             n=int(_attr(spec, "n")))
        else:
            pc = [_payloads(spec, sh_blocks[r][l - 1], xs[r], w, dst_prev_table=table) for r in range(num_parts)]
            mk = "softmax" if kind == "gat" else _MERGE[kind]
            agg, tot = merge(mk, np.stack([p[1] for p in pc]), np.stack([p[0] for p in pc]),
                             p=float(_attr(spec, "p", 0.0) or 0.0))
        out = update(spec, table, agg, tot, w)
        for i, g in enumerate(dst):
            state[int(down[i])][int(g)] = out[i]
    emb = np.zeros((num_queries, _attr(layers[-1], "out_dim")), dtype=np.float32)
    for qi in range(num_queries):
        g = num_base + qi
        emb[qi] = state[int(owner_of(np.array([g]))[0])][g]
    return dict(targets=targets, shards=sh_blocks, emb=emb, owner=owner)


def max_rel_err(a, r) -> float:
    """Parity metric from SURVEY.md 8(d): max|a-r| / max|r| (0/0 -> 0)."""
    a = np.asarray(a, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    denom = float(np.max(np.abs(r))) if r.size else 0.0
    num = float(np.max(np.abs(a - r))) if r.size else 0.0
    if denom == 0.0:
        return num
    return num / denom


_ = math  # keep import for readers comparing formulas
