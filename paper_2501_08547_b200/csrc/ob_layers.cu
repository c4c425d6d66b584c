// ob_layers.cu -- per-layer execution: input binding, segment aggregation,
// dense update on the tensor cores, GAT edge softmax, whole-graph PE precompute.
//
// Reference (paths relative to /root/reference/pkg/src/gnnserve):
//   resolve_block_inputs   models.py:231-267   FEATURE / PE / COMPUTED row binding
//   _aggregate             models.py:172-211   gcn, sage_mean, sage_max, power_mean, moments, gat
//   apply_update           models.py:214-228   relu([h_v | agg] @ [W_self; W_neigh]) etc.
//   forward_all_blocks     models.py:270-300
//   precompute_embeddings  graphstore.py:330-365
//
// Aggregation is split into edge-chunk work items (kAggChunk edges each) so hub
// destinations spread across the whole GPU; each item writes a partial
// (sum / max / online-softmax triple) and a finalize pass merges a
// destination's partials in item order -- the same ordered partial/merge
// algebra CGP uses across GPUs (cgpexec.py:189-240), which keeps results
// deterministic run to run.  Inputs are never materialised: every source
// carries a row pointer into features / query features / PE / the previous
// layer's output, and gathers read rows straight from HBM.
//
// Linear kinds whose layer narrows (gcn / sage_mean with in > out, e.g. the
// 602 -> 128 Reddit layer) run transform-first: Y = X W on the tensor cores
// over the block's unique sources, then the gather/reduce runs over Y's
// narrow rows -- the same sum reordered (sum_u x_u W = (sum_u x_u) W), which
// cuts the gathered bytes by in/out.
#include <type_traits>

#include <cstdlib>

#include "ob_engine.h"

namespace ob {

// kOpDSum / kOpMom2 accumulate in float64: the moments kind takes an n-th root
// of a central moment near zero, which amplifies float32 rounding (the reference
// keeps those payloads float64 for the same reason, cgpexec.py:24-28).
enum AggOp { kOpSum = 0, kOpMax = 1, kOpPow = 2, kOpMom2 = 3, kOpSoftmax = 4, kOpDSum = 5 };

__device__ __forceinline__ float softplus_f(float x) {
  // log(1 + e^x) without overflow (densemath.py:32-34)
  return fmaxf(x, 0.f) + log1pf(__expf(-fabsf(x)));
}

// ---------------------------------------------------------------------------
// binding (resolve_block_inputs)
// ---------------------------------------------------------------------------

// returns BIND_* kind and the row pointer (compgraph.py:287-305 binding rule)
__device__ __forceinline__ int bind_row(const BindCtx& c, int64_t T, int64_t s, int64_t g, const float** row,
                                        int* pe_layer) {
  *pe_layer = 0;
  if (c.layer == 1) {
    *row = g < c.N ? c.feats + (c.pos ? (int64_t)c.pos[g] : g) * c.F_ld : c.qfeat + (g - c.N) * c.F_ld;
    return 0;  // FEATURE
  }
  if (c.mode == 1) {
    *row = c.prev + s * c.in_ld;
    return 2;  // COMPUTED
  }
  if (g >= c.N) {
    *row = c.prev + (T + (g - c.N)) * c.in_ld;
    return 2;
  }
  if (bm_test(c.cbits, g)) {
    int32_t tp = c.tpos[bm_rank(c.cbits, c.cwpre, g)];
    if (tp >= 0) {
      *row = c.prev + (int64_t)tp * c.in_ld;
      return 2;
    }
  }
  *row = c.pe + (c.pos ? (int64_t)c.pos[g] : g) * c.in_ld;
  *pe_layer = c.layer - 1;
  return 1;  // PE
}

__global__ void k_resolve(BindCtx c, BlockCounters* cnt, const int32_t* __restrict__ src_ids, const float** rowp,
                          float* gscale, uint8_t* kind_out, int32_t* pe_layer_out) {
  pdl_wait();
  const CtaWords st = cta_ldv(&cnt->S, c.T_dev);
  const int64_t S = st.v[0];
  const int64_t T = st.v[1];
  int64_t nfeat = 0, npe = 0;
  OB_GRID_STRIDE(s, S) {
    int64_t g = src_ids[s];
    const float* r;
    int pl;
    int k = bind_row(c, T, s, g, &r, &pl);
    rowp[s] = r;
    if (c.yrow) {
      // FEATURE rows of training nodes and PE rows are static: their x W is in the table
      const bool stat = (k == 0 && g < c.N) || k == 1;
      if (stat) {
        c.yrow[s] = c.ytab + (c.pos ? (int64_t)c.pos[g] : g) * c.y_ld;
      } else if (c.qxw && g >= c.N) {
        c.yrow[s] = c.qxw + (g - c.N) * c.y_ld;
      } else {
        const unsigned act = __activemask();
        const unsigned b = __ballot_sync(act, 1);
        const int lane = threadIdx.x & 31, leader = __ffs(act) - 1;
        int64_t base = 0;
        if (lane == leader) base = (int64_t)atomicAdd((unsigned long long*)c.ndyn, (unsigned long long)__popc(b));
        base = __shfl_sync(act, base, leader);
        const int64_t slot = base + __popc(b & ((1u << lane) - 1u));
        c.dyn_src[slot] = (int32_t)s;
        c.yrow[s] = c.ydyn + slot * c.y_ld;
      }
    }
    if (gscale) {
      int64_t d = g < c.N ? c.indeg[g] : c.qdeg[g - c.N];
      gscale[s] = (float)(1.0 / sqrt((double)d + 1.0));
    }
    if (kind_out) {
      kind_out[s] = (uint8_t)k;
      pe_layer_out[s] = pl;
    }
    nfeat += (k == 0 && g < c.N);
    npe += (k == 1);
  }
  // warp-aggregated fetch-byte counters (graph_fetch_bytes, runtime.py:105-120)
  for (int o = 16; o; o >>= 1) {
    nfeat += __shfl_xor_sync(0xffffffffu, nfeat, o);
    npe += __shfl_xor_sync(0xffffffffu, npe, o);
  }
  if ((threadIdx.x & 31) == 0 && kind_out == nullptr) {
    if (nfeat) atomicAdd((unsigned long long*)&cnt->feat_src, (unsigned long long)nfeat);
    if (npe) atomicAdd((unsigned long long*)&cnt->pe_src, (unsigned long long)npe);
  }
}

// ---------------------------------------------------------------------------
// merge of a destination's partials (item order) and its normalisation /
// epilogue (k_reduce_groups + k_finalize after k_agg).  Merging inside k_agg was
// measured slower both ways it was tried: a per-item release fence + arrival
// counter (fences stall the gather), and one warp per small destination (load
// imbalance under the static item schedule); DESIGN.md "Tried".
// ---------------------------------------------------------------------------
constexpr int kAggWarps = 4;
constexpr int kSmHdr = 4;    // softmax partial rows: [max logit, sum exp, pad, pad | values]

struct FinArgs {
  // stored aggregates: raw CSR-part sum of each training destination, added before normalising
  const float* stat = nullptr;
  int64_t stat_ld = 0;
  const int32_t* stat_dst_ids = nullptr;
  int64_t stat_N = 0;
  const BlockCounters* cnt;
  const int64_t* dst_ptr;
  const int64_t* item_ptr;
  const int32_t* group_dst;  // destination per second-level group
  const float* partial;
  const int64_t* group_ptr;  // hub destinations: second-level partials in partial2
  float* partial2;
  int pw;     // partial row stride: ld4(width) (+ kSmHdr for softmax)
  int width;
  int kind;   // ob_kind
  float p;
  int n;
  float* out;  // [D][ldo]
  int64_t ldo;
  bool relu;
  bool gcn_norm;  // divide by sqrt(count + 1) (gcn)
  // own-row update of a transform-first SAGE layer 1 (k_self_update fused):
  // out = relu(own + mean), own = the stored x_v W_self of a training destination or the query's row
  const float* self_tab = nullptr;
  const float* self_q = nullptr;
  int64_t self_ld = 0;
  const int32_t* self_dst_ids = nullptr;
  int64_t self_N = 0;
  // delta rows for the next layer (k_delta_rows fused): dbuf[i] = out[i] - dpe[dst_ids[i]] for i < T
  float* dbuf = nullptr;
  const float* dpe = nullptr;
  const int64_t* dT = nullptr;
};

// partial-row loads (non-coherent path; CG = L2 loads for partials written by the same kernel)
template <bool CG>
__device__ __forceinline__ float4 ldp4(const float* p) {
  return CG ? __ldcg(reinterpret_cast<const float4*>(p)) : __ldg(reinterpret_cast<const float4*>(p));
}
template <bool CG>
__device__ __forceinline__ float2 ldp2(const float* p) {
  return CG ? __ldcg(reinterpret_cast<const float2*>(p)) : __ldg(reinterpret_cast<const float2*>(p));
}
__device__ __forceinline__ float4 ld4f(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// softmax partial header over items [i0, i1): running max logit and the
// rescaled sum of exps, lanes over items, fixed butterfly order
template <bool CG>
__device__ __forceinline__ void sm_header(const float* part, int64_t pw, int64_t i0, int64_t i1, float& ms,
                                          float& den) {
  const int lane = threadIdx.x & 31;
  float m = -INFINITY;
  for (int64_t it = i0 + lane; it < i1; it += 32) {
    const float2 h = ldp2<CG>(part + it * pw);
    if (h.y > 0.f) m = fmaxf(m, h.x);
  }
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float d = 0.f;
  for (int64_t it = i0 + lane; it < i1; it += 32) {
    const float2 h = ldp2<CG>(part + it * pw);
    if (h.y > 0.f) d += h.y * __expf(h.x - m);
  }
  for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  ms = m;
  den = d;
}

enum MergeKind { kMergeSum = 0, kMergeMax = 1, kMergeSoftmax = 2 };

__device__ __forceinline__ float4 f4_op(int mk, float4 a, float4 v, float sc) {
  if (mk == kMergeMax) return make_float4(fmaxf(a.x, v.x), fmaxf(a.y, v.y), fmaxf(a.z, v.z), fmaxf(a.w, v.w));
  if (mk == kMergeSoftmax) return make_float4(fmaf(sc, v.x, a.x), fmaf(sc, v.y, a.y), fmaf(sc, v.z, a.z), fmaf(sc, v.w, a.w));
  return make_float4(a.x + v.x, a.y + v.y, a.z + v.z, a.w + v.w);
}

// four columns [c4, c4+4) of items [i0, i1) merged with a fixed association:
// four interleaved accumulators, 4 rows in flight per lane
template <bool CG>
__device__ __forceinline__ float4 merge_cols(int mk, const float* part, int64_t pw, int64_t i0, int64_t i1, int hdr,
                                             int c4, float ms) {
  const float z = mk == kMergeMax ? -INFINITY : 0.f;
  float4 acc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = make_float4(z, z, z, z);
  int64_t it = i0;
  for (; it + 3 < i1; it += 4) {
    float4 v[4];
    float sc[4] = {1.f, 1.f, 1.f, 1.f};
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = ldp4<CG>(part + (it + j) * pw + hdr + c4);
    if (mk == kMergeSoftmax) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 h = ldp2<CG>(part + (it + j) * pw);
        sc[j] = h.y > 0.f ? __expf(h.x - ms) : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = f4_op(mk, acc[j], v[j], sc[j]);
  }
  for (; it < i1; ++it) {
    float sc = 1.f;
    if (mk == kMergeSoftmax) {
      const float2 h = ldp2<CG>(part + it * pw);
      sc = h.y > 0.f ? __expf(h.x - ms) : 0.f;
    }
    acc[0] = f4_op(mk, acc[0], ldp4<CG>(part + it * pw + hdr + c4), sc);
  }
  const int cm = mk == kMergeMax ? kMergeMax : kMergeSum;
  return f4_op(cm, f4_op(cm, acc[0], acc[1], 1.f), f4_op(cm, acc[2], acc[3], 1.f), 1.f);
}

__device__ __forceinline__ int merge_kind(int kind) {
  return kind == OB_KIND_GAT ? kMergeSoftmax : (kind == OB_KIND_SAGE_MAX ? kMergeMax : kMergeSum);
}

// Hub destinations (more than kItemGroup items): group g = kItemGroup consecutive
// items merged into one second-level partial of the same form (sum / max / softmax
// header + values), fixed association.
template <bool CG>
__device__ __forceinline__ void reduce_group(const FinArgs& a, int64_t g) {
  const int lane = threadIdx.x & 31;
  const int mk = merge_kind(a.kind);
  const int hdr = mk == kMergeSoftmax ? kSmHdr : 0;
  const int64_t i = __ldg(a.group_dst + g);
  const int64_t it0 = a.item_ptr[i] + (g - a.group_ptr[i]) * kItemGroup;
  const int64_t it1 = min(it0 + kItemGroup, a.item_ptr[i + 1]);
  float* out = a.partial2 + g * (int64_t)a.pw;
  float ms = 0.f, den = 0.f;
  if (mk == kMergeSoftmax) {
    sm_header<CG>(a.partial, a.pw, it0, it1, ms, den);
    if (lane == 0) {
      out[0] = ms;
      out[1] = den;
    }
  }
  for (int c4 = lane * 4; c4 < a.width; c4 += 128)
    *reinterpret_cast<float4*>(out + hdr + c4) = merge_cols<CG>(mk, a.partial, a.pw, it0, it1, hdr, c4, ms);
}

// columns [c4, c4 + 4) of destination i from its merged raw aggregate v (softmax:
// the sum exp * z with its header (ms, den)): add the stored CSR part, normalise,
// then the layer epilogue (activation, own-row update, the next layer's delta rows)
__device__ __forceinline__ void fin_cols(const FinArgs& a, int64_t i, int64_t cnt, int c4, float4 v, float ms,
                                         float den, int64_t dT) {
  if (c4 >= a.width) return;
  const int mk = merge_kind(a.kind);
  const float* st = nullptr;
  if (a.stat) {
    const int64_t u = a.stat_dst_ids[i];
    if (u < a.stat_N) st = a.stat + u * a.stat_ld;
  }
  if (st && mk == kMergeSoftmax) {  // the static (max, sum exp, sum exp z) triple joins the items
    const float2 h = __ldg(reinterpret_cast<const float2*>(st));
    if (h.y > 0.f) {
      const float M = den > 0.f ? fmaxf(ms, h.x) : h.x;
      const float sc_items = den > 0.f ? __expf(ms - M) : 0.f;
      const float sc_stat = __expf(h.x - M);
      den = den * sc_items + h.y * sc_stat;
      const float4 q = ld4f(st + kSmHdr + c4);
      v = make_float4(fmaf(sc_stat, q.x, v.x * sc_items), fmaf(sc_stat, q.y, v.y * sc_items),
                      fmaf(sc_stat, q.z, v.z * sc_items), fmaf(sc_stat, q.w, v.w * sc_items));
    }
  } else if (st) {
    const float4 q = ld4f(st + c4);
    v = make_float4(q.x + v.x, q.y + v.y, q.z + v.z, q.w + v.w);
  }
  const float* own = nullptr;
  if (a.self_tab) {
    const int64_t u = a.self_dst_ids[i];
    own = (u < a.self_N ? a.self_tab + u * a.self_ld : a.self_q + (u - a.self_N) * a.self_ld) + c4;
  }
  const float* dpe = nullptr;
  float* drow = nullptr;
  if (a.dbuf && i < dT) {
    const int64_t ld = (a.width + 3) & ~3;
    dpe = a.dpe + (int64_t)a.self_dst_ids[i] * ld + c4;
    drow = a.dbuf + i * ld + c4;
  }
  const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (c4 + t >= a.width) break;
    float r;
    if (mk == kMergeSoftmax) r = den > 0.f ? vv[t] / den : 0.f;
    else if (mk == kMergeMax) r = cnt > 0 ? vv[t] : 0.f;
    else if (a.gcn_norm) r = vv[t] / sqrtf((float)cnt + 1.f);  // agg / sqrt(|N(v)|+1) (models.py:217-218)
    else if (a.kind == OB_KIND_POWER_MEAN) r = cnt > 0 ? powf(vv[t] / (float)cnt, 1.f / a.p) : 0.f;
    else r = cnt > 0 ? vv[t] / (float)cnt : 0.f;  // mean
    if (own) r = fmaxf(own[t] + r, 0.f);  // the fp32 sum the own-row update formed (then relu)
    if (a.relu) r = fmaxf(r, 0.f);
    a.out[i * a.ldo + c4 + t] = r;
    if (drow) drow[t] = r - dpe[t];
  }
}

// destination i: merge its items (or hub groups) in item order, then fin_cols
// dT: the delta-row count (*a.dT, read once per kernel)
__device__ __forceinline__ void finalize_dst(const FinArgs& a, int64_t i, int64_t dT) {
  const int lane = threadIdx.x & 31;
  const int mk = merge_kind(a.kind);
  const int hdr = mk == kMergeSoftmax ? kSmHdr : 0;
  int64_t i0 = a.item_ptr[i], i1 = a.item_ptr[i + 1];
  const int64_t cnt = a.dst_ptr[i + 1] - a.dst_ptr[i];
  const float* part = a.partial;
  if (a.group_ptr && a.group_ptr[i + 1] > a.group_ptr[i]) {  // hub: merge the group partials
    i0 = a.group_ptr[i];
    i1 = a.group_ptr[i + 1];
    part = a.partial2;
  }
  float ms = 0.f, den = 0.f;
  // (max, sum exp, sum exp*z) merge in item order (cgpexec.py:225-239)
  if (mk == kMergeSoftmax) sm_header<false>(part, a.pw, i0, i1, ms, den);
  for (int c4 = lane * 4; c4 < a.width; c4 += 128)
    fin_cols(a, i, cnt, c4, merge_cols<false>(mk, part, a.pw, i0, i1, hdr, c4, ms), ms, den, dT);
}

// ---------------------------------------------------------------------------
// edge-chunk aggregation: one warp per (work item, 512-column slice)
// ---------------------------------------------------------------------------
struct AggArgs {
  const BlockCounters* cnt;
  const int64_t* dst_ptr;
  const int64_t* item_ptr;
  const int32_t* item_dst;
  const int32_t* edge_src;
  RowSrc x;              // input rows (16 B aligned, stride multiple of 4)
  int width;
  const float* gscale;   // sum with per-source weight (gcn) or null
  float p;               // power mean exponent
  int n;                 // moments order
  const double* mean;    // moments phase 2: [D][width] (float64)
  const float* s_src;    // softmax
  const float* s_dst;
  float* partial;        // [items][pw]
  int pw;                // partial row stride: ld4(width), softmax kSmHdr + ld4(width)
  // stored aggregates (layer 1): a training destination's CSR part is in the
  // table, so only its request span (the row's suffix of query sources) is gathered
  const int32_t* skip_dst_ids = nullptr;
  const int32_t* skip_indeg = nullptr;
  int64_t skip_N = 0;
  // delta mode (skip_dst_ids set too): CSR-part edges are kept only when their row
  // lies in dprev[0, T) (a recomputed target) and then read from the delta row at
  // the same index (dbuf); the request suffix is gathered as is
  const float* dprev = nullptr;
  const int64_t* dT = nullptr;
  const float* dbuf = nullptr;
  int64_t dld = 0;
  // source-range pass (sum): only sources [src_lo, src_hi) of each row (a row's
  // sources are ascending, so that is a contiguous run of every 32-edge group);
  // accumulate adds to the partials of the previous pass
  int pass = 0, passes = 1;  // pass p covers sources [S p / passes, S (p+1) / passes)
  int64_t S_max = 0;         // host side: bound on the block's sources (the profiler's row count)
};

template <int OP, int NV>
#ifndef OB_AGG_MINB_WIDE
#define OB_AGG_MINB_WIDE 1  // k_agg CTAs per SM for rows wider than 128 columns (NV = 2, 4)
#endif
__global__ void __launch_bounds__(32 * kAggWarps, (NV == 1 ? 8 : OB_AGG_MINB_WIDE)) k_agg(AggArgs a) {
  using AT = typename std::conditional<(OP == kOpDSum || OP == kOpMom2), double, float>::type;
  constexpr int kU = NV == 1 ? 8 : 4;  // edges whose rows are in flight together
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const CtaWords st = cta_ldv(&a.cnt->items, a.passes > 1 ? &a.cnt->S : nullptr, a.dprev ? a.dT : nullptr);
  const int64_t items = st.v[0];
  const int col0 = blockIdx.y * (32 * 4 * NV);
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int32_t src_lo = 0, src_hi = 0x7fffffff;
  if (a.passes > 1) {
    const int64_t S = st.v[1];
    src_lo = (int32_t)(S * a.pass / a.passes);
    src_hi = a.pass + 1 == a.passes ? 0x7fffffff : (int32_t)(S * (a.pass + 1) / a.passes);
  }
  // delta mode: recomputed rows are prev[0, T); their delta rows sit at the same offset in dbuf
  const float* d_lo = a.dprev;
  const float* d_hi = a.dprev ? a.dprev + st.v[2] * a.dld : nullptr;
  const ptrdiff_t d_shift = a.dprev ? a.dbuf - a.dprev : 0;
  __shared__ const float* c_row[kAggWarps][32];  // delta mode: the group's kept edges, compacted
  __shared__ float c_w[kAggWarps][32];
  const int wib = threadIdx.x >> 5;
  for (int64_t it = gw; it < items; it += nw) {
    const int64_t i = __ldg(a.item_dst + it);
    const int64_t j = it - a.item_ptr[i];
    int64_t e0 = a.dst_ptr[i] + j * kAggChunk;
    const int64_t e1 = min(e0 + kAggChunk, a.dst_ptr[i + 1]);
    int64_t csr_end = e0;  // delta mode: edges below this are the destination's CSR part
    if (a.skip_indeg) {
      const int64_t v = __ldg(a.skip_dst_ids + i);
      const int64_t ce = v < a.skip_N ? a.dst_ptr[i] + (int64_t)__ldg(a.skip_indeg + v) : a.dst_ptr[i];
      if (d_lo) csr_end = ce;
      else e0 = max(e0, ce);
    }
    AT acc[NV][4];
    float m_run = -INFINITY, den = 0.f;
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[q][t] = (OP == kOpMax) ? -INFINITY : 0.f;
    const float sd = (OP == kOpSoftmax) ? a.s_dst[i] : 0.f;
    for (int64_t eb = e0; eb < e1; eb += 32) {
      // lane-cooperative edge fetch, then broadcast
      const int64_t my = eb + lane;
      const int32_t s_l = my < e1 ? a.edge_src[my] : 0;
      bool in_l = my < e1 && s_l >= src_lo && s_l < src_hi;
      const float* r_l = in_l ? a.x.row(s_l) : nullptr;
      if (d_lo && in_l && my < csr_end) {  // CSR part: recomputed sources only, as delta rows
        in_l = r_l >= d_lo && r_l < d_hi;
        r_l += d_shift;
      }
      float w_l = 1.f;
      if (in_l) {
        if (OP == kOpSum && a.gscale) w_l = a.gscale[s_l];
        if (OP == kOpSoftmax) {
          float lg = a.s_src[s_l] + sd;
          w_l = lg >= 0.f ? lg : 0.2f * lg;  // leaky_relu(0.2)
        }
      }
      // the group's in-range edges are contiguous (ascending sources): [first, first + cnt);
      // in delta mode they are compacted through shared memory first (same edge order)
      const unsigned inb = __ballot_sync(0xffffffffu, in_l);
      if (!inb) continue;
      int first = __ffs(inb) - 1;
      const int cnt = __popc(inb);
      if (d_lo) {
        if (in_l) {
          const int slot = __popc(inb & ((1u << lane) - 1u));
          c_row[wib][slot] = r_l;
          c_w[wib][slot] = w_l;
        }
        __syncwarp();
        r_l = c_row[wib][lane];
        w_l = c_w[wib][lane];
        __syncwarp();
        first = 0;
      }
      for (int u = 0; u < cnt; u += kU) {
        float4 v[kU][NV];
        float wg[kU];
#pragma unroll
        for (int x = 0; x < kU; ++x) {  // issue kU row loads before consuming any
          const int uu = first + min(u + x, cnt - 1);
          const float* r = (const float*)__shfl_sync(0xffffffffu, (unsigned long long)r_l, uu);
          wg[x] = __shfl_sync(0xffffffffu, w_l, uu);
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const int col = col0 + (q * 32 + lane) * 4;
            v[x][q] = col < a.width ? __ldg(reinterpret_cast<const float4*>(r + col)) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int x = 0; x < kU; ++x) {
          if (u + x >= cnt) break;
          const float wgt = wg[x];
          float scale_old = 1.f, pe = 1.f;
          if (OP == kOpSoftmax) {
            float mn = fmaxf(m_run, wgt);
            scale_old = __expf(m_run - mn);
            pe = __expf(wgt - mn);
            den = den * scale_old + pe;
            m_run = mn;
          }
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const int col = col0 + (q * 32 + lane) * 4;
            if (col < a.width) {
              const float vv[4] = {v[x][q].x, v[x][q].y, v[x][q].z, v[x][q].w};
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                if (OP == kOpSum) acc[q][t] = fmaf(wgt, vv[t], acc[q][t]);
                else if (OP == kOpDSum) acc[q][t] += (double)vv[t];
                else if (OP == kOpMax) acc[q][t] = fmaxf(acc[q][t], vv[t]);
                else if (OP == kOpPow) acc[q][t] += powf(softplus_f(vv[t]), a.p);
                else if (OP == kOpMom2) {
                  if (col + t < a.width) {
                    double dlt = (double)vv[t] - a.mean[i * a.width + col + t];
                    double pw = dlt;
                    for (int r2 = 1; r2 < a.n; ++r2) pw *= dlt;
                    acc[q][t] += pw;
                  }
                } else {
                  acc[q][t] = fmaf(pe, vv[t], acc[q][t] * scale_old);
                }
              }
            }
          }
        }
      }
    }
    AT* out = reinterpret_cast<AT*>(a.partial) + it * (int64_t)a.pw;
    if (OP == kOpSoftmax) {
      if (blockIdx.y == 0 && lane == 0) {
        out[0] = (e1 > e0) ? m_run : -INFINITY;
        out[1] = den;
      }
      out += kSmHdr;
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int col = col0 + (q * 32 + lane) * 4;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (col + t < a.width) out[col + t] = a.pass > 0 ? out[col + t] + acc[q][t] : acc[q][t];
    }
  }
}

// Profiler only (launched after a stored-aggregate or delta k_agg, outside its events):
// the rows that launch loaded -- row loads (one per kept edge) into cnt->gathered and
// distinct rows into cnt->uniq.  Bit 2s + 1 marks source s's delta row, bit 2s its row.
__global__ void k_prof_rows(AggArgs a, uint32_t* bits) {
  const int lane = threadIdx.x & 31;
  const int64_t items = cta_ld(&a.cnt->items);
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float* d_lo = a.dprev;
  const float* d_hi = a.dprev ? a.dprev + cta_ld(a.dT) * a.dld : nullptr;
  unsigned long long loads = 0;
  for (int64_t it = gw; it < items; it += nw) {
    const int64_t i = a.item_dst[it];
    int64_t e0 = a.dst_ptr[i] + (it - a.item_ptr[i]) * kAggChunk;
    const int64_t e1 = min(e0 + kAggChunk, a.dst_ptr[i + 1]);
    int64_t csr_end = e0;
    if (a.skip_indeg) {
      const int64_t v = a.skip_dst_ids[i];
      const int64_t ce = v < a.skip_N ? a.dst_ptr[i] + (int64_t)a.skip_indeg[v] : a.dst_ptr[i];
      if (d_lo) csr_end = ce;
      else e0 = max(e0, ce);
    }
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int32_t src = a.edge_src[e];
      int64_t bit = 2 * (int64_t)src;
      if (d_lo && e < csr_end) {
        const float* r = a.x.row(src);
        if (r < d_lo || r >= d_hi) continue;
        bit += 1;
      }
      ++loads;
      atomicOr(bits + (bit >> 5), 1u << (bit & 31));
    }
  }
  for (int o = 16; o; o >>= 1) loads += __shfl_xor_sync(0xffffffffu, loads, o);
  if (lane == 0 && loads) atomicAdd((unsigned long long*)&const_cast<BlockCounters*>(a.cnt)->gathered, loads);
}

__global__ void k_prof_popc(const uint32_t* bits, int64_t words, const BlockCounters* cnt) {
  unsigned long long n = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
    n += __popc(bits[w]);
  for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd((unsigned long long*)&const_cast<BlockCounters*>(cnt)->uniq, n);
}

__global__ void __launch_bounds__(256) k_reduce_groups(FinArgs a) {
  pdl_wait();
  const int64_t G = cta_ld(&a.cnt->groups);
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = gw; g < G; g += nw) reduce_group<false>(a, g);
}

#ifndef OB_FIN_MINB
#define OB_FIN_MINB 4  // k_finalize CTAs resident per SM (64 registers, no spills)
#endif
__global__ void __launch_bounds__(256, OB_FIN_MINB) k_finalize(FinArgs a) {
  pdl_wait();
  const int64_t D = cta_ld(&a.cnt->D);
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  __shared__ int64_t s_dT;  // read once per CTA, from shared memory per row (no register held)
  if (threadIdx.x == 0) s_dT = a.dbuf ? ld_state(a.dT) : 0;
  __syncthreads();
  for (int64_t i = gw; i < D; i += nw) finalize_dst(a, i, s_dT);
}

// moments finalize in float64: phase 1 -> mean (double), phase 2 -> signed root (float)
__global__ void __launch_bounds__(256) k_finalize_moments(const BlockCounters* cnt_, const int64_t* dst_ptr,
                                                          const int64_t* item_ptr, const double* partial, int width,
                                                          int phase, int n, double* mean, float* agg, int64_t ldo) {
  pdl_wait();
  const int64_t D = cta_ld(&cnt_->D);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < D; i += nw) {
    const int64_t cnt = dst_ptr[i + 1] - dst_ptr[i];
    for (int col = lane; col < width; col += 32) {
      double s = 0.0;
      for (int64_t it = item_ptr[i]; it < item_ptr[i + 1]; ++it) s += partial[it * (int64_t)width + col];
      const double m = cnt > 0 ? s / (double)cnt : 0.0;
      if (phase == 1) {
        mean[i * width + col] = m;
      } else {
        const double r = (n & 1) ? copysign(pow(fabs(m), 1.0 / n), m) : pow(fmax(m, 0.0), 1.0 / n);
        agg[i * ldo + col] = (float)r;  // densemath.py:37-41
      }
    }
  }
}

// GAT attention scores: s[r] = z[row(r)] . a  (one warp per row)
// out[r] = z_row(self[r] or r) . av  (GAT source / destination scores)
// tab/stab (optional): rows inside the stored-transform table [tab, tab + tab_rows * tab_ld)
// take the precomputed score stab[row index] -- the same dot product, computed once per table
__global__ void k_rowdot_rows(const int64_t* M_dev, RowSrc z, const int32_t* self, int w,
                              const float* __restrict__ av, float* out) {
  pdl_wait();
  const int64_t M = cta_ld(M_dev);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < M; r += nw) {
    const float* row = z.row(self ? (int64_t)self[r] : r);
    float s = 0.f;
    for (int c = lane; c < w; c += 32) s = fmaf(row[c], av[c], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = s;
  }
}

// the same for source rows bound by pointer, where rows inside the stored-transform table
// [tab, tab + tab_rows * tab_ld) take the table's precomputed score stab[row index]
__global__ void k_rowdot_rows_tab(const int64_t* M_dev, RowSrc z, int w, const float* __restrict__ av, float* out,
                                  const float* tab, int64_t tab_rows, int64_t tab_ld, const float* __restrict__ stab) {
  pdl_wait();
  const int64_t M = cta_ld(M_dev);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool pow2 = (tab_ld & (tab_ld - 1)) == 0;  // row index by shift, not a 64-bit divide
  const int sh = pow2 ? __ffsll((long long)tab_ld) - 1 : 0;
  for (int64_t r = gw; r < M; r += nw) {
    const float* row = z.row(r);
    if (row >= tab && row < tab + tab_rows * tab_ld) {
      if (lane == 0) {
        const int64_t off = row - tab;
        out[r] = stab[pow2 ? off >> sh : off / tab_ld];
      }
      continue;
    }
    float s = 0.f;
    for (int c = lane; c < w; c += 32) s = fmaf(row[c], av[c], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = s;
  }
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
// Sum gathers over a source-row set larger than ~half the L2 run as source-range
// passes, each touching a slice of the rows that stays L2-resident.
constexpr int64_t kAggPassBytes = 64ll << 20;

// widest column slice per warp (OB_AGG_NV_MAX: 4 = 512 columns; 2 splits 512-wide rows into two
// 256-column slices on blockIdx.y, each warp then needs ~40 % fewer registers)
static int agg_nv_max() {
  static const int n = [] {
    const char* v = std::getenv("OB_AGG_NV_MAX");
    const int x = v && v[0] ? std::atoi(v) : 4;
    return x >= 4 ? 4 : (x >= 2 ? 2 : 1);
  }();
  return n;
}

template <int OP>
static void launch_agg(cudaStream_t s, const AggArgs& a0, int64_t items_max, int64_t S_max = 0) {
  // sum gathers of 512-wide rows run as two 256-column slices (measured +1-3 % on the
  // H = 512 GCN configs; the softmax kind keeps one 512-column warp, -4 % otherwise)
  const int nv_cap = OP == kOpSum ? std::min(agg_nv_max(), 2) : agg_nv_max();
  const int nv = std::min(nv_cap, a0.width <= 128 ? 1 : (a0.width <= 256 ? 2 : 4));
  dim3 grid(grid_for(items_max, kAggWarps, kNumSMs * 16), (a0.width + 128 * nv - 1) / (128 * nv));
  int passes = 1;
  if (OP == kOpSum && S_max > 0 && !a0.skip_indeg && !a0.dprev) {
    const int64_t rows_bytes = S_max * (int64_t)ld4(a0.width) * 4;
    passes = (int)std::min<int64_t>(4, (rows_bytes + kAggPassBytes - 1) / kAggPassBytes);
    if (passes < 1) passes = 1;
  }
  cudaEvent_t pa = prof_begin(s);
  for (int p = 0; p < passes; ++p) {
    AggArgs a = a0;
    a.pass = p;
    a.passes = passes;
    if (nv == 1) launch_pdl(k_agg<OP, 1>, grid, dim3(32 * kAggWarps), 0, s, a);
    else if (nv == 2) launch_pdl(k_agg<OP, 2>, grid, dim3(32 * kAggWarps), 0, s, a);
    else launch_pdl(k_agg<OP, 4>, grid, dim3(32 * kAggWarps), 0, s, a);
  }
  // K = -1 marks a stored-aggregate launch: it gathers only the request spans, which the
  // block counters do not size, so the profiler counts its edge list and partials only
  // (K = -2: delta launch -- edge list, the recomputed rows (<= D) and the partials)
  prof_end(s, pa, kProfAgg, a0.cnt, a0.width, a0.pw, a0.dprev ? -2 : (a0.skip_indeg ? -1 : 0), 0, 0);
  if (pa && a0.skip_indeg && a0.S_max > 0) {  // count the rows it loaded (profiler only, its own class)
    cudaEvent_t pc = prof_begin(s);
    const int64_t words = (2 * a0.S_max + 31) / 32;
    uint32_t* bits = g_prof->bits(words, s);
    k_prof_rows<<<grid_for(items_max, 8, kNumSMs * 16), 256, 0, s>>>(a0, bits);
    k_prof_popc<<<grid_for(words, 256, kNumSMs * 4), 256, 0, s>>>(bits, words, a0.cnt);
    OB_CUDA(cudaGetLastError());
    prof_end(s, pc, kProfCount, nullptr, 0, 0, 0, 0, 0);
  }
}

static void finalize(cudaStream_t s, const FinArgs& f, int64_t D_max, int64_t items_max) {
  cudaEvent_t pa = prof_begin(s);
  if (f.group_ptr) {
    launch_pdl(k_reduce_groups, dim3(grid_for(items_max / kItemGroup + 1, 8, kNumSMs * 16)), dim3(256), 0, s, f);
  }
  launch_pdl(k_finalize, dim3(grid_for(D_max, 8, kNumSMs * 16)), dim3(256), 0, s, f);
  prof_end(s, pa, kProfFinalize, f.cnt, f.width, f.pw, 0, 0, 0);
}

// aggregation, then the merge of each destination's partials and its epilogue
template <int OP>
static void agg_fin(cudaStream_t s, const AggArgs& a, const FinArgs& f, int64_t items_max, int64_t D_max,
                    int64_t S_split = 0) {
  launch_agg<OP>(s, a, items_max, S_split);
  finalize(s, f, D_max, items_max);
}

static void gemm(cudaStream_t s, const TcGemmArgs& g, int64_t M_max, const BlockCounters* cnt) {
  cudaEvent_t pa = prof_begin(s);
  tc_gemm(s, g, M_max);
  prof_end(s, pa, kProfGemm, cnt, 0, 0, g.K1 + g.K2, g.N, (cnt && g.M_dev == &cnt->S) ? 1 : 0);
}

// ---------------------------------------------------------------------------
// one layer over one block (shared by serving and precompute)
// ---------------------------------------------------------------------------


static TcGemmArgs gemm_args(const int64_t* M_dev, const TcWeights& w, float* C, int64_t ldc, bool relu) {
  TcGemmArgs g{};
  g.M_dev = M_dev;
  g.Bt = w.hi;
  g.Bt_lo = w.lo;
  g.w = &w;
  g.N = w.N;
  g.Np = w.Np;
  g.C = C;
  g.ldc = ldc;
  g.relu = relu;
  return g;
}

// Returns true when the layer's finalize also wrote the next layer's delta rows
// (r.dnext): the output then comes from the merge epilogue, not a GEMM.
bool run_layer(cudaStream_t s, const LayerDev& L, const LayerRun& r, const LayerScratch& sc, float* out,
               int64_t ldo) {
  const ob_layer& sp = L.spec;
  const int in = sp.in_dim, outd = sp.out_dim;
  const int64_t ld_out = ld4(outd);
  AggArgs a{};
  a.cnt = r.cnt;
  a.S_max = r.S_max;
  a.dst_ptr = r.dst_ptr;
  a.item_ptr = r.item_ptr;
  a.item_dst = r.item_dst;
  a.edge_src = r.edge_src;
  a.x = r.x;
  a.width = in;
  a.pw = sp.kind == OB_KIND_MOMENTS ? in : ld4(in);  // moments: float64 rows, unpadded
  a.partial = sc.partial;
  a.p = sp.p;
  a.n = sp.n;
  FinArgs f{};
  f.cnt = r.cnt;
  f.dst_ptr = r.dst_ptr;
  f.item_ptr = r.item_ptr;
  f.group_dst = r.group_dst;
  f.partial = sc.partial;
  f.partial2 = sc.partial2;
  f.group_ptr = r.group_ptr;
  f.pw = a.pw;
  f.width = in;
  f.kind = sp.kind;
  f.p = sp.p;
  f.n = sp.n;
  f.out = sc.agg;
  f.ldo = ld4(in);
  if (r.stat) {  // stored aggregates: gather only the request spans, add the static CSR part
    a.skip_dst_ids = r.dst_ids;
    a.skip_indeg = r.indeg;
    a.skip_N = r.N;
    if (r.delta) {
      a.dprev = r.dprev;
      a.dT = r.dT;
      a.dbuf = r.dbuf;
      a.dld = ld4(in);
    }
    f.stat = r.stat;
    f.stat_ld = r.stat_ld;
    f.stat_dst_ids = r.dst_ids;
    f.stat_N = r.N;
  }
  // the next layer's delta rows from this layer's merge epilogue (when it writes the output)
  auto with_dnext = [&](FinArgs& ff) {
    if (!r.dnext) return false;
    ff.dbuf = r.dnext;
    ff.dpe = r.dnext_pe;
    ff.dT = r.dnext_T;
    ff.self_dst_ids = r.dst_ids;
    return true;
  };
  const int64_t split = r.split_gather ? r.S_max : 0;

  if ((sp.kind == OB_KIND_GAT || L.transform_first) && r.yrow) {
    // stored transforms: only the listed sources (queries, recomputed rows) need x W now
    TcGemmArgs g = gemm_args(r.ndyn, L.tw_main, sc.z, ld_out, false);
    g.a1 = r.x;
    g.self = r.dyn_src;
    g.K1 = in;
    if (!r.no_dyn) gemm(s, g, r.dyn_max, nullptr);
    a.x = RowSrc{r.yrow, nullptr, 0};
    a.width = outd;
    a.pw = ld4(outd);
    f.width = outd;
    f.pw = ld4(outd);
    f.ldo = ld_out;
  } else if (sp.kind == OB_KIND_GAT || L.transform_first) {
    // Y = X W over every source row (GAT: z; transform-first: X W_neigh or X W)
    TcGemmArgs g = gemm_args(r.S_dev, L.tw_main, sc.z, ld_out, false);
    g.a1 = r.x;
    g.K1 = in;
    gemm(s, g, r.S_max, r.cnt);
    a.x = RowSrc{nullptr, sc.z, ld_out};
    a.width = outd;
    a.pw = ld4(outd);
    f.width = outd;
    f.pw = ld4(outd);
    f.ldo = ld_out;
  }
  if (sp.kind == OB_KIND_GAT) {
    const RowSrc z = r.yrow ? RowSrc{r.yrow, nullptr, 0} : RowSrc{nullptr, sc.z, ld_out};
    if (r.yrow && r.stab)  // stored rows' source scores from the table
      launch_pdl(k_rowdot_rows_tab, dim3(grid_for(r.S_max, 8)), dim3(256), 0, s, r.S_dev, z, outd, L.a_src, sc.s_src,
                 r.ytab, r.ytab_rows, r.ytab_ld, r.stab);
    else
      launch_pdl(k_rowdot_rows, dim3(grid_for(r.S_max, 8)), dim3(256), 0, s, r.S_dev, z, nullptr, outd, L.a_src, sc.s_src);
    launch_pdl(k_rowdot_rows, dim3(grid_for(r.D_max, 8)), dim3(256), 0, s, r.D_dev, z, r.self, outd, L.a_dst, sc.s_dst);
    a.pw = kSmHdr + ld4(outd);
    a.s_src = sc.s_src;
    a.s_dst = sc.s_dst;
    f.pw = a.pw;
    f.out = out;
    f.ldo = ldo;
    f.relu = true;
    const bool d = with_dnext(f);
    agg_fin<kOpSoftmax>(s, a, f, r.items_max, r.D_max);
    return d;
  }
  if (sp.kind == OB_KIND_GCN) {
    a.gscale = r.gscale;
    f.gcn_norm = true;
    if (L.transform_first) {  // relu(sum_u (x_u W) / sqrt(d_u+1) / sqrt(c+1))
      f.out = out;
      f.ldo = ldo;
      f.relu = true;
      const bool d = with_dnext(f);
      agg_fin<kOpSum>(s, a, f, r.items_max, r.D_max, split);
      return d;
    }
    agg_fin<kOpSum>(s, a, f, r.items_max, r.D_max, split);
    TcGemmArgs g = gemm_args(r.D_dev, L.tw_main, out, ldo, true);
    g.a2 = sc.agg;
    g.lda2 = ld4(in);
    g.K2 = in;
    gemm(s, g, r.D_max, r.cnt);
    return false;
  }
  if (sp.kind == OB_KIND_SAGE_MEAN && L.transform_first && r.self_tab) {
    // own-row term: training destinations from the stored table, the queries by a B-row GEMM
    // (done early, beside the request-index sort, when the query rows were staged ahead);
    // relu(own + mean) is the merge epilogue
    const float* qs = r.self_q;
    if (!qs) {
      TcGemmArgs g = gemm_args(r.B_dev, L.tw_self, sc.z, ld_out, false);
      g.a1 = RowSrc{nullptr, r.qpad, r.q_ld};
      g.K1 = in;
      gemm(s, g, r.B, nullptr);
      qs = sc.z;
    }
    f.self_tab = r.self_tab;
    f.self_q = qs;
    f.self_ld = ld_out;
    f.self_dst_ids = r.dst_ids;
    f.self_N = r.N;
    f.out = out;
    f.ldo = ldo;
    const bool d = with_dnext(f);
    agg_fin<kOpSum>(s, a, f, r.items_max, r.D_max, split);
    return d;
  }
  if (sp.kind == OB_KIND_SAGE_MEAN && L.transform_first) {
    agg_fin<kOpSum>(s, a, f, r.items_max, r.D_max, split);  // mean over Y = X W_neigh -> agg
    TcGemmArgs g = gemm_args(r.D_dev, L.tw_self, out, ldo, true);
    g.a1 = r.x;
    g.self = r.self;
    g.K1 = in;
    g.E = sc.agg;
    g.lde = ld_out;
    gemm(s, g, r.D_max, r.cnt);
    return false;
  }
  if (sp.kind == OB_KIND_SAGE_MAX) {
    agg_fin<kOpMax>(s, a, f, r.items_max, r.D_max);
  } else if (sp.kind == OB_KIND_POWER_MEAN) {
    agg_fin<kOpPow>(s, a, f, r.items_max, r.D_max);
  } else if (sp.kind == OB_KIND_MOMENTS) {
    double* mean = reinterpret_cast<double*>(sc.mean);
    launch_agg<kOpDSum>(s, a, r.items_max);
    launch_pdl(k_finalize_moments, dim3(grid_for(r.D_max, 8, kNumSMs * 16)), dim3(256), 0, s, 
        r.cnt, r.dst_ptr, r.item_ptr, (const double*)sc.partial, in, 1, sp.n, mean, nullptr, 0);
    a.mean = mean;
    launch_agg<kOpMom2>(s, a, r.items_max);
    launch_pdl(k_finalize_moments, dim3(grid_for(r.D_max, 8, kNumSMs * 16)), dim3(256), 0, s, 
        r.cnt, r.dst_ptr, r.item_ptr, (const double*)sc.partial, in, 2, sp.n, nullptr, sc.agg, ld4(in));
  } else {  // sage_mean aggregate-first
    agg_fin<kOpSum>(s, a, f, r.items_max, r.D_max, split);
  }
  // relu([h_v | agg] @ [W_self; W_neigh])
  TcGemmArgs g = gemm_args(r.D_dev, L.tw_main, out, ldo, true);
  g.a1 = r.x;
  g.self = r.self;
  g.K1 = in;
  g.a2 = sc.agg;
  g.lda2 = ld4(in);
  g.K2 = in;
  gemm(s, g, r.D_max, r.cnt);
  return false;
}

// ---------------------------------------------------------------------------
// CGP building blocks (cgpexec.py:111-240): raw local partials, partition-
// ordered merge, update with explicit destination rows
// ---------------------------------------------------------------------------
int cgp_partial_width(const LayerDev& L) {
  const int w = (L.spec.kind == OB_KIND_GAT || L.transform_first) ? L.spec.out_dim : L.spec.in_dim;
  return L.spec.kind == OB_KIND_GAT ? w + 2 : w;
}

// merge a destination's items (or hub groups) into one raw partial: sum / max /
// (max logit, sum exp, sum exp*z); count = local in-edges
__global__ void __launch_bounds__(256) k_local_raw(FinArgs a, float* lp, int64_t ldp, float* lcnt) {
  pdl_wait();
  const int64_t D = cta_ld(&a.cnt->D);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < D; i += nw) {
    int64_t i0 = a.item_ptr[i], i1 = a.item_ptr[i + 1];
    const float* part = a.partial;
    if (a.group_ptr && a.group_ptr[i + 1] > a.group_ptr[i]) {
      i0 = a.group_ptr[i];
      i1 = a.group_ptr[i + 1];
      part = a.partial2;
    }
    float* o = lp + i * ldp;
    if (lane == 0) lcnt[i] = (float)(a.dst_ptr[i + 1] - a.dst_ptr[i]);
    const int mk = merge_kind(a.kind);
    const int hdr = mk == kMergeSoftmax ? kSmHdr : 0;
    const int oh = mk == kMergeSoftmax ? 2 : 0;  // rank-partial layout: [max, sum exp | values]
    float ms = 0.f, den = 0.f;
    if (mk == kMergeSoftmax) {
      sm_header<false>(part, a.pw, i0, i1, ms, den);
      if (lane == 0) {
        o[0] = ms;
        o[1] = den;
      }
    }
    const float* st = nullptr;  // this partition's stored CSR-part sum (sum kinds, layer 1)
    if (a.stat) {
      const int64_t v = a.stat_dst_ids[i];
      if (v < a.stat_N) st = a.stat + v * a.stat_ld;
    }
    for (int c4 = lane * 4; c4 < a.width; c4 += 128) {
      float4 v = merge_cols<false>(mk, part, a.pw, i0, i1, hdr, c4, ms);
      if (st) {
        const float4 q = ld4f(st + c4);
        v = make_float4(q.x + v.x, q.y + v.y, q.z + v.z, q.w + v.w);
      }
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (c4 + t < a.width) o[oh + c4 + t] = vv[t];
    }
  }
}

// float64 raw sums for the moments kind (items carry float64 partials)
__global__ void __launch_bounds__(256) k_local_raw_f64(const BlockCounters* cnt_, const int64_t* dst_ptr,
                                                       const int64_t* item_ptr, const double* partial, int width,
                                                       double* lp, int64_t ldp, float* lcnt) {
  pdl_wait();
  const int64_t D = cta_ld(&cnt_->D);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < D; i += nw) {
    if (lane == 0) lcnt[i] = (float)(dst_ptr[i + 1] - dst_ptr[i]);
    for (int col = lane; col < width; col += 32) {
      double s = 0.0;
      for (int64_t it = item_ptr[i]; it < item_ptr[i + 1]; ++it) s += partial[it * (int64_t)width + col];
      lp[i * ldp + col] = s;
    }
  }
}

struct MergeArgs {
  int P;
  PartPtrs parts;             // partition p's partial rows / counts (local or a peer's, over NVLink)
  int64_t ldp;
  const int64_t* D_dev;
  OwnerFilter own;            // NCCL mode: merge only the destinations this rank owns
  int width, kind;
  float p;
  int n;
  bool gcn_norm, relu;
  float* out;
  int64_t ldo;
};

// merge in ascending partition order (cgpexec.py:189-240): sum / mean / max / powmean /
// softmax rescale, empty destinations aggregate to zero
__global__ void __launch_bounds__(256) k_merge_parts(MergeArgs m) {
  pdl_wait();
  const int64_t D = cta_ld(m.D_dev);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < D; i += nw) {
    if (!m.own.mine(i)) continue;
    float c = 0.f;
    for (int p = 0; p < m.P; ++p) c += __ldcg(m.parts.cnt[p] + i);
    float ms = -INFINITY;
    if (m.kind == OB_KIND_GAT) {
      for (int p = 0; p < m.P; ++p) {
        const float* o = m.parts.lp[p] + i * m.ldp;
        if (__ldcg(o + 1) > 0.f) ms = fmaxf(ms, __ldcg(o));
      }
    }
    for (int col = lane; col < m.width; col += 32) {
      float r;
      if (m.kind == OB_KIND_GAT) {
        float den = 0.f, num = 0.f;
        for (int p = 0; p < m.P; ++p) {
          const float* o = m.parts.lp[p] + i * m.ldp;
          if (__ldcg(o + 1) > 0.f) {
            const float sc = __expf(__ldcg(o) - ms);
            den += __ldcg(o + 1) * sc;
            num += __ldcg(o + 2 + col) * sc;
          }
        }
        r = den > 0.f ? num / den : 0.f;
      } else if (m.kind == OB_KIND_SAGE_MAX) {
        float mx = -INFINITY;
        for (int p = 0; p < m.P; ++p)
          if (__ldcg(m.parts.cnt[p] + i) > 0.f) mx = fmaxf(mx, __ldcg(m.parts.lp[p] + i * m.ldp + col));
        r = c > 0.f ? mx : 0.f;
      } else {
        float s = 0.f;
        for (int p = 0; p < m.P; ++p) s += __ldcg(m.parts.lp[p] + i * m.ldp + col);
        if (m.gcn_norm) r = s / sqrtf(c + 1.f);
        else if (m.kind == OB_KIND_POWER_MEAN) r = c > 0.f ? powf(s / c, 1.f / m.p) : 0.f;
        else r = c > 0.f ? s / c : 0.f;
      }
      if (m.relu) r = fmaxf(r, 0.f);
      m.out[i * m.ldo + col] = r;
    }
  }
}

__global__ void __launch_bounds__(256) k_merge_moments(int P, PartPtrs parts, int64_t ldp, const int64_t* D_dev,
                                                       OwnerFilter own, int width, int phase, int n, double* mean,
                                                       float* agg, int64_t ldo) {
  pdl_wait();
  const int64_t D = cta_ld(D_dev);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < D; i += nw) {
    if (!own.mine(i)) continue;
    float c = 0.f;
    for (int p = 0; p < P; ++p) c += __ldcg(parts.cnt[p] + i);
    for (int col = lane; col < width; col += 32) {
      double s = 0.0;
      for (int p = 0; p < P; ++p)
        s += __ldcg(reinterpret_cast<const double*>(parts.lp[p]) + i * ldp + col);
      const double v = c > 0.f ? s / (double)c : 0.0;
      if (phase == 1) {
        mean[i * width + col] = v;
      } else {
        const double r = (n & 1) ? copysign(pow(fabs(v), 1.0 / n), v) : pow(fmax(v, 0.0), 1.0 / n);
        agg[i * ldo + col] = (float)r;
      }
    }
  }
}

void launch_resolve(cudaStream_t s, const BindCtx& c, BlockCounters* cnt, int64_t S_max, const int32_t* src_ids,
                    const float** rowp, float* gscale) {
  launch_pdl(k_resolve, dim3(grid_for(S_max, 256)), dim3(256), 0, s, c, cnt, src_ids, rowp, gscale, nullptr, nullptr);
}

void cgp_local_partial(cudaStream_t s, const LayerDev& L, const LayerRun& r, const LayerScratch& sc,
                       const float* s_dst, float* lp, int64_t ldp, float* lcnt, int moments_phase,
                       const double* mean) {
  const ob_layer& sp = L.spec;
  const int in = sp.in_dim, outd = sp.out_dim;
  const int64_t ld_out = ld4(outd);
  AggArgs a{};
  a.cnt = r.cnt;
  a.S_max = r.S_max;
  a.dst_ptr = r.dst_ptr;
  a.item_ptr = r.item_ptr;
  a.item_dst = r.item_dst;
  a.edge_src = r.edge_src;
  a.x = r.x;
  a.width = in;
  a.pw = sp.kind == OB_KIND_MOMENTS ? in : ld4(in);
  a.partial = sc.partial;
  a.p = sp.p;
  a.n = sp.n;
  if (r.stat) {  // stored CSR-part sums of this partition: gather only the request suffix
    a.skip_dst_ids = r.dst_ids;
    a.skip_indeg = r.indeg;
    a.skip_N = r.N;
  }
  RowSrc zrows{nullptr, sc.z, ld_out};
  if ((sp.kind == OB_KIND_GAT || L.transform_first) && r.yrow) {
    // stored transforms: owned training rows from the table, the listed rows (this
    // partition's queries) through a GEMM
    TcGemmArgs g = gemm_args(r.ndyn, L.tw_main, sc.z, ld_out, false);
    g.a1 = r.x;
    g.self = r.dyn_src;
    g.K1 = in;
    gemm(s, g, r.dyn_max, nullptr);
    zrows = RowSrc{r.yrow, nullptr, 0};
    a.x = zrows;
    a.width = outd;
    a.pw = ld4(outd);
  } else if (sp.kind == OB_KIND_GAT || L.transform_first) {
    TcGemmArgs g = gemm_args(r.S_dev, L.tw_main, sc.z, ld_out, false);
    g.a1 = r.x;
    g.K1 = in;
    gemm(s, g, r.S_max, r.cnt);
    a.x = zrows;
    a.width = outd;
    a.pw = ld4(outd);
  }
  if (sp.kind == OB_KIND_MOMENTS) {
    a.mean = mean;
    if (moments_phase == 1) launch_agg<kOpDSum>(s, a, r.items_max);
    else launch_agg<kOpMom2>(s, a, r.items_max);
    launch_pdl(k_local_raw_f64, dim3(grid_for(r.D_max, 8, kNumSMs * 16)), dim3(256), 0, s, r.cnt, r.dst_ptr, r.item_ptr,
                                                                        (const double*)sc.partial, in, (double*)lp,
                                                                        ldp, lcnt);
    return;
  }
  if (sp.kind == OB_KIND_GAT) {
    launch_pdl(k_rowdot_rows, dim3(grid_for(r.S_max, 8)), dim3(256), 0, s, r.S_dev, zrows, nullptr, outd, L.a_src, sc.s_src);
    a.pw = kSmHdr + ld4(outd);
    a.s_src = sc.s_src;
    a.s_dst = s_dst;
    launch_agg<kOpSoftmax>(s, a, r.items_max);
  } else if (sp.kind == OB_KIND_GCN) {
    a.gscale = r.gscale;
    launch_agg<kOpSum>(s, a, r.items_max);
  } else if (sp.kind == OB_KIND_SAGE_MAX) {
    launch_agg<kOpMax>(s, a, r.items_max);
  } else if (sp.kind == OB_KIND_POWER_MEAN) {
    launch_agg<kOpPow>(s, a, r.items_max);
  } else {
    launch_agg<kOpSum>(s, a, r.items_max);
  }
  FinArgs f{};
  f.cnt = r.cnt;
  f.dst_ptr = r.dst_ptr;
  f.item_ptr = r.item_ptr;
  f.group_dst = r.group_dst;
  f.partial = sc.partial;
  f.partial2 = sc.partial2;
  f.group_ptr = r.group_ptr;
  f.pw = a.pw;
  f.width = a.width;
  f.kind = sp.kind;
  if (r.stat) {
    f.stat = r.stat;
    f.stat_ld = r.stat_ld;
    f.stat_dst_ids = r.dst_ids;
    f.stat_N = r.N;
  }
  launch_pdl(k_reduce_groups, dim3(grid_for(r.items_max / kItemGroup + 1, 8, kNumSMs * 16)), dim3(256), 0, s, f);
  launch_pdl(k_local_raw, dim3(grid_for(r.D_max, 8, kNumSMs * 16)), dim3(256), 0, s, f, lp, ldp, lcnt);
}

void cgp_merge(cudaStream_t s, const LayerDev& L, int P, const PartPtrs& parts, int64_t ldp, const OwnerFilter& own,
               const int64_t* D_dev, int64_t D_max, float* agg, float* out, int64_t ldo, int moments_phase,
               double* mean) {
  const ob_layer& sp = L.spec;
  if (sp.kind == OB_KIND_MOMENTS) {  // float64 partials, ldp counts float64 elements
    launch_pdl(k_merge_moments, dim3(grid_for(D_max, 8, kNumSMs * 16)), dim3(256), 0, s, P, parts, ldp, D_dev, own, sp.in_dim,
                                                                      moments_phase, sp.n, mean, agg, ld4(sp.in_dim));
    return;
  }
  MergeArgs m{};
  m.P = P;
  m.parts = parts;
  m.ldp = ldp;
  m.own = own;
  m.D_dev = D_dev;
  m.kind = sp.kind;
  m.p = sp.p;
  m.n = sp.n;
  const bool narrow = sp.kind == OB_KIND_GAT || L.transform_first;
  m.width = narrow ? sp.out_dim : sp.in_dim;
  m.gcn_norm = sp.kind == OB_KIND_GCN;
  if (sp.kind == OB_KIND_GAT || (sp.kind == OB_KIND_GCN && L.transform_first)) {
    m.relu = true;  // relu(agg) is the layer output
    m.out = out;
    m.ldo = ldo;
  } else {
    m.out = agg;
    m.ldo = ld4(m.width);
  }
  launch_pdl(k_merge_parts, dim3(grid_for(D_max, 8, kNumSMs * 16)), dim3(256), 0, s, m);
}

void cgp_update(cudaStream_t s, const LayerDev& L, const int64_t* D_dev, int64_t D_max, const float* const* hvp,
                const float* agg, float* out, int64_t ldo) {
  const ob_layer& sp = L.spec;
  const int in = sp.in_dim;
  if (sp.kind == OB_KIND_GAT || (sp.kind == OB_KIND_GCN && L.transform_first)) return;  // merged directly
  if (sp.kind == OB_KIND_GCN) {
    TcGemmArgs g = gemm_args(D_dev, L.tw_main, out, ldo, true);
    g.a2 = agg;
    g.lda2 = ld4(in);
    g.K2 = in;
    gemm(s, g, D_max, nullptr);
    return;
  }
  if (sp.kind == OB_KIND_SAGE_MEAN && L.transform_first) {
    TcGemmArgs g = gemm_args(D_dev, L.tw_self, out, ldo, true);
    g.a1 = RowSrc{hvp, nullptr, 0};
    g.K1 = in;
    g.E = agg;
    g.lde = ld4(sp.out_dim);
    gemm(s, g, D_max, nullptr);
    return;
  }
  TcGemmArgs g = gemm_args(D_dev, L.tw_main, out, ldo, true);
  g.a1 = RowSrc{hvp, nullptr, 0};
  g.K1 = in;
  g.a2 = agg;
  g.lda2 = ld4(in);
  g.K2 = in;
  gemm(s, g, D_max, nullptr);
}

// ---------------------------------------------------------------------------
// serving forward over the request's blocks
// ---------------------------------------------------------------------------
BindCtx bind_ctx(Engine& e, RequestWs& w, int l) {
  const bool full = khop(e.cfg);
  const LayerDev& L = e.layers[l - 1];
  BindCtx c{};
  c.mode = full ? 1 : 0;
  c.layer = l;
  c.N = e.g.N;
  c.F_ld = e.g.F_ld;
  c.pos = e.g.pos;
  c.feats = e.g.feats;
  c.qfeat = w.qpad;
  c.pe = (!full && l > 1) ? e.pe[l - 2] : nullptr;
  c.prev = l > 1 ? w.outs[l - 1] : nullptr;
  c.in_ld = ld4(L.spec.in_dim);
  c.cbits = w.cbits;
  c.cwpre = w.cwpre;
  c.tpos = w.cand_tpos;
  c.indeg = e.g.indeg;
  c.qdeg = w.qdeg;
  c.T_dev = &w.rc->T;
  return c;
}

__global__ void k_pad_rows(const ReqParams* rp, int64_t rows, int w, float* dst, int64_t ld) {
  pdl_wait();
  const float* __restrict__ src = rp->qfeat;
  const int64_t n = rows * ld;
  OB_GRID_STRIDE(i, n) {
    const int64_t r = i / ld;
    const int c = (int)(i - r * ld);
    dst[i] = c < w ? src[r * w + c] : 0.f;
  }
}

// delta rows of the recomputed targets: dbuf[t] = prev[t] - PE[targets[t]] (t < T)
__global__ void k_delta_rows(const int64_t* T_dev, const int32_t* __restrict__ targets, const float* __restrict__ prev,
                             const float* __restrict__ pe, int64_t ld, float* dbuf) {
  pdl_wait();
  const int64_t n = cta_ld(T_dev) * ld;
  OB_GRID_STRIDE(t, n) {
    const int64_t i = t / ld;
    const int64_t c = t - i * ld;
    dbuf[t] = prev[t] - pe[(int64_t)targets[i] * ld + c];
  }
}

void stage_forward(Engine& e, RequestWs& w, float* d_out) {
  cudaStream_t s = e.stream;
  const int k = (int)e.layers.size();
  // stage query features with 16 B aligned rows (unless staged early, stage_query_rows)
  if (!w.qpad_ready) {
    launch_pdl(k_pad_rows, dim3(grid_for((int64_t)w.B * e.g.F_ld, 256)), dim3(256), 0, s, w.rp, w.B, e.g.F, w.qpad, e.g.F_ld);
  }
  bool delta_ready = false;  // the previous layer's epilogue wrote this layer's delta rows
  for (int l = 1; l <= k; ++l) {
    const LayerDev& L = e.layers[l - 1];
    BlockDev& b = w.blocks[w.block_of_layer[l - 1]];
    BindCtx c = bind_ctx(e, w, l);
    const bool yt = e.ytab_ready && l - 1 < (int)e.ytab.size() && e.ytab[l - 1];
    if (yt) {
      c.ytab = e.ytab[l - 1];
      c.y_ld = ld4(L.spec.out_dim);
      c.yrow = w.yrow;
      c.ydyn = w.z;
      c.dyn_src = w.dyn_src;
      c.ndyn = w.ndyn;
      if (l == 1 && w.qrows_ready) c.qxw = w.qxw;  // layer 1: queries are the only non-table sources
      OB_CUDA(cudaMemsetAsync(w.ndyn, 0, sizeof(int64_t), s));
    }
    launch_pdl(k_resolve, dim3(grid_for(b.S_max, 256)), dim3(256), 0, s, c, b.cnt, (const int32_t*)b.src_ids, w.rowp,
               w.gscale, (uint8_t*)nullptr, (int32_t*)nullptr);
    LayerRun r{};
    if (yt) {
      r.yrow = w.yrow;
      r.dyn_src = w.dyn_src;
      r.ndyn = w.ndyn;
      r.dyn_max = b.S_max;
      r.no_dyn = l == 1 && w.qrows_ready;
      if (l - 1 < (int)e.stab.size() && e.stab[l - 1]) {
        r.ytab = e.ytab[l - 1];
        r.ytab_rows = e.g.N;
        r.ytab_ld = ld4(L.spec.out_dim);
        r.stab = e.stab[l - 1];
      }
    }
    if (l == 1 && e.yself1) {
      r.self_tab = e.yself1;
      r.dst_ids = b.dst_ids;
      r.N = e.g.N;
      r.qpad = w.qpad;
      r.q_ld = e.g.F_ld;
      r.B_dev = &w.blocks[(int)w.blocks.size() - 1].cnt->D;  // the query block: D = B
      r.B = w.B;
      if (w.qrows_ready) r.self_q = w.qself;
    }
    if (l > 1 && l < k && (int)e.sagg_l.size() >= l && e.sagg_l[l - 1] && w.delta) {
      // delta aggregates: static CSR-part sums of the stored rows + (h - PE) of recomputed sources
      const int64_t ld = ld4(L.spec.in_dim);
      if (!delta_ready) {
        launch_pdl(k_delta_rows, dim3(grid_for(b.D_max * ld, 256)), dim3(256), 0, s, &w.rc->T, w.targets, w.outs[l - 1], e.pe[l - 2],
                                                                   ld, w.delta);
      }
      r.delta = true;
      r.dprev = w.outs[l - 1];
      r.dT = &w.rc->T;
      r.dbuf = w.delta;
      r.stat = e.sagg_l[l - 1];
      r.stat_ld = ld;
      r.dst_ids = b.dst_ids;
      r.indeg = e.g.indeg;
      r.N = e.g.N;
    }
    // the next layer aggregates by deltas: this layer's merge epilogue may write them
    if (l + 1 < k && (int)e.sagg_l.size() > l && e.sagg_l[l] && w.delta) {
      r.dnext = w.delta;
      r.dnext_pe = e.pe[l - 1];
      r.dnext_T = &w.rc->T;
      r.dst_ids = b.dst_ids;
    }
    if (l == 1 && e.sagg1) {
      r.stat = e.sagg1;
      r.stat_ld = L.spec.kind == OB_KIND_GAT ? kSmHdr + ld4(L.spec.out_dim)
                                             : ld4(L.transform_first ? L.spec.out_dim : L.spec.in_dim);
      r.dst_ids = b.dst_ids;
      r.indeg = e.g.indeg;
      r.N = e.g.N;
    }
    r.cnt = b.cnt;
    r.D_dev = &b.cnt->D;
    r.S_dev = &b.cnt->S;
    r.D_max = b.D_max;
    r.S_max = b.S_max;
    r.items_max = b.items_max;
    r.dst_ptr = b.dst_ptr;
    r.item_ptr = b.item_ptr;
    r.item_dst = b.item_dst;
    r.group_dst = b.group_dst;
    r.edge_src = b.edge_src;
    r.self = b.self_src;
    r.x = RowSrc{w.rowp, nullptr, 0};
    r.gscale = w.gscale;
    r.group_ptr = b.group_ptr;
    // with several requests in flight, big sum gathers run as L2-sized source-range passes
    r.split_gather = e.nlanes > 1;
    LayerScratch sc{w.partial, w.partial2, w.agg, w.mean, w.z, w.s_src, w.s_dst};
    const bool last = l == k;
    float* out = last ? d_out : w.outs[l];
    delta_ready = run_layer(s, L, r, sc, out, last ? L.spec.out_dim : ld4(L.spec.out_dim));
  }
}

// Layer-1 query rows ahead of the block builds: padded features and, for layers with
// stored transforms, x_q W (and x_q W_self for the SAGE own-row table) over the B queries.
// Launched on the main stream beside the request-index sort, off the critical path.
void stage_query_rows(Engine& e, RequestWs& w) {
  cudaStream_t s = e.stream;
  w.qrows_ready = false;
  launch_pdl(k_pad_rows, dim3(grid_for((int64_t)w.B * e.g.F_ld, 256)), dim3(256), 0, s, w.rp, w.B, e.g.F, w.qpad, e.g.F_ld);
  w.qpad_ready = true;
  const LayerDev& L = e.layers[0];
  const bool yt = e.ytab_ready && !e.ytab.empty() && e.ytab[0] && w.qxw;
  const int64_t ld = ld4(L.spec.out_dim);
  if (yt) {
    TcGemmArgs g = gemm_args(&w.rp->B, L.tw_main, w.qxw, ld, false);
    g.a1 = RowSrc{nullptr, w.qpad, e.g.F_ld};
    g.K1 = L.spec.in_dim;
    gemm(s, g, w.B, nullptr);
  }
  if (yt && e.yself1) {
    TcGemmArgs g = gemm_args(&w.rp->B, L.tw_self, w.qself, ld, false);
    g.a1 = RowSrc{nullptr, w.qpad, e.g.F_ld};
    g.K1 = L.spec.in_dim;
    gemm(s, g, w.B, nullptr);
  }
  w.qrows_ready = yt;
}

void stage_qpad(Engine& e, RequestWs& w) {
  launch_pdl(k_pad_rows, dim3(grid_for((int64_t)w.B * e.g.F_ld, 256)), dim3(256), 0, e.stream, w.rp, w.B, e.g.F, w.qpad, e.g.F_ld);
}

// parity export of bind_kind / bind_pe_layer with the same binding rule
void export_bindings(Engine& e, RequestWs& w, BlockDev& b, int layer, uint8_t* d_kind, int32_t* d_pe_layer) {
  BindCtx c = bind_ctx(e, w, layer);
  launch_pdl(k_resolve, dim3(grid_for(b.S_max, 256)), dim3(256), 0, e.stream, c, b.cnt, b.src_ids, w.rowp, nullptr, d_kind, d_pe_layer);
}

// raw CSR-part sum per node: out[v] = sum_{u in N(v)} w_u x_u (w_u = 1/sqrt(deg u + 1) for gcn),
// warp per node, 4 columns per lane, rows in CSR order
__global__ void k_sagg_build(int64_t N, const int64_t* __restrict__ off, const int32_t* __restrict__ nbrs,
                             RowSrc x, int width, const int32_t* __restrict__ indeg, bool gcn, float* out,
                             int64_t ld, const int32_t* __restrict__ pos = nullptr) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < N; v += nw) {
    for (int c4 = lane * 4; c4 < ld; c4 += 128) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        const int32_t u = __ldg(nbrs + e);
        const float wgt = gcn ? (float)(1.0 / sqrt((double)__ldg(indeg + u) + 1.0)) : 1.f;
        const int64_t ru = pos ? (int64_t)__ldg(pos + u) : u;  // stored row of u (owned rows under CGP)
        const float4 q = c4 < width ? __ldg(reinterpret_cast<const float4*>(x.row(ru) + c4))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        acc.x = fmaf(wgt, q.x, acc.x);
        acc.y = fmaf(wgt, q.y, acc.y);
        acc.z = fmaf(wgt, q.z, acc.z);
        acc.w = fmaf(wgt, q.w, acc.w);
      }
      *reinterpret_cast<float4*>(out + v * ld + c4) = acc;
    }
  }
}

// GAT layer 1: the CSR part's softmax triple per node (max logit, sum exp,
// sum exp * z_u) with logit = leaky_relu_0.2(s_src[u] + z_v . a_dst) -- the
// destination score of a training node is static at layer 1 (models.py:199-206)
__global__ void k_sagg_gat_build(int64_t N, const int64_t* __restrict__ off, const int32_t* __restrict__ nbrs,
                                 const float* __restrict__ z, int64_t zld, int width, const float* __restrict__ ssrc,
                                 const float* __restrict__ a_dst, float* out, int64_t ld) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < N; v += nw) {
    float sd = 0.f;
    for (int c = lane; c < width; c += 32) sd = fmaf(z[v * zld + c], a_dst[c], sd);
    for (int o = 16; o; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
    const int64_t e0 = off[v], e1 = off[v + 1];
    float m = -INFINITY;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const float lg = ssrc[nbrs[e]] + sd;
      m = fmaxf(m, lg >= 0.f ? lg : 0.2f * lg);
    }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float den = 0.f;
    for (int c4 = lane * 4; c4 < ld - kSmHdr; c4 += 128) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      float dd = 0.f;
      for (int64_t e = e0; e < e1; ++e) {
        const int32_t u = __ldg(nbrs + e);
        const float lg0 = ssrc[u] + sd;
        const float p = __expf((lg0 >= 0.f ? lg0 : 0.2f * lg0) - m);
        dd += p;
        const float4 q = c4 < width ? __ldg(reinterpret_cast<const float4*>(z + (int64_t)u * zld + c4))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        acc.x = fmaf(p, q.x, acc.x);
        acc.y = fmaf(p, q.y, acc.y);
        acc.z = fmaf(p, q.z, acc.z);
        acc.w = fmaf(p, q.w, acc.w);
      }
      den = dd;
      *reinterpret_cast<float4*>(out + v * ld + kSmHdr + c4) = acc;
    }
    if (lane == 0) {
      out[v * ld] = e1 > e0 ? m : -INFINITY;
      out[v * ld + 1] = e1 > e0 ? den : 0.f;
      out[v * ld + 2] = 0.f;
      out[v * ld + 3] = 0.f;
    }
  }
}

// ---------------------------------------------------------------------------
// CGP ranks: layer-1 tables over the rows and edges a partition stores
//   * stored transforms (GAT / transform-first layer 1): x_u W for every stored
//     feature row (owned rows under NCCL partitioned storage, through pos)
//   * stored aggregates (sum kinds, layer 1): per local partition p, the CSR-part
//     sum over its source-split CSR, sum_{u in N_p(v)} w_u x_u (W), for every
//     destination v; a request then gathers only its slice's request spans
// Tables are skipped when they would take more than a third of free HBM (the
// papers-shaped cfg4: N x H per partition does not fit).
// ---------------------------------------------------------------------------
static void build_cgp_tables(Engine& e) {
  const char* off = std::getenv("OB_NO_STORED_TRANSFORMS");
  if ((off && off[0] && off[0] != '0') || !e.g.feats || e.layers.empty()) return;
  cudaStream_t s = e.stream;
  const LayerDev& L1 = e.layers[0];
  const int64_t N = e.g.N;
  const int64_t rows = e.g.pos ? e.g.N_local : N;
  const int k = (int)e.layers.size();
  e.ytab.assign(k, nullptr);
  size_t fb = 0, tb = 0;
  int64_t* n_dev = (int64_t*)e.dalloc(sizeof(int64_t));
  OB_CUDA(cudaMemcpyAsync(n_dev, &rows, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  if (L1.spec.kind == OB_KIND_GAT || L1.transform_first) {
    const int64_t ld = ld4(L1.spec.out_dim);
    OB_CUDA(cudaMemGetInfo(&fb, &tb));
    if ((size_t)rows * ld * 4 <= fb / 3) {
      e.ytab[0] = (float*)e.dalloc(sizeof(float) * std::max<int64_t>(rows, 1) * ld);
      TcGemmArgs g = gemm_args(n_dev, L1.tw_main, e.ytab[0], ld, false);
      g.a1 = RowSrc{nullptr, e.g.feats, e.g.F_ld};
      g.K1 = L1.spec.in_dim;
      tc_gemm(s, g, rows);
    }
  }
  const char* off_sa = std::getenv("OB_NO_STORED_AGGREGATES");
  const bool sa_off = off_sa && off_sa[0] && off_sa[0] != '0';
  const bool sum_kind = L1.spec.kind == OB_KIND_GCN || L1.spec.kind == OB_KIND_SAGE_MEAN;
  if (sum_kind && !sa_off && (!L1.transform_first || e.ytab[0])) {
    const int w = L1.transform_first ? L1.spec.out_dim : L1.spec.in_dim;
    const int64_t ld = ld4(w);
    OB_CUDA(cudaMemGetInfo(&fb, &tb));
    if ((size_t)N * ld * 4 * e.cgp.parts.size() <= fb / 3) {
      const RowSrc x = L1.transform_first ? RowSrc{nullptr, e.ytab[0], ld} : RowSrc{nullptr, e.g.feats, e.g.F_ld};
      for (auto& part : e.cgp.parts) {
        float* t = (float*)e.dalloc(sizeof(float) * N * ld);
        launch_pdl(k_sagg_build, dim3(grid_for(N, 8, kNumSMs * 16)), dim3(256), 0, s, N, part.off, part.src, x, w, e.g.indeg,
                                                                     L1.spec.kind == OB_KIND_GCN, t, ld, e.g.pos);
        e.cgp_sagg1.push_back(t);
      }
    }
  }
  OB_CUDA(cudaStreamSynchronize(s));
  e.dfree(n_dev);
}

// ---------------------------------------------------------------------------
// stored transforms: x_v W for every training node whose layer input is static
// ---------------------------------------------------------------------------
void build_stored_transforms(Engine& e) {
  if (e.ytab_ready) return;
  e.ytab_ready = true;  // decided once per (model, PE) state; tables may stay empty
  const char* off = std::getenv("OB_NO_STORED_TRANSFORMS");
  if (off && off[0] && off[0] != '0') return;
  if (e.cfg.strategy == OB_STRATEGY_SRPE_CGP) return build_cgp_tables(e);
  if (e.g.pos || !e.g.feats) return;  // centralized, full tables
  const int k = (int)e.layers.size();
  const int64_t N = e.g.N;
  std::vector<int> want(k, 0);
  size_t bytes = 0;
  for (int l = 1; l <= k; ++l) {
    const LayerDev& L = e.layers[l - 1];
    if (!(L.spec.kind == OB_KIND_GAT || L.transform_first)) continue;
    const bool stat_in = l == 1 || (!khop(e.cfg) && (int)e.pe.size() >= l - 1 && e.pe[l - 2]);
    if (!stat_in) continue;
    want[l - 1] = 1;
    bytes += (size_t)N * ld4(L.spec.out_dim) * 4;
  }
  size_t free_b = 0, total_b = 0;
  OB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  if (bytes > free_b / 3) want.assign(k, 0);  // keep room for request workspaces
  cudaStream_t s = e.stream;
  int64_t* n_dev = (int64_t*)e.dalloc(sizeof(int64_t));
  OB_CUDA(cudaMemcpyAsync(n_dev, &N, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  e.ytab.assign(k, nullptr);
  e.stab.assign(k, nullptr);
  for (int l = 1; l <= k; ++l) {
    if (!want[l - 1]) continue;
    const LayerDev& L = e.layers[l - 1];
    const int64_t ld = ld4(L.spec.out_dim);
    float* t = (float*)e.dalloc(sizeof(float) * N * ld);
    TcGemmArgs g = gemm_args(n_dev, L.tw_main, t, ld, false);
    g.a1 = l == 1 ? RowSrc{nullptr, e.g.feats, e.g.F_ld} : RowSrc{nullptr, e.pe[l - 2], ld4(L.spec.in_dim)};
    g.K1 = L.spec.in_dim;
    tc_gemm(s, g, N);
    e.ytab[l - 1] = t;
    // GAT, wide rows: the stored rows' source scores (k_rowdot_rows, same arithmetic).  Measured:
    // H = 512 (Amazon-shaped) p50 1.04 -> 0.85 ms; at H = 128 (cfg3) the per-request dot products
    // are cheap and warm L2 with the rows the gather reads next (p50 0.324 -> 0.348 ms without them)
    static const bool stab_off = [] {
      const char* v = std::getenv("OB_NO_GAT_SCORE_TABLE");
      return v && v[0] && v[0] != '0';
    }();
    if (L.spec.kind == OB_KIND_GAT && L.spec.out_dim >= 256 && !stab_off) {
      float* st = (float*)e.dalloc(sizeof(float) * N);
      launch_pdl(k_rowdot_rows, dim3(grid_for(N, 8)), dim3(256), 0, s, (const int64_t*)n_dev, RowSrc{nullptr, t, ld},
                 (const int32_t*)nullptr, L.spec.out_dim, (const float*)L.a_src, st);
      e.stab[l - 1] = st;
    }
  }
  // own-row transform of a transform-first SAGE layer 1 (its destinations' x_v W_self)
  const LayerDev& L1 = e.layers[0];
  if (L1.spec.kind == OB_KIND_SAGE_MEAN && L1.transform_first && e.ytab[0] &&
      (e.cfg.strategy == OB_STRATEGY_SRPE || e.cfg.strategy == OB_STRATEGY_FULL)) {
    const int64_t ld = ld4(L1.spec.out_dim);
    size_t fb = 0, tb = 0;
    OB_CUDA(cudaMemGetInfo(&fb, &tb));
    if ((size_t)N * ld * 4 <= fb / 3) {
      e.yself1 = (float*)e.dalloc(sizeof(float) * N * ld);
      TcGemmArgs g = gemm_args(n_dev, L1.tw_self, e.yself1, ld, false);
      g.a1 = RowSrc{nullptr, e.g.feats, e.g.F_ld};
      g.K1 = L1.spec.in_dim;
      tc_gemm(s, g, N);
    }
  }
  // stored aggregates of layer 1 (srpe / full: block-1 rows are CSR ++ request)
  {
    const char* off_g = std::getenv("OB_NO_STORED_AGGREGATES");
    const bool rows_full_g = e.cfg.strategy == OB_STRATEGY_SRPE || e.cfg.strategy == OB_STRATEGY_FULL;
    if (L1.spec.kind == OB_KIND_GAT && rows_full_g && !(off_g && off_g[0] && off_g[0] != '0') && e.g.offsets &&
        e.ytab[0]) {  // softmax triple over the CSR part
      const int w = L1.spec.out_dim;
      const int64_t zld = ld4(w), ld = kSmHdr + ld4(w);
      size_t fb = 0, tb = 0;
      OB_CUDA(cudaMemGetInfo(&fb, &tb));
      if ((size_t)N * (ld + 1) * 4 <= fb / 3) {
        float* ssrc = (float*)e.dalloc(sizeof(float) * N);
        launch_pdl(k_rowdot_rows, dim3(grid_for(N, 8)), dim3(256), 0, s, n_dev, RowSrc{nullptr, e.ytab[0], zld}, nullptr, w, L1.a_src,
                   ssrc);
        e.sagg1 = (float*)e.dalloc(sizeof(float) * N * ld);
        launch_pdl(k_sagg_gat_build, dim3(grid_for(N, 8, kNumSMs * 16)), dim3(256), 0, s, N, e.g.offsets, e.g.nbrs, e.ytab[0], zld, w,
                                                                        ssrc, L1.a_dst, e.sagg1, ld);
        OB_CUDA(cudaStreamSynchronize(s));
        e.dfree(ssrc);
      }
    }
  }
  const bool sum_kind = L1.spec.kind == OB_KIND_GCN || L1.spec.kind == OB_KIND_SAGE_MEAN;
  const bool rows_full = e.cfg.strategy == OB_STRATEGY_SRPE || e.cfg.strategy == OB_STRATEGY_FULL;
  const char* off_sa = std::getenv("OB_NO_STORED_AGGREGATES");
  const bool sa_off = off_sa && off_sa[0] && off_sa[0] != '0';
  if (sum_kind && rows_full && !sa_off && e.g.offsets && (!L1.transform_first || e.ytab[0])) {
    const int w = L1.transform_first ? L1.spec.out_dim : L1.spec.in_dim;
    const int64_t ld = ld4(w);
    size_t fb = 0, tb = 0;
    OB_CUDA(cudaMemGetInfo(&fb, &tb));
    if ((size_t)N * ld * 4 <= fb / 3) {
      e.sagg1 = (float*)e.dalloc(sizeof(float) * N * ld);
      const RowSrc x = L1.transform_first ? RowSrc{nullptr, e.ytab[0], ld} : RowSrc{nullptr, e.g.feats, e.g.F_ld};
      launch_pdl(k_sagg_build, dim3(grid_for(N, 8, kNumSMs * 16)), dim3(256), 0, s, N, e.g.offsets, e.g.nbrs, x, w, e.g.indeg,
                                                                   L1.spec.kind == OB_KIND_GCN, e.sagg1, ld, (const int32_t*)nullptr);
    }
  }
  // delta aggregates of srpe mid-block layers l = 2..k-1 (aggregate-first sum kinds): the CSR-part
  // sum of the stored rows PE_{l-1} per node; a request then gathers only recomputed sources
  const char* off_d = std::getenv("OB_NO_DELTA_AGGREGATES");
  const bool d_off = sa_off || (off_d && off_d[0] && off_d[0] != '0');
  e.sagg_l.assign(k, nullptr);
  for (int l = 2; l < k && e.cfg.strategy == OB_STRATEGY_SRPE && !d_off && e.g.offsets; ++l) {
    const LayerDev& L = e.layers[l - 1];
    if (!(L.spec.kind == OB_KIND_GCN || L.spec.kind == OB_KIND_SAGE_MEAN) || L.transform_first) continue;
    if ((int)e.pe.size() < l - 1 || !e.pe[l - 2]) continue;
    const int w = L.spec.in_dim;
    const int64_t ld = ld4(w);
    size_t fb = 0, tb = 0;
    OB_CUDA(cudaMemGetInfo(&fb, &tb));
    if ((size_t)N * ld * 4 > fb / 3) continue;
    e.sagg_l[l - 1] = (float*)e.dalloc(sizeof(float) * N * ld);
    launch_pdl(k_sagg_build, dim3(grid_for(N, 8, kNumSMs * 16)), dim3(256), 0, s, N, e.g.offsets, e.g.nbrs, RowSrc{nullptr, e.pe[l - 2], ld},
                                                                 w, e.g.indeg, L.spec.kind == OB_KIND_GCN,
                                                                 e.sagg_l[l - 1], ld, (const int32_t*)nullptr);
  }
  OB_CUDA(cudaStreamSynchronize(s));
  e.dfree(n_dev);
}

// ---------------------------------------------------------------------------
// precompute_embeddings: layers 1..k-1 over the whole graph (graphstore.py:330-365)
// ---------------------------------------------------------------------------
__global__ void k_node_scale(const int32_t* __restrict__ indeg, int64_t N, float* sc) {
  pdl_wait();
  OB_GRID_STRIDE(v, N) sc[v] = (float)(1.0 / sqrt((double)indeg[v] + 1.0));
}

void stage_precompute(Engine& e) {
  cudaStream_t s = e.stream;
  const int k = (int)e.layers.size();
  OB_CHECK(k >= 2, OB_EINVAL, "stored embeddings need a model with k >= 2 layers");
  OB_CHECK(e.g.N > 0, OB_ESTATE, "load a graph first");
  const int64_t N = e.g.N, E = e.g.E;
  int maxw = 0;
  bool mom = false, wide = false;
  for (auto& L : e.layers) {
    maxw = std::max(maxw, ld4(std::max(L.spec.in_dim, L.spec.out_dim)) + kSmHdr);
    mom |= L.spec.kind == OB_KIND_MOMENTS;
    wide |= L.spec.kind == OB_KIND_GAT || L.transform_first;
  }
  const int64_t items_max = E / kAggChunk + N + 1;
  std::vector<void*> tmp;
  auto talloc = [&](size_t bytes) {
    void* p = nullptr;
    OB_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
    tmp.push_back(p);
    return p;
  };
  try {
    BlockCounters* cnt = (BlockCounters*)talloc(sizeof(BlockCounters));
    BlockCounters hc{};
    hc.D = N;
    hc.E = E;
    hc.S = N;
    OB_CUDA(cudaMemcpyAsync(cnt, &hc, sizeof(hc), cudaMemcpyHostToDevice, s));
    int64_t* item_ptr = (int64_t*)talloc(sizeof(int64_t) * (N + 1));
    float* partial = (float*)talloc(sizeof(float) * items_max * maxw * (mom ? 2 : 1));
    float* partial2 = (float*)talloc(sizeof(float) * (items_max / kItemGroup + N + 1) * maxw);
    int64_t* group_ptr = (int64_t*)talloc(sizeof(int64_t) * (N + 1));
    int32_t* item_dst = (int32_t*)talloc(sizeof(int32_t) * items_max);
    int32_t* group_dst = (int32_t*)talloc(sizeof(int32_t) * (items_max / kItemGroup + N + 1));
    float* agg = (float*)talloc(sizeof(float) * N * maxw);
    float* mean = mom ? (float*)talloc(sizeof(double) * N * maxw) : nullptr;
    float* z = wide ? (float*)talloc(sizeof(float) * N * maxw) : nullptr;
    float* s_src = (float*)talloc(sizeof(float) * N);
    float* s_dst = (float*)talloc(sizeof(float) * N);
    float* gscale = (float*)talloc(sizeof(float) * N);
    launch_pdl(k_node_scale, dim3(grid_for(N, 256)), dim3(256), 0, s, e.g.indeg, N, gscale);
    ScanScratch sc_scan;
    sc_scan.cap = ScanScratch::bytes_for(N, 1);
    sc_scan.pool = (char*)talloc(sc_scan.cap);
    OB_CUDA(cudaMemsetAsync(sc_scan.pool, 0, sc_scan.cap, s));
    // dst_ptr = the graph's offsets
    const BlockStore3 bst{nullptr, item_ptr, group_ptr};
    device_scan_t<I3>(s, sc_scan, OffsetsLoad3{e.g.offsets}, bst, BlockTotal3{bst, cnt}, nullptr, N, N);
    expand_items(s, cnt, N, item_ptr, group_ptr, item_dst, group_dst);
    for (float* t : e.pe) e.dfree(t);  // replaced below
    e.pe.assign(k - 1, nullptr);
    e.pe_dim.assign(k - 1, 0);
    const float* h = e.g.feats;
    int64_t hld = e.g.F_ld;
    int hw = e.g.F;
    for (int l = 1; l < k; ++l) {
      const LayerDev& L = e.layers[l - 1];
      OB_CHECK(L.spec.in_dim == hw, OB_EINVAL, "model input width does not match the stored rows");
      const int64_t old = ld4(L.spec.out_dim);
      float* out = (float*)e.dalloc(sizeof(float) * N * old);
      OB_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * N * old, s));
      LayerRun r{};
      r.cnt = cnt;
      r.D_dev = &cnt->D;
      r.S_dev = &cnt->S;
      r.D_max = N;
      r.S_max = N;
      r.items_max = items_max;
      r.dst_ptr = e.g.offsets;
      r.item_ptr = item_ptr;
      r.item_dst = item_dst;
      r.group_dst = group_dst;
      r.edge_src = e.g.nbrs;
      r.self = nullptr;
      r.x = RowSrc{nullptr, h, hld};
      r.gscale = gscale;
      r.group_ptr = group_ptr;
      LayerScratch scr{partial, partial2, agg, mean, z, s_src, s_dst};
      run_layer(s, L, r, scr, out, old);
      e.pe[l - 1] = out;
      e.pe_dim[l - 1] = L.spec.out_dim;
      h = out;
      hld = old;
      hw = L.spec.out_dim;
    }
    OB_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    cudaStreamSynchronize(s);
    for (void* p : tmp) cudaFree(p);
    throw;
  }
  for (void* p : tmp) cudaFree(p);
}

}  // namespace ob
