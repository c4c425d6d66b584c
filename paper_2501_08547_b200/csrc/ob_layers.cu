// ob_layers.cu -- per-layer execution: input binding, segment aggregation,
// dense update, GAT edge softmax, and the whole-graph PE precompute.
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
#include <type_traits>

#include "ob_engine.h"

namespace ob {

// kOpDSum / kOpMom2 accumulate in float64: the moments kind takes an n-th root
// of a central moment near zero, which amplifies float32 rounding (the reference
// keeps those payloads float64 for the same reason, cgpexec.py:24-28).
enum AggOp { kOpSum = 0, kOpMax = 1, kOpPow = 2, kOpMom2 = 3, kOpSoftmax = 4, kOpDSum = 5 };

struct RowSrc {
  const float* const* rowp;  // per-source row pointers, or null for dense
  const float* base;
  int64_t ld;
  __device__ __forceinline__ const float* row(int64_t s) const { return rowp ? rowp[s] : base + s * ld; }
};

__device__ __forceinline__ float softplus_f(float x) {
  // log(1 + e^x) without overflow (densemath.py:32-34)
  return fmaxf(x, 0.f) + log1pf(__expf(-fabsf(x)));
}

// ---------------------------------------------------------------------------
// binding (resolve_block_inputs)
// ---------------------------------------------------------------------------
struct BindCtx {
  int mode;            // 0 = srpe, 1 = full (computed rows follow the source order)
  int layer;           // 1-based
  int64_t N;
  int F;
  const float* feats;
  const float* qfeat;
  const float* pe;     // stored layer (layer-1) rows, N x in
  const float* prev;   // previous layer output
  int in_dim;
  const int64_t* T_dev; // srpe: computed rows = [targets..., queries...]
  const uint32_t* cbits;
  const int64_t* cwpre;
  const int32_t* tpos;
  const int32_t* indeg;
  const int32_t* qdeg;
};

// returns BIND_* kind, row pointer and the gcn source degree
__device__ __forceinline__ int bind_row(const BindCtx& c, int64_t T, int64_t s, int64_t g, const float** row,
                                        int* pe_layer) {
  *pe_layer = 0;
  if (c.layer == 1) {
    *row = g < c.N ? c.feats + g * c.F : c.qfeat + (g - c.N) * c.F;
    return 0;  // FEATURE
  }
  if (c.mode == 1) {
    *row = c.prev + s * c.in_dim;
    return 2;  // COMPUTED
  }
  if (g >= c.N) {
    *row = c.prev + (T + (g - c.N)) * c.in_dim;
    return 2;
  }
  if (bm_test(c.cbits, g)) {
    int32_t tp = c.tpos[bm_rank(c.cbits, c.cwpre, g)];
    if (tp >= 0) {
      *row = c.prev + (int64_t)tp * c.in_dim;
      return 2;
    }
  }
  *row = c.pe + g * c.in_dim;
  *pe_layer = c.layer - 1;
  return 1;  // PE
}

__global__ void k_resolve(BindCtx c, BlockCounters* cnt, const int32_t* __restrict__ src_ids, const float** rowp,
                          float* gscale, uint8_t* kind_out, int32_t* pe_layer_out) {
  const int64_t S = cnt->S;
  const int64_t T = c.T_dev ? *c.T_dev : 0;
  int64_t nfeat = 0, npe = 0;
  OB_GRID_STRIDE(s, S) {
    int64_t g = src_ids[s];
    const float* r;
    int pl;
    int k = bind_row(c, T, s, g, &r, &pl);
    rowp[s] = r;
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
// edge-chunk aggregation
// ---------------------------------------------------------------------------
constexpr int kAggWarps = 4;
constexpr int kAggNV = 4;  // vectors per lane per column slice

__device__ __forceinline__ int64_t item_dst(const int64_t* __restrict__ item_ptr, int64_t D, int64_t it) {
  int64_t lo = 0, hi = D;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(item_ptr + mid) <= it) lo = mid;
    else hi = mid;
  }
  return lo;
}

template <int VEC>
struct Vec;
template <>
struct Vec<1> {
  using T = float;
  __device__ static void load(const float* p, float* v) { v[0] = __ldg(p); }
};
template <>
struct Vec<2> {
  __device__ static void load(const float* p, float* v) {
    float2 t = __ldg(reinterpret_cast<const float2*>(p));
    v[0] = t.x;
    v[1] = t.y;
  }
};
template <>
struct Vec<4> {
  __device__ static void load(const float* p, float* v) {
    float4 t = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = t.x;
    v[1] = t.y;
    v[2] = t.z;
    v[3] = t.w;
  }
};

struct AggArgs {
  const BlockCounters* cnt;
  const int64_t* dst_ptr;
  const int64_t* item_ptr;
  const int32_t* edge_src;
  RowSrc x;              // input rows (width `width`)
  int width;
  const float* gscale;   // sum with per-source weight (gcn) or null
  float p;               // power mean exponent
  int n;                 // moments order
  const double* mean;    // moments phase 2: [D][width] (float64)
  const float* s_src;    // softmax
  const float* s_dst;
  float* partial;        // [items][pw]
  int pw;                // partial row width (softmax: width + 2)
};

// one warp per (work item, column slice of 32*VEC*kAggNV floats)
template <int OP, int VEC>
__global__ void __launch_bounds__(32 * kAggWarps) k_agg(AggArgs a) {
  constexpr int SLICE = 32 * VEC * kAggNV;
  const int lane = threadIdx.x & 31;
  const int64_t D = a.cnt->D;
  const int64_t items = a.cnt->items;
  const int col0 = blockIdx.y * SLICE;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = gw; it < items; it += nw) {
    const int64_t i = item_dst(a.item_ptr, D, it);
    const int64_t j = it - a.item_ptr[i];
    const int64_t e0 = a.dst_ptr[i] + j * kAggChunk;
    const int64_t e1 = min(e0 + kAggChunk, a.dst_ptr[i + 1]);
    using AT = typename std::conditional<(OP == kOpDSum || OP == kOpMom2), double, float>::type;
    AT acc[kAggNV][VEC];
    float m_run = -INFINITY, den = 0.f;
#pragma unroll
    for (int q = 0; q < kAggNV; ++q)
#pragma unroll
      for (int t = 0; t < VEC; ++t) acc[q][t] = (OP == kOpMax) ? -INFINITY : 0.f;
    const float sd = (OP == kOpSoftmax) ? a.s_dst[i] : 0.f;
    for (int64_t eb = e0; eb < e1; eb += 32) {
      // lane-cooperative edge fetch, then broadcast
      int64_t my = eb + lane;
      int32_t s_l = my < e1 ? a.edge_src[my] : 0;
      const float* r_l = my < e1 ? a.x.row(s_l) : nullptr;
      float w_l = 1.f;
      if (my < e1) {
        if (OP == kOpSum && a.gscale) w_l = a.gscale[s_l];
        if (OP == kOpSoftmax) {
          float lg = a.s_src[s_l] + sd;
          w_l = lg >= 0.f ? lg : 0.2f * lg;  // leaky_relu(0.2)
        }
      }
      const int cnt = (int)min((int64_t)32, e1 - eb);
      for (int u = 0; u < cnt; ++u) {
        const float* r = (const float*)__shfl_sync(0xffffffffu, (unsigned long long)r_l, u);
        const float wgt = __shfl_sync(0xffffffffu, w_l, u);
        float scale_old = 1.f, pe = 1.f;
        if (OP == kOpSoftmax) {
          float mn = fmaxf(m_run, wgt);
          scale_old = __expf(m_run - mn);
          pe = __expf(wgt - mn);
          den = den * scale_old + pe;
          m_run = mn;
        }
#pragma unroll
        for (int q = 0; q < kAggNV; ++q) {
          const int col = col0 + (q * 32 + lane) * VEC;
          if (col < a.width) {
            float v[VEC];
            Vec<VEC>::load(r + col, v);
#pragma unroll
            for (int t = 0; t < VEC; ++t) {
              if (OP == kOpSum) acc[q][t] = fmaf(wgt, v[t], acc[q][t]);
              else if (OP == kOpDSum) acc[q][t] += (double)v[t];
              else if (OP == kOpMax) acc[q][t] = fmaxf(acc[q][t], v[t]);
              else if (OP == kOpPow) acc[q][t] += powf(softplus_f(v[t]), a.p);
              else if (OP == kOpMom2) {
                double dlt = (double)v[t] - a.mean[i * a.width + col + t];
                double pw = dlt;
                for (int r2 = 1; r2 < a.n; ++r2) pw *= dlt;
                acc[q][t] += pw;
              } else {
                acc[q][t] = fmaf(pe, v[t], acc[q][t] * scale_old);
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
      out += 2;
    }
#pragma unroll
    for (int q = 0; q < kAggNV; ++q) {
      const int col = col0 + (q * 32 + lane) * VEC;
      if (col < a.width) {
#pragma unroll
        for (int t = 0; t < VEC; ++t) out[col + t] = acc[q][t];
      }
    }
  }
}

// moments finalize in float64: phase 1 -> mean (double), phase 2 -> signed root (float)
__global__ void k_finalize_moments(const BlockCounters* cnt_, const int64_t* dst_ptr, const int64_t* item_ptr,
                                   const double* partial, int width, int phase, int n, double* mean,
                                   float* agg) {
  const int64_t D = cnt_->D;
  const int64_t total = D * width;
  OB_GRID_STRIDE(idx, total) {
    const int64_t i = idx / width;
    const int col = (int)(idx - i * width);
    const int64_t cnt = dst_ptr[i + 1] - dst_ptr[i];
    double s = 0.0;
    for (int64_t it = item_ptr[i]; it < item_ptr[i + 1]; ++it) s += partial[it * (int64_t)width + col];
    double m = cnt > 0 ? s / (double)cnt : 0.0;
    if (phase == 1) {
      mean[idx] = m;
    } else {
      double r = (n & 1) ? copysign(pow(fabs(m), 1.0 / n), m) : pow(fmax(m, 0.0), 1.0 / n);  // densemath.py:37-41
      agg[idx] = (float)r;
    }
  }
}

// merge a destination's partials in item order and normalise
struct FinArgs {
  const BlockCounters* cnt;
  const int64_t* dst_ptr;
  const int64_t* item_ptr;
  const float* partial;
  int pw;
  int width;
  int kind;   // ob_kind
  int phase;  // moments: 1 = mean, 2 = central moment
  float p;
  int n;
  float* out;  // [D][width]
  bool relu;   // gat writes the layer output directly
};

__global__ void k_finalize(FinArgs a) {
  const int64_t D = a.cnt->D;
  const int64_t total = D * a.width;
  OB_GRID_STRIDE(idx, total) {
    const int64_t i = idx / a.width;
    const int col = (int)(idx - i * a.width);
    const int64_t i0 = a.item_ptr[i], i1 = a.item_ptr[i + 1];
    const int64_t cnt = a.dst_ptr[i + 1] - a.dst_ptr[i];
    float r;
    if (a.kind == OB_KIND_GAT) {
      float ms = -INFINITY;
      for (int64_t it = i0; it < i1; ++it) {
        const float* pp = a.partial + it * (int64_t)a.pw;
        if (pp[1] > 0.f) ms = fmaxf(ms, pp[0]);
      }
      float den = 0.f, num = 0.f;
      for (int64_t it = i0; it < i1; ++it) {
        const float* pp = a.partial + it * (int64_t)a.pw;
        if (pp[1] > 0.f) {
          float sc = __expf(pp[0] - ms);
          den += pp[1] * sc;
          num += pp[2 + col] * sc;
        }
      }
      r = den > 0.f ? num / den : 0.f;
    } else if (a.kind == OB_KIND_SAGE_MAX) {
      float mx = -INFINITY;
      for (int64_t it = i0; it < i1; ++it) mx = fmaxf(mx, a.partial[it * (int64_t)a.pw + col]);
      r = cnt > 0 ? mx : 0.f;
    } else {
      float s = 0.f;
      for (int64_t it = i0; it < i1; ++it) s += a.partial[it * (int64_t)a.pw + col];
      if (a.kind == OB_KIND_GCN) {
        r = s / sqrtf((float)cnt + 1.f);  // agg / sqrt(|N(v)|+1) folded before @W (models.py:217-218)
      } else if (a.kind == OB_KIND_POWER_MEAN) {
        r = cnt > 0 ? powf(s / (float)cnt, 1.f / a.p) : 0.f;
      } else if (a.kind == OB_KIND_MOMENTS && a.phase == 2) {
        float cm = cnt > 0 ? s / (float)cnt : 0.f;
        if (a.n & 1) r = copysignf(powf(fabsf(cm), 1.f / a.n), cm);
        else r = powf(fmaxf(cm, 0.f), 1.f / a.n);
      } else {
        r = cnt > 0 ? s / (float)cnt : 0.f;  // mean
      }
    }
    if (a.relu) r = fmaxf(r, 0.f);
    a.out[i * a.width + col] = r;
  }
}

// ---------------------------------------------------------------------------
// dense update: C = act(A1 @ W[0:K1] + A2 @ W[K1:K1+K2]), fp32 FFMA
//   A1 rows: x.row(self(i)) (h_v);  A2 rows: dense agg
// ---------------------------------------------------------------------------
constexpr int GBM = 64, GBN = 64, GBK = 16;

struct GemmArgs {
  const int64_t* M_dev;  // rows (device count)
  RowSrc a1;
  const int32_t* self;   // A1 row index per output row (null = identity)
  int K1;
  const float* a2;       // dense [M][K2] or null
  int K2;
  const float* W;        // [(K1+K2)][Nc]
  int Nc;
  float* C;              // [M][Nc]
  bool relu;
};

__global__ void __launch_bounds__(256) k_gemm(GemmArgs g) {
  __shared__ float As[GBK][GBM + 4];
  __shared__ float Bs[GBK][GBN + 4];
  const int64_t M = *g.M_dev;
  const int K = g.K1 + g.K2;
  const int64_t tm = (M + GBM - 1) / GBM;
  const int tn = (g.Nc + GBN - 1) / GBN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (int64_t tile = blockIdx.x; tile < tm * tn; tile += gridDim.x) {
    const int64_t m0 = (tile / tn) * GBM;
    const int n0 = (int)(tile % tn) * GBN;
    float acc[4][4] = {};
    // each thread loads 4 A elements: rows (threadIdx.x>>2) , k = (threadIdx.x&3)*4..+3
    const int ar = threadIdx.x >> 2;
    const int ak = (threadIdx.x & 3) * 4;
    const int64_t arow = m0 + ar;
    const float* a1row = nullptr;
    const float* a2row = nullptr;
    if (arow < M) {
      if (g.K1) a1row = g.a1.row(g.self ? g.self[arow] : arow);
      if (g.K2) a2row = g.a2 + arow * g.K2;
    }
    const int br = threadIdx.x >> 4;        // 0..15
    const int bc = (threadIdx.x & 15) * 4;  // 0..60
    for (int k0 = 0; k0 < K; k0 += GBK) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        int k = k0 + ak + t;
        float v = 0.f;
        if (arow < M && k < K) v = k < g.K1 ? a1row[k] : a2row[k - g.K1];
        As[ak + t][ar] = v;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        int k = k0 + br, c = n0 + bc + t;
        Bs[br][bc + t] = (k < K && c < g.Nc) ? g.W[(int64_t)k * g.Nc + c] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < GBK; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) av[u] = As[kk][ty * 4 + u];
#pragma unroll
        for (int u = 0; u < 4; ++u) bv[u] = Bs[kk][tx * 4 + u];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int64_t r = m0 + ty * 4 + u;
      if (r >= M) continue;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        int c = n0 + tx * 4 + v;
        if (c < g.Nc) {
          float o = acc[u][v];
          g.C[r * g.Nc + c] = g.relu ? fmaxf(o, 0.f) : o;
        }
      }
    }
  }
}

// GAT attention scores: s[r] = z[row(r)] . a  (one warp per row)
__global__ void k_rowdot(const int64_t* M_dev, const float* __restrict__ z, const int32_t* self, int w,
                         const float* __restrict__ av, float* out) {
  const int64_t M = *M_dev;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < M; r += nw) {
    const float* row = z + (self ? (int64_t)self[r] : r) * w;
    float s = 0.f;
    for (int c = lane; c < w; c += 32) s = fmaf(row[c], av[c], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = s;
  }
}

// ---------------------------------------------------------------------------
// one layer over one block (shared by serving and precompute)
// ---------------------------------------------------------------------------
struct LayerRun {
  const BlockCounters* cnt;  // D, E, S, items (device)
  const int64_t* D_dev;
  const int64_t* S_dev;
  int64_t D_max, S_max, items_max;
  const int64_t* dst_ptr;
  const int64_t* item_ptr;
  const int32_t* edge_src;
  const int32_t* self;       // null = identity
  RowSrc x;                  // bound inputs
  const float* gscale;       // gcn
};

struct LayerScratch {
  float* partial;
  float* agg;
  float* mean;
  float* z;
  float* s_src;
  float* s_dst;
};

template <int OP>
static void launch_agg(cudaStream_t s, const AggArgs& a, int64_t items_max) {
  int vec = (a.width % 4 == 0) ? 4 : (a.width % 2 == 0 ? 2 : 1);
  // row pointers must be aligned for vector loads; all tables are 256B aligned
  // and rows are width*4 bytes apart, so width % VEC == 0 suffices.
  int slice = 32 * vec * kAggNV;
  dim3 grid(grid_for(items_max, kAggWarps, kNumSMs * 16), (a.width + slice - 1) / slice);
  cudaEvent_t pa = prof_begin(s);
  if (vec == 4) k_agg<OP, 4><<<grid, 32 * kAggWarps, 0, s>>>(a);
  else if (vec == 2) k_agg<OP, 2><<<grid, 32 * kAggWarps, 0, s>>>(a);
  else k_agg<OP, 1><<<grid, 32 * kAggWarps, 0, s>>>(a);
  OB_LAUNCHED();
  prof_end(s, pa, kProfAgg, a.cnt, a.width, a.pw, 0, 0, 0);
}

static void finalize(cudaStream_t s, FinArgs f, int64_t D_max) {
  cudaEvent_t pa = prof_begin(s);
  k_finalize<<<grid_for(D_max * f.width, 256), 256, 0, s>>>(f);
  OB_LAUNCHED();
  prof_end(s, pa, kProfFinalize, f.cnt, f.width, f.pw, 0, 0, 0);
}

static void gemm(cudaStream_t s, const GemmArgs& g, int64_t M_max, const BlockCounters* cnt = nullptr) {
  int64_t tiles = ((M_max + GBM - 1) / GBM) * ((g.Nc + GBN - 1) / GBN);
  cudaEvent_t pa = prof_begin(s);
  k_gemm<<<grid_for(tiles, 1, kNumSMs * 4), 256, 0, s>>>(g);
  OB_LAUNCHED();
  prof_end(s, pa, kProfGemm, cnt, 0, 0, g.K1 + g.K2, g.Nc, (cnt && g.M_dev == &cnt->S) ? 1 : 0);
}

void run_layer(cudaStream_t s, const LayerDev& L, const LayerRun& r, const LayerScratch& sc, float* out) {
  const ob_layer& sp = L.spec;
  const int in = sp.in_dim, outd = sp.out_dim;
  AggArgs a{};
  a.cnt = r.cnt;
  a.dst_ptr = r.dst_ptr;
  a.item_ptr = r.item_ptr;
  a.edge_src = r.edge_src;
  a.x = r.x;
  a.width = in;
  a.pw = in;
  a.partial = sc.partial;
  a.p = sp.p;
  a.n = sp.n;
  FinArgs f{};
  f.cnt = r.cnt;
  f.dst_ptr = r.dst_ptr;
  f.item_ptr = r.item_ptr;
  f.partial = sc.partial;
  f.pw = in;
  f.width = in;
  f.kind = sp.kind;
  f.p = sp.p;
  f.n = sp.n;
  f.out = sc.agg;
  if (sp.kind == OB_KIND_GAT) {
    // z = X @ W over every source row, then scores and the edge softmax
    GemmArgs g{r.S_dev, r.x, nullptr, in, nullptr, 0, L.w, outd, sc.z, false};
    gemm(s, g, r.S_max, r.cnt);
    k_rowdot<<<grid_for(r.S_max, 8), 256, 0, s>>>(r.S_dev, sc.z, nullptr, outd, L.a_src, sc.s_src);
    k_rowdot<<<grid_for(r.D_max, 8), 256, 0, s>>>(r.D_dev, sc.z, r.self, outd, L.a_dst, sc.s_dst);
    g_launches += 2;
    a.x = RowSrc{nullptr, sc.z, outd};
    a.width = outd;
    a.pw = outd + 2;
    a.s_src = sc.s_src;
    a.s_dst = sc.s_dst;
    launch_agg<kOpSoftmax>(s, a, r.items_max);
    f.pw = outd + 2;
    f.width = outd;
    f.out = out;
    f.relu = true;
    finalize(s, f, r.D_max);
    return;
  }
  bool finalize_skip = false;
  if (sp.kind == OB_KIND_GCN) {
    a.gscale = r.gscale;
    launch_agg<kOpSum>(s, a, r.items_max);
  } else if (sp.kind == OB_KIND_SAGE_MAX) {
    launch_agg<kOpMax>(s, a, r.items_max);
  } else if (sp.kind == OB_KIND_POWER_MEAN) {
    launch_agg<kOpPow>(s, a, r.items_max);
  } else if (sp.kind == OB_KIND_MOMENTS) {
    double* mean = reinterpret_cast<double*>(sc.mean);
    launch_agg<kOpDSum>(s, a, r.items_max);
    k_finalize_moments<<<grid_for(r.D_max * in, 256), 256, 0, s>>>(r.cnt, r.dst_ptr, r.item_ptr,
                                                                     (const double*)sc.partial, in, 1, sp.n, mean,
                                                                     nullptr);
    a.mean = mean;
    launch_agg<kOpMom2>(s, a, r.items_max);
    k_finalize_moments<<<grid_for(r.D_max * in, 256), 256, 0, s>>>(r.cnt, r.dst_ptr, r.item_ptr,
                                                                     (const double*)sc.partial, in, 2, sp.n, nullptr,
                                                                     sc.agg);
    g_launches += 2;
    finalize_skip = true;
  } else {
    launch_agg<kOpSum>(s, a, r.items_max);  // sage_mean
  }
  if (!finalize_skip) finalize(s, f, r.D_max);
  GemmArgs g{};
  g.M_dev = r.D_dev;
  g.Nc = outd;
  g.C = out;
  g.relu = true;
  if (sp.kind == OB_KIND_GCN) {
    g.K1 = 0;
    g.a2 = sc.agg;
    g.K2 = in;
    g.W = L.w;
  } else {
    g.a1 = r.x;
    g.self = r.self;
    g.K1 = in;
    g.a2 = sc.agg;
    g.K2 = in;
    g.W = L.wcat;
  }
  gemm(s, g, r.D_max, r.cnt);
}

// ---------------------------------------------------------------------------
// serving forward over the request's blocks
// ---------------------------------------------------------------------------
void stage_forward(Engine& e, RequestWs& w, float* d_out) {
  cudaStream_t s = e.stream;
  const int k = (int)e.layers.size();
  const bool full = e.cfg.strategy == OB_STRATEGY_FULL;
  for (int l = 1; l <= k; ++l) {
    const LayerDev& L = e.layers[l - 1];
    BlockDev& b = w.blocks[w.block_of_layer[l - 1]];
    BindCtx c{};
    c.mode = full ? 1 : 0;
    c.layer = l;
    c.N = e.g.N;
    c.F = e.g.F;
    c.feats = e.g.feats;
    c.qfeat = w.qfeat;
    c.pe = (!full && l > 1) ? e.pe[l - 2] : nullptr;
    c.prev = l > 1 ? w.outs[l - 1] : nullptr;
    c.in_dim = L.spec.in_dim;
    c.cbits = w.cbits;
    c.cwpre = w.cwpre;
    c.tpos = w.cand_tpos;
    c.indeg = e.g.indeg;
    c.qdeg = w.qdeg;
    c.T_dev = &w.rc->T;
    k_resolve<<<grid_for(b.S_max, 256), 256, 0, s>>>(c, b.cnt, b.src_ids, w.rowp, w.gscale, nullptr, nullptr);
    OB_LAUNCHED();
    LayerRun r{};
    r.cnt = b.cnt;
    r.D_dev = &b.cnt->D;
    r.S_dev = &b.cnt->S;
    r.D_max = b.D_max;
    r.S_max = b.S_max;
    r.items_max = b.items_max;
    r.dst_ptr = b.dst_ptr;
    r.item_ptr = b.item_ptr;
    r.edge_src = b.edge_src;
    r.self = b.self_src;
    r.x = RowSrc{w.rowp, nullptr, 0};
    r.gscale = w.gscale;
    LayerScratch sc{w.partial, w.agg, w.mean, w.z, w.s_src, w.s_dst};
    float* out = (l == k) ? d_out : w.outs[l];
    run_layer(s, L, r, sc, out);
  }
}

// parity export of bind_kind / bind_pe_layer with the same binding rule
void export_bindings(Engine& e, RequestWs& w, int layer, uint8_t* d_kind, int32_t* d_pe_layer) {
  const bool full = e.cfg.strategy == OB_STRATEGY_FULL;
  BlockDev& b = w.blocks[w.block_of_layer[layer - 1]];
  const LayerDev& L = e.layers[layer - 1];
  BindCtx c{};
  c.mode = full ? 1 : 0;
  c.layer = layer;
  c.N = e.g.N;
  c.F = e.g.F;
  c.feats = e.g.feats;
  c.qfeat = w.qfeat;
  c.pe = (!full && layer > 1) ? e.pe[layer - 2] : nullptr;
  c.prev = layer > 1 ? w.outs[layer - 1] : nullptr;
  c.in_dim = L.spec.in_dim;
  c.cbits = w.cbits;
  c.cwpre = w.cwpre;
  c.tpos = w.cand_tpos;
  c.indeg = e.g.indeg;
  c.qdeg = w.qdeg;
  c.T_dev = &w.rc->T;
  k_resolve<<<grid_for(b.S_max, 256), 256, 0, e.stream>>>(c, b.cnt, b.src_ids, w.rowp, nullptr, d_kind, d_pe_layer);
  OB_LAUNCHED();
}

// ---------------------------------------------------------------------------
// precompute_embeddings: layers 1..k-1 over the whole graph (graphstore.py:330-365)
// ---------------------------------------------------------------------------
__global__ void k_node_scale(const int32_t* __restrict__ indeg, int64_t N, float* sc) {
  OB_GRID_STRIDE(v, N) sc[v] = (float)(1.0 / sqrt((double)indeg[v] + 1.0));
}

void stage_precompute(Engine& e) {
  cudaStream_t s = e.stream;
  const int k = (int)e.layers.size();
  OB_CHECK(k >= 2, OB_EINVAL, "stored embeddings need a model with k >= 2 layers");
  OB_CHECK(e.g.N > 0, OB_ESTATE, "load a graph first");
  const int64_t N = e.g.N, E = e.g.E;
  int maxw = 0;
  for (auto& L : e.layers) maxw = std::max(maxw, std::max(L.spec.in_dim, L.spec.out_dim) + 2);
  const int64_t items_max = E / kAggChunk + N + 1;
  BlockCounters* cnt = (BlockCounters*)e.dalloc(sizeof(BlockCounters));
  BlockCounters hc{};
  hc.D = N;
  hc.E = E;
  hc.S = N;
  OB_CUDA(cudaMemcpyAsync(cnt, &hc, sizeof(hc), cudaMemcpyHostToDevice, s));
  int64_t* item_ptr = (int64_t*)e.dalloc(sizeof(int64_t) * (N + 1));
  bool mom = false;
  for (auto& L : e.layers) mom |= L.spec.kind == OB_KIND_MOMENTS;
  float* partial = (float*)e.dalloc(sizeof(float) * items_max * maxw * (mom ? 2 : 1));
  float* agg = (float*)e.dalloc(sizeof(float) * N * maxw);
  float* mean = nullptr;
  float* z = nullptr;
  float* s_src = nullptr;
  float* s_dst = nullptr;
  float* gscale = (float*)e.dalloc(sizeof(float) * N);
  k_node_scale<<<grid_for(N, 256), 256, 0, s>>>(e.g.indeg, N, gscale);
  OB_LAUNCHED();
  for (auto& L : e.layers) {
    if (L.spec.kind == OB_KIND_MOMENTS && !mean) mean = (float*)e.dalloc(sizeof(double) * N * maxw);
    if (L.spec.kind == OB_KIND_GAT && !z) {
      z = (float*)e.dalloc(sizeof(float) * N * maxw);
      s_src = (float*)e.dalloc(sizeof(float) * N);
      s_dst = (float*)e.dalloc(sizeof(float) * N);
    }
  }
  ScanScratch sc_scan;
  sc_scan.max_tiles = N / kScanTile + 2;
  sc_scan.tile_sums = (int64_t*)e.dalloc(sizeof(int64_t) * (sc_scan.max_tiles + 1));
  device_scan(s, sc_scan, ItemLoad{e.g.offsets, kAggChunk}, StoreI64{item_ptr}, nullptr, N, N, &cnt->items,
              item_ptr);
  e.pe.assign(k - 1, nullptr);
  e.pe_dim.assign(k - 1, 0);
  const float* h = e.g.feats;
  int hw = e.g.F;
  for (int l = 1; l < k; ++l) {
    const LayerDev& L = e.layers[l - 1];
    OB_CHECK(L.spec.in_dim == hw, OB_EINVAL, "model input width does not match the stored rows");
    float* out = (float*)e.dalloc(sizeof(float) * N * L.spec.out_dim);
    LayerRun r{};
    r.cnt = cnt;
    r.D_dev = &cnt->D;
    r.S_dev = &cnt->S;
    r.D_max = N;
    r.S_max = N;
    r.items_max = items_max;
    r.dst_ptr = e.g.offsets;
    r.item_ptr = item_ptr;
    r.edge_src = e.g.nbrs;
    r.self = nullptr;
    r.x = RowSrc{nullptr, h, hw};
    r.gscale = gscale;
    LayerScratch sc{partial, agg, mean, z, s_src, s_dst};
    run_layer(s, L, r, sc, out);
    e.pe[l - 1] = out;
    e.pe_dim[l - 1] = L.spec.out_dim;
    h = out;
    hw = L.spec.out_dim;
  }
  OB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace ob
