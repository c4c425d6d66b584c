// ob_engine.h -- engine state and stage entry points for libomega_b200.
//
// Data layout in HBM:
//   graph:  in_offsets int64[N+1], in_neighbors int32[E] (ascending per dst),
//           in_degree int32[N], features f32[N][F] (row-major)
//   PE:     f32[N][H_l] per stored layer (or owned rows + pos map under CGP)
//   model:  f32 weights; sage/power/moments keep [W_self; W_neigh] stacked
//   request workspace: one bump arena sized from per-request bounds, every
//           request-dependent count lives in a device-side counter block.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <memory>
#include <vector>

#include "ob_common.cuh"

namespace ob {

enum ErrBits : int64_t {
  kErrRange = 1,        // request edge endpoint out of range
  kErrNoQuery = 2,      // request edge without a query endpoint
  kErrZeroTotal = 4,    // candidate with zero total degree (policy.py:79-80)
  kErrNonFinite = 8,    // query feature not finite
  kErrComm = 16,        // a CGP peer never signalled (NVLink exchange timeout)
  kErrRandom = 32,      // RANDOM policy: the generated draw stream ran out (not reached in practice)
};

// Device-side counters of one request (one allocation, read back once).
struct ReqCounters {
  int64_t err;
  int64_t R;           // |candidates|
  int64_t budget;      // floor(gamma * R)
  int64_t T;           // |targets|
  int64_t RB;          // R + B request-CSR slots
  int64_t n_big;       // segments needing the CTA sort
  uint64_t sel_prefix; // radix-select state
  uint64_t sel_mask;
  int64_t sel_krem;
  int64_t sel_gt;      // keys strictly above the threshold
  int64_t sel_eq_take; // threshold-equal keys to take (lowest ids first)
  int64_t fetch_feat_rows;
  int64_t n_chunks;    // 4096-element sort chunks over the long segments
  int64_t pad[3];
};

struct BlockCounters {
  int64_t D, E, S, items;
  int64_t feat_src;    // FEATURE-bound training sources (fetch bytes)
  int64_t pe_src;      // PE-bound sources (fetch bytes)
  int64_t groups;      // second-level partial groups (hub destinations)
  int64_t gathered;    // profiler: row loads of the stored-aggregate / delta aggregation over this block
  int64_t uniq;        // profiler: distinct rows that aggregation loaded
};

// A computation block in device memory (CSR over destinations).
struct BlockDev {
  int64_t D_max = 0, E_max = 0, S_max = 0, items_max = 0;
  BlockCounters* cnt = nullptr;  // device
  int32_t* dst_ids = nullptr;    // [D] global ids (ascending)
  int64_t* dst_ptr = nullptr;    // [D+1]
  int32_t* edge_src = nullptr;   // [E] local source index, ascending within a dst
  int32_t* src_ids = nullptr;    // [S] ascending global ids
  int32_t* self_src = nullptr;   // [D] local index of dst's own row (centralized only)
  int64_t* item_ptr = nullptr;   // [D+1] aggregation work items per dst (edge chunks)
  int32_t* item_dst = nullptr;   // [items] destination of each work item
  int32_t* group_dst = nullptr;  // [groups] destination of each second-level group
  int64_t* group_ptr = nullptr;  // [D+1] groups of kItemGroup items (hub destinations only)
  bool has_self = true;
  // host mirror of counts after the request completes
  BlockCounters host{};
};

// Every row table in HBM uses a row stride padded to 4 floats (16 B) so rows
// can be staged with 16-byte cp.async and read with float4 vectors.
inline int ld4(int w) { return (w + 3) & ~3; }
// one block per layer, frontier expansion, no selection: full and sampled
inline bool khop(const ob_config& c) { return c.strategy == OB_STRATEGY_FULL || c.strategy == OB_STRATEGY_SAMPLED; }

// A row source: per-row pointers (gathered inputs) or a dense strided matrix.
struct RowSrc {
  const float* const* rowp;
  const float* base;
  int64_t ld;
  __device__ __forceinline__ const float* row(int64_t s) const { return rowp ? rowp[s] : base + s * ld; }
};

// Weights staged for the tensor-core GEMM: B^T (Np x Kp, K-major, zero padded)
// plus its 3xTF32 low part; K is the concatenation of 32-padded segments.
// Weights staged for the tcgen05 GEMM.  One TMEM accumulator pair covers at
// most 256 output columns; wider layers (Yelp/Amazon-shaped H = 512) are split
// into column slabs of <= 256, each its own staged operand and launch.
struct TcWeights {
  float* hi = nullptr;
  float* lo = nullptr;
  int N = 0, Np = 0, Kp = 0;
  int n0 = 0;  // first output column of this slab
  alignas(64) unsigned char map_hi[128] = {};  // CUtensorMap (TMA, 128B swizzle, box 32 x Np)
  alignas(64) unsigned char map_lo[128] = {};
  alignas(64) unsigned char map_hi64[128] = {};  // 64- and 32-row boxes: column slabs of small-M launches
  alignas(64) unsigned char map_lo64[128] = {};
  alignas(64) unsigned char map_hi32[128] = {};
  alignas(64) unsigned char map_lo32[128] = {};
  bool map_ready = false, map64_ready = false, map32_ready = false;
  std::shared_ptr<TcWeights> next;  // the following column slab (N > 256)
};

struct TcGemmArgs {
  const int64_t* M_dev;   // rows (device count)
  RowSrc a1;              // A1 rows (gathered), K1 wide
  const int32_t* self;    // A1 row index per output row (null = identity)
  int K1;
  const float* a2;        // dense A2 [M][lda2], K2 wide
  int64_t lda2;
  int K2;
  const float* Bt;
  const float* Bt_lo;
  const TcWeights* w;     // staged weights (TMA maps)
  int N, Np;
  float* C;
  int64_t ldc;
  const float* E;         // optional addend [M][lde] (before the activation)
  int64_t lde;
  bool relu;
  int nslab = 1;          // column slabs of Np / nslab per work unit (set by tc_gemm)
};

struct LayerDev {
  ob_layer spec{};
  float* a_src = nullptr;   // gat
  float* a_dst = nullptr;   // gat
  float* wa_dst = nullptr;  // gat: W a_dst (in_dim), s_dst = h_v . (W a_dst) for CGP owners
  bool transform_first = false;  // gcn / sage_mean with in > out: aggregate X W instead of X
  TcWeights tw_main;        // aggregate-first update ([W_self; W_neigh] or W) / gcn-gat W / tf: W_neigh
  TcWeights tw_self;        // transform-first sage_mean: W_self
};

struct GraphDev {
  int64_t N = 0, E = 0;
  int F = 0;
  int F_ld = 0;             // padded feature row stride
  int64_t* offsets = nullptr;
  int32_t* nbrs = nullptr;
  int32_t* indeg = nullptr;
  float* feats = nullptr;   // N x F_ld (or N_local x F_ld with pos)
  // CGP with partitioned storage: stored rows (features, PE) are the rank's
  // owned nodes only; pos maps a global id to its local row (-1: not stored).
  // Null: every row is stored at its global index.
  int32_t* pos = nullptr;
  int64_t N_local = 0;
  bool generated = false;   // built by the device generator (no host copy)
  std::vector<int64_t> topdeg_prefix;  // host: prefix sums of the largest in-degrees (descending)
};

void tc_gemm(cudaStream_t s, const TcGemmArgs& g, int64_t M_max);
void set_gemm_slabs(bool on);  // column-slab splitting of small-M GEMMs (single-lane engines)
struct Engine;
void prep_tc_weights(Engine& e, const std::vector<const float*>& segs, const std::vector<int>& seg_k, int N,
                     TcWeights* out);

// Bump allocator over one device allocation (reset per request).
struct Arena {
  char* base = nullptr;
  size_t cap = 0, used = 0;
  template <class T>
  T* take(int64_t count) {
    size_t bytes = ((size_t)(count > 0 ? count : 1) * sizeof(T) + 255) & ~(size_t)255;
    if (used + bytes > cap) throw Error(OB_ESTATE, "arena overflow");
    T* p = reinterpret_cast<T*>(base + used);
    used += bytes;
    return p;
  }
};

// Request sources bucketed by destination slot (slot: candidate rank, or R + query),
// ascending within a slot.  Built by an LSD radix sort of one packed key per
// edge (see RqKeyFmt); the slot offsets come from the per-slot counts.
struct RqCsr {
  int32_t* cnt = nullptr;       // [RB]
  int32_t* fill = nullptr;      // [RB]
  int64_t* ptr = nullptr;       // [RB+1]
  int32_t* src = nullptr;       // [m] ascending within a slot
  uint64_t* keys = nullptr;     // [m] packed keys (u32 or u64), radix ping
  uint64_t* keys2 = nullptr;    // [m] radix pong
  int32_t* rx_cnt = nullptr;    // [256 x tiles] digit counts per 4096-key tile (digit-major)
  int64_t* rx_off = nullptr;    // [256 x tiles + 1] their exclusive scan
  uint32_t* rx_st = nullptr;    // one-sweep: [8 passes][tiles][256] look-back words, 8 tickets,
                                // [8][256] digit totals (rx_st_words); nullptr: hist + scan passes
  int64_t* ctr = nullptr;       // device [4]: m (slice edge count), spare
};

// Packed request-edge key: (population, slot, source) so that ascending key
// order is the request CSR order.  Edges into a training candidate carry a
// query source (every edge has a query endpoint), edges into a query carry
// any source:
//   candidate slot:  [0 | rank (bR bits) | src - N (bB bits)]
//   query slot:      [1 | q (bB bits)    | src' (bN bits)]  (population bit at `body`)
// with src' = candidate rank of a training source (every training endpoint is a
// candidate and ranks follow ids) or R + q' for a query source.
struct RqKeyFmt {
  int bB, bN, bR, body, total;
  bool wide() const { return total > 32; }
  int passes() const { return (total + 7) / 8; }
};
constexpr int kRxTile = 4096;  // keys per radix tile (512 threads x 8)
inline int64_t rx_tiles(int64_t m_bound) { return m_bound / kRxTile + 1; }
inline int64_t rx_st_words(int64_t m_bound) { return 8 * 256 * rx_tiles(m_bound) + 8 + 8 * 256; }

// Request inputs as seen by the kernels: written (16 bytes of pointers + m) before
// each request so a captured CUDA graph can be replayed for any request whose
// size fits the graph's bucket.
struct ReqParams {
  const int64_t* edges;  // device [m][2]
  const float* qfeat;    // device [B][F]
  int64_t m;             // edge count of this request
  int64_t B;             // query count (GEMM row count of the early query transforms)
};

// one (src, dst) request edge: a single 16-byte load when the array allows it
__device__ __forceinline__ void ld_edge(const int64_t* __restrict__ edges, int64_t e, int64_t& s, int64_t& d) {
  if ((reinterpret_cast<uintptr_t>(edges) & 15) == 0) {
    const longlong2 v = __ldg(reinterpret_cast<const longlong2*>(edges) + e);
    s = v.x;
    d = v.y;
  } else {
    s = __ldg(edges + 2 * e);
    d = __ldg(edges + 2 * e + 1);
  }
}

// Scratch of one block assembly (two sets: the query block is assembled on the
// side stream while the mid block is assembled on the main stream).
struct BuildScratch {
  uint32_t* sbits = nullptr;       // source bitmap over [0, N+B)
  uint32_t* fill_bits = nullptr;   // [148][words_NB+1] per-CTA source bitmaps (small N only)
  int64_t* swpre = nullptr;        // [words_NB+1] popcount prefix
  int32_t* gcnt = nullptr;         // group-sparse rank: [words_NB/32 + 1] per-group counts (large N only)
  int64_t* gpre = nullptr;         //   and their prefix
  int32_t* src_global = nullptr;   // [E] global source id per edge
  int64_t* seg_len = nullptr;      // [D] CSR span + request span per destination
  int64_t* span_cs = nullptr;      // [D] CSR start/len, request start/len
  int32_t* span_cl = nullptr;
  int64_t* span_rs = nullptr;
  int32_t* span_rl = nullptr;
  int32_t* samp = nullptr;         // sampled: [D][fanout] kept source ids of the sampled rows
};

// Per-request device workspace for the centralized pipeline.
struct RequestWs {
  int B = 0;
  int64_t m = 0;                   // bucket bound on the edge count (sizes grids and buffers)
  const ReqParams* rp = nullptr;   // device
  ReqCounters* rc = nullptr;
  const int64_t* edges = nullptr;  // device [m][2]
  const float* qfeat = nullptr;    // device [B][F] as given
  float* qpad = nullptr;           // device [B][F_ld] staged copy (16 B aligned rows)
  int32_t* qdeg = nullptr;         // [B] request in-degree per query
  // candidate set (bitmap-rank over [0, N))
  uint32_t* cbits = nullptr;
  int64_t* cwpre = nullptr;        // [words+1]
  int32_t* c_gcnt = nullptr;       // group-sparse rank of the candidate bitmap (large N only)
  int64_t* c_gpre = nullptr;
  int32_t* cand_ids = nullptr;     // [R]
  int32_t* cand_nq = nullptr;      // [R]
  double* cand_score = nullptr;    // [R]
  uint64_t* cand_key = nullptr;    // [R]
  double* is_part = nullptr;       // [R] IS numerators (centralized; CGP: [P][R])
  // RANDOM policy: raw 32-bit draws, per-step draws j_i, per-value step lists
  uint32_t* rnd_raw = nullptr;     // [4 R_max + 4096]
  int32_t* rnd_j = nullptr;        // [R_max]
  int32_t* rnd_cnt = nullptr;      // [R_max + 1]
  int32_t* rnd_fill = nullptr;     // [R_max + 1]
  int64_t* rnd_off = nullptr;      // [R_max + 1]
  int32_t* rnd_lst = nullptr;      // [R_max]
  int64_t* rnd_lo = nullptr;       // chunked draw assignment: per chunk, the first evaluated entering step
  int32_t* rnd_exit = nullptr;     //   [chunks][4096] exit step per entering step
  int64_t* rnd_enter = nullptr;    //   [chunks] the true entering step
  int32_t* cand_tpos = nullptr;    // [R] position in targets or -1
  int32_t* targets = nullptr;      // [T]
  int64_t* sel_pos = nullptr;      // [R+1]
  uint32_t* sel_hist = nullptr;    // [256]
  // request CSR by destination slot (slot: candidate rank, or R + query)
  int32_t* rq_cnt = nullptr;       // [RB]
  int32_t* rq_fill = nullptr;      // [RB]
  int64_t* rq_ptr = nullptr;       // [RB+1]
  int32_t* rq_src = nullptr;       // [m] sources, ascending within a slot after sort
  uint64_t* rq_keys = nullptr;     // [m] radix keys (ping)
  uint64_t* rq_keys2 = nullptr;    // [m] radix keys (pong)
  int32_t* rx_cnt = nullptr;       // radix digit counts
  int64_t* rx_off = nullptr;       // radix digit offsets
  uint32_t* rx_st = nullptr;       // one-sweep look-back state (RqCsr::rx_st)
  int64_t* rq_ctr = nullptr;       // [4] csr counters
  RqCsr rq_view() const {
    RqCsr c;
    c.cnt = rq_cnt;
    c.fill = rq_fill;
    c.ptr = rq_ptr;
    c.src = rq_src;
    c.keys = rq_keys;
    c.keys2 = rq_keys2;
    c.rx_cnt = rx_cnt;
    c.rx_off = rx_off;
    c.rx_st = rx_st;
    c.ctr = rq_ctr;
    return c;
  }
  // block scratch
  // blocks
  std::vector<BlockDev> blocks;    // blocks[l-1] feeds layer l (mid blocks may alias)
  std::vector<int> block_of_layer; // layer -> index into blocks
  // execution scratch
  const float** rowp = nullptr;    // [S_max] input row per source
  const float** yrow = nullptr;    // [S_max] stored-transform row per source (wide layers)
  int32_t* dyn_src = nullptr;      // [S_max] sources whose transformed row is computed per request
  int64_t* ndyn = nullptr;
  float* qxw = nullptr;            // [B][ld] layer-1 x_q W of the queries (stored-transform layers)
  float* qself = nullptr;          // [B][ld] layer-1 x_q W_self (SAGE own-row table)
  bool qrows_ready = false;        // host: this enqueue staged qxw / qself early
  bool qpad_ready = false;         // host: this enqueue staged qpad early
  float* gscale = nullptr;         // [S_max] gcn source normaliser
  float* partial = nullptr;        // [items_max][w + 2]
  float* partial2 = nullptr;       // [groups_max][w + 2] second-level partials of hub destinations
  float* agg = nullptr;            // [D_max][ld4(w)]
  float* outs[8] = {};             // per-layer outputs [D_l][ld4(out)]
  float* z = nullptr;              // gat / transform-first: [S_max][ld4(out)]
  float* s_src = nullptr;          // gat: [S_max]
  float* s_dst = nullptr;          // gat: [D_max]
  float* mean = nullptr;           // moments: [D_max][in]
  float* delta = nullptr;          // [D_max][ld] delta rows h - PE of the targets (mid-block layers >= 2)
  int64_t words_N = 0, words_NB = 0;
  BuildScratch bs[2];
};

// in-library kernel profiler (CUDA events on the launching stream) -------------
// Used by bench.py to time the dominant kernel live inside the timed region.
enum ProfClass { kProfAgg = 0, kProfGemm = 1, kProfFinalize = 2, kProfBuild = 3, kProfSelect = 4,
                 kProfResolve = 5, kProfRequest = 6, kProfCsr = 7, kProfComm = 8, kProfCount = 9,
                 kProfClasses = 10 };

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  int slot;           // pinned snapshot of the block counters (-1: none)
  int width, pw;      // aggregation row width / partial width
  int K, Nc;          // gemm shape (M from the counters)
  int gemm_rows;      // 0 = D, 1 = S
};

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  std::vector<ProfRec> recs;
  BlockCounters* pinned = nullptr;  // snapshot slots
  int nslots = 0, used_slots = 0;
  std::vector<std::pair<const BlockCounters*, int>> pending;  // this request's snapshots
  uint32_t* rowbits = nullptr;  // device bitmap for the gathered-row count (profiler only)
  int64_t rowbits_words = 0;
  uint32_t* bits(int64_t words, cudaStream_t s);  // zeroed on s
  cudaEvent_t take();
  int slot_for(const BlockCounters* d);
  void request_end(cudaStream_t s);
  void reset();
  void prime(size_t events);  // allocate up front so profiled requests do no allocation
};
extern Profiler* g_prof;
cudaEvent_t prof_begin(cudaStream_t s);
void prof_end(cudaStream_t s, cudaEvent_t a, int cls, const BlockCounters* cnt, int width, int pw, int K, int Nc,
              int gemm_rows);


// layer execution building blocks (ob_layers.cu), shared with CGP (ob_cgp.cu) ---------
struct BindCtx {
  int mode;             // 0 = srpe, 1 = full (computed rows follow the source order)
  int layer;            // 1-based
  int64_t N;
  int64_t F_ld;
  const int32_t* pos;   // global -> stored row (null: identity)
  const float* feats;   // stored rows x F_ld
  const float* qfeat;   // B x F_ld
  const float* pe;      // stored layer (layer-1) rows, N x in_ld
  const float* prev;    // previous layer output, rows x in_ld
  int64_t in_ld;
  const int64_t* T_dev; // srpe: computed rows = [targets..., queries...]
  const uint32_t* cbits;
  const int64_t* cwpre;
  const int32_t* tpos;
  const int32_t* indeg;
  const int32_t* qdeg;
  // stored transforms (layers that gather X W rows): static rows of FEATURE /
  // PE-bound sources come from the table, the rest are listed for a GEMM
  const float* ytab;    // [N][y_ld] or null
  int64_t y_ld;
  const float** yrow;   // [S] row pointer of each source's transformed row
  float* ydyn;          // [dyn][y_ld] transformed rows of the listed sources
  int32_t* dyn_src;     // [dyn] source index per listed row
  int64_t* ndyn;        // device count of listed rows (zeroed before k_resolve)
  const float* qxw;     // layer 1: the queries' transformed rows, computed early (no listing)
};

struct LayerRun {
  const BlockCounters* cnt;  // D, E, S, items (device)
  const int64_t* D_dev;
  const int64_t* S_dev;
  int64_t D_max, S_max, items_max;
  const int64_t* dst_ptr;
  const int64_t* item_ptr;
  const int32_t* item_dst;   // destination per work item
  const int32_t* group_dst;  // destination per second-level group
  const int32_t* edge_src;
  const int32_t* self;       // null = identity
  RowSrc x;                  // bound inputs
  const float* gscale;       // gcn
  const int64_t* group_ptr;  // second-level partial groups (hub destinations)
  // stored transforms: Y rows by pointer, only the listed (dynamic) sources go through the GEMM
  const float** yrow = nullptr;
  const int32_t* dyn_src = nullptr;
  const int64_t* ndyn = nullptr;
  int64_t dyn_max = 0;
  // GAT: the table's source scores stab[v] = ytab[v] . a_src (rows that point into ytab
  // take their score from it instead of a dot product per request)
  const float* ytab = nullptr;
  int64_t ytab_rows = 0, ytab_ld = 0;
  const float* stab = nullptr;
  // stored aggregates (layer 1 of sum kinds): static CSR-part sums per training node
  // (delta mode, srpe mid-block layers >= 2: the stored rows' CSR-part sums; the
  // gather then visits only recomputed CSR sources, as (h - PE) delta rows)
  bool delta = false;
  const float* dprev = nullptr;  // previous layer's rows [T targets | B queries]
  const int64_t* dT = nullptr;   // device T
  const float* dbuf = nullptr;   // delta rows h - PE of the T targets (same row index)
  const float* stat = nullptr;
  int64_t stat_ld = 0;
  const int32_t* dst_ids = nullptr;
  const int32_t* indeg = nullptr;
  int64_t N = 0;
  bool split_gather = false;  // sum gathers as L2-sized source-range passes (request lanes)
  // layer-1 SAGE update from the stored own-row transform: only the B query rows need a GEMM
  const float* self_tab = nullptr;
  const float* qpad = nullptr;
  int64_t q_ld = 0;
  const int64_t* B_dev = nullptr;
  int64_t B = 0;
  const float* self_q = nullptr;   // the queries' own-row transforms, computed early
  bool no_dyn = false;             // every transformed row is a table row: skip the listed-row GEMM
  // the next layer's delta rows (dnext[i] = out[i] - dnext_pe[dst i], i < T), written by the
  // merge epilogue when this layer's output comes from it
  float* dnext = nullptr;
  const float* dnext_pe = nullptr;
  const int64_t* dnext_T = nullptr;
};

// CGP merge inputs: partition p's raw partial rows and local in-edge counts
// (contiguous in the single-process emulation, peers' exchange buffers over
// NVLink in NCCL mode); read with ld.global.cg so peer data is never stale in L1
constexpr int kMaxParts = 8;
struct PartPtrs {
  const float* lp[kMaxParts];
  const float* cnt[kMaxParts];
};
// IS policy: per-partition numerator arrays [R] summed in rank order (own / peers' buffers)
struct IsParts {
  const double* part[kMaxParts];
  int P;
};
// NCCL mode: a rank merges / updates only the destinations it owns
struct OwnerFilter {
  const int32_t* owner = nullptr;  // null: every destination
  const int32_t* dst_ids = nullptr;
  int64_t N = 0;
  int P = 1, rank = 0;
  __device__ __forceinline__ bool mine(int64_t i) const {
    if (!owner) return true;
    const int64_t g = dst_ids[i];
    return (g >= N ? (int)((g - N) % P) : owner[g]) == rank;
  }
};

struct LayerScratch {
  float* partial;
  float* partial2;
  float* agg;     // [D][ld4(w)]
  float* mean;    // moments (float64 [D][in])
  float* z;       // [S][ld4(out)]
  float* s_src;
  float* s_dst;
};

// returns true when the merge epilogue also wrote the next layer's delta rows (r.dnext)
bool run_layer(cudaStream_t s, const LayerDev& L, const LayerRun& r, const LayerScratch& sc, float* out,
               int64_t ldo);
void build_stored_transforms(Engine& e);
void launch_resolve(cudaStream_t s, const BindCtx& c, BlockCounters* cnt, int64_t S_max, const int32_t* src_ids,
                    const float** rowp, float* gscale);
// CGP: this partition's raw per-destination partial (cgpexec.py:111-164, not normalised)
void cgp_local_partial(cudaStream_t s, const LayerDev& L, const LayerRun& r, const LayerScratch& sc,
                       const float* s_dst, float* lp, int64_t ldp, float* lcnt, int moments_phase,
                       const double* mean);
// CGP: merge P raw partials in partition order (cgpexec.py:189-240) and normalise; GAT and
// transform-first GCN write the layer output, the others the aggregate for cgp_update
void cgp_merge(cudaStream_t s, const LayerDev& L, int P, const PartPtrs& parts, int64_t ldp, const OwnerFilter& own,
               const int64_t* D_dev, int64_t D_max, float* agg, float* out, int64_t ldo, int moments_phase,
               double* mean);
// CGP: apply_update with explicit destination rows h_v (models.py:214-228)
void cgp_update(cudaStream_t s, const LayerDev& L, const int64_t* D_dev, int64_t D_max, const float* const* hvp,
                const float* agg, float* out, int64_t ldo);
int cgp_partial_width(const LayerDev& L);  // raw partial row width (pw)

// stage entry points ---------------------------------------------------------
struct Engine;

constexpr int64_t kAggChunk = 128;  // edges per aggregation work item
constexpr int64_t kItemGroup = 16;  // items merged per second-level partial (hub destinations)

// aggregation work items: one per kAggChunk edges of a destination (at least one)
// Block offsets in one scan: (edges, aggregation work items, second-level
// groups) per destination.  A destination gets ceil(len / kAggChunk) items
// (at least one, so empty destinations still finalize), and destinations with
// more than kItemGroup items get ceil(items / kItemGroup) groups.
__device__ __forceinline__ I3 block_counts(int64_t len) {
  const int64_t items = len > kAggChunk ? (len + kAggChunk - 1) / kAggChunk : 1;
  const int64_t groups = items > kItemGroup ? (items + kItemGroup - 1) / kItemGroup : 0;
  return I3(len, items, groups);
}
struct SegLenLoad3 {  // from per-destination lengths
  const int64_t* seg_len;
  __device__ I3 operator()(int64_t i) const { return block_counts(seg_len[i]); }
};
struct OffsetsLoad3 {  // from an existing CSR offsets array
  const int64_t* off;
  __device__ I3 operator()(int64_t i) const { return block_counts(off[i + 1] - off[i]); }
};
struct BlockStore3 {
  int64_t* dst_ptr;  // null: offsets already exist
  int64_t* item_ptr;
  int64_t* group_ptr;
  __device__ void operator()(int64_t i, const I3& v) const {
    if (dst_ptr) dst_ptr[i] = v.a;
    item_ptr[i] = v.b;
    group_ptr[i] = v.c;
  }
};
struct BlockTotal3 {
  BlockStore3 st;
  BlockCounters* cnt;
  __device__ void operator()(int64_t n, const I3& v) const {
    st(n, v);
    cnt->E = v.a;
    cnt->items = v.b;
    cnt->groups = v.c;
  }
};

// item -> destination and group -> destination maps (warp per destination)
void configure_fill();  // shared-memory opt-in of the block fill (outside any capture)
void expand_items(cudaStream_t s, const BlockCounters* cnt, int64_t D_max, const int64_t* item_ptr,
                  const int64_t* group_ptr, int32_t* item_dst, int32_t* group_dst);
void export_bindings(Engine& e, RequestWs& w, BlockDev& b, int layer, uint8_t* d_kind, int32_t* d_pe_layer);
BindCtx bind_ctx(Engine& e, RequestWs& w, int l);
void stage_qpad(Engine& e, RequestWs& w);
void stage_query_rows(Engine& e, RequestWs& w);

void k_bitmap_compact_ext(Engine& e, const uint32_t* bits, const int64_t* wpre, int64_t words, int32_t* out);
// bitmaps above this many words take the group-sparse rank (bitmap_rank)
constexpr int64_t kSparseRankWords = 256 * 1024;  // 8.4M ids
void bitmap_rank(Engine& e, const uint32_t* bits, int64_t words, int64_t* wpre, int32_t* out, int64_t* total,
                 int32_t* gcnt, int64_t* gpre);

void stage_request_prep(Engine& e, RequestWs& w, bool need_scores);
void stage_request_post(Engine& e, RequestWs& w, bool need_scores);
void stage_select(Engine& e, RequestWs& w);
void launch_is_gather(Engine& e, RequestWs& w, const double* tab, double* out);
void build_is_table(Engine& e, const int64_t* off, const int32_t* src, double* out);
void ensure_is_tables(Engine& e);
void launch_score_is(Engine& e, RequestWs& w, const IsParts& parts);
void stage_request_csr(Engine& e, RequestWs& w);
void build_rq_csr(Engine& e, RequestWs& w, const int64_t* edges, int64_t m_bound, const int64_t* m_dev, RqCsr& c,
                  bool counts_ready);
// where a block's destinations pull their sources from
struct SpanSrc {
  const int64_t* offsets;  // CSR over all N destinations (whole graph or a rank's source-split CSR)
  const int32_t* nbrs;
  const int32_t* deg;      // CSR row lengths
  const int64_t* rq_ptr;   // request CSR (whole request or the rank's slice)
  const int32_t* rq_src;
};
// fan > 0 (sampled strategy): rows longer than fan keep the sources numpy's
// SeedSequence(seed, (layer, v)) choice picks (compgraph.py:266-274)
void assemble(Engine& e, RequestWs& w, BlockDev& b, const SpanSrc& src, const BuildScratch& sc, int fan = 0,
              int layer = 0);
void build_query_block(Engine& e, RequestWs& w);
void build_mid_block(Engine& e, RequestWs& w);
void write_mid_dst(Engine& e, RequestWs& w, BlockDev& b);
void write_query_dst(Engine& e, RequestWs& w, BlockDev& b);
void stage_build_full(Engine& e, RequestWs& w);
void stage_forward(Engine& e, RequestWs& w, float* d_out);
void stage_precompute(Engine& e);

// ---------------------------------------------------------------------------
// computation-graph parallelism (CGP): hash partitions and per-partition work
// ---------------------------------------------------------------------------
struct PartitionDev {
  int rank = 0;
  int64_t* off = nullptr;  // source-split CSR over all N destinations (graphstore.py:233-262)
  int32_t* src = nullptr;
  int32_t* deg = nullptr;
  int64_t E = 0;
};

struct CgpPartWs {
  int64_t* ledges = nullptr;  // this partition's request slice [m][2]
  RqCsr rq;                   // slice bucketed by destination slot (rq.ctr[0] = slice size)
  BlockDev blocks[2];         // mid (layers 1..k-1), last (layer k); no self rows
};

// CGP state of one request lane: the request's workspace pieces and the lane's
// own NVLink exchange (buffer, peer mappings, device step counter), so lanes on
// different streams never share exchange regions or flags
struct CgpLaneState {
  std::vector<CgpPartWs> ws;
  // per request
  const float** hvp = nullptr;  // [D_max] destination rows h_v (owned; zero row otherwise)
  float* zero_row = nullptr;
  float* lp = nullptr;          // raw partials [nparts][D_max][ldp] (float64 for moments)
  float* lcnt = nullptr;        // [nparts][D_max]
  float* sdst = nullptr;        // [D_max]
  float* lmax = nullptr;        // [D_max] softmax max exchange
  double* mean = nullptr;       // moments [D_max][in]
  float* fin = nullptr;         // [B][H] last-layer rows before the reduce to rank 0
  int64_t D_max = 0, ldp = 0;
  int64_t collective_bytes = 0;
  // NVLink exchange (NCCL mode): every rank's exchange buffer is mapped into
  // every peer (CUDA IPC); partials move with P2P loads, step flags with
  // system-scope stores -- only real rows, no padding, owner-only merges
  char* xbuf = nullptr;         // [flags 256 B][steps x region]
  size_t xregion = 0;           // bytes per step region
  int xsteps = 0;               // regions
  size_t x_need_region = 0;     // this plan's region bytes (carve_cgp)
  char* xpeer[kMaxParts] = {};  // every rank's buffer in this address space (own = xbuf)
  int64_t* xep = nullptr;       // device step counter
  int64_t* xerr = nullptr;      // device failure word of this lane's exchange (sticky after a timeout)
};

struct CgpState : CgpLaneState {
  int P = 1;
  int my_rank = 0;
  bool nccl = false;
  void* comm = nullptr;       // ncclComm_t
  int32_t* owner = nullptr;   // [N]
  std::vector<PartitionDev> parts;  // emulation: all P; NCCL: this rank's
  bool p2p = false;             // use the exchange (else padded ncclAllReduce)
  int64_t x_timeout_ns = 2000000000;  // flag-wait timeout of the exchange (OB_CGP_TIMEOUT_MS)
};

// release the current lane's exchange buffers (barrier with every peer first)
void cgp_release_exchange(Engine& e);

// (re)build the NVLink exchange when the plan needs bigger regions (all ranks
// call it at the same request: plans are identical); outside any capture
void cgp_ensure_exchange(Engine& e);

void cgp_build_partitions(Engine& e);
// NCCL-mode CGP on a host-loaded graph: keep only this rank's feature / PE rows
// (called before the first request; precompute must come first)
void cgp_localize_storage(Engine& e);
void owned_positions(Engine& e);
void localize_table(Engine& e, float*& table, int64_t ld);  // g.pos / g.N_local from cgp.owner and cgp.my_rank

// device generator (ob_gen.cu)
struct GenLaw {
  int64_t N;
  double s, inv1ms, c1, E, H;
  uint64_t seed, a, b;
};
GenLaw make_law(int64_t N, double avg, double exponent, uint64_t seed, cudaStream_t s, double* d_acc);
void generate_graph(Engine& e, int64_t N, double avg, double exponent, int F, uint64_t seed);
void generate_pe(Engine& e, int layer, int dim, uint64_t seed);
__global__ void k_owner(int64_t N, int P, uint64_t seed, int32_t* owner);
void carve_cgp(Engine& e, RequestWs& w, Arena& a);
// NVLink bytes of a request from its counters (all ranks) and the all-gather-of-rows alternative
void cgp_traffic(const Engine& e, const ReqCounters& rc, const std::vector<BlockCounters>& hc, int64_t* nvlink,
                 int64_t* allgather);
void serve_cgp(Engine& e, float* d_out);
void cgp_destroy(Engine& e);
void cgp_init_comm(Engine& e);

// One instantiated CUDA graph of the whole request pipeline.  Kernels read
// the request through the fixed ReqParams block and size their grids from
// the bucketed bound, so one graph serves every request with the same
// (B, m bucket) while the arena and output pointer stay put.
struct RequestGraph {
  int B = 0;
  int64_t m_bound = 0;
  const char* arena = nullptr;
  const float* out = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;           // kernel launches per replay (ob_launch_count)
  int64_t collective_bytes = 0;  // CGP accounting captured with the graph
  uint64_t last_use = 0;
};

// stage boundary marks: recorded as event nodes when the stream is being captured
inline void record_mark(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  OB_CUDA(cudaStreamIsCapturing(s, &st));
  if (st == cudaStreamCaptureStatusActive) OB_CUDA(cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal));
  else OB_CUDA(cudaEventRecord(ev, s));
}

// A request lane: everything a request writes (workspace arena, scan state,
// parameter block, captured graphs, streams, stage events).  The engine's own
// fields are lane 0; extra lanes are swapped in around a request, so two
// requests can be in flight on two streams at once (one's graph construction
// -- latency-bound small kernels -- overlapping the other's gathers).  The
// loaded graph, weights, stored embeddings and tables are shared read-only.
struct RequestGraph;
struct Lane {
  RequestWs ws;
  Arena arena;
  ScanScratch scan;
  ReqParams* params = nullptr;
  std::vector<RequestGraph> graphs;
  cudaStream_t stream = nullptr, side = nullptr, qside = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr, csr_ev = nullptr, done_ev = nullptr;
  cudaEvent_t qfork_ev = nullptr, qjoin_ev = nullptr;
  cudaEvent_t ev[6] = {};
  CgpLaneState cg;
};

struct Engine {
  ob_config cfg{};
  CgpState cgp;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // side stream for independent request stages (request-index sort next to the
  // top-k selection); forked and joined with events, so captured graphs branch
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr, csr_ev = nullptr;
  // third stream: the layer-1 query rows (padding, stored-transform GEMMs) need only the
  // request's features, so they run beside preparation and selection
  cudaStream_t qside = nullptr;
  cudaEvent_t qfork_ev = nullptr, qjoin_ev = nullptr;
  GraphDev g;
  std::vector<LayerDev> layers;
  std::vector<float*> pe;        // per stored layer, N x ld4(dim)
  std::vector<int> pe_dim;
  // stored transforms: per layer that gathers transformed rows (GAT z = x W,
  // transform-first X W_neigh / X W), the table x_v W over every training node
  // whose layer input is static (features at layer 1, stored embeddings above);
  // built lazily before the first request, dropped when weights / PE change
  std::vector<float*> ytab;
  // GAT layers with a table: the stored rows' source scores ytab[v] . a_src (N floats)
  std::vector<float*> stab;
  // stored aggregates: for sum kinds (gcn, sage_mean) the layer-1 aggregate of a
  // training node's CSR in-neighbours is static (only request edges, whose
  // sources are queries, change it): sagg1[v] = sum_u w_u x_u (W), raw, unnormalised
  float* sagg1 = nullptr;
  // SAGE-mean transform-first layer 1: x_v W_self per training node (the update's own-row term)
  float* yself1 = nullptr;
  // IS policy: per-node numerators of the whole CSR (centralized) or of each
  // local partition's source-split CSR (CGP), computed once per graph
  std::vector<double*> is_tab;
  // delta aggregates (srpe mid-block layers l >= 2 of sum kinds): sagg_l[l-1][v] =
  // sum_{u in N(v)} w_u PE_{l-1}(u), raw, unnormalised; null where unused
  std::vector<float*> sagg_l;
  // CGP: layer-1 stored aggregates per local partition (its source-split CSR)
  std::vector<float*> cgp_sagg1;
  bool ytab_ready = false;
  void drop_ytab() {
    for (float* t : sagg_l) dfree(t);
    sagg_l.clear();
    for (float* t : cgp_sagg1) dfree(t);
    cgp_sagg1.clear();
    for (float* t : ytab) dfree(t);
    ytab.clear();
    for (float* t : stab) dfree(t);
    stab.clear();
    dfree(sagg1);
    sagg1 = nullptr;
    dfree(yself1);
    yself1 = nullptr;
    for (double* t : is_tab) dfree(t);
    is_tab.clear();
    ytab_ready = false;
  }
  Arena arena;
  ScanScratch scan;
  RequestWs ws;
  bool have_request = false;
  cudaEvent_t ev[6] = {};
  int64_t launches_at_start = 0;
  Profiler prof;
  ReqParams* params = nullptr;   // device parameter block of the in-flight request
  bool use_graphs = true;        // replay captured request graphs (eager when profiling)
  int64_t m_reserved = 0;        // ob_reserve: edge-count bound every request is planned at (one graph)
  std::vector<RequestGraph> graphs;
  uint64_t graph_clock = 0;
  void drop_graphs() {
    for (auto& gr : graphs)
      if (gr.exec) cudaGraphExecDestroy(gr.exec);
    graphs.clear();
  }
  // A state change (graph, features, stored embeddings, weights) frees or
  // replaces buffers that captured request graphs and the stored tables point
  // at: wait for every in-flight request on every lane, then drop the graphs
  // of every lane and the derived tables (ob_api.cu)
  void invalidate_state();
  std::vector<void*> owned;      // device allocations to free
  void* dalloc(size_t bytes) {
    void* p = nullptr;
    OB_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
    owned.push_back(p);
    return p;
  }
  void dfree(void* p) {
    if (!p) return;
    for (auto& q : owned)
      if (q == p) {
        cudaFree(q);
        q = owned.back();
        owned.pop_back();
        return;
      }
  }
  bool comm_failed = false;  // a CGP exchange timed out: the engine refuses further requests
  bool localized = false;  // NCCL-mode CGP storage reduced to the owned rows
  // request lanes beyond lane 0 (ob_set_lanes); lane_rr round-robins device serves
  std::vector<Lane> lanes;
  int nlanes = 1;
  int64_t lane_rr = 0;
  int last_lane = 0;
  cudaEvent_t lane_fork_ev = nullptr;
  ~Engine();
};

}  // namespace ob
