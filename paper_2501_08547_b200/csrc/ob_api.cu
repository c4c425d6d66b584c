// ob_api.cu -- engine lifecycle, per-request workspace planning, the serve
// pipeline and the C ABI (include/ob_api.h).
//
// ServingEngine.serve (runtime.py:308-335) becomes one stream-ordered
// sequence: H2D request -> validate/mark -> candidates -> scores -> radix
// select -> request CSR -> blocks -> layers -> D2H rows.  Request-dependent
// sizes never leave the device; the host only sizes the workspace from
// bounds (m, B, dataset degree profile) and reads the counters back once.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>

#include "ob_engine.h"

#ifdef OB_WITH_NCCL
#include <nccl.h>
#endif

namespace ob {

static thread_local std::string t_err;

Engine::~Engine() {
  for (auto& L : lanes) {
    for (auto& gr : L.graphs)
      if (gr.exec) cudaGraphExecDestroy(gr.exec);
    if (L.arena.base) cudaFree(L.arena.base);
    if (L.scan.pool) cudaFree(L.scan.pool);
    for (auto& ev_ : L.ev)
      if (ev_) cudaEventDestroy(ev_);
    for (cudaEvent_t ev_ : {L.fork_ev, L.join_ev, L.csr_ev, L.done_ev})
      if (ev_) cudaEventDestroy(ev_);
    if (L.stream) cudaStreamDestroy(L.stream);
    if (L.side) cudaStreamDestroy(L.side);
    if (L.qside) cudaStreamDestroy(L.qside);
    for (cudaEvent_t ev_ : {L.qfork_ev, L.qjoin_ev})
      if (ev_) cudaEventDestroy(ev_);
  }
  if (lane_fork_ev) cudaEventDestroy(lane_fork_ev);
  drop_graphs();
  for (cudaEvent_t ev_ : prof.pool) cudaEventDestroy(ev_);
  if (prof.pinned) cudaFreeHost(prof.pinned);
  if (prof.rowbits) cudaFree(prof.rowbits);
  cgp_destroy(*this);
  if (arena.base) cudaFree(arena.base);
  if (scan.pool) cudaFree(scan.pool);
  for (void* p : owned) cudaFree(p);
  for (auto& ev_ : ev)
    if (ev_) cudaEventDestroy(ev_);
  if (own_stream && stream) cudaStreamDestroy(stream);
  if (side) cudaStreamDestroy(side);
  if (qside) cudaStreamDestroy(qside);
  for (cudaEvent_t ev_ : {qfork_ev, qjoin_ev})
    if (ev_) cudaEventDestroy(ev_);
  if (fork_ev) cudaEventDestroy(fork_ev);
  if (join_ev) cudaEventDestroy(join_ev);
  if (csr_ev) cudaEventDestroy(csr_ev);
}

void Engine::invalidate_state() {
  OB_CUDA(cudaDeviceSynchronize());
  drop_graphs();
  for (auto& L : lanes) {
    for (auto& gr : L.graphs)
      if (gr.exec) cudaGraphExecDestroy(gr.exec);
    L.graphs.clear();
  }
  drop_ytab();
}

// release a layer's device buffers (weights replaced by ob_load_model)
static void free_tc(Engine& e, TcWeights& t) {
  e.dfree(t.hi);
  e.dfree(t.lo);
  t.hi = t.lo = nullptr;
  for (auto n = t.next; n; n = n->next) {
    e.dfree(n->hi);
    e.dfree(n->lo);
    n->hi = n->lo = nullptr;
  }
}
static void free_layer(Engine& e, LayerDev& L) {
  free_tc(e, L.tw_main);
  free_tc(e, L.tw_self);
  e.dfree(L.a_src);
  e.dfree(L.a_dst);
  e.dfree(L.wa_dst);
  L.a_src = L.a_dst = L.wa_dst = nullptr;
}

// swap a lane's request state with the engine's current one (lane 0 lives in the engine)
static void swap_lane(Engine& e, Lane& L) {
  std::swap(e.ws, L.ws);
  std::swap(e.arena, L.arena);
  std::swap(e.scan, L.scan);
  std::swap(e.params, L.params);
  std::swap(e.graphs, L.graphs);
  std::swap(e.stream, L.stream);
  std::swap(e.side, L.side);
  std::swap(e.qside, L.qside);
  std::swap(e.qfork_ev, L.qfork_ev);
  std::swap(e.qjoin_ev, L.qjoin_ev);
  std::swap(e.fork_ev, L.fork_ev);
  std::swap(e.join_ev, L.join_ev);
  std::swap(e.csr_ev, L.csr_ev);
  for (int i = 0; i < 6; ++i) std::swap(e.ev[i], L.ev[i]);
  std::swap(static_cast<CgpLaneState&>(e.cgp), L.cg);
}

// RAII: lane `lane` is the engine's request state for the guard's lifetime
struct LaneGuard {
  Engine& e;
  Lane* L = nullptr;
  LaneGuard(Engine& e_, int lane) : e(e_) {
    if (lane > 0) {
      L = &e.lanes[lane - 1];
      swap_lane(e, *L);
    }
  }
  ~LaneGuard() {
    if (L) swap_lane(e, *L);
  }
};

// sum of the r largest in-degrees: bound on the CSR edges r destinations can pull
static int64_t topdeg(const GraphDev& g, int64_t r) {
  if (g.topdeg_prefix.empty()) return g.E;
  if (r >= (int64_t)g.topdeg_prefix.size() - 1 && (int64_t)g.topdeg_prefix.size() - 1 < g.N) return g.E;
  r = std::max<int64_t>(0, std::min<int64_t>(r, (int64_t)g.topdeg_prefix.size() - 1));
  return g.topdeg_prefix[r];
}

struct Plan {
  int64_t words_N, words_NB, R_max, RB_max, T_max, max_scan_n;
  std::vector<BlockDev> blocks;
};

static Plan plan_request(const Engine& e, int B, int64_t m) {
  Plan p{};
  const int64_t N = e.g.N;
  const int k = (int)e.layers.size();
  p.words_N = (N + 31) / 32;
  p.words_NB = (N + B + 31) / 32;
  p.R_max = std::min<int64_t>(N, 2 * m);
  p.RB_max = p.R_max + B;
  p.T_max = std::min<int64_t>(p.R_max, (int64_t)std::floor(e.cfg.gamma * (double)p.R_max) + 1);
  auto mk = [&](int64_t D, int64_t E, bool self) {
    BlockDev b;
    b.D_max = std::max<int64_t>(D, 1);
    b.E_max = std::max<int64_t>(E, 1);
    int64_t S = std::min<int64_t>(N + B, E + (self ? D : 0));
    b.S_max = std::max<int64_t>(S, 1);
    b.items_max = b.E_max / kAggChunk + b.D_max + 1;
    b.has_self = self;
    return b;
  };
  if (khop(e.cfg)) {
    p.blocks.resize(k);
    int64_t D = B;
    const bool samp = e.cfg.strategy == OB_STRATEGY_SAMPLED;
    for (int l = k; l >= 1; --l) {
      int64_t E = topdeg(e.g, std::min<int64_t>(N, D)) + m;
      E = std::min<int64_t>(E, e.g.E + m);
      if (samp) E = std::min<int64_t>(E, D * e.cfg.fanouts[l - 1]);  // at most fan sources per destination
      p.blocks[l - 1] = mk(D, E, true);
      D = p.blocks[l - 1].S_max;
    }
  } else {
    int64_t Dm = p.T_max + B;
    int64_t Em = std::min<int64_t>(topdeg(e.g, std::min<int64_t>(N, p.T_max)) + m, e.g.E + m);
    p.blocks.push_back(mk(Dm, Em, true));
    p.blocks.push_back(mk(B, m, true));
  }
  p.max_scan_n = std::max<int64_t>(std::max<int64_t>(p.words_NB, p.RB_max), 256 * rx_tiles(m));
  for (auto& b : p.blocks) p.max_scan_n = std::max<int64_t>(p.max_scan_n, b.D_max + 1);
  return p;
}

// carve the workspace out of an arena (dry-run with base == nullptr to size it)
static void carve(Engine& e, RequestWs& w, Plan& p, Arena& a) {
  const int k = (int)e.layers.size();
  const int64_t m = w.m;
  const int B = w.B;
  int maxw = e.g.F;
  for (auto& L : e.layers) maxw = std::max(maxw, std::max(L.spec.in_dim, L.spec.out_dim));
  w.words_N = p.words_N;
  w.words_NB = p.words_NB;
  w.rc = a.take<ReqCounters>(1);
  w.qdeg = a.take<int32_t>(B + 1);
  w.cbits = a.take<uint32_t>(p.words_N + 1);
  w.cwpre = a.take<int64_t>(p.words_N + 1);
  w.c_gcnt = p.words_N > kSparseRankWords ? a.take<int32_t>(p.words_N / 32 + 2) : nullptr;
  w.c_gpre = p.words_N > kSparseRankWords ? a.take<int64_t>(p.words_N / 32 + 2) : nullptr;
  w.cand_ids = a.take<int32_t>(p.R_max);
  w.cand_nq = a.take<int32_t>(p.R_max);
  w.cand_score = a.take<double>(p.R_max);
  w.cand_key = a.take<uint64_t>(p.R_max);
  // IS numerators: one array centralized, one per partition under CGP emulation,
  // [P][R] for the NCCL all-gather fallback
  w.is_part = e.cfg.policy == OB_POLICY_IS ? a.take<double>(p.R_max * std::max(1, e.cfg.num_partitions)) : nullptr;
  if (e.cfg.policy == OB_POLICY_RANDOM) {
    w.rnd_raw = a.take<uint32_t>(4 * p.R_max + 4096);
    w.rnd_j = a.take<int32_t>(p.R_max + 1);
    w.rnd_cnt = a.take<int32_t>(p.R_max + 2);
    w.rnd_fill = a.take<int32_t>(p.R_max + 2);
    w.rnd_off = a.take<int64_t>(p.R_max + 2);
    w.rnd_lst = a.take<int32_t>(p.R_max + 1);
    const int64_t chunks = (4 * p.R_max + 4096 + 2047) / 2048;
    w.rnd_lo = a.take<int64_t>(chunks + 1);
    w.rnd_exit = a.take<int32_t>((chunks + 1) * 4096);
    w.rnd_enter = a.take<int64_t>(chunks + 1);
  }
  w.cand_tpos = a.take<int32_t>(p.R_max);
  w.targets = a.take<int32_t>(p.T_max + 1);
  w.sel_hist = a.take<uint32_t>(257);  // [256] = round completion counter
  w.rq_cnt = a.take<int32_t>(p.RB_max + 1);
  w.rq_fill = a.take<int32_t>(p.RB_max + 1);
  w.rq_ptr = a.take<int64_t>(p.RB_max + 1);
  w.rq_src = a.take<int32_t>(m + 1);
  w.rq_keys = a.take<uint64_t>(m + 1);
  w.rq_keys2 = a.take<uint64_t>(m + 1);
  w.rx_cnt = a.take<int32_t>(256 * rx_tiles(m));
  w.rx_off = a.take<int64_t>(256 * rx_tiles(m) + 257);  // + per-digit totals
  w.rx_st = a.take<uint32_t>(rx_st_words(m));
  w.rq_ctr = a.take<int64_t>(4);
  int64_t Emax = 1, Dmax = 1, Smax = 1, Imax = 1;
  for (auto& b : p.blocks) {
    Emax = std::max(Emax, b.E_max);
    Dmax = std::max(Dmax, b.D_max);
    Smax = std::max(Smax, b.S_max);
    Imax = std::max(Imax, b.items_max);
  }
  auto take_scratch = [&](BuildScratch& sc, int64_t D, int64_t E) {
    sc.sbits = a.take<uint32_t>(p.words_NB + 1);
    sc.fill_bits = p.words_NB <= 48 * 1024 ? a.take<uint32_t>(kNumSMs * (p.words_NB + 1)) : nullptr;
    sc.swpre = a.take<int64_t>(p.words_NB + 1);
    sc.gcnt = p.words_NB > kSparseRankWords ? a.take<int32_t>(p.words_NB / 32 + 2) : nullptr;
    sc.gpre = p.words_NB > kSparseRankWords ? a.take<int64_t>(p.words_NB / 32 + 2) : nullptr;
    sc.src_global = a.take<int32_t>(E);
    sc.seg_len = a.take<int64_t>(D);
    sc.span_cs = a.take<int64_t>(D);
    sc.span_cl = a.take<int32_t>(D);
    sc.span_rs = a.take<int64_t>(D);
    sc.span_rl = a.take<int32_t>(D);
  };
  take_scratch(w.bs[0], Dmax, Emax);
  if (e.cfg.strategy == OB_STRATEGY_SAMPLED) {  // kept sources of the sampled rows, one block at a time
    int64_t n = 1;
    for (int l = 1; l <= k; ++l) n = std::max<int64_t>(n, p.blocks[l - 1].D_max * e.cfg.fanouts[l - 1]);
    w.bs[0].samp = a.take<int32_t>(n);
  }
  if (!khop(e.cfg)) take_scratch(w.bs[1], p.blocks[1].D_max, p.blocks[1].E_max);  // query block
  else w.bs[1] = w.bs[0];
  w.blocks = p.blocks;
  for (size_t i = 0; i < w.blocks.size(); ++i) {
    BlockDev& b = w.blocks[i];
    b.cnt = a.take<BlockCounters>(1);
    b.dst_ptr = a.take<int64_t>(b.D_max + 1);
    b.item_ptr = a.take<int64_t>(b.D_max + 1);
    b.item_dst = a.take<int32_t>(b.items_max);
    b.group_dst = a.take<int32_t>(b.items_max / kItemGroup + b.D_max + 1);
    b.group_ptr = a.take<int64_t>(b.D_max + 1);
    b.edge_src = a.take<int32_t>(b.E_max);
    b.src_ids = a.take<int32_t>(b.S_max);
    b.self_src = a.take<int32_t>(b.D_max);
    // full: block l-1's dst list aliases block l's src_ids (set below)
    b.dst_ids = a.take<int32_t>(b.D_max);
  }
  if (khop(e.cfg))  // block l-1's destinations are block l's sources
    for (int l = k - 1; l >= 1; --l) w.blocks[l - 1].dst_ids = w.blocks[l].src_ids;
  w.block_of_layer.assign(k, 0);
  for (int l = 1; l <= k; ++l)
    w.block_of_layer[l - 1] = khop(e.cfg) ? l - 1 : (l < k ? 0 : 1);
  w.rowp = a.take<const float*>(Smax);
  w.gscale = a.take<float>(Smax);
  bool gat = false, mom = false, wide = false;
  for (auto& L : e.layers) {
    gat |= L.spec.kind == OB_KIND_GAT;
    mom |= L.spec.kind == OB_KIND_MOMENTS;
    wide |= L.spec.kind == OB_KIND_GAT || L.transform_first;
  }
  const int64_t wl = ld4(maxw) + 4;
  w.qpad = a.take<float>((int64_t)B * e.g.F_ld + 4);
  w.partial = a.take<float>(Imax * wl * (mom ? 2 : 1));  // moments partials are float64
  w.partial2 = a.take<float>((Imax / kItemGroup + Dmax + 1) * wl);
  w.agg = a.take<float>(Dmax * wl);
  w.mean = mom ? a.take<float>(2 * Dmax * wl) : nullptr;
  w.z = wide ? a.take<float>(Smax * wl) : nullptr;
  w.yrow = wide ? a.take<const float*>(Smax) : nullptr;
  w.qxw = wide ? a.take<float>((int64_t)(B + 1) * wl) : nullptr;
  w.qself = wide ? a.take<float>((int64_t)(B + 1) * wl) : nullptr;
  w.dyn_src = wide ? a.take<int32_t>(Smax) : nullptr;
  w.ndyn = wide ? a.take<int64_t>(1) : nullptr;
  w.delta = (!khop(e.cfg) && k >= 3) ? a.take<float>(p.blocks[0].D_max * wl) : nullptr;
  w.s_src = gat ? a.take<float>(Smax) : nullptr;
  w.s_dst = gat ? a.take<float>(Dmax) : nullptr;
  for (int l = 1; l < k; ++l) {
    const BlockDev& b = w.blocks[w.block_of_layer[l - 1]];
    w.outs[l] = a.take<float>(b.D_max * ld4(e.layers[l - 1].spec.out_dim));
  }
}

struct PinnedReadback {
  ReqCounters rc;
  BlockCounters bc[8];
};

static void prepare_workspace(Engine& e, int B, int64_t m) {
  Plan p = plan_request(e, B, m);
  RequestWs& w = e.ws;
  w.B = B;
  w.m = m;
  Arena dry;
  dry.base = nullptr;
  dry.cap = (size_t)-1 / 2;
  carve(e, w, p, dry);
  if (e.cfg.strategy == OB_STRATEGY_SRPE_CGP) carve_cgp(e, w, dry);
  size_t need = dry.used + (1u << 20);
  if (need > e.arena.cap) {
    OB_CUDA(cudaStreamSynchronize(e.stream));
    e.drop_graphs();  // captured graphs point into the old arena
    const size_t cap = std::max(need, e.arena.cap * 3 / 2);
    if (e.arena.base) OB_CUDA(cudaFree(e.arena.base));
    e.arena.base = nullptr;
    e.arena.cap = 0;
    void* q = nullptr;
    OB_CUDA(cudaMalloc(&q, cap));
    e.arena.base = (char*)q;
    e.arena.cap = cap;
  }
  // scan state pool: its own allocation at a fixed address, zeroed once here
  // and by every request after use (graphs bake in its slices)
  const int nscans = 24 + 8 * std::max(1, e.cfg.num_partitions);
  const size_t pool = ScanScratch::bytes_for(p.max_scan_n, nscans);
  if (pool > e.scan.cap) {
    OB_CUDA(cudaStreamSynchronize(e.stream));
    e.drop_graphs();
    if (e.scan.pool) OB_CUDA(cudaFree(e.scan.pool));
    e.scan.pool = nullptr;
    e.scan.cap = 0;
    void* q = nullptr;
    OB_CUDA(cudaMalloc(&q, pool));
    OB_CUDA(cudaMemset(q, 0, pool));
    e.scan.pool = (char*)q;
    e.scan.cap = pool;
  }
  e.arena.used = 0;
  carve(e, w, p, e.arena);
  if (e.cfg.strategy == OB_STRATEGY_SRPE_CGP) {
    carve_cgp(e, w, e.arena);
    cgp_ensure_exchange(e);  // NCCL mode: NVLink exchange buffers for this plan
  }
}

static void check_ready(Engine& e) {
  OB_CHECK(e.g.N > 0, OB_ESTATE, "no graph loaded");
  OB_CHECK(!e.layers.empty(), OB_ESTATE, "no model loaded");
  OB_CHECK(e.layers[0].spec.in_dim == e.g.F, OB_EINVAL, "input width does not match layer in_dim");
  if (e.cfg.strategy == OB_STRATEGY_SAMPLED)
    OB_CHECK(e.cfg.num_fanouts == (int)e.layers.size(), OB_EINVAL, "sampled strategy needs one fanout per layer");
  if (!khop(e.cfg)) {
    OB_CHECK((int)e.layers.size() >= 2, OB_EINVAL, "reuse graphs need k >= 2");
    OB_CHECK((int)e.pe.size() >= (int)e.layers.size() - 1 && !e.pe.empty(), OB_EINVAL,
             "reuse strategy needs stored embeddings");
    for (int l = 1; l < (int)e.layers.size(); ++l)
      OB_CHECK(e.pe_dim[l - 1] == e.layers[l].spec.in_dim, OB_EINVAL, "stored embedding width mismatch");
  }
}

static void raise_request_errors(const ReqCounters& rc) {
  if (rc.err & kErrRange) throw Error(OB_EINVAL, "request edge endpoint out of range");
  if (rc.err & kErrNoQuery) throw Error(OB_EINVAL, "every request edge needs a query endpoint");
  if (rc.err & kErrNonFinite) throw Error(OB_EINVAL, "query features must be finite");
  if (rc.err & kErrZeroTotal) throw Error(OB_EINVAL, "candidate with zero total degree");
  if (rc.err & kErrRandom) throw Error(OB_ECUDA, "random policy: draw stream exhausted");
  if (rc.err & kErrComm) throw Error(OB_ECOMM, "CGP exchange: a peer rank did not signal in time (OB_CGP_TIMEOUT_MS)");
}

// fetch-byte accounting per layer (graph_fetch_bytes, runtime.py:105-120)
static int64_t fetch_bytes(const Engine& e, const RequestWs& w, const std::vector<BlockCounters>& per_layer) {
  int64_t total = 0;
  const int k = (int)e.layers.size();
  for (int l = 1; l <= k; ++l) {
    const BlockCounters& c = per_layer[l - 1];
    total += 16 * c.E;
    total += 4 * (int64_t)e.g.F * c.feat_src;
    if (l > 1 && !e.pe_dim.empty() && !khop(e.cfg)) total += 4 * (int64_t)e.pe_dim[l - 2] * c.pe_src;
  }
  (void)w;
  return total;
}

// request-size bucket: grids and the workspace are sized from this bound so
// one captured graph serves every request up to it (<= 25 % slack)
static int64_t bucket_m(int64_t m) {
  int64_t b = 1024;
  while (b < m) b = (b + b / 4 + 1023) / 1024 * 1024;
  return b;
}

__global__ void k_set_params(ReqParams* p, const int64_t* edges, const float* q, int64_t m, int64_t B) {
  pdl_wait();
  p->edges = edges;
  p->qfeat = q;
  p->m = m;
  p->B = B;
}

// every stage of one request, enqueued on e.stream (eagerly or under capture)
static void enqueue_stages(Engine& e, float* d_out);

static void enqueue_request(Engine& e, float* d_out) {
  e.scan.cursor = 0;
  try {
    enqueue_stages(e, d_out);
  } catch (...) {
    // the pool must be all zero for the next request whatever was enqueued
    cudaStreamSynchronize(e.stream);
    cudaMemset(e.scan.pool, 0, e.scan.cap);
    e.scan.cursor = 0;
    throw;
  }
  e.scan.clear(e.stream);  // zero the scan state this request used
}

static void enqueue_stages(Engine& e, float* d_out) {
  cudaStream_t s = e.stream;
  RequestWs& w = e.ws;
  const bool srpe = !khop(e.cfg);
  w.qrows_ready = w.qpad_ready = false;
  OB_CUDA(cudaMemsetAsync(w.rc, 0, sizeof(ReqCounters), s));
  for (auto& b : w.blocks) OB_CUDA(cudaMemsetAsync(b.cnt, 0, sizeof(BlockCounters), s));
  if (e.cfg.strategy == OB_STRATEGY_SRPE_CGP) {
    serve_cgp(e, d_out);  // marks ev[1] between build and layers
    return;
  }
  // the layer-1 query rows need only the request's features: third stream from the start
  // (OB_QROWS_SERIAL=1: on the main stream after the selection, as before)
  static const bool qserial = [] {
    const char* v = std::getenv("OB_QROWS_SERIAL");
    return v && v[0] && v[0] != '0';
  }();
  const bool qs = !qserial;
  if (qs) {
    OB_CUDA(cudaEventRecord(e.qfork_ev, s));
    OB_CUDA(cudaStreamWaitEvent(e.qside, e.qfork_ev, 0));
    e.stream = e.qside;
    try {
      stage_query_rows(e, w);
    } catch (...) {
      e.stream = s;
      throw;
    }
    e.stream = s;
    OB_CUDA(cudaEventRecord(e.qjoin_ev, e.qside));
  }
  cudaEvent_t p0 = prof_begin(s);
  stage_request_prep(e, w, srpe);
  // the request-index sort (side stream) and the top-k selection (main stream)
  // only share read-only inputs from here on: run them side by side
  // and, under srpe, the query block (it needs only the index) follows the sort there
  OB_CUDA(cudaEventRecord(e.fork_ev, s));
  OB_CUDA(cudaStreamWaitEvent(e.side, e.fork_ev, 0));
  {
    e.stream = e.side;  // stage functions launch on e.stream
    try {
      cudaEvent_t pc = prof_begin(e.side);
      stage_request_csr(e, w);
      prof_end(e.side, pc, kProfCsr, nullptr, 0, 0, 0, 0, 0);
      OB_CUDA(cudaEventRecord(e.csr_ev, e.side));
      if (srpe) {
        pc = prof_begin(e.side);
        build_query_block(e, w);
        prof_end(e.side, pc, kProfBuild, nullptr, 0, 0, 0, 0, 0);
      }
    } catch (...) {
      e.stream = s;
      throw;
    }
    e.stream = s;
  }
  stage_request_post(e, w, srpe);
  if (srpe) stage_select(e, w);
  prof_end(s, p0, kProfSelect, nullptr, 0, 0, 0, 0, 0);
  // query rows of layer 1 (padding, stored-transform rows) while the request index sorts
  if (!qs) stage_query_rows(e, w);
  OB_CUDA(cudaStreamWaitEvent(s, e.csr_ev, 0));
  p0 = prof_begin(s);
  if (srpe) build_mid_block(e, w);
  else stage_build_full(e, w);
  prof_end(s, p0, kProfBuild, nullptr, 0, 0, 0, 0, 0);
  OB_CUDA(cudaEventRecord(e.join_ev, e.side));
  OB_CUDA(cudaStreamWaitEvent(s, e.join_ev, 0));
  if (qs) OB_CUDA(cudaStreamWaitEvent(s, e.qjoin_ev, 0));
  record_mark(e.ev[1], s);
  stage_forward(e, w, d_out);
}

static RequestGraph& request_graph(Engine& e, float* d_out) {
  const RequestWs& w = e.ws;
  for (auto& gr : e.graphs)
    if (gr.B == w.B && gr.m_bound == w.m && gr.arena == e.arena.base && gr.out == d_out) return gr;
  cudaStream_t s = e.stream;
  const int64_t l0 = g_launches;
  OB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  cudaGraph_t graph = nullptr;
  try {
    enqueue_request(e, d_out);
  } catch (...) {
    cudaStreamEndCapture(s, &graph);
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    g_launches = l0;
    throw;
  }
  OB_CUDA(cudaStreamEndCapture(s, &graph));
  cudaGraphExec_t exec = nullptr;
  cudaError_t err = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  OB_CUDA(err);
  if (e.graphs.size() >= 16) {  // evict the least recently used
    auto lru = std::min_element(e.graphs.begin(), e.graphs.end(),
                                [](const RequestGraph& a, const RequestGraph& b) { return a.last_use < b.last_use; });
    cudaGraphExecDestroy(lru->exec);
    e.graphs.erase(lru);
  }
  RequestGraph gr;
  gr.B = w.B;
  gr.m_bound = w.m;
  gr.arena = e.arena.base;
  gr.out = d_out;
  gr.exec = exec;
  gr.kernels = g_launches - l0;
  gr.collective_bytes = e.cgp.collective_bytes;
  g_launches = l0;  // counted per replay
  e.graphs.push_back(gr);
  return e.graphs.back();
}

// IS numerator tables (once per graph; outside any capture)
void ensure_is_tables(Engine& e) {
  if (e.cfg.policy != OB_POLICY_IS || !e.is_tab.empty()) return;
  const int64_t N = e.g.N;
  if (e.cfg.strategy == OB_STRATEGY_SRPE_CGP) {
    for (auto& part : e.cgp.parts) {
      double* t = (double*)e.dalloc(sizeof(double) * N);
      build_is_table(e, part.off, part.src, t);
      e.is_tab.push_back(t);
    }
  } else {
    OB_CHECK(e.g.offsets, OB_ESTATE, "the IS policy needs the graph's CSR");
    double* t = (double*)e.dalloc(sizeof(double) * N);
    build_is_table(e, e.g.offsets, e.g.nbrs, t);
    e.is_tab.push_back(t);
  }
}

// blocks whose counters a breakdown reads: centralized blocks, or every partition's (mid, last)
static std::vector<BlockDev*> counted_blocks(Engine& e) {
  std::vector<BlockDev*> all;
  if (e.cfg.strategy == OB_STRATEGY_SRPE_CGP) {
    for (auto& pw : e.cgp.ws) all.insert(all.end(), {&pw.blocks[0], &pw.blocks[1]});
  } else {
    for (auto& b : e.ws.blocks) all.push_back(&b);
  }
  return all;
}

// The request pipeline, enqueued on the engine stream.  Inputs/outputs are device pointers.
static void enqueue_serve(Engine& e, int B, const float* d_q, int64_t m, const int64_t* d_edges, float* d_out) {
  check_ready(e);
  OB_CHECK(!e.comm_failed, OB_ECOMM,
           "a CGP exchange timed out on an earlier request: the exchange state is unusable, recreate the engines");
  OB_CHECK(B >= 0 && m >= 0, OB_EINVAL, "negative request size");
  OB_CHECK(e.g.N + B < ((int64_t)1 << 31) - 1, OB_EINVAL, "id space exceeds int32");
  cgp_localize_storage(e);  // NCCL CGP: keep only the owned rows (no-op otherwise)
  build_stored_transforms(e);  // once per (model, PE) state, outside any capture
  ensure_is_tables(e);
  set_gemm_slabs(e.nlanes == 1);  // baked into the captured graph (graphs are re-captured on ob_set_lanes)
  cudaStream_t s = e.stream;
  prepare_workspace(e, B, std::max(bucket_m(m), e.m_reserved));
  RequestWs& w = e.ws;
  if (!e.params) e.params = (ReqParams*)e.dalloc(sizeof(ReqParams));
  w.rp = e.params;
  w.edges = d_edges;
  w.qfeat = d_q;
  // kernel arguments are copied at launch: the block is stream-ordered with no host staging
  launch_pdl(k_set_params, dim3(1), dim3(1), 0, s, e.params, d_edges, d_q, m, B);
  OB_CUDA(cudaEventRecord(e.ev[0], s));
  if (e.prof.on || !e.use_graphs) {
    g_prof = e.prof.on ? &e.prof : nullptr;
    cudaEvent_t preq = prof_begin(s);
    try {
      enqueue_request(e, d_out);
    } catch (...) {
      g_prof = nullptr;
      throw;
    }
    prof_end(s, preq, kProfRequest, nullptr, 0, 0, 0, 0, 0);
    if (g_prof) g_prof->request_end(s);
    g_prof = nullptr;
  } else {
    RequestGraph& gr = request_graph(e, d_out);
    gr.last_use = ++e.graph_clock;
    OB_CUDA(cudaGraphLaunch(gr.exec, s));
    g_launches += gr.kernels;
    e.cgp.collective_bytes = gr.collective_bytes;
  }
  OB_CUDA(cudaEventRecord(e.ev[2], s));
  e.have_request = true;
}

// errors and the breakdown from the request's counters (read back to the host)
static void finish_breakdown(Engine& e, const ReqCounters& rc, const std::vector<BlockCounters>& hc, float t01,
                             float t12, ob_breakdown* bd) {
  RequestWs& w = e.ws;
  const int k = (int)e.layers.size();
  const bool srpe = !khop(e.cfg);
  const bool cgp = e.cfg.strategy == OB_STRATEGY_SRPE_CGP;
  std::vector<BlockDev*> all = counted_blocks(e);
  for (size_t i = 0; i < all.size() && i < hc.size(); ++i) all[i]->host = hc[i];
  if (rc.err & kErrComm) e.comm_failed = true;  // sticky: the exchange state is skewed
  raise_request_errors(rc);
  if (!bd) return;
  // graph_fetch_bytes per block set (runtime.py:105-120; CGP: _shard_fetch_bytes summed, :224-247)
  auto set_bytes = [&](const BlockCounters* blocks_of_layer[], const BlockCounters& mid) {
    std::vector<BlockCounters> per_layer(k);
    for (int l = 1; l <= k; ++l) per_layer[l - 1] = *blocks_of_layer[l - 1];
    if (srpe) {
      // the shared mid block accumulated layer 1's FEATURE rows and layers 2..k-1's PE rows
      for (int l = 1; l < k; ++l) {
        per_layer[l - 1].feat_src = (l == 1) ? mid.feat_src : 0;
        per_layer[l - 1].pe_src = (l == 1) ? 0 : mid.pe_src / std::max(1, k - 2);
      }
    }
    return fetch_bytes(e, w, per_layer);
  };
  int64_t fb = 0;
  std::vector<const BlockCounters*> bl(k);
  if (cgp) {
    for (auto& pw : e.cgp.ws) {
      for (int l = 1; l <= k; ++l) bl[l - 1] = &pw.blocks[l < k ? 0 : 1].host;
      fb += set_bytes(bl.data(), pw.blocks[0].host);
    }
  } else {
    for (int l = 1; l <= k; ++l) bl[l - 1] = &w.blocks[w.block_of_layer[l - 1]].host;
    fb = set_bytes(bl.data(), w.blocks[0].host);
  }
  std::memset(bd, 0, sizeof(*bd));
  bd->fetch_ms = t01;
  bd->compute_ms = t12;
  bd->fetch_bytes = fb;
  bd->collective_bytes = e.cgp.collective_bytes;
  if (cgp && e.cgp.nccl && e.cgp.p2p) {  // NVLink exchange: actual rows moved (all ranks)
    cgp_traffic(e, rc, hc, &bd->collective_bytes, &bd->allgather_bytes);
  } else if (cgp) {
    int64_t nv = 0;
    cgp_traffic(e, rc, hc, &nv, &bd->allgather_bytes);
  }
  bd->transfer_ms = (double)bd->fetch_bytes / 12e9 * 1e3;
  bd->num_candidates = rc.R;
  bd->num_targets = rc.T;
  bd->total_device_ms = t01 + t12;
}

static void serve_device(Engine& e, int B, const float* d_q, int64_t m, const int64_t* d_edges, float* d_out,
                         ob_breakdown* bd) {
  enqueue_serve(e, B, d_q, m, d_edges, d_out);
  if (!bd) return;
  cudaStream_t s = e.stream;
  PinnedReadback hb{};
  OB_CUDA(cudaMemcpyAsync(&hb.rc, e.ws.rc, sizeof(ReqCounters), cudaMemcpyDeviceToHost, s));
  std::vector<BlockDev*> all = counted_blocks(e);
  std::vector<BlockCounters> hc(all.size());
  for (size_t i = 0; i < all.size(); ++i)
    OB_CUDA(cudaMemcpyAsync(&hc[i], all[i]->cnt, sizeof(BlockCounters), cudaMemcpyDeviceToHost, s));
  OB_CUDA(cudaStreamSynchronize(s));
  OB_CUDA(cudaGetLastError());
  float t01 = 0, t12 = 0;
  OB_CUDA(cudaEventElapsedTime(&t01, e.ev[0], e.ev[1]));
  OB_CUDA(cudaEventElapsedTime(&t12, e.ev[1], e.ev[2]));
  finish_breakdown(e, hb.rc, hc, t01, t12, bd);
}

// ---------------------------------------------------------------------------
// loads
// ---------------------------------------------------------------------------
static void load_graph(Engine& e, int64_t N, const int64_t* off, const int64_t* nb, int64_t E, const float* feats,
                       int F) {
  OB_CHECK(N > 0 && N < ((int64_t)1 << 31) - 4096, OB_EINVAL, "num_nodes out of range");
  OB_CHECK(off && (E == 0 || nb) && (F == 0 || feats), OB_EINVAL, "null graph array");
  OB_CHECK(off[0] == 0 && off[N] == E, OB_EINVAL, "offsets inconsistent with num_edges");
  std::vector<int32_t> nbrs32((size_t)E);
  std::vector<int32_t> deg((size_t)N);
  for (int64_t v = 0; v < N; ++v) {
    int64_t a = off[v], b = off[v + 1];
    OB_CHECK(b >= a, OB_EINVAL, "offsets must be non-decreasing");
    deg[v] = (int32_t)(b - a);
    bool sorted = true;
    for (int64_t i = a; i < b; ++i) {
      int64_t u = nb[i];
      OB_CHECK(u >= 0 && u < N, OB_EINVAL, "edge endpoint out of range");
      nbrs32[i] = (int32_t)u;
      if (i > a && nbrs32[i] < nbrs32[i - 1]) sorted = false;
    }
    // edges are consumed in (dst, src) order (compgraph.py:197-201): sort rows once at load
    if (!sorted) std::sort(nbrs32.begin() + a, nbrs32.begin() + b);
  }
  GraphDev& g = e.g;
  g.N = N;
  g.E = E;
  g.F = F;
  g.offsets = (int64_t*)e.dalloc(sizeof(int64_t) * (N + 1));
  g.nbrs = (int32_t*)e.dalloc(sizeof(int32_t) * std::max<int64_t>(E, 1));
  g.indeg = (int32_t*)e.dalloc(sizeof(int32_t) * N);
  g.F_ld = ld4(std::max(F, 1));
  g.feats = (float*)e.dalloc(sizeof(float) * std::max<int64_t>(N * g.F_ld, 1));
  OB_CUDA(cudaMemcpy(g.offsets, off, sizeof(int64_t) * (N + 1), cudaMemcpyHostToDevice));
  if (E) OB_CUDA(cudaMemcpy(g.nbrs, nbrs32.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice));
  OB_CUDA(cudaMemcpy(g.indeg, deg.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice));
  // rows padded to 16 B for cp.async / float4 staging
  OB_CUDA(cudaMemset(g.feats, 0, sizeof(float) * N * g.F_ld));
  if (N * F)
    OB_CUDA(cudaMemcpy2D(g.feats, sizeof(float) * g.F_ld, feats, sizeof(float) * F, sizeof(float) * F, N,
                         cudaMemcpyHostToDevice));
  std::sort(deg.begin(), deg.end(), std::greater<int32_t>());
  g.topdeg_prefix.assign((size_t)N + 1, 0);
  for (int64_t i = 0; i < N; ++i) g.topdeg_prefix[i + 1] = g.topdeg_prefix[i] + deg[i];
}

static int nmats(int kind) {
  switch (kind) {
    case OB_KIND_GCN: return 1;
    case OB_KIND_GAT: return 3;
    default: return 2;
  }
}

static void load_model(Engine& e, int k, const ob_layer* layers, const float* const* mats) {
  OB_CHECK(k >= 1 && k <= 7, OB_EINVAL, "model needs 1..7 layers");
  std::vector<LayerDev> out(k);
  int mi = 0;
  for (int l = 0; l < k; ++l) {
    const ob_layer& sp = layers[l];
    OB_CHECK(sp.kind >= 0 && sp.kind <= 5, OB_EINVAL, "unknown layer kind");
    OB_CHECK(sp.in_dim > 0 && sp.out_dim > 0, OB_EINVAL, "layer dims must be positive");
    if (l) OB_CHECK(layers[l - 1].out_dim == sp.in_dim, OB_EINVAL, "adjacent layer dimensions do not chain");
    if (sp.kind == OB_KIND_POWER_MEAN) OB_CHECK(sp.p != 0.f, OB_EINVAL, "power_mean needs p != 0");
    if (sp.kind == OB_KIND_MOMENTS) OB_CHECK(sp.n >= 2, OB_EINVAL, "moments needs n >= 2");
    OB_CHECK(sp.out_dim <= 2048, OB_EINVAL, "layer out_dim above 2048 is not supported");
    LayerDev& L = out[l];
    L.spec = sp;
    const int in = sp.in_dim, o = sp.out_dim;
    // narrowing linear layers aggregate X W instead of X (fewer gathered bytes)
    L.transform_first = (sp.kind == OB_KIND_GCN || sp.kind == OB_KIND_SAGE_MEAN) && in > o;
    if (sp.kind == OB_KIND_GCN) {
      prep_tc_weights(e, {mats[mi]}, {in}, o, &L.tw_main);
    } else if (sp.kind == OB_KIND_GAT) {
      prep_tc_weights(e, {mats[mi]}, {in}, o, &L.tw_main);
      L.a_src = (float*)e.dalloc(sizeof(float) * o);
      L.a_dst = (float*)e.dalloc(sizeof(float) * o);
      {  // W a_dst for owner-side destination scores under CGP (models.py:199-200 reassociated)
        std::vector<float> wa(in);
        for (int i = 0; i < in; ++i) {
          double acc = 0.0;
          for (int j = 0; j < o; ++j) acc += (double)mats[mi][(size_t)i * o + j] * (double)mats[mi + 2][j];
          wa[i] = (float)acc;
        }
        L.wa_dst = (float*)e.dalloc(sizeof(float) * in);
        OB_CUDA(cudaMemcpy(L.wa_dst, wa.data(), sizeof(float) * in, cudaMemcpyHostToDevice));
      }
      OB_CUDA(cudaMemcpy(L.a_src, mats[mi + 1], sizeof(float) * o, cudaMemcpyHostToDevice));
      OB_CUDA(cudaMemcpy(L.a_dst, mats[mi + 2], sizeof(float) * o, cudaMemcpyHostToDevice));
    } else if (L.transform_first) {
      prep_tc_weights(e, {mats[mi + 1]}, {in}, o, &L.tw_main);  // X W_neigh
      prep_tc_weights(e, {mats[mi]}, {in}, o, &L.tw_self);      // h_v W_self (+ mean(X W_neigh))
    } else {
      // [W_self; W_neigh] so the update is one GEMM over [h_v | agg]
      prep_tc_weights(e, {mats[mi], mats[mi + 1]}, {in, in}, o, &L.tw_main);
    }
    mi += nmats(sp.kind);
  }
  for (auto& L : e.layers) free_layer(e, L);  // the old weights (no request can still use them)
  e.layers = out;
}

// ---------------------------------------------------------------------------
// parity export helpers
// ---------------------------------------------------------------------------
__global__ void k_src_degree(const int32_t* __restrict__ src_ids, const BlockCounters* cnt, int64_t N,
                             const int32_t* indeg, const int32_t* qdeg, int64_t* out) {
  pdl_wait();
  const int64_t S = ld_state(&cnt->S);
  OB_GRID_STRIDE(s, S) {
    int64_t g = src_ids[s];
    out[s] = g < N ? indeg[g] : qdeg[g - N];
  }
}

template <class T>
static std::vector<T> d2h(const T* d, int64_t n, cudaStream_t s) {
  std::vector<T> h((size_t)std::max<int64_t>(n, 0));
  if (n > 0) OB_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost, s));
  OB_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace ob

// =============================================================================
// C ABI
// =============================================================================
using namespace ob;

// One slot of the pipelined host path: device staging for one request's
// inputs/outputs, pinned counter readback, and the events that order its H2D
// copy -> request graph -> D2H copy across the three streams.
struct PipeSlot {
  int64_t* d_edges = nullptr;
  float* d_q = nullptr;
  float* d_out = nullptr;
  size_t cap_edges = 0, cap_q = 0, cap_out = 0;
  ReqCounters* h_rc = nullptr;        // pinned
  BlockCounters* h_bc = nullptr;      // pinned [kMaxCounted]
  int n_bc = 0;
  cudaEvent_t h2d_done = nullptr, start = nullptr, comp_done = nullptr, d2h_done = nullptr;
  bool busy = false;
  int64_t ticket = -1;
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  int64_t collective_bytes = 0;
  // pageable `out`: the rows come back into this pinned buffer and are copied
  // to the caller's array in ob_serve_wait (a D2H copy into pageable memory
  // would block the submit until the request finished on the device)
  float* h_out = nullptr;
  size_t cap_h_out = 0;
  float* user_out = nullptr;
  size_t out_bytes = 0;
  int32_t* d_edges32 = nullptr;  // int32 host edges land here and are widened on the device
  size_t cap_edges32 = 0;
};
constexpr int kMaxCounted = 64;
constexpr int kPipeSlots = 4;  // requests in flight on the pipelined host path

struct ob_engine {
  Engine impl;
  std::mutex mu;  // one in-flight request per engine
  // persistent request I/O buffers for the host-pointer path
  int64_t* d_edges = nullptr;
  float* d_q = nullptr;
  float* d_out = nullptr;
  size_t cap_edges = 0, cap_q = 0, cap_out = 0;
  int32_t* d_edges32 = nullptr;
  size_t cap_edges32 = 0;
  // pipelined host path (ob_serve_submit / ob_serve_wait): two slots, so request
  // t+1's inputs cross PCIe while request t runs and t-1's rows come back
  PipeSlot slot[kPipeSlots];
  cudaStream_t h2d = nullptr, d2h = nullptr;
  int64_t next_ticket = 0;
};

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return OB_OK;
  } catch (const Error& err) {
    t_err = err.what();
    return err.code;
  } catch (const std::exception& ex) {
    t_err = ex.what();
    return OB_ECUDA;
  } catch (...) {
    t_err = "unknown error";
    return OB_ECUDA;
  }
}

template <class T>
static void ensure(T*& p, size_t& cap, size_t n) {
  if (n <= cap && p) return;
  if (p) OB_CUDA(cudaFree(p));
  p = nullptr;
  size_t c = std::max<size_t>(n, 64);
  OB_CUDA(cudaMalloc(&p, sizeof(T) * c));
  cap = c;
}

// int32 (src, dst) request edges -> the int64 pairs the pipeline reads (8 host bytes
// per edge over PCIe instead of 16)
__global__ void k_widen_edges(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  pdl_wait();
  const int64_t n4 = n / 4;
  OB_GRID_STRIDE(i, n4) {
    const int4 v = __ldg(reinterpret_cast<const int4*>(in) + i);
    reinterpret_cast<longlong2*>(out)[2 * i] = make_longlong2(v.x, v.y);
    reinterpret_cast<longlong2*>(out)[2 * i + 1] = make_longlong2(v.z, v.w);
  }
  OB_GRID_STRIDE(j, n - 4 * n4) out[4 * n4 + j] = in[4 * n4 + j];
}

template <class T>
static void stage_edges(const T* src, int64_t m, int64_t*& d64, size_t& cap64, int32_t*& d32, size_t& cap32,
                        cudaStream_t copy_s) {
  ensure(d64, cap64, (size_t)(2 * m));
  if (!m) return;
  if constexpr (sizeof(T) == 8) {
    OB_CUDA(cudaMemcpyAsync(d64, src, sizeof(int64_t) * 2 * m, cudaMemcpyHostToDevice, copy_s));
  } else {
    ensure(d32, cap32, (size_t)(2 * m));
    OB_CUDA(cudaMemcpyAsync(d32, src, sizeof(int32_t) * 2 * m, cudaMemcpyHostToDevice, copy_s));
  }
}
template <class T>
static void widen_edges(int64_t m, int64_t* d64, const int32_t* d32, cudaStream_t s) {
  if (sizeof(T) == 8 || !m) return;
  launch_pdl(k_widen_edges, dim3(grid_for(m / 2 + 1, 256)), dim3(256), 0, s, d32, 2 * m, d64);
}

extern "C" {

const char* ob_last_error(void) { return t_err.c_str(); }
int ob_version(void) { return OB_API_VERSION; }

int ob_engine_create(const ob_config* cfg, ob_engine** out) {
  return guarded([&] {
    OB_CHECK(cfg && out, OB_EINVAL, "null argument");
    OB_CHECK(cfg->gamma >= 0.0 && cfg->gamma <= 1.0, OB_EINVAL, "gamma must lie in [0, 1]");
    OB_CHECK(cfg->strategy == OB_STRATEGY_FULL || cfg->strategy == OB_STRATEGY_SAMPLED ||
                 cfg->strategy == OB_STRATEGY_SRPE || cfg->strategy == OB_STRATEGY_SRPE_CGP,
             OB_EINVAL, "unknown strategy");
    if (cfg->strategy == OB_STRATEGY_SAMPLED) {
      OB_CHECK(cfg->num_fanouts >= 1 && cfg->num_fanouts <= OB_MAX_LAYERS, OB_EINVAL, "sampled strategy needs fanouts");
      for (int l = 0; l < cfg->num_fanouts; ++l) {
        OB_CHECK(cfg->fanouts[l] >= 1, OB_EINVAL, "fanouts must be >= 1");
        OB_CHECK(cfg->fanouts[l] <= OB_MAX_FANOUT, OB_EINVAL, "fanout above OB_MAX_FANOUT (200)");
      }
    }
    OB_CHECK(cfg->policy == OB_POLICY_RATIO || cfg->policy == OB_POLICY_IS || cfg->policy == OB_POLICY_RANDOM,
             OB_EINVAL, "unknown policy (ratio, is and random run on the device)");
    OB_CHECK(cfg->num_partitions >= 1, OB_EINVAL, "num_partitions must be >= 1");
    OB_CHECK(cfg->strategy == OB_STRATEGY_SRPE_CGP || cfg->num_partitions == 1, OB_EINVAL,
             "num_partitions > 1 needs strategy srpe-cgp");
    OB_CHECK(cfg->nccl_id == nullptr || (cfg->rank >= 0 && cfg->rank < cfg->num_partitions), OB_EINVAL,
             "rank out of range");
    int ndev = 0;
    OB_CUDA(cudaGetDeviceCount(&ndev));
    OB_CHECK(cfg->device >= 0 && cfg->device < ndev, OB_EINVAL, "no such CUDA device");
    OB_CUDA(cudaSetDevice(cfg->device));
    auto* h = new ob_engine();
    Engine& e = h->impl;
    e.cfg = *cfg;
    if (cfg->stream) {
      e.stream = (cudaStream_t)(uintptr_t)cfg->stream;
    } else {
      OB_CUDA(cudaStreamCreateWithFlags(&e.stream, cudaStreamNonBlocking));
      e.own_stream = true;
    }
    for (auto& ev_ : e.ev) OB_CUDA(cudaEventCreate(&ev_));
    OB_CUDA(cudaStreamCreateWithFlags(&e.side, cudaStreamNonBlocking));
    OB_CUDA(cudaStreamCreateWithFlags(&e.qside, cudaStreamNonBlocking));
    OB_CUDA(cudaEventCreateWithFlags(&e.qfork_ev, cudaEventDisableTiming));
    OB_CUDA(cudaEventCreateWithFlags(&e.qjoin_ev, cudaEventDisableTiming));
    OB_CUDA(cudaEventCreateWithFlags(&e.fork_ev, cudaEventDisableTiming));
    OB_CUDA(cudaEventCreateWithFlags(&e.join_ev, cudaEventDisableTiming));
    OB_CUDA(cudaEventCreateWithFlags(&e.csr_ev, cudaEventDisableTiming));
    configure_fill();
    if (const char* v = std::getenv("OB_NO_GRAPHS")) e.use_graphs = !(v[0] && v[0] != '0');
    if (cfg->nccl_id && cfg->strategy == OB_STRATEGY_SRPE_CGP) {
      try {
        cgp_init_comm(e);
      } catch (...) {
        delete h;
        throw;
      }
    }
    *out = h;
  });
}

int ob_engine_destroy(ob_engine* h) {
  return guarded([&] {
    if (!h) return;
    cudaSetDevice(h->impl.cfg.device);
    for (int i = 1; i <= (int)h->impl.lanes.size(); ++i) {  // every lane's NVLink exchange, with the peers
      LaneGuard lg(h->impl, i);
      cgp_release_exchange(h->impl);
    }
    if (h->h2d) cudaStreamSynchronize(h->h2d);
    if (h->d2h) cudaStreamSynchronize(h->d2h);
    cudaStreamSynchronize(h->impl.stream);
    if (h->d_edges) cudaFree(h->d_edges);
    if (h->d_edges32) cudaFree(h->d_edges32);
    if (h->d_q) cudaFree(h->d_q);
    if (h->d_out) cudaFree(h->d_out);
    for (auto& sl : h->slot) {
      if (sl.d_edges) cudaFree(sl.d_edges);
      if (sl.d_edges32) cudaFree(sl.d_edges32);
      if (sl.d_q) cudaFree(sl.d_q);
      if (sl.d_out) cudaFree(sl.d_out);
      if (sl.h_rc) cudaFreeHost(sl.h_rc);
      if (sl.h_bc) cudaFreeHost(sl.h_bc);
      if (sl.h_out) cudaFreeHost(sl.h_out);
      for (cudaEvent_t ev : {sl.h2d_done, sl.start, sl.comp_done, sl.d2h_done})
        if (ev) cudaEventDestroy(ev);
    }
    if (h->h2d) cudaStreamDestroy(h->h2d);
    if (h->d2h) cudaStreamDestroy(h->d2h);
    delete h;
  });
}

int ob_load_graph(ob_engine* h, int64_t N, const int64_t* off, const int64_t* nb, int64_t E, const float* feats,
                  int32_t F) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    OB_CUDA(cudaSetDevice(h->impl.cfg.device));
    h->impl.invalidate_state();  // graphs and stored tables follow the weights, features and PE
    load_graph(h->impl, N, off, nb, E, feats, F);
    if (h->impl.cfg.strategy == OB_STRATEGY_SRPE_CGP) cgp_build_partitions(h->impl);
  });
}

int ob_generate_graph(ob_engine* h, int64_t N, double avg_degree, double exponent, int32_t F, uint64_t seed) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    OB_CUDA(cudaSetDevice(h->impl.cfg.device));
    h->impl.invalidate_state();  // graphs and stored tables follow the weights, features and PE
    generate_graph(h->impl, N, avg_degree, exponent, F, seed);
  });
}

int ob_generate_pe(ob_engine* h, int32_t layer, int32_t dim, uint64_t seed) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    OB_CUDA(cudaSetDevice(h->impl.cfg.device));
    h->impl.invalidate_state();  // graphs and stored tables follow the weights, features and PE
    generate_pe(h->impl, layer, dim, seed);
  });
}

int ob_graph_info(ob_engine* h, int64_t* num_nodes, int64_t* num_edges, int64_t* local_rows, int64_t* local_edges) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    const Engine& e = h->impl;
    if (num_nodes) *num_nodes = e.g.N;
    if (num_edges) *num_edges = e.g.E;
    if (local_rows) *local_rows = e.g.pos ? e.g.N_local : e.g.N;
    if (local_edges) {
      int64_t le = 0;
      if (e.cfg.strategy == OB_STRATEGY_SRPE_CGP && e.cgp.nccl)
        for (const auto& p : e.cgp.parts) le += p.E;
      else
        le = e.g.E;
      *local_edges = le;
    }
  });
}

int ob_graph_csr(ob_engine* h, int32_t partition, int64_t* offsets, int64_t* nbrs, int32_t* indeg) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    const int64_t N = e.g.N;
    OB_CHECK(N > 0, OB_ESTATE, "no graph loaded");
    const int64_t* off = e.g.offsets;
    const int32_t* nb = e.g.nbrs;
    int64_t E = e.g.E;
    if (partition >= 0) {
      const PartitionDev* p = nullptr;
      for (const auto& q : e.cgp.parts)
        if (q.rank == partition) p = &q;
      OB_CHECK(p, OB_EINVAL, "partition not held by this engine");
      off = p->off;
      nb = p->src;
      E = p->E;
    }
    OB_CHECK(off, OB_ESTATE, "the whole in-CSR is not held by this engine");
    if (offsets) OB_CUDA(cudaMemcpy(offsets, off, sizeof(int64_t) * (N + 1), cudaMemcpyDeviceToHost));
    if (nbrs && E) {
      std::vector<int32_t> t((size_t)E);
      OB_CUDA(cudaMemcpy(t.data(), nb, sizeof(int32_t) * E, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < E; ++i) nbrs[i] = t[i];
    }
    if (indeg) OB_CUDA(cudaMemcpy(indeg, e.g.indeg, sizeof(int32_t) * N, cudaMemcpyDeviceToHost));
  });
}

int ob_read_rows(ob_engine* h, int32_t table, int64_t n, const int64_t* ids, float* out) {
  return guarded([&] {
    OB_CHECK(h && (n == 0 || (ids && out)), OB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    OB_CHECK(table >= 0 && table <= (int)e.pe.size(), OB_EINVAL, "table: 0 = features, l = stored layer l");
    const float* base = table == 0 ? e.g.feats : e.pe[table - 1];
    const int w = table == 0 ? e.g.F : e.pe_dim[table - 1];
    OB_CHECK(base, OB_EINVAL, "table not loaded");
    std::vector<int32_t> pos;
    if (e.g.pos) {
      pos.resize((size_t)e.g.N);
      OB_CUDA(cudaMemcpy(pos.data(), e.g.pos, sizeof(int32_t) * e.g.N, cudaMemcpyDeviceToHost));
    }
    for (int64_t i = 0; i < n; ++i) {
      OB_CHECK(ids[i] >= 0 && ids[i] < e.g.N, OB_EINVAL, "row id out of range");
      const int64_t r = e.g.pos ? pos[ids[i]] : ids[i];
      OB_CHECK(r >= 0, OB_ENOTFOUND, "row not stored on this rank");
      OB_CUDA(cudaMemcpy(out + i * w, base + r * ld4(w), sizeof(float) * w, cudaMemcpyDeviceToHost));
    }
  });
}

int ob_load_pe(ob_engine* h, int32_t layer, const float* rows, int64_t n, int32_t dim) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    e.invalidate_state();  // graphs and stored tables follow the weights, features and PE
    OB_CHECK(e.g.N > 0, OB_ESTATE, "load the graph before stored embeddings");
    OB_CHECK(layer >= 1 && layer <= 7, OB_EINVAL, "bad stored-embedding layer");
    OB_CHECK(n == e.g.N, OB_EINVAL, "stored embeddings must cover every node");
    OB_CHECK(dim > 0 && rows, OB_EINVAL, "bad stored-embedding rows");
    if ((int)e.pe.size() < layer) {
      e.pe.resize(layer, nullptr);
      e.pe_dim.resize(layer, 0);
    }
    OB_CHECK(!e.g.generated || !e.g.pos, OB_ESTATE, "partitioned generated graph: use ob_generate_pe");
    const int ld = ld4(dim);
    float* d = (float*)e.dalloc(sizeof(float) * n * ld);
    OB_CUDA(cudaMemset(d, 0, sizeof(float) * n * ld));
    OB_CUDA(cudaMemcpy2D(d, sizeof(float) * ld, rows, sizeof(float) * dim, sizeof(float) * dim, n,
                         cudaMemcpyHostToDevice));
    e.dfree(e.pe[layer - 1]);
    e.pe[layer - 1] = d;
    e.pe_dim[layer - 1] = dim;
    if (e.localized) localize_table(e, e.pe[layer - 1], ld);  // keep the owned rows only
  });
}

int ob_load_model(ob_engine* h, int32_t k, const ob_layer* layers, const float* const* mats) {
  return guarded([&] {
    OB_CHECK(h && layers && mats, OB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(h->mu);
    OB_CUDA(cudaSetDevice(h->impl.cfg.device));
    h->impl.invalidate_state();  // graphs and stored tables follow the weights, features and PE
    load_model(h->impl, k, layers, mats);
  });
}

int ob_precompute_pe(ob_engine* h) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    OB_CUDA(cudaSetDevice(h->impl.cfg.device));
    h->impl.invalidate_state();  // graphs and stored tables follow the weights, features and PE
    OB_CHECK(!h->impl.layers.empty(), OB_ESTATE, "load a model first");
    OB_CHECK(h->impl.layers[0].spec.in_dim == h->impl.g.F, OB_EINVAL, "input width does not match layer in_dim");
    OB_CHECK(h->impl.g.offsets && !h->impl.g.pos, OB_ESTATE,
             "precompute needs the whole graph on this device (partitioned engines: precompute before serving)");
    stage_precompute(h->impl);
    OB_CUDA(cudaGetLastError());
  });
}

int ob_read_pe(ob_engine* h, int32_t layer, float* out) {
  return guarded([&] {
    OB_CHECK(h && out, OB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    OB_CHECK(layer >= 1 && layer <= (int)e.pe.size() && e.pe[layer - 1], OB_EINVAL,
             "no stored embeddings for that layer");
    OB_CHECK(!e.g.pos, OB_ESTATE, "stored embeddings are partitioned across ranks on this engine");
    const int dim = e.pe_dim[layer - 1];
    OB_CUDA(cudaMemcpy2D(out, sizeof(float) * dim, e.pe[layer - 1], sizeof(float) * ld4(dim), sizeof(float) * dim,
                         e.g.N, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C" (the host-path templates have C++ linkage)

template <class T>
static int serve_host(ob_engine* h, int32_t B, const float* q, int64_t m, const T* edges, float* out,
                      ob_breakdown* bd) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    check_ready(e);
    OB_CHECK(B >= 0 && m >= 0, OB_EINVAL, "negative request size");
    OB_CHECK(m == 0 || edges, OB_EINVAL, "null edges");
    OB_CHECK(out, OB_EINVAL, "null output");
    const int H = e.layers.back().spec.out_dim;
    cudaStream_t s = e.stream;
    stage_edges(edges, m, h->d_edges, h->cap_edges, h->d_edges32, h->cap_edges32, s);
    ensure(h->d_q, h->cap_q, (size_t)B * e.g.F);
    ensure(h->d_out, h->cap_out, (size_t)B * H);
    if ((int64_t)B * e.g.F) OB_CUDA(cudaMemcpyAsync(h->d_q, q, sizeof(float) * B * e.g.F, cudaMemcpyHostToDevice, s));
    widen_edges<T>(m, h->d_edges, h->d_edges32, s);
    ob_breakdown local{};
    serve_device(e, B, h->d_q, m, h->d_edges, h->d_out, &local);
    e.last_lane = 0;
    if ((int64_t)B * H) OB_CUDA(cudaMemcpyAsync(out, h->d_out, sizeof(float) * B * H, cudaMemcpyDeviceToHost, s));
    OB_CUDA(cudaStreamSynchronize(s));
    local.h2d_bytes = 2 * (int64_t)sizeof(T) * m + 4 * (int64_t)B * e.g.F;
    local.d2h_bytes = 4 * (int64_t)B * H;
    if (bd) *bd = local;
  });
}

extern "C" {

int ob_serve(ob_engine* h, int32_t B, const float* q, int64_t m, const int64_t* edges, float* out,
             ob_breakdown* bd) {
  return serve_host(h, B, q, m, edges, out, bd);
}

int ob_serve_i32(ob_engine* h, int32_t B, const float* q, int64_t m, const int32_t* edges, float* out,
                 ob_breakdown* bd) {
  return serve_host(h, B, q, m, edges, out, bd);
}

// Pipelined host path.  Request t uses slot t % kPipeSlots (four slots): its
// H2D copy runs on the h2d stream (after slot t's previous request finished on
// the device), its request graph on its request lane's stream (after the copy
// and after the slot's previous D2H), its D2H copy and counter readback on the
// d2h stream.  Up to kPipeSlots requests are outstanding; ob_serve_wait(t)
// returns request t's rows in `out` and its breakdown (errors of request t are
// raised there).  The D2H into `out` overlaps only when `out` is pinned
// (page-locked) host memory; a pageable `out` makes the submit wait for it.
}  // extern "C"

template <class T>
static int submit_host(ob_engine* h, int32_t B, const float* q, int64_t m, const T* edges, float* out,
                       int64_t* ticket) {
  return guarded([&] {
    OB_CHECK(h && ticket, OB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    check_ready(e);
    OB_CHECK(B >= 0 && m >= 0, OB_EINVAL, "negative request size");
    OB_CHECK(m == 0 || edges, OB_EINVAL, "null edges");
    OB_CHECK(out, OB_EINVAL, "null output");
    const int64_t t = h->next_ticket;
    PipeSlot& sl = h->slot[t % kPipeSlots];
    OB_CHECK(!sl.busy, OB_ESTATE, "four requests already outstanding: wait for the oldest first");
    if (!h->h2d) {
      OB_CUDA(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking));
      OB_CUDA(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking));
    }
    if (!sl.h2d_done) {
      for (cudaEvent_t* ev : {&sl.h2d_done, &sl.start, &sl.comp_done, &sl.d2h_done}) OB_CUDA(cudaEventCreate(ev));
      OB_CUDA(cudaMallocHost(&sl.h_rc, sizeof(ReqCounters)));
      OB_CUDA(cudaMallocHost(&sl.h_bc, sizeof(BlockCounters) * kMaxCounted));
    }
    const int H = e.layers.back().spec.out_dim;
    // the slot is idle: its previous request was waited for, so its buffers can be resized
    stage_edges(edges, m, sl.d_edges, sl.cap_edges, sl.d_edges32, sl.cap_edges32, h->h2d);
    ensure(sl.d_q, sl.cap_q, (size_t)B * e.g.F);
    ensure(sl.d_out, sl.cap_out, (size_t)B * H);
    if ((int64_t)B * e.g.F)
      OB_CUDA(cudaMemcpyAsync(sl.d_q, q, sizeof(float) * B * e.g.F, cudaMemcpyHostToDevice, h->h2d));
    OB_CUDA(cudaEventRecord(sl.h2d_done, h->h2d));
    const int lane = (int)(t % kPipeSlots) % e.nlanes;  // with several lanes the slots' requests overlap
    LaneGuard lg(e, lane);
    e.last_lane = lane;
    cudaStream_t s = e.stream;
    OB_CUDA(cudaStreamWaitEvent(s, sl.h2d_done, 0));
    OB_CUDA(cudaEventRecord(sl.start, s));
    widen_edges<T>(m, sl.d_edges, sl.d_edges32, s);
    enqueue_serve(e, B, sl.d_q, m, sl.d_edges, sl.d_out);
    std::vector<BlockDev*> all = counted_blocks(e);
    OB_CHECK((int)all.size() <= kMaxCounted, OB_ESTATE, "too many blocks for the pipelined readback");
    OB_CUDA(cudaMemcpyAsync(sl.h_rc, e.ws.rc, sizeof(ReqCounters), cudaMemcpyDeviceToHost, s));
    for (size_t i = 0; i < all.size(); ++i)
      OB_CUDA(cudaMemcpyAsync(sl.h_bc + i, all[i]->cnt, sizeof(BlockCounters), cudaMemcpyDeviceToHost, s));
    OB_CUDA(cudaEventRecord(sl.comp_done, s));
    OB_CUDA(cudaStreamWaitEvent(h->d2h, sl.comp_done, 0));
    // pinned (page-locked or registered) `out` takes the copy directly, pageable goes through h_out
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, out) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    sl.out_bytes = sizeof(float) * (size_t)B * H;
    sl.user_out = pinned ? nullptr : out;
    if (!pinned && sl.out_bytes > sl.cap_h_out) {
      if (sl.h_out) OB_CUDA(cudaFreeHost(sl.h_out));
      sl.h_out = nullptr;
      sl.cap_h_out = 0;
      OB_CUDA(cudaMallocHost(&sl.h_out, sl.out_bytes));
      sl.cap_h_out = sl.out_bytes;
    }
    if (sl.out_bytes)
      OB_CUDA(cudaMemcpyAsync(pinned ? out : sl.h_out, sl.d_out, sl.out_bytes, cudaMemcpyDeviceToHost, h->d2h));
    OB_CUDA(cudaEventRecord(sl.d2h_done, h->d2h));
    sl.n_bc = (int)all.size();
    sl.busy = true;
    sl.ticket = t;
    sl.h2d_bytes = 2 * (int64_t)sizeof(T) * m + 4 * (int64_t)B * e.g.F;
    sl.d2h_bytes = 4 * (int64_t)B * H;
    sl.collective_bytes = e.cgp.collective_bytes;
    h->next_ticket = t + 1;
    *ticket = t;
  });
}

extern "C" {

int ob_serve_submit(ob_engine* h, int32_t B, const float* q, int64_t m, const int64_t* edges, float* out,
                    int64_t* ticket) {
  return submit_host(h, B, q, m, edges, out, ticket);
}

int ob_serve_submit_i32(ob_engine* h, int32_t B, const float* q, int64_t m, const int32_t* edges, float* out,
                        int64_t* ticket) {
  return submit_host(h, B, q, m, edges, out, ticket);
}

int ob_serve_wait(ob_engine* h, int64_t ticket, ob_breakdown* bd) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    OB_CHECK(ticket >= 0, OB_EINVAL, "bad ticket");
    PipeSlot& sl = h->slot[ticket % kPipeSlots];
    OB_CHECK(sl.busy && sl.ticket == ticket, OB_ESTATE, "ticket is not outstanding");
    // the next slot's request keeps running; only this one's D2H is awaited
    OB_CUDA(cudaEventSynchronize(sl.d2h_done));
    sl.busy = false;
    if (sl.user_out && sl.out_bytes) std::memcpy(sl.user_out, sl.h_out, sl.out_bytes);
    OB_CUDA(cudaGetLastError());
    float ms = 0;
    OB_CUDA(cudaEventElapsedTime(&ms, sl.start, sl.comp_done));
    std::vector<BlockCounters> hc(sl.h_bc, sl.h_bc + sl.n_bc);
    LaneGuard lg(e, (int)(ticket % kPipeSlots) % e.nlanes);
    ob_breakdown local{};
    // counters of the request that was last enqueued describe the workspace
    // layout; both slots share one plan once the shape is reserved
    finish_breakdown(e, *sl.h_rc, hc, 0.f, ms, &local);
    local.fetch_ms = 0.0;  // the stage split is not recorded per slot
    local.compute_ms = ms;
    local.total_device_ms = ms;
    if (!(e.cfg.strategy == OB_STRATEGY_SRPE_CGP && e.cgp.nccl && e.cgp.p2p)) local.collective_bytes = sl.collective_bytes;
    local.h2d_bytes = sl.h2d_bytes;
    local.d2h_bytes = sl.d2h_bytes;
    if (bd) *bd = local;
  });
}

int ob_serve_device(ob_engine* h, int32_t B, const float* d_q, int64_t m, const int64_t* d_edges, float* d_out,
                    ob_breakdown* bd) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    const int lane = e.nlanes > 1 ? (int)(e.lane_rr++ % e.nlanes) : 0;
    LaneGuard g(e, lane);
    serve_device(e, B, d_q, m, d_edges, d_out, bd);
    e.last_lane = lane;
  });
}

int ob_set_lanes(ob_engine* h, int32_t n) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    OB_CHECK(n >= 1 && n <= 8, OB_EINVAL, "lanes must be 1..8");
    OB_CHECK(n == 1 || e.cfg.strategy != OB_STRATEGY_SRPE_CGP || !e.cgp.nccl || e.cgp.p2p, OB_EINVAL,
             "CGP lanes need the NVLink exchange (each lane has its own; OB_CGP_NCCL=1 serialises on one comm)");
    OB_CHECK(n == 1 || !e.prof.on, OB_ESTATE, "profiling runs on one lane");
    for (auto& sl : h->slot) OB_CHECK(!sl.busy, OB_ESTATE, "wait for the outstanding pipelined requests first");
    OB_CUDA(cudaDeviceSynchronize());
    if (!e.lane_fork_ev) OB_CUDA(cudaEventCreateWithFlags(&e.lane_fork_ev, cudaEventDisableTiming));
    while ((int)e.lanes.size() < n - 1) {
      e.lanes.emplace_back();
      Lane& L = e.lanes.back();
      OB_CUDA(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking));
      OB_CUDA(cudaStreamCreateWithFlags(&L.side, cudaStreamNonBlocking));
      OB_CUDA(cudaStreamCreateWithFlags(&L.qside, cudaStreamNonBlocking));
      OB_CUDA(cudaEventCreateWithFlags(&L.qfork_ev, cudaEventDisableTiming));
      OB_CUDA(cudaEventCreateWithFlags(&L.qjoin_ev, cudaEventDisableTiming));
      for (auto& ev_ : L.ev) OB_CUDA(cudaEventCreate(&ev_));
      for (cudaEvent_t* ev_ : {&L.fork_ev, &L.join_ev, &L.csr_ev, &L.done_ev})
        OB_CUDA(cudaEventCreateWithFlags(ev_, cudaEventDisableTiming));
    }
    if (n != e.nlanes) {  // the gather plan depends on the lane count: re-capture every lane's graphs
      e.drop_graphs();
      for (auto& L : e.lanes) {
        for (auto& gr : L.graphs)
          if (gr.exec) cudaGraphExecDestroy(gr.exec);
        L.graphs.clear();
      }
    }
    e.nlanes = n;
    e.lane_rr = 0;
  });
}

// order every lane after the work enqueued so far on lane 0's stream
int ob_lanes_fork(ob_engine* h) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    if (e.nlanes < 2) return;
    OB_CUDA(cudaEventRecord(e.lane_fork_ev, e.stream));
    for (int i = 0; i + 1 < e.nlanes; ++i) OB_CUDA(cudaStreamWaitEvent(e.lanes[i].stream, e.lane_fork_ev, 0));
  });
}

// order lane 0's stream after everything enqueued on the other lanes
int ob_lanes_join(ob_engine* h) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    for (int i = 0; i + 1 < e.nlanes; ++i) {
      OB_CUDA(cudaEventRecord(e.lanes[i].done_ev, e.lanes[i].stream));
      OB_CUDA(cudaStreamWaitEvent(e.stream, e.lanes[i].done_ev, 0));
    }
  });
}

int ob_last_plan(ob_engine* h, int64_t* nc, int64_t* nt, int64_t* ids, int64_t* nq, int64_t* total, double* scores,
                 int64_t* targets) {
  return guarded([&] {
    OB_CHECK(h && nc && nt, OB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    OB_CHECK(e.have_request && !khop(e.cfg), OB_ESTATE, "no srpe request served");
    LaneGuard lg(e, e.last_lane);
    OB_CUDA(cudaDeviceSynchronize());
    RequestWs& w = e.ws;
    cudaStream_t s = e.stream;
    ReqCounters rc = d2h(w.rc, 1, s)[0];
    *nc = rc.R;
    *nt = rc.T;
    if (ids) {
      auto a = d2h(w.cand_ids, rc.R, s);
      auto b = d2h(w.cand_nq, rc.R, s);
      std::vector<int32_t> deg((size_t)rc.R);
      // total = training in-degree + nq (policy.py:64-67)
      std::vector<int32_t> indeg = d2h(e.g.indeg, e.g.N, s);
      for (int64_t i = 0; i < rc.R; ++i) {
        ids[i] = a[i];
        if (nq) nq[i] = b[i];
        if (total) total[i] = (int64_t)indeg[a[i]] + b[i];
      }
      if (scores) {
        auto c = d2h(w.cand_score, rc.R, s);
        std::copy(c.begin(), c.end(), scores);
      }
    }
    if (targets) {
      auto t = d2h(w.targets, rc.T, s);
      for (int64_t i = 0; i < rc.T; ++i) targets[i] = t[i];
    }
  });
}

// the block that fed `layer` on partition `part` (centralized: part 0)
static BlockDev& block_of(Engine& e, int part, int layer) {
  OB_CHECK(e.have_request, OB_ESTATE, "no request served");
  OB_CHECK(layer >= 1 && layer <= (int)e.layers.size(), OB_EINVAL, "layer out of range");
  const int k = (int)e.layers.size();
  if (e.cfg.strategy == OB_STRATEGY_SRPE_CGP) {
    const CgpState& c = e.cgp;
    int idx = -1;
    for (size_t i = 0; i < c.parts.size(); ++i)
      if (c.parts[i].rank == part) idx = (int)i;
    OB_CHECK(idx >= 0, OB_EINVAL, "partition not held by this engine");
    return e.cgp.ws[idx].blocks[layer < k ? 0 : 1];
  }
  OB_CHECK(part == 0, OB_EINVAL, "partition index out of range");
  return e.ws.blocks[e.ws.block_of_layer[layer - 1]];
}

int ob_last_block_sizes(ob_engine* h, int32_t part, int32_t layer, int64_t* ns, int64_t* nd, int64_t* ne) {
  return guarded([&] {
    OB_CHECK(h && ns && nd && ne, OB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    LaneGuard lg(e, e.last_lane);
    OB_CUDA(cudaDeviceSynchronize());
    BlockDev& b = block_of(e, part, layer);
    BlockCounters c = d2h(b.cnt, 1, e.stream)[0];
    *ns = c.S;
    *nd = c.D;
    *ne = c.E;
  });
}

int ob_last_block(ob_engine* h, int32_t part, int32_t layer, int64_t* src_ids, int64_t* dst_ids, int64_t* edge_src,
                  int64_t* edge_dst, uint8_t* bind_kind, int32_t* bind_pe_layer, int64_t* src_degree,
                  int64_t* dst_self_src) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    LaneGuard lg(e, e.last_lane);
    OB_CUDA(cudaDeviceSynchronize());
    RequestWs& w = e.ws;
    BlockDev& b = block_of(e, part, layer);
    cudaStream_t s = e.stream;
    BlockCounters c = d2h(b.cnt, 1, s)[0];
    auto cp32 = [&](const int32_t* d, int64_t n, int64_t* o) {
      if (!o) return;
      auto v = d2h(d, n, s);
      for (int64_t i = 0; i < n; ++i) o[i] = v[i];
    };
    cp32(b.src_ids, c.S, src_ids);
    cp32(b.dst_ids, c.D, dst_ids);
    cp32(b.edge_src, c.E, edge_src);
    if (b.has_self) cp32(b.self_src, c.D, dst_self_src);
    if (edge_dst) {
      auto ptr = d2h(b.dst_ptr, c.D + 1, s);
      for (int64_t i = 0; i < c.D; ++i)
        for (int64_t j = ptr[i]; j < ptr[i + 1]; ++j) edge_dst[j] = i;
    }
    if (bind_kind || bind_pe_layer || src_degree) {
      uint8_t* dk = nullptr;
      int32_t* dp = nullptr;
      int64_t* dd = nullptr;
      OB_CUDA(cudaMalloc(&dk, std::max<int64_t>(c.S, 1)));
      OB_CUDA(cudaMalloc(&dp, sizeof(int32_t) * std::max<int64_t>(c.S, 1)));
      OB_CUDA(cudaMalloc(&dd, sizeof(int64_t) * std::max<int64_t>(c.S, 1)));
      export_bindings(e, w, b, layer, dk, dp);
      launch_pdl(k_src_degree, dim3(grid_for(std::max<int64_t>(c.S, 1), 256)), dim3(256), 0, s, b.src_ids, b.cnt, e.g.N, e.g.indeg,
                                                                             w.qdeg, dd);
      auto k1 = d2h(dk, c.S, s);
      auto k2 = d2h(dp, c.S, s);
      auto k3 = d2h(dd, c.S, s);
      if (bind_kind) std::copy(k1.begin(), k1.end(), bind_kind);
      if (bind_pe_layer) std::copy(k2.begin(), k2.end(), bind_pe_layer);
      if (src_degree) std::copy(k3.begin(), k3.end(), src_degree);
      cudaFree(dk);
      cudaFree(dp);
      cudaFree(dd);
    }
  });
}

int ob_reserve(ob_engine* h, int32_t B, int64_t m) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    check_ready(e);
    cgp_localize_storage(e);
    e.m_reserved = bucket_m(m);
    prepare_workspace(e, B, e.m_reserved);
    const int H = e.layers.back().spec.out_dim;
    ensure(h->d_edges, h->cap_edges, (size_t)(2 * m));
    ensure(h->d_q, h->cap_q, (size_t)B * e.g.F);
    ensure(h->d_out, h->cap_out, (size_t)B * H);
  });
}

int ob_set_graphs(ob_engine* h, int32_t enable) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    OB_CUDA(cudaSetDevice(h->impl.cfg.device));
    OB_CUDA(cudaStreamSynchronize(h->impl.stream));
    h->impl.use_graphs = enable != 0;
    if (!enable) h->impl.drop_graphs();
  });
}

int ob_profile(ob_engine* h, int32_t enable) {
  return guarded([&] {
    OB_CHECK(h, OB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lk(h->mu);
    OB_CUDA(cudaSetDevice(h->impl.cfg.device));
    OB_CHECK(!enable || h->impl.nlanes == 1, OB_ESTATE, "profiling runs on one lane (ob_set_lanes(e, 1))");
    OB_CUDA(cudaStreamSynchronize(h->impl.stream));
    h->impl.prof.reset();
    h->impl.prof.on = enable != 0;
    if (enable) h->impl.prof.prime(8192);
  });
}

int ob_profile_read(ob_engine* h, int32_t cls, double* total_ms, int64_t* launches, double* alg_bytes,
                    double* flops) {
  return guarded([&] {
    OB_CHECK(h && total_ms && launches && alg_bytes && flops, OB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    OB_CUDA(cudaStreamSynchronize(e.stream));
    double ms = 0, by = 0, fl = 0;
    int64_t n = 0;
    for (const ProfRec& r : e.prof.recs) {
      if (cls == kProfRequest && r.cls == kProfCount) {  // the profiler's own row counts are not request time
        float t = 0;
        OB_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
        ms -= t;
        continue;
      }
      if (r.cls != cls) continue;
      float t = 0;
      OB_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
      ms += t;
      ++n;
      if (r.slot < 0) continue;
      const BlockCounters& c = e.prof.pinned[r.slot];
      if (cls == kProfAgg && r.K < 0) {
        // stored-aggregate (K = -1) or delta (K = -2) launch: edge list, every distinct row it
        // loaded once (request-span sources, delta rows of recomputed CSR sources; counted on the
        // device by k_prof_rows) and the partials
        by += 4.0 * c.E + 4.0 * r.width * c.uniq + 4.0 * r.pw * c.items;
        fl += 4.0 * r.width * c.gathered;  // row bytes it loaded (one row per kept edge)
      } else if (cls == kProfAgg) {
        // edge list + every source row once + partial rows out
        by += 4.0 * c.E + 4.0 * r.width * c.S + 4.0 * r.pw * c.items;
        fl += 4.0 * r.width * c.E;  // gathered row bytes (rows are re-read once per edge, mostly from L2)
      } else if (cls == kProfFinalize) {
        by += 4.0 * r.pw * c.items + 4.0 * r.width * c.D;
      } else if (cls == kProfGemm) {
        double M = r.gemm_rows ? c.S : c.D;
        fl += 2.0 * M * r.K * r.Nc;
        by += 4.0 * (M * r.K + (double)r.K * r.Nc + M * r.Nc);
      }
    }
    *total_ms = ms;
    *launches = n;
    *alg_bytes = by;
    *flops = fl;
  });
}

int ob_partition_owner(ob_engine* h, int64_t* owner) {
  return guarded([&] {
    OB_CHECK(h && owner, OB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(h->mu);
    Engine& e = h->impl;
    OB_CUDA(cudaSetDevice(e.cfg.device));
    OB_CHECK(e.cfg.strategy == OB_STRATEGY_SRPE_CGP && e.cgp.owner, OB_ESTATE, "engine is not partitioned");
    auto v = d2h(e.cgp.owner, e.g.N, e.stream);
    for (int64_t i = 0; i < e.g.N; ++i) owner[i] = v[i];
  });
}

int64_t ob_launch_count(ob_engine* h) {
  (void)h;
  return g_launches;
}

int ob_nccl_unique_id(void* out128) {
  return guarded([&] {
    OB_CHECK(out128, OB_EINVAL, "null argument");
#ifdef OB_WITH_NCCL
    ncclUniqueId id;
    OB_CHECK(ncclGetUniqueId(&id) == ncclSuccess, OB_ECOMM, "ncclGetUniqueId failed");
    std::memcpy(out128, &id, sizeof(id));
#else
    OB_CHECK(false, OB_ECOMM, "built without NCCL");
#endif
  });
}

}  // extern "C"
