// ob_cgp.cu -- computation-graph parallelism (CGP) on B200s.
//
// Reference (paths relative to /root/reference/pkg/src/gnnserve):
//   partition_random_hash    graphstore.py:219-263  owner = splitmix64(v ^ splitmix64(seed)) % P,
//                                                   edges stored at their source's owner
//   partition_request        compgraph.py:367-392   request edge -> owner of its source
//   select_targets_distributed runtime.py:151-192   identical plan on every rank
//   build_partitioned        compgraph.py:395-459   global dst lists, local sources only
//   execute_layer/_model     cgpexec.py:308-439     local partials -> owner merge -> update
//
// B200 mapping.  Every rank receives the whole request (it is small next to the
// graph), so candidate scoring and the top-k run redundantly and identically on
// every rank -- the reference's stats all-gather disappears.  A rank builds the
// part of both blocks whose sources it owns (its source-split CSR + its request
// slice) with the same device builder as the centralized path, aggregates
// locally into one raw partial per destination (sum / max / softmax triple), and
// the partials are combined across ranks:
//   * NCCL mode (one process per GPU, ob_config.nccl_id): by default every
//     rank writes its partial rows into its own CUDA-IPC exchange region and the
//     owners read the peers' regions in place over NVLink ("NVLink exchange"
//     below: device step counters, release/acquire flags, owner-only merges);
//     OB_CGP_NCCL=1 selects ncclAllReduce on destination-indexed buffers padded
//     to the request bound instead; owners then update their destinations and
//     the query rows go to rank 0;
//   * emulation (nccl_id == NULL, P > 1): all P partitions run on this device and
//     the merge walks the P partials in ascending rank order (cgpexec.py:189-240).
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "ob_engine.h"

#ifdef OB_WITH_NCCL
#include <nccl.h>
#endif

namespace ob {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser (graphstore.py:25-30)
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_owner(int64_t N, int P, uint64_t seed, int32_t* owner) {
  pdl_wait();  // declared in ob_engine.h
  const uint64_t key = mix64(seed);
  OB_GRID_STRIDE(v, N) owner[v] = (int32_t)(mix64((uint64_t)v ^ key) % (uint64_t)P);
}

// per destination row: number of in-neighbours owned by partition r (warp per row)
__global__ void k_part_deg(int64_t N, const int64_t* __restrict__ off, const int32_t* __restrict__ nbrs,
                           const int32_t* __restrict__ owner, int r, int32_t* deg) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < N; v += nw) {
    int c = 0;
    for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32) c += owner[nbrs[e]] == r;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) deg[v] = c;
  }
}

// ordered compaction of the owned in-neighbours (ascending order preserved)
__global__ void k_part_fill(int64_t N, const int64_t* __restrict__ off, const int32_t* __restrict__ nbrs,
                            const int32_t* __restrict__ owner, int r, const int64_t* __restrict__ poff,
                            int32_t* psrc) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < N; v += nw) {
    int64_t out = poff[v];
    for (int64_t e0 = off[v]; e0 < off[v + 1]; e0 += 32) {
      const int64_t e = e0 + lane;
      const bool keep = e < off[v + 1] && owner[nbrs[e]] == r;
      const unsigned b = __ballot_sync(0xffffffffu, keep);
      if (keep) psrc[out + __popc(b & ((1u << lane) - 1u))] = nbrs[e];
      out += __popc(b);
    }
  }
}

void cgp_build_partitions(Engine& e) {
  CgpState& c = e.cgp;
  cudaStream_t s = e.stream;
  const int64_t N = e.g.N;
  c.P = e.cfg.num_partitions;
  c.nccl = e.cfg.nccl_id != nullptr;
  c.my_rank = c.nccl ? e.cfg.rank : 0;
  c.owner = (int32_t*)e.dalloc(sizeof(int32_t) * N);
  launch_pdl(k_owner, dim3(grid_for(N, 256)), dim3(256), 0, s, N, c.P, e.cfg.seed, c.owner);
  ScanScratch sc;
  sc.cap = ScanScratch::bytes_for(N, c.P);
  sc.pool = (char*)e.dalloc(sc.cap);
  OB_CUDA(cudaMemsetAsync(sc.pool, 0, sc.cap, s));
  int64_t* total = (int64_t*)e.dalloc(sizeof(int64_t));
  c.parts.clear();
  for (int r = 0; r < c.P; ++r) {
    if (c.nccl && r != c.my_rank) continue;
    PartitionDev p;
    p.rank = r;
    p.deg = (int32_t*)e.dalloc(sizeof(int32_t) * N);
    p.off = (int64_t*)e.dalloc(sizeof(int64_t) * (N + 1));
    launch_pdl(k_part_deg, dim3(grid_for(N, 8, kNumSMs * 16)), dim3(256), 0, s, N, e.g.offsets, e.g.nbrs, c.owner, r, p.deg);
    device_scan(s, sc, LoadI32{p.deg}, StoreI64{p.off}, nullptr, N, N, total, p.off);
    OB_CUDA(cudaMemcpyAsync(&p.E, total, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    OB_CUDA(cudaStreamSynchronize(s));
    p.src = (int32_t*)e.dalloc(sizeof(int32_t) * std::max<int64_t>(p.E, 1));
    launch_pdl(k_part_fill, dim3(grid_for(N, 8, kNumSMs * 16)), dim3(256), 0, s, N, e.g.offsets, e.g.nbrs, c.owner, r, p.off, p.src);
    c.parts.push_back(p);
  }
  OB_CUDA(cudaStreamSynchronize(s));
}

__global__ void k_flag_owned(int64_t N, const int32_t* owner, int rank, int32_t* flag) {
  pdl_wait();
  OB_GRID_STRIDE(v, N) flag[v] = owner[v] == rank;
}
__global__ void k_pos_owned(int64_t N, const int32_t* owner, int rank, const int64_t* excl, int32_t* pos) {
  pdl_wait();
  OB_GRID_STRIDE(v, N) pos[v] = owner[v] == rank ? (int32_t)excl[v] : -1;
}
__global__ void k_gather_owned(int64_t N, int64_t ld, const int32_t* __restrict__ pos, const float* __restrict__ full,
                               float* local) {
  pdl_wait();
  const int64_t n = N * ld;
  OB_GRID_STRIDE(i, n) {
    const int64_t v = i / ld;
    const int32_t p = pos[v];
    if (p >= 0) local[(int64_t)p * ld + (i - v * ld)] = full[i];
  }
}

// owned-row map of this rank: pos[v] = local row of v, -1 when another rank owns it
void owned_positions(Engine& e) {
  CgpState& c = e.cgp;
  cudaStream_t s = e.stream;
  const int64_t N = e.g.N;
  int32_t* flag = (int32_t*)e.dalloc(sizeof(int32_t) * N);
  int64_t* excl = (int64_t*)e.dalloc(sizeof(int64_t) * (N + 1));
  ScanScratch sc;
  sc.cap = ScanScratch::bytes_for(N, 1);
  sc.pool = (char*)e.dalloc(sc.cap);
  OB_CUDA(cudaMemsetAsync(sc.pool, 0, sc.cap, s));
  launch_pdl(k_flag_owned, dim3(grid_for(N, 256)), dim3(256), 0, s, N, c.owner, c.my_rank, flag);
  device_scan(s, sc, LoadI32{flag}, StoreI64{excl}, nullptr, N, N, nullptr, excl);
  e.g.pos = (int32_t*)e.dalloc(sizeof(int32_t) * N);
  launch_pdl(k_pos_owned, dim3(grid_for(N, 256)), dim3(256), 0, s, N, c.owner, c.my_rank, excl, e.g.pos);
  OB_CUDA(cudaMemcpyAsync(&e.g.N_local, excl + N, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  OB_CUDA(cudaStreamSynchronize(s));
  e.dfree(flag);
  e.dfree(excl);
  e.dfree(sc.pool);
}

// replace a full (N x ld) row table by this rank's owned rows (g.pos order)
void localize_table(Engine& e, float*& table, int64_t ld) {
  if (!table) return;
  cudaStream_t s = e.stream;
  const int64_t N = e.g.N;
  float* local = (float*)e.dalloc(sizeof(float) * std::max<int64_t>(e.g.N_local, 1) * ld);
  launch_pdl(k_gather_owned, dim3(grid_for(N * ld, 256)), dim3(256), 0, s, N, ld, e.g.pos, table, local);
  OB_CUDA(cudaStreamSynchronize(s));
  e.dfree(table);
  table = local;
}

// NCCL-mode CGP: every rank keeps only the feature and stored-embedding rows of
// the nodes it owns (graphstore.py:233-262); aggregation sources are always
// owned (source-split edges) and destinations are updated by their owner, so
// no request ever needs another rank's rows.  The full in-CSR is dropped too
// (the rank's source-split CSR replaces it).
void cgp_localize_storage(Engine& e) {
  if (e.localized || !e.cgp.nccl || e.cfg.strategy != OB_STRATEGY_SRPE_CGP) return;
  cudaStream_t s = e.stream;
  const int64_t N = e.g.N;
  if (!e.g.pos) owned_positions(e);
  (void)s;
  (void)N;
  if (!e.g.generated) {
    localize_table(e, e.g.feats, e.g.F_ld);
    for (size_t l = 0; l < e.pe.size(); ++l) localize_table(e, e.pe[l], ld4(e.pe_dim[l]));
    e.dfree(e.g.offsets);
    e.dfree(e.g.nbrs);
    e.g.offsets = nullptr;
    e.g.nbrs = nullptr;
  }
  e.localized = true;
}

// request slice of partition r: edges whose source it owns (queries: round robin)
__global__ void k_filter_slice(const ReqParams* rp, int64_t N, int P, int r, const int32_t* __restrict__ owner,
                               const ReqCounters* rc, int64_t* out, int64_t* count) {
  pdl_wait();
  const CtaWords st = cta_ldv(&rc->err, &rp->m);
  if (st.v[0] & (kErrRange | kErrNoQuery)) return;
  const int64_t* __restrict__ edges = rp->edges;
  const int64_t m = st.v[1];
  OB_GRID_STRIDE(e, m) {
    const int64_t s = edges[2 * e];
    const int o = s >= N ? (int)((s - N) % P) : owner[s];
    const bool keep = o == r;
    const unsigned act = __activemask();
    const unsigned b = __ballot_sync(act, keep);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(act) - 1;
    int64_t base = 0;
    if (lane == leader && b) base = (int64_t)atomicAdd((unsigned long long*)count, (unsigned long long)__popc(b));
    base = __shfl_sync(act, base, leader);
    if (keep) {
      const int64_t at = base + __popc(b & ((1u << lane) - 1u));
      out[2 * at] = s;
      out[2 * at + 1] = edges[2 * e + 1];
    }
  }
}

// destination rows h_v for a layer (dst-indexed); non-owned rows read a zero row
__global__ void k_dst_rows(const int32_t* __restrict__ dst_ids, const int64_t* D_dev, int64_t N, int layer, int k,
                           const int32_t* pos, const float* feats, const float* qpad, int64_t F_ld,
                           const float* prev, int64_t in_ld,
                           const int64_t* T_dev, const int32_t* owner, int P, int rank, const float* zero,
                           const float** hvp) {
  pdl_wait();
  const CtaWords st = cta_ldv(D_dev, T_dev);
  const int64_t D = st.v[0], T = st.v[1];
  OB_GRID_STRIDE(i, D) {
    const int64_t g = dst_ids[i];
    bool mine = true;
    if (owner) mine = (g >= N ? (int)((g - N) % P) : owner[g]) == rank;
    const float* r;
    if (!mine) r = zero;
    else if (layer == 1) r = g < N ? feats + (pos ? (int64_t)pos[g] : g) * F_ld : qpad + (g - N) * F_ld;
    else if (layer == k) r = prev + (T + (g - N)) * in_ld;  // last block: queries in the mid table
    else r = prev + i * in_ld;                              // mid blocks share one destination list
    hvp[i] = r;
  }
}

__global__ void k_rowdot_ptr(const int64_t* M_dev, const float* const* rows, int w, const float* __restrict__ av,
                             float* out) {
  pdl_wait();
  const int64_t M = cta_ld(M_dev);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < M; r += nw) {
    const float* row = rows[r];
    float s = 0.f;
    for (int c = lane; c < w; c += 32) s = fmaf(row[c], av[c], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = s;
  }
}

// softmax exchange: pull the max-logit column out, then rescale (den, num) to the
// global max so the triples can be summed (cgpexec.py:225-239)
__global__ void k_sm_extract(const int64_t* D_dev, const float* lp, int64_t ldp, float* lmax) {
  pdl_wait();
  const int64_t D = cta_ld(D_dev);
  OB_GRID_STRIDE(i, D) lmax[i] = lp[i * ldp + 1] > 0.f ? lp[i * ldp] : -INFINITY;
}
__global__ void k_sm_rescale(const int64_t* D_dev, float* lp, int64_t ldp, int w, const float* gmax) {
  pdl_wait();
  const int64_t D = cta_ld(D_dev);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < D; i += nw) {
    float* o = lp + i * ldp;
    const float sc = o[1] > 0.f ? __expf(o[0] - gmax[i]) : 0.f;
    __syncwarp();
    for (int c = lane; c < w; c += 32) o[2 + c] *= sc;
    __syncwarp();
    if (lane == 0) {
      o[1] *= sc;
      o[0] = 0.f;
    }
  }
}
__global__ void k_sm_restore(const int64_t* D_dev, float* lp, int64_t ldp, const float* gmax) {
  pdl_wait();
  const int64_t D = cta_ld(D_dev);
  OB_GRID_STRIDE(i, D) lp[i * ldp] = gmax[i];
}

// final rows: zero the queries this rank does not own before the reduce to rank 0
__global__ void k_zero_foreign_queries(float* rows, int B, int H, int P, int rank) {
  pdl_wait();
  const int64_t n = (int64_t)B * H;
  OB_GRID_STRIDE(i, n) if ((int)((i / H) % P) != rank) rows[i] = 0.f;
}

void carve_cgp(Engine& e, RequestWs& w, Arena& a) {
  CgpState& c = e.cgp;
  const int np = (int)c.parts.size();
  const BlockDev& mid = w.blocks[0];
  const BlockDev& last = w.blocks[1];
  c.ws.assign(np, CgpPartWs{});
  const int64_t RB_max = std::min<int64_t>(e.g.N, 2 * w.m) + w.B;
  for (int p = 0; p < np; ++p) {
    CgpPartWs& pw = c.ws[p];
    pw.ledges = a.take<int64_t>(2 * w.m + 2);
    pw.rq.cnt = a.take<int32_t>(RB_max + 1);
    pw.rq.fill = a.take<int32_t>(RB_max + 1);
    pw.rq.ptr = a.take<int64_t>(RB_max + 1);
    pw.rq.src = a.take<int32_t>(w.m + 1);
    pw.rq.keys = a.take<uint64_t>(w.m + 1);
    pw.rq.keys2 = a.take<uint64_t>(w.m + 1);
    pw.rq.rx_cnt = a.take<int32_t>(256 * rx_tiles(w.m));
    pw.rq.rx_off = a.take<int64_t>(256 * rx_tiles(w.m) + 257);  // + per-digit totals
    pw.rq.ctr = a.take<int64_t>(4);
    for (int bi = 0; bi < 2; ++bi) {
      BlockDev b = bi == 0 ? mid : last;
      b.has_self = false;
      b.cnt = a.take<BlockCounters>(1);
      b.dst_ptr = a.take<int64_t>(b.D_max + 1);
      b.item_ptr = a.take<int64_t>(b.D_max + 1);
      b.item_dst = a.take<int32_t>(b.items_max);
      b.group_dst = a.take<int32_t>(b.items_max / kItemGroup + b.D_max + 1);
      b.group_ptr = a.take<int64_t>(b.D_max + 1);
      b.edge_src = a.take<int32_t>(b.E_max);
      b.src_ids = a.take<int32_t>(b.S_max);
      b.self_src = nullptr;
      b.dst_ids = a.take<int32_t>(b.D_max);
      pw.blocks[bi] = b;
    }
  }
  int maxw = 4;
  bool mom = false;
  for (auto& L : e.layers) {
    maxw = std::max(maxw, cgp_partial_width(L));
    mom |= L.spec.kind == OB_KIND_MOMENTS;
  }
  c.D_max = mid.D_max;
  c.ldp = ld4(maxw);
  const int64_t part_elems = c.D_max * c.ldp * (mom ? 2 : 1);
  c.lp = a.take<float>(np * part_elems);
  c.lcnt = a.take<float>(np * c.D_max);
  c.hvp = a.take<const float*>(c.D_max);
  c.zero_row = a.take<float>(ld4(std::max(e.g.F, 4)) + 512);
  c.sdst = a.take<float>(c.D_max);
  c.lmax = a.take<float>(c.D_max);
  c.mean = mom ? a.take<double>(c.D_max * ld4(maxw)) : nullptr;
  c.fin = a.take<float>((int64_t)w.B * e.layers.back().spec.out_dim + 4);
  // exchange region: the largest single-step payload (partials + counts, s_dst,
  // moments means, final query rows)
  const int64_t esz = mom ? 8 : 4;
  const size_t parts_b = (((size_t)c.D_max * c.ldp * esz + 255) & ~(size_t)255) + (size_t)c.D_max * 4;
  const size_t mean_b = mom ? (size_t)c.D_max * ld4(maxw) * 8 : 0;
  const size_t fin_b = (size_t)w.B * e.layers.back().spec.out_dim * 4;
  const size_t is_b = e.cfg.policy == OB_POLICY_IS ? (size_t)std::min<int64_t>(e.g.N, 2 * w.m) * 8 : 0;
  c.x_need_region = (std::max(std::max(std::max(parts_b, mean_b), std::max(fin_b, (size_t)c.D_max * 4)), is_b) + 4095) &
                    ~(size_t)4095;
}

#ifdef OB_WITH_NCCL
#define OB_NCCL(x)                                                                               \
  do {                                                                                           \
    ncclResult_t _r = (x);                                                                       \
    if (_r != ncclSuccess) throw Error(OB_ECOMM, std::string(#x) + ": " + ncclGetErrorString(_r)); \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// NVLink exchange over CUDA-IPC-mapped peer buffers (NCCL mode)
//
// Buffer of rank r: ready[p] (int64, written by rank p when its step-k data is
// in p's region), done[p] (written by rank p when it has read r's step-k data),
// then one region per exchange step of a request.  One step:
//   x_begin    wait until every peer finished reading the previous step
//   producer   kernels write this rank's region (local stores)
//   x_publish  fence; bump the device step counter k; ready[me] = k at every peer
//   x_wait     spin until ready[p] >= k for every peer (acquire, system scope)
//   consumer   kernels read peers' regions with ld.global.cg over NVLink
//   x_done     done[me] = k at every peer
// The step counter lives on the device, so a replayed CUDA graph keeps
// counting; spins give up after OB_CGP_TIMEOUT_MS (default 2 s of %globaltimer
// wall time) and raise OB_ECOMM instead of hanging.  The failure is sticky: the
// lane's failure word skips every later step and the timed-out rank poisons its
// peers' flags, so no rank carries on with a skewed step counter.
// ---------------------------------------------------------------------------
struct XCtx {
  char* peer[kMaxParts];
  int P, rank;
  int64_t* ep;
  int64_t* err;     // the request's error word (kErrComm on a flag timeout)
  int64_t* sticky;  // the lane's persistent failure word: once set, every later step is skipped
  int64_t timeout_ns;
};
constexpr size_t kXFlags = 256;   // ready[8] @0, done[8] @64, poison @128
constexpr size_t kXPoison = 128;  // set by a peer that timed out: this exchange is unusable

__device__ __forceinline__ int64_t ld_acq_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// the exchange failed earlier (this lane timed out, or a peer poisoned our flags)
__device__ __forceinline__ bool x_failed(const XCtx& x) {
  return *reinterpret_cast<volatile int64_t*>(x.sticky) != 0 ||
         ld_acq_sys(reinterpret_cast<const int64_t*>(x.peer[x.rank] + kXPoison)) != 0;
}
// Sticky failure: flag this request, remember it for the lane and poison every
// peer's flags so their spins end with kErrComm too instead of reading regions
// this rank may overwrite (no rank proceeds on a skewed step counter silently)
__device__ __noinline__ void x_fail(const XCtx& x) {
  atomicOr((unsigned long long*)x.err, (unsigned long long)kErrComm);
  atomicExch((unsigned long long*)x.sticky, 1ull);
  for (int q = 0; q < x.P; ++q)
    if (q != x.rank) st_rel_sys(reinterpret_cast<int64_t*>(x.peer[q] + kXPoison), 1);
}
__device__ __forceinline__ void spin_geq(const XCtx& x, const int64_t* f, int64_t k) {
  const uint64_t t0 = globaltimer_ns();
  while (ld_acq_sys(f) < k) {
    if (x_failed(x) || globaltimer_ns() - t0 > (uint64_t)x.timeout_ns) {  // a peer is gone
      x_fail(x);
      return;
    }
    __nanosleep(256);
  }
}

__global__ void k_x_begin(XCtx x) {
  pdl_wait();  // peers done with the previous step
  const int q = threadIdx.x;
  if (q >= x.P || q == x.rank) return;
  if (x_failed(x)) {
    atomicOr((unsigned long long*)x.err, (unsigned long long)kErrComm);
    return;
  }
  const int64_t k = ld_state(x.ep);
  if (k > 0) spin_geq(x, reinterpret_cast<const int64_t*>(x.peer[x.rank] + 64) + q, k);
}
__global__ void k_x_publish(XCtx x) {
  pdl_wait();
  __threadfence_system();
  const int64_t k = ld_state(x.ep) + 1;
  __syncthreads();
  if (threadIdx.x == 0) *x.ep = k;
  const int q = threadIdx.x;
  if (q < x.P && q != x.rank) st_rel_sys(reinterpret_cast<int64_t*>(x.peer[q]) + x.rank, k);
}
__global__ void k_x_wait(XCtx x) {
  pdl_wait();
  const int p = threadIdx.x;
  if (p >= x.P || p == x.rank) return;
  if (x_failed(x)) {
    atomicOr((unsigned long long*)x.err, (unsigned long long)kErrComm);
    return;
  }
  spin_geq(x, reinterpret_cast<const int64_t*>(x.peer[x.rank]) + p, ld_state(x.ep));
}
__global__ void k_x_done(XCtx x) {
  pdl_wait();
  const int q = threadIdx.x;
  if (q < x.P && q != x.rank)
    st_rel_sys(reinterpret_cast<int64_t*>(x.peer[q] + 64) + x.rank, ld_state(x.ep));
}

// rows[i] of destination i from its owner's copy (s_dst, moments means, final rows)
__global__ void k_x_gather_rows(XCtx x, size_t off, const int32_t* dst_ids, const int64_t* D_dev, int64_t D_fixed,
                                int64_t N, const int32_t* owner, int esize, int64_t width_el, float* out) {
  pdl_wait();
  const int64_t D = D_dev ? cta_ld(D_dev) : D_fixed;
  const int64_t words = width_el * esize / 4;  // 4-byte words per row
  const int64_t n = D * words;
  OB_GRID_STRIDE(t, n) {
    const int64_t i = t / words;
    const int64_t g = dst_ids ? (int64_t)dst_ids[i] : N + i;
    const int o = g >= N ? (int)((g - N) % x.P) : owner[g];
    const float* src = reinterpret_cast<const float*>(x.peer[o] + kXFlags + off);
    out[t] = __ldcg(src + t);
  }
}

static XCtx xctx(Engine& e) {
  CgpState& c = e.cgp;
  XCtx x{};
  for (int p = 0; p < c.P; ++p) x.peer[p] = c.xpeer[p];
  x.P = c.P;
  x.rank = c.my_rank;
  x.ep = c.xep;
  x.err = &e.ws.rc->err;
  x.sticky = c.xerr;
  x.timeout_ns = c.x_timeout_ns;
  return x;
}
static void x_launch(cudaStream_t s, void (*kern)(XCtx), const XCtx& x) {
  launch_pdl(kern, dim3(1), dim3(32), 0, s, x);
}

// offset (from the region base past the flags) of step j's region
static size_t xoff(const CgpState& c, int j) { return (size_t)j * c.xregion; }
static char* xregion_ptr(const CgpState& c, int j) { return c.xbuf + kXFlags + xoff(c, j); }

static void allreduce(Engine& e, void* buf, size_t count, bool is_double, bool max) {
#ifdef OB_WITH_NCCL
  CgpState& c = e.cgp;
  cudaEvent_t p0 = prof_begin(e.stream);
  OB_NCCL(ncclAllReduce(buf, buf, count, is_double ? ncclDouble : ncclFloat, max ? ncclMax : ncclSum,
                        (ncclComm_t)c.comm, e.stream));
  prof_end(e.stream, p0, kProfComm, nullptr, 0, 0, 0, 0, 0);
  c.collective_bytes += (int64_t)(2.0 * (c.P - 1) / c.P * count * (is_double ? 8 : 4));
#else
  (void)e, (void)buf, (void)count, (void)is_double, (void)max;
  throw Error(OB_ECOMM, "built without NCCL");
#endif
}

void serve_cgp(Engine& e, float* d_out) {
  CgpState& c = e.cgp;
  RequestWs& w = e.ws;
  cudaStream_t s = e.stream;
  const int k = (int)e.layers.size();
  const int np = (int)c.parts.size();
  const int64_t N = e.g.N;
  c.collective_bytes = 0;
  const bool p2p = c.nccl && c.p2p;
  const XCtx x = p2p ? xctx(e) : XCtx{};
  int xj = 0;  // exchange step within this request (selects the region)
  auto x_begin = [&] { x_launch(s, k_x_begin, x); };
  auto x_exchange = [&] {  // publish this rank's region, wait for everyone's
    cudaEvent_t pc = prof_begin(s);
    x_launch(s, k_x_publish, x);
    x_launch(s, k_x_wait, x);
    prof_end(s, pc, kProfComm, nullptr, 0, 0, 0, 0, 0);
  };
  auto x_done = [&] {
    x_launch(s, k_x_done, x);
    ++xj;
  };
  // identical plan on every rank from the whole request (runtime.py:151-192)
  cudaEvent_t p0 = prof_begin(s);
  stage_request_prep(e, w, true);
  static const bool serial_env = [] {  // OB_CGP_SERIAL=1: slice sorts on the main stream (A/B)
    const char* v = std::getenv("OB_CGP_SERIAL");
    return v && v[0] && v[0] != '0';
  }();
  // With request lanes on more than two ranks the two-stream request graphs stall each
  // other across ranks (measured cfg4 P = 4, 4 lanes: 0.72 M vs 3.57 M queries/s serial);
  // at P = 2 the overlap still pays with lanes (4.51 vs 4.17 M), and always without them
  const bool serial = serial_env || (e.nlanes > 1 && c.P > 2);
  cudaStream_t side = serial ? s : e.side;
  // the slices' request-index sorts and query blocks (side stream) need only the
  // request and the candidate set: they run beside the selection (main stream);
  // the mid blocks follow the targets (as in the centralized pipeline)
  OB_CUDA(cudaEventRecord(e.fork_ev, s));
  OB_CUDA(cudaStreamWaitEvent(side, e.fork_ev, 0));
  {
    e.stream = side;
    try {
      cudaEvent_t pc = prof_begin(side);
      for (int p = 0; p < np; ++p) {
        CgpPartWs& pw = c.ws[p];
        const PartitionDev& part = c.parts[p];
        OB_CUDA(cudaMemsetAsync(pw.rq.ctr, 0, sizeof(int64_t) * 4, side));
        OB_CUDA(cudaMemsetAsync(pw.blocks[0].cnt, 0, sizeof(BlockCounters), side));
        OB_CUDA(cudaMemsetAsync(pw.blocks[1].cnt, 0, sizeof(BlockCounters), side));
        if (w.m > 0) {
          launch_pdl(k_filter_slice, dim3(grid_for(w.m, 256)), dim3(256), 0, side, w.rp, N, c.P, part.rank, c.owner, w.rc, pw.ledges,
                                                                  pw.rq.ctr);
        }
        build_rq_csr(e, w, pw.ledges, w.m, pw.rq.ctr, pw.rq, /*counts_ready=*/false);
        const SpanSrc src{part.off, part.src, part.deg, pw.rq.ptr, pw.rq.src};
        write_query_dst(e, w, pw.blocks[1]);
        assemble(e, w, pw.blocks[1], src, w.bs[1]);
      }
      prof_end(side, pc, kProfBuild, nullptr, 0, 0, 0, 0, 0);
      OB_CUDA(cudaEventRecord(e.csr_ev, side));
    } catch (...) {
      e.stream = s;
      throw;
    }
    e.stream = s;
  }
  stage_request_post(e, w, true);
  const int64_t r_max = std::min<int64_t>(N, 2 * w.m);
  if (e.cfg.policy == OB_POLICY_IS && r_max > 0) {
    // importance numerators per partition over its source-split CSR
    // (policy.py:98-107), summed in rank order on every rank (runtime.py:168-175)
    IsParts ip{};
    ip.P = c.P;
    if (p2p) {
      x_begin();
      launch_is_gather(e, w, e.is_tab[0], reinterpret_cast<double*>(xregion_ptr(c, xj)));
      x_exchange();
      for (int q = 0; q < c.P; ++q)
        ip.part[q] = reinterpret_cast<const double*>(c.xpeer[q] + kXFlags + xoff(c, xj));
      launch_score_is(e, w, ip);
      x_done();
    } else {
      for (int p = 0; p < np; ++p)
        launch_is_gather(e, w, e.is_tab[p], w.is_part + (int64_t)c.parts[p].rank * r_max);
#ifdef OB_WITH_NCCL
      if (c.nccl) {
        OB_NCCL(ncclAllGather(w.is_part + (int64_t)c.my_rank * r_max, w.is_part, (size_t)r_max, ncclDouble,
                              (ncclComm_t)c.comm, s));
        c.collective_bytes += r_max * 8 * (c.P - 1);
      }
#endif
      for (int q = 0; q < c.P; ++q) ip.part[q] = w.is_part + (int64_t)q * r_max;
      launch_score_is(e, w, ip);
    }
  }
  stage_select(e, w);
  prof_end(s, p0, kProfSelect, nullptr, 0, 0, 0, 0, 0);
  OB_CUDA(cudaStreamWaitEvent(s, e.csr_ev, 0));
  p0 = prof_begin(s);
  for (int p = 0; p < np; ++p) {
    CgpPartWs& pw = c.ws[p];
    const PartitionDev& part = c.parts[p];
    const SpanSrc src{part.off, part.src, part.deg, pw.rq.ptr, pw.rq.src};
    write_mid_dst(e, w, pw.blocks[0]);
    assemble(e, w, pw.blocks[0], src, w.bs[0]);
  }
  prof_end(s, p0, kProfBuild, nullptr, 0, 0, 0, 0, 0);
  record_mark(e.ev[1], s);
  stage_qpad(e, w);
  OB_CUDA(cudaMemsetAsync(c.zero_row, 0, sizeof(float) * (ld4(std::max(e.g.F, 4)) + 512), s));
  const int64_t part_stride_f = c.D_max * c.ldp;  // floats between partitions (x2 for float64 partials)
  OwnerFilter own{};
  if (p2p) {
    own.owner = c.owner;
    own.N = N;
    own.P = c.P;
    own.rank = c.my_rank;
  }
  for (int l = 1; l <= k; ++l) {
    const LayerDev& L = e.layers[l - 1];
    const int bi = l < k ? 0 : 1;
    const BlockDev& b0 = c.ws[0].blocks[bi];
    const int64_t* D_dev = &b0.cnt->D;
    const int64_t D_max = b0.D_max;
    const bool mom = L.spec.kind == OB_KIND_MOMENTS;
    const int64_t pstride = mom ? 2 * part_stride_f : part_stride_f;
    BindCtx bc = bind_ctx(e, w, l);
    own.dst_ids = b0.dst_ids;
    // destination rows h_v (owned ones; zero row elsewhere under NCCL)
    launch_pdl(k_dst_rows, dim3(grid_for(D_max, 256)), dim3(256), 0, s, b0.dst_ids, D_dev, N, l, k, e.g.pos, e.g.feats, w.qpad, e.g.F_ld,
                                                    l > 1 ? w.outs[l - 1] : nullptr, ld4(L.spec.in_dim), &w.rc->T,
                                                    c.nccl ? c.owner : nullptr, c.P, c.my_rank, c.zero_row, c.hvp);
    if (L.spec.kind == OB_KIND_GAT) {  // s_dst = h_v . (W a_dst), computed by the owner
      if (p2p) {
        x_begin();
        float* reg = reinterpret_cast<float*>(xregion_ptr(c, xj));
        launch_pdl(k_rowdot_ptr, dim3(grid_for(D_max, 8)), dim3(256), 0, s, D_dev, c.hvp, L.spec.in_dim, L.wa_dst, reg);
        x_exchange();
        launch_pdl(k_x_gather_rows, dim3(grid_for(D_max, 256)), dim3(256), 0, s, x, xoff(c, xj), b0.dst_ids, D_dev, 0, N, c.owner, 4, 1,
                                                             c.sdst);
        x_done();
      } else {
        launch_pdl(k_rowdot_ptr, dim3(grid_for(D_max, 8)), dim3(256), 0, s, D_dev, c.hvp, L.spec.in_dim, L.wa_dst, c.sdst);
        if (c.nccl) allreduce(e, c.sdst, D_max, false, false);
      }
    }
    const int phases = mom ? 2 : 1;
    for (int ph = 1; ph <= phases; ++ph) {
      // this rank's raw partials: into its exchange region (p2p) or the arena
      float* lp0 = c.lp;
      float* cnt0 = c.lcnt;
      if (p2p) {
        x_begin();
        char* reg = xregion_ptr(c, xj);
        lp0 = reinterpret_cast<float*>(reg);
        cnt0 = reinterpret_cast<float*>(reg + (((size_t)c.D_max * c.ldp * (mom ? 8 : 4) + 255) & ~(size_t)255));
      }
      // layer 1 from the stored tables: transformed rows of the stored features, and the
      // partitions' CSR-part sums (sum kinds)
      const bool yt = l == 1 && e.ytab_ready && !e.ytab.empty() && e.ytab[0] && w.yrow;
      if (yt) {
        bc.ytab = e.ytab[0];
        bc.y_ld = ld4(L.spec.out_dim);
        bc.yrow = w.yrow;
        bc.ydyn = w.z;
        bc.dyn_src = w.dyn_src;
        bc.ndyn = w.ndyn;
      }
      const bool sa = l == 1 && (int)e.cgp_sagg1.size() == np;
      for (int p = 0; p < np; ++p) {
        const BlockDev& b = c.ws[p].blocks[bi];
        if (yt) OB_CUDA(cudaMemsetAsync(w.ndyn, 0, sizeof(int64_t), s));
        launch_resolve(s, bc, b.cnt, b.S_max, b.src_ids, w.rowp, w.gscale);
        LayerRun r{};
        if (yt) {
          r.yrow = w.yrow;
          r.dyn_src = w.dyn_src;
          r.ndyn = w.ndyn;
          r.dyn_max = b.S_max;
        }
        if (sa) {
          r.stat = e.cgp_sagg1[p];
          r.stat_ld = ld4(L.transform_first ? L.spec.out_dim : L.spec.in_dim);
          r.dst_ids = b.dst_ids;
          r.indeg = c.parts[p].deg;
          r.N = N;
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
        r.self = nullptr;
        r.x = RowSrc{w.rowp, nullptr, 0};
        r.gscale = w.gscale;
        r.group_ptr = b.group_ptr;
        LayerScratch sc{w.partial, w.partial2, w.agg, w.mean, w.z, w.s_src, w.s_dst};
        cgp_local_partial(s, L, r, sc, c.sdst, lp0 + p * pstride, c.ldp, cnt0 + p * c.D_max, ph, c.mean);
      }
      PartPtrs pp{};
      int Pm = np;
      const size_t cnt_off = (((size_t)c.D_max * c.ldp * (mom ? 8 : 4) + 255) & ~(size_t)255);
      if (p2p) {
        x_exchange();
        Pm = c.P;
        for (int q = 0; q < c.P; ++q) {  // every rank's partials, read in place over NVLink
          const char* reg = c.xpeer[q] + kXFlags + xoff(c, xj);
          pp.lp[q] = reinterpret_cast<const float*>(reg);
          pp.cnt[q] = reinterpret_cast<const float*>(reg + cnt_off);
        }
      } else {
        if (c.nccl) {
          const int64_t pw = cgp_partial_width(L);
          if (L.spec.kind == OB_KIND_GAT) {
            launch_pdl(k_sm_extract, dim3(grid_for(D_max, 256)), dim3(256), 0, s, D_dev, c.lp, c.ldp, c.lmax);
            allreduce(e, c.lmax, D_max, false, true);
            launch_pdl(k_sm_rescale, dim3(grid_for(D_max, 8)), dim3(256), 0, s, D_dev, c.lp, c.ldp, (int)pw - 2, c.lmax);
            allreduce(e, c.lp, D_max * c.ldp, false, false);
            launch_pdl(k_sm_restore, dim3(grid_for(D_max, 256)), dim3(256), 0, s, D_dev, c.lp, c.ldp, c.lmax);
          } else if (L.spec.kind == OB_KIND_SAGE_MAX) {
            allreduce(e, c.lp, D_max * c.ldp, false, true);  // empty partials hold -inf
          } else {
            allreduce(e, c.lp, D_max * c.ldp, mom, false);
          }
          allreduce(e, c.lcnt, D_max, false, false);
          Pm = 1;
        }
        for (int q = 0; q < Pm; ++q) {
          pp.lp[q] = c.lp + q * pstride;
          pp.cnt[q] = c.lcnt + q * c.D_max;
        }
      }
      const bool last = l == k;
      float* out = last ? (c.nccl ? c.fin : d_out) : w.outs[l];
      const int64_t ldo = last ? L.spec.out_dim : ld4(L.spec.out_dim);
      cgp_merge(s, L, Pm, pp, c.ldp, own, D_dev, D_max, w.agg, out, ldo, ph, c.mean);
      if (p2p) x_done();
      if (mom && ph == 1 && p2p) {  // owners' means to every rank (phase 2 needs them for all destinations)
        x_begin();
        const int64_t mw = L.spec.in_dim;  // mean rows are in_dim float64 wide (k_merge_moments)
        OB_CUDA(cudaMemcpyAsync(xregion_ptr(c, xj), c.mean, sizeof(double) * D_max * mw, cudaMemcpyDeviceToDevice, s));
        x_exchange();
        launch_pdl(k_x_gather_rows, dim3(grid_for(D_max * mw * 2, 256)), dim3(256), 0, s, x, xoff(c, xj), b0.dst_ids, D_dev, 0, N, c.owner,
                                                                      8, mw, reinterpret_cast<float*>(c.mean));
        x_done();
      }
      if (ph == phases) cgp_update(s, L, D_dev, D_max, c.hvp, w.agg, out, ldo);
    }
  }
#ifdef OB_WITH_NCCL
  if (p2p) {  // rank 0 collects every query row from its owner
    const int H = e.layers.back().spec.out_dim;
    x_begin();
    OB_CUDA(cudaMemcpyAsync(xregion_ptr(c, xj), c.fin, sizeof(float) * w.B * H, cudaMemcpyDeviceToDevice, s));
    x_exchange();
    if (c.my_rank == 0) {
      launch_pdl(k_x_gather_rows, dim3(grid_for((int64_t)w.B * H, 256)), dim3(256), 0, s, x, xoff(c, xj), nullptr, nullptr, w.B, N,
                                                                      c.owner, 4, H, d_out);
    }
    x_done();
  } else if (c.nccl) {
    const int H = e.layers.back().spec.out_dim;
    launch_pdl(k_zero_foreign_queries, dim3(grid_for((int64_t)w.B * H, 256)), dim3(256), 0, s, c.fin, w.B, H, c.P, c.my_rank);
    OB_NCCL(ncclReduce(c.fin, d_out, (size_t)w.B * H, ncclFloat, ncclSum, 0, (ncclComm_t)c.comm, s));
    c.collective_bytes += (int64_t)w.B * H * 4;
  }
#endif
}

// NVLink traffic of one request from its actual sizes (the block counters read
// back after the request), summed over the P ranks, next to the all-gather-of-
// source-rows alternative sum_l (P-1) S_l row_bytes_l.  The
// exchange reads only real rows: an owner reads P-1 peers' partial rows of each
// destination it owns (+ a 4-byte count); GAT destination scores and moments
// means are read by every rank from the owners; rank 0 reads the query rows.
void cgp_traffic(const Engine& e, const ReqCounters& rc, const std::vector<BlockCounters>& hc, int64_t* nvlink,
                 int64_t* allgather) {
  const CgpState& c = e.cgp;
  const int k = (int)e.layers.size();
  const double P = c.P, q = c.P - 1;
  *nvlink = 0;
  *allgather = 0;
  if (c.P < 2 || hc.size() < 2) return;
  const int np = (int)hc.size() / 2;  // (mid, last) per local partition
  auto S_of = [&](int bi) {         // union of the partitions' sources (NCCL: P x this rank's)
    double S = 0;
    for (int p = 0; p < np; ++p) S += (double)hc[2 * p + bi].S;
    return np == c.P ? S : S * P / np;
  };
  double nv = 0, ag = 0;
  if (e.cfg.policy == OB_POLICY_IS) nv += P * q * (double)rc.R * 8;  // every rank reads every peer's numerators
  for (int l = 1; l <= k; ++l) {
    const LayerDev& L = e.layers[l - 1];
    const int bi = l < k ? 0 : 1;
    const double D = (double)hc[bi].D;
    const bool mom = L.spec.kind == OB_KIND_MOMENTS;
    if (L.spec.kind == OB_KIND_GAT) nv += q * D * 4;                       // s_dst from the owners
    nv += (mom ? 2 : 1) * q * D * ((double)cgp_partial_width(L) * (mom ? 8 : 4) + 4);  // partials to owners
    if (mom) nv += q * D * L.spec.in_dim * 8.0;                            // owners' means to every rank
    ag += q * S_of(bi) * L.spec.in_dim * 4.0;
  }
  nv += q / P * (double)hc[1].D * e.layers.back().spec.out_dim * 4;       // query rows to rank 0
  *nvlink = (int64_t)nv;
  *allgather = (int64_t)ag;
}

#ifdef OB_WITH_NCCL
static void comm_barrier(Engine& e) {
  CgpState& c = e.cgp;
  int* d = (int*)e.dalloc(sizeof(int));
  OB_CUDA(cudaMemsetAsync(d, 0, sizeof(int), e.stream));
  OB_NCCL(ncclAllReduce(d, d, 1, ncclInt, ncclSum, (ncclComm_t)c.comm, e.stream));
  OB_CUDA(cudaStreamSynchronize(e.stream));
  e.dfree(d);
}
#endif

static void close_exchange(Engine& e) {
  CgpState& c = e.cgp;
  for (int p = 0; p < c.P && p < kMaxParts; ++p) {
    if (c.xpeer[p] && c.xpeer[p] != c.xbuf) cudaIpcCloseMemHandle(c.xpeer[p]);
    c.xpeer[p] = nullptr;
  }
  if (c.xbuf) cudaFree(c.xbuf);
  c.xbuf = nullptr;
  c.xregion = 0;
  c.xsteps = 0;
}

void cgp_release_exchange(Engine& e) {
#ifdef OB_WITH_NCCL
  if (e.cgp.comm && e.cgp.xbuf) {
    try {
      cudaStreamSynchronize(e.stream);
      comm_barrier(e);  // no peer still reads this lane's buffer
      close_exchange(e);
      comm_barrier(e);
    } catch (...) {
      close_exchange(e);
    }
  }
#else
  (void)e;
#endif
}

void cgp_ensure_exchange(Engine& e) {
#ifdef OB_WITH_NCCL
  CgpState& c = e.cgp;
  if (!c.nccl || !c.p2p) return;
  const int steps = 4 * (int)e.layers.size() + 3;  // + the IS numerator exchange
  if (c.xbuf && c.x_need_region <= c.xregion && steps <= c.xsteps) return;
  cudaStream_t s = e.stream;
  OB_CUDA(cudaStreamSynchronize(s));
  e.drop_graphs();  // captured graphs hold the old buffer addresses
  comm_barrier(e);  // every peer stopped using the old buffers
  close_exchange(e);
  comm_barrier(e);
  const size_t region = std::max(c.x_need_region, c.xregion * 3 / 2);
  const size_t bytes = kXFlags + (size_t)steps * region;
  void* q = nullptr;
  OB_CUDA(cudaMalloc(&q, bytes));
  OB_CUDA(cudaMemset(q, 0, bytes));
  c.xbuf = (char*)q;
  c.xregion = region;
  c.xsteps = steps;
  if (!c.xep) {
    c.xep = (int64_t*)e.dalloc(sizeof(int64_t));
    c.xerr = (int64_t*)e.dalloc(sizeof(int64_t));
  }
  OB_CUDA(cudaMemset(c.xep, 0, sizeof(int64_t)));
  OB_CUDA(cudaMemset(c.xerr, 0, sizeof(int64_t)));
  // everyone's IPC handle to everyone
  cudaIpcMemHandle_t mine;
  OB_CUDA(cudaIpcGetMemHandle(&mine, c.xbuf));
  char* dh = (char*)e.dalloc(sizeof(cudaIpcMemHandle_t) * c.P);
  OB_CUDA(cudaMemcpy(dh + sizeof(mine) * c.my_rank, &mine, sizeof(mine), cudaMemcpyHostToDevice));
  OB_NCCL(ncclAllGather(dh + sizeof(mine) * c.my_rank, dh, sizeof(mine), ncclChar, (ncclComm_t)c.comm, s));
  std::vector<cudaIpcMemHandle_t> all(c.P);
  OB_CUDA(cudaMemcpyAsync(all.data(), dh, sizeof(mine) * c.P, cudaMemcpyDeviceToHost, s));
  OB_CUDA(cudaStreamSynchronize(s));
  e.dfree(dh);
  for (int p = 0; p < c.P; ++p) {
    if (p == c.my_rank) {
      c.xpeer[p] = c.xbuf;
      continue;
    }
    void* ptr = nullptr;
    OB_CUDA(cudaIpcOpenMemHandle(&ptr, all[p], cudaIpcMemLazyEnablePeerAccess));
    c.xpeer[p] = (char*)ptr;
  }
  comm_barrier(e);  // every peer mapped before any request uses the flags
#else
  (void)e;
#endif
}

void cgp_init_comm(Engine& e) {
#ifdef OB_WITH_NCCL
  ncclUniqueId id;
  std::memcpy(&id, e.cfg.nccl_id, sizeof(id));
  ncclComm_t comm;
  OB_NCCL(ncclCommInitRank(&comm, e.cfg.num_partitions, id, e.cfg.rank));
  e.cgp.comm = comm;
  // partial exchange over CUDA-IPC-mapped peer buffers unless OB_CGP_NCCL=1 asks for
  // the padded ncclAllReduce path
  const char* v = std::getenv("OB_CGP_NCCL");
  e.cgp.p2p = !(v && v[0] && v[0] != '0') && e.cfg.num_partitions <= kMaxParts;
  // flag-wait timeout of the NVLink exchange (wall time, %globaltimer)
  const char* t = std::getenv("OB_CGP_TIMEOUT_MS");
  const double ms = t && t[0] ? std::atof(t) : 2000.0;
  e.cgp.x_timeout_ns = (int64_t)(std::max(ms, 1.0) * 1e6);
#else
  throw Error(OB_ECOMM, "built without NCCL");
#endif
}

void cgp_destroy(Engine& e) {
#ifdef OB_WITH_NCCL
  cgp_release_exchange(e);
  if (e.cgp.comm) ncclCommDestroy((ncclComm_t)e.cgp.comm);
#endif
  e.cgp.comm = nullptr;
}

}  // namespace ob
