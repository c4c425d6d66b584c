// ob_select.cu -- SRPE candidate set, ratio scores, budgeted top-k, request CSR.
//
// Reference (paths relative to /root/reference/pkg/src/gnnserve):
//   candidate_arrays / find_candidates  compgraph.py:108-121, policy.py:64-67
//   score_query_edge_ratio              policy.py:77-81   (IEEE fp64 nq / total)
//   select_targets                      policy.py:110-135 (floor(gamma*|R|), score desc, id asc)
//   _EdgeIndex                          compgraph.py:155-171 (request edges by dst, src ascending)
//
// B200 design: the candidate set is a bitmap over [0, N) whose word-popcount
// prefix gives ascending order and an O(1) id -> candidate-rank map.  The
// top-k is a radix select over the 64-bit score bit patterns (non-negative
// doubles order like their bits) followed by an ordered compaction, so the
// (score desc, id asc) order never needs a full sort.  Request edges are
// bucketed by destination slot with shared-memory aggregation for the hot
// query slots (every query receives hundreds of edges), then each bucket is
// sorted: warp sorts for short buckets, and a chunked CTA radix sort plus
// multi-CTA merge-path levels for long ones.  Everything runs off
// device-side counts.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/warp/warp_merge_sort.cuh>

#include "ob_engine.h"

namespace ob {

int64_t g_launches = 0;

__global__ void k_fill_i32(int32_t* a, const int64_t* n_dev, int64_t n_host, int32_t v) {
  const int64_t n = dev_count(n_dev, n_host);
  OB_GRID_STRIDE(i, n) a[i] = v;
}
__global__ void k_fill_i64(int64_t* a, const int64_t* n_dev, int64_t n_host, int64_t v) {
  const int64_t n = dev_count(n_dev, n_host);
  OB_GRID_STRIDE(i, n) a[i] = v;
}

// warp-aggregated atomicAdd of 1 on base[slot]; returns this lane's old value
__device__ __forceinline__ int32_t warp_agg_inc(int32_t* base, int64_t slot) {
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, (unsigned long long)slot);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  int32_t old = 0;
  if (lane == leader) old = atomicAdd(base + slot, __popc(peers));
  old = __shfl_sync(peers, old, leader);
  return old + __popc(peers & ((1u << lane) - 1u));
}

// ---------------------------------------------------------------------------
// 1. validate + mark training endpoints + per-query in-degree
// ---------------------------------------------------------------------------
constexpr int kEdgeTile = 4096;  // request edges per CTA pass
constexpr int kMaxSmemQueries = 12288;

__global__ void __launch_bounds__(256) k_request_mark(const ReqParams* rp, int64_t N, int B, uint32_t* cbits,
                                                      int32_t* qdeg, ReqCounters* rc) {
  extern __shared__ int32_t sq[];  // per-CTA query in-degree histogram (B entries) when B fits
  const int64_t* __restrict__ edges = rp->edges;
  const int64_t m = rp->m;
  const bool smem = B <= kMaxSmemQueries;
  const int64_t hi = N + B;
  int64_t err = 0;
  for (int64_t t0 = (int64_t)blockIdx.x * kEdgeTile; t0 < m; t0 += (int64_t)gridDim.x * kEdgeTile) {
    if (smem) {
      for (int q = threadIdx.x; q < B; q += blockDim.x) sq[q] = 0;
      __syncthreads();
    }
    const int64_t t1 = min(t0 + kEdgeTile, m);
    for (int64_t e = t0 + threadIdx.x; e < t1; e += blockDim.x) {
      int64_t s, d;
      ld_edge(edges, e, s, d);
      if (s < 0 || s >= hi || d < 0 || d >= hi) {
        err |= kErrRange;
        continue;
      }
      if (s < N && d < N) err |= kErrNoQuery;
      if (s < N) bm_set(cbits, s);
      if (d < N) bm_set(cbits, d);
      else if (smem) atomicAdd(sq + (d - N), 1);
      else atomicAdd(qdeg + (d - N), 1);
    }
    if (smem) {
      __syncthreads();
      for (int q = threadIdx.x; q < B; q += blockDim.x)
        if (sq[q]) atomicAdd(qdeg + q, sq[q]);
      __syncthreads();
    }
  }
  if (err) atomicOr((unsigned long long*)&rc->err, (unsigned long long)err);
}

__global__ void k_check_finite(const ReqParams* rp, int64_t n, ReqCounters* rc) {
  const float* __restrict__ q = rp->qfeat;
  bool bad = false;
  OB_GRID_STRIDE(i, n) bad |= !isfinite(q[i]);
  if (bad) atomicOr((unsigned long long*)&rc->err, (unsigned long long)kErrNonFinite);
}

// ids of set bits in ascending order (bitmap -> sorted unique list)
__global__ void k_bitmap_compact(const uint32_t* __restrict__ bits, const int64_t* __restrict__ wpre, int64_t words,
                                 int32_t* out) {
  OB_GRID_STRIDE(w, words) {
    uint32_t b = bits[w];
    int64_t pos = wpre[w];
    while (b) {
      int t = __ffs(b) - 1;
      out[pos++] = (int32_t)(w * 32 + t);
      b &= b - 1;
    }
  }
}

void k_bitmap_compact_ext(Engine& e, const uint32_t* bits, const int64_t* wpre, int64_t words, int32_t* out) {
  k_bitmap_compact<<<grid_for(words, 256), 256, 0, e.stream>>>(bits, wpre, words, out);
  OB_LAUNCHED();
}

// RB = R + B slots; query slots take their counts from the per-query in-degrees
__global__ void k_slots_init(ReqCounters* rc, int B, const int32_t* qdeg, int32_t* rq_cnt, int32_t* rq_fill) {
  const int64_t R = rc->R;
  if (blockIdx.x == 0 && threadIdx.x == 0) rc->RB = R + B;
  const int64_t RB = R + B;
  OB_GRID_STRIDE(i, RB) {
    rq_cnt[i] = i < R ? 0 : qdeg[i - R];
    rq_fill[i] = 0;
  }
}

__global__ void k_rq_count(const ReqParams* rp, int64_t N, const uint32_t* cbits, const int64_t* cwpre,
                           const ReqCounters* rc, int32_t* rq_cnt) {
  if (rc->err & (kErrRange | kErrNoQuery)) return;
  const int64_t* __restrict__ edges = rp->edges;
  const int64_t m = rp->m;
  OB_GRID_STRIDE(e, m) {
    int64_t d = edges[2 * e + 1];
    if (d < N) warp_agg_inc(rq_cnt, bm_rank(cbits, cwpre, d));
  }
}

// request-CSR slot of a destination: candidate rank for training ids, R + q for queries
__device__ __forceinline__ int64_t rq_slot(int64_t d, int64_t N, const uint32_t* cbits, const int64_t* cwpre,
                                           int64_t R) {
  return d < N ? bm_rank(cbits, cwpre, d) : R + (d - N);
}

// every slot (candidate and query) of an edge subset -- a CGP rank's slice
__global__ void k_rq_count_all(const int64_t* __restrict__ edges, int64_t m_host, const int64_t* m_dev, int64_t N,
                               const uint32_t* cbits, const int64_t* cwpre, const ReqCounters* rc, int32_t* rq_cnt) {
  if (rc->err & (kErrRange | kErrNoQuery)) return;
  const int64_t R = rc->R, m = dev_count(m_dev, m_host);  // a CGP slice: edges live in the arena
  OB_GRID_STRIDE(e, m) warp_agg_inc(rq_cnt, rq_slot(edges[2 * e + 1], N, cbits, cwpre, R));
}

__global__ void k_zero_slots(const ReqCounters* rc, int B, int32_t* a, int32_t* b) {
  const int64_t RB = rc->R + B;
  OB_GRID_STRIDE(i, RB) a[i] = b[i] = 0;
}

// ---------------------------------------------------------------------------
// 2. ratio scores (policy.py:77-81) and budget
// ---------------------------------------------------------------------------
__global__ void k_score(const int32_t* __restrict__ cand_ids, const int32_t* __restrict__ rq_cnt,
                        const int32_t* __restrict__ indeg, ReqCounters* rc, int32_t* cand_nq, double* score,
                        uint64_t* key, int32_t* tpos) {
  const int64_t R = rc->R;
  bool bad = false;
  OB_GRID_STRIDE(c, R) {
    int32_t nq = rq_cnt[c];
    int64_t total = (int64_t)indeg[cand_ids[c]] + nq;
    if (total <= 0) bad = true;
    double s = total > 0 ? (double)nq / (double)total : 0.0;
    cand_nq[c] = nq;
    score[c] = s;
    key[c] = (uint64_t)__double_as_longlong(s);  // s >= +0.0: bit order == value order
    tpos[c] = -1;
  }
  if (bad) atomicOr((unsigned long long*)&rc->err, (unsigned long long)kErrZeroTotal);
}

__global__ void k_budget(ReqCounters* rc, double gamma, uint32_t* hist) {
  // budget = int(np.floor(gamma * m)) with gamma a Python float: one IEEE fp64 multiply
  const int64_t R = rc->R;
  const int64_t b = (int64_t)floor(gamma * (double)R);
  if (threadIdx.x == 0) {
    rc->budget = b;
    rc->sel_prefix = 0;
    rc->sel_mask = 0;
    rc->sel_krem = b;
    rc->sel_gt = 0;
    rc->sel_eq_take = 0;
    rc->T = 0;
  }
  if (threadIdx.x < 256) hist[threadIdx.x] = 0;
}

// radix select, MSB-first 8-bit digits: find the budget-th largest key
__global__ void k_sel_hist(const uint64_t* __restrict__ key, const ReqCounters* rc, int shift, uint32_t* hist) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t R = rc->R, b = rc->budget;
  if (b > 0 && b < R) {
    const uint64_t pre = rc->sel_prefix, msk = rc->sel_mask;
    OB_GRID_STRIDE(c, R) {
      uint64_t k = key[c];
      if ((k & msk) == pre) atomicAdd(&h[(k >> shift) & 255], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, h[i]);
}

__global__ void __launch_bounds__(256) k_sel_pick(ReqCounters* rc, int shift, uint32_t* hist) {
  using BS = cub::BlockScan<int64_t, 256>;
  __shared__ typename BS::TempStorage tmp;
  const int64_t R = rc->R, b = rc->budget;
  const int d = 255 - threadIdx.x;  // scan from the top digit down
  int64_t c = hist[d];
  int64_t excl;
  BS(tmp).ExclusiveSum(c, excl);  // keys in digits above d
  hist[d] = 0;
  if (!(b > 0 && b < R)) return;
  const int64_t krem = rc->sel_krem;
  if (excl < krem && krem <= excl + c) {
    rc->sel_krem = krem - excl;
    rc->sel_gt += excl;
    rc->sel_prefix |= (uint64_t)d << shift;
    rc->sel_mask |= (uint64_t)255 << shift;
    if (shift == 0) rc->sel_eq_take = krem - excl;
  }
}

struct EqLoad {
  const uint64_t* key;
  const ReqCounters* rc;
  __device__ int64_t operator()(int64_t c) const {
    const int64_t R = rc->R, b = rc->budget;
    return (b > 0 && b < R && key[c] == rc->sel_prefix) ? 1 : 0;
  }
};
// selected = above the threshold, or at it among the lowest ids (score desc, id asc)
struct EqStore {
  int32_t* flag;
  const uint64_t* key;
  const ReqCounters* rc;
  __device__ void operator()(int64_t c, int64_t eqpos) const {
    const int64_t R = rc->R, b = rc->budget;
    int sel;
    if (b <= 0) sel = 0;
    else if (b >= R) sel = 1;
    else {
      uint64_t k = key[c], thr = rc->sel_prefix;
      sel = (k > thr) || (k == thr && eqpos < rc->sel_eq_take);
    }
    flag[c] = sel;
  }
};
struct SelStore {
  const int32_t* flag;
  const int32_t* cand_ids;
  int32_t* targets;
  int32_t* tpos;
  __device__ void operator()(int64_t c, int64_t pos) const {
    if (flag[c]) {
      targets[pos] = cand_ids[c];
      tpos[c] = (int32_t)pos;
    }
  }
};

// ---------------------------------------------------------------------------
// 3. request CSR fill: per-CTA reservation for query slots, warp-aggregated
//    atomics for candidate slots
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_rq_fill(const int64_t* __restrict__ edges_arg, int64_t m_host,
                                                 const int64_t* m_dev, const ReqParams* rp, int64_t N, int B,
                                                 const uint32_t* cbits, const int64_t* cwpre, const ReqCounters* rc,
                                                 const int64_t* rq_ptr, int32_t* rq_fill, int32_t* rq_src) {
  extern __shared__ int32_t sm[];  // [B] counts, then [B] base offsets
  const bool smem = B <= kMaxSmemQueries / 2;
  if (rc->err & (kErrRange | kErrNoQuery)) return;
  const int64_t R = rc->R;
  // the whole request (edges from the parameter block) or a CGP slice in the arena
  const int64_t* __restrict__ edges = rp ? rp->edges : edges_arg;
  const int64_t m = rp ? rp->m : dev_count(m_dev, m_host);
  int32_t* cnt = sm;
  int32_t* base = sm + B;
  for (int64_t t0 = (int64_t)blockIdx.x * kEdgeTile; t0 < m; t0 += (int64_t)gridDim.x * kEdgeTile) {
    const int64_t t1 = min(t0 + kEdgeTile, m);
    if (smem) {
      for (int q = threadIdx.x; q < B; q += blockDim.x) cnt[q] = 0;
      __syncthreads();
      for (int64_t e = t0 + threadIdx.x; e < t1; e += blockDim.x) {
        int64_t d = edges[2 * e + 1];
        if (d >= N) atomicAdd(cnt + (d - N), 1);
      }
      __syncthreads();
      for (int q = threadIdx.x; q < B; q += blockDim.x) {
        base[q] = cnt[q] ? atomicAdd(rq_fill + R + q, cnt[q]) : 0;
        cnt[q] = 0;
      }
      __syncthreads();
    }
    for (int64_t e = t0 + threadIdx.x; e < t1; e += blockDim.x) {
      int64_t s, d;
      ld_edge(edges, e, s, d);
      int64_t pos;
      if (d >= N) {
        int64_t q = d - N;
        pos = rq_ptr[R + q] + (smem ? base[q] + atomicAdd(cnt + q, 1) : atomicAdd(rq_fill + R + q, 1));
      } else {
        int64_t c = bm_rank(cbits, cwpre, d);
        pos = rq_ptr[c] + warp_agg_inc(rq_fill, c);
      }
      rq_src[pos] = (int32_t)s;
    }
    if (smem) __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// 4. per-slot sort of request sources
// ---------------------------------------------------------------------------
constexpr int kWarpSortItems = 8;     // warp sort handles <= 256
constexpr int kChunkThreads = 512;
constexpr int kChunkItems = 8;
constexpr int kChunk = kChunkThreads * kChunkItems;  // 4096-element CTA sort tiles

__device__ __forceinline__ void warp_bitonic32(int32_t& v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      int32_t o = __shfl_xor_sync(0xffffffffu, v, j);
      bool up = ((lane & k) == 0);
      bool lower = ((lane & j) == 0);
      v = (lower == up) ? min(v, o) : max(v, o);
    }
  }
}

struct LessI32 {
  __device__ bool operator()(const int32_t& a, const int32_t& b) const { return a < b; }
};

__global__ void __launch_bounds__(256) k_segsort_warp(const int64_t* __restrict__ ptr, const ReqCounters* rc,
                                                      int64_t* ctr, int32_t* vals, int32_t* big_list) {
  using WS = cub::WarpMergeSort<int32_t, kWarpSortItems, 32>;
  __shared__ typename WS::TempStorage tmp[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nseg = rc->RB;
  for (int64_t s = (int64_t)blockIdx.x * 8 + warp; s < nseg; s += (int64_t)gridDim.x * 8) {
    const int64_t b = ptr[s], len = ptr[s + 1] - b;
    if (len <= 1) continue;
    if (len <= 32) {
      int32_t v = lane < len ? vals[b + lane] : INT32_MAX;
      warp_bitonic32(v);
      if (lane < len) vals[b + lane] = v;
    } else if (len <= 32 * kWarpSortItems) {
      int32_t k[kWarpSortItems];
#pragma unroll
      for (int i = 0; i < kWarpSortItems; ++i) {
        int64_t idx = (int64_t)lane * kWarpSortItems + i;
        k[i] = idx < len ? vals[b + idx] : INT32_MAX;
      }
      WS(tmp[warp]).Sort(k, LessI32());
#pragma unroll
      for (int i = 0; i < kWarpSortItems; ++i) {
        int64_t idx = (int64_t)lane * kWarpSortItems + i;
        if (idx < len) vals[b + idx] = k[i];
      }
    } else if (lane == 0) {
      int64_t at = atomicAdd((unsigned long long*)&ctr[1], 1ull);
      big_list[at] = (int32_t)s;
    }
  }
}

struct ChunkLoad {
  const int32_t* big_list;
  const int64_t* ptr;
  __device__ int64_t operator()(int64_t i) const {
    int64_t s = big_list[i];
    return (ptr[s + 1] - ptr[s] + kChunk - 1) / kChunk;
  }
};

// (big segment, chunk) of chunk index ci
__device__ __forceinline__ void chunk_of(const int64_t* cptr, int64_t nbig, int64_t ci, int64_t* seg, int64_t* j) {
  int64_t lo = 0, hi = nbig;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (cptr[mid] <= ci) lo = mid;
    else hi = mid;
  }
  *seg = lo;
  *j = ci - cptr[lo];
}

// sort every 4096-element chunk of every long segment in shared memory
__device__ __forceinline__ int levels_for(int64_t len);

// ids are < 2^end_bit, so only end_bit radix bits are sorted; the merge levels the
// longest segment needs are published in ctr[3] (later levels exit at once)
__global__ void __launch_bounds__(kChunkThreads) k_chunk_sort(const int64_t* __restrict__ ptr, int64_t* ctr,
                                                              const int32_t* big_list, const int64_t* cptr,
                                                              int32_t* vals, int end_bit) {
  using BRS = cub::BlockRadixSort<int32_t, kChunkThreads, kChunkItems>;
  __shared__ typename BRS::TempStorage tmp;
  const int64_t nbig = ctr[1], nch = ctr[2];
  for (int64_t ci = blockIdx.x; ci < nch; ci += gridDim.x) {
    int64_t bi, j;
    chunk_of(cptr, nbig, ci, &bi, &j);
    const int64_t s = big_list[bi];
    const int64_t b = ptr[s] + j * kChunk, len = min((int64_t)kChunk, ptr[s + 1] - b);
    if (j == 0 && threadIdx.x == 0)
      atomicMax((unsigned long long*)&ctr[3], (unsigned long long)levels_for(ptr[s + 1] - ptr[s]));
    int32_t k[kChunkItems];
#pragma unroll
    for (int i = 0; i < kChunkItems; ++i) {
      int64_t idx = (int64_t)threadIdx.x * kChunkItems + i;
      k[i] = idx < len ? vals[b + idx] : INT32_MAX;  // padding sorts last (stable, all-ones low bits)
    }
    BRS(tmp).Sort(k, 0, end_bit);
#pragma unroll
    for (int i = 0; i < kChunkItems; ++i) {
      int64_t idx = (int64_t)threadIdx.x * kChunkItems + i;
      if (idx < len) vals[b + idx] = k[i];
    }
    __syncthreads();
  }
}

// number of elements of a[0,na) that are < v (strict) or <= v
__device__ __forceinline__ int lower_cnt(const int32_t* a, int na, int32_t v, bool inclusive) {
  int lo = 0, hi = na;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    bool go = inclusive ? (a[mid] <= v) : (a[mid] < v);
    if (go) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// merge levels a segment of `len` needs after the 4096-element chunk sort
__device__ __forceinline__ int levels_for(int64_t len) {
  int l = 0;
  for (int64_t w = kChunk; w < len; w *= 2) ++l;
  return l;
}

// merge level `level` (run width 4096 << level): runs merge pairwise from the
// buffer the segment's data currently sits in (parity of the level) into the
// other; segments that need fewer levels are skipped.  Each CTA produces one
// 4096-element output tile (merge-path split, then rank-merge in shared memory).
__global__ void __launch_bounds__(kChunkThreads) k_merge_level(const int64_t* __restrict__ ptr, const int64_t* ctr,
                                                               const int32_t* big_list, const int64_t* cptr,
                                                               int32_t* vals, int32_t* tmp, int level) {
  __shared__ int32_t sa[kChunk];
  __shared__ int32_t sb[kChunk];
  __shared__ int64_t split[2];
  const int64_t nbig = ctr[1], nch = ctr[2];
  if (level >= ctr[3]) return;  // no segment needs this level
  const int64_t w = (int64_t)kChunk << level;
  for (int64_t ci = blockIdx.x; ci < nch; ci += gridDim.x) {
    int64_t bi, j;
    chunk_of(cptr, nbig, ci, &bi, &j);
    const int64_t s = big_list[bi];
    const int64_t sb0 = ptr[s], len = ptr[s + 1] - sb0;
    if (level >= levels_for(len)) continue;  // uniform per CTA
    const int32_t* src = (level & 1) ? tmp : vals;
    int32_t* dst = (level & 1) ? vals : tmp;
    const int64_t o0 = j * kChunk, o1 = min(o0 + kChunk, len);
    const int64_t ps = (o0 / (2 * w)) * (2 * w);
    const int64_t na = min(w, len - ps), nb = max((int64_t)0, min(w, len - ps - na));
    const int32_t* A = src + sb0 + ps;
    const int32_t* Bp = A + na;
    if (nb == 0) {  // lone run: copy through
      for (int64_t o = o0 + threadIdx.x; o < o1; o += blockDim.x) dst[sb0 + o] = src[sb0 + o];
      __syncthreads();
      continue;
    }
    if (threadIdx.x < 2) {
      const int64_t d = (threadIdx.x == 0 ? o0 : o1) - ps;
      int64_t lo = max((int64_t)0, d - nb), hi = min(d, na);
      while (lo < hi) {  // merge path: A elements precede equal B elements
        int64_t mid = (lo + hi) >> 1;
        if (A[mid] <= Bp[d - 1 - mid]) lo = mid + 1;
        else hi = mid;
      }
      split[threadIdx.x] = lo;
    }
    __syncthreads();
    const int64_t a0 = split[0], a1 = split[1];
    const int64_t b0 = (o0 - ps) - a0, b1 = (o1 - ps) - a1;
    const int la = (int)(a1 - a0), lb = (int)(b1 - b0);
    for (int i = threadIdx.x; i < la; i += blockDim.x) sa[i] = A[a0 + i];
    for (int i = threadIdx.x; i < lb; i += blockDim.x) sb[i] = Bp[b0 + i];
    __syncthreads();
    int32_t* out = dst + sb0 + o0;
    for (int i = threadIdx.x; i < la; i += blockDim.x) out[i + lower_cnt(sb, lb, sa[i], false)] = sa[i];
    for (int i = threadIdx.x; i < lb; i += blockDim.x) out[i + lower_cnt(sa, la, sb[i], true)] = sb[i];
    __syncthreads();
  }
}

// segments whose level count is odd finished in tmp: copy their tiles back
__global__ void __launch_bounds__(kChunkThreads) k_merge_copyback(const int64_t* __restrict__ ptr,
                                                                  const int64_t* ctr, const int32_t* big_list,
                                                                  const int64_t* cptr, int32_t* vals,
                                                                  const int32_t* tmp) {
  const int64_t nbig = ctr[1], nch = ctr[2];
  for (int64_t ci = blockIdx.x; ci < nch; ci += gridDim.x) {
    int64_t bi, j;
    chunk_of(cptr, nbig, ci, &bi, &j);
    const int64_t s = big_list[bi];
    const int64_t sb0 = ptr[s], len = ptr[s + 1] - sb0;
    if (!(levels_for(len) & 1)) continue;
    const int64_t o0 = j * kChunk, o1 = min(o0 + kChunk, len);
    for (int64_t o = o0 + threadIdx.x; o < o1; o += blockDim.x) vals[sb0 + o] = tmp[sb0 + o];
  }
}

// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------
void stage_request_prep(Engine& e, RequestWs& w, bool need_scores) {
  cudaStream_t s = e.stream;
  const int64_t N = e.g.N;
  const int64_t m = w.m;
  OB_CUDA(cudaMemsetAsync(w.cbits, 0, sizeof(uint32_t) * (w.words_N + 1), s));
  OB_CUDA(cudaMemsetAsync(w.qdeg, 0, sizeof(int32_t) * (w.B + 1), s));
  const size_t sq = w.B <= kMaxSmemQueries ? sizeof(int32_t) * w.B : 0;
  if (m > 0) {
    k_request_mark<<<grid_for(m, kEdgeTile, kNumSMs * 4), 256, sq, s>>>(w.rp, N, w.B, w.cbits, w.qdeg, w.rc);
    OB_LAUNCHED();
  }
  if ((int64_t)w.B * e.g.F > 0) {
    k_check_finite<<<grid_for((int64_t)w.B * e.g.F, 256), 256, 0, s>>>(w.rp, (int64_t)w.B * e.g.F, w.rc);
    OB_LAUNCHED();
  }
  // candidate set: popcount prefix, ascending ids
  device_scan(s, e.scan, LoadPopc{w.cbits}, StoreI64{w.cwpre}, nullptr, w.words_N, w.words_N, &w.rc->R, w.cwpre);
  k_bitmap_compact<<<grid_for(w.words_N, 256), 256, 0, s>>>(w.cbits, w.cwpre, w.words_N, w.cand_ids);
  OB_LAUNCHED();
  const int64_t rb_max = std::min<int64_t>(N, 2 * m) + w.B;
  k_slots_init<<<grid_for(rb_max, 256), 256, 0, s>>>(w.rc, w.B, w.qdeg, w.rq_cnt, w.rq_fill);
  OB_LAUNCHED();
  if (m > 0) {
    k_rq_count<<<grid_for(m, 256), 256, 0, s>>>(w.rp, N, w.cbits, w.cwpre, w.rc, w.rq_cnt);
    OB_LAUNCHED();
  }
  if (need_scores) {
    const int64_t r_max = std::min<int64_t>(N, 2 * m);
    k_score<<<grid_for(r_max, 256), 256, 0, s>>>(w.cand_ids, w.rq_cnt, e.g.indeg, w.rc, w.cand_nq, w.cand_score,
                                                 w.cand_key, w.cand_tpos);
    OB_LAUNCHED();
  }
}

void stage_select(Engine& e, RequestWs& w) {
  cudaStream_t s = e.stream;
  const int64_t r_max = std::min<int64_t>(e.g.N, 2 * w.m);
  k_budget<<<1, 256, 0, s>>>(w.rc, e.cfg.gamma, w.sel_hist);
  OB_LAUNCHED();
  for (int shift = 56; shift >= 0; shift -= 8) {
    k_sel_hist<<<grid_for(r_max, 256, kNumSMs * 2), 256, 0, s>>>(w.cand_key, w.rc, shift, w.sel_hist);
    k_sel_pick<<<1, 256, 0, s>>>(w.rc, shift, w.sel_hist);
    g_launches += 2;
  }
  // ordered compaction: ties at the threshold resolved by ascending id
  device_scan(s, e.scan, EqLoad{w.cand_key, w.rc}, EqStore{w.sel_flag, w.cand_key, w.rc}, &w.rc->R, 0, r_max,
              nullptr);
  device_scan(s, e.scan, LoadI32{w.sel_flag}, SelStore{w.sel_flag, w.cand_ids, w.targets, w.cand_tpos}, &w.rc->R, 0,
              r_max, &w.rc->T);
}

// Request CSR over an edge set (the whole request via the parameter block when
// edges == nullptr, or one CGP rank's slice in the arena): bucket by destination
// slot, then sort each slot's sources ascending.
void build_rq_csr(Engine& e, RequestWs& w, const int64_t* edges, int64_t m_bound, const int64_t* m_dev, RqCsr& c,
                  bool counts_ready) {
  const ReqParams* rp = edges ? nullptr : w.rp;
  cudaStream_t s = e.stream;
  const int64_t rb_max = std::min<int64_t>(e.g.N, 2 * w.m) + w.B;
  OB_CUDA(cudaMemsetAsync(c.ctr + 1, 0, 3 * sizeof(int64_t), s));
  if (!counts_ready) {
    k_zero_slots<<<grid_for(rb_max, 256), 256, 0, s>>>(w.rc, w.B, c.cnt, c.fill);
    OB_LAUNCHED();
    if (m_bound > 0) {
      k_rq_count_all<<<grid_for(m_bound, 256), 256, 0, s>>>(edges, m_bound, m_dev, e.g.N, w.cbits, w.cwpre, w.rc,
                                                              c.cnt);
      OB_LAUNCHED();
    }
  }
  device_scan(s, e.scan, LoadI32{c.cnt}, StoreI64{c.ptr}, &w.rc->RB, 0, rb_max, nullptr, c.ptr);
  if (m_bound <= 0) return;
  const size_t sm = w.B <= kMaxSmemQueries / 2 ? 2 * sizeof(int32_t) * w.B : 0;
  k_rq_fill<<<grid_for(m_bound, kEdgeTile, kNumSMs * 4), 256, sm, s>>>(edges, m_bound, m_dev, rp, e.g.N, w.B,
                                                                         w.cbits, w.cwpre, w.rc, c.ptr, c.fill, c.src);
  k_segsort_warp<<<grid_for(rb_max, 8), 256, 0, s>>>(c.ptr, w.rc, c.ctr, c.src, c.big_list);
  g_launches += 2;
  // long segments: chunk sort + merge levels (ping-pong src <-> sort_tmp)
  device_scan(s, e.scan, ChunkLoad{c.big_list, c.ptr}, StoreI64{c.big_cptr}, c.ctr + 1, 0, rb_max, c.ctr + 2,
              c.big_cptr);
  const int64_t ch_max = m_bound / kChunk + rb_max / 256 + 2;
  const int g = grid_for(ch_max, 1, kNumSMs * 4);
  int end_bit = 1;
  while (end_bit < 31 && ((int64_t)1 << end_bit) <= e.g.N + w.B) ++end_bit;
  k_chunk_sort<<<g, kChunkThreads, 0, s>>>(c.ptr, c.ctr, c.big_list, c.big_cptr, c.src, end_bit);
  OB_LAUNCHED();
  // the longest possible segment is the whole edge set; levels past a segment's
  // own count exit immediately
  int level = 0;
  for (int64_t wd = kChunk; wd < m_bound; wd *= 2, ++level) {
    k_merge_level<<<g, kChunkThreads, 0, s>>>(c.ptr, c.ctr, c.big_list, c.big_cptr, c.src, c.sort_tmp, level);
    OB_LAUNCHED();
  }
  if (level > 0) {
    k_merge_copyback<<<g, kChunkThreads, 0, s>>>(c.ptr, c.ctr, c.big_list, c.big_cptr, c.src, c.sort_tmp);
    OB_LAUNCHED();
  }
}

void stage_request_csr(Engine& e, RequestWs& w) {
  RqCsr c = w.rq_view();
  build_rq_csr(e, w, nullptr, w.m, nullptr, c, /*counts_ready=*/true);
}

}  // namespace ob
