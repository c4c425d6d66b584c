// ob_select.cu -- SRPE candidate set, ratio scores, budgeted top-k, request CSR.
//
// Reference (paths relative to /root/reference/pkg/src/gnnserve):
//   candidate_arrays / find_candidates  compgraph.py:108-121, policy.py:64-67
//   score_query_edge_ratio              policy.py:77-81   (IEEE fp64 nq / total)
//   score_importance / partial sums     policy.py:84-107, runtime.py:168-175 (numpy pairwise fp64 sums)
//   select_targets                      policy.py:110-135 (floor(gamma*|R|), score desc, id asc)
//   _EdgeIndex                          compgraph.py:155-171 (request edges by dst, src ascending)
//
// B200 design: the candidate set is a bitmap over [0, N) whose word-popcount
// prefix gives ascending order and an O(1) id -> candidate-rank map.  The
// top-k is a radix select over the 64-bit score bit patterns (non-negative
// doubles order like their bits) followed by an ordered compaction, so the
// (score desc, id asc) order never needs a full sort.  The request CSR
// (sources by destination slot, ascending) is one stable LSD radix sort of a
// packed (population, slot, source) key per edge -- usually 29 bits, so four
// 8-bit passes over 32-bit keys -- which handles hub queries with 10^5 in-edges
// and the ~10^5 tiny candidate slots alike.  Everything runs off device-side
// counts.
#include <cstdlib>
#include <cooperative_groups.h>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "ob_engine.h"

namespace ob {

int64_t g_launches = 0;

// exclusive scan of the tile sums in place (one CTA; long scans only)
__global__ void __launch_bounds__(1024) k_scan_spine(const int64_t* n_dev, int64_t n_host, int64_t* tile_sums) {
  pdl_wait();
  using BS = cub::BlockScan<int64_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t carry;
  const int64_t n = cta_count(n_dev, n_host);
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b = 0; b < ntiles; b += 1024) {
    const int64_t i = b + threadIdx.x;
    int64_t v = i < ntiles ? tile_sums[i] : 0, agg;
    BS(tmp).ExclusiveSum(v, v, agg);
    if (i < ntiles) tile_sums[i] = v + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
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
  pdl_wait();
  extern __shared__ int32_t sq[];  // per-CTA query in-degree histogram (B entries) when B fits
  const int64_t* __restrict__ edges = rp->edges;
  const int64_t m = cta_ld(&rp->m);
  const bool smem = B <= kMaxSmemQueries;
  const int64_t hi = N + B;
  int64_t err = 0;
  for (int64_t t0 = (int64_t)blockIdx.x * kEdgeTile; t0 < m; t0 += (int64_t)gridDim.x * kEdgeTile) {
    if (smem) {
      for (int q = threadIdx.x; q < B; q += blockDim.x) sq[q] = 0;
      __syncthreads();
    }
    const int64_t t1 = min(t0 + kEdgeTile, m);
    constexpr int kU = 4;  // edges per thread with their loads in flight together
    for (int64_t e00 = t0 + threadIdx.x; e00 < t1; e00 += (int64_t)kU * blockDim.x) {
      int64_t sv[kU], dv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t e = e00 + (int64_t)u * blockDim.x;
        sv[u] = dv[u] = 0;
        if (e < t1) ld_edge(edges, e, sv[u], dv[u]);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (e00 + (int64_t)u * blockDim.x >= t1) break;
        const int64_t s = sv[u], d = dv[u];
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
  pdl_wait();
  const float* __restrict__ q = rp->qfeat;
  bool bad = false;
  OB_GRID_STRIDE(i, n) bad |= !isfinite(q[i]);
  if (bad) atomicOr((unsigned long long*)&rc->err, (unsigned long long)kErrNonFinite);
}

// ids of set bits in ascending order (bitmap -> sorted unique list)
__global__ void k_bitmap_compact(const uint32_t* __restrict__ bits, const int64_t* __restrict__ wpre, int64_t words,
                                 int32_t* out) {
  pdl_wait();
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
  launch_pdl(k_bitmap_compact, dim3(grid_for(words, 256)), dim3(256), 0, e.stream, bits, wpre, words, out);
}

// Bitmap-rank over a huge id space (papers scale: 3.5M words for 111M ids) with
// few set bits: count per 32-word group (one warp reads a group's 128 bytes), scan
// the group counts (32x shorter than the words), then only the non-empty groups
// write their words' prefixes and their ids.  The dense path scans every word and
// writes an int64 prefix for all of them (~100 MB of traffic at 111M ids); this one
// reads the bitmap once.  Word prefixes of empty groups are left unwritten: ranks
// are only taken of set bits.
__global__ void __launch_bounds__(256) k_bm_group_popc(const uint32_t* __restrict__ bits, int64_t words,
                                                       int64_t groups, int32_t* gcnt) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = gw; g < groups; g += nw) {
    const int64_t w = g * 32 + lane;
    int c = w < words ? __popc(__ldg(bits + w)) : 0;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) gcnt[g] = c;
  }
}

__global__ void __launch_bounds__(256) k_bm_group_fin(const uint32_t* __restrict__ bits, int64_t words, int64_t groups,
                                                      const int32_t* __restrict__ gcnt,
                                                      const int64_t* __restrict__ gpre, int64_t* wpre, int32_t* out) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (gw == 0 && lane == 0) wpre[words] = gpre[groups];  // the total, like the dense scan's out_arr
  for (int64_t g = gw; g < groups; g += nw) {
    if (__ldg(gcnt + g) == 0) continue;
    const int64_t w = g * 32 + lane;
    uint32_t b = w < words ? __ldg(bits + w) : 0u;
    const int c = __popc(b);
    int x = c;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    int64_t pos = __ldg(gpre + g) + (x - c);
    if (w < words) wpre[w] = pos;
    while (b) {
      const int t = __ffs(b) - 1;
      out[pos++] = (int32_t)(w * 32 + t);
      b &= b - 1;
    }
  }
}

// prefix of set bits per word + the sorted ids of the set bits + their count:
// the dense scan, or the group-sparse one for large bitmaps
void bitmap_rank(Engine& e, const uint32_t* bits, int64_t words, int64_t* wpre, int32_t* out, int64_t* total,
                 int32_t* gcnt, int64_t* gpre) {
  cudaStream_t s = e.stream;
  if (words <= kSparseRankWords || !gcnt) {
    device_scan(s, e.scan, LoadPopc{bits}, StoreI64{wpre}, nullptr, words, words, total, wpre);
    k_bitmap_compact_ext(e, bits, wpre, words, out);
    return;
  }
  const int64_t groups = (words + 31) / 32;
  launch_pdl(k_bm_group_popc, dim3(grid_for(groups, 8, kNumSMs * 16)), dim3(256), 0, s, bits, words, groups, gcnt);
  device_scan(s, e.scan, LoadI32{gcnt}, StoreI64{gpre}, nullptr, groups, groups, total, gpre);
  launch_pdl(k_bm_group_fin, dim3(grid_for(groups, 8, kNumSMs * 16)), dim3(256), 0, s, bits, words, groups,
             (const int32_t*)gcnt, (const int64_t*)gpre, wpre, out);
}

// RB = R + B slots; query slots take their counts from the per-query in-degrees
__global__ void k_slots_init(ReqCounters* rc, int B, const int32_t* qdeg, int32_t* rq_cnt, int32_t* rq_fill) {
  pdl_wait();
  const int64_t R = cta_ld(&rc->R);
  if (blockIdx.x == 0 && threadIdx.x == 0) rc->RB = R + B;
  const int64_t RB = R + B;
  OB_GRID_STRIDE(i, RB) {
    rq_cnt[i] = i < R ? 0 : qdeg[i - R];
    rq_fill[i] = 0;
  }
}

// packed request-edge key (RqKeyFmt); candidate ranks come from the bitmap
// Sources into a query slot are stored by candidate rank (every training
// endpoint of the request is a candidate, and ranks follow id order) or R + q'
// for a query source, so the key needs bits(R + B) for them, not bits(N + B).
template <class K>
__device__ __forceinline__ K rq_key(int64_t s, int64_t d, int64_t N, const uint32_t* cbits, const int64_t* cwpre,
                                    int64_t R, const RqKeyFmt& f) {
  if (d < N) return ((K)bm_rank(cbits, cwpre, d) << f.bB) | (K)(s - N);
  const int64_t sr = s < N ? bm_rank(cbits, cwpre, s) : R + (s - N);
  return ((K)1 << f.body) | ((K)(d - N) << f.bN) | (K)sr;
}

// candidate-slot counts (query slots take qdeg) + one radix key per edge
template <class K>
__global__ void k_rq_count(const ReqParams* rp, int64_t N, const uint32_t* cbits, const int64_t* cwpre,
                           const ReqCounters* rc, int32_t* rq_cnt, K* keys, RqKeyFmt f) {
  pdl_wait();
  const CtaWords st = cta_ldv(&rc->err, &rp->m, &rc->R);
  if (st.v[0] & (kErrRange | kErrNoQuery)) return;
  const int64_t* __restrict__ edges = rp->edges;
  const int64_t m = st.v[1], R = st.v[2];
  OB_GRID_STRIDE(e, m) {
    int64_t s, d;
    ld_edge(edges, e, s, d);
    if (d < N) warp_agg_inc(rq_cnt, bm_rank(cbits, cwpre, d));
    keys[e] = rq_key<K>(s, d, N, cbits, cwpre, R, f);
  }
}

// request-CSR slot of a destination: candidate rank for training ids, R + q for queries
__device__ __forceinline__ int64_t rq_slot(int64_t d, int64_t N, const uint32_t* cbits, const int64_t* cwpre,
                                           int64_t R) {
  return d < N ? bm_rank(cbits, cwpre, d) : R + (d - N);
}

// every slot (candidate and query) of an edge subset -- a CGP rank's slice -- + keys
template <class K>
__global__ void k_rq_count_all(const int64_t* __restrict__ edges, const int64_t* m_dev, int64_t N,
                               const uint32_t* cbits, const int64_t* cwpre, const ReqCounters* rc, int32_t* rq_cnt,
                               K* keys, RqKeyFmt f) {
  pdl_wait();
  const CtaWords st = cta_ldv(&rc->err, &rc->R, m_dev);
  if (st.v[0] & (kErrRange | kErrNoQuery)) return;
  const int64_t R = st.v[1], m = st.v[2];  // a CGP slice: edges live in the arena
  OB_GRID_STRIDE(e, m) {
    int64_t s, d;
    ld_edge(edges, e, s, d);
    warp_agg_inc(rq_cnt, rq_slot(d, N, cbits, cwpre, R));
    keys[e] = rq_key<K>(s, d, N, cbits, cwpre, R, f);
  }
}

__global__ void k_zero_slots(const ReqCounters* rc, int B, int32_t* a, int32_t* b) {
  pdl_wait();
  const int64_t RB = cta_ld(&rc->R) + B;
  OB_GRID_STRIDE(i, RB) a[i] = b[i] = 0;
}

// ---------------------------------------------------------------------------
// 2. ratio scores (policy.py:77-81) and budget
// ---------------------------------------------------------------------------
// ratio == false (IS policy): counts only; k_score_is writes the scores and the
// zero-total check does not apply (score_importance never divides by the total)
__global__ void k_score(const int32_t* __restrict__ cand_ids, const int32_t* __restrict__ rq_cnt,
                        const int32_t* __restrict__ indeg, ReqCounters* rc, int32_t* cand_nq, double* score,
                        uint64_t* key, int32_t* tpos, bool ratio) {
  pdl_wait();
  const int64_t R = cta_ld(&rc->R);
  bool bad = false;
  OB_GRID_STRIDE(c, R) {
    int32_t nq = rq_cnt[c];
    cand_nq[c] = nq;
    tpos[c] = -1;
    if (!ratio) continue;
    int64_t total = (int64_t)indeg[cand_ids[c]] + nq;
    if (total <= 0) bad = true;
    double s = total > 0 ? (double)nq / (double)total : 0.0;
    score[c] = s;
    key[c] = (uint64_t)__double_as_longlong(s);  // s >= +0.0: bit order == value order
  }
  if (bad) atomicOr((unsigned long long*)&rc->err, (unsigned long long)kErrZeroTotal);
}

// ---------------------------------------------------------------------------
// 2b. importance scores (policy.py:84-107, runtime.py:168-175)
//
// IS(v) = (1/deg v) * sum_{u in N(v)} [deg u > 0] / deg u over the training
// CSR, in fp64.  The reference sums each row with np.sum, i.e. numpy's
// pairwise summation: rows under 8 terms add sequentially from 0.0; rows of
// 8..128 terms run eight strided accumulators combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail; longer rows
// split at n2 = n/2 - (n/2)%8 and add the halves.  One warp per candidate
// reproduces that association exactly: the leaves (64..128 terms) of the
// split tree are summed by 8-lane groups, four leaves at a time, and lane 0
// adds the leaf sums back up the same tree.  Under CGP each partition sums
// its source-split row and the partials are added in rank order.
// ---------------------------------------------------------------------------
constexpr int kPwChunk = 16384;           // rows above this split at warp level first
constexpr int kPwLeafCap = kPwChunk / 64;  // leaves are >= 64 terms
constexpr int kIsWarps = 8;

__device__ __forceinline__ double is_term(const int32_t* __restrict__ indeg, int32_t u) {
  const int32_t d = __ldg(indeg + u);
  return d > 0 ? 1.0 / (double)d : 0.0;
}

__device__ __forceinline__ int pw_split(int n) {
  const int n2 = n / 2;
  return n2 - n2 % 8;
}

// The split tree of a row depends only on its length; walk it without recursion
// (device recursion costs stack and cannot be sized statically).  Leaves of
// the tree are visited left to right; kPwDepth bounds the depth for n < 2^31.
constexpr int kPwDepth = 32;

// leaf start offsets of an n-term row (n <= kPwChunk), left to right
__device__ int pw_leaves(int n, int* starts) {
  int st_off[kPwDepth], st_n[kPwDepth], sp = 0, L = 0;
  st_off[sp] = 0;
  st_n[sp++] = n;
  while (sp) {
    --sp;
    const int o = st_off[sp], m = st_n[sp];
    if (m <= 128) {
      starts[L++] = o;
      continue;
    }
    const int m2 = pw_split(m);
    st_off[sp] = o + m2;  // right half below the left so the left pops first
    st_n[sp++] = m - m2;
    st_off[sp] = o;
    st_n[sp++] = m2;
  }
  return L;
}

// add the leaf sums back up the split tree of an n-term row: post-order walk
// with an explicit stack of (length, state, left value)
__device__ double pw_combine(int n, const double* sums) {
  int st_n[kPwDepth], st_s[kPwDepth], sp = 0, li = 0;
  double st_v[kPwDepth];
  st_n[sp] = n;
  st_s[sp++] = 0;
  double v = 0.0;
  bool have = false;  // v holds a finished subtree value to hand to the parent
  while (true) {
    if (!have) {
      const int m = st_n[sp - 1];
      if (m <= 128) {
        v = sums[li++];
        --sp;
        have = true;
      } else {  // descend into the left half
        st_n[sp] = pw_split(m);
        st_s[sp++] = 0;
      }
      continue;
    }
    if (sp == 0) return v;
    int& state = st_s[sp - 1];
    if (state == 0) {  // left done: keep it, descend into the right half
      st_v[sp - 1] = v;
      state = 1;
      const int m = st_n[sp - 1];
      st_n[sp] = m - pw_split(m);
      st_s[sp++] = 0;
      have = false;
    } else {  // both halves done
      v = st_v[sp - 1] + v;
      --sp;
    }
  }
}

// one leaf (8 <= n <= 128) by the 8-lane group of this lane; every lane of the
// group returns the leaf sum.  All 32 lanes must call it (butterfly shuffles).
__device__ __forceinline__ double pw_leaf(const int32_t* __restrict__ a, int n, const int32_t* __restrict__ indeg,
                                          bool valid) {
  const int j = threadIdx.x & 7;
  const int full = n - (n & 7);
  int32_t u[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int i = j + 8 * t;
    u[t] = valid && i < full ? __ldg(a + i) : -1;
  }
  double r = 0.0;
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    if (u[t] >= 0) {
      const double x = is_term(indeg, u[t]);
      r = t == 0 ? x : r + x;
    }
  }
  // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)): IEEE addition commutes, so the butterfly is exact
  r += __shfl_xor_sync(0xffffffffu, r, 1);
  r += __shfl_xor_sync(0xffffffffu, r, 2);
  r += __shfl_xor_sync(0xffffffffu, r, 4);
  if (valid)
    for (int i = full; i < n; ++i) r += is_term(indeg, __ldg(a + i));
  return r;
}

// pairwise sum of a row of at most kPwChunk terms (warp-uniform n)
__device__ double pw_chunk(const int32_t* __restrict__ a, int n, const int32_t* __restrict__ indeg, int* starts,
                           double* sums) {
  const int lane = threadIdx.x & 31;
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += is_term(indeg, __ldg(a + i));
    return r;
  }
  if (n <= 128) return pw_leaf(a, n, indeg, true);
  int L = 0;
  if (lane == 0) L = pw_leaves(n, starts);
  L = __shfl_sync(0xffffffffu, L, 0);
  __syncwarp();
  const int g = lane >> 3;
  for (int l0 = 0; l0 < L; l0 += 4) {
    const int li = l0 + g;
    const bool valid = li < L;
    const int st = valid ? starts[li] : 0;
    const int len = valid ? (li + 1 < L ? starts[li + 1] : n) - st : 8;
    const double v = pw_leaf(a + st, len, indeg, valid);
    if (valid && (lane & 7) == 0) sums[li] = v;
  }
  __syncwarp();
  double r = 0.0;
  if (lane == 0) r = pw_combine(n, sums);
  __syncwarp();
  return __shfl_sync(0xffffffffu, r, 0);
}

// pairwise sum of any row: the top of the split tree (halves above kPwChunk)
// walked warp-uniformly with an explicit stack, chunks summed by pw_chunk
__device__ double pw_row(const int32_t* __restrict__ a, int64_t n, const int32_t* __restrict__ indeg, int* starts,
                         double* sums) {
  if (n <= kPwChunk) return pw_chunk(a, (int)n, indeg, starts, sums);
  int64_t st_off[kPwDepth], st_n[kPwDepth];
  int st_s[kPwDepth], sp = 0;
  double st_v[kPwDepth];
  st_off[sp] = 0;
  st_n[sp] = n;
  st_s[sp++] = 0;
  double v = 0.0;
  bool have = false;
  while (true) {
    if (!have) {
      const int64_t m = st_n[sp - 1], o = st_off[sp - 1];
      if (m <= kPwChunk) {
        v = pw_chunk(a + o, (int)m, indeg, starts, sums);
        --sp;
        have = true;
      } else {
        int64_t m2 = m / 2;
        m2 -= m2 % 8;
        st_off[sp] = o;
        st_n[sp] = m2;
        st_s[sp++] = 0;
      }
      continue;
    }
    if (sp == 0) return v;
    if (st_s[sp - 1] == 0) {
      st_v[sp - 1] = v;
      st_s[sp - 1] = 1;
      const int64_t m = st_n[sp - 1], o = st_off[sp - 1];
      int64_t m2 = m / 2;
      m2 -= m2 % 8;
      st_off[sp] = o + m2;
      st_n[sp] = m - m2;
      st_s[sp++] = 0;
      have = false;
    } else {
      v = st_v[sp - 1] + v;
      --sp;
    }
  }
}

// IS numerators depend only on the training graph (and a partition's source
// split), so they are computed once per graph for every node and gathered per
// request.  Rows up to kPwChunk terms: a warp each; longer rows are queued for
// k_is_big, where a CTA's warps sum the top-level chunks and one thread adds
// them back up the split tree.
__global__ void __launch_bounds__(32 * kIsWarps) k_is_rows(int64_t N, const int64_t* __restrict__ off,
                                                           const int32_t* __restrict__ src,
                                                           const int32_t* __restrict__ indeg, double* out,
                                                           int32_t* big, int32_t* nbig) {
  pdl_wait();
  __shared__ int starts[kIsWarps][kPwLeafCap];
  __shared__ double sums[kIsWarps][kPwLeafCap];
  const int wid = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < N; v += nw) {
    const int64_t b = off[v], n = off[v + 1] - b;
    if (n > kPwChunk) {
      if ((threadIdx.x & 31) == 0) big[atomicAdd(nbig, 1)] = (int32_t)v;
      continue;
    }
    const double r = pw_chunk(src + b, (int)n, indeg, starts[wid], sums[wid]);
    if ((threadIdx.x & 31) == 0) out[v] = r;
  }
}

constexpr int kIsBigChunks = 1024;  // rows up to 1024 top-level chunks (~16.7M terms)

__global__ void __launch_bounds__(32 * kIsWarps) k_is_big(const int32_t* __restrict__ big, const int32_t* nbig,
                                                          const int64_t* __restrict__ off,
                                                          const int32_t* __restrict__ src,
                                                          const int32_t* __restrict__ indeg, double* out) {
  pdl_wait();
  __shared__ int starts[kIsWarps][kPwLeafCap];
  __shared__ double sums[kIsWarps][kPwLeafCap];
  __shared__ int64_t c_off[kIsBigChunks];
  __shared__ int c_len[kIsBigChunks];
  __shared__ double c_val[kIsBigChunks];
  __shared__ int nchunks;
  const int wid = threadIdx.x >> 5;
  for (int bi = blockIdx.x; bi < *nbig; bi += gridDim.x) {
    const int32_t v = big[bi];
    const int64_t b = off[v], n = off[v + 1] - b;
    if (threadIdx.x == 0) {  // top-level chunks of the split tree, left to right
      int64_t st_off[kPwDepth], st_n[kPwDepth];
      int sp = 0, L = 0;
      st_off[sp] = 0;
      st_n[sp++] = n;
      while (sp) {
        --sp;
        const int64_t o = st_off[sp], m = st_n[sp];
        if (m <= kPwChunk) {
          if (L < kIsBigChunks) {
            c_off[L] = o;
            c_len[L] = (int)m;
          }
          ++L;
          continue;
        }
        int64_t m2 = m / 2;
        m2 -= m2 % 8;
        st_off[sp] = o + m2;
        st_n[sp++] = m - m2;
        st_off[sp] = o;
        st_n[sp++] = m2;
      }
      nchunks = L;
    }
    __syncthreads();
    const int L = min(nchunks, kIsBigChunks);
    for (int c = wid; c < L; c += kIsWarps) {
      const double r = pw_chunk(src + b + c_off[c], c_len[c], indeg, starts[wid], sums[wid]);
      if ((threadIdx.x & 31) == 0) c_val[c] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // add the chunk sums back up the same tree (post-order)
      int64_t st_n[kPwDepth];
      int st_s[kPwDepth], sp = 0, li = 0;
      double st_v[kPwDepth];
      st_n[sp] = n;
      st_s[sp++] = 0;
      double val = 0.0;
      bool have = false;
      while (true) {
        if (!have) {
          const int64_t m = st_n[sp - 1];
          if (m <= kPwChunk) {
            val = c_val[li++];
            --sp;
            have = true;
          } else {
            int64_t m2 = m / 2;
            m2 -= m2 % 8;
            st_n[sp] = m2;
            st_s[sp++] = 0;
          }
          continue;
        }
        if (sp == 0) break;
        if (st_s[sp - 1] == 0) {
          st_v[sp - 1] = val;
          st_s[sp - 1] = 1;
          const int64_t m = st_n[sp - 1];
          int64_t m2 = m / 2;
          m2 -= m2 % 8;
          st_n[sp] = m - m2;
          st_s[sp++] = 0;
          have = false;
        } else {
          val = st_v[sp - 1] + val;
          --sp;
        }
      }
      out[v] = nchunks <= kIsBigChunks ? val : __longlong_as_double(0x7FF8000000000000ll);  // NaN: too long
    }
    __syncthreads();
  }
}

// numerator table of one CSR (the whole graph, or a partition's source split) over all N nodes
void build_is_table(Engine& e, const int64_t* off, const int32_t* src, double* out) {
  cudaStream_t s = e.stream;
  const int64_t N = e.g.N;
  int32_t* big = (int32_t*)e.dalloc(sizeof(int32_t) * (N + 1));
  int32_t* nbig = (int32_t*)e.dalloc(sizeof(int32_t));
  OB_CUDA(cudaMemsetAsync(nbig, 0, sizeof(int32_t), s));
  launch_pdl(k_is_rows, dim3(grid_for(N, kIsWarps, kNumSMs * 8)), dim3(32 * kIsWarps), 0, s, N, off, src, e.g.indeg, out, big, nbig);
  launch_pdl(k_is_big, dim3(kNumSMs), dim3(32 * kIsWarps), 0, s, big, nbig, off, src, e.g.indeg, out);
  OB_CUDA(cudaStreamSynchronize(s));
  e.dfree(big);
  e.dfree(nbig);
}

__global__ void k_is_gather(const int32_t* __restrict__ cand_ids, const ReqCounters* rc,
                            const double* __restrict__ tab, double* out) {
  pdl_wait();
  const int64_t R = cta_ld(&rc->R);
  OB_GRID_STRIDE(c, R) out[c] = tab[cand_ids[c]];
}

void launch_is_gather(Engine& e, RequestWs& w, const double* tab, double* out) {
  const int64_t r_max = std::min<int64_t>(e.g.N, 2 * w.m);
  launch_pdl(k_is_gather, dim3(grid_for(r_max, 256)), dim3(256), 0, e.stream, w.cand_ids, w.rc, tab, out);
}

// scores from P partial arrays, summed in rank order (P = 1: the centralized row sum)
__global__ void k_score_is(const int32_t* __restrict__ cand_ids, const int32_t* __restrict__ indeg,
                           const ReqCounters* rc, IsParts parts, double* score, uint64_t* key) {
  pdl_wait();
  const int64_t R = cta_ld(&rc->R);
  OB_GRID_STRIDE(c, R) {
    double sum = 0.0;
    for (int p = 0; p < parts.P; ++p) sum += __ldcg(parts.part[p] + c);
    const int32_t d = indeg[cand_ids[c]];
    const double s = d > 0 ? sum / (double)d : 0.0;
    score[c] = s;
    key[c] = (uint64_t)__double_as_longlong(s);
  }
}

void launch_score_is(Engine& e, RequestWs& w, const IsParts& parts) {
  const int64_t r_max = std::min<int64_t>(e.g.N, 2 * w.m);
  launch_pdl(k_score_is, dim3(grid_for(r_max, 256)), dim3(256), 0, e.stream, w.cand_ids, e.g.indeg, w.rc, parts, w.cand_score,
                                                         w.cand_key);
}

__global__ void k_budget(ReqCounters* rc, double gamma, uint32_t* hist) {
  pdl_wait();
  // budget = int(np.floor(gamma * m)) with gamma a Python float: one IEEE fp64 multiply
  const int64_t R = cta_ld(&rc->R);
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
  if (threadIdx.x == 0) hist[256] = 0;
}

// One radix-select round in one launch: per-CTA digit histograms of the keys that
// still match the chosen prefix are merged into hist; the last CTA to finish
// picks this round's digit (scan from the top digit) and clears hist.
__global__ void __launch_bounds__(256) k_sel_round(const uint64_t* __restrict__ key, ReqCounters* rc, int shift,
                                                   uint32_t* hist) {
  pdl_wait();
  using BS = cub::BlockScan<int64_t, 256>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t h[256];
  __shared__ bool last;
  h[threadIdx.x] = 0;
  __syncthreads();
  const CtaWords st = cta_ldv(&rc->R, &rc->budget, &rc->sel_prefix, &rc->sel_mask);
  const int64_t R = st.v[0], b = st.v[1];
  const bool active = b > 0 && b < R;
  if (active) {
    const uint64_t pre = (uint64_t)st.v[2], msk = (uint64_t)st.v[3];
    OB_GRID_STRIDE(c, R) {
      const uint64_t k = key[c];
      if ((k & msk) == pre) atomicAdd(&h[(k >> shift) & 255], 1u);
    }
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(hist + threadIdx.x, h[threadIdx.x]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(hist + 256, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int d = 255 - threadIdx.x;  // scan from the top digit down
  const int64_t c = __ldcg(hist + d);
  int64_t excl;
  BS(tmp).ExclusiveSum(c, excl);  // keys in digits above d
  hist[d] = 0;
  if (threadIdx.x == 0) hist[256] = 0;
  if (!active) return;
  const int64_t krem = ld_state(&rc->sel_krem);
  if (excl < krem && krem <= excl + c) {
    rc->sel_krem = krem - excl;
    rc->sel_gt = ld_state(&rc->sel_gt) + excl;
    rc->sel_prefix = ld_state(&rc->sel_prefix) | ((uint64_t)d << shift);
    rc->sel_mask = ld_state(&rc->sel_mask) | ((uint64_t)255 << shift);
    if (shift == 0) rc->sel_eq_take = krem - excl;
  }
}

// Ordered compaction of the selection in one scan over (above-threshold,
// at-threshold) counts: candidate c is selected when its key is above the
// threshold, or equal to it with fewer than eq_take equal keys before it (ties
// go to the lowest ids, policy.py:131); its target position is then
// (# above before c) + min(# equal before c, eq_take).
struct SelLoad {
  const uint64_t* key;
  const ReqCounters* rc;
  int64_t R = 0, b = 0;  // cached by prepare() (once per thread, after pdl_wait)
  uint64_t thr = 0;
  __device__ void prepare() {
    const CtaWords st = cta_ldv(&rc->R, &rc->budget, &rc->sel_prefix);
    R = st.v[0];
    b = st.v[1];
    thr = (uint64_t)st.v[2];
  }
  __device__ I3 operator()(int64_t c) const {
    if (b <= 0) return I3(0);
    if (b >= R) return I3(1, 0, 0);
    const uint64_t k = key[c];
    return I3(k > thr ? 1 : 0, k == thr ? 1 : 0, 0);
  }
};
struct SelStore3 {
  SelLoad ld;
  const int32_t* cand_ids;
  int32_t* targets;
  int32_t* tpos;
  int64_t take = 0;
  __device__ void prepare() {
    const CtaWords st = cta_ldv(&ld.rc->R, &ld.rc->budget, &ld.rc->sel_prefix, &ld.rc->sel_eq_take);
    ld.R = st.v[0];
    ld.b = st.v[1];
    ld.thr = (uint64_t)st.v[2];
    take = st.v[3];
  }
  __device__ void operator()(int64_t c, const I3& pre) const {
    const I3 me = ld(c);
    if (me.a || (me.b && pre.b < take)) {
      const int64_t pos = pre.a + (pre.b < take ? pre.b : take);
      targets[pos] = cand_ids[c];
      tpos[c] = (int32_t)pos;
    }
  }
};
struct SelTotal {
  ReqCounters* rc;
  __device__ void operator()(int64_t, const I3& t) const {
    const int64_t take = ld_state(&rc->sel_eq_take);
    rc->T = t.a + (t.b < take ? t.b : take);
  }
};

// ---------------------------------------------------------------------------
// 2d. The whole top-k in one launch of one 16-CTA thread-block cluster: the budget
// (policy.py:127), the eight 8-bit radix-select rounds over the fp64 score bits and
// the ordered compaction (ties to the lowest ids, policy.py:131).  Each CTA keeps its
// contiguous chunk of the keys in shared memory; a round's digit histograms are summed
// across the cluster through distributed shared memory (every CTA reads all 16 and
// takes the same decision), one cluster barrier per round.  Replaces k_budget, the
// eight k_sel_round launches and the compaction scan whenever |R| fits the cluster's
// shared memory (16 x 24576 keys).
// ---------------------------------------------------------------------------
constexpr int kSelCl = 16;
constexpr int kSelClThreads = 512;
constexpr int kSelClKeys = 24576;  // keys per CTA (192 KB of shared memory)
constexpr int64_t kSelClSoloEdges = 1 << 18;  // single-lane engines: requests up to this many edges

__global__ void __launch_bounds__(kSelClThreads, 1)
    k_select_cluster(const uint64_t* __restrict__ key, const int32_t* __restrict__ cand_ids, ReqCounters* rc,
                     double gamma, int32_t* targets, int32_t* tpos) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  using Scan = cub::BlockScan<unsigned long long, kSelClThreads>;
  using Red = cub::BlockReduce<unsigned long long, kSelClThreads>;
  extern __shared__ uint64_t sk[];
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Red::TempStorage red;
  } tmp;
  __shared__ uint32_t hist[2][256];
  __shared__ int64_t wsum[8];
  __shared__ uint64_t s_pre, s_msk;
  __shared__ int64_t s_krem, s_take;
  __shared__ unsigned long long s_tot;  // this CTA's (above << 32 | equal) counts
  pdl_wait();
  const int t = threadIdx.x, lane = t & 31;
  const int64_t R = cta_ld(&rc->R);
  const int64_t b = (int64_t)floor(gamma * (double)R);  // int(np.floor(gamma * m)): one fp64 multiply
  const int rank = (int)cl.block_rank();
  const int64_t chunk = (R + kSelCl - 1) / kSelCl;
  const int64_t c0 = min(R, (int64_t)rank * chunk), c1 = min(R, c0 + chunk);
  const int n = (int)(c1 - c0);
  for (int i = t; i < n; i += kSelClThreads) sk[i] = key[c0 + i];
  if (t < 256) hist[0][t] = hist[1][t] = 0;
  if (t == 0) {
    s_pre = 0;
    s_msk = 0;
    s_krem = b;
    s_take = 0;
  }
  __syncthreads();
  const bool active = b > 0 && b < R;
  if (active) {
    for (int r = 0; r < 8; ++r) {
      const int shift = 56 - 8 * r, buf = r & 1;
      const uint64_t pre = s_pre, msk = s_msk;
      for (int base = 0; base < n; base += kSelClThreads) {  // warp-uniform trip count
        const int i = base + t;
        const uint64_t k = i < n ? sk[i] : 0;
        const bool in = i < n && (k & msk) == pre;
        const int d = (int)((k >> shift) & 255);
        const unsigned peers = __match_any_sync(0xffffffffu, in ? d : 256 + lane);
        if (in && lane == __ffs(peers) - 1) atomicAdd(&hist[buf][d], (uint32_t)__popc(peers));
      }
      cl.sync();  // every CTA's histogram of this round is complete and visible
      int64_t c = 0, incl = 0;
      if (t < 256) {
        const int d = 255 - t;  // scan from the top digit down
        for (int q = 0; q < kSelCl; ++q) c += cl.map_shared_rank(&hist[buf][0], q)[d];
        incl = c;
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[t >> 5] = incl;
      }
      if (t < 256) hist[buf ^ 1][t] = 0;  // the next round's buffer (its last readers passed this barrier)
      __syncthreads();
      if (t < 256) {
        int64_t excl = incl - c;
        for (int wq = 0; wq < (t >> 5); ++wq) excl += wsum[wq];
        const int64_t krem = s_krem;
        if (excl < krem && krem <= excl + c) {
          const int d = 255 - t;
          s_pre = pre | ((uint64_t)d << shift);
          s_msk = msk | ((uint64_t)255 << shift);
          s_krem = krem - excl;
          if (shift == 0) s_take = krem - excl;
        }
      }
      __syncthreads();
    }
  }
  // ordered compaction: c is selected when above the threshold, or equal to it with fewer
  // than take equal keys before it; its position is (# above before) + min(# equal before, take)
  const uint64_t thr = s_pre;
  const int64_t take = s_take;
  auto flags = [&](int i) -> unsigned long long {
    if (i >= n || b <= 0) return 0ull;
    if (b >= R) return 1ull << 32;
    const uint64_t k = sk[i];
    return k > thr ? (1ull << 32) : (k == thr ? 1ull : 0ull);
  };
  unsigned long long mine = 0;
  for (int i = t; i < n; i += kSelClThreads) mine += flags(i);
  const unsigned long long tot = Red(tmp.red).Sum(mine);
  if (t == 0) s_tot = tot;
  cl.sync();  // every CTA's totals are visible
  unsigned long long basep = 0, allp = 0;
  if (t == 0) {
    for (int q = 0; q < kSelCl; ++q) {
      const unsigned long long v = *cl.map_shared_rank(&s_tot, q);
      if (q < rank) basep += v;
      allp += v;
    }
    if (rank == 0) {
      const int64_t above = (int64_t)(allp >> 32), eq = (int64_t)(allp & 0xffffffffu);
      rc->budget = b;
      rc->sel_prefix = thr;
      rc->sel_eq_take = take;
      rc->T = above + (eq < take ? eq : take);
    }
  }
  cl.sync();  // every remote read of s_tot is done before it is reused (and before any CTA exits)
  if (t == 0) s_tot = basep;  // this CTA's base counts
  __syncthreads();
  unsigned long long run = s_tot;
  for (int base = 0; base < n; base += kSelClThreads) {
    const int i = base + t;
    const unsigned long long f = flags(i);
    unsigned long long ex, tile;
    Scan(tmp.scan).ExclusiveSum(f, ex, tile);
    const unsigned long long p = run + ex;
    const int64_t above_b = (int64_t)(p >> 32), eq_b = (int64_t)(p & 0xffffffffu);
    const bool sel = (f >> 32) || ((f & 1ull) && eq_b < take);
    if (sel) {
      const int64_t pos = above_b + (eq_b < take ? eq_b : take);
      targets[pos] = cand_ids[c0 + i];
      tpos[c0 + i] = (int32_t)pos;
    }
    run += tile;
    __syncthreads();  // tmp.scan reuse
  }
}

static bool select_cluster_ok() {
  static const bool ok = [] {
    const char* v = std::getenv("OB_NO_CLUSTER_SELECT");
    if (v && v[0] && v[0] != '0') return false;
    if (cudaFuncSetAttribute(k_select_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        cudaFuncSetAttribute(k_select_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kSelClKeys * sizeof(uint64_t))) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return true;
  }();
  return ok;
}

static void launch_select_cluster(cudaStream_t s, const uint64_t* key, const int32_t* cand_ids, ReqCounters* rc,
                                  double gamma, int32_t* targets, int32_t* tpos) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kSelCl);
  cfg.blockDim = dim3(kSelClThreads);
  cfg.dynamicSmemBytes = kSelClKeys * sizeof(uint64_t);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kSelCl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1 + launch_attrs(at + 1);
  OB_CUDA(cudaLaunchKernelEx(&cfg, k_select_cluster, key, cand_ids, rc, gamma, targets, tpos));
  OB_LAUNCHED();
}

// ---------------------------------------------------------------------------
// 3. request CSR order: stable LSD radix sort of the packed keys, 8-bit digits,
//    4096-key tiles.  Per pass: digit counts per tile (digit-major), one scan,
//    then a stable scatter -- keys are ranked inside the tile warp by warp
//    (match_any over the digit, items in index order), exchanged through shared
//    memory into tile order and written out in coalesced runs.  The last pass
//    writes the decoded source ids straight into the CSR.
// ---------------------------------------------------------------------------
constexpr int kRxThreads = 512;
#ifndef OB_RX_MINB
#define OB_RX_MINB 2  // scatter CTAs resident per SM (caps registers at 64)
#endif
constexpr int kRxWarps = kRxThreads / 32;
constexpr int kRxItems = kRxTile / kRxThreads;  // 8 keys per thread, warp-striped

template <class K>
__global__ void __launch_bounds__(kRxThreads) k_rx_hist(const K* __restrict__ keys, const int64_t* m_dev, int shift,
                                                        int64_t tiles_b, int32_t* cnt) {
  pdl_wait();
  __shared__ int32_t h[256];
  const int64_t m = cta_ld(m_dev);
  const int64_t tiles = (m + kRxTile - 1) / kRxTile;
  for (int64_t t = blockIdx.x; t < tiles_b; t += gridDim.x) {
    if (threadIdx.x < 256) h[threadIdx.x] = 0;
    __syncthreads();
    if (t < tiles) {
      const int64_t e1 = min((t + 1) * kRxTile, m);
      for (int64_t e = t * kRxTile + threadIdx.x; e < e1; e += kRxThreads) atomicAdd(&h[(keys[e] >> shift) & 255], 1);
    }
    __syncthreads();
    if (threadIdx.x < 256) cnt[(int64_t)threadIdx.x * tiles_b + t] = h[threadIdx.x];
    __syncthreads();
  }
}

// one-sweep: every pass's digit totals from one read of the keys ([pass][256])
template <class K>
__global__ void __launch_bounds__(kRxThreads) k_rx_ghist(const K* __restrict__ keys, const int64_t* m_dev, int passes,
                                                         uint32_t* ghist) {
  pdl_wait();
  __shared__ uint32_t h[8 * 256];
  for (int i = threadIdx.x; i < passes * 256; i += kRxThreads) h[i] = 0;
  __syncthreads();
  const int64_t m = cta_ld(m_dev);
  OB_GRID_STRIDE(e, m) {
    const K k = keys[e];
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p * 256 + (int)((k >> (8 * p)) & 255)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += kRxThreads)
    if (h[i]) atomicAdd(ghist + i, h[i]);
}

// Digit d's tile counts -> their exclusive prefix over tiles (row d of the digit-major
// count matrix) and the digit's total; one CTA per digit.  The scatter adds the
// exclusive prefix over digit totals, so no grid-wide scan is needed between passes.
constexpr int kRowScanThreads = 256;
__global__ void __launch_bounds__(kRowScanThreads) k_rx_rowscan(const int32_t* __restrict__ cnt, int64_t tiles_b,
                                                               int64_t* off, int64_t* dtot) {
  pdl_wait();
  using BS = cub::BlockScan<int64_t, kRowScanThreads>;
  __shared__ typename BS::TempStorage tmp;
  const int d = blockIdx.x;
  const int32_t* row = cnt + (int64_t)d * tiles_b;
  int64_t carry = 0;
  for (int64_t t0 = 0; t0 < tiles_b; t0 += kRowScanThreads) {
    const int64_t t = t0 + threadIdx.x;
    const int64_t v = t < tiles_b ? row[t] : 0;
    int64_t x, agg;
    BS(tmp).ExclusiveSum(v, x, agg);
    __syncthreads();
    if (t < tiles_b) off[(int64_t)d * tiles_b + t] = carry + x;
    carry += agg;
  }
  if (threadIdx.x == 0) dtot[d] = carry;
}

// look-back word: flag in the top two bits (1 tile count, 2 inclusive prefix), count below
constexpr uint32_t kRxAgg = 1u << 30, kRxInc = 2u << 30, kRxCount = kRxAgg - 1u;

template <class K, bool FINAL>
__global__ void __launch_bounds__(kRxThreads, OB_RX_MINB) k_rx_scatter(const K* __restrict__ in, K* out, int32_t* src_out,
                                                           const int64_t* m_dev, int shift, int64_t tiles_b,
                                                           const int64_t* __restrict__ off,
                                                           const int32_t* __restrict__ cnt, RqKeyFmt f, int64_t N,
                                                           const int32_t* __restrict__ cand_ids,
                                                           const ReqCounters* rc, uint32_t* st, uint32_t* ticket,
                                                           const uint32_t* __restrict__ ghist,
                                                           const int64_t* __restrict__ dtot) {
  pdl_wait();
  using BS = cub::BlockScan<int32_t, kRxThreads>;
  using BS64 = cub::BlockScan<int64_t, kRxThreads>;
  __shared__ typename BS64::TempStorage scan_tmp64;
  __shared__ union {
    int32_t wcnt[kRxWarps][256];  // per-warp digit counts, then per-warp offsets
    K exch[kRxTile];              // the tile in (digit, index) order
  } u;
  __shared__ typename BS::TempStorage scan_tmp;
  __shared__ int32_t bstart[256];
  __shared__ int64_t gofs[256];
  __shared__ int64_t gbase[256];  // one-sweep: keys of smaller digits (whole input)
  __shared__ int64_t s_t;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t m = cta_ld(m_dev);
  const int64_t tiles = (m + kRxTile - 1) / kRxTile;
  if (st || dtot) {  // keys of smaller digits: one-sweep totals, or the row scans' digit totals
    int64_t g = threadIdx.x < 256 ? (st ? (int64_t)ghist[threadIdx.x] : dtot[threadIdx.x]) : 0, gx;
    BS64(scan_tmp64).ExclusiveSum(g, gx);
    if (threadIdx.x < 256) gbase[threadIdx.x] = gx;
  }
  for (int64_t t = blockIdx.x;; t += gridDim.x) {
    // one-sweep tiles come from a ticket, so every look-back target is already running
    if (st) {
      if (threadIdx.x == 0) s_t = (int64_t)atomicAdd(ticket, 1u);
      __syncthreads();
      t = s_t;
    }
    if (t >= tiles) break;
    for (int i = threadIdx.x; i < kRxWarps * 256; i += kRxThreads) (&u.wcnt[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = t * kRxTile + warp * 256;
    K k[kRxItems];
    int dg[kRxItems], rk[kRxItems];
#pragma unroll
    for (int i = 0; i < kRxItems; ++i) {
      const int64_t idx = base + i * 32 + lane;
      k[i] = idx < m ? in[idx] : (K)0;
      dg[i] = idx < m ? (int)((k[i] >> shift) & 255) : 256 + lane;  // padding never matches
    }
#pragma unroll
    for (int i = 0; i < kRxItems; ++i) {
      const unsigned peers = __match_any_sync(0xffffffffu, dg[i]);
      const int leader = __ffs(peers) - 1;
      int b0 = 0;
      if (lane == leader && dg[i] < 256) {
        b0 = u.wcnt[warp][dg[i]];
        u.wcnt[warp][dg[i]] = b0 + __popc(peers);
      }
      rk[i] = __shfl_sync(0xffffffffu, b0, leader) + __popc(peers & lt);
      __syncwarp();
    }
    __syncthreads();
    int32_t tot = 0;
    if (threadIdx.x < 256) {  // per digit: warps' exclusive offsets, tile total
      for (int w2 = 0; w2 < kRxWarps; ++w2) {
        const int32_t c = u.wcnt[w2][threadIdx.x];
        u.wcnt[w2][threadIdx.x] = tot;
        tot += c;
      }
    }
    int32_t start;
    BS(scan_tmp).ExclusiveSum(tot, start);
    if (st) {
      if (threadIdx.x < 256) {  // publish this tile's digit count, then look back for the prefix
        const int d = threadIdx.x;
        volatile uint32_t* vs = st;
        vs[t * 256 + d] = (t == 0 ? kRxInc : kRxAgg) | (uint32_t)tot;
        uint32_t excl = 0;
        if (t > 0) {
          for (int64_t j = t - 1;; --j) {
            uint32_t v;
            do v = vs[j * 256 + d];
            while ((v & ~kRxCount) == 0);
            excl += v & kRxCount;
            if (v & kRxInc) break;
          }
          vs[t * 256 + d] = kRxInc | (excl + (uint32_t)tot);
        }
        bstart[d] = start;
        gofs[d] = gbase[d] + excl;
      }
    } else if (off) {
      if (threadIdx.x < 256) {
        bstart[threadIdx.x] = start;
        gofs[threadIdx.x] = gbase[threadIdx.x] + off[(int64_t)threadIdx.x * tiles_b + t];
      }
    } else {
      // few tiles: derive this tile's global digit offsets from the raw counts
      // (digit d starts after every key of smaller digits, then after digit d's
      // keys in earlier tiles) instead of a separate grid-wide scan
      int64_t dtot = 0, before = 0;
      if (threadIdx.x < 256)
        for (int64_t t2 = 0; t2 < tiles_b; ++t2) {
          const int64_t c = cnt[(int64_t)threadIdx.x * tiles_b + t2];
          dtot += c;
          if (t2 < t) before += c;
        }
      __syncthreads();  // scan_tmp reuse
      int64_t dstart;
      BS64(scan_tmp64).ExclusiveSum(dtot, dstart);
      if (threadIdx.x < 256) {
        bstart[threadIdx.x] = start;
        gofs[threadIdx.x] = dstart + before;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRxItems; ++i)
      if (dg[i] < 256) rk[i] += bstart[dg[i]] + u.wcnt[warp][dg[i]];
    __syncthreads();  // offsets read before the exchange overwrites them
#pragma unroll
    for (int i = 0; i < kRxItems; ++i)
      if (dg[i] < 256) u.exch[rk[i]] = k[i];
    __syncthreads();
    const int n = (int)min((int64_t)kRxTile, m - t * kRxTile);
    const int64_t R_fin = FINAL ? ld_state(&rc->R) : 0;  // query-slot source codes >= R are queries
    for (int p = threadIdx.x; p < n; p += kRxThreads) {
      const K kk = u.exch[p];
      const int d = (int)((kk >> shift) & 255);
      const int64_t pos = gofs[d] + (p - bstart[d]);
      if (FINAL) {
        const bool query_slot = (kk >> f.body) & 1;
        if (query_slot) {
          const int64_t sr = (int64_t)(kk & (((K)1 << f.bN) - 1));
          src_out[pos] = sr < R_fin ? cand_ids[sr] : (int32_t)(N + (sr - R_fin));
        } else {
          src_out[pos] = (int32_t)(N + (kk & (((K)1 << f.bB) - 1)));
        }
      } else {
        out[pos] = kk;
      }
    }
    __syncthreads();
  }
}

#ifndef OB_RX_ONESWEEP
#define OB_RX_ONESWEEP 0  // measured: cfg2 p50 +2 % (look-back spins contend with the side stream), cfg1/cfg3 ±1 %
#endif

template <class K>
static void rx_sort(Engine& e, RequestWs& w, RqCsr& c, const int64_t* m_dev, int64_t m_bound, const RqKeyFmt& f) {
  cudaStream_t s = e.stream;
  const int64_t tiles_b = rx_tiles(m_bound);
  const int g = grid_for(tiles_b, 1, kNumSMs * (OB_RX_MINB > 2 ? OB_RX_MINB : 2));
  K* a = reinterpret_cast<K*>(c.keys);
  K* b = reinterpret_cast<K*>(c.keys2);
  const int passes = f.passes();
  // OB_RX_ONESWEEP in the environment overrides the build default (read per sort;
  // a captured request graph keeps the path it was captured with)
  const char* os_env = std::getenv("OB_RX_ONESWEEP");
  const bool onesweep = os_env ? std::atoi(os_env) != 0 : OB_RX_ONESWEEP != 0;
  if (onesweep && c.rx_st && m_bound < (int64_t)kRxCount) {
    // one sweep per pass: digit totals for every pass from one read, then each
    // scatter tile publishes its digit counts and looks back for its offsets
    uint32_t* st = c.rx_st;
    uint32_t* ticket = st + 8 * 256 * tiles_b;
    uint32_t* ghist = ticket + 8;
    OB_CUDA(cudaMemsetAsync(st, 0, sizeof(uint32_t) * rx_st_words(m_bound), s));
    launch_pdl(k_rx_ghist<K>, dim3(grid_for(m_bound, kRxThreads * 8, kNumSMs * 2)), dim3(kRxThreads), 0, s, a, m_dev, passes, ghist);
    for (int p = 0; p < passes; ++p) {
      const int shift = 8 * p;
      uint32_t* sp = st + (int64_t)p * 256 * tiles_b;
      if (p + 1 == passes) {
        launch_pdl(k_rx_scatter<K, true>, dim3(g), dim3(kRxThreads), 0, s, a, nullptr, c.src, m_dev, shift, tiles_b, nullptr, c.rx_cnt, f,
                                                        e.g.N, w.cand_ids, w.rc, sp, ticket + p, ghist + 256 * p, nullptr);
      } else {
        launch_pdl(k_rx_scatter<K, false>, dim3(g), dim3(kRxThreads), 0, s, a, b, nullptr, m_dev, shift, tiles_b, nullptr, c.rx_cnt, f,
                                                         e.g.N, w.cand_ids, w.rc, sp, ticket + p, ghist + 256 * p, nullptr);
        std::swap(a, b);
      }
      OB_LAUNCHED();
    }
    return;
  }
  const bool fused = tiles_b <= 32;  // few tiles: offsets come straight from the counts
  const int64_t* off = fused ? nullptr : c.rx_off;
  const int64_t* dtot = fused ? nullptr : c.rx_off + 256 * tiles_b;  // per-digit totals (row scans)
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    launch_pdl(k_rx_hist<K>, dim3(g), dim3(kRxThreads), 0, s, a, m_dev, shift, tiles_b, c.rx_cnt);
    if (!fused)  // each digit's tile counts scanned by its own CTA; the digit prefix is taken in the scatter
      launch_pdl(k_rx_rowscan, dim3(256), dim3(kRowScanThreads), 0, s, (const int32_t*)c.rx_cnt, tiles_b, c.rx_off,
                 c.rx_off + 256 * tiles_b);
    if (p + 1 == passes) {
      launch_pdl(k_rx_scatter<K, true>, dim3(g), dim3(kRxThreads), 0, s, a, nullptr, c.src, m_dev, shift, tiles_b, off, c.rx_cnt, f,
                                                      e.g.N, w.cand_ids, w.rc, nullptr, nullptr, nullptr, dtot);
    } else {
      launch_pdl(k_rx_scatter<K, false>, dim3(g), dim3(kRxThreads), 0, s, a, b, nullptr, m_dev, shift, tiles_b, off, c.rx_cnt, f,
                                                       e.g.N, w.cand_ids, w.rc, nullptr, nullptr, nullptr, dtot);
      std::swap(a, b);
    }
  }
}

static int bits_for(int64_t n) {  // bits to hold values in [0, n)
  int b = 1;
  while (b < 62 && ((int64_t)1 << b) < n) ++b;
  return b;
}

RqKeyFmt rq_key_fmt(const Engine& e, const RequestWs& w) {
  RqKeyFmt f;
  f.bB = bits_for(std::max(w.B, 1));
  f.bR = bits_for(std::max<int64_t>(1, std::min<int64_t>(e.g.N, 2 * w.m)));
  f.bN = bits_for(std::min<int64_t>(e.g.N, 2 * w.m) + w.B);  // query-slot sources by candidate rank
  f.body = std::max(f.bR + f.bB, f.bB + f.bN);
  f.total = f.body + 1;
  OB_CHECK(f.total <= 64, OB_EINVAL, "request key does not fit 64 bits");
  return f;
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
    launch_pdl(k_request_mark, dim3(grid_for(m, kEdgeTile, kNumSMs * 4)), dim3(256), sq, s, w.rp, N, w.B, w.cbits, w.qdeg, w.rc);
  }
  // candidate set: popcount prefix, ascending ids
  bitmap_rank(e, w.cbits, w.words_N, w.cwpre, w.cand_ids, &w.rc->R, w.c_gcnt, w.c_gpre);
  const int64_t rb_max = std::min<int64_t>(N, 2 * m) + w.B;
  launch_pdl(k_slots_init, dim3(grid_for(rb_max, 256)), dim3(256), 0, s, w.rc, w.B, w.qdeg, w.rq_cnt, w.rq_fill);
  if (m > 0) {  // candidate-slot counts + the request CSR's radix keys
    const RqKeyFmt f = rq_key_fmt(e, w);
    if (f.wide())
      launch_pdl(k_rq_count<uint64_t>, dim3(grid_for(m, 256)), dim3(256), 0, s, w.rp, N, w.cbits, w.cwpre, w.rc, w.rq_cnt, w.rq_keys, f);
    else
      launch_pdl(k_rq_count<uint32_t>, dim3(grid_for(m, 256)), dim3(256), 0, s, w.rp, N, w.cbits, w.cwpre, w.rc, w.rq_cnt,
                                                            reinterpret_cast<uint32_t*>(w.rq_keys), f);
  }
  (void)need_scores;
}

// the request's checks and scores: off the request-index sort's critical path
// (launched on the main stream after the fork; only the selection needs them)
void stage_request_post(Engine& e, RequestWs& w, bool need_scores) {
  cudaStream_t s = e.stream;
  const int64_t N = e.g.N;
  const int64_t m = w.m;
  if ((int64_t)w.B * e.g.F > 0) {
    launch_pdl(k_check_finite, dim3(grid_for((int64_t)w.B * e.g.F, 256)), dim3(256), 0, s, w.rp, (int64_t)w.B * e.g.F, w.rc);
  }
  if (need_scores) {
    const int64_t r_max = std::min<int64_t>(N, 2 * m);
    launch_pdl(k_score, dim3(grid_for(r_max, 256)), dim3(256), 0, s, w.cand_ids, w.rq_cnt, e.g.indeg, w.rc, w.cand_nq, w.cand_score,
                                                 w.cand_key, w.cand_tpos, e.cfg.policy == OB_POLICY_RATIO);
  }
}

static void select_random(Engine& e, RequestWs& w, int64_t r_max);  // RANDOM policy (below)

void stage_select(Engine& e, RequestWs& w) {
  cudaStream_t s = e.stream;
  const int64_t r_max = std::min<int64_t>(e.g.N, 2 * w.m);
  if (e.cfg.policy == OB_POLICY_IS && e.cfg.strategy != OB_STRATEGY_SRPE_CGP && r_max > 0) {
    // centralized importance scores over the whole training CSR (policy.py:84-95)
    launch_is_gather(e, w, e.is_tab[0], w.is_part);
    IsParts ip{};
    ip.P = 1;
    ip.part[0] = w.is_part;
    launch_score_is(e, w, ip);
  }
  // the cluster needs 16 SMs of one GPC at once: with one lane and a long request-index sort
  // on the side stream (whose CTAs fill the SMs) it waits for them (cfg2: p50 0.76 -> 0.80 ms),
  // so that case keeps the multi-launch rounds, which slot into whatever SMs free up
  static const int64_t solo_edges = [] {  // OB_SEL_CLUSTER_EDGES overrides the single-lane bound
    const char* v = std::getenv("OB_SEL_CLUSTER_EDGES");
    return v && v[0] ? std::atoll(v) : kSelClSoloEdges;
  }();
  const bool cluster = e.nlanes > 1 || w.m <= solo_edges;
  if (e.cfg.policy != OB_POLICY_RANDOM && cluster && r_max <= (int64_t)kSelCl * kSelClKeys && select_cluster_ok()) {
    launch_select_cluster(s, w.cand_key, w.cand_ids, w.rc, e.cfg.gamma, w.targets, w.cand_tpos);
    return;
  }
  launch_pdl(k_budget, dim3(1), dim3(256), 0, s, w.rc, e.cfg.gamma, w.sel_hist);
  if (e.cfg.policy == OB_POLICY_RANDOM) {
    // zero scores (runtime.py:182-183); the chosen ranks' keys are 1 against threshold 0
    OB_CUDA(cudaMemsetAsync(w.cand_score, 0, sizeof(double) * std::max<int64_t>(r_max, 1), s));
    select_random(e, w, r_max);
  }
  for (int shift = 56; shift >= 0 && e.cfg.policy != OB_POLICY_RANDOM; shift -= 8) {
    static const int sel_cap = [] {  // OB_SEL_GRID: CTAs per radix-select round (A/B)
      const char* v = std::getenv("OB_SEL_GRID");
      return v && v[0] ? std::max(1, std::atoi(v)) : kNumSMs * 2;
    }();
    launch_pdl(k_sel_round, dim3(grid_for(r_max, 256, sel_cap)), dim3(256), 0, s, w.cand_key, w.rc, shift, w.sel_hist);
  }
  // ordered compaction: ties at the threshold resolved by ascending id
  const SelLoad ld{w.cand_key, w.rc};
  device_scan_t<I3>(s, e.scan, ld, SelStore3{ld, w.cand_ids, w.targets, w.cand_tpos}, SelTotal{w.rc}, &w.rc->R, 0,
                    r_max);
}

// ---------------------------------------------------------------------------
// 2c. RANDOM policy (policy.py:122-124): order = default_rng(tie_seed).permutation(|R|),
//     targets = sort(ids[order[:budget]]).
//
// numpy's permutation is a Fisher-Yates shuffle of arange(R): for i = R-1 .. 1,
// j_i = random_interval(i) (masked rejection on the PCG64 stream's 32-bit draws, low
// half of each 64-bit output first), swap a[i], a[j_i].  The device never performs the
// swaps:
//   1. k_rnd_raw: the raw 32-bit draw stream, each thread jumping the 128-bit LCG
//      ahead to its chunk (O(log n) affine-map squaring) -- fully parallel;
//   2. k_rnd_draws: one warp assigns draws to steps.  Acceptance of draw r depends on
//      how many earlier draws were rejected, so each lane evaluates its draw under 16
//      hypotheses (k earlier rejections) and the warp resolves the chain with one
//      ballot per hypothesis: ~32 draws per iteration instead of one;
//   3. position p's final value is found by tracing p through the transpositions
//      (oracle/sampling.py permutation_prefix_traced): it becomes j_p at step p and
//      afterwards hops to the first later step whose draw equals its current value --
//      per-value step lists (count, scan, fill, sort the short lists), one thread per
//      p < budget;
//   4. the chosen ranks are flagged in the selection keys and the existing ordered
//      compaction writes the targets ascending.
// ---------------------------------------------------------------------------
constexpr int kRndHyp = 16;  // rejections one warp iteration can resolve
constexpr int kRndChunk = 64;  // 64-bit outputs per thread in k_rnd_raw

__host__ __device__ inline int64_t rnd_raw_len(int64_t R) { return 4 * R + 4096; }  // 32-bit draws generated

struct Pcg128 {
  unsigned __int128 s, inc;
};

__device__ __forceinline__ unsigned __int128 pcg_mult() {
  return ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
}

// state after `delta` steps of s <- a s + inc (pcg's affine-map squaring)
__device__ __forceinline__ unsigned __int128 pcg_advance(unsigned __int128 st, unsigned __int128 inc, uint64_t delta) {
  unsigned __int128 acc_m = 1, acc_p = 0, cur_m = pcg_mult(), cur_p = inc;
  while (delta) {
    if (delta & 1) {
      acc_m *= cur_m;
      acc_p = acc_p * cur_m + cur_p;
    }
    cur_p = (cur_m + 1) * cur_p;
    cur_m *= cur_m;
    delta >>= 1;
  }
  return acc_m * st + acc_p;
}

__device__ __forceinline__ uint64_t pcg_out(unsigned __int128 st) {  // XSL-RR
  const uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64 - rot) & 63));
}

__global__ void k_rnd_raw(Pcg128 g, const ReqCounters* rc, uint32_t* raw) {
  pdl_wait();
  const int64_t n64 = rnd_raw_len(cta_ld(&rc->R)) / 2;
  const int64_t chunks = (n64 + kRndChunk - 1) / kRndChunk;
  OB_GRID_STRIDE(c, chunks) {
    const int64_t o0 = c * kRndChunk;
    unsigned __int128 st = pcg_advance(g.s, g.inc, (uint64_t)o0);
    const int64_t o1 = min(o0 + kRndChunk, n64);
    for (int64_t o = o0; o < o1; ++o) {
      st = st * pcg_mult() + g.inc;  // next64: step, then output
      const uint64_t v = pcg_out(st);
      raw[2 * o] = (uint32_t)v;  // the bit generator's 32-bit buffer: low half first
      raw[2 * o + 1] = (uint32_t)(v >> 32);
    }
  }
}

// random_interval's mask: the smallest all-ones value >= m (m >= 1)
__device__ __forceinline__ uint32_t interval_mask(uint32_t m) { return 0xFFFFFFFFu >> __clz(m); }

// one warp: j[i] for i = R-1 .. 1 from the raw stream
__global__ void __launch_bounds__(32) k_rnd_draws(const uint32_t* __restrict__ raw, ReqCounters* rc, int32_t* jd) {
  pdl_wait();
  __shared__ uint32_t buf[2048];
  const int lane = threadIdx.x;
  const int64_t R = cta_ld(&rc->R);
  const int64_t L = rnd_raw_len(R);
  int64_t i = R - 1, r = 0, base = 0;
  for (int k = lane; k < 2048; k += 32) buf[k] = k < L ? raw[k] : 0u;
  __syncwarp();
  while (i >= 1) {
    if (r + 32 > base + 2048) {  // refill the window at r
      __syncwarp();
      base = r;
      for (int k = lane; k < 2048; k += 32) buf[k] = base + k < L ? raw[base + k] : 0u;
      __syncwarp();
    }
    if (r + 32 > L) {  // not reached in practice: 4R + 4096 draws for <= R-1 acceptances of p >= 1/2
      if (lane == 0) atomicOr((unsigned long long*)&rc->err, (unsigned long long)kErrRandom);
      return;
    }
    const uint32_t x = buf[r - base + lane];
    // hypothesis h: h rejections among the earlier lanes -> this lane's step is i - lane + h
    unsigned rej[kRndHyp];
    uint32_t vh[kRndHyp];
#pragma unroll
    for (int h = 0; h < kRndHyp; ++h) {
      const int64_t st = i - lane + h;
      bool acc = false;
      uint32_t v = 0;
      if (st >= 1 && st <= i) {
        v = x & interval_mask((uint32_t)st);
        acc = v <= (uint32_t)st;
      }
      vh[h] = v;
      rej[h] = __ballot_sync(0xffffffffu, !acc);
    }
    // resolve: lanes up to the first rejection under h = 0 are accepted with h = 0, the next
    // run up to the first rejection under h = 1 with h = 1, ... (unrolled, predicated)
    int cur = -1, myh = -1;
#pragma unroll
    for (int h = 0; h < kRndHyp; ++h) {
      if (cur < 32) {
        const unsigned above = cur >= 31 ? 0u : (0xffffffffu << (cur + 1));
        const unsigned b = rej[h] & above;
        const int f = b ? __ffs(b) - 1 : 32;
        if (lane > cur && lane < f) myh = h;
        cur = f;
      }
    }
    const int consumed = cur >= 32 ? 32 : cur + 1;  // through the last resolved rejection
    // lanes past the last resolved rejection are re-read next iteration
    bool wrote = false;
    if (myh >= 0 && lane < consumed) {
      int64_t st = i - lane + myh;
      uint32_t v = 0;
#pragma unroll
      for (int hh = 0; hh < kRndHyp; ++hh)
        if (hh == myh) v = vh[hh];
      if (st >= 1) {
        jd[st] = (int32_t)v;
        wrote = true;
      }
    }
    const int acc_n = __popc(__ballot_sync(0xffffffffu, wrote));
    i -= acc_n;
    r += consumed;
  }
}

// Chunked draw assignment (replaces the one-warp walk for large |R|).  Draws are cut
// into chunks of kRndW; a chunk maps the step it is entered with to the step it
// leaves with.  Phase A evaluates that map for a window of kRndK entering steps
// around the expected one (one thread per entering step, the chunk's draws
// broadcast from shared memory); phase B walks the chunks on one thread with the
// maps (falling back to simulating a chunk when the true step left its window);
// phase C re-runs every chunk from its true entering step and writes the draws.
constexpr int kRndW = 2048;      // draws per chunk
constexpr int kRndK = 4096;      // entering steps evaluated per chunk (4.7 sigma of the random walk at |R| = 2e5)
constexpr int kRndKCta = 1024;

__device__ __forceinline__ int64_t rnd_step_exit(const uint32_t* d, int n, int64_t s) {
  int r = 0;
  for (; r + 8 <= n && s >= 1; r += 8) {  // eight draws loaded ahead of the dependent chain
    uint32_t x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = d[r + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (s >= 1) {
        const uint32_t v = x[q] & interval_mask((uint32_t)s);
        s -= v <= (uint32_t)s;
      }
    }
  }
  for (; r < n && s >= 1; ++r) {
    const uint32_t v = d[r] & interval_mask((uint32_t)s);
    s -= v <= (uint32_t)s;
  }
  return s;
}

// the expected entering step of every chunk (deterministic: expected acceptances,
// four sub-steps per chunk at the local acceptance rate (i + 1) / (mask(i) + 1))
__global__ void k_rnd_estimate(const ReqCounters* rc, int64_t chunks, int64_t* lo) {
  pdl_wait();
  if (threadIdx.x || blockIdx.x) return;
  float i = (float)(ld_state(&rc->R) - 1);
  int64_t tail = 4;  // chunks evaluated past the expected end of the walk
  for (int64_t c = 0; c < chunks; ++c) {
    if (i < 1.f && --tail < 0) {
      lo[c] = INT64_MIN;  // never reached in expectation: k_rnd_chunkmap skips it
      continue;
    }
    lo[c] = (int64_t)lrintf(i) - kRndK / 2;
    for (int q = 0; q < 4 && i >= 1.f; ++q) {
      const float m = (float)interval_mask((uint32_t)i) + 1.f;
      i -= (kRndW / 4) * (i + 1.f) / m;
    }
  }
}

__global__ void __launch_bounds__(kRndKCta) k_rnd_chunkmap(const uint32_t* __restrict__ raw, const ReqCounters* rc,
                                                           const int64_t* __restrict__ lo, int32_t* exit_) {
  pdl_wait();
  __shared__ uint32_t d[kRndW];
  const int64_t R = cta_ld(&rc->R);
  const int64_t L = rnd_raw_len(R);
  const int64_t c = blockIdx.x / (kRndK / kRndKCta);
  const int k = (int)(blockIdx.x % (kRndK / kRndKCta)) * kRndKCta + threadIdx.x;
  const int64_t r0 = c * kRndW;
  if (r0 >= L || lo[c] == INT64_MIN) return;
  const int n = (int)min((int64_t)kRndW, L - r0);
  for (int r = threadIdx.x; r < n; r += kRndKCta) d[r] = raw[r0 + r];
  __syncthreads();
  const int64_t s0 = lo[c] + k;
  exit_[c * kRndK + k] = s0 >= 1 && s0 < R ? (int32_t)rnd_step_exit(d, n, s0) : -1;
}

__global__ void k_rnd_walk(const uint32_t* __restrict__ raw, ReqCounters* rc, int64_t chunks,
                           const int64_t* __restrict__ lo, const int32_t* __restrict__ exit_, int64_t* enter) {
  pdl_wait();
  if (threadIdx.x || blockIdx.x) return;
  const int64_t R = ld_state(&rc->R);
  const int64_t L = rnd_raw_len(R);
  int64_t i = R - 1;
  for (int64_t c = 0; c < chunks; ++c) {
    enter[c] = i;
    if (i < 1) continue;
    const int64_t r0 = c * kRndW;
    if (r0 >= L) {  // not reached in practice: the stream holds 4R + 4096 draws
      atomicOr((unsigned long long*)&rc->err, (unsigned long long)kErrRandom);
      return;
    }
    const int64_t k = lo[c] == INT64_MIN ? -1 : i - lo[c];
    if (k >= 0 && k < kRndK && exit_[c * kRndK + k] >= 0) i = exit_[c * kRndK + k];
    else i = rnd_step_exit(raw + r0, (int)min((int64_t)kRndW, L - r0), i);  // outside the window: walk it
  }
  if (i >= 1) atomicOr((unsigned long long*)&rc->err, (unsigned long long)kErrRandom);
}

__global__ void __launch_bounds__(32) k_rnd_emit(const uint32_t* __restrict__ raw, const ReqCounters* rc,
                                                 int64_t chunks, const int64_t* __restrict__ enter, int32_t* jd) {
  pdl_wait();
  __shared__ uint32_t d[kRndW];
  const int64_t L = rnd_raw_len(cta_ld(&rc->R));
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    int64_t s = enter[c];
    if (s < 1) continue;
    const int64_t r0 = c * kRndW;
    const int n = (int)max((int64_t)0, min((int64_t)kRndW, L - r0));
    __syncwarp();
    for (int r = threadIdx.x; r < n; r += 32) d[r] = raw[r0 + r];
    __syncwarp();
    if (threadIdx.x == 0) {
      for (int r = 0; r < n && s >= 1; ++r) {
        const uint32_t v = d[r] & interval_mask((uint32_t)s);
        if (v <= (uint32_t)s) {
          jd[s] = (int32_t)v;
          --s;
        }
      }
    }
  }
}

__global__ void k_rnd_count(const ReqCounters* rc, const int32_t* __restrict__ jd, int32_t* cnt) {
  pdl_wait();
  const int64_t R = cta_ld(&rc->R);
  OB_GRID_STRIDE(t, R) {
    if (t >= 1) atomicAdd(cnt + jd[t], 1);
  }
}

__global__ void k_rnd_fill(const ReqCounters* rc, const int32_t* __restrict__ jd, const int64_t* __restrict__ off,
                           int32_t* fill, int32_t* lst) {
  pdl_wait();
  const int64_t R = cta_ld(&rc->R);
  OB_GRID_STRIDE(t, R) {
    if (t >= 1) {
      const int32_t v = jd[t];
      lst[off[v] + atomicAdd(fill + v, 1)] = (int32_t)t;
    }
  }
}

// sort each value's (short) step list, then trace the chosen positions
__global__ void k_rnd_sort_lists(const ReqCounters* rc, const int64_t* __restrict__ off, int32_t* lst) {
  pdl_wait();
  const int64_t R = cta_ld(&rc->R);
  OB_GRID_STRIDE(v, R) {
    const int64_t a = off[v], b = off[v + 1];
    for (int64_t x = a + 1; x < b; ++x) {  // insertion sort (expected length <= ln R + 1)
      const int32_t key = lst[x];
      int64_t y = x - 1;
      while (y >= a && lst[y] > key) {
        lst[y + 1] = lst[y];
        --y;
      }
      lst[y + 1] = key;
    }
  }
}

__global__ void k_rnd_trace(ReqCounters* rc, const int32_t* __restrict__ jd, const int64_t* __restrict__ off,
                            const int32_t* __restrict__ lst, uint64_t* key) {
  pdl_wait();
  const CtaWords st = cta_ldv(&rc->R, &rc->budget);
  const int64_t R = st.v[0], budget = st.v[1];
  if (budget <= 0 || budget >= R) return;  // SelLoad takes none / all
  OB_GRID_STRIDE(p, budget) {
    int64_t x = p > 0 ? jd[p] : 0, s = p;
    for (int64_t guard = 0; guard < R; ++guard) {
      // first step > s whose draw equals x
      int64_t lo = off[x], hi = off[x + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (lst[mid] <= s) lo = mid + 1;
        else hi = mid;
      }
      if (lo == off[x + 1]) break;
      x = s = lst[lo];
    }
    key[x] = 1;  // candidate rank x is chosen (ranks follow ids: the compaction sorts by id)
  }
}

// host: SeedSequence(seed).generate_state(4, uint64) (numpy/random/bit_generator.pyx) and
// PCG64's seeding (pcg_setseq_128_srandom_r)
static Pcg128 pcg64_from_seed(uint64_t seed) {
  const uint32_t INIT_A = 0x43B0D7E5u, MULT_A = 0x931E8875u, INIT_B = 0x8B51F9DDu, MULT_B = 0x58F38DEDu;
  const uint32_t MIX_L = 0xCA01F9DDu, MIX_R = 0x4973F715u;
  std::vector<uint32_t> ent;
  if (seed == 0) ent.push_back(0);
  for (uint64_t x = seed; x; x >>= 32) ent.push_back((uint32_t)x);
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [&](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u);
  for (int a = 0; a < 4; ++a)
    for (int d = 0; d < 4; ++d)
      if (a != d) pool[d] = mix(pool[d], hashmix(pool[a]));
  for (size_t a = 4; a < ent.size(); ++a)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[a]));
  uint32_t hb = INIT_B, o[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4] ^ hb;
    hb *= MULT_B;
    v *= hb;
    o[i] = v ^ (v >> 16);
  }
  uint64_t st[4];
  for (int i = 0; i < 4; ++i) st[i] = (uint64_t)o[2 * i] | ((uint64_t)o[2 * i + 1] << 32);
  const unsigned __int128 mult = ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
  Pcg128 g;
  g.inc = ((((unsigned __int128)st[2] << 64) | st[3]) << 1) | 1u;
  g.s = 0;
  g.s = g.s * mult + g.inc;
  g.s += ((unsigned __int128)st[0] << 64) | st[1];
  g.s = g.s * mult + g.inc;
  return g;
}

static void select_random(Engine& e, RequestWs& w, int64_t r_max) {
  cudaStream_t s = e.stream;
  const Pcg128 g = pcg64_from_seed(e.cfg.seed);
  OB_CUDA(cudaMemsetAsync(w.cand_key, 0, sizeof(uint64_t) * std::max<int64_t>(r_max, 1), s));
  OB_CUDA(cudaMemsetAsync(w.rnd_cnt, 0, sizeof(int32_t) * (r_max + 1), s));
  OB_CUDA(cudaMemsetAsync(w.rnd_fill, 0, sizeof(int32_t) * (r_max + 1), s));
  launch_pdl(k_rnd_raw, dim3(grid_for(rnd_raw_len(r_max) / 2, kRndChunk * 128, kNumSMs * 4)), dim3(128), 0, s, g, w.rc, w.rnd_raw);
  // draws -> steps: the chunk maps + one walk + re-emission (large |R|); the one-warp walk
  // over the whole stream below kRndSmall candidates (a few chunks are not worth three launches)
  const int64_t chunks = (rnd_raw_len(r_max) + kRndW - 1) / kRndW;
  if (r_max > 8192) {
    launch_pdl(k_rnd_estimate, dim3(1), dim3(32), 0, s, w.rc, chunks, w.rnd_lo);
    launch_pdl(k_rnd_chunkmap, dim3((unsigned)(chunks * (kRndK / kRndKCta))), dim3(kRndKCta), 0, s, w.rnd_raw, w.rc, w.rnd_lo, w.rnd_exit);
    launch_pdl(k_rnd_walk, dim3(1), dim3(32), 0, s, w.rnd_raw, w.rc, chunks, w.rnd_lo, w.rnd_exit, w.rnd_enter);
    launch_pdl(k_rnd_emit, dim3((unsigned)std::min<int64_t>(chunks, kNumSMs * 16)), dim3(32), 0, s, w.rnd_raw, w.rc, chunks, w.rnd_enter,
                                                                                 w.rnd_j);
  } else {
    launch_pdl(k_rnd_draws, dim3(1), dim3(32), 0, s, w.rnd_raw, w.rc, w.rnd_j);
  }
  launch_pdl(k_rnd_count, dim3(grid_for(r_max, 256)), dim3(256), 0, s, w.rc, w.rnd_j, w.rnd_cnt);
  device_scan(s, e.scan, LoadI32{w.rnd_cnt}, StoreI64{w.rnd_off}, nullptr, r_max + 1, r_max + 1, nullptr);
  launch_pdl(k_rnd_fill, dim3(grid_for(r_max, 256)), dim3(256), 0, s, w.rc, w.rnd_j, w.rnd_off, w.rnd_fill, w.rnd_lst);
  launch_pdl(k_rnd_sort_lists, dim3(grid_for(r_max, 256)), dim3(256), 0, s, w.rc, w.rnd_off, w.rnd_lst);
  launch_pdl(k_rnd_trace, dim3(grid_for(r_max, 256)), dim3(256), 0, s, w.rc, w.rnd_j, w.rnd_off, w.rnd_lst, w.cand_key);
}

// Request CSR over an edge set (the whole request via the parameter block when
// edges == nullptr, or one CGP rank's slice in the arena): slot offsets from
// the per-slot counts, source order from the radix sort of the packed keys.
void build_rq_csr(Engine& e, RequestWs& w, const int64_t* edges, int64_t m_bound, const int64_t* m_dev, RqCsr& c,
                  bool counts_ready) {
  cudaStream_t s = e.stream;
  const int64_t rb_max = std::min<int64_t>(e.g.N, 2 * w.m) + w.B;
  const RqKeyFmt f = rq_key_fmt(e, w);
  if (!edges) m_dev = &w.rp->m;  // the whole request: its edge count lives in the parameter block
  if (!counts_ready) {
    launch_pdl(k_zero_slots, dim3(grid_for(rb_max, 256)), dim3(256), 0, s, w.rc, w.B, c.cnt, c.fill);
    if (m_bound > 0) {
      if (f.wide())
        launch_pdl(k_rq_count_all<uint64_t>, dim3(grid_for(m_bound, 256)), dim3(256), 0, s, edges, m_dev, e.g.N, w.cbits, w.cwpre, w.rc,
                                                                          c.cnt, c.keys, f);
      else
        launch_pdl(k_rq_count_all<uint32_t>, dim3(grid_for(m_bound, 256)), dim3(256), 0, s, 
            edges, m_dev, e.g.N, w.cbits, w.cwpre, w.rc, c.cnt, reinterpret_cast<uint32_t*>(c.keys), f);
    }
  }
  device_scan(s, e.scan, LoadI32{c.cnt}, StoreI64{c.ptr}, &w.rc->RB, 0, rb_max, nullptr, c.ptr);
  if (m_bound <= 0) return;
  if (f.wide()) rx_sort<uint64_t>(e, w, c, m_dev, m_bound, f);
  else rx_sort<uint32_t>(e, w, c, m_dev, m_bound, f);
}

void stage_request_csr(Engine& e, RequestWs& w) {
  RqCsr c = w.rq_view();
  build_rq_csr(e, w, nullptr, w.m, nullptr, c, /*counts_ready=*/true);
}

}  // namespace ob
