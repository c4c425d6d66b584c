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
#include <cub/block/block_scan.cuh>

#include "ob_engine.h"

namespace ob {

int64_t g_launches = 0;

// exclusive scan of the tile sums in place (one CTA; long scans only)
__global__ void __launch_bounds__(1024) k_scan_spine(const int64_t* n_dev, int64_t n_host, int64_t* tile_sums) {
  using BS = cub::BlockScan<int64_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t carry;
  const int64_t n = dev_count(n_dev, n_host);
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
  if (rc->err & (kErrRange | kErrNoQuery)) return;
  const int64_t* __restrict__ edges = rp->edges;
  const int64_t m = rp->m;
  OB_GRID_STRIDE(e, m) {
    int64_t s, d;
    ld_edge(edges, e, s, d);
    if (d < N) warp_agg_inc(rq_cnt, bm_rank(cbits, cwpre, d));
    keys[e] = rq_key<K>(s, d, N, cbits, cwpre, rc->R, f);
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
  if (rc->err & (kErrRange | kErrNoQuery)) return;
  const int64_t R = rc->R, m = *m_dev;  // a CGP slice: edges live in the arena
  OB_GRID_STRIDE(e, m) {
    int64_t s, d;
    ld_edge(edges, e, s, d);
    warp_agg_inc(rq_cnt, rq_slot(d, N, cbits, cwpre, R));
    keys[e] = rq_key<K>(s, d, N, cbits, cwpre, R, f);
  }
}

__global__ void k_zero_slots(const ReqCounters* rc, int B, int32_t* a, int32_t* b) {
  const int64_t RB = rc->R + B;
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
  const int64_t R = rc->R;
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
  k_is_rows<<<grid_for(N, kIsWarps, kNumSMs * 8), 32 * kIsWarps, 0, s>>>(N, off, src, e.g.indeg, out, big, nbig);
  OB_LAUNCHED();
  k_is_big<<<kNumSMs, 32 * kIsWarps, 0, s>>>(big, nbig, off, src, e.g.indeg, out);
  OB_LAUNCHED();
  OB_CUDA(cudaStreamSynchronize(s));
  e.dfree(big);
  e.dfree(nbig);
}

__global__ void k_is_gather(const int32_t* __restrict__ cand_ids, const ReqCounters* rc,
                            const double* __restrict__ tab, double* out) {
  const int64_t R = rc->R;
  OB_GRID_STRIDE(c, R) out[c] = tab[cand_ids[c]];
}

void launch_is_gather(Engine& e, RequestWs& w, const double* tab, double* out) {
  const int64_t r_max = std::min<int64_t>(e.g.N, 2 * w.m);
  k_is_gather<<<grid_for(r_max, 256), 256, 0, e.stream>>>(w.cand_ids, w.rc, tab, out);
  OB_LAUNCHED();
}

// scores from P partial arrays, summed in rank order (P = 1: the centralized row sum)
__global__ void k_score_is(const int32_t* __restrict__ cand_ids, const int32_t* __restrict__ indeg,
                           const ReqCounters* rc, IsParts parts, double* score, uint64_t* key) {
  const int64_t R = rc->R;
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
  k_score_is<<<grid_for(r_max, 256), 256, 0, e.stream>>>(w.cand_ids, e.g.indeg, w.rc, parts, w.cand_score,
                                                         w.cand_key);
  OB_LAUNCHED();
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
  if (threadIdx.x == 0) hist[256] = 0;
}

// One radix-select round in one launch: per-CTA digit histograms of the keys that
// still match the chosen prefix are merged into hist; the last CTA to finish
// picks this round's digit (scan from the top digit) and clears hist.
__global__ void __launch_bounds__(256) k_sel_round(const uint64_t* __restrict__ key, ReqCounters* rc, int shift,
                                                   uint32_t* hist) {
  using BS = cub::BlockScan<int64_t, 256>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t h[256];
  __shared__ bool last;
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t R = rc->R, b = rc->budget;
  const bool active = b > 0 && b < R;
  if (active) {
    const uint64_t pre = rc->sel_prefix, msk = rc->sel_mask;
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
  const int64_t krem = rc->sel_krem;
  if (excl < krem && krem <= excl + c) {
    rc->sel_krem = krem - excl;
    rc->sel_gt += excl;
    rc->sel_prefix |= (uint64_t)d << shift;
    rc->sel_mask |= (uint64_t)255 << shift;
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
  __device__ I3 operator()(int64_t c) const {
    const int64_t R = rc->R, b = rc->budget;
    if (b <= 0) return I3(0);
    if (b >= R) return I3(1, 0, 0);
    const uint64_t k = key[c], thr = rc->sel_prefix;
    return I3(k > thr ? 1 : 0, k == thr ? 1 : 0, 0);
  }
};
struct SelStore3 {
  SelLoad ld;
  const int32_t* cand_ids;
  int32_t* targets;
  int32_t* tpos;
  __device__ void operator()(int64_t c, const I3& pre) const {
    const I3 me = ld(c);
    const int64_t take = ld.rc->sel_eq_take;
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
    const int64_t take = rc->sel_eq_take;
    rc->T = t.a + (t.b < take ? t.b : take);
  }
};

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
  __shared__ int32_t h[256];
  const int64_t m = *m_dev;
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
  __shared__ uint32_t h[8 * 256];
  for (int i = threadIdx.x; i < passes * 256; i += kRxThreads) h[i] = 0;
  __syncthreads();
  const int64_t m = *m_dev;
  OB_GRID_STRIDE(e, m) {
    const K k = keys[e];
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p * 256 + (int)((k >> (8 * p)) & 255)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += kRxThreads)
    if (h[i]) atomicAdd(ghist + i, h[i]);
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
                                                           const uint32_t* __restrict__ ghist) {
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
  const int64_t m = *m_dev;
  const int64_t tiles = (m + kRxTile - 1) / kRxTile;
  if (st) {
    int64_t g = threadIdx.x < 256 ? (int64_t)ghist[threadIdx.x] : 0, gx;
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
        gofs[threadIdx.x] = off[(int64_t)threadIdx.x * tiles_b + t];
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
    for (int p = threadIdx.x; p < n; p += kRxThreads) {
      const K kk = u.exch[p];
      const int d = (int)((kk >> shift) & 255);
      const int64_t pos = gofs[d] + (p - bstart[d]);
      if (FINAL) {
        const bool query_slot = (kk >> f.body) & 1;
        if (query_slot) {
          const int64_t sr = (int64_t)(kk & (((K)1 << f.bN) - 1)), R = rc->R;
          src_out[pos] = sr < R ? cand_ids[sr] : (int32_t)(N + (sr - R));
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
    k_rx_ghist<K><<<grid_for(m_bound, kRxThreads * 8, kNumSMs * 2), kRxThreads, 0, s>>>(a, m_dev, passes, ghist);
    OB_LAUNCHED();
    for (int p = 0; p < passes; ++p) {
      const int shift = 8 * p;
      uint32_t* sp = st + (int64_t)p * 256 * tiles_b;
      if (p + 1 == passes) {
        k_rx_scatter<K, true><<<g, kRxThreads, 0, s>>>(a, nullptr, c.src, m_dev, shift, tiles_b, nullptr, c.rx_cnt, f,
                                                        e.g.N, w.cand_ids, w.rc, sp, ticket + p, ghist + 256 * p);
      } else {
        k_rx_scatter<K, false><<<g, kRxThreads, 0, s>>>(a, b, nullptr, m_dev, shift, tiles_b, nullptr, c.rx_cnt, f,
                                                         e.g.N, w.cand_ids, w.rc, sp, ticket + p, ghist + 256 * p);
        std::swap(a, b);
      }
      OB_LAUNCHED();
    }
    return;
  }
  const bool fused = tiles_b <= 32;  // few tiles: offsets come straight from the counts
  const int64_t* off = fused ? nullptr : c.rx_off;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    k_rx_hist<K><<<g, kRxThreads, 0, s>>>(a, m_dev, shift, tiles_b, c.rx_cnt);
    OB_LAUNCHED();
    if (!fused)
      device_scan(s, e.scan, LoadI32{c.rx_cnt}, StoreI64{c.rx_off}, nullptr, 256 * tiles_b, 256 * tiles_b, nullptr);
    if (p + 1 == passes) {
      k_rx_scatter<K, true><<<g, kRxThreads, 0, s>>>(a, nullptr, c.src, m_dev, shift, tiles_b, off, c.rx_cnt, f,
                                                      e.g.N, w.cand_ids, w.rc, nullptr, nullptr, nullptr);
    } else {
      k_rx_scatter<K, false><<<g, kRxThreads, 0, s>>>(a, b, nullptr, m_dev, shift, tiles_b, off, c.rx_cnt, f,
                                                       e.g.N, w.cand_ids, w.rc, nullptr, nullptr, nullptr);
      std::swap(a, b);
    }
    OB_LAUNCHED();
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
    k_request_mark<<<grid_for(m, kEdgeTile, kNumSMs * 4), 256, sq, s>>>(w.rp, N, w.B, w.cbits, w.qdeg, w.rc);
    OB_LAUNCHED();
  }
  // candidate set: popcount prefix, ascending ids
  device_scan(s, e.scan, LoadPopc{w.cbits}, StoreI64{w.cwpre}, nullptr, w.words_N, w.words_N, &w.rc->R, w.cwpre);
  k_bitmap_compact<<<grid_for(w.words_N, 256), 256, 0, s>>>(w.cbits, w.cwpre, w.words_N, w.cand_ids);
  OB_LAUNCHED();
  const int64_t rb_max = std::min<int64_t>(N, 2 * m) + w.B;
  k_slots_init<<<grid_for(rb_max, 256), 256, 0, s>>>(w.rc, w.B, w.qdeg, w.rq_cnt, w.rq_fill);
  OB_LAUNCHED();
  if (m > 0) {  // candidate-slot counts + the request CSR's radix keys
    const RqKeyFmt f = rq_key_fmt(e, w);
    if (f.wide())
      k_rq_count<uint64_t><<<grid_for(m, 256), 256, 0, s>>>(w.rp, N, w.cbits, w.cwpre, w.rc, w.rq_cnt, w.rq_keys, f);
    else
      k_rq_count<uint32_t><<<grid_for(m, 256), 256, 0, s>>>(w.rp, N, w.cbits, w.cwpre, w.rc, w.rq_cnt,
                                                            reinterpret_cast<uint32_t*>(w.rq_keys), f);
    OB_LAUNCHED();
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
    k_check_finite<<<grid_for((int64_t)w.B * e.g.F, 256), 256, 0, s>>>(w.rp, (int64_t)w.B * e.g.F, w.rc);
    OB_LAUNCHED();
  }
  if (need_scores) {
    const int64_t r_max = std::min<int64_t>(N, 2 * m);
    k_score<<<grid_for(r_max, 256), 256, 0, s>>>(w.cand_ids, w.rq_cnt, e.g.indeg, w.rc, w.cand_nq, w.cand_score,
                                                 w.cand_key, w.cand_tpos, e.cfg.policy == OB_POLICY_RATIO);
    OB_LAUNCHED();
  }
}

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
  k_budget<<<1, 256, 0, s>>>(w.rc, e.cfg.gamma, w.sel_hist);
  OB_LAUNCHED();
  for (int shift = 56; shift >= 0; shift -= 8) {
    k_sel_round<<<grid_for(r_max, 256, kNumSMs * 2), 256, 0, s>>>(w.cand_key, w.rc, shift, w.sel_hist);
    OB_LAUNCHED();
  }
  // ordered compaction: ties at the threshold resolved by ascending id
  const SelLoad ld{w.cand_key, w.rc};
  device_scan_t<I3>(s, e.scan, ld, SelStore3{ld, w.cand_ids, w.targets, w.cand_tpos}, SelTotal{w.rc}, &w.rc->R, 0,
                    r_max);
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
    k_zero_slots<<<grid_for(rb_max, 256), 256, 0, s>>>(w.rc, w.B, c.cnt, c.fill);
    OB_LAUNCHED();
    if (m_bound > 0) {
      if (f.wide())
        k_rq_count_all<uint64_t><<<grid_for(m_bound, 256), 256, 0, s>>>(edges, m_dev, e.g.N, w.cbits, w.cwpre, w.rc,
                                                                          c.cnt, c.keys, f);
      else
        k_rq_count_all<uint32_t><<<grid_for(m_bound, 256), 256, 0, s>>>(
            edges, m_dev, e.g.N, w.cbits, w.cwpre, w.rc, c.cnt, reinterpret_cast<uint32_t*>(c.keys), f);
      OB_LAUNCHED();
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
