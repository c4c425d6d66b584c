// ob_build.cu -- computation-graph construction on the device.
//
// Reference (paths relative to /root/reference/pkg/src/gnnserve):
//   _serving_in_sources   compgraph.py:216-221  CSR(v) ++ request sources into v
//   _make_block           compgraph.py:180-213  dedup, relabel, (dst, src) edge order
//   build_srpe            compgraph.py:308-345  last block = queries; mid = targets U queries
//   build_full_k_hop      compgraph.py:224-245  k-hop frontier expansion
//   DegreeView            compgraph.py:124-152  source normaliser degrees
//
// One generic builder serves every strategy.  A destination's source list is
// described by two spans -- a CSR span (training in-neighbours, ascending) and
// a request span (request sources into it, ascending after the per-slot sort)
// -- and the concatenation is ascending because request sources of a training
// destination are queries, which are numbered above every training id.  The
// builder then: scans the span lengths into dst_ptr, gathers the global
// source ids edge-parallel (hub destinations are split across warps), marks
// them (and the destinations' own rows) in a bitmap over [0, N+B), and uses
// the bitmap's popcount prefix both as the ascending unique source list and
// as the global -> local relabel.  Edges come out already ordered by
// (dst, src), so no sort is needed.
//
// Sampled strategy (build_sampled, compgraph.py:248-284): after the spans are
// known, k_sample_spans replaces every row longer than the block's fanout by
// the fanout sources numpy would keep -- one thread per destination runs
// numpy's SeedSequence(seed, (l, v)) -> PCG64 -> Floyd choice stream
// (restated in oracle/sampling.py) and writes the kept sources, ascending,
// to a per-block buffer that the fill reads instead of the CSR span.
#include "ob_engine.h"

namespace ob {

struct SegSpans {
  int64_t* cs;  // csr start (sampled row: start in samp)
  int32_t* cl;  // csr length (sampled row: -fanout, every source in samp)
  int64_t* rs;  // request-span start
  int32_t* rl;  // request-span length
  const int32_t* samp;  // sampled rows' kept sources
};

// spans for a destination list (global ids ascending)
__global__ void k_block_spans(const int32_t* __restrict__ dst_ids, const BlockCounters* cnt, int64_t N,
                              const int64_t* __restrict__ offsets, const int32_t* __restrict__ indeg,
                              const uint32_t* cbits, const int64_t* cwpre, const int64_t* rq_ptr,
                              const ReqCounters* rc, SegSpans sp, int64_t* seg_len) {
  pdl_wait();
  const CtaWords st = cta_ldv(&cnt->D, &rc->R, &rc->err);
  const int64_t D = st.v[0];
  const int64_t R = st.v[1];
  const bool bad = st.v[2] & (kErrRange | kErrNoQuery);
  OB_GRID_STRIDE(i, D) {
    int64_t v = dst_ids[i];
    int64_t cs = 0, rs = 0;
    int32_t cl = 0, rl = 0;
    if (v < N) {
      cs = offsets[v];
      cl = indeg[v];
      if (!bad && bm_test(cbits, v)) {
        int64_t c = bm_rank(cbits, cwpre, v);
        rs = rq_ptr[c];
        rl = (int32_t)(rq_ptr[c + 1] - rs);
      }
    } else if (!bad) {
      int64_t slot = R + (v - N);
      rs = rq_ptr[slot];
      rl = (int32_t)(rq_ptr[slot + 1] - rs);
    }
    sp.cs[i] = cs;
    sp.cl[i] = cl;
    sp.rs[i] = rs;
    sp.rl[i] = rl;
    seg_len[i] = (int64_t)cl + rl;
  }
}

// gather global source ids: one warp per aggregation work item (kAggChunk edges
// of one destination), so a destination's CSR row and request span are copied
// with contiguous, coalesced loads and hub destinations spread over many warps.
// SMEM variant (source bitmap fits in shared memory): each CTA marks its
// sources in a private shared bitmap and writes it out once; k_bitmap_or
// merges the per-CTA bitmaps.  Hub sources that appear in thousands of rows
// then cost shared-memory atomics instead of serialised L2 atomics on one word.
template <bool SMEM>
__global__ void __launch_bounds__(1024) k_block_fill(const BlockCounters* cnt, const int64_t* __restrict__ dst_ptr,
                                                     const int64_t* __restrict__ item_ptr,
                                                     const int32_t* __restrict__ item_dst, SegSpans sp,
                                                     const int32_t* __restrict__ nbrs,
                                                     const int32_t* __restrict__ rq_src, int32_t* src_global,
                                                     uint32_t* sbits, int64_t words, uint32_t* part_bits) {
  pdl_wait();
  extern __shared__ uint32_t sbm[];
  const int64_t items = cta_ld(&cnt->items);
  const int lane = threadIdx.x & 31;
  if (SMEM) {
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) sbm[w] = 0u;
    __syncthreads();
  }
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = gw; it < items; it += nw) {
    const int64_t i = __ldg(item_dst + it);
    const int64_t d0 = __ldg(dst_ptr + i);
    const int64_t e0 = d0 + (it - __ldg(item_ptr + i)) * kAggChunk;
    const int64_t e1 = min(e0 + kAggChunk, __ldg(dst_ptr + i + 1));
    const int64_t cs = __ldg(sp.cs + i), rs = __ldg(sp.rs + i);
    const int32_t cl0 = __ldg(sp.cl + i);
    const int32_t* __restrict__ row = cl0 < 0 ? sp.samp : nbrs;  // a sampled row lives in samp
    const int32_t cl = cl0 < 0 ? -cl0 : cl0;
    int32_t v[kAggChunk / 32];
#pragma unroll
    for (int u = 0; u < kAggChunk / 32; ++u) {  // all loads in flight first
      const int64_t e = e0 + u * 32 + lane, j = e - d0;
      v[u] = e < e1 ? (j < cl ? __ldg(row + cs + j) : __ldg(rq_src + rs + (j - cl))) : -1;
    }
#pragma unroll
    for (int u = 0; u < kAggChunk / 32; ++u) {
      if (v[u] < 0) continue;
      src_global[e0 + u * 32 + lane] = v[u];
      if (SMEM) {
        const uint32_t m = 1u << (v[u] & 31);
        if (!(sbm[v[u] >> 5] & m)) atomicOr(sbm + (v[u] >> 5), m);
      } else {
        bm_set(sbits, v[u]);  // test before set: a re-marked source costs a read, not an atomic
      }
    }
  }
  if (SMEM) {
    __syncthreads();
    uint32_t* out = part_bits + (int64_t)blockIdx.x * words;
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) out[w] = sbm[w];
  }
}

// --- numpy's per-destination sampling stream -----------------------------------
// SeedSequence(entropy=seed, spawn_key=(l, v)).generate_state(4, uint64)
// (numpy/random/bit_generator.pyx): uint32 limbs, entropy zero-padded to the
// 4-word pool because a spawn key is present, hashmix/mix pool, INIT_B draw.
__device__ void ss_generate(uint64_t seed, uint32_t l, uint32_t v, uint64_t st[4]) {
  uint32_t ent[6];
  int ne = 0;
  ent[ne++] = (uint32_t)seed;
  if (seed >> 32) ent[ne++] = (uint32_t)(seed >> 32);
  while (ne < 4) ent[ne++] = 0u;
  ent[4] = l;
  ent[5] = v;
  uint32_t hc = 0x43b0d7e5u;
  auto hashmix = [&hc](uint32_t x) {
    x ^= hc;
    hc *= 0x931e8875u;
    x *= hc;
    return x ^ (x >> 16);
  };
  auto mix = [](uint32_t x, uint32_t y) {
    const uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    return r ^ (r >> 16);
  };
  uint32_t mx[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) mx[i] = hashmix(ent[i]);
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int d = 0; d < 4; ++d)
      if (a != d) mx[d] = mix(mx[d], hashmix(mx[a]));
#pragma unroll
  for (int a = 4; a < 6; ++a)
#pragma unroll
    for (int d = 0; d < 4; ++d) mx[d] = mix(mx[d], hashmix(ent[a]));
  uint32_t hb = 0x8b51f9ddu, o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t x = mx[i & 3] ^ hb;
    hb *= 0x58f38dedu;
    x *= hb;
    o[i] = x ^ (x >> 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) st[i] = (uint64_t)o[2 * i] | ((uint64_t)o[2 * i + 1] << 32);
}

// numpy's PCG64 (XSL-RR 128/64, pcg_setseq_128_srandom_r seeding) with the
// bit generator's 32-bit draw buffer (low half of a 64-bit output first)
struct Pcg64 {
  unsigned __int128 s, inc;
  uint32_t buf;
  bool has;
  __device__ void step() {
    const unsigned __int128 mult = ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    s = s * mult + inc;
  }
  __device__ explicit Pcg64(const uint64_t st[4]) {
    const unsigned __int128 seed = ((unsigned __int128)st[0] << 64) | st[1];
    inc = ((((unsigned __int128)st[2] << 64) | st[3]) << 1) | 1u;
    s = 0;
    step();
    s += seed;
    step();
    has = false;
    buf = 0;
  }
  __device__ uint64_t next64() {
    step();
    const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    const unsigned rot = (unsigned)(hi >> 58);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ uint32_t next32() {
    if (has) {
      has = false;
      return buf;
    }
    const uint64_t n = next64();
    has = true;
    buf = (uint32_t)(n >> 32);
    return (uint32_t)n;
  }
  // random_bounded_uint64(0, rng) for 0 < rng < 2^32 - 1: Lemire's rejection method
  __device__ uint32_t bounded(uint32_t rng) {
    const uint32_t ex = rng + 1u;
    uint64_t m = (uint64_t)next32() * ex;
    uint32_t left = (uint32_t)m;
    if (left < ex) {
      const uint32_t thr = (0xFFFFFFFFu - rng) % ex;
      while (left < thr) {
        m = (uint64_t)next32() * ex;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

// rows longer than fan keep Generator.choice(n, fan, replace=False)'s set
// (Floyd: j = n-fan .. n-1, t = bounded(j), keep t unless chosen, else j),
// ascending; the row's source list is ascending, so the kept values come out
// in the order np.sort(nbrs[keep]) gives
__global__ void __launch_bounds__(128) k_sample_spans(const int32_t* __restrict__ dst_ids, const BlockCounters* cnt,
                                                      SegSpans sp, const int32_t* __restrict__ nbrs,
                                                      const int32_t* __restrict__ rq_src, int fan, int layer,
                                                      uint64_t seed, int32_t* samp, int64_t* seg_len) {
  pdl_wait();
  const int64_t D = cta_ld(&cnt->D);
  OB_GRID_STRIDE(i, D) {
    const int32_t cl = sp.cl[i], rl = sp.rl[i];
    const int64_t n = (int64_t)cl + rl;
    if (n <= fan) continue;
    uint64_t st[4];
    ss_generate(seed, (uint32_t)layer, (uint32_t)dst_ids[i], st);
    Pcg64 g(st);
    int32_t pick[OB_MAX_FANOUT];
    int c = 0;
    for (int64_t j = n - fan; j < n; ++j) {
      const int32_t t = j > 0 ? (int32_t)g.bounded((uint32_t)j) : 0;
      bool dup = false;
      for (int q = 0; q < c; ++q) dup |= pick[q] == t;
      // insertion into the ascending list of picks
      int32_t x = dup ? (int32_t)j : t;
      int q = c++;
      while (q > 0 && pick[q - 1] > x) {
        pick[q] = pick[q - 1];
        --q;
      }
      pick[q] = x;
    }
    const int64_t cs = sp.cs[i], rs = sp.rs[i];
    int32_t* out = samp + i * fan;
    for (int q = 0; q < fan; ++q) {
      const int32_t j = pick[q];
      out[q] = j < cl ? nbrs[cs + j] : rq_src[rs + (j - cl)];
    }
    sp.cs[i] = i * fan;
    sp.cl[i] = -fan;
    sp.rl[i] = 0;
    seg_len[i] = fan;
  }
}

// OR of the per-CTA bitmaps: a CTA takes 32 words; each of its 8 warps ORs every
// 8th part over those words (a warp reads 32 consecutive words: one coalesced
// 128-byte line per part), then warp 0 combines the 8 partial words
__global__ void __launch_bounds__(256) k_bitmap_or(const uint32_t* __restrict__ part_bits, int nparts, int64_t words,
                                                   uint32_t* sbits) {
  pdl_wait();
  __shared__ uint32_t acc[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t w0 = (int64_t)blockIdx.x * 32; w0 < words; w0 += (int64_t)gridDim.x * 32) {
    const int64_t w = w0 + lane;
    uint32_t v = 0;
    if (w < words) {
#pragma unroll 4
      for (int p = warp; p < nparts; p += 8) v |= __ldg(part_bits + (int64_t)p * words + w);
    }
    acc[warp][lane] = v;
    __syncthreads();
    if (warp == 0 && w < words) {
      uint32_t o = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) o |= acc[q][lane];
      sbits[w] = o;
    }
    __syncthreads();
  }
}

constexpr int64_t kFillSmemWords = 48 * 1024;  // 192 KB: source bitmaps up to 1.5M ids stay on chip

void configure_fill() {
  OB_CUDA(cudaFuncSetAttribute(k_block_fill<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(kFillSmemWords * 4)));
}

__global__ void __launch_bounds__(256) k_expand_items(const BlockCounters* cnt, const int64_t* __restrict__ item_ptr,
                                                      const int64_t* __restrict__ group_ptr, int32_t* item_dst,
                                                      int32_t* group_dst) {
  pdl_wait();
  const int64_t D = cta_ld(&cnt->D);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < D; i += nw) {
    for (int64_t it = item_ptr[i] + lane; it < item_ptr[i + 1]; it += 32) item_dst[it] = (int32_t)i;
    for (int64_t g = group_ptr[i] + lane; g < group_ptr[i + 1]; g += 32) group_dst[g] = (int32_t)i;
  }
}

void expand_items(cudaStream_t s, const BlockCounters* cnt, int64_t D_max, const int64_t* item_ptr,
                  const int64_t* group_ptr, int32_t* item_dst, int32_t* group_dst) {
  launch_pdl(k_expand_items, dim3(grid_for(D_max, 8, kNumSMs * 16)), dim3(256), 0, s, cnt, item_ptr, group_ptr, item_dst, group_dst);
}

__global__ void k_mark_ids(const int32_t* __restrict__ ids, const BlockCounters* cnt, uint32_t* sbits) {
  pdl_wait();
  const int64_t D = cta_ld(&cnt->D);
  OB_GRID_STRIDE(i, D) bm_set(sbits, ids[i]);
}

__global__ void k_relabel(const BlockCounters* cnt, const int32_t* __restrict__ src_global, const uint32_t* sbits,
                          const int64_t* swpre, int32_t* edge_src) {
  pdl_wait();
  const int64_t E = cta_ld(&cnt->E);
  OB_GRID_STRIDE(e, E) edge_src[e] = (int32_t)bm_rank(sbits, swpre, src_global[e]);
}

__global__ void k_self_rows(const BlockCounters* cnt, const int32_t* __restrict__ dst_ids, const uint32_t* sbits,
                            const int64_t* swpre, int32_t* self_src) {
  pdl_wait();
  const int64_t D = cta_ld(&cnt->D);
  OB_GRID_STRIDE(i, D) self_src[i] = (int32_t)bm_rank(sbits, swpre, dst_ids[i]);
}

// srpe destination lists ------------------------------------------------------
__global__ void k_mid_dst(const ReqCounters* rc, int64_t N, int B, const int32_t* targets, int32_t* dst_ids,
                          BlockCounters* cnt) {
  pdl_wait();
  const int64_t T = cta_ld(&rc->T), D = T + B;
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt->D = D;
  OB_GRID_STRIDE(i, D) dst_ids[i] = i < T ? targets[i] : (int32_t)(N + (i - T));
}

__global__ void k_query_dst(int64_t N, int B, int32_t* dst_ids, BlockCounters* cnt) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt->D = B;
  OB_GRID_STRIDE(i, (int64_t)B) dst_ids[i] = (int32_t)(N + i);
}

__global__ void k_copy_count_D(BlockCounters* dst, const BlockCounters* src) {
  pdl_wait(); dst->D = ld_state(&src->S); }

// generic block assembly over an already written dst list + counts->D.
// `src` names the CSR the destinations pull from (the whole graph, or a CGP
// rank's source-split CSR) and the request CSR (whole request or the rank's slice).
void assemble(Engine& e, RequestWs& w, BlockDev& b, const SpanSrc& src, const BuildScratch& sc, int fan,
              int layer) {
  cudaStream_t s = e.stream;
  SegSpans sp;  // transient, shared by every block of the request
  sp.cs = sc.span_cs;
  sp.cl = sc.span_cl;
  sp.rs = sc.span_rs;
  sp.rl = sc.span_rl;
  sp.samp = sc.samp;
  launch_pdl(k_block_spans, dim3(grid_for(b.D_max, 256)), dim3(256), 0, s, b.dst_ids, b.cnt, e.g.N, src.offsets, src.deg, w.cbits,
                                                        w.cwpre, src.rq_ptr, w.rc, sp, sc.seg_len);
  if (fan > 0) {
    launch_pdl(k_sample_spans, dim3(grid_for(b.D_max, 128)), dim3(128), 0, s, b.dst_ids, b.cnt, sp, src.nbrs, src.rq_src, fan, layer,
                                                           e.cfg.seed, sc.samp, sc.seg_len);
  }
  // dst_ptr / item_ptr / group_ptr (+ E, items, groups) in one pass; the work
  // items double as the fill's edge chunks
  const BlockStore3 st{b.dst_ptr, b.item_ptr, b.group_ptr};
  device_scan_t<I3>(s, e.scan, SegLenLoad3{sc.seg_len}, st, BlockTotal3{st, b.cnt}, &b.cnt->D, 0, b.D_max);
  expand_items(s, b.cnt, b.D_max, b.item_ptr, b.group_ptr, b.item_dst, b.group_dst);
  if (w.words_NB <= kFillSmemWords) {  // per-CTA shared bitmaps, then one OR pass
    const int64_t words = w.words_NB + 1;
    launch_pdl(k_block_fill<true>, dim3(kNumSMs), dim3(1024), words * 4, s, b.cnt, b.dst_ptr, b.item_ptr, b.item_dst, sp, src.nbrs,
                                                        src.rq_src, sc.src_global, nullptr, words, sc.fill_bits);
    launch_pdl(k_bitmap_or, dim3(grid_for(words, 32, kNumSMs * 8)), dim3(256), 0, s, (const uint32_t*)sc.fill_bits,
               (int)kNumSMs, words, sc.sbits);
  } else {
    OB_CUDA(cudaMemsetAsync(sc.sbits, 0, sizeof(uint32_t) * (w.words_NB + 1), s));
    launch_pdl(k_block_fill<false>, dim3(grid_for(b.items_max, 32, kNumSMs * 2)), dim3(1024), 0, s, 
        b.cnt, b.dst_ptr, b.item_ptr, b.item_dst, sp, src.nbrs, src.rq_src, sc.src_global, sc.sbits, 0, nullptr);
  }
  if (b.has_self) {
    launch_pdl(k_mark_ids, dim3(grid_for(b.D_max, 256)), dim3(256), 0, s, b.dst_ids, b.cnt, sc.sbits);
  }
  bitmap_rank(e, sc.sbits, w.words_NB, sc.swpre, b.src_ids, &b.cnt->S, sc.gcnt, sc.gpre);
  launch_pdl(k_relabel, dim3(grid_for(b.E_max, 256)), dim3(256), 0, s, b.cnt, sc.src_global, sc.sbits, sc.swpre, b.edge_src);
  if (b.has_self) {
    launch_pdl(k_self_rows, dim3(grid_for(b.D_max, 256)), dim3(256), 0, s, b.cnt, b.dst_ids, sc.sbits, sc.swpre, b.self_src);
  }
}

void write_mid_dst(Engine& e, RequestWs& w, BlockDev& b) {
  launch_pdl(k_mid_dst, dim3(grid_for(b.D_max, 256)), dim3(256), 0, e.stream, w.rc, e.g.N, w.B, w.targets, b.dst_ids, b.cnt);
}

void write_query_dst(Engine& e, RequestWs& w, BlockDev& b) {
  launch_pdl(k_query_dst, dim3(grid_for(w.B, 256)), dim3(256), 0, e.stream, e.g.N, w.B, b.dst_ids, b.cnt);
}


// the two srpe blocks separately: the query block needs only the request index,
// the mid block also the targets
void build_query_block(Engine& e, RequestWs& w) {
  const SpanSrc src{e.g.offsets, e.g.nbrs, e.g.indeg, w.rq_ptr, w.rq_src};
  write_query_dst(e, w, w.blocks[1]);
  assemble(e, w, w.blocks[1], src, w.bs[1]);
}
void build_mid_block(Engine& e, RequestWs& w) {
  const SpanSrc src{e.g.offsets, e.g.nbrs, e.g.indeg, w.rq_ptr, w.rq_src};
  write_mid_dst(e, w, w.blocks[0]);
  assemble(e, w, w.blocks[0], src, w.bs[0]);
}

void stage_build_full(Engine& e, RequestWs& w) {
  cudaStream_t s = e.stream;
  const int k = (int)e.layers.size();
  const SpanSrc src{e.g.offsets, e.g.nbrs, e.g.indeg, w.rq_ptr, w.rq_src};
  // blocks[l-1] feeds layer l; block k's dst = queries; block l-1's dst = block l's sources
  write_query_dst(e, w, w.blocks[k - 1]);
  for (int l = k; l >= 1; --l) {
    BlockDev& b = w.blocks[l - 1];
    if (l < k) {
      BlockDev& up = w.blocks[l];  // b.dst_ids aliases up.src_ids (carve)
      launch_pdl(k_copy_count_D, dim3(1), dim3(1), 0, s, b.cnt, up.cnt);
    }
    const bool samp = e.cfg.strategy == OB_STRATEGY_SAMPLED;
    assemble(e, w, b, src, w.bs[0], samp ? e.cfg.fanouts[l - 1] : 0, l);
  }
}

}  // namespace ob
