// ob_gen.cu -- synthetic power-law graphs generated on the device (SURVEY.md
// 8(f)2: "needed for papers-scale inputs that cannot exist on host or disk").
//
// Reference law (gnnserve/workload.py:119-168): configuration-model graph whose
// in- and out-degree sequences follow the same power law P(k) ~ k^-exponent
// with a given average degree.  The device generator draws from that law but
// is not the numpy stream (bit-identity is impossible at 10^9 edges and is not
// claimed; DESIGN.md says so):
//   * popularity ranks are Zipf(s) with s = 1 / (exponent - 1), which gives a
//     degree distribution with the same tail exponent;
//   * in-degree of node v: max(1, round(E * p(rank_in(v)))) with rank_in an
//     affine bijection of v and p the Zipf pmf normalised over N;
//   * in-edge j of v takes its source by inverse-CDF sampling of the Zipf law at
//     the stratified point (j + u) / d_v, so each CSR row comes out already
//     ascending (the (dst, src) order of compgraph.py:197-201) and source
//     out-degrees follow the same law (source ids are popularity ranks);
//   * features N(0, 1) by Box-Muller on a counter hash.
// Everything is a pure function of (v, j, seed), so a CGP rank generates exactly
// its own source-split CSR and owned feature rows without ever holding the
// whole graph (graphstore.py:219-263 layout).
#include <algorithm>
#include <cmath>
#include <functional>
#include <vector>

#include "ob_engine.h"

namespace ob {

__device__ __forceinline__ uint64_t gmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

// rank in [0, N) of the Zipf(s) law at cumulative probability x in [0, 1)
__device__ __forceinline__ int64_t zipf_rank(const GenLaw& L, double x) {
  const double r = pow(1.0 + x * L.c1, L.inv1ms);  // continuous inverse CDF on [1, N + 1)
  int64_t k = (int64_t)r - 1;
  return k < 0 ? 0 : (k >= L.N ? L.N - 1 : k);
}

__device__ __forceinline__ int32_t gen_indeg(const GenLaw& L, int64_t v) {
  const int64_t r = (int64_t)(((unsigned __int128)L.a * (uint64_t)v + L.b) % (uint64_t)L.N);  // rank_in(v)
  const double d = L.E * pow((double)(r + 1), -L.s) / L.H;
  const double c = d < 1.0 ? 1.0 : (d > 2.0e9 ? 2.0e9 : floor(d + 0.5));
  return (int32_t)c;
}

__device__ __forceinline__ int64_t gen_src(const GenLaw& L, int64_t v, int64_t j, int32_t d) {
  const double x = ((double)j + u01(gmix(L.seed ^ gmix((uint64_t)v * 0x9E3779B97F4A7C15ull + (uint64_t)j)))) / d;
  return zipf_rank(L, x);
}

__global__ void k_zipf_norm(GenLaw L, double* acc) {
  pdl_wait();
  double s = 0.0;
  OB_GRID_STRIDE(r, L.N) s += pow((double)(r + 1), -L.s);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc, s);
}

__global__ void k_gen_indeg(GenLaw L, int32_t* indeg) {
  pdl_wait(); OB_GRID_STRIDE(v, L.N) indeg[v] = gen_indeg(L, v); }

// owned in-neighbours per destination row (owner == nullptr: all); warp per row
__global__ void k_gen_count(GenLaw L, const int32_t* __restrict__ indeg, const int32_t* __restrict__ owner, int rank,
                            int32_t* cnt) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < L.N; v += nw) {
    const int32_t d = indeg[v];
    int c = 0;
    for (int64_t j = lane; j < d; j += 32) {
      const int64_t u = gen_src(L, v, j, d);
      c += owner ? owner[u] == rank : 1;
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[v] = c;
  }
}

__global__ void k_gen_fill(GenLaw L, const int32_t* __restrict__ indeg, const int32_t* __restrict__ owner, int rank,
                           const int64_t* __restrict__ off, int32_t* src) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < L.N; v += nw) {
    const int32_t d = indeg[v];
    int64_t out = off[v];
    for (int64_t j0 = 0; j0 < d; j0 += 32) {
      const int64_t j = j0 + lane;
      int64_t u = 0;
      bool keep = false;
      if (j < d) {
        u = gen_src(L, v, j, d);
        keep = owner ? owner[u] == rank : true;
      }
      const unsigned b = __ballot_sync(0xffffffffu, keep);
      if (keep) src[out + __popc(b & ((1u << lane) - 1u))] = (int32_t)u;
      out += __popc(b);
    }
  }
}

// N(0, 1) rows for the stored nodes (global id -> local row via pos)
__global__ void k_gen_rows(int64_t N, int F, int ld, uint64_t seed, const int32_t* pos, float* rows) {
  pdl_wait();
  const int64_t n = N * (int64_t)ld;
  OB_GRID_STRIDE(i, n) {
    const int64_t v = i / ld;
    const int f = (int)(i - v * ld);
    const int32_t p = pos ? pos[v] : (int32_t)v;
    if (p < 0) continue;
    float x = 0.f;
    if (f < F) {
      const uint64_t h1 = gmix(seed ^ gmix((uint64_t)v * 0xD1B54A32D192ED03ull + (uint64_t)f));
      const uint64_t h2 = gmix(h1 ^ 0xA0761D6478BD642Full);
      const float a = 1.f - (float)(h1 >> 40) * (1.f / 16777216.f), b = (float)(h2 >> 40) * (1.f / 16777216.f);
      x = sqrtf(-2.f * __logf(a)) * __cosf(6.2831853f * b);
    }
    rows[(int64_t)p * ld + f] = x;
  }
}

GenLaw make_law(int64_t N, double avg, double exponent, uint64_t seed, cudaStream_t s, double* d_acc) {
  OB_CHECK(N >= 2 && N < ((int64_t)1 << 31) - 4096, OB_EINVAL, "generator: num_nodes out of range");
  OB_CHECK(avg >= 1.0 && exponent > 1.0, OB_EINVAL, "generator: need avg_degree >= 1 and exponent > 1");
  GenLaw L{};
  L.N = N;
  L.s = 1.0 / (exponent - 1.0);
  L.inv1ms = 1.0 / (1.0 - L.s);
  L.c1 = std::pow((double)N + 1.0, 1.0 - L.s) - 1.0;
  L.E = avg * (double)N;
  L.seed = seed;
  // affine bijection rank_in(v) = (a v + b) mod N with gcd(a, N) = 1
  uint64_t a = 0x9E3779B97F4A7C15ull % (uint64_t)N;
  auto gcd = [](uint64_t x, uint64_t y) {
    while (y) {
      uint64_t t = x % y;
      x = y;
      y = t;
    }
    return x;
  };
  if (a < 2) a = 2;
  while (gcd(a, (uint64_t)N) != 1) ++a;
  L.a = a;
  L.b = (seed * 0xBF58476D1CE4E5B9ull) % (uint64_t)N;
  OB_CUDA(cudaMemsetAsync(d_acc, 0, sizeof(double), s));
  launch_pdl(k_zipf_norm, dim3(kNumSMs * 8), dim3(256), 0, s, L, d_acc);
  OB_CUDA(cudaMemcpyAsync(&L.H, d_acc, sizeof(double), cudaMemcpyDeviceToHost, s));
  OB_CUDA(cudaStreamSynchronize(s));
  return L;
}

}  // namespace ob

namespace ob {

__global__ void k_sum_i32(const int32_t* a, int64_t n, unsigned long long* out) {
  pdl_wait();
  unsigned long long s = 0;
  OB_GRID_STRIDE(i, n) s += (unsigned long long)a[i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

// prefix of the largest in-degrees (the request planner's edge bounds): the top
// 4M degrees are enough for any request bucket; beyond that the planner uses E
static void topdeg_from_device(Engine& e) {
  GraphDev& g = e.g;
  std::vector<int32_t> deg((size_t)g.N);
  OB_CUDA(cudaMemcpy(deg.data(), g.indeg, sizeof(int32_t) * g.N, cudaMemcpyDeviceToHost));
  const int64_t K = std::min<int64_t>(g.N, (int64_t)1 << 22);
  std::nth_element(deg.begin(), deg.begin() + (K - 1), deg.end(), std::greater<int32_t>());
  std::sort(deg.begin(), deg.begin() + K, std::greater<int32_t>());
  g.topdeg_prefix.assign((size_t)K + 1, 0);
  for (int64_t i = 0; i < K; ++i) g.topdeg_prefix[i + 1] = g.topdeg_prefix[i] + deg[i];
}

// Build the serving graph on the device.  NCCL-mode CGP engines get only their
// rank's share (source-split CSR, owned feature rows, global in-degrees);
// every other engine gets the whole in-CSR and feature table.
void generate_graph(Engine& e, int64_t N, double avg, double exponent, int F, uint64_t seed) {
  OB_CHECK(e.g.N == 0, OB_ESTATE, "graph already loaded");
  OB_CHECK(F >= 1, OB_EINVAL, "generator: feature_dim must be >= 1");
  cudaStream_t s = e.stream;
  double* acc = (double*)e.dalloc(sizeof(double) * 2);
  const GenLaw L = make_law(N, avg, exponent, seed, s, acc);
  GraphDev& g = e.g;
  g.N = N;
  g.F = F;
  g.F_ld = ld4(F);
  g.generated = true;
  g.indeg = (int32_t*)e.dalloc(sizeof(int32_t) * N);
  launch_pdl(k_gen_indeg, dim3(grid_for(N, 256)), dim3(256), 0, s, L, g.indeg);
  {
    unsigned long long* tot = reinterpret_cast<unsigned long long*>(acc + 1);
    OB_CUDA(cudaMemsetAsync(tot, 0, sizeof(*tot), s));
    launch_pdl(k_sum_i32, dim3(kNumSMs * 8), dim3(256), 0, s, g.indeg, N, tot);
    unsigned long long h = 0;
    OB_CUDA(cudaMemcpyAsync(&h, tot, sizeof(h), cudaMemcpyDeviceToHost, s));
    OB_CUDA(cudaStreamSynchronize(s));
    g.E = (int64_t)h;
  }
  ScanScratch sc;
  sc.cap = ScanScratch::bytes_for(N, 2);
  sc.pool = (char*)e.dalloc(sc.cap);
  OB_CUDA(cudaMemsetAsync(sc.pool, 0, sc.cap, s));
  int64_t* total = (int64_t*)e.dalloc(sizeof(int64_t));
  const uint64_t fseed = seed ^ 0x5851F42D4C957F2Dull;
  const bool part = e.cfg.strategy == OB_STRATEGY_SRPE_CGP && e.cfg.nccl_id != nullptr;
  if (part) {
    CgpState& c = e.cgp;
    c.P = e.cfg.num_partitions;
    c.nccl = true;
    c.my_rank = e.cfg.rank;
    c.owner = (int32_t*)e.dalloc(sizeof(int32_t) * N);
    launch_pdl(k_owner, dim3(grid_for(N, 256)), dim3(256), 0, s, N, c.P, e.cfg.seed, c.owner);
    owned_positions(e);  // pos map + N_local
    g.feats = (float*)e.dalloc(sizeof(float) * std::max<int64_t>(g.N_local, 1) * g.F_ld);
    launch_pdl(k_gen_rows, dim3(grid_for(N * g.F_ld, 256)), dim3(256), 0, s, N, F, g.F_ld, fseed, g.pos, g.feats);
    // this rank's source-split CSR, rows ascending
    PartitionDev p;
    p.rank = c.my_rank;
    p.deg = (int32_t*)e.dalloc(sizeof(int32_t) * N);
    p.off = (int64_t*)e.dalloc(sizeof(int64_t) * (N + 1));
    launch_pdl(k_gen_count, dim3(grid_for(N, 8, kNumSMs * 16)), dim3(256), 0, s, L, g.indeg, c.owner, c.my_rank, p.deg);
    device_scan(s, sc, LoadI32{p.deg}, StoreI64{p.off}, nullptr, N, N, total, p.off);
    OB_CUDA(cudaMemcpyAsync(&p.E, total, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    OB_CUDA(cudaStreamSynchronize(s));
    p.src = (int32_t*)e.dalloc(sizeof(int32_t) * std::max<int64_t>(p.E, 1));
    launch_pdl(k_gen_fill, dim3(grid_for(N, 8, kNumSMs * 16)), dim3(256), 0, s, L, g.indeg, c.owner, c.my_rank, p.off, p.src);
    c.parts.clear();
    c.parts.push_back(p);
    e.localized = true;
  } else {
    g.offsets = (int64_t*)e.dalloc(sizeof(int64_t) * (N + 1));
    device_scan(s, sc, LoadI32{g.indeg}, StoreI64{g.offsets}, nullptr, N, N, total, g.offsets);
    g.nbrs = (int32_t*)e.dalloc(sizeof(int32_t) * std::max<int64_t>(g.E, 1));
    launch_pdl(k_gen_fill, dim3(grid_for(N, 8, kNumSMs * 16)), dim3(256), 0, s, L, g.indeg, nullptr, 0, g.offsets, g.nbrs);
    g.feats = (float*)e.dalloc(sizeof(float) * N * g.F_ld);
    launch_pdl(k_gen_rows, dim3(grid_for(N * g.F_ld, 256)), dim3(256), 0, s, N, F, g.F_ld, fseed, nullptr, g.feats);
    g.N_local = N;
  }
  OB_CUDA(cudaStreamSynchronize(s));
  e.dfree(sc.pool);
  e.dfree(total);
  e.dfree(acc);
  topdeg_from_device(e);
  if (!part && e.cfg.strategy == OB_STRATEGY_SRPE_CGP) cgp_build_partitions(e);
}

// Synthetic stored embeddings for layer `layer` (rows of the stored nodes only):
// serving kernels are data-independent, so papers-scale benches use these in
// place of a full-graph precompute (DESIGN.md says so).
void generate_pe(Engine& e, int layer, int dim, uint64_t seed) {
  OB_CHECK(e.g.N > 0, OB_ESTATE, "generate the graph before stored embeddings");
  OB_CHECK(layer >= 1 && layer <= 7 && dim >= 1, OB_EINVAL, "bad stored-embedding layer or width");
  if ((int)e.pe.size() < layer) {
    e.pe.resize(layer, nullptr);
    e.pe_dim.resize(layer, 0);
  }
  const int ld = ld4(dim);
  const int64_t rows = e.g.pos ? std::max<int64_t>(e.g.N_local, 1) : e.g.N;
  e.dfree(e.pe[layer - 1]);
  float* d = (float*)e.dalloc(sizeof(float) * rows * ld);
  launch_pdl(k_gen_rows, dim3(grid_for(e.g.N * ld, 256)), dim3(256), 0, e.stream, e.g.N, dim, ld, seed * 0x9E3779B97F4A7C15ull + layer,
                                                              e.g.pos, d);
  OB_CUDA(cudaStreamSynchronize(e.stream));
  e.pe[layer - 1] = d;
  e.pe_dim[layer - 1] = dim;
}

}  // namespace ob
