// ob_common.cuh -- shared device helpers for libomega_b200 (sm_100a).
//
// * error plumbing (ob::Error carries an ob_status code up to the C ABI)
// * bitmap-rank sets: dedup + ascending order + O(1) relabel in one structure
//   (bit per id, exclusive popcount prefix per 32-bit word)
// * device-count scans: every size a request produces lives in device memory,
//   so kernels are launched persistently (grid = k x 148 SMs) and loop over
//   the count they read; no host round trip between stages.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_exchange.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <type_traits>
#include <stdexcept>
#include <string>

#include "../../include/ob_api.h"

namespace ob {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define OB_CUDA(x)                                                                       \
  do {                                                                                   \
    cudaError_t _e = (x);                                                                \
    if (_e != cudaSuccess)                                                               \
      throw ::ob::Error(_e == cudaErrorMemoryAllocation ? OB_ENOMEM : OB_ECUDA,          \
                        std::string(#x) + ": " + cudaGetErrorString(_e));                \
  } while (0)

#define OB_CHECK(cond, code, msg)                  \
  do {                                             \
    if (!(cond)) throw ::ob::Error((code), (msg)); \
  } while (0)

constexpr int kNumSMs = 148;        // B200: 2 dies x 74 SMs
constexpr int kPersistCTAs = kNumSMs * 8;

// Launch accounting (own kernels only) -- reported as gpu_launches by bench.py.
extern int64_t g_launches;
#define OB_LAUNCHED() (++::ob::g_launches)

// Programmatic dependent launch for the per-layer kernel chain: the next kernel's
// CTAs are scheduled onto SMs as the previous kernel's tail drains and run their
// prologue; every such kernel calls pdl_wait() before it touches its
// predecessors' results (griddepcontrol.wait: returns once the prerequisite grid
// has completed and flushed; a no-op for an ordinary launch).  OB_NO_PDL=1 turns
// the attribute off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
// programmatic dependent launch on every kernel (OB_NO_PDL=1 turns it off)
inline int launch_attrs(cudaLaunchAttribute* at) {
  if (!pdl_enabled()) return 0;
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  return 1;
}
template <class... KArgs, class... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  cfg.attrs = at;
  cfg.numAttrs = launch_attrs(at);
  OB_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  OB_LAUNCHED();
}

inline int grid_for(int64_t work, int per_cta, int cap = kPersistCTAs) {
  int64_t g = (work + per_cta - 1) / per_cta;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// Request state that earlier kernels of the same request update (counters, selection state)
// is read past L1 (ld.global.cg): an SM's L1 may still hold a sector cached by a CTA of a
// concurrent kernel from the request's other streams after the writer's update reached L2.
__device__ __forceinline__ int64_t ld_state(const int64_t* p) { return __ldcg(reinterpret_cast<const long long*>(p)); }
__device__ __forceinline__ uint64_t ld_state(const uint64_t* p) {
  return __ldcg(reinterpret_cast<const unsigned long long*>(p));
}
__device__ __forceinline__ int64_t dev_count(const int64_t* p, int64_t fallback) {
  return p ? ld_state(p) : fallback;
}
// The same, one L2 read per CTA broadcast through shared memory: every thread of the CTA
// must reach it (a per-thread ld.global.cg of one hot word from every warp of a large grid
// queues thousands of requests on a single L2 line)
__device__ __forceinline__ int64_t cta_ld(const int64_t* p) {
  __shared__ int64_t s_cta_word;
  __syncthreads();  // every thread has taken the previous broadcast
  if (threadIdx.x == 0) s_cta_word = ld_state(p);
  __syncthreads();
  return s_cta_word;
}
__device__ __forceinline__ uint64_t cta_ld(const uint64_t* p) {
  return (uint64_t)cta_ld(reinterpret_cast<const int64_t*>(p));
}
__device__ __forceinline__ int64_t cta_count(const int64_t* p, int64_t fallback) {
  return p ? cta_ld(p) : fallback;
}
// Up to four words in one round trip (null pointers read as 0); every thread of the CTA must
// reach it and the CTA must have at least as many threads as non-null pointers
struct CtaWords {
  int64_t v[4];
};
__device__ __forceinline__ CtaWords cta_ldv(const void* p0, const void* p1, const void* p2 = nullptr,
                                            const void* p3 = nullptr) {
  __shared__ int64_t s_cta_words[4];
  __syncthreads();
  if (threadIdx.x < 4) {
    const void* p = threadIdx.x == 0 ? p0 : threadIdx.x == 1 ? p1 : threadIdx.x == 2 ? p2 : p3;
    s_cta_words[threadIdx.x] = p ? ld_state(static_cast<const int64_t*>(p)) : 0;
  }
  __syncthreads();
  return CtaWords{{s_cta_words[0], s_cta_words[1], s_cta_words[2], s_cta_words[3]}};
}

// ---------------------------------------------------------------------------
// bitmap-rank set over [0, n_bits)
// ---------------------------------------------------------------------------
// test before set: re-marking an already set bit (the common case when a
// source feeds many destinations) costs an L2 read instead of an L2 atomic
__device__ __forceinline__ void bm_set(uint32_t* bits, int64_t v) {
  const uint32_t m = 1u << (v & 31);
  if (!(__ldcg(bits + (v >> 5)) & m)) atomicOr(bits + (v >> 5), m);
}
__device__ __forceinline__ bool bm_test(const uint32_t* bits, int64_t v) {
  return (__ldg(bits + (v >> 5)) >> (v & 31)) & 1u;
}
// warp-aggregated bm_set: lanes hitting the same word OR their bits first
__device__ __forceinline__ void bm_set_warp(uint32_t* bits, int64_t v) {
  const unsigned act = __activemask();
  const uint32_t word = (uint32_t)(v >> 5);
  const unsigned peers = __match_any_sync(act, word);
  const uint32_t orv = __reduce_or_sync(peers, 1u << (v & 31));
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1 && (__ldcg(bits + word) & orv) != orv) atomicOr(bits + word, orv);
}
// rank of v among set bits (v need not be set: counts set bits below v)
__device__ __forceinline__ int64_t bm_rank(const uint32_t* bits, const int64_t* wpre, int64_t v) {
  uint32_t w = __ldg(bits + (v >> 5));
  return __ldg(wpre + (v >> 5)) + __popc(w & ((1u << (v & 31)) - 1u));
}

// ---------------------------------------------------------------------------
// Single-pass exclusive scan (decoupled look-back) with a device-resident count
//   out[i] = sum_{j<i} load(j) for i in [0, n]; total(n, out[n])
// Tiles are claimed in order from an atomic ticket, so every predecessor of a
// tile is already resident and the look-back cannot deadlock.  Each tile
// publishes its aggregate, then its inclusive prefix; warp 0 of a tile walks
// back 32 predecessors at a time until it meets an inclusive prefix.
// The per-scan state (ticket, flags, aggregates, prefixes) is a slice of a
// zeroed pool; the request zeroes what it used when it finishes.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
#ifndef OB_SCAN_MINB
#define OB_SCAN_MINB 2  // int64 scan CTAs resident per SM (I3 scans keep one: 3x the registers)
#endif

// three running sums scanned together (block assembly: edges, items, groups)
struct I3 {
  int64_t a, b, c;
  I3() = default;
  __host__ __device__ constexpr I3(int64_t x) : a(x), b(x), c(x) {}
  __host__ __device__ constexpr I3(int64_t x, int64_t y, int64_t z) : a(x), b(y), c(z) {}
};
__host__ __device__ inline I3 operator+(const I3& x, const I3& y) { return I3(x.a + y.a, x.b + y.b, x.c + y.c); }

__device__ __forceinline__ int64_t shfl_xor_t(int64_t v, int o) {
  return (int64_t)__shfl_xor_sync(0xffffffffu, (long long)v, o);
}
__device__ __forceinline__ I3 shfl_xor_t(const I3& v, int o) {
  return I3(shfl_xor_t(v.a, o), shfl_xor_t(v.b, o), shfl_xor_t(v.c, o));
}
__device__ __forceinline__ int64_t ldcg_t(const int64_t* p) { return __ldcg(reinterpret_cast<const long long*>(p)); }
__device__ __forceinline__ I3 ldcg_t(const I3* p) {
  const long long* q = reinterpret_cast<const long long*>(p);
  return I3(__ldcg(q), __ldcg(q + 1), __ldcg(q + 2));
}

template <class T>
struct ScanTiles {
  unsigned long long* ticket;
  int* flag;  // 0 empty, 1 aggregate published, 2 inclusive prefix published
  T* agg;
  T* incl;
};

// Load / Store functors may cache request state once per thread (prepare(), run after
// pdl_wait on a per-thread copy); functors without it are used in place (no copy)
template <class F, class = void>
struct has_prepare : std::false_type {};
template <class F>
struct has_prepare<F, std::void_t<decltype(std::declval<F&>().prepare())>> : std::true_type {};

template <class T, int ITEMS, class Load, class Store, class Total>
__device__ __forceinline__ void scan_tiles(const Load& load, const Store& store, const Total& total,
                                           const int64_t* n_dev, int64_t n_host, const ScanTiles<T>& st);

template <class T, int ITEMS, class Load, class Store, class Total>
__global__ void __launch_bounds__(kScanThreads, sizeof(T) == 8 ? OB_SCAN_MINB : 1) k_scan(Load load, Store store, Total total, const int64_t* n_dev,
                                                       int64_t n_host, ScanTiles<T> st) {
  pdl_wait();
  if constexpr (has_prepare<Load>::value || has_prepare<Store>::value) {
    Load l = load;
    Store o = store;
    if constexpr (has_prepare<Load>::value) l.prepare();
    if constexpr (has_prepare<Store>::value) o.prepare();
    scan_tiles<T, ITEMS>(l, o, total, n_dev, n_host, st);
  } else {
    scan_tiles<T, ITEMS>(load, store, total, n_dev, n_host, st);
  }
}

template <class T, int ITEMS, class Load, class Store, class Total>
__device__ __forceinline__ void scan_tiles(const Load& load, const Store& store, const Total& total,
                                           const int64_t* n_dev, int64_t n_host, const ScanTiles<T>& st) {
  using BS = cub::BlockScan<T, kScanThreads>;
  using BX = cub::BlockExchange<T, kScanThreads, ITEMS>;
  // 8-byte values move warp-striped (coalesced loads and stores) and are
  // transposed to the blocked order the scan needs through shared memory
  constexpr bool kStriped = sizeof(T) == 8;
  struct NoExchange {};
  using XT = typename std::conditional<kStriped, typename BX::TempStorage, NoExchange>::type;
  constexpr int64_t kTile = (int64_t)kScanThreads * ITEMS;
  __shared__ union {
    typename BS::TempStorage scan;
    XT ex;
  } tmp;
  __shared__ int64_t s_tile;
  __shared__ T s_prefix;
  const int64_t n = cta_count(n_dev, n_host);
  const int64_t ntiles = (n + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31;
  if (n <= 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) total(0, T(0));
    return;
  }
  for (;;) {
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(st.ticket, 1ull);
    __syncthreads();
    const int64_t t = s_tile;
    if (t >= ntiles) break;
    T v[ITEMS];
    if constexpr (kStriped) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int64_t idx = t * kTile + (int64_t)i * kScanThreads + threadIdx.x;
        v[i] = idx < n ? T(load(idx)) : T(0);
      }
      BX(tmp.ex).StripedToBlocked(v);
      __syncthreads();
    } else {
      const int64_t base = t * kTile + (int64_t)threadIdx.x * ITEMS;  // blocked arrangement
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) v[i] = (base + i < n) ? T(load(base + i)) : T(0);
    }
    T agg;
    BS(tmp.scan).ExclusiveSum(v, v, agg);
    if (threadIdx.x < 32) {
      T excl(0);
      volatile int* vf = st.flag;
      if (t == 0) {
        if (lane == 0) {
          st.incl[0] = agg;
          __threadfence();
          vf[0] = 2;
        }
      } else {
        if (lane == 0) {
          st.agg[t] = agg;
          __threadfence();
          vf[t] = 1;
        }
        for (int64_t hi = t - 1;;) {
          const int64_t j = hi - lane;
          int f = j >= 0 ? vf[j] : 2;
          const unsigned inc = __ballot_sync(0xffffffffu, f == 2);
          const int first = inc ? __ffs(inc) - 1 : 32;  // nearest inclusive predecessor
          const unsigned need = first == 32 ? 0xffffffffu : (first == 31 ? 0xffffffffu : ((2u << first) - 1u));
          if (__ballot_sync(0xffffffffu, f == 0) & need) continue;  // a predecessor has not published yet
          __threadfence();
          T x(0);
          if (j >= 0 && lane < first) x = ldcg_t(st.agg + j);
          else if (j >= 0 && lane == first) x = ldcg_t(st.incl + j);
#pragma unroll
          for (int o = 16; o; o >>= 1) x = x + shfl_xor_t(x, o);
          excl = excl + x;
          if (first < 32) break;
          hi -= 32;
        }
        if (lane == 0) {
          st.incl[t] = excl + agg;
          __threadfence();
          vf[t] = 2;
        }
      }
      if (lane == 0) s_prefix = excl;
    }
    __syncthreads();
    const T off = s_prefix;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) v[i] = v[i] + off;
    if constexpr (kStriped) {
      BX(tmp.ex).BlockedToStriped(v);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int64_t idx = t * kTile + (int64_t)i * kScanThreads + threadIdx.x;
        if (idx < n) store(idx, v[i]);
      }
    } else {
      const int64_t base = t * kTile + (int64_t)threadIdx.x * ITEMS;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        if (base + i < n) store(base + i, v[i]);
    }
    if (t == ntiles - 1 && threadIdx.x == 0) total(n, off + agg);
    __syncthreads();  // s_tile / s_prefix / tmp are reused by the next tile
  }
}

// Pool of zeroed per-scan state.  `cursor` advances per scan on the host (so a
// captured graph bakes in fixed slices); clear() zeroes the used part.
struct ScanScratch {
  char* pool = nullptr;
  size_t cap = 0;
  size_t cursor = 0;
  static size_t slice_bytes(int64_t max_n) {
    const size_t tiles = (size_t)(max_n / kScanTile + 2);
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    return 256 + al(tiles * sizeof(int)) + 2 * al(tiles * sizeof(I3));
  }
  static size_t bytes_for(int64_t max_n, int scans) { return slice_bytes(max_n) * (size_t)scans; }
  template <class T>
  ScanTiles<T> take(int64_t max_n) {
    const size_t tiles = (size_t)(max_n / kScanTile + 2);
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t need = 256 + al(tiles * sizeof(int)) + 2 * al(tiles * sizeof(T));
    if (cursor + need > cap) throw Error(OB_ESTATE, "scan pool too small");
    char* p = pool + cursor;
    cursor += need;
    ScanTiles<T> st;
    st.ticket = reinterpret_cast<unsigned long long*>(p);
    st.flag = reinterpret_cast<int*>(p + 256);
    st.agg = reinterpret_cast<T*>(p + 256 + al(tiles * sizeof(int)));
    st.incl = reinterpret_cast<T*>(p + 256 + al(tiles * sizeof(int)) + al(tiles * sizeof(T)));
    return st;
  }
  void clear(cudaStream_t s) {
    if (cursor) OB_CUDA(cudaMemsetAsync(pool, 0, cursor, s));
    cursor = 0;
  }
};

struct TotalI64 {
  int64_t* total_out;
  int64_t* out_arr;
  __device__ void operator()(int64_t n, int64_t v) const {
    if (total_out) *total_out = v;
    if (out_arr) out_arr[n] = v;
  }
};

// Reduce-then-scan variant for very long inputs (bitmaps over 10^8 ids): with
// thousands of 4096-element tiles the single-pass look-back chain, not
// bandwidth, sets the time; three bandwidth-bound passes are shorter.
template <class Load>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(Load load, const int64_t* n_dev, int64_t n_host,
                                                              int64_t* tile_sums) {
  pdl_wait();
  using BR = cub::BlockReduce<int64_t, kScanThreads>;
  __shared__ typename BR::TempStorage tmp;
  const int64_t n = cta_count(n_dev, n_host);
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int64_t v = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const int64_t idx = t * kScanTile + (int64_t)i * kScanThreads + threadIdx.x;
      if (idx < n) v += load(idx);
    }
    const int64_t r = BR(tmp).Sum(v);
    if (threadIdx.x == 0) tile_sums[t] = r;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) k_scan_spine(const int64_t* n_dev, int64_t n_host, int64_t* tile_sums);

template <class Load, class Store, class Total>
__global__ void __launch_bounds__(kScanThreads, OB_SCAN_MINB) k_scan_down(Load load, Store store, Total total,
                                                            const int64_t* n_dev, int64_t n_host,
                                                            const int64_t* tile_off) {
  pdl_wait();
  using BS = cub::BlockScan<int64_t, kScanThreads>;
  using BX = cub::BlockExchange<int64_t, kScanThreads, kScanItems>;
  __shared__ union {
    typename BS::TempStorage scan;
    typename BX::TempStorage ex;
  } tmp;
  const int64_t n = cta_count(n_dev, n_host);
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  if (n <= 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) total(0, 0);
    return;
  }
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int64_t v[kScanItems];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const int64_t idx = t * kScanTile + (int64_t)i * kScanThreads + threadIdx.x;
      v[i] = idx < n ? (int64_t)load(idx) : 0;
    }
    BX(tmp.ex).StripedToBlocked(v);
    __syncthreads();
    int64_t agg;
    BS(tmp.scan).ExclusiveSum(v, v, agg);
    const int64_t off = tile_off[t];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) v[i] += off;
    __syncthreads();
    BX(tmp.ex).BlockedToStriped(v);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const int64_t idx = t * kScanTile + (int64_t)i * kScanThreads + threadIdx.x;
      if (idx < n) store(idx, v[i]);
    }
    if (t == ntiles - 1 && threadIdx.x == 0) total(n, off + agg);
    __syncthreads();
  }
}

template <class T, class Load, class Store, class Total>
void device_scan_t(cudaStream_t s, ScanScratch& sc, Load load, Store store, Total total, const int64_t* n_dev,
                   int64_t n_host, int64_t max_n) {
  ScanTiles<T> st = sc.take<T>(max_n);
  const int64_t tiles = (max_n + kScanTile - 1) / kScanTile;
  const int g = grid_for(tiles < 1 ? 1 : tiles, 1, kNumSMs * 2);
  if constexpr (std::is_same<T, int64_t>::value) {
    if (tiles > 4 * kNumSMs) {  // long input: reduce, spine, downsweep
      int64_t* sums = reinterpret_cast<int64_t*>(st.agg);
      launch_pdl(k_scan_reduce<Load>, dim3(g), dim3(kScanThreads), 0, s, load, n_dev, n_host, sums);
      launch_pdl(k_scan_spine, dim3(1), dim3(1024), 0, s, n_dev, n_host, sums);
      launch_pdl(k_scan_down<Load, Store, Total>, dim3(g), dim3(kScanThreads), 0, s, load, store, total, n_dev, n_host,
                 (const int64_t*)sums);
      return;
    }
  }
  launch_pdl(k_scan<T, kScanItems, Load, Store, Total>, dim3(g), dim3(kScanThreads), 0, s, load, store, total, n_dev,
             n_host, st);
}

// int64 scan; out_arr (optional): the plain array behind `store`, out_arr[n] = total.
template <class Load, class Store>
void device_scan(cudaStream_t s, ScanScratch& sc, Load load, Store store, const int64_t* n_dev, int64_t n_host,
                 int64_t max_n, int64_t* total_out, int64_t* out_arr = nullptr) {
  device_scan_t<int64_t>(s, sc, load, store, TotalI64{total_out, out_arr}, n_dev, n_host, max_n);
}

// Common loaders / stores.
struct LoadPopc {
  const uint32_t* bits;
  __device__ int64_t operator()(int64_t i) const { return __popc(bits[i]); }
};
struct LoadI64 {
  const int64_t* a;
  __device__ int64_t operator()(int64_t i) const { return a[i]; }
};
struct LoadI32 {
  const int32_t* a;
  __device__ int64_t operator()(int64_t i) const { return a[i]; }
};
struct StoreI64 {
  int64_t* a;
  __device__ void operator()(int64_t i, int64_t v) const { a[i] = v; }
};

// Simple grid-stride helpers.
#define OB_GRID_STRIDE(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)


}  // namespace ob
