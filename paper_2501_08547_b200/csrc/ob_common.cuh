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
#include <cub/block/block_scan.cuh>
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

inline int grid_for(int64_t work, int per_cta, int cap = kPersistCTAs) {
  int64_t g = (work + per_cta - 1) / per_cta;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

__device__ __forceinline__ int64_t dev_count(const int64_t* p, int64_t fallback) {
  return p ? *p : fallback;
}

// ---------------------------------------------------------------------------
// bitmap-rank set over [0, n_bits)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bm_set(uint32_t* bits, int64_t v) {
  atomicOr(bits + (v >> 5), 1u << (v & 31));
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
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicOr(bits + word, orv);
}
// rank of v among set bits (v need not be set: counts set bits below v)
__device__ __forceinline__ int64_t bm_rank(const uint32_t* bits, const int64_t* wpre, int64_t v) {
  uint32_t w = __ldg(bits + (v >> 5));
  return __ldg(wpre + (v >> 5)) + __popc(w & ((1u << (v & 31)) - 1u));
}

// ---------------------------------------------------------------------------
// 3-phase exclusive scan with a device-resident item count
//   out[i] = sum_{j<i} load(j) for i in [0, n]; *total = out[n]
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class Load>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(Load load, const int64_t* n_dev, int64_t n_host,
                                                              int64_t* tile_sums) {
  using BR = cub::BlockReduce<int64_t, kScanThreads>;
  __shared__ typename BR::TempStorage tmp;
  const int64_t n = dev_count(n_dev, n_host);
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int64_t base = t * kScanTile;
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
      if (idx < n) s += load(idx);
    }
    int64_t r = BR(tmp).Sum(s);
    if (threadIdx.x == 0) tile_sums[t] = r;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) k_scan_tiles(const int64_t* n_dev, int64_t n_host, int64_t* tile_sums,
                                                     int64_t* total_out, int64_t* out_arr);

template <class Load, class Store>
__global__ void __launch_bounds__(kScanThreads) k_scan_downsweep(Load load, Store store, const int64_t* n_dev,
                                                                 int64_t n_host, const int64_t* tile_sums) {
  using BS = cub::BlockScan<int64_t, kScanThreads>;
  __shared__ typename BS::TempStorage tmp;
  const int64_t n = dev_count(n_dev, n_host);
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int64_t base = t * kScanTile + (int64_t)threadIdx.x * kScanItems;  // blocked arrangement
    int64_t v[kScanItems];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) v[i] = (base + i < n) ? load(base + i) : 0;
    int64_t agg;
    BS(tmp).ExclusiveSum(v, v, agg);
    int64_t off = tile_sums[t];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
      if (base + i < n) store(base + i, v[i] + off);
    __syncthreads();
  }
}

// Host driver.  `max_n` bounds the device count (sizes tile_sums).  Writes
// out[n] via the tile kernel (out_total) and optionally a second copy.
struct ScanScratch {
  int64_t* tile_sums = nullptr;  // >= max_tiles + 1
  int64_t max_tiles = 0;
};

// out_arr (optional): the plain array behind `store`; out_arr[n] = total is written.
template <class Load, class Store>
void device_scan(cudaStream_t s, const ScanScratch& sc, Load load, Store store, const int64_t* n_dev,
                 int64_t n_host, int64_t max_n, int64_t* total_out, int64_t* out_arr = nullptr) {
  int64_t tiles = (max_n + kScanTile - 1) / kScanTile;
  if (tiles < 1) tiles = 1;
  OB_CHECK(tiles <= sc.max_tiles, OB_ESTATE, "scan scratch too small");
  int g = grid_for(tiles, 1, kNumSMs * 2);
  k_scan_reduce<<<g, kScanThreads, 0, s>>>(load, n_dev, n_host, sc.tile_sums);
  k_scan_tiles<<<1, 1024, 0, s>>>(n_dev, n_host, sc.tile_sums, total_out, out_arr);
  k_scan_downsweep<<<g, kScanThreads, 0, s>>>(load, store, n_dev, n_host, sc.tile_sums);
  g_launches += 3;
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

__global__ void k_fill_i32(int32_t* a, const int64_t* n_dev, int64_t n_host, int32_t v);
__global__ void k_fill_i64(int64_t* a, const int64_t* n_dev, int64_t n_host, int64_t v);

}  // namespace ob
