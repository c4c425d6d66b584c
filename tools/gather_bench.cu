// gather_bench.cu -- how fast can a B200 gather 512-byte rows at random?
//
// The aggregation kernel (k_agg) reads one 128-float row per edge from a
// table that is ~L2-sized, so its ceiling is the row-gather rate of the memory
// system, not HBM.  This standalone probe measures that rate three ways on the
// same indices (uniform random over S rows, E edges, 128-edge work items):
//   ldg<U>   one warp per item, U rows in flight per warp (the k_agg scheme)
//   tma      one warp per item, rows fetched by TMA (cp.async.bulk.tensor 2D,
//            one 1 x 128 box per row) into a 16-slot shared ring, mbarrier per slot
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda tools/gather_bench.cu -o /tmp/gb
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));       \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

constexpr int W = 128;  // row width (floats)

template <int U>
__global__ void __launch_bounds__(128) k_ldg(const float* __restrict__ tab, const int* __restrict__ idx, long E,
                                             float* out) {
  const int lane = threadIdx.x & 31;
  const long items = E / 128;
  const long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long it = gw; it < items; it += nw) {
    const int my[4] = {idx[it * 128 + lane], idx[it * 128 + 32 + lane], idx[it * 128 + 64 + lane],
                       idx[it * 128 + 96 + lane]};
    float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll
    for (int b = 0; b < 128; b += U) {
      float4 v[U];
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const int r = __shfl_sync(0xffffffffu, my[(b + x) >> 5], (b + x) & 31);
        v[x] = __ldg(reinterpret_cast<const float4*>(tab + (long)r * W) + lane);
      }
#pragma unroll
      for (int x = 0; x < U; ++x) acc.x += v[x].x, acc.y += v[x].y, acc.z += v[x].z, acc.w += v[x].w;
    }
    reinterpret_cast<float4*>(out)[it * 32 + lane] = acc;
  }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kSlots = 16;
__global__ void __launch_bounds__(128) k_tma(const __grid_constant__ CUtensorMap map, const int* __restrict__ idx,
                                             long E, float* out) {
  __shared__ __align__(1024) float ring[4][kSlots][W];  // 4 warps x 16 slots x 512 B = 32 KB
  __shared__ __align__(8) uint64_t bar[4][kSlots];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane < kSlots) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[warp][lane])));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t phase = 0;  // bit s = parity of slot s
  const long items = E / 128;
  const long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long it = gw; it < items; it += nw) {
    const int my[4] = {idx[it * 128 + lane], idx[it * 128 + 32 + lane], idx[it * 128 + 64 + lane],
                       idx[it * 128 + 96 + lane]};
    auto issue = [&](int r, int slot) {  // lane 0 issues
      const int row = __shfl_sync(0xffffffffu, my[r >> 5], r & 31);
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[warp][slot])),
                     "r"(W * 4)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(su32(&ring[warp][slot][0])),
            "l"(&map), "r"(0), "r"(row), "r"(su32(&bar[warp][slot]))
            : "memory");
      }
    };
#pragma unroll
    for (int r = 0; r < kSlots; ++r) issue(r, r);
    float4 acc = make_float4(0, 0, 0, 0);
    for (int r = 0; r < 128; ++r) {
      const int slot = r % kSlots;
      const uint32_t par = (phase >> slot) & 1u;
      asm volatile(
          "{\n\t.reg .pred P1;\n"
          "W_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra W_%=;\n"
          "D_%=:\n\t}" ::"r"(su32(&bar[warp][slot])),
          "r"(par)
          : "memory");
      phase ^= 1u << slot;
      const float4 v = reinterpret_cast<const float4*>(ring[warp][slot])[lane];
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
      __syncwarp();
      if (r + kSlots < 128) issue(r + kSlots, slot);
    }
    reinterpret_cast<float4*>(out)[it * 32 + lane] = acc;
  }
}

int main(int argc, char** argv) {
  const long S = argc > 1 ? atol(argv[1]) : 222000;
  const long E = (argc > 2 ? atol(argv[2]) : 5900000) / 128 * 128;
  std::vector<int> h(E);
  unsigned long long x = 88172645463325252ull;
  for (long i = 0; i < E; ++i) {
    x ^= x << 13, x ^= x >> 7, x ^= x << 17;
    h[i] = (int)(x % S);
  }
  float *tab, *out;
  int* idx;
  CK(cudaMalloc(&tab, S * W * 4));
  CK(cudaMalloc(&out, E / 128 * W * 4));
  CK(cudaMalloc(&idx, E * 4));
  CK(cudaMemset(tab, 0, S * W * 4));
  CK(cudaMemcpy(idx, h.data(), E * 4, cudaMemcpyHostToDevice));
  void* big;
  CK(cudaMalloc(&big, 512 << 20));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)S};
  cuuint64_t strides[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {W, 1}, es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("tensor map encode failed\n");
    return 1;
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemset(big, rep, 512 << 20));  // flush L2
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) best = ms < best ? ms : best;
    }
    CK(cudaGetLastError());
    printf("%-10s %8.1f us   %6.2f TB/s of gathered rows\n", name, best * 1e3, E * W * 4.0 / (best * 1e-3) / 1e12);
  };
  for (int g : {148 * 7, 148 * 14, 148 * 16}) {
    printf("grid %d\n", g);
    run("ldg<4>", [&] { k_ldg<4><<<g, 128>>>(tab, idx, E, out); });
    run("ldg<8>", [&] { k_ldg<8><<<g, 128>>>(tab, idx, E, out); });
    run("ldg<16>", [&] { k_ldg<16><<<g, 128>>>(tab, idx, E, out); });
    run("tma16", [&] { k_tma<<<g, 128>>>(map, idx, E, out); });
  }
  return 0;
}
