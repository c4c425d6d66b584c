// ob_gemm.cu -- dense layer transforms on the 5th-gen tensor cores (tcgen05).
//
// C[M x N] = epi( [A1 | A2] @ B ), M device-resident, K = K1 + K2, N <= 256.
//   A1 rows are gathered through per-row pointers (features / query features /
//   stored embeddings / previous layer rows -- never materialised), A2 rows are
//   a dense matrix (the aggregation result).
//
// Precision: the reference accumulates in float64 (models.py:214-228) and the
// parity bar is 1e-4 relative in fp32, which single-pass TF32 (10-bit mantissa)
// misses.  We use the 3xTF32 split: A = A_hi + A_lo, B = B_hi + B_lo, and
// D = A_hi B_hi + A_hi B_lo + A_lo B_hi accumulated in an fp32 TMEM tile.
// B_hi / B_lo are prepared once at model load (weights are static).
//
// Warp-specialized persistent kernel, one CTA per SM, 128-row tiles:
//   warps 0-3  A producers: gather A k-blocks (32 fp32 = one 128-byte row
//              segment per tile row; 8 threads per segment, coalesced) with
//              cp.async into the canonical K-major SWIZZLE_128B layout of an
//              SA-deep ring, completion via cp.async.mbarrier.arrive.noinc
//   warp 13    weight tiles: B_hi / B_lo k-blocks by TMA (cp.async.bulk.tensor,
//              128B swizzle) into a separate, shorter SB-deep ring
//   warps 4-7  transform: A_lo = a - trunc_tf32(a) written to TMEM with
//              tcgen05.st (N <= 128; in place in shared memory for N = 256);
//              the tensor core truncates the raw tile to A_hi itself
//   warp 12    MMA issuer: 12 x tcgen05.mma.kind::tf32 (A B_hi, A B_lo from
//              shared memory, A_lo B_hi with A from TMEM; 4 K=8 steps) per
//              k-block into one of two TMEM accumulators; tcgen05.commit frees
//              the A and B stages / publishes the accumulator
//   warps 8-11 epilogue: tcgen05.ld 32x32b -> smem transpose -> coalesced
//              addend + activation + store, overlapping the next tile's MMAs
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "ob_engine.h"

namespace ob {

namespace {

constexpr int kTcBM = 128;
constexpr int kTcBK = 32;                  // fp32 per k-block: one 128-byte swizzle row
constexpr int kTileA = kTcBM * kTcBK * 4;  // 16 KB
constexpr int kWarpsProd = 4, kWarpsXf = 4, kWarpsEpi = 4;
constexpr int kTcThreads = (kWarpsProd + kWarpsXf + kWarpsEpi + 2) * 32;  // 448: + MMA warp + TMA warp
constexpr int kMmaWarp = kWarpsProd + kWarpsXf + kWarpsEpi;               // 12

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
// arrive on the barrier when all of this thread's prior cp.async have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, SWIZZLE_128B shared-memory matrix descriptor (sm_100 "version 1")
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);  // start address
  d |= (uint64_t)1 << 16;                   // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;         // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                   // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
  return d;
}

// kind::tf32 instruction descriptor: fp32 accumulate, K-major A and B, M = 128
__host__ __device__ constexpr uint32_t tf32_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t addr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace

// Shared memory: an SA-stage ring of gathered A tiles (+ A_lo when it cannot
// live in TMEM), a separate SB-stage ring of {B_hi, B_lo} tiles, and the
// epilogue transpose tiles.  Splitting the rings lets the A gather (HBM
// latency, the long pole) run up to SA k-blocks ahead while the weight tiles
// (L2-resident, shared by every CTA) only need a short ring.
constexpr int cmin(int a, int b) { return a < b ? a : b; }

template <int NP>
struct TcSmem {
  // A_lo lives in TMEM (written by the transform warps with tcgen05.st) when the
  // two accumulators leave room for it
  static constexpr bool kLoTmem = NP <= 128;
  static constexpr int kTileB = NP * kTcBK * 4;
  static constexpr int kStageA = (kLoTmem ? 1 : 2) * kTileA;
  static constexpr int kStageB = 2 * kTileB;
  static constexpr int kEpi = kWarpsEpi * 32 * 32 * 4;  // 16 KB
  static constexpr int kFixed = kEpi + 1024 /*align*/ + 1024 /*bars*/;
  static constexpr int kBudget = 227 * 1024 - kFixed;
  static constexpr int kSB = NP >= 256 ? 2 : 3;
  static constexpr uint32_t kAccCols = 2 * NP;  // two accumulators
  static constexpr int kSA0 = cmin(8, cmin((kBudget - kSB * kStageB) / kStageA,
                                           kLoTmem ? (int)((512 - kAccCols) / kTcBK) : 8));
  static constexpr int kSA = kSA0 < 2 ? 2 : kSA0;
  static constexpr int kBytes = kSA * kStageA + kSB * kStageB + kFixed;
  static constexpr uint32_t kLoCol = kAccCols;  // then kSA x 32 A_lo columns
  static constexpr uint32_t kNeed = kAccCols + (kLoTmem ? kSA * kTcBK : 0);
  static constexpr uint32_t kCols = kNeed <= 64 ? 64 : (kNeed <= 128 ? 128 : (kNeed <= 256 ? 256 : 512));
  static_assert(kNeed <= 512, "TMEM budget");
  static_assert(kBytes <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ void tmem_st32(uint32_t addr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// A operand from TMEM (the A_lo x B_hi product)
__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc),
      "r"(idesc));
}

template <int NP>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_tc_gemm(TcGemmArgs g, const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo) {
  using SM = TcSmem<NP>;
  constexpr int SA = SM::kSA, SB = SM::kSB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // offset (not an integer cast) keeps the pointer in the shared window -> LDS/STS
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring_a = base;
  uint8_t* ring_b = base + SA * SM::kStageA;
  float* epi_buf = reinterpret_cast<float*>(ring_b + SB * SM::kStageB);
  uint64_t* full_a = reinterpret_cast<uint64_t*>(ring_b + SB * SM::kStageB + SM::kEpi);
  uint64_t* ready_a = full_a + SA;
  uint64_t* empty_a = ready_a + SA;
  uint64_t* full_b = empty_a + SA;
  uint64_t* empty_b = full_b + SB;
  uint64_t* tfull = empty_b + SB;  // [2]
  uint64_t* tempty = tfull + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KB1 = (g.K1 + kTcBK - 1) / kTcBK, KB2 = (g.K2 + kTcBK - 1) / kTcBK, KB = KB1 + KB2;

  if (tid == 0) {
    for (int i = 0; i < SA; ++i) {
      mbar_init(full_a + i, kWarpsProd * 32);  // cp.async arrivals
      mbar_init(ready_a + i, kWarpsXf * 32);
      mbar_init(empty_a + i, 1);
    }
    for (int i = 0; i < SB; ++i) {
      mbar_init(full_b + i, 1);  // the TMA expect_tx arrival
      mbar_init(empty_b + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, kWarpsEpi * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(SM::kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the set-up above (barriers, TMEM allocation) overlaps the previous kernel's tail;
  // everything below may read its results (the row count M is one of them)
  pdl_wait();
  const int64_t M = ld_state(g.M_dev);
  const int64_t tiles = (M + kTcBM - 1) / kTcBM;
  // work units: (row tile, column slab); small-M GEMMs split the columns across
  // CTAs (nslab > 1) so more SMs share the tile's MMAs and epilogue
  const int ns = g.nslab;
  const int64_t units = tiles * ns;

  if (warp < kWarpsProd) {
    // ---------------- A producers ----------------
    // thread t copies 16-byte chunk (t & 7) of rows (t >> 3) + 16 i: each warp
    // instruction moves four whole 128-byte row segments (coalesced), not 32
    // scattered 16-byte pieces
    constexpr int kRowsPer = kTcBM / (kWarpsProd * 32 / 8);  // 8 rows per thread
    const int c = tid & 7, r0 = tid >> 3;
    uint32_t gk = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int64_t tile = u / ns;
      const float* p1[kRowsPer];
      const float* p2[kRowsPer];
#pragma unroll
      for (int i = 0; i < kRowsPer; ++i) {
        const int64_t row = tile * kTcBM + r0 + 16 * i;
        p1[i] = (row < M && g.K1) ? g.a1.row(g.self ? (int64_t)g.self[row] : row) : nullptr;
        p2[i] = (row < M && g.K2) ? g.a2 + row * g.lda2 : nullptr;
      }
      for (int kb = 0; kb < KB; ++kb, ++gk) {
        const int s = gk % SA;
        if (gk >= (uint32_t)SA) mbar_wait(empty_a + s, ((gk / SA) - 1) & 1);
        const uint32_t a_s = smem_u32(ring_a + s * SM::kStageA);
        const bool first = kb < KB1;
        const int k = (first ? kb : kb - KB1) * kTcBK + c * 4;
        const int rem = (first ? g.K1 : g.K2) - k;
        const int vb = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
#pragma unroll
        for (int i = 0; i < kRowsPer; ++i) {
          const int r = r0 + 16 * i;
          const float* rp = first ? p1[i] : p2[i];
          const int bytes = rp ? vb : 0;
          const float* src = bytes ? rp + k : g.Bt;  // any valid address when 0 bytes are read
          cp_async16(a_s + r * 128 + ((c ^ (r & 7)) << 4), src, bytes);
        }
        cp_async_arrive(full_a + s);
      }
    }
  } else if (warp < kWarpsProd + kWarpsXf) {
    // ---------------- transform: A_lo = a - trunc_tf32(a) ----------------
    uint32_t gk = 0;
    if constexpr (SM::kLoTmem) {
      // row r = this warp's TMEM lane quadrant x 32 + lane: read the (swizzled)
      // 128-byte row, write A_lo to this stage's TMEM columns
      const int q = warp & 3, r = q * 32 + lane;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        for (int kb = 0; kb < KB; ++kb, ++gk) {
          const int s = gk % SA;
          mbar_wait(full_a + s, (gk / SA) & 1);
          const uint8_t* rowp = ring_a + s * SM::kStageA + r * 128;
          float lo[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = *reinterpret_cast<const float4*>(rowp + ((c ^ (r & 7)) << 4));
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) lo[c * 4 + j] = vv[j] - __uint_as_float(__float_as_uint(vv[j]) & 0xFFFFE000u);
          }
          tmem_st32(tmem + ((uint32_t)(q * 32) << 16) + SM::kLoCol + s * kTcBK, lo);
          fence_proxy_async();  // the cp.async-written A tile is read by the tensor core
          tc_fence_before();
          mbar_arrive(ready_a + s);
        }
      }
    } else {
      // in place: trunc_tf32(a) in the A tile, A_lo in the stage's second tile
      const int t = tid - kWarpsProd * 32;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        for (int kb = 0; kb < KB; ++kb, ++gk) {
          const int s = gk % SA;
          mbar_wait(full_a + s, (gk / SA) & 1);
          float* a = reinterpret_cast<float*>(ring_a + s * SM::kStageA);
          float* alo = a + kTcBM * kTcBK;
#pragma unroll
          for (int i = t * 4; i < kTcBM * kTcBK; i += kWarpsXf * 32 * 4) {
            const float4 v = *reinterpret_cast<const float4*>(a + i);
            float4 h, o;
            h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
            h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
            h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
            h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
            o.x = v.x - h.x, o.y = v.y - h.y, o.z = v.z - h.z, o.w = v.w - h.w;
            *reinterpret_cast<float4*>(a + i) = h;
            *reinterpret_cast<float4*>(alo + i) = o;
          }
          fence_proxy_async();
          mbar_arrive(ready_a + s);
        }
      }
    }
  } else if (warp < kMmaWarp) {
    // ---------------- epilogue: TMEM -> smem transpose -> global ----------------
    const int q = warp - (kWarpsProd + kWarpsXf);  // TMEM lane quadrant (warp % 4)
    float* buf = epi_buf + q * 1024;
    uint32_t ti = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++ti) {
      const int64_t tile = u / ns;
      const int n0 = (int)(u % ns) * NP;  // first column of this unit's slab
      const int acc = ti & 1;
      mbar_wait(tfull + acc, (ti >> 1) & 1);
      tc_fence_after();
      const int64_t m0 = tile * kTcBM;
#pragma unroll 1
      for (int c0 = 0; c0 < NP; c0 += 32) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * NP + c0, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) buf[lane * 32 + (j ^ lane)] = v[j];
        __syncwarp();
        const int col = n0 + c0 + lane;
        const int64_t r0 = m0 + q * 32;
        if (g.E) {  // all 32 addend loads in flight before any is consumed
#pragma unroll
          for (int r = 0; r < 32; ++r)
            v[r] = (r0 + r < M && col < g.N) ? __ldg(g.E + (r0 + r) * g.lde + col) : 0.f;
        }
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const int64_t row = r0 + r;
          if (row < M && col < g.N) {
            float o = buf[r * 32 + (lane ^ r)];
            if (g.E) o += v[r];
            if (g.relu) o = fmaxf(o, 0.f);
            g.C[row * g.ldc + col] = o;
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(tempty + acc);
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer (one elected thread) ----------------
    if (lane == 0) {
      const uint32_t idesc = tf32_idesc(NP);
      uint32_t gk = 0, ti = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++ti) {
        const int acc = ti & 1;
        if (ti >= 2) mbar_wait(tempty + acc, ((ti >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t dcol = tmem + acc * NP;
        for (int kb = 0; kb < KB; ++kb, ++gk) {
          const int sa = gk % SA, sb = gk % SB;
          mbar_wait(ready_a + sa, (gk / SA) & 1);
          mbar_wait(full_b + sb, (gk / SB) & 1);
          tc_fence_after();
          const uint32_t a_s = smem_u32(ring_a + sa * SM::kStageA), alo_s = a_s + kTileA;
          const uint32_t b_s = smem_u32(ring_b + sb * SM::kStageB), blo_s = b_s + SM::kTileB;
#pragma unroll
          for (int kk = 0; kk < kTcBK / 8; ++kk) {
            const uint32_t off = kk * 32;  // 8 tf32 per MMA
            const uint64_t da = sw128_desc(a_s + off);
            const uint64_t db = sw128_desc(b_s + off), dbl = sw128_desc(blo_s + off);
            mma_tf32(dcol, da, db, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
            mma_tf32(dcol, da, dbl, idesc, 1u);
            if constexpr (SM::kLoTmem) mma_tf32_ta(dcol, tmem + SM::kLoCol + sa * kTcBK + kk * 8, db, idesc);
            else mma_tf32(dcol, sw128_desc(alo_s + off), db, idesc, 1u);
          }
          mma_commit(empty_a + sa);  // stages free once these MMAs retire
          mma_commit(empty_b + sb);
        }
        mma_commit(tfull + acc);  // accumulator complete
      }
    }
    __syncwarp();
  } else {
    // ---------------- weight tiles: TMA into the B ring ----------------
    if (lane == 0) {
      uint32_t gk = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int n0 = (int)(u % ns) * NP;
        for (int kb = 0; kb < KB; ++kb, ++gk) {
          const int s = gk % SB;
          if (gk >= (uint32_t)SB) mbar_wait(empty_b + s, ((gk / SB) - 1) & 1);
          const uint32_t b_s = smem_u32(ring_b + s * SM::kStageB);
          mbar_expect_tx(full_b + s, SM::kStageB);
          tma_load_2d(b_s, &map_hi, kb * kTcBK, n0, full_b + s);
          tma_load_2d(b_s + SM::kTileB, &map_lo, kb * kTcBK, n0, full_b + s);
        }
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(SM::kCols));
  }
}

static void tc_gemm_slab(cudaStream_t s, const TcGemmArgs& g, int64_t M_max);

// one launch per <= 256-column weight slab (TMEM holds two 256-column accumulators)
void tc_gemm(cudaStream_t s, const TcGemmArgs& g, int64_t M_max) {
  OB_CHECK(g.w && g.w->map_ready, OB_ESTATE, "tc_gemm: weights not staged");
  if (!g.w->next) return tc_gemm_slab(s, g, M_max);
  for (const TcWeights* w = g.w; w; w = w->next.get()) {
    TcGemmArgs gs = g;
    gs.w = w;
    gs.Bt = w->hi;
    gs.Bt_lo = w->lo;
    gs.N = w->N;
    gs.Np = w->Np;
    gs.C = g.C + w->n0;
    gs.E = g.E ? g.E + w->n0 : nullptr;
    tc_gemm_slab(s, gs, M_max);
  }
}

// Column slabs spread a small-M GEMM over more SMs: lower latency for one request
// at a time, but with request lanes the wider grids take whole SMs (smem, TMEM)
// from the other lanes' kernels, so engines with lanes launch one slab per tile
static thread_local bool t_gemm_slabs = true;
void set_gemm_slabs(bool on) { t_gemm_slabs = on; }

static void tc_gemm_slab(cudaStream_t s, const TcGemmArgs& g0, int64_t M_max) {
  OB_CHECK(g0.N >= 1 && g0.N <= 256, OB_ESTATE, "tc_gemm: N out of range");
  OB_CHECK(g0.w && g0.w->map_ready, OB_ESTATE, "tc_gemm: weights not staged");
  const int64_t tiles = (M_max + kTcBM - 1) / kTcBM;
  TcGemmArgs g = g0;
  // column slabs: pick the split with the fewest unit rounds on 148 SMs per unit of
  // work, charging 15 % per extra slab for re-gathering the A rows
  int np = g.Np, ns = 1;
  double best = 1e30;
  for (int sw : {g.Np, 64, 32}) {
    if (sw > g.Np || (sw != g.Np && !(sw == 64 ? g.w->map64_ready : g.w->map32_ready))) continue;
    const int n = g.Np / sw;
    const double rounds = (double)((tiles * n + kNumSMs - 1) / kNumSMs);
    const double cost = rounds / n * (1.0 + 0.15 * (n - 1));
    if (cost < best - 1e-9) {
      best = cost;
      np = sw;
      ns = n;
    }
  }
  if (const char* v = std::getenv("OB_GEMM_NO_SLABS")) {
    if (v[0] && v[0] != '0') np = g.Np, ns = 1;
  }
  if (!t_gemm_slabs) np = g.Np, ns = 1;
  g.nslab = ns;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles * ns, kNumSMs));
  const unsigned char* mh_raw = np == g.Np ? g.w->map_hi : (np == 64 ? g.w->map_hi64 : g.w->map_hi32);
  const unsigned char* ml_raw = np == g.Np ? g.w->map_lo : (np == 64 ? g.w->map_lo64 : g.w->map_lo32);
  const CUtensorMap& mh = *reinterpret_cast<const CUtensorMap*>(mh_raw);
  const CUtensorMap& ml = *reinterpret_cast<const CUtensorMap*>(ml_raw);
  // smem opt-in is set at weight preparation (tc_gemm_configure), never while a
  // request is being captured into a CUDA graph
  auto go = [&](auto kern, int bytes) { launch_pdl(kern, dim3(grid), dim3(kTcThreads), (size_t)bytes, s, g, mh, ml); };
  if (np == 32) go(k_tc_gemm<32>, TcSmem<32>::kBytes);
  else if (np == 64) go(k_tc_gemm<64>, TcSmem<64>::kBytes);
  else if (np == 128) go(k_tc_gemm<128>, TcSmem<128>::kBytes);
  else if (np == 256) go(k_tc_gemm<256>, TcSmem<256>::kBytes);
  else throw Error(OB_ESTATE, "tc_gemm: padded N must be 32/64/128/256");
}

static void tc_gemm_configure() {
  OB_CUDA(cudaFuncSetAttribute(k_tc_gemm<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<32>::kBytes));
  OB_CUDA(cudaFuncSetAttribute(k_tc_gemm<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<64>::kBytes));
  OB_CUDA(cudaFuncSetAttribute(k_tc_gemm<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<128>::kBytes));
  OB_CUDA(cudaFuncSetAttribute(k_tc_gemm<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<256>::kBytes));
}

// ---------------------------------------------------------------------------
// weight preparation: W (K x N row-major) segments -> Bt / Bt_lo (Np x Kp, K-major,
// zero padded), each K segment padded to 32; TMA maps over both (128B swizzle)
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    OB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    OB_CHECK(p && q == cudaDriverEntryPointSuccess, OB_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static void make_map(void* out, float* base, int Np, int Kp, int box_rows = 0) {
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(out);
  const cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)Np};
  const cuuint64_t strides[1] = {(cuuint64_t)Kp * 4};
  const cuuint32_t box[2] = {(cuuint32_t)kTcBK, (cuuint32_t)(box_rows ? box_rows : Np)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  OB_CHECK(r == CUDA_SUCCESS, OB_ECUDA, "cuTensorMapEncodeTiled failed");
}

static void prep_slab(Engine& e, const std::vector<const float*>& segs, const std::vector<int>& seg_k, int Ntot,
                      int n0, TcWeights* out);

void prep_tc_weights(Engine& e, const std::vector<const float*>& segs, const std::vector<int>& seg_k, int N,
                     TcWeights* out) {
  tc_gemm_configure();
  TcWeights* cur = out;
  for (int n0 = 0; n0 < N; n0 += 256) {  // column slabs of <= 256
    if (n0) {
      cur->next = std::make_shared<TcWeights>();
      cur = cur->next.get();
    }
    prep_slab(e, segs, seg_k, N, n0, cur);
  }
}

static void prep_slab(Engine& e, const std::vector<const float*>& segs, const std::vector<int>& seg_k, int Ntot,
                      int n0, TcWeights* out) {
  const int N = std::min(256, Ntot - n0);
  int Np = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  int Kp = 0;
  for (int k : seg_k) Kp += (k + kTcBK - 1) / kTcBK * kTcBK;
  std::vector<float> hi((size_t)Np * Kp, 0.f), lo((size_t)Np * Kp, 0.f);
  int kbase = 0;
  for (size_t si = 0; si < segs.size(); ++si) {
    const float* W = segs[si];
    const int K = seg_k[si];
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < N; ++n) {
        float v = W[(size_t)k * Ntot + n0 + n];
        uint32_t b;
        std::memcpy(&b, &v, 4);
        b &= 0xFFFFE000u;
        float h;
        std::memcpy(&h, &b, 4);
        hi[(size_t)n * Kp + kbase + k] = h;
        lo[(size_t)n * Kp + kbase + k] = v - h;
      }
    kbase += (K + kTcBK - 1) / kTcBK * kTcBK;
  }
  out->N = N;
  out->Np = Np;
  out->Kp = Kp;
  out->n0 = n0;
  out->hi = (float*)e.dalloc(sizeof(float) * hi.size());
  out->lo = (float*)e.dalloc(sizeof(float) * lo.size());
  OB_CUDA(cudaMemcpy(out->hi, hi.data(), sizeof(float) * hi.size(), cudaMemcpyHostToDevice));
  OB_CUDA(cudaMemcpy(out->lo, lo.data(), sizeof(float) * lo.size(), cudaMemcpyHostToDevice));
  make_map(out->map_hi, out->hi, Np, Kp);
  make_map(out->map_lo, out->lo, Np, Kp);
  if (Np > 64) {  // column-slab boxes for small-M launches
    make_map(out->map_hi64, out->hi, Np, Kp, 64);
    make_map(out->map_lo64, out->lo, Np, Kp, 64);
    out->map64_ready = true;
  }
  if (Np > 32) {
    make_map(out->map_hi32, out->hi, Np, Kp, 32);
    make_map(out->map_lo32, out->lo, Np, Kp, 32);
    out->map32_ready = true;
  }
  out->map_ready = true;
}

}  // namespace ob
