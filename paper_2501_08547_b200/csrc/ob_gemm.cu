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
// D = A_hi B_hi + A_hi B_lo + A_lo B_hi accumulated in an fp32 TMEM tile.  The
// tensor core truncates fp32 operands to TF32, so the raw fp32 tile *is* A_hi;
// A_lo = a - trunc(a) is formed in shared memory per k-block, B_lo is prepared
// once at model load (weights are static).
//
// Structure (one CTA per SM, persistent over 128-row tiles):
//   * 256 threads stage A/B k-blocks (32 fp32 = one 128-byte row) with cp.async
//     into the canonical K-major SWIZZLE_128B layout, up to a 4-stage ring;
//     A_lo lives in its own double buffer so the ring holds only raw loads;
//   * one elected thread issues 12 tcgen05.mma.kind::tf32 (3 products x 4 K=8
//     steps) per k-block and tcgen05.commit's an mbarrier per stage;
//   * epilogue: 8 warps tcgen05.ld 32x32b (lane quadrant x column half) ->
//     registers -> optional addend + activation -> global.
#include <algorithm>
#include <cstring>

#include "ob_engine.h"

namespace ob {

namespace {

constexpr int kTcThreads = 256;
constexpr int kTcBM = 128;
constexpr int kTcBK = 32;  // fp32 per k-block: one 128-byte swizzle row
constexpr int kTileA = kTcBM * kTcBK * 4;  // 16 KB

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

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
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

// Shared memory: S-stage ring of {A, B, B_lo} k-blocks + a double-buffered A_lo.
template <int NP>
struct TcSmem {
  static constexpr int kTileB = NP * kTcBK * 4;
  static constexpr int kStage = kTileA + 2 * kTileB;
  static constexpr int kBudget = 227 * 1024 - 2 * kTileA - (1024 + 256 + kTcBM * 8);
  static constexpr int kStages = (kBudget / kStage) >= 4 ? 4 : ((kBudget / kStage) >= 3 ? 3 : 2);
  static constexpr int kBytes = kStages * kStage + 2 * kTileA + 1024 /*align*/ + 256 /*bars*/ + kTcBM * 8;
};

template <int NP>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_gemm(TcGemmArgs g) {
  using SM = TcSmem<NP>;
  constexpr int S = SM::kStages;
  constexpr uint32_t kCols = NP <= 32 ? 32 : (NP <= 64 ? 64 : (NP <= 128 ? 128 : 256));
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // offset (not an integer cast) keeps the pointer in the shared window -> LDS/STS
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* alo_base = base + S * SM::kStage;  // 2 x 16 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(alo_base + 2 * kTileA);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + S + 1);
  const float** rows = reinterpret_cast<const float**>(alo_base + 2 * kTileA + 256);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = *g.M_dev;
  const int64_t tiles = (M + kTcBM - 1) / kTcBM;
  const int KB1 = (g.K1 + kTcBK - 1) / kTcBK, KB2 = (g.K2 + kTcBK - 1) / kTcBK, KB = KB1 + KB2;
  const int Kp = KB * kTcBK;

  if (tid == 0) {
    for (int i = 0; i < S + 1; ++i) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = tf32_idesc(NP);

  uint32_t it = 0;  // global k-block counter across tiles (stage / phase bookkeeping)
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t m0 = tile * kTcBM;
    if (tid < kTcBM) {  // per-tile A1 row pointers
      const int64_t r = m0 + tid;
      const float* p = nullptr;
      if (r < M && g.K1) p = g.a1.row(g.self ? (int64_t)g.self[r] : r);
      rows[tid] = p;
    }
    __syncthreads();

    auto load = [&](int kb, int stage) {
      uint8_t* sA = base + stage * SM::kStage;
      const uint32_t a_s = smem_u32(sA), b_s = a_s + kTileA, bl_s = b_s + SM::kTileB;
      const bool first = kb < KB1;
      const int k0 = (first ? kb : kb - KB1) * kTcBK;
      const int Kv = first ? g.K1 : g.K2;
#pragma unroll
      for (int i = 0; i < (kTcBM * 8) / kTcThreads; ++i) {
        const int q = tid + i * kTcThreads;
        const int r = q >> 3, c = q & 7;
        const int k = k0 + c * 4;
        const float* src = nullptr;
        int bytes = 0;
        if (m0 + r < M) {
          const float* rowp = first ? rows[r] : g.a2 + (m0 + r) * g.lda2;
          const int rem = Kv - k;
          bytes = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
          src = rowp + (bytes ? k : 0);
        }
        if (!src) src = g.Bt;  // any valid address; 0 bytes are read
        cp_async16(a_s + r * 128 + ((c ^ (r & 7)) << 4), src, bytes);
      }
#pragma unroll
      for (int i = 0; i < (NP * 8 + kTcThreads - 1) / kTcThreads; ++i) {
        const int q = tid + i * kTcThreads;
        if (q < NP * 8) {
          const int n = q >> 3, c = q & 7;
          const int64_t off = (int64_t)n * Kp + kb * kTcBK + c * 4;
          const uint32_t so = n * 128 + ((c ^ (n & 7)) << 4);
          cp_async16(b_s + so, g.Bt + off, 16);
          cp_async16(bl_s + so, g.Bt_lo + off, 16);
        }
      }
    };

#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
      if (s < KB) load(s, (it + s) % S);
      cp_async_commit();
    }
    for (int kb = 0; kb < KB; ++kb) {
      const uint32_t gk = it + kb;
      const int stage = gk % S;
      cp_async_wait<S - 2>();
      __syncthreads();
      // A_lo = a - trunc_tf32(a) into the double buffer (MMAs of k-block gk-2 have retired:
      // we waited for gk-2 before refilling its stage one iteration ago)
      {
        const float* a = reinterpret_cast<const float*>(base + stage * SM::kStage);
        float* alo = reinterpret_cast<float*>(alo_base + (gk & 1) * kTileA);
#pragma unroll 4
        for (int i = tid * 4; i < kTcBM * kTcBK; i += kTcThreads * 4) {
          const float4 v = *reinterpret_cast<const float4*>(a + i);
          float4 o;
          o.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          o.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          o.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          o.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          *reinterpret_cast<float4*>(alo + i) = o;
        }
      }
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t a_s = smem_u32(base + stage * SM::kStage);
        const uint32_t b_s = a_s + kTileA, blo_s = b_s + SM::kTileB;
        const uint32_t alo_s = smem_u32(alo_base + (gk & 1) * kTileA);
#pragma unroll
        for (int kk = 0; kk < kTcBK / 8; ++kk) {
          const uint32_t off = kk * 32;  // 8 tf32 per MMA
          const uint64_t da = sw128_desc(a_s + off), dal = sw128_desc(alo_s + off);
          const uint64_t db = sw128_desc(b_s + off), dbl = sw128_desc(blo_s + off);
          mma_tf32(tmem, da, db, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          mma_tf32(tmem, da, dbl, idesc, 1u);
          mma_tf32(tmem, dal, db, idesc, 1u);
        }
        mma_commit(bars + stage);
      }
      // refill the stage consumed by the previous k-block once its MMAs retired
      const int nk = kb + S - 1;
      if (nk < KB) {
        if (kb > 0) mbar_wait(bars + ((gk - 1) % S), ((gk - 1) / S) & 1);
        load(nk, (gk + S - 1) % S);
      }
      cp_async_commit();
    }
    {
      const uint32_t glast = it + KB - 1;
      mbar_wait(bars + (glast % S), (glast / S) & 1);
    }
    it += KB;
    tc_fence_after();
    // epilogue: warp w reads TMEM lanes [32(w%4), +32) = tile rows, column half w/4;
    // each 32x32 block is transposed through shared memory (the free A_lo buffers,
    // XOR-swizzled) so E loads and C stores run with lanes along a row (coalesced)
    {
      const int quad = warp & 3, half = warp >> 2;
      constexpr int kHalf = NP >= 64 ? NP / 2 : NP;
      float* buf = reinterpret_cast<float*>(alo_base) + warp * 1024;
      if (NP >= 64 || half == 0) {
#pragma unroll 1
        for (int c0 = half * kHalf; c0 < (half + 1) * kHalf; c0 += 32) {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + c0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) buf[lane * 32 + (j ^ lane)] = v[j];
          __syncwarp();
          const int col = c0 + lane;
#pragma unroll 4
          for (int r = 0; r < 32; ++r) {
            const int64_t row = m0 + quad * 32 + r;
            if (row < M && col < g.N) {
              float o = buf[r * 32 + (lane ^ r)];
              if (g.E) o += g.E[row * g.lde + col];
              if (g.relu) o = fmaxf(o, 0.f);
              g.C[row * g.ldc + col] = o;
            }
          }
          __syncwarp();
        }
      }
    }
    tc_fence_before();
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
  }
}

void tc_gemm(cudaStream_t s, const TcGemmArgs& g, int64_t M_max) {
  OB_CHECK(g.N >= 1 && g.N <= 256, OB_ESTATE, "tc_gemm: N out of range");
  const int64_t tiles = (M_max + kTcBM - 1) / kTcBM;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, kNumSMs));
  const int np = g.Np;
  auto go = [&](auto kern, int bytes) {
    static bool configured[4] = {false, false, false, false};
    int slot = np <= 32 ? 0 : np <= 64 ? 1 : np <= 128 ? 2 : 3;
    if (!configured[slot]) {
      OB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      configured[slot] = true;
    }
    kern<<<grid, kTcThreads, bytes, s>>>(g);
  };
  if (np == 32) go(k_tc_gemm<32>, TcSmem<32>::kBytes);
  else if (np == 64) go(k_tc_gemm<64>, TcSmem<64>::kBytes);
  else if (np == 128) go(k_tc_gemm<128>, TcSmem<128>::kBytes);
  else if (np == 256) go(k_tc_gemm<256>, TcSmem<256>::kBytes);
  else throw Error(OB_ESTATE, "tc_gemm: padded N must be 32/64/128/256");
  OB_LAUNCHED();
}

// ---------------------------------------------------------------------------
// weight preparation: W (K x N row-major) blocks -> Bt / Bt_lo (Np x Kp, K-major,
// zero padded), K-blocks of each operand segment padded to 32
// ---------------------------------------------------------------------------
void prep_tc_weights(Engine& e, const std::vector<const float*>& segs, const std::vector<int>& seg_k, int N,
                     TcWeights* out) {
  int Np = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  OB_CHECK(N <= 256, OB_EINVAL, "layer width above 256 is not supported by the tensor-core path");
  int Kp = 0;
  for (int k : seg_k) Kp += (k + kTcBK - 1) / kTcBK * kTcBK;
  std::vector<float> hi((size_t)Np * Kp, 0.f), lo((size_t)Np * Kp, 0.f);
  int kbase = 0;
  for (size_t si = 0; si < segs.size(); ++si) {
    const float* W = segs[si];
    const int K = seg_k[si];
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < N; ++n) {
        float v = W[(size_t)k * N + n];
        uint32_t b;
        std::memcpy(&b, &v, 4);
        b &= 0xFFFFE000u;
        float h;
        std::memcpy(&h, &b, 4);
        hi[(size_t)n * Kp + kbase + k] = v;
        lo[(size_t)n * Kp + kbase + k] = v - h;
      }
    kbase += (K + kTcBK - 1) / kTcBK * kTcBK;
  }
  out->N = N;
  out->Np = Np;
  out->Kp = Kp;
  out->hi = (float*)e.dalloc(sizeof(float) * hi.size());
  out->lo = (float*)e.dalloc(sizeof(float) * lo.size());
  OB_CUDA(cudaMemcpy(out->hi, hi.data(), sizeof(float) * hi.size(), cudaMemcpyHostToDevice));
  OB_CUDA(cudaMemcpy(out->lo, lo.data(), sizeof(float) * lo.size(), cudaMemcpyHostToDevice));
}

}  // namespace ob
