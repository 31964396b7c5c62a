// tcgen05 bf16 GEMM for the decoder-shaped chain (BASELINE north_star (2):
// "tensor cores (tcgen05) used only for the small dense GEMM nodes").
//
//   out[M, N] = epi( A[M, K] · W[N, K]^T + bias[N] )   epi = [GELU] [+ residual[M, N]], bf16 out
//
// One CTA per 128 x BN output tile (UMMA M = 128, cta_group::1, fp32 accumulator in TMEM).
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + single-thread MMA
// issuer, warps 2..5 = epilogue (warp w reads TMEM lane quarter w % 4).
// Operands are K-major, staged by TMA with the 128-byte swizzle into a STAGES-deep mbarrier ring.
//
// Programmatic dependent launch: W is a STATIC slot (weights never written by the chain), so the
// producer prefetches this CTA's whole W slab into L2 and issues the first stages' W tiles BEFORE
// griddepcontrol.wait; only the A tiles (the predecessor's output) wait. At the C3 shapes the
// GEMMs are weight-streaming bound (M = 128: ~128 FLOP/B, below the ~210 FLOP/B ridge), so
// overlapping the weight fetch with the previous node's tail is the main lever.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <cstdlib>
#include <mutex>

#include "../../include/cgx.h"
#include "cgx_decoder.h"
#include "cgx_device.cuh"

namespace cgx {

static constexpr int kBM = 128;
static constexpr int kBK = 64;          // 64 bf16 = 128 B = one swizzle-128B row
// Stage count per N tile (4: deeper rings measured no faster at the C3 shapes, profiles/r01).
template <int BN>
struct Stages {
  static constexpr int value = 4;
};
static constexpr int kGemmThreads = 192;
static constexpr uint32_t kGemmTriggerAfterWait = 1u << 8;   // internal flag bit (above CGX_GEMM_*)

struct alignas(64) GemmArgs {
  CUtensorMap tmA;            // A [M, K] bf16, box {64, 128}
  CUtensorMap tmB;            // W [N, K] bf16, box {64, BN}
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  __nv_bfloat16* out;
  float* ws;                  // split-K partial tiles [split][tiles][128][BN] (split > 1)
  unsigned long long* cnt;    // per-tile monotonic arrival counters (split > 1)
  uint32_t M, N, K, flags;
  uint32_t split;             // K splits (gridDim.z)
  unsigned long long* trace;  // optional per-CTA %globaltimer trace [cta][8] (diagnostics)
};

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* tm, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];\n" ::"l"(tm), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(tm) : "memory");
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle: 8-row x 128-B atoms, SBO = 1024 B.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);          // start address [0,14)
  d |= (uint64_t)(16 >> 4) << 16;                   // LBO (unused for swizzled K-major) [16,30)
  d |= (uint64_t)(1024 >> 4) << 32;                 // SBO [32,46)
  d |= (uint64_t)1 << 46;                           // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                           // layout: SWIZZLE_128B
  return d;
}
// Instruction descriptor: kind::f16, A = B = BF16, D = F32, K-major A and B, M = 128, N = BN.
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void trace_at(const GemmArgs& a, int slot) {
  if (a.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const uint32_t cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    a.trace[cta * 8 + slot] = t;
  }
}

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanhf(k0 * (x + k1 * x * x * x)));
}

// ------------------------------------------------------------------ kernel
// Split-K (gridDim.z = split, launched as thread-block clusters (1, 1, split)): CTA z accumulates
// k-blocks [z*nk/split, (z+1)*nk/split) in TMEM, parks its fp32 partial tile in its own shared
// memory, and after a cluster barrier reduces 1/split of the tile over DSMEM in fixed split order
// (deterministic, no float atomics, no global workspace) before running the epilogue on it. At M = 128 every N tile re-reads the whole A panel, so without split-K the per-CTA
// bytes (up to 128 x 3072 x 2 for FC2) bound the kernel; split-K spreads them over ~148 CTAs.
__device__ __forceinline__ void epilogue_store(const GemmArgs& a, int m, int n, float* v) {
  if (a.flags & CGX_GEMM_BIAS) {
    const uint4* bp = reinterpret_cast<const uint4*>(a.bias + n);
    const uint4 b0 = __ldg(bp), b1 = __ldg(bp + 1);
    const __nv_bfloat16* bb0 = reinterpret_cast<const __nv_bfloat16*>(&b0);
    const __nv_bfloat16* bb1 = reinterpret_cast<const __nv_bfloat16*>(&b1);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] += __bfloat162float(bb0[i]);
      v[8 + i] += __bfloat162float(bb1[i]);
    }
  }
  if (a.flags & CGX_GEMM_GELU) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = gelu_tanh(v[i]);
  }
  if (a.flags & CGX_GEMM_RESIDUAL) {
    const uint4* rp = reinterpret_cast<const uint4*>(a.residual + (size_t)m * a.N + n);
    const uint4 r0 = rp[0], r1 = rp[1];
    const __nv_bfloat16* rb0 = reinterpret_cast<const __nv_bfloat16*>(&r0);
    const __nv_bfloat16* rb1 = reinterpret_cast<const __nv_bfloat16*>(&r1);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] += __bfloat162float(rb0[i]);
      v[8 + i] += __bfloat162float(rb1[i]);
    }
  }
  uint4 o[2];
  __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(o);
#pragma unroll
  for (int i = 0; i < 16; ++i) ob[i] = __float2bfloat16_rn(v[i]);
  uint4* op = reinterpret_cast<uint4*>(a.out + (size_t)m * a.N + n);
  op[0] = o[0];
  op[1] = o[1];
}

__device__ __forceinline__ void epilogue_store4(const GemmArgs& a, int m, int n, float4 acc, uint2 bu) {
  float v[4] = {acc.x, acc.y, acc.z, acc.w};
  if (a.flags & CGX_GEMM_BIAS) {
    const __nv_bfloat16* bb = reinterpret_cast<const __nv_bfloat16*>(&bu);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] += __bfloat162float(bb[i]);
  }
  if (a.flags & CGX_GEMM_GELU) {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = gelu_tanh(v[i]);
  }
  if (a.flags & CGX_GEMM_RESIDUAL) {
    const uint2 ru = *reinterpret_cast<const uint2*>(a.residual + (size_t)m * a.N + n);
    const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&ru);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] += __bfloat162float(rb[i]);
  }
  uint2 o;
  __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
  for (int i = 0; i < 4; ++i) ob[i] = __float2bfloat16_rn(v[i]);
  *reinterpret_cast<uint2*>(a.out + (size_t)m * a.N + n) = o;
}

template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm_bf16(const __grid_constant__ GemmArgs a) {
  constexpr uint32_t kABytes = kBM * kBK * 2;     // 16 KiB
  constexpr uint32_t kBBytes = BN * kBK * 2;
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  constexpr int kStages = Stages<BN>::value;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tmem_full + 1);

  if (threadIdx.x == 0) trace_at(a, 0);
  const bool late_trigger = a.flags & kGemmTriggerAfterWait;
  if (!late_trigger) pdl_trigger();   // dependents may start their prologues (they read our output after their wait)
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN;
  const int m0 = blockIdx.y * kBM;
  const int kps = (int)(a.K / kBK / a.split);     // k-blocks per split
  const int kbase = (int)blockIdx.z * kps;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&a.tmA);
    prefetch_tmap(&a.tmB);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {   // TMEM allocation (whole warp), address published through shared memory
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer. Weights first (independent of the predecessor), then wait, then A.
      for (int i = 0; i < kps; ++i) tma_prefetch_l2(&a.tmB, (kbase + i) * kBK, n0);
      const int pre = kps < kStages ? kps : kStages;
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(&full[i], kABytes + kBBytes);
        tma_load_2d(sB + i * kBBytes, &a.tmB, &full[i], (kbase + i) * kBK, n0);
      }
      pdl_wait();
      if (late_trigger) pdl_trigger();
      for (int i = 0; i < pre; ++i) tma_load_2d(sA + i * kABytes, &a.tmA, &full[i], (kbase + i) * kBK, m0);
      for (int i = pre; i < kps; ++i) {
        const int s = i % kStages;
        const uint32_t ph = (uint32_t)(i / kStages) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_expect_tx(&full[s], kABytes + kBBytes);
        tma_load_2d(sB + s * kBBytes, &a.tmB, &full[s], (kbase + i) * kBK, n0);
        tma_load_2d(sA + s * kABytes, &a.tmA, &full[s], (kbase + i) * kBK, m0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- single-thread MMA issuer
      constexpr uint32_t idesc = umma_idesc(kBM, BN);
      for (int i = 0; i < kps; ++i) {
        const int s = i % kStages;
        const uint32_t ph = (uint32_t)(i / kStages) & 1u;
        mbar_wait(&full[s], ph);
        if (i == 0) trace_at(a, 2);
        tc_fence_after();
        const uint64_t da = umma_desc_sw128(smem_u32(sA + s * kABytes));
        const uint64_t db = umma_desc_sw128(smem_u32(sB + s * kBBytes));
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)   // UMMA_K = 16 bf16 = 32 B -> +2 in the >>4 address field
          umma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
      trace_at(a, 3);
    }
  } else {
    // ---- epilogue warps (128 threads): TMEM -> registers -> [split-K reduction] -> epilogue
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const uint32_t q = warp & 3;                  // TMEM lane quarter this warp may access
    const uint32_t row = q * 32 + lane;
    const int m = m0 + (int)row;
    const bool live = m < (int)a.M;
    if (a.split == 1) {
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((q * 32u) << 16) + (uint32_t)c0, v);
        if (live) epilogue_store(a, m, n0 + c0, v);
      }
    } else {
      // split-K: park this split's fp32 partial tile in OWN shared memory (the operand ring is
      // idle now): row-major [128][BN + 4] floats (padding keeps the 16-B column accesses of a
      // quarter warp on distinct banks)
      float* sP = reinterpret_cast<float*>(smem);
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((q * 32u) << 16) + (uint32_t)c0, v);
        float4* d = reinterpret_cast<float4*>(sP + row * (BN + 4) + c0);
#pragma unroll
        for (int i = 0; i < 4; ++i) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
      if (threadIdx.x == 64) trace_at(a, 5);
    }
  }
  if (a.split > 1) {
    // The S splits of a tile form one thread-block cluster (1, 1, S). After a cluster barrier
    // every CTA reduces 1/S of the tile, reading the S partials from the CTAs' shared memory
    // (DSMEM) in fixed split order 0..S-1 — deterministic, no global round trips or atomics —
    // then runs the epilogue on it. A second barrier keeps every partial alive until all reads
    // are done.
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (threadIdx.x == 64) trace_at(a, 6);
    if (warp >= 2) {
      const uint32_t S = a.split;
      const uint32_t my_rank = blockIdx.z;          // cluster (1,1,S) over gridDim.z == S
      constexpr uint32_t kQuads = kBM * BN / 4;
      const uint32_t q_lo = (uint32_t)((uint64_t)kQuads * my_rank / S);
      const uint32_t q_hi = (uint32_t)((uint64_t)kQuads * (my_rank + 1) / S);
      const uint32_t et = threadIdx.x - 64;          // epilogue thread 0..127
      const uint32_t local = smem_u32(smem);
      // this thread's quads: q_lo + et + 128 j, j < kQMax (<= BN/8 for any split >= 1)
      constexpr int kQMax = BN / 8;
      uint32_t offs[kQMax];
      bool have[kQMax];
      uint2 bias_q[kQMax];
      float4 acc[kQMax];
#pragma unroll
      for (int j = 0; j < kQMax; ++j) {
        const uint32_t qi = q_lo + et + 128u * j;
        have[j] = qi < q_hi;
        const uint32_t r = qi / (BN / 4), c = 4 * (qi % (BN / 4));
        offs[j] = (r * (BN + 4) + c) * 4;
        acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        bias_q[j] = make_uint2(0u, 0u);
        if (have[j] && (a.flags & CGX_GEMM_BIAS)) bias_q[j] = __ldg(reinterpret_cast<const uint2*>(a.bias + n0 + c));
      }
      for (uint32_t z = 0; z < S; ++z) {            // fixed split order: deterministic sums
        float4 t[kQMax];
#pragma unroll
        for (int j = 0; j < kQMax; ++j) {           // all of this split's loads in flight at once
          if (have[j]) {
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local + offs[j]), "r"(z));
            asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                         : "=f"(t[j].x), "=f"(t[j].y), "=f"(t[j].z), "=f"(t[j].w) : "r"(remote));
          }
        }
#pragma unroll
        for (int j = 0; j < kQMax; ++j)
          if (have[j]) {
            acc[j].x += t[j].x;
            acc[j].y += t[j].y;
            acc[j].z += t[j].z;
            acc[j].w += t[j].w;
          }
      }
      if (threadIdx.x == 64) trace_at(a, 1);
#pragma unroll
      for (int j = 0; j < kQMax; ++j) {
        if (!have[j]) continue;
        const uint32_t qi = q_lo + et + 128u * j;
        const uint32_t r = qi / (BN / 4), c = 4 * (qi % (BN / 4));
        const int mr = m0 + (int)r;
        if (mr < (int)a.M) epilogue_store4(a, mr, n0 + (int)c, acc[j], bias_q[j]);
      }
      if (threadIdx.x == 64) trace_at(a, 4);
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_at(a, 7);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static int get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode ? CGX_OK : CGX_E_CUDA;
}

static int encode_kmajor(CUtensorMap* tm, const void* base, uint64_t rows, uint64_t K, uint32_t box_rows) {
  cuuint64_t dims[2] = {K, rows};
  cuuint64_t strides[1] = {K * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? CGX_OK : CGX_E_CUDA;
}

// Tiling (measured per C3 shape with scripts/diag_gemm_tiling.py, profiles/r01/gemm_tiling.txt):
// BN = 32 everywhere; no split-K when there are already >= 64 N tiles (the DSMEM reduction costs
// more than the smaller A slice saves), else the largest split S <= 4 dividing the k-block count
// with tiles * S <= 148 (one wave; the S CTAs of a tile form a thread-block cluster).
static void pick_tiling(uint32_t M, uint32_t N, uint32_t K, int* bn_out, uint32_t* split_out) {
  const char* env_bn = getenv("CGX_GEMM_BN");          // measurement knobs
  const char* env_ms = getenv("CGX_GEMM_MAXSPLIT");
  int bn = (N % 32 == 0) ? 32 : 64;
  if (env_bn && N % atoi(env_bn) == 0) bn = atoi(env_bn);
  const uint32_t tiles = (N / bn) * ((M + kBM - 1) / kBM);
  const uint32_t nk = K / kBK;
  uint32_t max_split = env_ms ? (uint32_t)atoi(env_ms) : (tiles >= 64 ? 1u : 4u);
  uint32_t best = 1;
  for (uint32_t sp = 1; sp <= max_split && sp <= 8 && sp <= nk; ++sp)
    if (nk % sp == 0 && tiles * sp <= 148) best = sp;
  *bn_out = bn;
  *split_out = best;
}

template <int BN>
static size_t smem_bytes() {
  constexpr int kStages = Stages<BN>::value;
  return 1024 + kStages * (kBM * kBK * 2 + BN * kBK * 2) + (2 * kStages + 1) * 8 + 16;
}

void decoder_gemm_plan(uint32_t, uint32_t, uint32_t, size_t* ws_bytes, size_t* cnt_bytes) {
  // split-K partials are reduced through distributed shared memory: no global workspace
  *ws_bytes = 0;
  *cnt_bytes = 0;
}

template <int BN>
static const void* setup_kernel() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(k_gemm_bf16<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<BN>());
    cudaFuncSetAttribute(k_gemm_bf16<BN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  });
  return (const void*)k_gemm_bf16<BN>;
}

void decoder_gemm_set_trace(void* args, unsigned long long* trace) {
  static_cast<GemmArgs*>(args)->trace = trace;
}

void decoder_gemm_set_trigger_after_wait(void* args) {
  static_cast<GemmArgs*>(args)->flags |= kGemmTriggerAfterWait;
}

bool decoder_gemm_supported(uint32_t M, uint32_t N, uint32_t K) {
  return M >= 1 && K >= kBK && K % kBK == 0 && (N % 32 == 0);
}

int decoder_gemm_build(uint32_t M, uint32_t N, uint32_t K, uint32_t flags, const void* A, const void* W,
                       const void* bias, const void* residual, void* out, void* ws, void* cnt, void* args_out,
                       size_t* argbytes, dim3* grid, dim3* block, size_t* smem, const void** func) {
  if (!decoder_gemm_supported(M, N, K)) return CGX_E_UNSUPPORTED;
  int bn = 0;
  uint32_t sp = 1;
  pick_tiling(M, N, K, &bn, &sp);
  *argbytes = sizeof(GemmArgs);
  *grid = dim3(N / bn, (M + kBM - 1) / kBM, sp);
  *block = dim3(kGemmThreads);
  if (bn == 64) {
    *smem = smem_bytes<64>();
    *func = setup_kernel<64>();
  } else {
    *smem = smem_bytes<32>();
    *func = setup_kernel<32>();
  }
  if (!args_out) return CGX_OK;
  if (get_encode() != CGX_OK) return CGX_E_CUDA;
  GemmArgs* g = static_cast<GemmArgs*>(args_out);
  if (encode_kmajor(&g->tmA, A, M, K, kBM) != CGX_OK) return CGX_E_CUDA;
  if (encode_kmajor(&g->tmB, W, N, K, (uint32_t)bn) != CGX_OK) return CGX_E_CUDA;
  g->bias = static_cast<const __nv_bfloat16*>(bias);
  g->residual = static_cast<const __nv_bfloat16*>(residual);
  g->out = static_cast<__nv_bfloat16*>(out);
  g->ws = static_cast<float*>(ws);
  g->cnt = static_cast<unsigned long long*>(cnt);
  g->M = M;
  g->N = N;
  g->K = K;
  g->flags = flags;
  g->split = sp;
  g->trace = nullptr;

  return CGX_OK;
}

}  // namespace cgx
