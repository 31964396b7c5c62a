// Persistent decoder executor (cgx_mega.h): one CTA per SM runs every stage of a fused decoder
// range; stages hand over through L2 behind grid barriers.
//
// Stage kinds:
//  * GEMM  (tcgen05): warp 0 issues TMA (W slice of the CTA's task, prefetched one GEMM stage
//    ahead into one of two W buffers; A after the stage's barrier through a 2-slot ring of
//    4-k-block boxes), warp 1 issues the UMMAs (converged warp, elect.sync) into a TMEM
//    accumulator allocated once per launch, warps 4-7 drain TMEM (warp w reads lane quarter w % 4)
//    and either apply the epilogue (bias, GELU, residual, bf16 store) or store the fp32 partial of
//    a K-split task for a later ROW-stage fixup.
//  * ATTN  (mma.sync): the per-node kernel's attention tile (cgx_attn.cuh), one (q-block, head)
//    task at a time.
//  * ROW: row-local ops (split-K fixup, bf16 ADD, LayerNorm) on row r = CTA + i*G, each thread
//    owning 4-column chunks, values kept in registers between the ops of the stage.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/cgx.h"
#include "cgx_args.h"
#include "cgx_attn.cuh"
#include "cgx_device.cuh"
#include "cgx_mega.h"
#include "cgx_umma.cuh"

namespace cgx {

static constexpr uint32_t kMegaKB = 128u * 64u * 2u;   // one A k-block: 128 rows x 128 B (16 KiB)
static constexpr uint32_t kMegaSlotBytes = kMegaAGroup * kMegaKB;
static_assert(kMegaASlots * kMegaSlotBytes == kMegaABytes, "A ring layout");
static constexpr uint32_t kMegaBarBytes = 64;          // full_a[2] empty_a[2] full_w[2] tmem_full row_full
static constexpr uint32_t kMegaMiscBytes = 256;        // tmem address, abort flag, ext pointers, reductions
static constexpr size_t kMegaSmem = 1024 + kMegaABytes + 2 * kMegaWBytes + kMegaBarBytes + kMegaMiscBytes + kMegaRec;
static_assert(kMegaSmem <= 232448, "shared memory budget");
static constexpr uint32_t kMegaRowPartBytes = 64u * 1024u;   // ROW stage: split partials of the fixup (else L2 loads)
static_assert(kMegaRowPartBytes + kMegaMaxRowOps * 4 * kMegaMaxCols * 2 <= kMegaABytes, "ROW prefetch layout");

// CGX_MEGA_TRACE: [stage][cta][8] %globaltimer stamps (0 start after the barrier, 1 end, 2-6 phase
// marks of the stage kind, 7 barrier arrival)
__device__ __forceinline__ void mtrace(const MegaArgs& a, uint32_t si, uint32_t slot) {
  if (a.strace) a.strace[((size_t)si * a.G + blockIdx.x) * 8 + slot] = gtimer();
}

__device__ __forceinline__ const void* mref(const MegaRef& r, const uint64_t* s_ext) {
  return r.ext >= 0 ? reinterpret_cast<const void*>(s_ext[r.ext]) : r.p;
}

__device__ __forceinline__ float mega_warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Sum over the CTA's 256 threads in a fixed order (warp tree, then warps 0..7): deterministic.
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = mega_warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int w = 0; w < kMegaThreads / 32; ++w) t += red[w];
  __syncthreads();
  return t;
}

// Grid-wide barrier. Default (mode 3): each CTA adds 1 to one of kBarGroups counters (its CTA index
// mod 16, each counter on its own L2 line) after a gpu-scope fence, and warp 0 of every CTA polls
// the 16 counters until group g has reached (barrier count) x (CTAs in g). Every launch passes the
// same number of barriers with all G CTAs, so the counts are monotonic across replays (a CTA's own
// word flags[cta] keeps its count). Measured on the C3 decoder (scripts/diag_mega.py, profiles/r02/
// mega_*): one counter for all 148 CTAs ~2.2 us per barrier (same-address atomics serialise at ~27
// cycles each, B300_MICROARCH "L2-atom multi-CTA"); per-CTA words polled by every CTA 4-7 us (the
// polls saturate the L2 slices holding the words); a master CTA polling the words and releasing a
// "go" word 2.4-3.0 us (mode 1); 16 counters 1.7-1.9 us (1.3 us with empty stages). Inter-SM
// flag latency on this part is ~0.42 us one way (scripts/pingpong_microbench.cu), so any barrier
// costs >= 2 hops. A CTA that never arrives is reported through the status word (kDevErrBarrier)
// and the launch stops instead of hanging. CGX_MEGA_BAR / CGX_MEGA_BAR_NS select the variant and a
// poll back-off (measurement knobs).
static constexpr uint32_t kBarGroups = 16, kBarGroup0 = 544;   // mode 3 counters: words 544 + 32 g
__device__ __forceinline__ bool grid_barrier(const MegaArgs& a, uint32_t& cnt, volatile uint32_t* s_abort) {
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x, target = cnt + 1u;
    const uint32_t mode = a.bar_mode & 15u, ns = a.bar_sleep_ns;
    const bool rel_store = a.bar_mode & 16u, no_proxy = a.bar_mode & 32u;
    if (lane == 0) {
      if (!rel_store) __threadfence();
      if (!no_proxy) asm volatile("fence.proxy.async.global;\n" ::: "memory");
      if (mode == 2) asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(a.flags + 256 + 32 * (blockIdx.x & 7)) : "memory");
      else if (mode == 3) {
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;\n" ::"l"(a.flags + kBarGroup0 + 32 * (blockIdx.x % kBarGroups)) : "memory");
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;\n" ::"l"(a.flags + blockIdx.x), "r"(target) : "memory");
      } else if (rel_store) asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(a.flags + blockIdx.x), "r"(target) : "memory");
      else asm volatile("st.relaxed.gpu.global.u32 [%0], %1;\n" ::"l"(a.flags + blockIdx.x), "r"(target) : "memory");
    }
    uint64_t spins = 0;
    const unsigned long long t0 = gtimer();
    const bool poll_all = mode == 0 || (mode == 1 && blockIdx.x == 0);
    for (;;) {
      bool ok = true;
      if (poll_all) {
        for (uint32_t i = 4u * lane; i < a.G; i += 128u) {
          uint32_t v0, v1, v2, v3;
          asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                       : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                       : "l"(a.flags + i)
                       : "memory");
          ok = ok && (int32_t)(v0 - target) >= 0 && (i + 1 >= a.G || (int32_t)(v1 - target) >= 0) &&
               (i + 2 >= a.G || (int32_t)(v2 - target) >= 0) && (i + 3 >= a.G || (int32_t)(v3 - target) >= 0);
        }
      } else if (mode == 1) {
        uint32_t v = target;
        if (lane == 0) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(a.flags + 512) : "memory");
        ok = (int32_t)(__shfl_sync(0xffffffffu, v, 0) - target) >= 0;
      } else if (mode == 3) {   // kBarGroups spread counters, group g reaches target * (its CTAs)
        if (lane < kBarGroups) {
          uint32_t v;
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(a.flags + kBarGroup0 + 32 * lane) : "memory");
          const uint32_t members = a.G / kBarGroups + (lane < a.G % kBarGroups ? 1u : 0u);
          ok = (int32_t)(v - target * members) >= 0;
        }
      } else {   // mode 2: 8 spread counters, each reaches target * (CTAs in its group)
        if (lane < 8) {
          uint32_t v;
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(a.flags + 256 + 32 * lane) : "memory");
          const uint32_t members = a.G / 8 + (lane < a.G % 8 ? 1u : 0u);
          ok = (int32_t)(v - target * members) >= 0;
        }
      }
      if (__all_sync(0xffffffffu, ok)) break;
      uint32_t quit = 0;
      if (lane == 0 && spin_expired(a.st, t0, spins, kDevErrBarrier)) {
        *s_abort = 1u;
        quit = 1;
      }
      if (__shfl_sync(0xffffffffu, quit, 0)) break;
      if (ns) __nanosleep(ns);
    }
    if (mode == 1 && blockIdx.x == 0 && lane == 0) {
      if (rel_store) asm volatile("fence.acq_rel.gpu;\n st.relaxed.gpu.global.u32 [%0], %1;\n" ::"l"(a.flags + 512), "r"(target) : "memory");
      else asm volatile("st.relaxed.gpu.global.u32 [%0], %1;\n" ::"l"(a.flags + 512), "r"(target) : "memory");
    }
    if (lane == 0) asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    cnt = target;
  }
  __syncthreads();
  return *s_abort == 0u;
}

// ---------------------------------------------------------------- GEMM epilogue (warps 4-7)
// TMEM row -> registers (+ bias prefetched before the accumulator wait, GELU, residual) -> a padded
// staging tile in the idle A ring -> coalesced 16-B row stores by the 128 epilogue threads. Each
// thread owning one tile row and storing it straight out made every warp store instruction touch 32
// rows 3 KiB apart: ~2 us for a 32 KiB partial tile, measured with the stage trace.
template <int BN>
__device__ __forceinline__ void mega_epilogue(const MegaStage& S, const uint64_t* s_ext, uint32_t tmem, uint32_t q,
                                              uint32_t row, int m0, int n0, uint32_t split, const float* bias,
                                              uint8_t* stg) {
  const uint32_t et = threadIdx.x - 128u;   // epilogue thread 0..127 (warps 4-7)
  const uint32_t m = (uint32_t)m0 + row;
  float v[BN];
#pragma unroll
  for (int c0 = 0; c0 < BN; c0 += 16) tmem_ld16_nw(tmem + ((q * 32u) << 16) + (uint32_t)c0, v + c0);
  tmem_wait_regs<BN>(v);
  if (S.deferred) {
    constexpr uint32_t kRowF = BN + 4;   // padded fp32 row: conflict-free 16-B writes
    float* t = reinterpret_cast<float*>(stg);
#pragma unroll
    for (int i = 0; i < BN / 4; ++i)
      *reinterpret_cast<float4*>(t + row * kRowF + 4 * i) = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    constexpr uint32_t kQ = BN / 4;      // float4 per row
    for (uint32_t i = et; i < 128u * kQ; i += 128u) {
      const uint32_t r = i / kQ, c = i % kQ;
      if ((uint32_t)m0 + r < S.M)
        reinterpret_cast<float4*>(S.ws + ((size_t)split * S.M + m0 + r) * S.N + n0)[c] =
            *reinterpret_cast<const float4*>(t + r * kRowF + 4 * c);
    }
    return;
  }
  if (S.flags & CGX_GEMM_BIAS) {
#pragma unroll
    for (int i = 0; i < BN; ++i) v[i] += bias[i];
  }
  if (S.flags & CGX_GEMM_GELU) {
#pragma unroll
    for (int i = 0; i < BN; ++i) v[i] = gelu_tanh(v[i]);
  }
  if ((S.flags & CGX_GEMM_RESIDUAL) && m < S.M) {
    const uint4* rp = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(mref(S.res, s_ext)) +
                                                     (size_t)m * S.N + n0);
#pragma unroll
    for (int c8 = 0; c8 < BN / 8; ++c8) {
      const uint4 u = rp[c8];
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[8 * c8 + i] += __bfloat162float(b[i]);
    }
  }
  constexpr uint32_t kRowB = BN * 2 + 16;   // padded bf16 row (bytes)
#pragma unroll
  for (int c8 = 0; c8 < BN / 8; ++c8) {
    uint4 o;
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
    for (int i = 0; i < 8; ++i) ob[i] = __float2bfloat16_rn(v[8 * c8 + i]);
    *reinterpret_cast<uint4*>(stg + row * kRowB + 16 * c8) = o;
  }
  asm volatile("bar.sync 1, 128;\n" ::: "memory");
  constexpr uint32_t kQ = BN / 8;           // 16-B chunks per row
  for (uint32_t i = et; i < 128u * kQ; i += 128u) {
    const uint32_t r = i / kQ, c = i % kQ;
    if ((uint32_t)m0 + r < S.M)
      reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(S.out) + (size_t)(m0 + r) * S.N + n0)[c] =
          *reinterpret_cast<const uint4*>(stg + r * kRowB + 16 * c);
  }
}

// ---------------------------------------------------------------- ROW stage
// Every global operand of every op of the stage (bf16 rows / column parameters, and the split-K
// partials of a fixup) is fetched with cp.async at the start of the row, all in flight at once,
// into the (idle) A region: a ROW stage is one L2 round trip plus arithmetic instead of one
// dependent round trip per op. A thread only ever reads the chunks it fetched, so
// cp.async.wait_all alone orders them. Values produced by an earlier op of the stage stay in
// registers (MegaRef::reg; the planner keeps a stage to kMegaMaxRowOps ops so none is evicted).
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16cg(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n cp.async.wait_all;\n" ::: "memory");
}
__device__ __forceinline__ void unpack4(uint2 u, float* out) {
  const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) out[i] = __bfloat162float(b[i]);
}

__device__ void mega_row_stage(const MegaArgs& a, uint32_t si, const MegaStage& S, const MegaRowOp* ops,
                               const uint64_t* s_ext, float* red, uint8_t* sA, uint64_t* row_full, uint32_t& row_par) {
  float4* sP = reinterpret_cast<float4*>(sA);                         // fixup partials [S][cols] fp32
  uint2* sO = reinterpret_cast<uint2*>(sA + kMegaRowPartBytes);        // operands [op][x][cols] bf16
  const uint32_t t = threadIdx.x, cols = S.cols;
  float R[kMegaMaxRegs][2][4];
  // operand (oi, x): cols bf16 at sO + (oi * 4 + x) * kMegaMaxCols / 4 (uint2 units); chunk j of thread t
  auto oslot = [&](uint32_t oi, uint32_t x, uint32_t j) {
    return sO + (oi * 4u + x) * (kMegaMaxCols / 4u) + t + 256u * j;
  };
  auto operand = [&](const MegaRowOp& op, uint32_t oi, uint32_t x, uint32_t j, float* out) {
    const MegaRef& ref = (&op.a)[x];
    if (ref.reg >= 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) out[i] = R[ref.reg][j][i];
    } else {
      unpack4(*oslot(oi, x, j), out);
    }
  };
  auto store = [&](const MegaRowOp& op, uint32_t r, uint32_t c, uint32_t j, const float* v) {
    uint2 u;
    __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = __float2bfloat16_rn(v[i]);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(op.out) + (size_t)r * cols + c) = u;
    if (op.out_reg >= 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) R[op.out_reg][j][i] = __bfloat162float(b[i]);
    }
  };
  // operands land with ONE mbarrier: thread 0 issues a bulk copy per contiguous row / column
  // vector / split partial (a handful of instructions instead of one LSU request per 8-16 B)
  const bool part_smem = ops[0].kind == kRowFixup && (size_t)ops[0].S * cols * 4 <= kMegaRowPartBytes;
  for (uint32_t r = blockIdx.x; r < S.rows; r += a.G) {
    if (t == 0) {
      if (!(a.dbg & 2u)) asm volatile("fence.proxy.async.global;\n" ::: "memory");   // generic stores -> bulk-copy reads
      uint32_t bytes = 0;
      for (uint32_t oi = 0; oi < S.n_ops; ++oi) {
        const MegaRowOp& op = ops[oi];
        if (op.kind == kRowFixup && part_smem) bytes += op.S * cols * 4u;
        for (uint32_t x = 0; x < 4; ++x)
          if ((op.pf >> x) & 1u) bytes += cols * 2u;
      }
      mbar_expect_tx(row_full, bytes);
      for (uint32_t oi = 0; oi < S.n_ops; ++oi) {
        const MegaRowOp& op = ops[oi];
        if (op.kind == kRowFixup && part_smem)
          for (uint32_t sp = 0; sp < op.S; ++sp)
            bulk_g2s(reinterpret_cast<float*>(sP) + sp * cols, op.ws + ((size_t)sp * S.rows + r) * cols, cols * 4u, row_full);
        for (uint32_t x = 0; x < 4; ++x)
          if ((op.pf >> x) & 1u) {
            const __nv_bfloat16* base = reinterpret_cast<const __nv_bfloat16*>(mref((&op.a)[x], s_ext));
            bulk_g2s(sO + (oi * 4u + x) * (kMegaMaxCols / 4u), base + (((op.col >> x) & 1u) ? 0 : (size_t)r * cols),
                     cols * 2u, row_full);
          }
      }
    }
    mbar_wait(row_full, row_par);
    row_par ^= 1u;
    if (threadIdx.x == 0 && r == blockIdx.x) mtrace(a, si, 2);   // operands landed
    // ---- compute
    for (uint32_t oi = 0; oi < S.n_ops; ++oi) {
      const MegaRowOp& op = ops[oi];
      if (op.kind == kRowLn) {
        float xv[2][4];
        float sum = 0.f;
#pragma unroll
        for (uint32_t j = 0; j < 2; ++j)
          if (4u * t + 1024u * j < cols) {
            operand(op, oi, 0, j, xv[j]);
            sum += (xv[j][0] + xv[j][1]) + (xv[j][2] + xv[j][3]);
          }
        const float mean = block_sum(sum, red) / (float)cols;
        float qs = 0.f;
#pragma unroll
        for (uint32_t j = 0; j < 2; ++j)
          if (4u * t + 1024u * j < cols)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float d = xv[j][i] - mean;
              qs += d * d;
            }
        const float var = block_sum(qs, red) / (float)cols;
        const float rstd = 1.0f / sqrtf(var + op.eps);
#pragma unroll
        for (uint32_t j = 0; j < 2; ++j) {
          const uint32_t c = 4u * t + 1024u * j;
          if (c < cols) {
            float g[4], b[4], y[4];
            operand(op, oi, 2, j, g);
            operand(op, oi, 3, j, b);
#pragma unroll
            for (int i = 0; i < 4; ++i) y[i] = (xv[j][i] - mean) * rstd * g[i] + b[i];
            store(op, r, c, j, y);
          }
        }
      } else if (op.kind == kRowAdd) {
#pragma unroll
        for (uint32_t j = 0; j < 2; ++j) {
          const uint32_t c = 4u * t + 1024u * j;
          if (c < cols) {
            float u[4], w[4], y[4];
            operand(op, oi, 0, j, u);
            operand(op, oi, 1, j, w);
#pragma unroll
            for (int i = 0; i < 4; ++i) y[i] = u[i] + w[i];
            store(op, r, c, j, y);
          }
        }
      } else {   // kRowFixup: the S partials in split order, then the GEMM node's epilogue
#pragma unroll
        for (uint32_t j = 0; j < 2; ++j) {
          const uint32_t c = 4u * t + 1024u * j;
          if (c >= cols) continue;
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          for (uint32_t sp = 0; sp < op.S; ++sp) {
            const float4 v = part_smem ? *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(sP) + sp * cols + c)
                                       : __ldcg(reinterpret_cast<const float4*>(op.ws + ((size_t)sp * S.rows + r) * cols + c));
            acc[0] += v.x;
            acc[1] += v.y;
            acc[2] += v.z;
            acc[3] += v.w;
          }
          if (op.flags & CGX_GEMM_BIAS) {
            float b[4];
            operand(op, oi, 2, j, b);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] += b[i];
          }
          if (op.flags & CGX_GEMM_GELU) {
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] = gelu_tanh(acc[i]);
          }
          if (op.flags & CGX_GEMM_RESIDUAL) {
            float rr[4];
            operand(op, oi, 3, j, rr);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] += rr[i];
          }
          store(op, r, c, j, acc);
        }
      }
    }
  }
}

// stage record (descriptor + row ops) -> shared memory with cp.async, issued before the stage's
// barrier (the barrier's L1 invalidation would otherwise turn every descriptor read after it into
// a dependent L2 round trip)
__device__ __forceinline__ const MegaStage& mstage(const MegaArgs& a, int32_t si) {
  return *reinterpret_cast<const MegaStage*>(a.recs + (size_t)si * kMegaRec);
}
__device__ __forceinline__ void stage_fetch(const MegaArgs& a, uint32_t si, uint8_t* s_desc) {
  if (threadIdx.x < kMegaRec / 16)
    cp_async16cg(s_desc + 16 * threadIdx.x, a.recs + (size_t)si * kMegaRec + 16 * threadIdx.x);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(kMegaThreads, 1) k_mega(const __grid_constant__ MegaArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sW = smem + kMegaABytes;
  uint64_t* full_a = reinterpret_cast<uint64_t*>(sW + 2 * kMegaWBytes);
  uint64_t* empty_a = full_a + kMegaASlots;
  uint64_t* full_w = empty_a + kMegaASlots;
  uint64_t* tmem_full = full_w + 2;
  uint64_t* row_full = tmem_full + 1;
  uint32_t* s_misc = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(full_a) + kMegaBarBytes);
  volatile uint32_t* s_abort = s_misc + 1;
  uint64_t* s_ext = reinterpret_cast<uint64_t*>(s_misc + 2);            // [kMegaMaxExt]
  float* s_red = reinterpret_cast<float*>(s_ext + kMegaMaxExt);           // [8]
  uint8_t* s_desc = reinterpret_cast<uint8_t*>(s_misc) + kMegaMiscBytes; // stage + row ops
  const MegaStage& S = *reinterpret_cast<const MegaStage*>(s_desc);
  const MegaRowOp* s_ops = reinterpret_cast<const MegaRowOp*>(s_desc + kMegaDescStage);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    node_stamp(a.ntrace, 0);
    for (uint32_t s = 0; s < kMegaASlots; ++s) {
      mbar_init(&full_a[s], 1);
      mbar_init(&empty_a[s], 1);
    }
    mbar_init(&full_w[0], 1);
    mbar_init(&full_w[1], 1);
    mbar_init(tmem_full, 1);
    mbar_init(row_full, 1);
    *s_abort = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(s_misc)),
                 "r"(kMegaMaxBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  // every input of the fused range was written before this launch (or is an input / weight); the
  // dependents launch only when this grid completes (no early trigger)
  pdl_wait();
  if (threadIdx.x < a.n_ext)   // PI: de-reference the externals once, at kernel start
    s_ext[threadIdx.x] = a.ext_t[threadIdx.x] >= 0 ? ld_table(a.table + a.ext_t[threadIdx.x])
                                                   : reinterpret_cast<uint64_t>(a.ext_ptr[threadIdx.x]);
  if (a.n_stages) stage_fetch(a, 0, s_desc);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) node_stamp(a.ntrace, 1);
  const uint32_t tmem = s_misc[0];

  // W slice of this CTA's first task of a GEMM stage (STATIC weights: no dependency) -> its buffer
  auto issue_w = [&](const MegaStage& G, uint32_t t) {
    const uint32_t split = t % G.split, tile = t / G.split;
    const int n0 = (int)((tile % G.n_tiles) * G.bn), kb0 = (int)(split * G.kps);
    mbar_expect_tx_w(&full_w[G.w_buf], G.bn * G.kps * 128u);
    tma_load_3d_w(sW + G.w_buf * kMegaWBytes, reinterpret_cast<const CUtensorMap*>(G.tmW), &full_w[G.w_buf], 0, n0,
                  kb0);
  };
  auto gemm_tasks = [](const MegaStage& G) { return G.m_tiles * G.n_tiles * G.split; };
  if (warp == 0 && a.first_gemm >= 0) {
    const MegaStage& G = mstage(a, a.first_gemm);
    if (blockIdx.x < gemm_tasks(G)) issue_w(G, blockIdx.x);
  }

  // pipeline state (each counter lives in the role that uses it; all advance identically)
  uint32_t a_it = 0, a_ct = 0;                 // A groups issued (warp 0) / consumed (warp 1)
  uint32_t w_par[2] = {0u, 0u};                // W buffer phases (warp 1)
  uint32_t acc_par = 0;                        // tmem_full phase (epilogue warps)
  uint32_t row_par = 0;                        // row_full phase (all threads)
  uint32_t bar_cnt = a.flags[blockIdx.x];     // this CTA's arrivals so far (its own word)

  for (uint32_t si = 0; si < a.n_stages; ++si) {
    const bool need_bar = si > 0 && S.bar_next;   // (S: the previous stage's record)
    __syncthreads();
    if (threadIdx.x == 0) mtrace(a, si, 7);
    if (si > 0) stage_fetch(a, si, s_desc);   // the previous stage is done with its record
    if (need_bar && !grid_barrier(a, bar_cnt, s_abort)) break;
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) mtrace(a, si, 0);
    if (a.null_work) {                       // diagnostics: barriers and stage bookkeeping only
    } else if (S.kind == kMegaGemm) {
      const uint32_t tasks = gemm_tasks(S);
      const uint32_t ngroups = S.kps / S.ga;
      for (uint32_t t = blockIdx.x, it = 0; t < tasks; t += a.G, ++it) {
        const uint32_t split = t % S.split, tile = t / S.split;
        const int n0 = (int)((tile % S.n_tiles) * S.bn), m0 = (int)((tile / S.n_tiles) * 128u);
        const int kb0 = (int)(split * S.kps);
        if (warp == 0) {
          if (it > 0) issue_w(S, t);   // later tasks of this CTA: the buffer is free (CTA synchronised)
          if (lane == 0 && it == 0) mtrace(a, si, 2);   // A issued
          if (!(a.dbg & 4u)) asm volatile("fence.proxy.async.global;\n" ::: "memory");   // other CTAs' generic stores -> TMA reads
          for (uint32_t g = 0; g < ngroups; ++g, ++a_it) {
            const uint32_t slot = a_it % kMegaASlots;
            if (a_it >= kMegaASlots) mbar_wait(&empty_a[slot], ((a_it / kMegaASlots) - 1u) & 1u);
            mbar_expect_tx_w(&full_a[slot], S.ga * kMegaKB);
            tma_load_3d_w(sA + slot * kMegaSlotBytes, reinterpret_cast<const CUtensorMap*>(S.tmA), &full_a[slot], 0,
                          m0, kb0 + (int)(g * S.ga));
          }
          // prefetch the next GEMM stage's W into the other buffer (its last user, the previous
          // GEMM stage, has drained: every stage ends with the CTA synchronised after its epilogue)
          if (it == 0 && S.next_gemm >= 0) {
            const MegaStage& Nx = mstage(a, S.next_gemm);
            if (blockIdx.x < gemm_tasks(Nx)) issue_w(Nx, blockIdx.x);
          }
        } else if (warp == 1) {
          const uint32_t idesc = umma_idesc(128, (int)S.bn);
          const uint32_t wb = S.w_buf;
          mbar_wait(&full_w[wb], w_par[wb]);
          w_par[wb] ^= 1u;
          if (lane == 0 && it == 0) mtrace(a, si, 3);   // W landed
          for (uint32_t g = 0; g < ngroups; ++g, ++a_ct) {
            const uint32_t slot = a_ct % kMegaASlots;
            mbar_wait(&full_a[slot], (a_ct / kMegaASlots) & 1u);
            if (lane == 0 && it == 0 && g == 0) mtrace(a, si, 4);   // first A group landed
            tc_fence_after();
            for (uint32_t kk = 0; kk < S.ga; ++kk) {
              const uint32_t kl = g * S.ga + kk;   // k-block within the task
              const uint64_t da = umma_desc_sw128(smem_u32(sA + slot * kMegaSlotBytes + kk * kMegaKB));
              const uint64_t db = umma_desc_sw128(smem_u32(sW + wb * kMegaWBytes + kl * S.bn * 128u));
#pragma unroll
              for (int k = 0; k < 4; ++k) umma_bf16_w(tmem, da + 2 * k, db + 2 * k, idesc, (kl | (uint32_t)k) != 0);
            }
            umma_commit_w(&empty_a[slot]);
          }
          umma_commit_w(tmem_full);
          if (lane == 0 && it == 0) mtrace(a, si, 5);   // all MMAs issued
        } else if (warp >= 4) {
          // the bias slice (STATIC) is fetched while the MMAs run
          float bias[kMegaMaxBN];
          if (!S.deferred && (S.flags & CGX_GEMM_BIAS)) {
            const uint4* bp = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(mref(S.bias, s_ext)) + n0);
#pragma unroll
            for (uint32_t c8 = 0; c8 < kMegaMaxBN / 8; ++c8)
              if (c8 < S.bn / 8) {
                const uint4 u = __ldg(bp + c8);
                const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
                for (int i = 0; i < 8; ++i) bias[8 * c8 + i] = __bfloat162float(b[i]);
              }
          }
          mbar_wait(tmem_full, acc_par);
          if (threadIdx.x == 128 && it == 0) mtrace(a, si, 6);   // accumulator ready
          acc_par ^= 1u;
          tc_fence_after();
          const uint32_t q = warp & 3u, row = q * 32u + lane;
          // the A ring is idle once the accumulator is complete: it stages the output tile
          if (S.bn == 64) mega_epilogue<64>(S, s_ext, tmem, q, row, m0, n0, split, bias, sA);
          else if (S.bn == 32) mega_epilogue<32>(S, s_ext, tmem, q, row, m0, n0, split, bias, sA);
          else mega_epilogue<16>(S, s_ext, tmem, q, row, m0, n0, split, bias, sA);
          tc_fence_before();
          // generic staging-tile accesses in the A ring -> the next TMA writes into it
          if (!(a.dbg & 1u)) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        }
        __syncthreads();
      }
      if (blockIdx.x >= tasks && warp == 0 && S.next_gemm >= 0) {   // no task here: still prefetch
        const MegaStage& Nx = mstage(a, S.next_gemm);
        if (blockIdx.x < gemm_tasks(Nx)) issue_w(Nx, blockIdx.x);
      }
    } else if (S.kind == kMegaAttn) {
      const uint32_t nqb = (S.T + 15u) / 16u, tasks = nqb * S.H;
      const __nv_bfloat16* qkv = reinterpret_cast<const __nv_bfloat16*>(mref(S.qkv, s_ext));
      for (uint32_t t = blockIdx.x; t < tasks; t += a.G) {
        attn_tile(qkv, reinterpret_cast<__nv_bfloat16*>(S.aout), S.T, S.H, S.scale, t % nqb, t / nqb, sA);
        __syncthreads();
      }
    } else {
      mega_row_stage(a, si, S, s_ops, s_ext, s_red, sA, row_full, row_par);
    }
    if (S.kind != kMegaGemm)   // generic shared-memory writes in the A region -> later TMA writes
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) mtrace(a, si, 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kMegaMaxBN));
  }
  if (threadIdx.x == 0) node_stamp(a.ntrace, 2);
}

const void* kfn_mega() {
  cudaFuncSetAttribute(k_mega, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMegaSmem);
  return (const void*)k_mega;
}
size_t mega_smem_bytes() { return kMegaSmem; }

}  // namespace cgx
