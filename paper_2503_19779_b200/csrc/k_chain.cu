// Chain kernels for sm_100a: elementwise (ADD/MUL/SCALE_IMM/COPY, f32 and bf16), row reduction,
// the multi-tensor copy of the COPY arm, the INDIRECT root table writers, and small utilities.
//
// All of them are HBM/L2-bandwidth or latency bound (no dense contraction): 128-bit coalesced
// accesses, several loads in flight per thread, one CTA wave where possible, no tensor cores.
//
// Parameter indirection: an operand whose table index is >= 0 is fetched as
// table[idx] ONCE at kernel start, before griddepcontrol.wait unless kFlagTableAfterWait is set
// (the first node after a root table-writer node). The arithmetic after the fetch is the same code
// for the direct and indirect variants, so all arms are bit-identical.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "cgx_args.h"
#include "cgx_device.cuh"

namespace cgx {

static constexpr int kElemThreads = 256;
#ifndef CGX_ELEM_VEC
#define CGX_ELEM_VEC 4
#endif
static constexpr int kElemVec = CGX_ELEM_VEC;   // 16-B vectors per thread per operand (loads in flight)

enum { OP_ADD = 0, OP_MUL = 1, OP_SCALE = 2, OP_COPY = 3, OP_SCALE_T = 4,
       // training-shaped chain (bf16): a - b, a + s*b, GELU(a), dy * GELU'(x)
       OP_SUB = 5, OP_AXPY = 6, OP_GELU = 7, OP_GELU_BWD = 8 };

// tanh-approximate GELU and its derivative in fp32 with libm tanhf (SURVEY ambiguity 11)
__device__ __forceinline__ float gelu_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanhf(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = tanhf(k0 * (x + k1 * x * x * x));
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * k0 * (1.0f + 3.0f * k1 * x * x);
}

template <int OP>
__device__ __forceinline__ float apply_f32(float x, float y, float s) {
  if (OP == OP_ADD) return __fadd_rn(x, y);
  if (OP == OP_MUL) return __fmul_rn(x, y);
  if (OP == OP_SCALE || OP == OP_SCALE_T) return __fmul_rn(x, s);
  if (OP == OP_SUB) return __fsub_rn(x, y);
  if (OP == OP_AXPY) return __fmaf_rn(s, y, x);          // x + s*y, one fp32 rounding
  if (OP == OP_GELU) return gelu_f(x);
  if (OP == OP_GELU_BWD) return __fmul_rn(x, gelu_grad_f(y));   // x = dy, y = pre-activation
  return x;
}
template <int OP>
__host__ __device__ constexpr bool elem_binary() {
  return OP == OP_ADD || OP == OP_MUL || OP == OP_SUB || OP == OP_AXPY || OP == OP_GELU_BWD;
}

__device__ __forceinline__ void fetch_operands(const ElemArgs& a, const void*& p0, const void*& p1) {
  p0 = a.in0;
  p1 = a.in1;
  if (a.t0 >= 0) p0 = reinterpret_cast<const void*>(ld_table(a.table + a.t0));
  if (a.t1 >= 0) p1 = reinterpret_cast<const void*>(ld_table(a.table + a.t1));
}

// Prologue shared by the chain kernels: trigger dependents (at entry unless the node is the first
// consumer after a root table-writer), table fetch (pre- or post-wait), PDL wait.
#define CGX_PROLOGUE(a, p0, p1)                                        \
  const void* p0;                                                      \
  const void* p1;                                                      \
  if ((a).flags & kFlagEpochBump) df_bump(a);                          \
  if (!((a).flags & kFlagTriggerAfterWait)) pdl_trigger();             \
  if ((a).flags & kFlagDbgNoop) return;                                \
  if (!((a).flags & kFlagTableAfterWait)) fetch_operands((a), p0, p1); \
  sync_in(a);                                                          \
  if ((a).flags & kFlagTableAfterWait) fetch_operands((a), p0, p1);    \
  if ((a).flags & kFlagTriggerAfterWait) pdl_trigger();

// The point where a node may start reading other nodes' outputs: griddepcontrol.wait (PDL chain),
// nothing yet (deferred wait: at sync_out), or the dataflow counters (plus the PDL wait when the
// node follows a root table-writer node, kFlagTableAfterWait).
__device__ __forceinline__ void sync_in(const ElemArgs& a) {
  if (a.flags & kFlagDataflow) {
    if (a.flags & kFlagDfPdlWait) pdl_wait();
    df_wait(a);
  } else if (!(a.flags & kFlagDeferWait)) {
    pdl_wait();
  }
  trace_at(a, 1);
}
// Every CTA (all threads) must reach this once, at the very end.
__device__ __forceinline__ void sync_out(const ElemArgs& a) {
  if (a.flags & kFlagDfSignal) df_signal(a);
  else if (a.flags & kFlagDeferWait) pdl_wait();
  trace_at(a, 2);
}

// ---------------------------------------------------------------------------- f32 elementwise
// Operands whose `pre` bit is set (EXTERNAL / STATIC slots: never written inside the graph) are
// loaded before griddepcontrol.wait, overlapping the predecessors; the rest after the wait.
template <int OP, int TW>
__global__ void __launch_bounds__(kElemThreads) k_elem_f32(const __grid_constant__ ArgsTW<ElemArgs, TW> A) {
  const ElemArgs& a = A.a;
  trace_at(a, 0);
  tw_publish(A);
  constexpr bool kBinary = (OP == OP_ADD || OP == OP_MUL);
  const bool late = a.flags & kFlagTableAfterWait;
  if (a.flags & kFlagEpochBump) df_bump(a);
  if (!(a.flags & kFlagTriggerAfterWait)) pdl_trigger();
  if (a.flags & kFlagDbgNoop) return;
  const void* p0;
  const void* p1;
  if (!late) fetch_operands(a, p0, p1);
  const float4* x = reinterpret_cast<const float4*>(p0);
  const float4* y = reinterpret_cast<const float4*>(p1);
  const uint64_t n4 = a.n >> 2;
  const uint64_t base = (uint64_t)blockIdx.x * (kElemThreads * kElemVec) + threadIdx.x;
  float4 xv[kElemVec], yv[kElemVec];
  const bool pre_x = !late && (a.pre & 1u);
  const bool pre_y = kBinary && !late && (a.pre & 2u);
  // SCALE_T: the scalar operand is a 1-element device tensor (pre-wait when never written in graph)
  float sval = a.scalar;
  const bool pre_s = OP == OP_SCALE_T && !late && (a.pre & 2u);
  if (OP == OP_SCALE_T && pre_s) sval = *reinterpret_cast<const float*>(p1);
  if (pre_x) {
#pragma unroll
    for (int j = 0; j < kElemVec; ++j) {
      const uint64_t i = base + (uint64_t)j * kElemThreads;
      if (i < n4) xv[j] = ld_global_f4(x + i);
    }
  }
  if (pre_y) {
#pragma unroll
    for (int j = 0; j < kElemVec; ++j) {
      const uint64_t i = base + (uint64_t)j * kElemThreads;
      if (i < n4) yv[j] = ld_global_f4(y + i);
    }
  }
  sync_in(a);
  if (a.flags & kFlagDbgNoWork) {
    sync_out(a);
    return;
  }
  if (late) {
    fetch_operands(a, p0, p1);
    x = reinterpret_cast<const float4*>(p0);
    y = reinterpret_cast<const float4*>(p1);
  }
  if (a.flags & kFlagTriggerAfterWait) pdl_trigger();
  if (OP == OP_SCALE_T && !pre_s) sval = *reinterpret_cast<const float*>(p1);
  if (!pre_x) {
#pragma unroll
    for (int j = 0; j < kElemVec; ++j) {
      const uint64_t i = base + (uint64_t)j * kElemThreads;
      if (i < n4) xv[j] = ld_global_f4(x + i);
    }
  }
  if (kBinary && !pre_y) {
#pragma unroll
    for (int j = 0; j < kElemVec; ++j) {
      const uint64_t i = base + (uint64_t)j * kElemThreads;
      if (i < n4) yv[j] = ld_global_f4(y + i);
    }
  }
  float4* o = reinterpret_cast<float4*>(a.out);
#pragma unroll
  for (int j = 0; j < kElemVec; ++j) {
    const uint64_t i = base + (uint64_t)j * kElemThreads;
    if (i < n4) {
      float4 r;
      r.x = apply_f32<OP>(xv[j].x, yv[j].x, sval);
      r.y = apply_f32<OP>(xv[j].y, yv[j].y, sval);
      r.z = apply_f32<OP>(xv[j].z, yv[j].z, sval);
      r.w = apply_f32<OP>(xv[j].w, yv[j].w, sval);
      o[i] = r;
    }
  }
  // further tiles when the grid is capped below the tile count (grid-stride over tiles)
  for (uint64_t b2 = base + (uint64_t)gridDim.x * (kElemThreads * kElemVec); b2 < n4;
       b2 += (uint64_t)gridDim.x * (kElemThreads * kElemVec)) {
#pragma unroll
    for (int j = 0; j < kElemVec; ++j) {
      const uint64_t i = b2 + (uint64_t)j * kElemThreads;
      if (i < n4) {
        xv[j] = ld_global_f4(x + i);
        if (kBinary) yv[j] = ld_global_f4(y + i);
      }
    }
#pragma unroll
    for (int j = 0; j < kElemVec; ++j) {
      const uint64_t i = b2 + (uint64_t)j * kElemThreads;
      if (i < n4) {
        float4 r;
        r.x = apply_f32<OP>(xv[j].x, yv[j].x, sval);
        r.y = apply_f32<OP>(xv[j].y, yv[j].y, sval);
        r.z = apply_f32<OP>(xv[j].z, yv[j].z, sval);
        r.w = apply_f32<OP>(xv[j].w, yv[j].w, sval);
        o[i] = r;
      }
    }
  }
  // scalar tail (n not a multiple of 4): block 0 only
  if (blockIdx.x == 0) {
    const uint64_t t = (n4 << 2) + threadIdx.x;
    if (t < a.n) {
      const float* xs = reinterpret_cast<const float*>(p0);
      const float* ys = reinterpret_cast<const float*>(p1);
      const float yy = kBinary ? ys[t] : 0.f;
      reinterpret_cast<float*>(a.out)[t] = apply_f32<OP>(xs[t], yy, sval);
    }
  }
  sync_out(a);
}

// ---------------------------------------------------------------------------- bf16 elementwise
// Math in f32 with one RNE rounding to bf16 (exact sums/products of bf16 values whenever the
// exponent gap is < 16; SURVEY ambiguity 11).
template <int OP>
__device__ __forceinline__ __nv_bfloat16 apply_bf16(__nv_bfloat16 x, __nv_bfloat16 y, float s) {
  return __float2bfloat16_rn(apply_f32<OP>(__bfloat162float(x), __bfloat162float(y), s));
}

template <int OP, int TW>
__global__ void __launch_bounds__(kElemThreads) k_elem_bf16(const __grid_constant__ ArgsTW<ElemArgs, TW> A) {
  const ElemArgs& a = A.a;
  trace_at(a, 0);
  tw_publish(A);
  CGX_PROLOGUE(a, p0, p1)
  const uint4* x = reinterpret_cast<const uint4*>(p0);
  const uint4* y = reinterpret_cast<const uint4*>(p1);
  uint4* o = reinterpret_cast<uint4*>(a.out);
  const uint64_t n8 = a.n >> 3;
  const uint64_t base = (uint64_t)blockIdx.x * (kElemThreads * kElemVec) + threadIdx.x;
  uint4 xv[kElemVec], yv[kElemVec];
#pragma unroll
  for (int j = 0; j < kElemVec; ++j) {
    const uint64_t i = base + (uint64_t)j * kElemThreads;
    if (i < n8) {
      xv[j] = x[i];
      if (elem_binary<OP>()) yv[j] = y[i];
    }
  }
#pragma unroll
  for (int j = 0; j < kElemVec; ++j) {
    const uint64_t i = base + (uint64_t)j * kElemThreads;
    if (i < n8) {
      const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&xv[j]);
      const __nv_bfloat16* yb = reinterpret_cast<const __nv_bfloat16*>(&yv[j]);
      uint4 r;
      __nv_bfloat16* rb = reinterpret_cast<__nv_bfloat16*>(&r);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        rb[e] = apply_bf16<OP>(xb[e], elem_binary<OP>() ? yb[e] : xb[e], a.scalar);
      o[i] = r;
    }
  }
  if (blockIdx.x == 0) {
    const uint64_t t = (n8 << 3) + threadIdx.x;
    if (t < a.n) {
      const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(p0);
      const __nv_bfloat16* ys = reinterpret_cast<const __nv_bfloat16*>(p1);
      reinterpret_cast<__nv_bfloat16*>(a.out)[t] =
          apply_bf16<OP>(xs[t], elem_binary<OP>() ? ys[t] : xs[t], a.scalar);
    }
  }
  sync_out(a);
}

// ---------------------------------------------------------------------------- TRANSPOSE bf16
// out[c, r] = in[r, c] for a [rows, cols] bf16 matrix (rows = n / cols): 32 x 32 tiles staged in
// shared memory (33-column padding: conflict-free column reads), 8 rows per warp pass. A pure copy:
// bit-exact. Used by the training-shaped chain to feed transposed operands to the K-major GEMM.
static constexpr int kTrTile = 32;
template <int TW>
__global__ void __launch_bounds__(256) k_transpose_bf16(const __grid_constant__ ArgsTW<ElemArgs, TW> A) {
  const ElemArgs& a = A.a;
  trace_at(a, 0);
  tw_publish(A);
  CGX_PROLOGUE(a, p0, p1)
  (void)p1;
  __shared__ __nv_bfloat16 tile[kTrTile][kTrTile + 1];
  const uint32_t cols = a.cols, rows = (uint32_t)(a.n / a.cols);
  const __nv_bfloat16* in = reinterpret_cast<const __nv_bfloat16*>(p0);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(a.out);
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;      // 32 x 8 threads
  const uint32_t tiles_c = (cols + kTrTile - 1) / kTrTile, tiles_r = (rows + kTrTile - 1) / kTrTile;
  for (uint32_t t = blockIdx.x; t < tiles_c * tiles_r; t += gridDim.x) {
    const uint32_t r0 = (t / tiles_c) * kTrTile, c0 = (t % tiles_c) * kTrTile;
#pragma unroll
    for (uint32_t k = 0; k < kTrTile; k += 8) {
      const uint32_t r = r0 + ty + k, c = c0 + tx;
      if (r < rows && c < cols) tile[ty + k][tx] = in[(size_t)r * cols + c];
    }
    __syncthreads();
#pragma unroll
    for (uint32_t k = 0; k < kTrTile; k += 8) {
      const uint32_t c = c0 + ty + k, r = r0 + tx;                  // out row c, out col r
      if (c < cols && r < rows) out[(size_t)c * rows + r] = tile[tx][ty + k];
    }
    __syncthreads();
  }
  sync_out(a);
}

// ---------------------------------------------------------------------------- REDUCE_SUM f32
// One warp per row of `cols` floats; per-lane float64 accumulation in a fixed order, then a fixed
// xor-shuffle tree; one rounding to f32. No atomics: every arm produces identical bits.
static constexpr int kReduceThreads = 256;

template <int TW>
__global__ void __launch_bounds__(kReduceThreads) k_reduce_sum_f32(const __grid_constant__ ArgsTW<ElemArgs, TW> A) {
  const ElemArgs& a = A.a;
  trace_at(a, 0);
  tw_publish(A);
  CGX_PROLOGUE(a, p0, p1)
  (void)p1;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t rows = (a.flags & kFlagDbgNoWork) ? 0 : a.n / a.cols;
  for (uint64_t r = (uint64_t)blockIdx.x * (kReduceThreads / 32) + warp; r < rows;
       r += (uint64_t)gridDim.x * (kReduceThreads / 32)) {
    const float4* row = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p0) + r * a.cols);
    const uint32_t c4 = a.cols >> 2;
    double acc = 0.0;
    uint32_t c = lane;
    for (; c + 32 < c4; c += 64) {            // two loads in flight, same summation order
      const float4 v = ld_global_f4(row + c);
      const float4 u = ld_global_f4(row + c + 32);
      acc += (double)v.x;
      acc += (double)v.y;
      acc += (double)v.z;
      acc += (double)v.w;
      acc += (double)u.x;
      acc += (double)u.y;
      acc += (double)u.z;
      acc += (double)u.w;
    }
    if (c < c4) {
      const float4 v = ld_global_f4(row + c);
      acc += (double)v.x;
      acc += (double)v.y;
      acc += (double)v.z;
      acc += (double)v.w;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) reinterpret_cast<float*>(a.out)[r] = __double2float_rn(acc);
  }
  sync_out(a);
}

// ---------------------------------------------------------------------------- multi-tensor copy
// COPY arm: ph_j <- y_j for every tensor whose fresh source differs from
// its placeholder. The concatenation of all tensors is cut into 2 KiB blocks (one warp moves one
// block: 4 x 16-B vectors per lane, all loads before the stores); warps walk the block space with
// a grid-wide warp stride and find a block's tensor by binary search over the tensors' first
// block indices (staged in shared memory), so small and large tensors share the machine evenly. Measured on this B200 (scripts/copy_microbench.cu,
// profiles/r01): warp-contiguous 2 KiB blocks with only 2 x 256 threads per SM sustain ~6.65 TB/s
// on 3 x 1 GiB, above cudaMemcpyAsync (~6.52 TB/s); more requests in flight per SM lower it.
static constexpr int kCopyThreads = 256;
static constexpr int kCopyVec = 4;
static constexpr uint32_t kCopyBlock = 32 * kCopyVec * 16;   // 2 KiB per warp-block

template <int CAP>
__global__ void __launch_bounds__(kCopyThreads) k_copy(const __grid_constant__ CopyArgs<CAP> a) {
  // first block index of every tensor, staged once per CTA; block -> tensor is a binary search
  __shared__ uint32_t s_begin[CAP + 1];
  for (uint32_t t = threadIdx.x; t < a.n_tensors; t += kCopyThreads) s_begin[t] = (uint32_t)a.desc[t].chunk_begin;
  if (threadIdx.x == 0) s_begin[a.n_tensors] = (uint32_t)a.n_chunks;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * kCopyThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * kCopyThreads) >> 5;
  for (uint64_t q = warp; q < a.n_chunks; q += nwarps) {
    uint32_t lo = 0, hi = a.n_tensors;          // largest t with s_begin[t] <= q
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_begin[mid] <= q) lo = mid; else hi = mid;
    }
    const uint32_t t = lo;
    const char* src = reinterpret_cast<const char*>(a.src[t]);
    const CopyDesc d = a.desc[t];
    char* dst = reinterpret_cast<char*>(d.dst);
    if (src == dst) continue;                                   // SURVEY reading 1
    const uint64_t off = (q - s_begin[t]) * (uint64_t)kCopyBlock;
    const uint64_t rem = d.nbytes - off;
    const uint32_t len = (uint32_t)(rem < kCopyBlock ? rem : kCopyBlock);
    const int4* s4 = reinterpret_cast<const int4*>(src + off);
    int4* d4 = reinterpret_cast<int4*>(dst + off);
    if (len == kCopyBlock) {
      int4 v[kCopyVec];
#pragma unroll
      for (int j = 0; j < kCopyVec; ++j) v[j] = s4[j * 32 + lane];
#pragma unroll
      for (int j = 0; j < kCopyVec; ++j) d4[j * 32 + lane] = v[j];
    } else {
      const uint32_t nv = len >> 4;
      for (uint32_t i = lane; i < nv; i += 32) d4[i] = s4[i];
      const uint32_t tail = len & 15u;
      if (lane < tail) dst[off + (nv << 4) + lane] = src[off + (nv << 4) + lane];
    }
  }
}

uint32_t copy_block_bytes() { return kCopyBlock; }

// TMA bulk-copy variant (copy_impl = 2): one warp per CTA; lane 0 streams chunks through a
// kBulkStages-deep shared-memory ring with cp.async.bulk (global -> smem, mbarrier completion) and
// cp.async.bulk (smem -> global, bulk async-group completion). No register staging at all.
static constexpr int kBulkStages = 4;
static constexpr uint32_t kBulkChunk = 32768;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int CAP>
__global__ void __launch_bounds__(32, 1) k_copy_bulk(const __grid_constant__ CopyArgs<CAP> a) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t bar[kBulkStages];
  const uint32_t lane = threadIdx.x;
  if (lane == 0) {
    for (int s = 0; s < kBulkStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  // chunk list of this CTA: c_i = blockIdx.x + i * gridDim.x
  const uint32_t my_n = a.n_chunks > blockIdx.x ? (uint32_t)((a.n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
  auto chunk_of = [&](uint32_t i, const char*& src, char*& dst, uint32_t& len, uint32_t& tail) -> bool {
    const uint32_t c = blockIdx.x + i * gridDim.x;
    const uint32_t t = a.chunk_tensor[c];
    const CopyDesc d = a.desc[t];
    src = reinterpret_cast<const char*>(a.src[t]);
    dst = reinterpret_cast<char*>(d.dst);
    if (src == dst) return false;
    const uint64_t off = (uint64_t)(c - d.chunk_begin) * a.chunk_bytes;
    const uint64_t rem = d.nbytes - off;
    const uint32_t l = (uint32_t)(rem < a.chunk_bytes ? rem : a.chunk_bytes);
    src += off;
    dst += off;
    len = l & ~15u;
    tail = l & 15u;
    return true;
  };
  if (lane == 0) {
    const uint32_t pre = my_n < (uint32_t)kBulkStages ? my_n : (uint32_t)kBulkStages;
    for (uint32_t i = 0; i < pre; ++i) {
      const char* src; char* dst; uint32_t len, tail;
      if (!chunk_of(i, src, dst, len, tail) || len == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(&bar[i])) : "memory");
        continue;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(&bar[i])), "r"(len) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(smem_addr(ring + i * kBulkChunk)), "l"(src), "r"(len), "r"(smem_addr(&bar[i])) : "memory");
    }
    for (uint32_t i = 0; i < my_n; ++i) {
      const uint32_t s = i % kBulkStages;
      const uint32_t ph = (i / kBulkStages) & 1u;
      uint32_t done;
      do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(smem_addr(&bar[s])), "r"(ph) : "memory");
      } while (!done);
      const char* src; char* dst; uint32_t len, tail;
      if (chunk_of(i, src, dst, len, tail) && len) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                     ::"l"(dst), "r"(smem_addr(ring + s * kBulkChunk)), "r"(len) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      // reuse the stage of chunk i for chunk i + kBulkStages once store i has read it
      const uint32_t nx = i + kBulkStages;
      if (nx < my_n) {
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        if (!chunk_of(nx, src, dst, len, tail) || len == 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(&bar[s])) : "memory");
        } else {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(&bar[s])), "r"(len) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                       ::"r"(smem_addr(ring + s * kBulkChunk)), "l"(src), "r"(len), "r"(smem_addr(&bar[s])) : "memory");
        }
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
  __syncwarp();
  // bytewise tails (< 16 B per chunk) by the warp
  for (uint32_t i = 0; i < my_n; ++i) {
    const char* src; char* dst; uint32_t len, tail;
    if (chunk_of(i, src, dst, len, tail) && lane < tail) dst[len + lane] = src[len + lane];
  }
}

// ---------------------------------------------------------------------------- INDIRECT roots
template <int CAP>
__global__ void k_table_write(const __grid_constant__ TableWriteArgs<CAP> a) {
  pdl_trigger();   // node 1 fetches the table after its wait and triggers only after it
  for (uint32_t i = threadIdx.x; i < a.n; i += blockDim.x) a.table[i] = a.ptr[i];
}

__global__ void k_table_mapped(const __grid_constant__ MappedTableArgs a) {
  __shared__ unsigned long long s_seq;
  pdl_trigger();
  if (threadIdx.x == 0) s_seq = *a.seq;
  __syncthreads();
  const uint32_t slot = (uint32_t)(s_seq % a.ring);
  const uint64_t* src = a.staging + (uint64_t)slot * a.n_pad;
  for (uint32_t i = threadIdx.x; i < a.n; i += blockDim.x) {
    uint64_t v;
    asm volatile("ld.volatile.global.u64 %0, [%1];\n" : "=l"(v) : "l"(src + i));
    a.table[i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.seq = s_seq + 1;
    __threadfence_system();
    asm volatile("st.volatile.global.u64 [%0], %1;\n" :: "l"(a.ack), "l"(s_seq + 1) : "memory");
  }
}

// ---------------------------------------------------------------------------- utilities
__global__ void k_empty() {}
// A node that follows the chain kernels' PDL protocol but does no work: trigger at entry, wait.
__global__ void k_pdl_nop() {
  pdl_trigger();
  pdl_wait();
}

// Output gather (cgx_output_gather): CTA i copies source i (a library-owned output slot, 256-B
// aligned) to its 16-B aligned offset of the caller's packed buffer: 16-B vectors, then the tail
// bytes. One launch replaces one small device-to-host copy per output with a single one.
__global__ void __launch_bounds__(256) k_gather(const __grid_constant__ GatherArgs a) {
  const uint32_t i = blockIdx.x;
  if (i >= a.n) return;
  const uint8_t* src = static_cast<const uint8_t*>(a.src[i]);
  uint8_t* dst = static_cast<uint8_t*>(a.dst[i]);
  const uint64_t nb = a.nbytes[i], n16 = nb >> 4;
  for (uint64_t j = threadIdx.x; j < n16; j += blockDim.x)
    reinterpret_cast<uint4*>(dst)[j] = reinterpret_cast<const uint4*>(src)[j];
  for (uint64_t j = (n16 << 4) + threadIdx.x; j < nb; j += blockDim.x) dst[j] = src[j];
}

// ---------------------------------------------------------------------------- peer all-reduce
// One-shot bf16 sum across `world` ranks over peer memory (NVLink P2P stores on an NVSwitch box;
// plain device memory when the ranks share one GPU): CTA c owns vectors [c*nv/C, (c+1)*nv/C).
//  1. push: copy this rank's chunk into slot `rank` (parity buffer) of EVERY rank's receive
//     region, itself included;
//  2. publish: bar.sync, then one thread: sys-scope fence and st.release.sys of the generation g
//     into flag[ar][rank][c] of every rank;
//  3. wait until flag[ar][s][c] == g in its own region for every source s (ld.acquire.sys polls,
//     bounded: a lost peer is reported through the exec's status word, DevStatus, instead of
//     hanging), then fence + bar.sync;
//  4. sum the world slots in fixed rank order 0..world-1 in fp32 and round once: every rank
//     computes bit-identical results.
// g = ++counter[ar][c] (chain-owned, the same sequence on every rank). Every all-reduce node owns
// two receive buffers (recv[] points at this node's [2][world][slot] block); generation g uses
// parity (g - 1) & 1. A writer reaches generation g + 2 of this node only after it received every
// peer's generation g + 1 flag, which each peer publishes only after it finished reading
// generation g: reuse is safe whatever other all-reduces (or execs) run in between.
// PDL: this kernel triggers its dependents only once every source has arrived (after step 3), so
// no successor sits resident on the SMs while the all-reduce spins for its peers (a desynchronised
// rank, or ranks sharing one GPU as in the tests, could otherwise starve the peers it waits for).
__global__ void __launch_bounds__(256) k_allreduce_peer(const __grid_constant__ PeerArArgs a) {
  pdl_wait();
  __shared__ uint32_t s_g;
  const uint32_t c = blockIdx.x, C = gridDim.x;
  const uint64_t nv = a.n / 8;
  const uint64_t lo = nv * c / C, hi = nv * (c + 1) / C;
  if (threadIdx.x == 0) {
    const uint32_t g = a.counters[a.ar_index * kArMaxCtas + c] + 1;
    a.counters[a.ar_index * kArMaxCtas + c] = g;
    s_g = g;
  }
  __syncthreads();
  const uint32_t g = s_g;
  const uint32_t par = (g - 1u) & 1u;
  const uint4* in = reinterpret_cast<const uint4*>(a.in);
  // 1. push
  for (uint64_t v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    const uint4 x = in[v];
    for (uint32_t p = 0; p < a.world; ++p)
      reinterpret_cast<uint4*>(a.recv[p] + ((uint64_t)par * a.world + a.rank) * a.slot_elems)[v] = x;
  }
  __syncthreads();
  // 2. publish
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;\n" ::: "memory");
    for (uint32_t p = 0; p < a.world; ++p) {
      uint32_t* f = a.flags_of[p] + ((uint64_t)a.ar_index * kArMaxWorld + a.rank) * kArMaxCtas + c;
      asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(f), "r"(g) : "memory");
    }
    // 3. wait for every source
    for (uint32_t s2 = 0; s2 < a.world; ++s2) {
      const uint32_t* f = a.flags_of[a.rank] + ((uint64_t)a.ar_index * kArMaxWorld + s2) * kArMaxCtas + c;
      uint64_t spins = 0;
      const unsigned long long t0 = gtimer();
      for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
        if (v == g) break;
        if (spin_expired(a.st, t0, spins, kDevErrPeer)) break;   // lost peer: reported, no trap
      }
    }
    asm volatile("fence.acq_rel.sys;\n" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  // 4. fixed-order sum
  const __nv_bfloat16* mine = a.recv[a.rank] + (uint64_t)par * a.world * a.slot_elems;
  for (uint64_t v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (uint32_t s2 = 0; s2 < a.world; ++s2) {
      const uint4 x = reinterpret_cast<const uint4*>(mine + (uint64_t)s2 * a.slot_elems)[v];
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&x);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += __bfloat162float(b[e]);
    }
    uint4 o;
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
    for (int e = 0; e < 8; ++e) ob[e] = __float2bfloat16_rn(acc[e]);
    reinterpret_cast<uint4*>(a.out)[v] = o;
  }
}

// ---------------------------------------------------------------------------- NVLS all-reduce
// One-shot bf16 sum across `world` ranks through an NVSwitch multicast object (SURVEY §8(f)
// NEXT-4): every rank's region is bound to the object at the same offsets, so one multimem load
// at an address returns the reduction of that address over every rank's copy, done in the switch.
// CTA c owns vectors [c*nv/C, (c+1)*nv/C):
//  1. store this rank's chunk into its OWN copy of the parity slot (plain stores, no pushes);
//  2. arrive: bar.sync, then one thread: sys-scope fence and multimem.red.release.sys.add of 1 to
//     counter[ar][c] — on every rank's copy at once;
//  3. wait until its own copy of counter[ar][c] reaches world * g (ld.acquire.sys polls, bounded:
//     a lost rank is reported through the exec's status word), then fence + bar.sync;
//  4. multimem.ld_reduce.add.acc::f32 of the chunk through the multicast mapping (fp32
//     accumulation in the switch, one bf16 rounding) into the output.
// g = ++counter[ar][c] (chain-owned, the same sequence on every rank); parity (g - 1) & 1 — a rank
// writes generation g + 2's partial only after every rank arrived at g + 1, i.e. finished reading
// g (the peer kernel's argument). PDL trigger after step 3, as in the peer kernel.
__global__ void __launch_bounds__(256) k_allreduce_mc(const __grid_constant__ McArArgs a) {
  pdl_wait();
  __shared__ uint32_t s_g;
  const uint32_t c = blockIdx.x, C = gridDim.x;
  const uint64_t nv = a.n / 8;
  const uint64_t lo = nv * c / C, hi = nv * (c + 1) / C;
  if (threadIdx.x == 0) {
    const uint32_t g = a.counters[a.ar_index * kArMaxCtas + c] + 1;
    a.counters[a.ar_index * kArMaxCtas + c] = g;
    s_g = g;
  }
  __syncthreads();
  const uint32_t g = s_g;
  const uint64_t off = (uint64_t)((g - 1u) & 1u) * a.slot_elems;
  const uint4* in = reinterpret_cast<const uint4*>(a.in);
  uint4* mine = reinterpret_cast<uint4*>(a.uc_data + off);
  for (uint64_t v = lo + threadIdx.x; v < hi; v += blockDim.x) mine[v] = in[v];   // 1. own copy
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;\n" ::: "memory");
    asm volatile("multimem.red.release.sys.global.add.u32 [%0], 1;\n" ::"l"(a.mc_flags + c) : "memory");   // 2.
    const uint32_t target = a.world * g;   // 3. (monotonic: every rank adds 1 per generation)
    uint64_t spins = 0;
    const unsigned long long t0 = gtimer();
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(a.uc_flags + c) : "memory");
      if ((int32_t)(v - target) >= 0) break;
      if (spin_expired(a.st, t0, spins, kDevErrPeer)) break;   // lost rank: reported, no trap
    }
    asm volatile("fence.acq_rel.sys;\n" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  const __nv_bfloat16* mc = a.mc_data + off;   // 4. in-switch reduction
  for (uint64_t v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    uint4 o;
    asm volatile("multimem.ld_reduce.weak.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w) : "l"(mc + 8 * v) : "memory");
    reinterpret_cast<uint4*>(a.out)[v] = o;
  }
}

struct FillArgs { float* out; uint64_t n; uint64_t base; };
__global__ void k_fill_uniform_f32(const __grid_constant__ FillArgs a) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = splitmix_mix(a.base + i) >> 40;           // synth.splitmix recipe
    a.out[i] = __fsub_rn(__fmul_rn((float)k, 0x1p-23f), 1.0f);  // exact: k*2^-23 - 1
  }
}

// ---------------------------------------------------------------------------- handles
template <int TW>
static const void* elem_fn(int op, int dtype) {
  if (dtype == 0) {
    switch (op) {
      case OP_ADD: return (const void*)k_elem_f32<OP_ADD, TW>;
      case OP_MUL: return (const void*)k_elem_f32<OP_MUL, TW>;
      case OP_SCALE: return (const void*)k_elem_f32<OP_SCALE, TW>;
      case OP_COPY: return (const void*)k_elem_f32<OP_COPY, TW>;
      case OP_SCALE_T: return (const void*)k_elem_f32<OP_SCALE_T, TW>;
    }
  } else {
    switch (op) {
      case OP_ADD: return (const void*)k_elem_bf16<OP_ADD, TW>;
      case OP_MUL: return (const void*)k_elem_bf16<OP_MUL, TW>;
      case OP_SCALE: return (const void*)k_elem_bf16<OP_SCALE, TW>;
      case OP_COPY: return (const void*)k_elem_bf16<OP_COPY, TW>;
      case OP_SUB: return (const void*)k_elem_bf16<OP_SUB, TW>;
      case OP_AXPY: return (const void*)k_elem_bf16<OP_AXPY, TW>;
      case OP_GELU: return (const void*)k_elem_bf16<OP_GELU, TW>;
      case OP_GELU_BWD: return (const void*)k_elem_bf16<OP_GELU_BWD, TW>;
    }
  }
  return nullptr;
}
const void* kfn_elem(int op, int dtype, int tw) {
  switch (tw) {
    case 0: return elem_fn<0>(op, dtype);
    case 8: return elem_fn<8>(op, dtype);
    case 64: return elem_fn<64>(op, dtype);
    case 512: return elem_fn<512>(op, dtype);
  }
  return nullptr;
}
const void* kfn_transpose_bf16(int tw) {
  switch (tw) {
    case 0: return (const void*)k_transpose_bf16<0>;
    case 8: return (const void*)k_transpose_bf16<8>;
    case 64: return (const void*)k_transpose_bf16<64>;
    case 512: return (const void*)k_transpose_bf16<512>;
  }
  return nullptr;
}
const void* kfn_reduce_sum_f32(int tw) {
  switch (tw) {
    case 0: return (const void*)k_reduce_sum_f32<0>;
    case 8: return (const void*)k_reduce_sum_f32<8>;
    case 64: return (const void*)k_reduce_sum_f32<64>;
    case 512: return (const void*)k_reduce_sum_f32<512>;
  }
  return nullptr;
}
int tw_cap(int n) { return n <= 8 ? 8 : n <= 64 ? 64 : n <= 512 ? 512 : 0; }
const void* kfn_copy(int cap) {
  if (cap <= 8) return (const void*)k_copy<8>;
  if (cap <= 64) return (const void*)k_copy<64>;
  return (const void*)k_copy<1024>;
}
const void* kfn_copy_bulk(int cap) {
  const void* f;
  if (cap <= 8) f = (const void*)k_copy_bulk<8>;
  else if (cap <= 64) f = (const void*)k_copy_bulk<64>;
  else f = (const void*)k_copy_bulk<1024>;
  // per call (build time, cheap): function attributes belong to the current device's context
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kBulkStages * kBulkChunk);
  return f;
}
size_t copy_bulk_smem() { return (size_t)kBulkStages * kBulkChunk; }
uint32_t copy_bulk_chunk() { return kBulkChunk; }

const void* kfn_table_write(int cap) {
  if (cap <= 8) return (const void*)k_table_write<8>;
  if (cap <= 64) return (const void*)k_table_write<64>;
  return (const void*)k_table_write<512>;
}
const void* kfn_table_mapped() { return (const void*)k_table_mapped; }
const void* kfn_empty() { return (const void*)k_empty; }
const void* kfn_pdl_nop() { return (const void*)k_pdl_nop; }
const void* kfn_fill_uniform_f32() { return (const void*)k_fill_uniform_f32; }
const void* kfn_gather() { return (const void*)k_gather; }
const void* kfn_allreduce_peer() { return (const void*)k_allreduce_peer; }
const void* kfn_allreduce_mc() { return (const void*)k_allreduce_mc; }
int elem_block_threads() { return kElemThreads; }
int elem_tile_vecs() { return kElemVec; }

}  // namespace cgx
