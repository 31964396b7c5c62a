// Decoder-shaped chain nodes: LayerNorm and causal attention on CUDA cores.
// Both are latency-bound at the C3 shapes (T = 128 rows of 768 bf16 = 196 KB per LN; 12 heads x
// 128 x 128 scores per attention), so the design goal is a short critical path per launch:
// warp-per-row, registers/shared memory only, PDL wait placed before the first dependent load.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "cgx_args.h"
#include "cgx_decoder.h"
#include "cgx_device.cuh"

namespace cgx {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------- LayerNorm
static constexpr int kLnWarps = 4;
static constexpr int kLnMaxVec = 8;    // 8 x 16 B per lane -> cols <= 2048

template <int TW>
__global__ void __launch_bounds__(kLnWarps * 32) k_layernorm(const __grid_constant__ ArgsTW<LnArgs, TW> A) {
  const LnArgs& a = A.a;
  tw_publish(A);
  const void* px = a.x;
  const bool late = a.flags & kFlagTableAfterWait;
  if (!(a.flags & kFlagTriggerAfterWait)) pdl_trigger();
  if (a.tx >= 0 && !late) px = reinterpret_cast<const void*>(ld_table(a.table + a.tx));
  pdl_wait();
  if (a.tx >= 0 && late) px = reinterpret_cast<const void*>(ld_table(a.table + a.tx));
  if (a.flags & kFlagTriggerAfterWait) pdl_trigger();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row = blockIdx.x * kLnWarps + warp;
  if (row >= a.rows) return;
  const uint32_t nv = a.cols >> 3;
  const uint4* xr = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(px) + (size_t)row * a.cols);
  float v[kLnMaxVec][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kLnMaxVec; ++i) {
    const uint32_t idx = lane + i * 32;
    if (idx < nv) {
      const uint4 u = xr[idx];
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[i][e] = __bfloat162float(b[e]);
        s += v[i][e];
      }
    }
  }
  const float mean = warp_sum(s) / (float)a.cols;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < kLnMaxVec; ++i)
    if (lane + i * 32 < nv)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = v[i][e] - mean;
        q += d * d;
      }
  const float var = warp_sum(q) / (float)a.cols;
  const float rstd = 1.0f / sqrtf(var + a.eps);
  const uint4* gr = reinterpret_cast<const uint4*>(a.g);
  const uint4* br = reinterpret_cast<const uint4*>(a.b);
  uint4* orow = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.cols);
#pragma unroll
  for (int i = 0; i < kLnMaxVec; ++i) {
    const uint32_t idx = lane + i * 32;
    if (idx < nv) {
      const uint4 gu = gr[idx], bu = br[idx];
      const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&gu);
      const __nv_bfloat16* bb = reinterpret_cast<const __nv_bfloat16*>(&bu);
      uint4 r;
      __nv_bfloat16* rb = reinterpret_cast<__nv_bfloat16*>(&r);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        rb[e] = __float2bfloat16_rn((v[i][e] - mean) * rstd * __bfloat162float(gb[e]) + __bfloat162float(bb[e]));
      orow[idx] = r;
    }
  }
}

const void* kfn_layernorm(int tw) {
  switch (tw) {
    case 0: return (const void*)k_layernorm<0>;
    case 8: return (const void*)k_layernorm<8>;
    case 64: return (const void*)k_layernorm<64>;
    case 512: return (const void*)k_layernorm<512>;
  }
  return nullptr;
}
void decoder_ln_launch_dims(uint32_t rows, uint32_t cols, dim3* grid, dim3* block) {
  (void)cols;
  *grid = dim3((rows + kLnWarps - 1) / kLnWarps);
  *block = dim3(kLnWarps * 32);
}

// ---------------------------------------------------------------------------- causal attention
// CTA = (8 query rows, 1 head), 8 warps, one warp per query row; ceil(T/8) x H CTAs (192 at the C3
// shape) so every SM runs several warps. K and V rows [0, q_end) are staged in shared memory as
// bf16x2 words with a 33-word row stride (conflict-free column walks), loaded as 16-B vectors with
// all of a thread's loads in flight. Scores: lane l owns keys j = l + 32 t and keeps the query row
// in registers (4 independent FMA chains per dot). P·V: lane l owns output dims (2l, 2l+1); the
// probabilities are broadcast with shuffles, 8 keys per step, two accumulator pairs.
static constexpr int kAttnRows = 8;
static constexpr int kAttnWarps = 8;
static constexpr int kAttnMaxT = 256;
static constexpr int kAttnD = 64;
static constexpr int kKStride = kAttnD / 2 + 1;   // words per staged row

__device__ __forceinline__ float2 bf2f(uint32_t u) {
  const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u);
  return make_float2(__bfloat162float(b.x), __bfloat162float(b.y));
}

__global__ void __launch_bounds__(kAttnWarps * 32) k_attention(const __grid_constant__ AttnArgs a) {
  extern __shared__ uint32_t sm[];
  if (!(a.flags & kFlagTriggerAfterWait)) pdl_trigger();
  pdl_wait();
  if (a.flags & kFlagTriggerAfterWait) pdl_trigger();
  const uint32_t T = a.T, H = a.H;
  const uint32_t h = blockIdx.y;
  const uint32_t q0 = blockIdx.x * kAttnRows;
  const uint32_t q_end = min(T, q0 + kAttnRows);
  const uint32_t row_vec = 3 * H * kAttnD / 8;        // qkv row in 16-B vectors
  const uint4* qkv = reinterpret_cast<const uint4*>(a.qkv);
  uint32_t* sK = sm;
  uint32_t* sV = sK + T * kKStride;
  // ---- stage K and V rows [0, q_end): 8 vectors per row each, up to 8 loads per thread in flight
  {
    constexpr int kPer = (kAttnMaxT * 8 * 2) / (kAttnWarps * 32);   // max vectors per thread
    const uint32_t nvec = q_end * 8;                                  // per matrix
    uint4 buf[kPer];
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const uint32_t idx = threadIdx.x + r * kAttnWarps * 32;         // over [K vectors | V vectors]
      if (idx < 2 * nvec) {
        const uint32_t which = idx >= nvec, v = idx - which * nvec;
        const uint32_t j = v >> 3, c = v & 7;
        buf[r] = qkv[(size_t)j * row_vec + (1 + which) * H * 8 + h * 8 + c];
      }
    }
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const uint32_t idx = threadIdx.x + r * kAttnWarps * 32;
      if (idx < 2 * nvec) {
        const uint32_t which = idx >= nvec, v = idx - which * nvec;
        const uint32_t j = v >> 3, c = v & 7;
        uint32_t* d = (which ? sV : sK) + j * kKStride + 4 * c;
        d[0] = buf[r].x;
        d[1] = buf[r].y;
        d[2] = buf[r].z;
        d[3] = buf[r].w;
      }
    }
  }
  __syncthreads();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t i = q0 + warp;
  if (i >= q_end) return;
  // ---- query row in registers (each lane holds all 64 values)
  float q[kAttnD];
  {
    const uint4* qr = qkv + (size_t)i * row_vec + h * 8;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint4 u = qr[c];
      const float2 f0 = bf2f(u.x), f1 = bf2f(u.y), f2 = bf2f(u.z), f3 = bf2f(u.w);
      q[8 * c + 0] = f0.x; q[8 * c + 1] = f0.y; q[8 * c + 2] = f1.x; q[8 * c + 3] = f1.y;
      q[8 * c + 4] = f2.x; q[8 * c + 5] = f2.y; q[8 * c + 6] = f3.x; q[8 * c + 7] = f3.y;
    }
  }
  float sc[kAttnMaxT / 32];
  float m = -INFINITY;
#pragma unroll
  for (int t = 0; t < kAttnMaxT / 32; ++t) {
    const uint32_t j = lane + 32 * t;
    sc[t] = -INFINITY;
    if (32 * t <= i && j <= i) {
      const uint32_t* kr = sK + j * kKStride;
      float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll
      for (int w = 0; w < kAttnD / 2; w += 2) {
        const float2 k0 = bf2f(kr[w]), k1 = bf2f(kr[w + 1]);
        d0 = fmaf(q[2 * w], k0.x, d0);
        d1 = fmaf(q[2 * w + 1], k0.y, d1);
        d2 = fmaf(q[2 * w + 2], k1.x, d2);
        d3 = fmaf(q[2 * w + 3], k1.y, d3);
      }
      sc[t] = ((d0 + d1) + (d2 + d3)) * a.scale;
      m = fmaxf(m, sc[t]);
    }
  }
  m = warp_max(m);
  float l = 0.f;
#pragma unroll
  for (int t = 0; t < kAttnMaxT / 32; ++t) {
    const uint32_t j = lane + 32 * t;
    sc[t] = (j <= i) ? __expf(sc[t] - m) : 0.f;
    l += sc[t];
  }
  l = warp_sum(l);
  float oa0 = 0.f, oa1 = 0.f, ob0 = 0.f, ob1 = 0.f;
#pragma unroll
  for (int t = 0; t < kAttnMaxT / 32; ++t) {
    if (32 * t > i) break;
    const uint32_t jn = min(32u, i + 1 - 32 * t);     // keys of this 32-block that are <= i
    const uint32_t* vb = sV + (32 * t) * kKStride + lane;
    uint32_t jj = 0;
    for (; jj + 8 <= jn; jj += 8) {
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        const float p0 = __shfl_sync(0xffffffffu, sc[t], jj + u);
        const float p1 = __shfl_sync(0xffffffffu, sc[t], jj + u + 1);
        const float2 v0 = bf2f(vb[(jj + u) * kKStride]), v1 = bf2f(vb[(jj + u + 1) * kKStride]);
        oa0 = fmaf(p0, v0.x, oa0);
        oa1 = fmaf(p0, v0.y, oa1);
        ob0 = fmaf(p1, v1.x, ob0);
        ob1 = fmaf(p1, v1.y, ob1);
      }
    }
    for (; jj < jn; ++jj) {
      const float p0 = __shfl_sync(0xffffffffu, sc[t], jj);
      const float2 v0 = bf2f(vb[jj * kKStride]);
      oa0 = fmaf(p0, v0.x, oa0);
      oa1 = fmaf(p0, v0.y, oa1);
    }
  }
  const float inv = 1.0f / l;
  __nv_bfloat162 r;
  r.x = __float2bfloat16_rn((oa0 + ob0) * inv);
  r.y = __float2bfloat16_rn((oa1 + ob1) * inv);
  reinterpret_cast<uint32_t*>(a.out)[(size_t)i * (H * kAttnD / 2) + h * (kAttnD / 2) + lane] =
      *reinterpret_cast<uint32_t*>(&r);
}

const void* kfn_attention() { return (const void*)k_attention; }
bool decoder_attn_supported(uint32_t T, uint32_t H, uint32_t D) {
  return D == kAttnD && T >= 1 && T <= kAttnMaxT && H >= 1 && H <= 64;
}
void decoder_attn_launch_dims(uint32_t T, uint32_t H, uint32_t D, dim3* grid, dim3* block, size_t* smem) {
  (void)D;
  *grid = dim3((T + kAttnRows - 1) / kAttnRows, H);
  *block = dim3(kAttnWarps * 32);
  *smem = (size_t)2 * T * kKStride * 4;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kAttnMaxT * kKStride * 4);
    attr_set = true;
  }
}

}  // namespace cgx
