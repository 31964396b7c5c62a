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
// CTA = (16 query rows, 1 head); K and V rows [0, q_end) staged in shared memory as 32-bit bf16
// pairs with a 33-word row stride (conflict-free column walks). One warp per query row: lanes own
// keys j = lane + 32 m for the scores, then dims (2 lane, 2 lane + 1) for P·V.
static constexpr int kAttnRows = 16;
static constexpr int kAttnWarps = 4;
static constexpr int kAttnMaxT = 256;
static constexpr int kAttnD = 64;
static constexpr int kKStride = kAttnD / 2 + 1;   // words per staged row

__global__ void __launch_bounds__(kAttnWarps * 32) k_attention(const __grid_constant__ AttnArgs a) {
  extern __shared__ uint32_t sm[];
  if (!(a.flags & kFlagTriggerAfterWait)) pdl_trigger();
  pdl_wait();
  if (a.flags & kFlagTriggerAfterWait) pdl_trigger();
  const uint32_t T = a.T, H = a.H;
  const uint32_t h = blockIdx.y;
  const uint32_t q0 = blockIdx.x * kAttnRows;
  const uint32_t q_end = min(T, q0 + kAttnRows);
  const uint32_t row_words = 3 * H * kAttnD / 2;      // qkv row in 32-bit words
  const uint32_t* qkv = reinterpret_cast<const uint32_t*>(a.qkv);
  uint32_t* sK = sm;
  uint32_t* sV = sK + T * kKStride;
  float* sQ = reinterpret_cast<float*>(sV + T * kKStride);   // [kAttnRows][64]
  for (uint32_t idx = threadIdx.x; idx < q_end * (kAttnD / 2); idx += blockDim.x) {
    const uint32_t j = idx / (kAttnD / 2), w = idx % (kAttnD / 2);
    const uint32_t* r = qkv + (size_t)j * row_words;
    sK[j * kKStride + w] = r[(1 * H + h) * (kAttnD / 2) + w];
    sV[j * kKStride + w] = r[(2 * H + h) * (kAttnD / 2) + w];
  }
  for (uint32_t idx = threadIdx.x; idx < (q_end - q0) * (kAttnD / 2); idx += blockDim.x) {
    const uint32_t i = idx / (kAttnD / 2), w = idx % (kAttnD / 2);
    const uint32_t u = qkv[(size_t)(q0 + i) * row_words + h * (kAttnD / 2) + w];
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u);
    sQ[i * kAttnD + 2 * w] = __bfloat162float(b.x);
    sQ[i * kAttnD + 2 * w + 1] = __bfloat162float(b.y);
  }
  __syncthreads();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* out = reinterpret_cast<uint32_t*>(a.out);
  for (uint32_t i = q0 + warp; i < q_end; i += kAttnWarps) {
    const float* q = sQ + (i - q0) * kAttnD;
    float sc[kAttnMaxT / 32];
    float m = -INFINITY;
#pragma unroll
    for (int t = 0; t < kAttnMaxT / 32; ++t) {
      const uint32_t j = lane + 32 * t;
      sc[t] = -INFINITY;
      if (j <= i) {
        const uint32_t* kr = sK + j * kKStride;
        float dot = 0.f;
#pragma unroll
        for (int w = 0; w < kAttnD / 2; ++w) {
          const uint32_t u = kr[w];
          const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u);
          dot = fmaf(q[2 * w], __bfloat162float(b.x), dot);
          dot = fmaf(q[2 * w + 1], __bfloat162float(b.y), dot);
        }
        sc[t] = dot * a.scale;
        m = fmaxf(m, sc[t]);
      }
    }
    m = warp_max(m);
    float l = 0.f;
#pragma unroll
    for (int t = 0; t < kAttnMaxT / 32; ++t) {
      const uint32_t j = lane + 32 * t;
      sc[t] = (j <= i) ? expf(sc[t] - m) : 0.f;
      l += sc[t];
    }
    l = warp_sum(l);
    float o0 = 0.f, o1 = 0.f;
    for (uint32_t j = 0; j <= i; ++j) {
      float p = 0.f;
#pragma unroll
      for (int t = 0; t < kAttnMaxT / 32; ++t)
        if ((j >> 5) == (uint32_t)t) p = sc[t];
      p = __shfl_sync(0xffffffffu, p, j & 31);
      const uint32_t u = sV[j * kKStride + lane];
      const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u);
      o0 = fmaf(p, __bfloat162float(b.x), o0);
      o1 = fmaf(p, __bfloat162float(b.y), o1);
    }
    const float inv = 1.0f / l;
    __nv_bfloat162 r;
    r.x = __float2bfloat16_rn(o0 * inv);
    r.y = __float2bfloat16_rn(o1 * inv);
    out[(size_t)i * (H * kAttnD / 2) + h * (kAttnD / 2) + lane] = *reinterpret_cast<uint32_t*>(&r);
  }
}

const void* kfn_attention() { return (const void*)k_attention; }
bool decoder_attn_supported(uint32_t T, uint32_t H, uint32_t D) {
  return D == kAttnD && T >= 1 && T <= kAttnMaxT && H >= 1 && H <= 64;
}
void decoder_attn_launch_dims(uint32_t T, uint32_t H, uint32_t D, dim3* grid, dim3* block, size_t* smem) {
  (void)D;
  *grid = dim3((T + kAttnRows - 1) / kAttnRows, H);
  *block = dim3(kAttnWarps * 32);
  *smem = (size_t)2 * T * kKStride * 4 + (size_t)kAttnRows * kAttnD * 4;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * kAttnMaxT * kKStride * 4 + kAttnRows * kAttnD * 4);
    attr_set = true;
  }
}

}  // namespace cgx
