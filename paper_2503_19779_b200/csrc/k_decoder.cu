// Decoder-shaped chain nodes: LayerNorm and causal attention on CUDA cores.
// Both are latency-bound at the C3 shapes (T = 128 rows of 768 bf16 = 196 KB per LN; 12 heads x
// 128 x 128 scores per attention), so the design goal is a short critical path per launch:
// warp-per-row, registers/shared memory only, PDL wait placed before the first dependent load.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "cgx_args.h"
#include "cgx_decoder.h"
#include "cgx_device.cuh"
#include "cgx_attn.cuh"

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
static constexpr int kLnWarps = 8;   // rows per CTA (8: 443.8 -> see profiles/r02/c3_knobs.txt)
static constexpr int kLnMaxVec = 8;    // 8 x 16 B per lane -> cols <= 2048
static_assert(kLnMaxVec * 8 * 32 == (int)kLnMaxCols, "k_layernorm row capacity");

// ADD: the fused ADD -> LAYERNORM pair (LnArgs::add_b / add_out): h = bf16(x + add_b) is stored to
// the ADD's slot and normalised from registers — the same values and the same reduction order as
// the unfused LN reading h back, so both paths are bit-identical.
// VEC: 16-B vectors per lane held in registers (cols <= VEC x 256): 3 for GPT-2's 768 columns keeps
// the kernel at a register budget that lets it sit beside a GEMM CTA under PDL, 8 for up to 2048
template <int TW, bool ADD, int VEC>
__global__ void __launch_bounds__(256) k_layernorm(const __grid_constant__ ArgsTW<LnArgs, TW> A) {
  const LnArgs& a = A.a;
  if (threadIdx.x == 0) node_stamp(a.ntrace, 0);
  tw_publish(A);
  const void* px = a.x;
  const bool late = a.flags & kFlagTableAfterWait;
  if (!(a.flags & kFlagTriggerAfterWait)) pdl_trigger();
  if (a.tx >= 0 && !late) px = reinterpret_cast<const void*>(ld_table(a.table + a.tx));
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row = blockIdx.x * (blockDim.x >> 5) + warp;
  const uint32_t nv = a.cols >> 3;
  // gamma / beta are STATIC (never written in the graph): fetched before the wait, overlapping
  // the predecessor, so the only post-wait round trip is the row itself
  uint4 gu[VEC], bu[VEC];
  const uint4* gr = reinterpret_cast<const uint4*>(a.g);
  const uint4* br = reinterpret_cast<const uint4*>(a.b);
  const bool params_pre = a.flags & kFlagLnParamsPre;
  if (params_pre) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const uint32_t idx = lane + i * 32;
      if (idx < nv) {
        gu[i] = __ldg(gr + idx);
        bu[i] = __ldg(br + idx);
      }
    }
  }
  pdl_wait();
  if (!params_pre) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const uint32_t idx = lane + i * 32;
      if (idx < nv) {
        gu[i] = gr[idx];
        bu[i] = br[idx];
      }
    }
  }
  if (a.tx >= 0 && late) px = reinterpret_cast<const void*>(ld_table(a.table + a.tx));
  const void* pb = a.add_b;
  if (ADD && a.tb >= 0) pb = reinterpret_cast<const void*>(ld_table(a.table + a.tb));
  if (a.flags & kFlagTriggerAfterWait) pdl_trigger();
  if (threadIdx.x == 0) node_stamp(a.ntrace, 1);
  if (row >= a.rows) {
    if (a.ntrace && lane == 0) node_stamp(a.ntrace, 2);
    return;
  }
  const uint4* xr = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(px) + (size_t)row * a.cols);
  uint4 xu[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i)
    if (lane + i * 32 < nv) xu[i] = xr[lane + i * 32];
  if constexpr (ADD) {   // h = bf16(x + b) (k_elem_bf16 ADD: fp32 sum, one rounding), stored
    const uint4* br2 = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(pb) + (size_t)row * a.cols);
    uint4* hr = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.add_out) + (size_t)row * a.cols);
    uint4 yu[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i)
      if (lane + i * 32 < nv) yu[i] = br2[lane + i * 32];
#pragma unroll
    for (int i = 0; i < VEC; ++i)
      if (lane + i * 32 < nv) {
        __nv_bfloat16* xb = reinterpret_cast<__nv_bfloat16*>(&xu[i]);
        const __nv_bfloat16* yb = reinterpret_cast<const __nv_bfloat16*>(&yu[i]);
#pragma unroll
        for (int e = 0; e < 8; ++e) xb[e] = __float2bfloat16_rn(__bfloat162float(xb[e]) + __bfloat162float(yb[e]));
        hr[lane + i * 32] = xu[i];
      }
  }
  float v[VEC][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    if (lane + i * 32 < nv) {
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&xu[i]);
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
  for (int i = 0; i < VEC; ++i)
    if (lane + i * 32 < nv)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = v[i][e] - mean;
        q += d * d;
      }
  const float var = warp_sum(q) / (float)a.cols;
  const float rstd = 1.0f / sqrtf(var + a.eps);
  uint4* orow = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.cols);
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const uint32_t idx = lane + i * 32;
    if (idx < nv) {
      const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&gu[i]);
      const __nv_bfloat16* bb = reinterpret_cast<const __nv_bfloat16*>(&bu[i]);
      uint4 r;
      __nv_bfloat16* rb = reinterpret_cast<__nv_bfloat16*>(&r);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        rb[e] = __float2bfloat16_rn((v[i][e] - mean) * rstd * __bfloat162float(gb[e]) + __bfloat162float(bb[e]));
      orow[idx] = r;
    }
  }
  if (a.ntrace && lane == 0) node_stamp(a.ntrace, 2);
}

template <int VEC>
static const void* kfn_layernorm_v(int tw, bool add) {
  if (add) return tw == 0 ? (const void*)k_layernorm<0, true, VEC> : nullptr;
  switch (tw) {
    case 0: return (const void*)k_layernorm<0, false, VEC>;
    case 8: return (const void*)k_layernorm<8, false, VEC>;
    case 64: return (const void*)k_layernorm<64, false, VEC>;
    case 512: return (const void*)k_layernorm<512, false, VEC>;
  }
  return nullptr;
}
const void* kfn_layernorm(int tw, bool add, uint32_t cols) {
  return cols <= 3u * 256u ? kfn_layernorm_v<3>(tw, add) : kfn_layernorm_v<kLnMaxVec>(tw, add);
}
void decoder_ln_launch_dims(uint32_t rows, uint32_t cols, dim3* grid, dim3* block) {
  (void)cols;
  // warps (rows) per CTA: CGX_LN_WARPS measurement knob (1..8), default kLnWarps
  static const uint32_t w = [] {
    const char* v = getenv("CGX_LN_WARPS");
    const int x = v ? atoi(v) : kLnWarps;
    return (uint32_t)(x >= 1 && x <= 8 ? x : kLnWarps);
  }();
  *grid = dim3((rows + w - 1) / w);
  *block = dim3(w * 32);
}

// ---------------------------------------------------------------------------- causal attention
// (tile body: cgx_attn.cuh)
template <bool kBulk>
__global__ void __launch_bounds__(kAttnMaxWarps * 32) k_attention(const __grid_constant__ AttnArgs a) {
  extern __shared__ __align__(16) uint8_t sm_attn[];
  unsigned long long* ct = a.ctrace ? a.ctrace + 8 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (ct && threadIdx.x == 0) ct[0] = gtimer();
  __shared__ __align__(8) uint64_t s_bar;   // the Q / K / V row copies (one phase per launch)
  if (kBulk && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&s_bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) node_stamp(a.ntrace, 0);
  if (!(a.flags & kFlagTriggerAfterWait)) pdl_trigger();
  pdl_wait();
  if (a.flags & kFlagTriggerAfterWait) pdl_trigger();
  if (threadIdx.x == 0) node_stamp(a.ntrace, 1);
  if (ct && threadIdx.x == 0) ct[1] = gtimer();
  attn_tile<kBulk>(reinterpret_cast<const __nv_bfloat16*>(a.qkv), reinterpret_cast<__nv_bfloat16*>(a.out), a.T, a.H,
                  a.scale, blockIdx.x, blockIdx.y, sm_attn, ct, &s_bar, a.flags & kAttnQAll);
  if (a.ntrace || ct) {
    __syncthreads();
    if (threadIdx.x == 0) node_stamp(a.ntrace, 2);
    if (ct && threadIdx.x == 0) ct[4] = gtimer();
  }
}

// Staging of Q / K / V: the register path by default; CGX_ATTN_BULK=1 (measurement knob, read per
// call) selects 128-B cp.async.bulk row copies on an mbarrier (attn_tile<true>), which measured
// 3.5 us per 12-layer C3 replay SLOWER (342.8 vs 339.2 us, A/B in one process,
// profiles/r02/ab_attn_bulk.txt) although it needs 61 instead of 117 registers
static bool attn_bulk() {
  const char* v = getenv("CGX_ATTN_BULK");
  return v && v[0] == '1';
}
const void* kfn_attention() { return attn_bulk() ? (const void*)k_attention<true> : (const void*)k_attention<false>; }
bool decoder_attn_supported(uint32_t T, uint32_t H, uint32_t D) {
  return D == kAttnD && T >= 1 && T <= kAttnMaxT && H >= 1 && H <= 64;
}
void decoder_attn_launch_dims(uint32_t T, uint32_t H, uint32_t D, dim3* grid, dim3* block, size_t* smem) {
  (void)D;
  *grid = dim3((T + kAttnQRows - 1) / kAttnQRows, H);
  const uint32_t warps = (T + kAttnKChunk - 1) / kAttnKChunk;   // one warp per 32-key chunk of the longest range
  uint32_t nw = warps < 1 ? 1 : warps > (uint32_t)kAttnMaxWarps ? kAttnMaxWarps : warps;
  // extra warps only help with the K/V / Q loads (all 8 by default: C3 459.1 -> 444.8 us per
  // 12-layer replay, profiles/r02/c3_knobs.txt); CGX_ATTN_WARPS measurement knob (>= the chunks)
  static const uint32_t min_w = [] {
    const char* v = getenv("CGX_ATTN_WARPS");
    const int x = v ? atoi(v) : kAttnMaxWarps;
    return (uint32_t)(x >= 1 && x <= kAttnMaxWarps ? x : kAttnMaxWarps);
  }();
  if (nw < min_w) nw = min_w;
  *block = dim3(32 * nw);
  *smem = attn_smem_bytes(T, attn_bulk());
  // per call (build time, cheap): function attributes belong to the current device's context
  cudaFuncSetAttribute(k_attention<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attn_smem_bytes(kAttnMaxT, true));
  cudaFuncSetAttribute(k_attention<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attn_smem_bytes(kAttnMaxT));
}

}  // namespace cgx
