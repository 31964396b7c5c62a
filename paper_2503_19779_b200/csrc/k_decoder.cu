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
static_assert(kLnMaxVec * 8 * 32 == (int)kLnMaxCols, "k_layernorm row capacity");

template <int TW>
__global__ void __launch_bounds__(kLnWarps * 32) k_layernorm(const __grid_constant__ ArgsTW<LnArgs, TW> A) {
  const LnArgs& a = A.a;
  if (threadIdx.x == 0) node_stamp(a.ntrace, 0);
  tw_publish(A);
  const void* px = a.x;
  const bool late = a.flags & kFlagTableAfterWait;
  if (!(a.flags & kFlagTriggerAfterWait)) pdl_trigger();
  if (a.tx >= 0 && !late) px = reinterpret_cast<const void*>(ld_table(a.table + a.tx));
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row = blockIdx.x * kLnWarps + warp;
  const uint32_t nv = a.cols >> 3;
  // gamma / beta are STATIC (never written in the graph): fetched before the wait, overlapping
  // the predecessor, so the only post-wait round trip is the row itself
  uint4 gu[kLnMaxVec], bu[kLnMaxVec];
  const uint4* gr = reinterpret_cast<const uint4*>(a.g);
  const uint4* br = reinterpret_cast<const uint4*>(a.b);
  const bool params_pre = a.flags & kFlagLnParamsPre;
  if (params_pre) {
#pragma unroll
    for (int i = 0; i < kLnMaxVec; ++i) {
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
    for (int i = 0; i < kLnMaxVec; ++i) {
      const uint32_t idx = lane + i * 32;
      if (idx < nv) {
        gu[i] = gr[idx];
        bu[i] = br[idx];
      }
    }
  }
  if (a.tx >= 0 && late) px = reinterpret_cast<const void*>(ld_table(a.table + a.tx));
  if (a.flags & kFlagTriggerAfterWait) pdl_trigger();
  if (threadIdx.x == 0) node_stamp(a.ntrace, 1);
  if (row >= a.rows) {
    if (a.ntrace && lane == 0) node_stamp(a.ntrace, 2);
    return;
  }
  const uint4* xr = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(px) + (size_t)row * a.cols);
  uint4 xu[kLnMaxVec];
#pragma unroll
  for (int i = 0; i < kLnMaxVec; ++i)
    if (lane + i * 32 < nv) xu[i] = xr[lane + i * 32];
  float v[kLnMaxVec][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kLnMaxVec; ++i) {
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
  for (int i = 0; i < kLnMaxVec; ++i)
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
  for (int i = 0; i < kLnMaxVec; ++i) {
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
// softmax(Q K^T * scale + causal mask) V per head, bf16 in/out, on the warp-level bf16 tensor-core
// MMA (mma.sync m16n8k16, fp32 accumulate): at T = 128, D = 64 a head is 2 x 0.5 MFLOP, far too
// small for tcgen05 tiles, and the node is latency-bound (one L2 round trip for Q/K/V, a few
// dozen MMAs, one store).
// CTA = (16 query rows, 1 head); warp w owns keys [32 w, 32 w + 32) of the causal range (split-KV
// inside the CTA, FlashDecoding-style): S_w = Q K_w^T (16 MMAs), row max / exp / row sum on the
// accumulator fragments, O_w = P_w V_w (16 MMAs, P re-used from the S fragments as bf16 A
// operands), then the warps' (m_w, l_w, O_w) are merged in fixed warp order through shared memory
// (deterministic). K and V rows are staged in shared memory (padded rows: conflict-free ldmatrix),
// Q fragments are loaded straight from global memory into registers, all loads in flight at once.
static constexpr int kAttnQRows = 16;
static constexpr int kAttnKChunk = 32;
static constexpr int kAttnMaxT = 256;
static constexpr int kAttnMaxWarps = kAttnMaxT / kAttnKChunk;   // 8
static constexpr int kAttnD = 64;
static constexpr int kKVRowB = kAttnD * 2 + 16;                   // padded smem row (bytes)

__device__ __forceinline__ void mma_bf16_16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_trans(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

__global__ void __launch_bounds__(kAttnMaxWarps * 32) k_attention(const __grid_constant__ AttnArgs a) {
  extern __shared__ __align__(16) uint8_t sm_attn[];
  if (threadIdx.x == 0) node_stamp(a.ntrace, 0);
  if (!(a.flags & kFlagTriggerAfterWait)) pdl_trigger();
  pdl_wait();
  if (a.flags & kFlagTriggerAfterWait) pdl_trigger();
  if (threadIdx.x == 0) node_stamp(a.ntrace, 1);
  const uint32_t T = a.T, H = a.H;
  const uint32_t h = blockIdx.y;
  const uint32_t q0 = blockIdx.x * kAttnQRows;
  const uint32_t kend = min(T, q0 + kAttnQRows);                 // keys [0, kend) are visible to the block
  const uint32_t nchunk = (kend + kAttnKChunk - 1) / kAttnKChunk;
  const uint32_t row_el = 3 * H * kAttnD;                         // qkv row length (elements)
  const __nv_bfloat16* qkv = reinterpret_cast<const __nv_bfloat16*>(a.qkv);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t g = lane >> 2, t4 = lane & 3;
  const uint32_t cap_rows = (T + kAttnKChunk - 1) / kAttnKChunk * kAttnKChunk;   // sized per T (host agrees)
  uint8_t* sK = sm_attn;                                          // [cap_rows][kKVRowB]
  uint8_t* sV = sK + cap_rows * kKVRowB;
  float* sO = reinterpret_cast<float*>(sV + cap_rows * kKVRowB);  // [warps][16][64]
  float* sML = sO + (cap_rows / kAttnKChunk) * kAttnQRows * kAttnD; // [warps][16][2]

  // ---- loads: Q fragments (registers), K/V rows [0, nchunk*32) -> smem (zero beyond kend)
  uint32_t qa[4][4];
  {
    const uint32_t r0 = q0 + g, r1 = q0 + g + 8;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t c = h * kAttnD + 16 * kk + 2 * t4;
      qa[kk][0] = r0 < T ? *reinterpret_cast<const uint32_t*>(qkv + (size_t)r0 * row_el + c) : 0u;
      qa[kk][1] = r1 < T ? *reinterpret_cast<const uint32_t*>(qkv + (size_t)r1 * row_el + c) : 0u;
      qa[kk][2] = r0 < T ? *reinterpret_cast<const uint32_t*>(qkv + (size_t)r0 * row_el + c + 8) : 0u;
      qa[kk][3] = r1 < T ? *reinterpret_cast<const uint32_t*>(qkv + (size_t)r1 * row_el + c + 8) : 0u;
    }
  }
  {
    const uint32_t nrow = nchunk * kAttnKChunk, nvec = nrow * 8;   // 16-B vectors per matrix
    constexpr int kPer = kAttnMaxT * 8 * 2 / (kAttnMaxWarps * 32);  // <= 16 per thread
    uint4 buf[kPer];
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const uint32_t idx = threadIdx.x + r * blockDim.x;
      buf[r] = make_uint4(0u, 0u, 0u, 0u);
      if (idx < 2 * nvec) {
        const uint32_t which = idx >= nvec, v = idx - which * nvec, j = v >> 3, c = v & 7;
        if (j < kend)
          buf[r] = *reinterpret_cast<const uint4*>(qkv + (size_t)j * row_el + (1 + which) * H * kAttnD + h * kAttnD + 8 * c);
      }
    }
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const uint32_t idx = threadIdx.x + r * blockDim.x;
      if (idx < 2 * nvec) {
        const uint32_t which = idx >= nvec, v = idx - which * nvec, j = v >> 3, c = v & 7;
        *reinterpret_cast<uint4*>((which ? sV : sK) + j * kKVRowB + 16 * c) = buf[r];
      }
    }
  }
  __syncthreads();

  if (warp < nchunk) {
    const uint32_t k0 = warp * kAttnKChunk;
    // ---- S = Q K^T over this warp's 32 keys: 4 n-tiles of 8 keys x 4 k-steps of 16 dims
    float sacc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        // matrices: keys k0+8j..+8 x dims 16kk..+8 and 16kk+8..+16 (lanes 0-7 / 8-15 give rows)
        const uint32_t rr = k0 + 8 * j + (lane & 7);
        const uint32_t addr = (uint32_t)__cvta_generic_to_shared(sK + rr * kKVRowB + (16 * kk + ((lane >> 3) & 1) * 8) * 2);
        uint32_t b0, b1;
        ldsm_x2(addr, b0, b1);
        mma_bf16_16816(sacc[j], qa[kk], b0, b1);
      }
    }
    // ---- scale, causal mask, row max / exp / row sum (rows g and g+8 of the 16; quad-reduced)
    const uint32_t qi0 = q0 + g, qi1 = q0 + g + 8;
    float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t key = k0 + 8 * j + 2 * t4 + (e & 1);
        const uint32_t qi = e < 2 ? qi0 : qi1;
        float v = sacc[j][e] * a.scale;
        if (key > qi || key >= T) v = -INFINITY;
        sacc[j][e] = v;
        if (e < 2) m0 = fmaxf(m0, v);
        else m1 = fmaxf(m1, v);
      }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
      m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    // rows past T (ragged tail) have no visible key: keep them finite, they are never stored
    const float mm0 = m0 == -INFINITY ? 0.f : m0, mm1 = m1 == -INFINITY ? 0.f : m1;
    float l0 = 0.f, l1 = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sacc[j][0] = __expf(sacc[j][0] - mm0);
      sacc[j][1] = __expf(sacc[j][1] - mm0);
      sacc[j][2] = __expf(sacc[j][2] - mm1);
      sacc[j][3] = __expf(sacc[j][3] - mm1);
      l0 += sacc[j][0] + sacc[j][1];
      l1 += sacc[j][2] + sacc[j][3];
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, o);
      l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    // ---- O = P V: 2 k-steps of 16 keys x 8 n-tiles of 8 dims; P fragments from the S accumulators
    float oacc[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) oacc[n][0] = oacc[n][1] = oacc[n][2] = oacc[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16(sacc[2 * kk][0], sacc[2 * kk][1]);
      pa[1] = pack_bf16(sacc[2 * kk][2], sacc[2 * kk][3]);
      pa[2] = pack_bf16(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
      pa[3] = pack_bf16(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3]);
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        // matrices: keys k0+16kk..+8 and +8..+16 x dims 8n..+8, transposed
        const uint32_t rr = k0 + 16 * kk + (lane & 7) + ((lane >> 3) & 1) * 8;
        const uint32_t addr = (uint32_t)__cvta_generic_to_shared(sV + rr * kKVRowB + 8 * n * 2);
        uint32_t b0, b1;
        ldsm_x2_trans(addr, b0, b1);
        mma_bf16_16816(oacc[n], pa, b0, b1);
      }
    }
    // ---- publish this warp's partial (m, l, O) for the merge
    float* o = sO + warp * kAttnQRows * kAttnD;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const uint32_t c = 8 * n + 2 * t4;
      *reinterpret_cast<float2*>(o + g * kAttnD + c) = make_float2(oacc[n][0], oacc[n][1]);
      *reinterpret_cast<float2*>(o + (g + 8) * kAttnD + c) = make_float2(oacc[n][2], oacc[n][3]);
    }
    if (t4 == 0) {
      sML[(warp * kAttnQRows + g) * 2 + 0] = m0;
      sML[(warp * kAttnQRows + g) * 2 + 1] = l0;
      sML[(warp * kAttnQRows + g + 8) * 2 + 0] = m1;
      sML[(warp * kAttnQRows + g + 8) * 2 + 1] = l1;
    }
  }
  __syncthreads();
  // ---- merge the warps' partials in fixed order: out = sum_w e^{m_w - m} O_w / sum_w e^{m_w - m} l_w
  for (uint32_t idx = threadIdx.x; idx < kAttnQRows * kAttnD / 2; idx += blockDim.x) {
    const uint32_t r = idx / (kAttnD / 2), c = 2 * (idx % (kAttnD / 2));
    const uint32_t qi = q0 + r;
    if (qi >= T) continue;
    float m = -INFINITY;
    for (uint32_t w = 0; w < nchunk; ++w) m = fmaxf(m, sML[(w * kAttnQRows + r) * 2]);
    float l = 0.f, ox = 0.f, oy = 0.f;
    for (uint32_t w = 0; w < nchunk; ++w) {
      const float mw = sML[(w * kAttnQRows + r) * 2];
      const float f = mw == -INFINITY ? 0.f : __expf(mw - m);
      l += f * sML[(w * kAttnQRows + r) * 2 + 1];
      const float2 ov = *reinterpret_cast<const float2*>(sO + (w * kAttnQRows + r) * kAttnD + c);
      ox += f * ov.x;
      oy += f * ov.y;
    }
    const float inv = 1.0f / l;
    *reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)qi * (H * kAttnD) + h * kAttnD + c) =
        pack_bf16(ox * inv, oy * inv);
  }
  if (a.ntrace) {
    __syncthreads();
    if (threadIdx.x == 0) node_stamp(a.ntrace, 2);
  }
}

const void* kfn_attention() { return (const void*)k_attention; }
bool decoder_attn_supported(uint32_t T, uint32_t H, uint32_t D) {
  return D == kAttnD && T >= 1 && T <= kAttnMaxT && H >= 1 && H <= 64;
}
static size_t attn_smem_bytes(uint32_t T) {
  const size_t rows = (T + kAttnKChunk - 1) / kAttnKChunk * kAttnKChunk, warps = rows / kAttnKChunk;
  return 2 * rows * kKVRowB + warps * kAttnQRows * kAttnD * 4 + warps * kAttnQRows * 2 * 4;
}
void decoder_attn_launch_dims(uint32_t T, uint32_t H, uint32_t D, dim3* grid, dim3* block, size_t* smem) {
  (void)D;
  *grid = dim3((T + kAttnQRows - 1) / kAttnQRows, H);
  const uint32_t warps = (T + kAttnKChunk - 1) / kAttnKChunk;   // one warp per 32-key chunk of the longest range
  *block = dim3(32 * (warps < 1 ? 1 : warps > (uint32_t)kAttnMaxWarps ? kAttnMaxWarps : warps));
  *smem = attn_smem_bytes(T);
  // per call (build time, cheap): function attributes belong to the current device's context
  cudaFuncSetAttribute(k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attn_smem_bytes(kAttnMaxT));
}

}  // namespace cgx
