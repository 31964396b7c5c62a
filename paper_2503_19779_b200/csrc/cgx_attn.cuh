// Causal attention tile on the warp-level bf16 tensor cores (mma.sync), shared by the per-node
// kernel (k_decoder.cu k_attention) and the persistent decoder executor (k_mega.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace cgx {

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
__device__ __forceinline__ unsigned long long attn_gtime() {   // diagnostics (per-CTA phase stamps)
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// One attention tile: query rows [16 qblock, 16 qblock + 16) of head h, with blockDim.x threads
// (>= one warp per 32-key chunk of the causal range; extra warps only help with the loads).
// Shared by k_attention (one tile per CTA) and the persistent decoder executor (k_mega.cu).
// kBulk (per-node kernel, CGX_ATTN_BULK=1 measurement variant): Q / K / V rows arrive by 128-B
// cp.async.bulk copies issued one row per thread on the mbarrier `bar` (initialised by the caller
// before its PDL wait), rows past the causal range zero-filled, Q fragments read from shared memory
// with ldmatrix.x4 — instead of every thread computing and guarding 16 vector loads plus 16
// Q-fragment loads (the deployed replay's per-CTA trace put the K/V staging at ~2 us after the
// wait, profiles/r02/attn_cta.txt). It staged sooner (median 1.5 us) but replayed the C3 chain
// 3.5 us slower, so the register path stays the default.
template <bool kBulk = false>
__device__ __forceinline__ void attn_tile(const __nv_bfloat16* qkv_in, __nv_bfloat16* out, uint32_t T, uint32_t H,
                                          float scale, uint32_t qblock, uint32_t h, uint8_t* smem,
                                          unsigned long long* ct = nullptr, uint64_t* bar = nullptr,
                                          bool qall = false) {
  const uint32_t q0 = qblock * kAttnQRows;
  const uint32_t kend = min(T, q0 + kAttnQRows);                 // keys [0, kend) are visible to the block
  const uint32_t nchunk = (kend + kAttnKChunk - 1) / kAttnKChunk;
  const uint32_t row_el = 3 * H * kAttnD;                         // qkv row length (elements)
  const __nv_bfloat16* qkv = qkv_in;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t g = lane >> 2, t4 = lane & 3;
  const uint32_t cap_rows = (T + kAttnKChunk - 1) / kAttnKChunk * kAttnKChunk;   // sized per T (host agrees)
  uint8_t* sK = smem;                                          // [cap_rows][kKVRowB]
  uint8_t* sV = sK + cap_rows * kKVRowB;
  float* sO = reinterpret_cast<float*>(sV + cap_rows * kKVRowB);  // [warps][16][64]
  float* sML = sO + (cap_rows / kAttnKChunk) * kAttnQRows * kAttnD; // [warps][16][2]
  uint8_t* sQ = reinterpret_cast<uint8_t*>(sML + (cap_rows / kAttnKChunk) * kAttnQRows * 2);   // kBulk: [16][kKVRowB]

  // ---- loads: Q fragments (registers), K/V rows [0, nchunk*32) -> smem (zero beyond kend)
  uint32_t qa[4][4];
  if constexpr (kBulk) {
    const uint32_t nrow = nchunk * kAttnKChunk;
    const uint32_t qrows = min((uint32_t)kAttnQRows, T - q0);
    const uint32_t ncopy = 2 * kend + qrows;
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                   "r"(ncopy * (uint32_t)(kAttnD * 2)) : "memory");
    for (uint32_t i = threadIdx.x; i < ncopy; i += blockDim.x) {
      const uint32_t which = i < kend ? 0u : i < 2 * kend ? 1u : 2u;   // K, V, Q
      const uint32_t j = which == 0 ? i : which == 1 ? i - kend : q0 + (i - 2 * kend);
      const __nv_bfloat16* src = qkv + (size_t)j * row_el + (which == 2 ? 0u : (1 + which) * H * kAttnD) + h * kAttnD;
      uint8_t* dst = which == 0 ? sK + j * kKVRowB : which == 1 ? sV + j * kKVRowB : sQ + (j - q0) * kKVRowB;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"((uint32_t)(kAttnD * 2)),
                   "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
    }
    // rows past the causal range / past T: zeros (P = 0 there, and 0 * garbage could be NaN)
    const uint32_t zkv = (nrow - kend) * 8, nz = 2 * zkv + (kAttnQRows - qrows) * 8;
    for (uint32_t i = threadIdx.x; i < nz; i += blockDim.x) {
      uint8_t* d = i < zkv ? sK + (kend + i / 8) * kKVRowB + 16 * (i % 8)
                 : i < 2 * zkv ? sV + (kend + (i - zkv) / 8) * kKVRowB + 16 * ((i - zkv) % 8)
                               : sQ + (qrows + (i - 2 * zkv) / 8) * kKVRowB + 16 * ((i - 2 * zkv) % 8);
      *reinterpret_cast<uint4*>(d) = make_uint4(0u, 0u, 0u, 0u);
    }
    {
      const uint32_t ba = (uint32_t)__cvta_generic_to_shared(bar);
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(ba) : "memory");
    }
    __syncthreads();   // (the zero fill)
    // Q fragments from the staged rows: matrices rows 0-7 / 8-15 x dims 16kk..+8 / +8..+16
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t addr = (uint32_t)__cvta_generic_to_shared(sQ + (lane & 15) * kKVRowB + (16 * kk + (lane >> 4) * 8) * 2);
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                   : "=r"(qa[kk][0]), "=r"(qa[kk][1]), "=r"(qa[kk][2]), "=r"(qa[kk][3]) : "r"(addr));
    }
  } else {
  // Q fragments: only the warps that own a key chunk (the others only help stage K / V) — every
  // warp loading them made the 4-B Q loads ~4x the request count of the K / V vectors
  if (warp < nchunk || qall) {
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
  }
  if (ct && threadIdx.x == 0) ct[2] = attn_gtime();   // (diagnostics: K/V staged)

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
        float v = sacc[j][e] * scale;
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
    if (nchunk == 1) {
      // one 32-key chunk (the first two query blocks; every block at T <= 16, decode): warp 0's
      // partial is the result — normalised and stored from registers, no merge round trip
      // (bit-identical to the merge, whose single weight is __expf(0) = 1)
      const float inv0 = 1.0f / l0, inv1 = 1.0f / l1;
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const uint32_t c = h * kAttnD + 8 * n + 2 * t4;
        if (qi0 < T) *reinterpret_cast<uint32_t*>(out + (size_t)qi0 * (H * kAttnD) + c) =
            pack_bf16(oacc[n][0] * inv0, oacc[n][1] * inv0);
        if (qi1 < T) *reinterpret_cast<uint32_t*>(out + (size_t)qi1 * (H * kAttnD) + c) =
            pack_bf16(oacc[n][2] * inv1, oacc[n][3] * inv1);
      }
      return;
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
  if (nchunk == 1) return;   // (CTA-uniform: warp 0 stored the result above)
  __syncthreads();
  if (ct && threadIdx.x == 0) ct[3] = attn_gtime();   // (diagnostics: partials published)
  // ---- merge the warps' partials in fixed order: out = sum_w e^{m_w - m} O_w / sum_w e^{m_w - m} l_w
  // (4 columns per item: one float4 of each warp's partial, 256 items = one per thread at 8 warps;
  // per element the same operations in the same order as one column at a time)
  for (uint32_t idx = threadIdx.x; idx < kAttnQRows * kAttnD / 4; idx += blockDim.x) {
    const uint32_t r = idx / (kAttnD / 4), c = 4 * (idx % (kAttnD / 4));
    const uint32_t qi = q0 + r;
    if (qi >= T) continue;
    float2 ml[kAttnMaxWarps];
    float m = -INFINITY;
#pragma unroll
    for (uint32_t w = 0; w < (uint32_t)kAttnMaxWarps; ++w)
      if (w < nchunk) {
        ml[w] = *reinterpret_cast<const float2*>(sML + (w * kAttnQRows + r) * 2);
        m = fmaxf(m, ml[w].x);
      }
    float l = 0.f;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (uint32_t w = 0; w < (uint32_t)kAttnMaxWarps; ++w) {
      if (w >= nchunk) break;
      const float mw = ml[w].x;
      const float f = mw == -INFINITY ? 0.f : __expf(mw - m);
      l += f * ml[w].y;
      const float4 ov = *reinterpret_cast<const float4*>(sO + (w * kAttnQRows + r) * kAttnD + c);
      o.x += f * ov.x;
      o.y += f * ov.y;
      o.z += f * ov.z;
      o.w += f * ov.w;
    }
    const float inv = 1.0f / l;
    *reinterpret_cast<uint2*>(out + (size_t)qi * (H * kAttnD) + h * kAttnD + c) =
        make_uint2(pack_bf16(o.x * inv, o.y * inv), pack_bf16(o.z * inv, o.w * inv));
  }
}

static inline size_t attn_smem_bytes(uint32_t T, bool bulk = false) {
  const size_t rows = (T + kAttnKChunk - 1) / kAttnKChunk * kAttnKChunk, warps = rows / kAttnKChunk;
  return 2 * rows * kKVRowB + warps * kAttnQRows * kAttnD * 4 + warps * kAttnQRows * 2 * 4 +
         (bulk ? kAttnQRows * kKVRowB : 0);
}

}  // namespace cgx
