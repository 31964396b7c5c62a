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
// Programmatic dependent launch: when W is a STATIC slot (weights never written by the chain) the
// producer prefetches this CTA's whole W slab into L2 and issues the first stages' W tiles BEFORE
// griddepcontrol.wait; only the A tiles (the predecessor's output) wait (kGemmWAfterWait moves the
// W loads behind the wait when a node writes W: the training chain). At the C3 shapes the GEMMs are
// weight-streaming / latency bound (M = 128: ~128 FLOP/B, below the ~210 FLOP/B ridge), so
// overlapping the weight fetch with the previous node's tail is the main lever.
//
// Also here: split-K over a thread-block cluster with bulk-DSMEM pushes (below), the fused
// tensor-parallel all-reduce epilogue (CGX_GEMM_ALLREDUCE), and the small-M (decode) path
// k_gemv_bf16.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/cgx.h"
#include "cgx_args.h"
#include "cgx_attn.cuh"
#include "cgx_decoder.h"
#include "cgx_device.cuh"
#include "cgx_umma.cuh"

namespace cgx {

static constexpr int kBM = 128;
static constexpr int kBK = 64;          // 64 bf16 = 128 B = one swizzle-128B row
// Operand pipelines (r02, profiles/r02/tma_issue_microbench.txt): A and W flow through SEPARATE
// mbarrier rings of groups of G k-blocks (one 3-D TMA box {64, rows, G} per group, landing as G
// stacked SW128 K-major tiles = the UMMA operand layout). One SM pulls ~160 GB/s from L2 when all
// of a CTA's boxes are in flight at once (12 x 16 KiB in 1.25 us), whereas a ring that refills a
// slot only after the MMA consumed it exposes one L2 round trip per refill. So the activation A
// (the operand that arrives after the PDL wait, on the critical path) is held WHOLE in shared
// memory whenever it fits ("one-shot": every A box is issued right after the wait, one barrier per
// k-block so the MMAs start with the first), and the small weight slab W (static: issued before
// the wait) cycles through the remaining space.
static constexpr int kMaxGroupKb = 8;   // k-blocks per box
static constexpr uint32_t kSmemLimit = 232448u;   // dynamic shared memory per block (227 KiB)
static constexpr uint32_t kSmemFixed = 1024u + 512u + 16u + 256u + 512u;   // align, bias, words, tensor map, barriers
static constexpr int kGemmThreads = 192;
static constexpr uint32_t kGemmTriggerAfterWait = 1u << 8;   // internal flag bit (above CGX_GEMM_*)
// W (and bias) written by an earlier node of the graph (training chain: transposed activations,
// updated weights): no pre-wait weight prefetch / loads
static constexpr uint32_t kGemmWAfterWait = 1u << 11;
// A is rebound per replay (EXTERNAL A operand, PI through the TMA descriptor; "de-
// references these pointers-to-pointers before performing any computation"): the producer warp
// builds this CTA's own copy of the A tensor map in global memory with the replay's address
// (table[ta] under INDIRECT, the patched a_ptr field in the patch modes) and loads A through it.
static constexpr uint32_t kGemmADynamic = 1u << 12;
// EAGER: two launches of the same node may overlap under PDL (node k of iteration i + 1 can start
// while node k of iteration i still waits), so the per-CTA map is rewritten only after this
// launch's griddepcontrol.wait (every earlier launch in the stream has then completed). In graphs
// a node runs once per replay and replays are stream-serialised: the map is built pre-wait.
static constexpr uint32_t kGemmADynAfterWait = 1u << 13;
static constexpr uint32_t kGemmFenceOnWait = 1u << 14;   // experiment: tcgen05 fence only after a barrier wait
// LayerNorm folded into the GEMM (exec option fuse & CGX_FUSE_LN_GEMM). With
// a = LN(h) = (h - mean) * rstd * gamma + beta:
//   a W^T [m, n] = rstd_m * (h W'^T)[m, n] - rstd_m * mean_m * c1[n] + c2[n],
//   W' = bf16(gamma * W) (per column k), c1[n] = sum_k W'[n, k], c2[n] = sum_k beta_k W[n, k],
// so the MMAs run on the LN's INPUT h with the gamma-scaled weights W' (prepared once at exec
// creation, cgx_ln_fold_prep) and the epilogue applies the row correction before bias / GELU /
// residual; mean / rstd come from the row sums the producer GEMM wrote (kGemmStatsOut). While the
// MMAs run, the epilogue warps of every CTA also store a slice of a = LN(h) to the LN node's output
// slot, so every node output is still materialised.
static constexpr uint32_t kGemmLnA = 1u << 15;
static constexpr uint32_t kLnMaxTiles = 64;   // producer N tiles whose row sums a kGemmLnA GEMM combines
// This GEMM's epilogue writes per-row {sum, sum of squares} of its bf16 output tile to
// stats_out[n_tile][M] (float2) for a kGemmLnA consumer.
static constexpr uint32_t kGemmStatsOut = 1u << 16;
// Phase tracer (GemmArgs::trace) in SM clock cycles (clock64) instead of %globaltimer, whose 256 ns
// tick is too coarse for sub-µs phases; cycle stamps are only comparable within one CTA.
static constexpr uint32_t kGemmTraceClk = 1u << 17;
// Causal attention folded into the small-M (GEMV) consumer (exec option fuse & CGX_FUSE_ATTN_GEMM,
// T = M = 1, the decode step): every warp forms its K slice of A = softmax(q k^T *
// scale) v from the qkv row itself (one visible key: exactly v, gv_attn_row); the first column
// group's warps of CTA 0 store the ATTN node's output row, so every node output is still
// materialised.
static constexpr uint32_t kGemmAttnA = 1u << 18;

struct alignas(64) GemmArgs {
  CUtensorMap tmA;            // A [M, K] bf16 as 3-D {64, M, K/64}, box {64, 128, group}
  CUtensorMap tmB;            // W [N, K] bf16 as 3-D {64, N, K/64}, box {64, BN, group}
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  __nv_bfloat16* out;
  float* ws;                  // split-K partial tiles [split][tiles][128][BN] (split > 1)
  unsigned long long* cnt;    // per-tile monotonic arrival counters (split > 1)
  uint32_t M, N, K, flags;
  uint32_t split;             // K splits (gridDim.z)
  uint32_t ga, ra;            // A: k-blocks per box, groups resident (ra * ga >= k-blocks: one-shot)
  uint32_t gw, rw;            // W: k-blocks per box, groups resident
  unsigned long long* trace;  // optional per-CTA %globaltimer trace [cta][16] (diagnostics)
  const uint64_t* table;      // INDIRECT: pointer table; residual = table[tres] when tres >= 0
  int32_t tres;               // table index of an EXTERNAL residual (-1: `residual` is direct)
  int32_t ta;                 // kGemmADynamic: table index of A (-1: a_ptr, a patched field)
  CUtensorMap* tm_ws;         // kGemmADynamic: per-CTA tensor-map workspace [ctas] (128-B aligned)
  const __nv_bfloat16* a_ptr; // small-M path (k_gemv_bf16): A and W by plain pointers
  const __nv_bfloat16* w_ptr;
  // CGX_GEMM_ALLREDUCE: the epilogue's peer all-reduce (same protocol and regions as
  // k_allreduce_peer, flags indexed by this GEMM's CTA)
  uint32_t ar_rank, ar_world, ar_index, ar_nar;
  uint64_t ar_slot;
  uint32_t* ar_counters;
  __nv_bfloat16* ar_recv[kArMaxWorld];
  uint32_t* ar_flags[kArMaxWorld];
  DevStatus st;               // spin bound / lost-peer report (CGX_GEMM_ALLREDUCE)
  unsigned long long* ntrace; // CGX_NODE_TRACE=1: replay timeline [entry, ready, exit] ns
  float2* stats_out;          // kGemmStatsOut: [N / BN][M] row sums of this GEMM's output
  const float2* ln_stats;     // kGemmLnA: the producer's [ln_ntiles][M] row sums of h
  const __nv_bfloat16* ln_g;  // kGemmLnA: gamma / beta [K]
  const __nv_bfloat16* ln_b;
  __nv_bfloat16* ln_out;      // kGemmLnA: the LN node's output slot [M][K]
  const __nv_bfloat16* ln_h;  // kGemmLnA: the LN input h [M][K] (also A)
  const float* ln_c1;         // kGemmLnA: [N] row sums of W'
  const float* ln_c2;         // kGemmLnA: [N] beta . W
  uint32_t ln_ntiles;
  float ln_eps;
  uint32_t ln_dbg;            // measurement knob (CGX_LN_DBG): 1 = serial stats loop, 2 = skip the LN output
  const __nv_bfloat16* attn_qkv;  // kGemmAttnA: the ATTN node's input [M][3 K] (q | k | v, head-major)
  __nv_bfloat16* attn_out;        // kGemmAttnA: the ATTN node's output slot [M][K]
  uint32_t attn_H;                // kGemmAttnA, tcgen05 path: heads (qkv row = 3 H k-blocks of 64)
  float attn_scale;               // kGemmAttnA, tcgen05 path: softmax scale
};

__device__ __forceinline__ void trace_at(const GemmArgs& a, int slot) {
  if (a.trace) {
    unsigned long long t;
    if (a.flags & kGemmTraceClk) t = clock64();
    else asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const uint32_t cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    a.trace[cta * 16 + slot] = t;
  }
}

// ------------------------------------------------------------------ kernel
// Split-K (gridDim.z = S, launched as thread-block clusters (1, 1, S)): CTA z accumulates the
// k-blocks [nk*z/S, nk*(z+1)/S) in TMEM. The output rows of the tile are partitioned over the S
// CTAs (CTA o owns rows [ceil(128 o/S), ceil(128 (o+1)/S))). Each CTA stages its fp32 partial tile
// in its (now idle) operand ring, then pushes every peer owner's row block into that owner's
// receive slot z with ONE bulk shared::cta -> shared::cluster copy that completes bytes on the
// owner's receive mbarrier (expect_tx armed at init). The owner sums the S slots of its rows in
// fixed split order 0..S-1 (deterministic, no float atomics, no global workspace; its own slot is
// read from its staging tile) and runs the epilogue. Cluster barriers: phase 0 publishes the
// receive mbarriers' initialisation (armed at entry, waited just before the first push); phase 1
// is arrived at as soon as a CTA's incoming copies are complete and waited on at exit, so no CTA
// releases a staging tile a peer is still copying from. (Per-thread st.async pushes of 16 B each
// measured slower for BN >= 64: the DSMEM transaction rate bounds them.)
__host__ __device__ constexpr uint32_t split_row_lo(uint32_t z, uint32_t S) { return (128u * z + S - 1) / S; }
__host__ __device__ constexpr uint32_t split_rows_max(uint32_t S) { return (128u + S - 1) / S; }

// ---- CGX_GEMM_ALLREDUCE epilogue helpers (protocol of k_allreduce_peer, k_chain.cu)
__device__ __forceinline__ __nv_bfloat16* ar_slot_ptr(const GemmArgs& a, uint32_t region, uint32_t par, uint32_t src) {
  return a.ar_recv[region] + ((uint64_t)par * a.ar_world + src) * a.ar_slot;
}
// Epilogue threads only (named barrier 1): publish this CTA's generation to every rank, wait for
// every source's, with sys-scope release / acquire.
__device__ __forceinline__ void ar_publish_wait(const GemmArgs& a, uint32_t cta, uint32_t g, uint32_t et) {
  asm volatile("bar.sync 1, 128;\n" ::: "memory");
  if (et == 0) {
    asm volatile("fence.acq_rel.sys;\n" ::: "memory");
    for (uint32_t p = 0; p < a.ar_world; ++p) {
      uint32_t* f = a.ar_flags[p] + ((uint64_t)a.ar_index * kArMaxWorld + a.ar_rank) * kArMaxCtas + cta;
      asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(f), "r"(g) : "memory");
    }
    for (uint32_t s2 = 0; s2 < a.ar_world; ++s2) {
      const uint32_t* f = a.ar_flags[a.ar_rank] + ((uint64_t)a.ar_index * kArMaxWorld + s2) * kArMaxCtas + cta;
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
  asm volatile("bar.sync 1, 128;\n" ::: "memory");
}


// ---- attention folded into the O-proj GEMM's A operand (ATT instantiation, exec option fuse &
// CGX_FUSE_ATTN_GEMM with T <= 128). K split S = H / HP: split z holds k-blocks
// [HP z, HP z + HP) of A = heads HP z .. HP z + HP - 1, so the CTA computes those 64-column blocks
// of A itself — causal attention of its heads over all M <= 128 query rows — on the tensor cores,
// HP <= 2 heads per CTA, double-buffered: the producer TMA-loads every head's Q, K, V tiles up front
// ([128][128 B] SW128, rows >= T zero-filled by the tensor map); the MMA warp issues S = Q K^T
// (M 128, N 128, K 64) for every head as its tiles land (TMEM S region per head, so head 1's S
// overlaps head 0's softmax); each epilogue thread owns one query row (its TMEM lane): causal mask,
// max, p = 2^(s * scale * log2 e - max'), l = sum p, and writes bf16(p) into the P tile (K-major
// SW128, two 64-key k-blocks over the head's dead Q / K tiles; key groups past the warp's causal
// range are zeros without a TMEM read); the MMA warp issues O = P V (N 64, K 128, V read MN-major
// straight from its TMA tile) into the O region; the thread scales its O row by 1 / l,
// rounds to bf16 into the UMMA A tile (and, in N tile 0, into the ATTN node's output slot, so every
// node output is materialised). The O-proj MMAs then run as in any split-K GEMM (columns [0, 32)).
// Each N tile recomputes its heads' attention (N / BN times: tensor-core work, cheap) — instead of a
// separate attention launch and the activation round trip through L2 between the two nodes.
// TMEM columns: O-proj accumulator [0, 32), S of head 0 / 1 [32, 160) / [160, 288), O [288, 352)
static constexpr uint32_t kAttTmemS = 32, kAttTmemO = 288, kAttTmemCols = 512;
static constexpr uint32_t kAttQkvBytes = 3u * 128u * 128u;   // one head's Q | K | V tiles
// UMMA smem descriptor, MN-major, 128-byte swizzle (V as the B operand of P V: rows = keys (K),
// 64 contiguous head dims (N) per 128-B row, 8-key atoms of 1024 B): SBO = 1024 B between K atoms,
// LBO = stride between 64-wide N blocks (one block here).
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(8192 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t chunk) {   // byte offset of 16-B chunk of row r
  return r * 128u + (((chunk ^ r) & 7u) << 4);
}

template <int BN, bool AR, bool ATT = false>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm_bf16(const __grid_constant__ GemmArgs a) {
  constexpr uint32_t kABytes = kBM * kBK * 2;     // 16 KiB
  constexpr uint32_t kBBytes = BN * kBK * 2;
  constexpr uint32_t kTmemCols = ATT ? kAttTmemCols : BN < 32 ? 32 : BN;
  const uint32_t GA = a.ga, RA = a.ra, GW = a.gw, RW = a.rw;
  constexpr uint32_t kRowF = BN + 4;              // partial-tile row stride (floats): 16-B aligned, bank-spread
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment (SWIZZLE_128B) by offsetting the __shared__ array itself, so every derived
  // pointer stays in the shared address space (LDS/STS; a uintptr_t round trip made them generic)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t S = a.split;
  const uint32_t z = blockIdx.z;                   // cluster (1,1,S) over gridDim.z == S: rank == z
  const uint32_t rows_max = split_rows_max(S);
  uint8_t* sA = smem;                              // [RA][GA][128 x 128 B]
  uint8_t* sB = smem + RA * GA * kABytes;          // [RW][GW][BN x 128 B]
  // The operand rings double as the epilogue staging area once the MMAs are done: the fp32
  // partial tile [128][kRowF] (split-K).
  const uint32_t ring_bytes = RA * GA * kABytes + RW * GW * kBBytes;
  const uint32_t stage_bytes = S > 1 ? 128u * kRowF * 4u : 0u;
  float* recv = reinterpret_cast<float*>(smem + (ring_bytes > stage_bytes ? ring_bytes : stage_bytes));  // [S][rows_max][kRowF]
  float* sbias = recv + (S > 1 ? S * rows_max * kRowF : 0);                     // [BN] fp32 bias slice
  uint64_t* full_a = reinterpret_cast<uint64_t*>(sbias + BN);
  uint64_t* empty_a = full_a + RA;
  uint64_t* full_w = empty_a + RA;
  uint64_t* empty_w = full_w + RW;
  uint64_t* tmem_full = empty_w + RW;
  uint64_t* recv_full = tmem_full + 1;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(recv_full + 1);   // [0] TMEM address, [1] AR generation
  uint32_t* s_tm = reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(s_tmem + 4) + 127) & ~uintptr_t(127));
  float2* s_mr = reinterpret_cast<float2*>(s_tm + 32);              // kGemmLnA: [128] (mean, rstd) per tile row
  float2* s_cc = s_mr + kBM;                                         // kGemmLnA: [BN] (c1, c2) of the tile's columns
  uint64_t* qkv_full = reinterpret_cast<uint64_t*>(s_cc + BN);       // ATT: [2] head i's Q / K / V tiles landed
  uint64_t* s_full = qkv_full + 2;                                   // ATT: [2] head i's S = Q K^T in TMEM
  uint64_t* p_full = qkv_full + 4;                                   // ATT: a P tile written (4 warps)
  uint64_t* o_full = qkv_full + 5;                                   // ATT: O = P V in TMEM
  uint8_t* sQKV = smem + ((smem_u32(qkv_full + 6) - smem_u32(smem) + 1023u) & ~1023u);   // ATT: [2][3][128][128 B]
  // the folded LayerNorm is a runtime flag of the one kernel, not a separate instantiation: a
  // dedicated <BN, AR, LN> kernel (128 vs 164 registers) replayed the fused-LN C3 chain in 424 us
  // against 379 us for this generic one, every other node unchanged (profiles/r02/c3_fuse_ln_gemm.txt)
  const bool ln_a = a.flags & kGemmLnA;

  if (threadIdx.x == 0) {
    trace_at(a, 0);
    node_stamp(a.ntrace, 0);
  }
  // an all-reducing GEMM never triggers early: no successor may sit resident while it waits for
  // its peers (dependents then launch at its completion)
  constexpr bool ar = AR;                        // CGX_GEMM_ALLREDUCE instantiation
  const bool late_trigger = (a.flags & kGemmTriggerAfterWait) && !ar;
  if (!late_trigger && !ar) pdl_trigger();   // dependents may start their prologues (they read our output after their wait)
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN;
  const int m0 = blockIdx.y * kBM;
  const int nk = (int)(a.K / kBK);
  const int kbase = (int)((uint32_t)nk * z / S);
  const int kps = (int)((uint32_t)nk * (z + 1) / S) - kbase;   // k-blocks of this split (>= 1)
  const int nga = (kps + (int)GA - 1) / (int)GA, ngw = (kps + (int)GW - 1) / (int)GW;   // operand groups
  const uint32_t my_lo = split_row_lo(z, S), my_rows = split_row_lo(z + 1, S) - my_lo;
  const bool dyn_a = a.flags & kGemmADynamic;

  if (warp == 0 && lane == 0) {
    if (!dyn_a) prefetch_tmap(&a.tmA);
    prefetch_tmap(&a.tmB);
    for (uint32_t s = 0; s < RA; ++s) {
      mbar_init(&full_a[s], ATT ? 4u : 1u);   // ATT: the 4 attention warps write the A tile
      mbar_init(&empty_a[s], 1);
    }
    if (ATT) {
      mbar_init(&qkv_full[0], 1);
      mbar_init(&qkv_full[1], 1);
      mbar_init(&s_full[0], 1);
      mbar_init(&s_full[1], 1);
      mbar_init(p_full, 4);
      mbar_init(o_full, 1);
    }
    for (uint32_t s = 0; s < RW; ++s) {
      mbar_init(&full_w[s], 1);
      mbar_init(&empty_w[s], 1);
    }
    mbar_init(tmem_full, 1);
    if (S > 1) {
      mbar_init(recv_full, 1);
      // armed now, before the cluster barrier that lets peers push: one arrival + the peers' bytes
      mbar_expect_tx(recv_full, (S - 1) * my_rows * kRowF * 4u);
    }
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
  if (threadIdx.x == 0) trace_at(a, 1);
  // (relaxed: fence.mbarrier_init above already orders the barrier initialisation at cluster scope;
  // a .release arrive compiles to MEMBAR.ALL.GPU, which drains this thread's outstanding memory ops)
  if (S > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  const uint32_t tmem = *s_tmem;

  if (warp == 0) {
    // ---- TMA producer (lane 0; the whole warp builds a dynamic A tensor map). Weights first
    // (independent of the predecessor), then the PDL wait, then A. One 3-D box per operand per
    // group of G k-blocks; the box bytes always count in full (a short last group's extra k-blocks
    // are fetched, or zero-filled past K, and never multiplied).
    const CUtensorMap* tmA = &a.tmA;
    const bool dyn_late = dyn_a && (a.flags & kGemmADynAfterWait);
    auto build_a = [&]() {
      // the replay's A address: the pointer table (written before the graph's first consumer; a
      // GEMM never is the first consumer after a root table writer) or the patched a_ptr field
      uint64_t addr = 0;
      if (lane == 0) addr = a.ta >= 0 ? ld_table(a.table + a.ta) : reinterpret_cast<uint64_t>(a.a_ptr);
      addr = __shfl_sync(0xffffffffu, addr, 0);
      const uint32_t cta_lin = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      tmA = build_dynamic_tmap(&a.tmA, a.tm_ws + cta_lin, s_tm, addr, lane);
    };
    if (dyn_a && !dyn_late) build_a();
    // the whole warp runs the producer loop (converged: elect.sync picks the issuing lane)
    const int pre_a = nga < (int)RA ? nga : (int)RA, pre_w = ngw < (int)RW ? ngw : (int)RW;
    const bool w_late = a.flags & kGemmWAfterWait;
    if (w_late) pdl_wait();
    if (lane == 0)
      for (int g = pre_w; g < ngw; ++g) tma_prefetch_l2_3d(&a.tmB, 0, n0, kbase + g * (int)GW);   // beyond the ring
    __syncwarp();
    for (int g = 0; g < pre_w; ++g) {
      mbar_expect_tx_w(&full_w[g], GW * kBBytes);
      tma_load_3d_w(sB + g * GW * kBBytes, &a.tmB, &full_w[g], 0, n0, kbase + g * (int)GW);
    }
    if (!w_late) pdl_wait();
    if (lane == 0) node_stamp(a.ntrace, 1);
    if (dyn_late) build_a();                        // every lane has passed the wait
    if (late_trigger) pdl_trigger();
    if constexpr (ATT) {   // each head's Q, K, V tiles (tmA maps qkv [M][3 H * 64]; k-block = part * H + head)
      for (int i = 0; i < kps; ++i) {   // (kps <= 2: one buffer per head)
        mbar_expect_tx_w(&qkv_full[i], 3 * kABytes);
#pragma unroll
        for (int part = 0; part < 3; ++part)
          tma_load_3d_w(sQKV + i * kAttQkvBytes + part * kABytes, tmA, &qkv_full[i], 0, m0,
                        part * (int)a.attn_H + kbase + i);
      }
    } else {
      for (int g = 0; g < pre_a; ++g) {             // the whole A slice (one-shot) or the first RA groups
        mbar_expect_tx_w(&full_a[g], GA * kABytes);
        tma_load_3d_w(sA + g * GA * kABytes, tmA, &full_a[g], 0, m0, kbase + g * (int)GA);
      }
    }
    if (lane == 0) trace_at(a, 11);
    // refills in the order the MMAs consume k-blocks (deadlock-free: each waits for an earlier
    // k-block's release); slot / phase counters advance incrementally (no divisions)
    // (the first refill of a ring reuses slot 0 and waits for its release #1, i.e. parity 0)
    int ia = pre_a, iw = pre_w, sa = 0, sw = 0;
    uint32_t pha = 0u, phw = 0u;
    while (ia < nga || iw < ngw) {
      const int ka = ia < nga ? ia * (int)GA : 1 << 30, kw = iw < ngw ? iw * (int)GW : 1 << 30;
      if (ka <= kw) {
        mbar_wait(&empty_a[sa], pha);
        mbar_expect_tx_w(&full_a[sa], GA * kABytes);
        tma_load_3d_w(sA + sa * GA * kABytes, tmA, &full_a[sa], 0, m0, kbase + ia * (int)GA);
        ++ia;
        if (++sa == (int)RA) {
          sa = 0;
          pha ^= 1u;
        }
      } else {
        mbar_wait(&empty_w[sw], phw);
        mbar_expect_tx_w(&full_w[sw], GW * kBBytes);
        tma_load_3d_w(sB + sw * GW * kBBytes, &a.tmB, &full_w[sw], 0, n0, kbase + iw * (int)GW);
        ++iw;
        if (++sw == (int)RW) {
          sw = 0;
          phw ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: the whole warp runs the loop, elect.sync issues (k-block by k-block, 4
    // UMMA_K steps each, waiting for the A and W groups as they land; a group's slot is released
    // with a commit when it will be refilled)
    constexpr uint32_t idesc = umma_idesc(kBM, BN);
    if constexpr (ATT) {
      constexpr uint32_t idesc_s = umma_idesc(kBM, 128);                  // S = Q K^T: N = 128 keys
      constexpr uint32_t idesc_o = umma_idesc(kBM, 64) | (1u << 16);      // O = P V: N = 64 dims, B MN-major
      for (int i = 0; i < kps; ++i) {   // every head's S as soon as its tiles land
        const uint32_t bQ = smem_u32(sQKV + i * kAttQkvBytes), bK = bQ + kABytes;
        mbar_wait(&qkv_full[i], 0);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          umma_bf16_w(tmem + kAttTmemS + 128u * i, umma_desc_sw128(bQ) + 2 * k, umma_desc_sw128(bK) + 2 * k, idesc_s,
                      k != 0);
        umma_commit_w(&s_full[i]);
      }
      for (int i = 0; i < kps; ++i) {   // then O = P V per head, as the P tiles are written
        const uint32_t bP = smem_u32(sQKV + i * kAttQkvBytes), bV = bP + 2 * kABytes;
        mbar_wait(p_full, (uint32_t)i & 1u);
        tc_fence_after();
#pragma unroll
        for (int j = 0; j < 8; ++j)   // 16 keys per step: P k-block j / 4 (+32 B per step), V atoms 2 j, 2 j + 1
          umma_bf16_w(tmem + kAttTmemO, umma_desc_sw128(bP + (j >> 2) * kABytes) + 2 * (j & 3),
                      umma_desc_sw128_mn(bV + 2048u * j), idesc_o, j != 0);
        umma_commit_w(o_full);
      }
    }
    int sa = 0, sw = 0, oa = 0, ow = 0, ia = 0, iw = 0;
    uint32_t pha = 0u, phw = 0u;
    for (int kb = 0; kb < kps; ++kb) {
      if (oa == 0) mbar_wait(&full_a[sa], pha);
      if (ow == 0) mbar_wait(&full_w[sw], phw);
      if (kb == 0 && lane == 0) trace_at(a, 2);
      tc_fence_after();
      const uint64_t da = umma_desc_sw128(smem_u32(sA + (sa * GA + oa) * kABytes));
      const uint64_t db = umma_desc_sw128(smem_u32(sB + (sw * GW + ow) * kBBytes));
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k)   // UMMA_K = 16 bf16 = 32 B -> +2 in the >>4 address field
        umma_bf16_w(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
      const bool last = kb + 1 == kps;
      if (++oa == (int)GA || last) {
        if (ia + (int)RA < nga) umma_commit_w(&empty_a[sa]);
        oa = 0;
        ++ia;
        if (++sa == (int)RA) {
          sa = 0;
          pha ^= 1u;
        }
      }
      if (++ow == (int)GW || last) {
        if (iw + (int)RW < ngw) umma_commit_w(&empty_w[sw]);
        ow = 0;
        ++iw;
        if (++sw == (int)RW) {
          sw = 0;
          phw ^= 1u;
        }
      }
    }
    if (lane == 0) trace_at(a, 15);
    umma_commit_w(tmem_full);
    if (lane == 0) trace_at(a, 3);
  } else {
    // ---- epilogue warps (128 threads): TMEM -> registers -> [split-K push/reduce] -> epilogue.
    // Everything the epilogue reads from global memory is fetched BEFORE the accumulator is ready:
    // the bias slice (STATIC) into shared memory pre-wait, the residual (written by an earlier
    // node) into registers right after this thread's own griddepcontrol.wait. The TMEM row is
    // read with all tcgen05.ld in flight behind one wait. (Serial per-chunk global loads after
    // the MMA cost ~0.5 us each, measured with the phase tracer.)
    const uint32_t q = warp & 3;                  // TMEM lane quarter this warp may access
    const uint32_t row = q * 32 + lane;
    const uint32_t et = threadIdx.x - 64;          // epilogue thread 0..127
    const bool has_bias = a.flags & CGX_GEMM_BIAS, has_res = a.flags & CGX_GEMM_RESIDUAL;
    const bool gelu = a.flags & CGX_GEMM_GELU;
    if (has_bias && (a.flags & kGemmWAfterWait)) pdl_wait();
    for (uint32_t i = et; i < (uint32_t)BN; i += 128u)
      sbias[i] = has_bias ? __bfloat162float(a.bias[n0 + i]) : 0.f;
    if (ln_a)   // the fold's column terms (prepared at exec creation: STATIC, before the wait)
      for (uint32_t i = et; i < (uint32_t)BN; i += 128u) s_cc[i] = make_float2(a.ln_c1[n0 + i], a.ln_c2[n0 + i]);
    const uint32_t cta_lin = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    uint32_t& s_ar_g = s_tmem[1];                  // dynamic smem word after the TMEM address
    if (ar && et == 0) {
      const uint32_t g = a.ar_counters[a.ar_index * kArMaxCtas + cta_lin] + 1;
      a.ar_counters[a.ar_index * kArMaxCtas + cta_lin] = g;
      s_ar_g = g;
    }
    constexpr uint32_t kQRow = BN / 4;             // 4-column quads per tile row
    constexpr int kQMax = BN / 8;                  // quads per thread in the split reduction (rows_max <= 64)
    uint4 res_row[BN / 8];                         // S == 1: this thread's residual row (bf16 x 8 per uint4)
    uint2 res_q[kQMax];                            // S > 1: the residual quads this thread outputs
    if (has_res) {
      pdl_wait();
      // an EXTERNAL residual under INDIRECT comes from the pointer table (published before the
      // graph's first consumer; read after this thread's wait)
      const __nv_bfloat16* resp = a.tres >= 0 ? reinterpret_cast<const __nv_bfloat16*>(ld_table(a.table + a.tres))
                                              : a.residual;
      if (S == 1) {
        const int m = m0 + (int)row;
        if (m < (int)a.M) {
          const uint4* rp = reinterpret_cast<const uint4*>(resp + (size_t)m * a.N + n0);
#pragma unroll
          for (int i = 0; i < BN / 8; ++i) res_row[i] = rp[i];
        }
      } else {
#pragma unroll
        for (int j = 0; j < kQMax; ++j) {
          const uint32_t qi = et + 128u * j;
          if (qi < my_rows * kQRow) {
            const int mr = m0 + (int)(my_lo + qi / kQRow);
            if (mr < (int)a.M)
              res_q[j] = *reinterpret_cast<const uint2*>(resp + (size_t)mr * a.N + n0 + 4 * (qi % kQRow));
          }
        }
      }
    }
    asm volatile("bar.sync 1, 128;\n" ::: "memory");   // bias slice (and LN gamma / beta) staged
    if constexpr (ATT) {   // A = this split's heads of the causal attention, computed here (row = thread)
      const uint32_t T = a.M, r = row;                          // query row = TMEM lane
      const uint32_t trow = tmem + ((q * 32u) << 16);
      const uint32_t kvis = min(r + 1u, T);                     // keys [0, kvis) visible to this row
      const float sl2 = a.attn_scale * 1.4426950408889634f;   // softmax in base 2: p = 2^(s sl2 - max s sl2)
      const uint32_t bA = smem_u32(sA);
      // key groups of 32 this warp's rows can see (warp-uniform: the TMEM loads are warp-collective)
      const uint32_t ngrp = (min(32u * q + 32u, T) + 31u) / 32u;
      for (int i = 0; i < kps; ++i) {
        const uint32_t bP = smem_u32(sQKV + i * kAttQkvBytes), tS = trow + kAttTmemS + 128u * i;
        mbar_wait(&s_full[i], 0);
        tc_fence_after();
        if (threadIdx.x == 64 && i == 0) trace_at(a, 12);     // (phase tracer: S ready)
        float v[32];
        float mx = -INFINITY;
        for (uint32_t gi = 0; gi < ngrp; ++gi) {               // pass 1: row max over the visible keys
          tmem_ld16_nw(tS + 32u * gi, v);
          tmem_ld16_nw(tS + 32u * gi + 16u, v + 16);
          tmem_wait_regs<32>(v);
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (32u * gi + (uint32_t)c < kvis) mx = fmaxf(mx, v[c]);
        }
        const float mxl = mx * sl2;
        float l = 0.f;
        for (uint32_t gi = 0; gi < 4; ++gi) {                  // pass 2: p, l, bf16(p) -> P tile
          if (gi < ngrp) {
            tmem_ld16_nw(tS + 32u * gi, v);
            tmem_ld16_nw(tS + 32u * gi + 16u, v + 16);
            tmem_wait_regs<32>(v);
          }
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            uint32_t w4[4] = {0u, 0u, 0u, 0u};
            if (gi < ngrp) {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const uint32_t k0 = 32u * gi + 8u * c8 + 2u * e;
                float p0 = 0.f, p1 = 0.f;
                if (k0 < kvis) asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(fmaf(v[8 * c8 + 2 * e], sl2, -mxl)));
                if (k0 + 1u < kvis) asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(fmaf(v[8 * c8 + 2 * e + 1], sl2, -mxl)));
                l += p0 + p1;
                w4[e] = pack_bf16(p0, p1);
              }
            }
            const uint32_t key8 = 32u * gi + 8u * c8;          // 8 keys = one 16-B chunk of k-block key8 / 64
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(bP + (key8 >> 6) * kABytes +
                                                                         sw128_off(r, (key8 & 63u) >> 3)),
                         "r"(w4[0]), "r"(w4[1]), "r"(w4[2]), "r"(w4[3]) : "memory");
          }
        }
        fence_proxy_async_smem();   // generic-proxy stores -> visible to the tensor core
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        mbar_wait(o_full, (uint32_t)i & 1u);
        tc_fence_after();
        float vo[64];
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) tmem_ld16_nw(trow + kAttTmemO + (uint32_t)c0, vo + c0);
        tmem_wait_regs<64>(vo);
        const float inv = 1.0f / l;
        const uint32_t hd = (uint32_t)(kbase + i);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          uint4 o;
          o.x = pack_bf16(vo[8 * c8 + 0] * inv, vo[8 * c8 + 1] * inv);
          o.y = pack_bf16(vo[8 * c8 + 2] * inv, vo[8 * c8 + 3] * inv);
          o.z = pack_bf16(vo[8 * c8 + 4] * inv, vo[8 * c8 + 5] * inv);
          o.w = pack_bf16(vo[8 * c8 + 6] * inv, vo[8 * c8 + 7] * inv);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(bA + (uint32_t)i * kABytes + sw128_off(r, c8)),
                       "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w) : "memory");
          if (blockIdx.x == 0 && r < T)   // N tile 0 materialises the ATTN node's output
            *reinterpret_cast<uint4*>(a.attn_out + (size_t)r * a.K + hd * 64u + 8u * c8) = o;
        }
        tc_fence_before();
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_a[0]);
      if (lane == 0) trace_at(a, 13 + (warp == 2u ? 0 : 1));   // (13: warp 2's rows done; 14: the others')
    }
    if (ln_a) {
      // ---- folded LayerNorm (kGemmLnA): this thread's tile row statistics from the producer's
      // per-tile row sums (fixed tile order) into shared memory, then — while the MMAs run — this
      // CTA's share of the LN output slot a = (h - mean) * rstd * gamma + beta (16-B chunks of the
      // [M, K] matrix dealt round-robin over all CTAs of the grid), one bf16 rounding.
      pdl_wait();
      {
        const int m = m0 + (int)row;
        float mean = 0.f, rstd = 0.f;
        if (m < (int)a.M) {
          float s1 = 0.f, s2 = 0.f;                // the tiles' sums in fixed tile order
          uint32_t t = 0;
          if (!(a.ln_dbg & 1u)) {
            for (; t + 8 <= a.ln_ntiles; t += 8) {   // 8 loads in flight, summed in order
              float2 v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) v[u] = __ldcg(a.ln_stats + (size_t)(t + u) * a.M + m);
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                s1 += v[u].x;
                s2 += v[u].y;
              }
            }
          }
          for (; t < a.ln_ntiles; ++t) {
            const float2 v = __ldcg(a.ln_stats + (size_t)t * a.M + m);
            s1 += v.x;
            s2 += v.y;
          }
          mean = s1 / (float)a.K;
          const float var = fmaxf(s2 / (float)a.K - mean * mean, 0.f);
          rstd = 1.0f / sqrtf(var + a.ln_eps);
        }
        s_mr[row] = make_float2(mean, rstd);
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      const uint32_t nctas = gridDim.x * gridDim.y * gridDim.z;
      const uint32_t kc = a.K / 8;                       // 16-B chunks per row
      const uint64_t chunks = (uint64_t)a.M * kc;
      for (uint64_t i = (uint64_t)cta_lin * 128u + et; (a.ln_dbg & 2u) == 0 && i < chunks; i += (uint64_t)nctas * 128u) {
        const uint32_t mm = (uint32_t)(i / kc), k8 = (uint32_t)(i % kc) * 8;
        // the row's statistics: from shared memory when the row is in this CTA's M tile, else
        // recomputed from the sums (only when T > 128 spreads rows over several M tiles)
        float2 mr;
        if ((int)mm >= m0 && (int)mm < m0 + (int)kBM) {
          mr = s_mr[mm - m0];
        } else {
          float s1 = 0.f, s2 = 0.f;
          for (uint32_t t = 0; t < a.ln_ntiles; ++t) {
            const float2 v = __ldcg(a.ln_stats + (size_t)t * a.M + mm);
            s1 += v.x;
            s2 += v.y;
          }
          const float mean = s1 / (float)a.K;
          mr = make_float2(mean, 1.0f / sqrtf(fmaxf(s2 / (float)a.K - mean * mean, 0.f) + a.ln_eps));
        }
        const uint4 hx = *reinterpret_cast<const uint4*>(a.ln_h + (size_t)mm * a.K + k8);
        const uint4 gx = __ldg(reinterpret_cast<const uint4*>(a.ln_g + k8));
        const uint4 bx = __ldg(reinterpret_cast<const uint4*>(a.ln_b + k8));
        const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&hx);
        const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&gx);
        const __nv_bfloat16* bb = reinterpret_cast<const __nv_bfloat16*>(&bx);
        uint4 y;
        __nv_bfloat16* yb = reinterpret_cast<__nv_bfloat16*>(&y);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          yb[e] = __float2bfloat16_rn((__bfloat162float(hb[e]) - mr.x) * mr.y * __bfloat162float(gb[e]) +
                                      __bfloat162float(bb[e]));
        *reinterpret_cast<uint4*>(a.ln_out + (size_t)mm * a.K + k8) = y;
      }
    }
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    if (threadIdx.x == 64) trace_at(a, 8);
    float v[BN];
#pragma unroll
    for (int c0 = 0; c0 < BN; c0 += 16) tmem_ld16_nw(tmem + ((q * 32u) << 16) + (uint32_t)c0, v + c0);
    tmem_wait_regs<BN>(v);
    if (threadIdx.x == 64) trace_at(a, 9);
    if (S == 1) {
      // bias / GELU / residual in registers, 16-B stores straight from registers (measured faster
      // than staging the tile and bulk-storing rows: the bulk store's read-completion wait is ~1 us)
      const int m = m0 + (int)row;
      if (m < (int)a.M) {
        uint4* op = reinterpret_cast<uint4*>(a.out + (size_t)m * a.N + n0);
        if (ln_a) {   // folded LayerNorm: rstd * acc - rstd * mean * c1 + c2
          const float2 mr = s_mr[row];
#pragma unroll
          for (int i = 0; i < BN; ++i) v[i] = mr.y * v[i] - mr.y * mr.x * s_cc[i].x + s_cc[i].y;
        }
#pragma unroll
        for (int c8 = 0; c8 < BN / 8; ++c8) {
          const float4 b0 = *reinterpret_cast<const float4*>(sbias + 8 * c8);
          const float4 b1 = *reinterpret_cast<const float4*>(sbias + 8 * c8 + 4);
          const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i) v[8 * c8 + i] += bb[i];
        }
        if (gelu) {
#pragma unroll
          for (int i = 0; i < BN; ++i) v[i] = gelu_tanh(v[i]);
        }
        if (has_res) {
#pragma unroll
          for (int c8 = 0; c8 < BN / 8; ++c8) {
            const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&res_row[c8]);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[8 * c8 + i] += __bfloat162float(rb[i]);
          }
        }
        float q1 = 0.f, q2 = 0.f;                  // kGemmStatsOut: row sums of the rounded output
#pragma unroll
        for (int c8 = 0; c8 < BN / 8; ++c8) {
          uint4 o;
          __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            ob[i] = __float2bfloat16_rn(v[8 * c8 + i]);
            const float y = __bfloat162float(ob[i]);
            q1 += y;
            q2 += y * y;
          }
          if (!ar) {
            op[c8] = o;
          } else {                                 // this rank's bf16 tile row -> slot `rank` everywhere
            const uint32_t par = (s_ar_g - 1u) & 1u;
            for (uint32_t p = 0; p < a.ar_world; ++p)
              reinterpret_cast<uint4*>(ar_slot_ptr(a, p, par, a.ar_rank) + (size_t)m * a.N + n0)[c8] = o;
          }
        }
        if (a.flags & kGemmStatsOut) a.stats_out[(size_t)blockIdx.x * a.M + m] = make_float2(q1, q2);
      }
      if (ar) {
        const uint32_t g = s_ar_g;
        const uint32_t par = (g - 1u) & 1u;
        ar_publish_wait(a, cta_lin, g, et);
        if (m < (int)a.M) {                       // fixed rank order, fp32, one rounding
          uint4* op = reinterpret_cast<uint4*>(a.out + (size_t)m * a.N + n0);
#pragma unroll
          for (int c8 = 0; c8 < BN / 8; ++c8) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (uint32_t s2 = 0; s2 < a.ar_world; ++s2) {
              const uint4 x = reinterpret_cast<const uint4*>(ar_slot_ptr(a, a.ar_rank, par, s2) + (size_t)m * a.N + n0)[c8];
              const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&x);
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[i] += __bfloat162float(xb[i]);
            }
            uint4 o;
            __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
            for (int i = 0; i < 8; ++i) ob[i] = __float2bfloat16_rn(acc[i]);
            op[c8] = o;
          }
        }
      }
      if (threadIdx.x == 64) trace_at(a, 4);
    } else {
      // stage this row of the partial tile locally, then one thread per peer owner pushes that
      // owner's row block to its receive slot z with a single bulk DSMEM copy (complete_tx on
      // the owner's receive barrier). Own rows are reduced straight from the staging tile.
      float* stg = reinterpret_cast<float*>(smem);
      {
        float4* d4 = reinterpret_cast<float4*>(stg + row * kRowF);
#pragma unroll
        for (int i = 0; i < BN / 4; ++i) d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
      fence_proxy_async_smem();
      if (threadIdx.x == 64) trace_at(a, 10);
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");   // peers' receive barriers are armed
      asm volatile("bar.sync 1, 128;\n" ::: "memory");                         // staging tile complete
      if (et < S && et != z) {
        const uint32_t o = et, lo = split_row_lo(o, S), n = split_row_lo(o + 1, S) - lo;
        bulk_s2dsmem(mapa(smem_u32(recv + (size_t)z * rows_max * kRowF), o), smem_u32(stg + lo * kRowF),
                     n * kRowF * 4u, mapa(smem_u32(recv_full), o));
      }
      if (threadIdx.x == 64) trace_at(a, 5);
      mbar_wait(recv_full, 0);                            // every peer's rows have landed
      // our incoming copies are complete (so the peers' staging reads are done): let them exit
      // (no data of ours is published by this arrive: relaxed)
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
      if (threadIdx.x == 64) trace_at(a, 6);
      const uint32_t nq = my_rows * kQRow;
      if (!ar) {
        // The owner's quads (up to kQMax per thread) in stages over all of them, every flag test
        // hoisted out of the per-quad work: the four quads' dependency chains interleave. (One quad
        // at a time, with the flag branches inside, ran ~570 cycles per quad at one warp per
        // scheduler: serial short-latency waits and branch resolution, profiles/r02/gemm_epilogue.txt.)
        float4 acc[kQMax];
        uint32_t qr[kQMax], qc[kQMax];
        bool qv[kQMax];
#pragma unroll
        for (int j = 0; j < kQMax; ++j) {
          const uint32_t qi = et + 128u * j;
          qv[j] = qi < nq;
          qr[j] = qi / kQRow;
          qc[j] = 4u * (qi % kQRow);
          const float* src = recv + (size_t)qr[j] * kRowF + qc[j];
          const float* own = stg + (size_t)(my_lo + qr[j]) * kRowF + qc[j];
          acc[j] = qv[j] ? *reinterpret_cast<const float4*>(z == 0 ? own : src) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (uint32_t zz = 1; zz < S; ++zz) {          // fixed split order: deterministic sums
#pragma unroll
          for (int j = 0; j < kQMax; ++j) {
            if (!qv[j]) continue;
            const float* src = recv + (size_t)qr[j] * kRowF + qc[j];
            const float* own = stg + (size_t)(my_lo + qr[j]) * kRowF + qc[j];
            const float4 t = *reinterpret_cast<const float4*>(zz == z ? own : src + (size_t)zz * rows_max * kRowF);
            acc[j].x += t.x;
            acc[j].y += t.y;
            acc[j].z += t.z;
            acc[j].w += t.w;
          }
        }
        float w[kQMax][4];
        if (ln_a) {   // folded LayerNorm: rstd * acc - rstd * mean * c1 + c2 (after the split sum)
#pragma unroll
          for (int j = 0; j < kQMax; ++j) {
            const float2 m2 = qv[j] ? s_mr[my_lo + qr[j]] : make_float2(0.f, 0.f);   // (rows of s_mr only)
            const uint32_t c = qc[j];
            acc[j].x = m2.y * acc[j].x - m2.y * m2.x * s_cc[c].x + s_cc[c].y;
            acc[j].y = m2.y * acc[j].y - m2.y * m2.x * s_cc[c + 1].x + s_cc[c + 1].y;
            acc[j].z = m2.y * acc[j].z - m2.y * m2.x * s_cc[c + 2].x + s_cc[c + 2].y;
            acc[j].w = m2.y * acc[j].w - m2.y * m2.x * s_cc[c + 3].x + s_cc[c + 3].y;
          }
        }
#pragma unroll
        for (int j = 0; j < kQMax; ++j) {
          const float4 b4 = *reinterpret_cast<const float4*>(sbias + qc[j]);
          w[j][0] = acc[j].x + b4.x;
          w[j][1] = acc[j].y + b4.y;
          w[j][2] = acc[j].z + b4.z;
          w[j][3] = acc[j].w + b4.w;
        }
        if (gelu) {
#pragma unroll
          for (int j = 0; j < kQMax; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) w[j][i] = gelu_tanh(w[j][i]);
        }
        if (has_res) {
#pragma unroll
          for (int j = 0; j < kQMax; ++j) {
            const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&res_q[j]);
#pragma unroll
            for (int i = 0; i < 4; ++i) w[j][i] += __bfloat162float(rb[i]);
          }
        }
        uint2 ov[kQMax];
#pragma unroll
        for (int j = 0; j < kQMax; ++j) {
          __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&ov[j]);
#pragma unroll
          for (int i = 0; i < 4; ++i) ob[i] = __float2bfloat16_rn(w[j][i]);
        }
        if (a.flags & kGemmStatsOut) {
          // row sums of the ROUNDED output for a fused LN consumer: the kQRow threads holding a
          // row's quads are consecutive lanes (every lane of the warp takes part: the planner keeps
          // my_rows * kQRow a multiple of 32), reduced by a fixed shuffle tree
#pragma unroll
          for (int j = 0; j < kQMax; ++j) {
            if (128u * j >= nq) break;                 // (warp-uniform: nq % 32 == 0)
            const int mr = m0 + (int)(my_lo + qr[j]);
            const bool valid = qv[j] && mr < (int)a.M;
            float q1 = 0.f, q2 = 0.f;
            if (valid) {
              const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(&ov[j]);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float y = __bfloat162float(ob[i]);
                q1 += y;
                q2 += y * y;
              }
            }
#pragma unroll
            for (uint32_t o = kQRow / 2; o > 0; o >>= 1) {
              q1 += __shfl_xor_sync(0xffffffffu, q1, o);
              q2 += __shfl_xor_sync(0xffffffffu, q2, o);
            }
            if (valid && (et + 128u * j) % kQRow == 0) a.stats_out[(size_t)blockIdx.x * a.M + mr] = make_float2(q1, q2);
          }
        }
#pragma unroll
        for (int j = 0; j < kQMax; ++j) {
          const int mr = m0 + (int)(my_lo + qr[j]);
          if (qv[j] && mr < (int)a.M) *reinterpret_cast<uint2*>(a.out + (size_t)mr * a.N + n0 + qc[j]) = ov[j];
        }
      } else {
#pragma unroll
      for (int j = 0; j < kQMax; ++j) {
        const uint32_t qi = et + 128u * j;
        if (qi >= nq) break;
        const uint32_t r = qi / kQRow, c = 4u * (qi % kQRow);
        const int mr = m0 + (int)(my_lo + r);
        const float* src = recv + (size_t)r * kRowF + c;
        const float* own = stg + (size_t)(my_lo + r) * kRowF + c;
        float4 acc = *reinterpret_cast<const float4*>(z == 0 ? own : src);
        for (uint32_t zz = 1; zz < S; ++zz) {        // fixed split order: deterministic sums
          const float4 t = *reinterpret_cast<const float4*>(zz == z ? own : src + (size_t)zz * rows_max * kRowF);
          acc.x += t.x;
          acc.y += t.y;
          acc.z += t.z;
          acc.w += t.w;
        }
        if (mr >= (int)a.M) continue;
        float w[4] = {acc.x + sbias[c], acc.y + sbias[c + 1], acc.z + sbias[c + 2], acc.w + sbias[c + 3]};
        if (gelu) {
#pragma unroll
          for (int i = 0; i < 4; ++i) w[i] = gelu_tanh(w[i]);
        }
        if (has_res) {
          const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&res_q[j]);
#pragma unroll
          for (int i = 0; i < 4; ++i) w[i] += __bfloat162float(rb[i]);
        }
        uint2 ov;
        __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&ov);
#pragma unroll
        for (int i = 0; i < 4; ++i) ob[i] = __float2bfloat16_rn(w[i]);
        // this rank's bf16 quad -> slot `rank` everywhere (the AR path: no folded LN, no stats)
        const uint32_t par = (s_ar_g - 1u) & 1u;
        for (uint32_t p = 0; p < a.ar_world; ++p)
          *reinterpret_cast<uint2*>(ar_slot_ptr(a, p, par, a.ar_rank) + (size_t)mr * a.N + n0 + c) = ov;
      }
      }
      if (ar) {
        const uint32_t g = s_ar_g;
        const uint32_t par = (g - 1u) & 1u;
        ar_publish_wait(a, cta_lin, g, et);
#pragma unroll
        for (int j = 0; j < kQMax; ++j) {          // fixed rank order, fp32, one rounding
          const uint32_t qi = et + 128u * j;
          if (qi >= nq) break;
          const uint32_t r = qi / kQRow, c = 4u * (qi % kQRow);
          const int mr = m0 + (int)(my_lo + r);
          if (mr >= (int)a.M) continue;
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          for (uint32_t s2 = 0; s2 < a.ar_world; ++s2) {
            const uint2 x = *reinterpret_cast<const uint2*>(ar_slot_ptr(a, a.ar_rank, par, s2) + (size_t)mr * a.N + n0 + c);
            const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&x);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] += __bfloat162float(xb[i]);
          }
          uint2 ov;
          __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&ov);
#pragma unroll
          for (int i = 0; i < 4; ++i) ob[i] = __float2bfloat16_rn(acc[i]);
          *reinterpret_cast<uint2*>(a.out + (size_t)mr * a.N + n0 + c) = ov;
        }
      }
      if (threadIdx.x == 64) trace_at(a, 4);
    }
  }
  if (S > 1) {
    // phase 0 (receive barriers armed) for the non-epilogue warps; phase 1: no CTA exits before
    // every peer has received the rows it copied out of this CTA's staging tile
    if (warp < 2) {
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    trace_at(a, 7);
    node_stamp(a.ntrace, 2);
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
  }
}

// ------------------------------------------------------------------ small-M path (decode, T <= 8)
// At M <= 4 (the C3 T = 1 decode variant) a 128-row UMMA tile wastes 127/128 of the tensor core and
// still pays the TMA/TMEM latency chain, while the node is a pure weight stream (N x K x 2 bytes).
// KS warps per output column, each holding a K slice of kGvKV 16-B vectors per lane: the warps
// stream their W slices (STATIC) into registers BEFORE griddepcontrol.wait — the whole weight matrix
// is in flight while the predecessor drains — then load the M activation rows (L2), form M partial
// dot products in fp32 (fixed lane order + fixed shuffle tree), and the slice-0 warp sums the KS
// partials in slice order (deterministic) and applies bias / GELU / residual, rounding once.
// The K split keeps every variant at 3 vectors per lane (80 registers, 3 CTAs of 256 threads per
// SM), so the next node's CTAs fit beside this one's and start their own weight stream early: one
// warp holding a whole K = 3072 row (207-224 registers) blocked that (profiles/r02/decode_gemv_ks.txt).
static constexpr int kGvWarps = 8;
static constexpr int kGvMaxM = 4;    // decode replays measured faster than tcgen05 up to T = 4, not at 8
static constexpr int kGvKV = 3;      // 16-B vectors per lane per K slice: a slice covers 768 columns
static constexpr int kGvMaxKS = 8;   // slices per column: K <= 8 * 768 = 6144

__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// kGemmAttnA (M = 1): this lane's kGvKV 16-B vectors of the attention output row. With T = 1 the
// causal softmax has one visible key, so p_0 = __expf(s_0 - s_0) = 1, l = 1 and the output row is
// bf16(1 * v_0 * (1 / 1)) = v_0 exactly — what the attention kernel (cgx_attn.cuh) computes for a
// one-key tile, bit for bit — and the q / k segments of the qkv row do not enter it.
__device__ __forceinline__ void gv_attn_row(const GemmArgs& a, uint32_t v0, uint32_t lane, uint32_t kv,
                                            uint4 (&x)[kGvKV]) {
  const uint4* vrow = reinterpret_cast<const uint4*>(a.attn_qkv) + 2 * kv;   // v segment of qkv row 0
#pragma unroll
  for (int i = 0; i < kGvKV; ++i) {
    const uint32_t v = v0 + lane + 32u * i;
    if (v < kv) x[i] = vrow[v];
  }
}

template <int KS, int MT, int R>
__global__ void __launch_bounds__(kGvWarps * 32, MT == 1 ? (R == 1 ? 4 : 3) : 3) k_gemv_bf16(const __grid_constant__ GemmArgs a) {
  static_assert(kGvWarps % KS == 0, "slices of a column stay in one CTA");
  const bool late_trigger = a.flags & kGemmTriggerAfterWait;
  if (threadIdx.x == 0) node_stamp(a.ntrace, 0);
  if (!late_trigger) pdl_trigger();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t slice = warp % KS;                                    // this warp's K slice
  const uint32_t n0 = (blockIdx.x * (kGvWarps / KS) + warp / KS) * R;  // this warp's R output columns
  const uint32_t M = MT == 1 ? 1u : a.M;                               // activation rows
  const uint32_t kv = a.K / 8;                                         // 16-B vectors per row
  const uint32_t v0 = slice * (kGvKV * 32u);                           // the slice's first vector
  // ---- W rows n0 .. n0 + R - 1, this slice (STATIC): all loads in flight before the wait
  const bool w_late = a.flags & kGemmWAfterWait;
  if (w_late) pdl_wait();
  uint4 w[R][kGvKV];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int i = 0; i < kGvKV; ++i) {
      const uint32_t v = v0 + lane + 32u * i;
      if (n0 + r < a.N && v < kv) w[r][i] = *(reinterpret_cast<const uint4*>(a.w_ptr + (size_t)(n0 + r) * a.K) + v);
    }
  // epilogue operands no node of the graph writes (bias unless kGemmWAfterWait, the folded-LN
  // column sums c1 / c2) and the gamma / beta of the materialised LN row: fetched before the wait
  // too, so the epilogue after the dot products issues no dependent load but the residual's
  const bool has_bias = a.flags & CGX_GEMM_BIAS, gelu = a.flags & CGX_GEMM_GELU;
  const bool has_res = a.flags & CGX_GEMM_RESIDUAL;
  const bool ln_a = a.flags & kGemmLnA;
  const bool owner = slice == 0 && lane == 0;                          // applies the columns' epilogue
  float e_b[R], e_c1[R], e_c2[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    e_b[r] = e_c1[r] = e_c2[r] = 0.f;
    if (owner && n0 + r < a.N) {
      if (has_bias && !w_late) e_b[r] = __bfloat162float(a.bias[n0 + r]);
      if (ln_a) {
        e_c1[r] = a.ln_c1[n0 + r];
        e_c2[r] = a.ln_c2[n0 + r];
      }
    }
  }
  // (gamma / beta staged in shared memory by the storing warps — the first column's KS warps of
  // CTA 0 — registers would cost occupancy; each lane reads back only what it stored itself)
  __shared__ uint4 s_gb[2][KS][kGvKV * 32];
  __shared__ float s_part[kGvWarps][R][MT];                            // KS > 1: per-slice partials
  __shared__ float s_st[kGvWarps];                                     // KS > 1: per-slice LN sums
  const bool ln_mat = ln_a && blockIdx.x == 0 && warp < (uint32_t)KS;
  if (ln_mat)
#pragma unroll
    for (int i = 0; i < kGvKV; ++i) {
      const uint32_t v = v0 + lane + 32u * i;
      if (v < kv) {
        s_gb[0][slice][lane + 32u * i] = __ldg(reinterpret_cast<const uint4*>(a.ln_g) + v);
        s_gb[1][slice][lane + 32u * i] = __ldg(reinterpret_cast<const uint4*>(a.ln_b) + v);
      }
    }
  if (!w_late) pdl_wait();
  if (late_trigger) pdl_trigger();
  if (threadIdx.x == 0) node_stamp(a.ntrace, 1);
  if (has_bias && w_late && owner)
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (n0 + r < a.N) e_b[r] = __bfloat162float(a.bias[n0 + r]);
  // A: the patched / direct a_ptr, or table[ta] for an EXTERNAL A under INDIRECT (after the wait)
  const __nv_bfloat16* ap = a.ta >= 0 ? reinterpret_cast<const __nv_bfloat16*>(ld_table(a.table + a.ta)) : a.a_ptr;
  // the residual (written by an earlier node): in flight together with the A rows
  float e_res[R][MT];
  if (has_res && owner) {
    const __nv_bfloat16* resp = a.tres >= 0 ? reinterpret_cast<const __nv_bfloat16*>(ld_table(a.table + a.tres))
                                            : a.residual;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int m = 0; m < MT; ++m)
        e_res[r][m] = (m < (int)M && n0 + r < a.N) ? __bfloat162float(resp[(size_t)m * a.N + n0 + r]) : 0.f;
  }
  float acc[R][MT];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[r][m] = 0.f;
  // folded LayerNorm (kGemmLnA, A = the LN input h): the dot products run on the raw h (with W'), so
  // only the epilogue needs the row statistics; the first column group's KS warps (they hold whole
  // rows between them) compute them from their loads while the other warps go on — at KS = 1
  // (K <= 768) with the LN kernel's reduction (per-lane chunk order, then the xor tree), so mean /
  // rstd and the materialised a are bit-identical to the LN node; at KS > 1 the slices' sums are
  // added in slice order through shared memory. (Every warp computing them measured ~1.2 us per
  // GEMV of SM issue time at T = 1, profiles/r02/decode_gemv_ks.txt.)
  __shared__ float2 s_mr[MT];
  const bool ln_warp = ln_a && warp < (uint32_t)KS;
  const bool attn_a = a.flags & kGemmAttnA;
  const bool attn_mat = attn_a && blockIdx.x == 0 && warp < (uint32_t)KS;
  for (uint32_t m = 0; m < M; ++m) {
    uint4 x[kGvKV];
    if (MT == 1 && attn_a) {   // (M = 1 instantiations only: the M <= 4 ones keep their registers)
      gv_attn_row(a, v0, lane, kv, x);
      if (attn_mat)   // the ATTN node's output row, materialised once (each slice by its warp)
#pragma unroll
        for (int i = 0; i < kGvKV; ++i) {
          const uint32_t v = v0 + lane + 32u * i;
          if (v < kv) reinterpret_cast<uint4*>(a.attn_out + (size_t)m * a.K)[v] = x[i];
        }
    } else {
      const uint4* ar = reinterpret_cast<const uint4*>(ap + (size_t)m * a.K);
#pragma unroll
      for (int i = 0; i < kGvKV; ++i) {
        const uint32_t v = v0 + lane + 32u * i;
        if (v < kv) x[i] = ar[v];
      }
    }
    if (ln_warp) {
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < kGvKV; ++i)
        if (v0 + lane + 32u * i < kv) {
          const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&x[i]);
#pragma unroll
          for (int e = 0; e < 8; ++e) s += __bfloat162float(xb[e]);
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if constexpr (KS > 1) {
        if (lane == 0) s_st[warp] = s;
        asm volatile("bar.sync 1, %0;\n" ::"r"(KS * 32) : "memory");
        s = 0.f;
#pragma unroll
        for (int j = 0; j < KS; ++j) s += s_st[j];
        asm volatile("bar.sync 1, %0;\n" ::"r"(KS * 32) : "memory");
      }
      const float mean = s / (float)a.K;
      float q = 0.f;
#pragma unroll
      for (int i = 0; i < kGvKV; ++i)
        if (v0 + lane + 32u * i < kv) {
          const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&x[i]);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float d = __bfloat162float(xb[e]) - mean;
            q += d * d;
          }
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
      if constexpr (KS > 1) {
        if (lane == 0) s_st[warp] = q;
        asm volatile("bar.sync 1, %0;\n" ::"r"(KS * 32) : "memory");
        q = 0.f;
#pragma unroll
        for (int j = 0; j < KS; ++j) q += s_st[j];
        asm volatile("bar.sync 1, %0;\n" ::"r"(KS * 32) : "memory");
      }
      const float rstd = 1.0f / sqrtf(q / (float)a.K + a.ln_eps);
      if (warp == 0 && lane == 0) s_mr[m] = make_float2(mean, rstd);
      if (ln_mat)   // the LN node's output row, materialised once (each slice by its warp)
#pragma unroll
        for (int i = 0; i < kGvKV; ++i) {
          const uint32_t v = v0 + lane + 32u * i;
          if (v < kv) {
            const uint4 gx = s_gb[0][slice][lane + 32u * i], bx = s_gb[1][slice][lane + 32u * i];
            const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&x[i]);
            const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&gx);
            const __nv_bfloat16* bb = reinterpret_cast<const __nv_bfloat16*>(&bx);
            uint4 y;
            __nv_bfloat16* yb = reinterpret_cast<__nv_bfloat16*>(&y);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              yb[e] = __float2bfloat16_rn((__bfloat162float(xb[e]) - mean) * rstd * __bfloat162float(gb[e]) +
                                          __bfloat162float(bb[e]));
            reinterpret_cast<uint4*>(a.ln_out + (size_t)m * a.K)[v] = y;
          }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int i = 0; i < kGvKV; ++i) {
        if (v0 + lane + 32u * i < kv) {
          const uint32_t* xp = reinterpret_cast<const uint32_t*>(&x[i]);
          const uint32_t* wp = reinterpret_cast<const uint32_t*>(&w[r][i]);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            s0 = fmaf(bf16lo(xp[q]), bf16lo(wp[q]), s0);
            s1 = fmaf(bf16hi(xp[q]), bf16hi(wp[q]), s1);
          }
        }
      }
      float t = s0 + s1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
#pragma unroll
      for (int mm = 0; mm < MT; ++mm)
        if (mm == (int)m) acc[r][mm] = t;
    }
  }
  if constexpr (KS > 1) {   // the slices' partials (summed below in slice order by the slice-0 warp)
    if (lane == 0)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int m = 0; m < MT; ++m) s_part[warp][r][m] = acc[r][m];
  }
  if (KS > 1 || ln_a) __syncthreads();   // partials and row statistics in shared memory
  if constexpr (KS > 1) {
    if (owner)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          float t = s_part[warp][r][m];
#pragma unroll
          for (int j = 1; j < KS; ++j) t += s_part[warp + j][r][m];
          acc[r][m] = t;
        }
  }
  if (owner) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t n = n0 + r;
      if (n >= a.N) break;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (m >= (int)M) break;
        float v = acc[r][m];
        if (ln_a) v = s_mr[m].y * v - s_mr[m].y * s_mr[m].x * e_c1[r] + e_c2[r];   // folded LN
        v += e_b[r];
        if (gelu) v = gelu_tanh(v);
        if (has_res) v += e_res[r][m];
        a.out[(size_t)m * a.N + n] = __float2bfloat16_rn(v);
      }
    }
  }
  if (a.ntrace) {
    __syncthreads();
    if (threadIdx.x == 0) node_stamp(a.ntrace, 2);   // after every warp's stores
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

// K-major operand [rows, K] bf16 viewed as 3-D {64 (k in block), rows, K/64 (k-block)} with strides
// {K * 2 B, 128 B}: a box {64, box_rows, G} lands in shared memory as G stacked [box_rows][128 B]
// SW128 tiles (the swizzle phase repeats every 8 rows; box_rows % 8 == 0).
static int encode_kmajor(CUtensorMap* tm, const void* base, uint64_t rows, uint64_t K, uint32_t box_rows,
                         uint32_t group) {
  cuuint64_t dims[3] = {(cuuint64_t)kBK, rows, K / kBK};
  cuuint64_t strides[2] = {K * 2, (cuuint64_t)kBK * 2};
  cuuint32_t box[3] = {(cuuint32_t)kBK, box_rows, group};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? CGX_OK : CGX_E_CUDA;
}

// Tiling. Every CTA of an M = 128 GEMM streams its A panel slice through its SM, so per-SM operand
// ingress (k-blocks per CTA x (16 KiB of A + BN x 128 B of W)) and the serial latency chain (first
// TMA, MMA, epilogue) bound it; split-K cuts the ingress S-fold at the price of the push
// reduction. Rule measured on the deployed C3 replay (scripts/diag_c3_tiling.py,
// profiles/r01/c3_tiling.txt: 562 -> 514 us per 12-layer replay): BN = 32 (64 for M >= 1024 with
// K >= 512, profiles/r01/gemm_large.txt), and the largest
// S in {1, 2, 4, 8} with tiles x S <= 192 CTAs (up to two co-resident per SM) and >= 3 k-blocks
// per split. CGX_GEMM_TILING / CGX_GEMM_BN / CGX_GEMM_SPLIT pin a tiling for measurement.
static uint32_t split_rows_max_h(uint32_t S) { return (128u + S - 1) / S; }

static size_t recv_bytes(int bn, uint32_t S) { return S > 1 ? (size_t)S * split_rows_max_h(S) * (bn + 4) * 4 : 0; }
struct GemmPipes {
  uint32_t ga, ra, gw, rw;
};
static size_t smem_bytes(int bn, uint32_t S, const GemmPipes& p) {
  size_t ring = (size_t)p.ra * p.ga * kBM * kBK * 2 + (size_t)p.rw * p.gw * bn * kBK * 2;
  const size_t stage = S > 1 ? (size_t)128 * (bn + 4) * 4 : 0;
  if (stage > ring) ring = stage;
  // align + rings + split receive slots + bias slice + barriers + TMEM/AR words + dynamic tensor map
  return 1024 + ring + recv_bytes(bn, S) + bn * 4 + (2 * p.ra + 2 * p.rw + 2) * 8 + 16 + 256;
}
// Operand pipelines: A whole (one-shot, one box per k-block so the MMAs start with the first) when
// its K slice fits beside a W ring of >= 2 k-blocks, else an A ring of 4-k-block boxes; W per
// k-block through the rest of the budget (>= 2 slots). CGX_GEMM_PIPES="GA/RA/GW/RW" pins all shapes,
// CGX_GEMM_TILING="NxK=BN/S/GA/RA/GW/RW" one shape (measurement knobs).
static GemmPipes pick_pipes(int bn, uint32_t S, uint32_t nk) {
  // Lean rings (r02 sweeps, profiles/r02/gemm_pipes_sweep.txt): groups of 2 k-blocks, 2 groups of A
  // and 2 of W resident (80 KiB at BN = 32), so two GEMM CTAs fit on one SM and a node's CTAs can
  // become resident — and stream their weights before griddepcontrol.wait — while its predecessor
  // still runs. Holding the whole A slice (one-shot, ~200 KiB) made each GEMM ~1 us shorter alone
  // but cost as much in launch gaps in the deployed chain (FC1 -> FC2: 2.9-3.7 us), and the
  // per-CTA floor is the tcgen05 issue rate (~50-60 cycles per 128 x 32 x 16 MMA), not the loads.
  const uint32_t kps = (nk + S - 1) / S;
  GemmPipes p{1, 1, 1, 1};
  p.ga = p.gw = kps < 2 ? kps : 2;
  const uint32_t ng = (kps + p.ga - 1) / p.ga;
  p.ra = p.rw = ng < 2 ? ng : 2;
  (void)bn;
  return p;
}

static bool parse_pipes(const char* s, GemmPipes* p) {
  int ga = 0, ra = 0, gw = 0, rw = 0;
  if (sscanf(s, "%d/%d/%d/%d", &ga, &ra, &gw, &rw) != 4) return false;
  if (ga < 1 || ga > kMaxGroupKb || gw < 1 || gw > kMaxGroupKb || ra < 1 || rw < 1) return false;
  *p = GemmPipes{(uint32_t)ga, (uint32_t)ra, (uint32_t)gw, (uint32_t)rw};
  return true;
}
static void clamp_pipes(GemmPipes* p, uint32_t kps) {
  if (p->ga > kps) p->ga = kps;
  if (p->gw > kps) p->gw = kps;
  const uint32_t nga = (kps + p->ga - 1) / p->ga, ngw = (kps + p->gw - 1) / p->gw;
  if (p->ra > nga) p->ra = nga;
  if (p->rw > ngw) p->rw = ngw;
}

static void pick_tiling(uint32_t M, uint32_t N, uint32_t K, int* bn_out, uint32_t* split_out) {
  // CGX_GEMM_TILING="NxK=BN/S,..." pins a tiling per shape (measurement knob)
  if (const char* t = getenv("CGX_GEMM_TILING")) {
    char key[32];
    snprintf(key, sizeof key, "%ux%u=", N, K);
    if (const char* p = strstr(t, key)) {
      int bn = 0, sp = 0;
      if (sscanf(p + strlen(key), "%d/%d", &bn, &sp) == 2 && (bn == 32 || bn == 64 || bn == 128) && N % bn == 0 &&
          sp >= 1 && sp <= 16 && (uint32_t)sp <= K / kBK) {
        *bn_out = bn;
        *split_out = (uint32_t)sp;
        return;
      }
    }
  }
  const char* env_bn = getenv("CGX_GEMM_BN");          // measurement knobs
  const char* env_sp = getenv("CGX_GEMM_SPLIT");
  const uint32_t nk = K / kBK;
  // large, compute-bound shapes (many M tiles and a long K) take BN = 64: two CTAs per SM overlap one
  // tile's epilogue with the other's mainloop (gemm_large.txt: 753 vs 422 TFLOP/s at BN = 32)
  int bn = (M >= 1024 && K >= 512 && N % 64 == 0) ? 64 : 32;
  if (env_bn && (atoi(env_bn) == 32 || atoi(env_bn) == 64 || atoi(env_bn) == 128) && N % atoi(env_bn) == 0)
    bn = atoi(env_bn);
  const uint32_t tiles = (N / bn) * ((M + kBM - 1) / kBM);
  uint32_t sp = 1;
  if (env_sp && atoi(env_sp) >= 1 && (uint32_t)atoi(env_sp) <= nk && atoi(env_sp) <= 16) {
    sp = (uint32_t)atoi(env_sp);
  } else {
    // the largest S in {2, 3, 4, 8} with <= 192 CTAs and >= 4 k-blocks per split (O-proj 768 x 768:
    // S = 3 instead of 4, C3 327 -> 321.5 us; the other decoder shapes unchanged, every 32 / S
    // alternative slower: profiles/r02/sweep_c3_split*.txt)
    for (uint32_t c : {2u, 3u, 4u, 8u})
      if (tiles * c <= 192 && nk >= 4 * c) sp = c;
  }
  *bn_out = bn;
  *split_out = sp;
}

int decoder_encode_kmajor(void* tm, const void* base, uint64_t rows, uint64_t K, uint32_t box_rows, uint32_t group) {
  if (get_encode() != CGX_OK) return CGX_E_CUDA;
  return encode_kmajor(static_cast<CUtensorMap*>(tm), base, rows, K, box_rows, group);
}

int decoder_gemm_set_stats_out(void* args, void* stats, dim3 grid) {
  GemmArgs* g = static_cast<GemmArgs*>(args);
  if (g->flags & CGX_GEMM_ALLREDUCE) return CGX_E_UNSUPPORTED;
  const uint32_t S = grid.z, bn = g->N / grid.x, rows = split_rows_max_h(S);
  // every lane of an owner warp takes part in the row-sum shuffles: my_rows * BN / 4 % 32 == 0
  // (every thread of the 4 epilogue warps runs the row-sum shuffles, with zeros past its owner rows:
  // a row's bn / 4 quads sit in consecutive, aligned lanes whatever my_rows is)
  if (g->split != S || (S != 1 && (rows * (bn / 4) > 128u * (bn / 8)))) return CGX_E_UNSUPPORTED;
  g->stats_out = static_cast<float2*>(stats);
  g->flags |= kGemmStatsOut;
  return CGX_OK;
}

static bool gemv_shape(uint32_t M, uint32_t N, uint32_t K);
int decoder_gemm_set_ln_a(void* args, dim3 grid, const void* stats, uint32_t ntiles, const void* h, const void* w_fold,
                          const float* c1, const float* c2, const void* gamma, const void* beta, void* ln_out,
                          float eps, size_t* smem, const void** func) {
  GemmArgs* g = static_cast<GemmArgs*>(args);
  if (g->flags & CGX_GEMM_ALLREDUCE) return CGX_E_UNSUPPORTED;
  if (gemv_shape(g->M, g->N, g->K)) {   // small-M path: the statistics come from its own A loads
    g->w_ptr = static_cast<const __nv_bfloat16*>(w_fold);
    g->ln_h = static_cast<const __nv_bfloat16*>(h);
    g->ln_c1 = c1;
    g->ln_c2 = c2;
    g->ln_g = static_cast<const __nv_bfloat16*>(gamma);
    g->ln_b = static_cast<const __nv_bfloat16*>(beta);
    g->ln_out = static_cast<__nv_bfloat16*>(ln_out);
    g->ln_eps = eps;
    g->flags |= kGemmLnA;
    (void)stats, (void)ntiles, (void)grid, (void)smem, (void)func;
    return CGX_OK;
  }
  if (get_encode() != CGX_OK) return CGX_E_CUDA;
  const uint32_t bn = g->N / grid.x;
  if (ntiles > kLnMaxTiles) return CGX_E_UNSUPPORTED;
  const size_t extra = 128 + (size_t)kBM * 8 + (size_t)bn * 8;
  if (*smem + extra > kSmemLimit) return CGX_E_UNSUPPORTED;
  // the MMAs stream the gamma-scaled weights W'
  if (encode_kmajor(&g->tmB, w_fold, g->N, g->K, bn, g->gw) != CGX_OK) return CGX_E_CUDA;
  g->w_ptr = static_cast<const __nv_bfloat16*>(w_fold);
  *smem += extra;
  g->ln_stats = static_cast<const float2*>(stats);
  g->ln_ntiles = ntiles;
  g->ln_h = static_cast<const __nv_bfloat16*>(h);
  g->ln_c1 = c1;
  g->ln_c2 = c2;
  g->ln_g = static_cast<const __nv_bfloat16*>(gamma);
  g->ln_b = static_cast<const __nv_bfloat16*>(beta);
  g->ln_out = static_cast<__nv_bfloat16*>(ln_out);
  g->ln_eps = eps;
  g->ln_dbg = getenv("CGX_LN_DBG") ? (uint32_t)atoi(getenv("CGX_LN_DBG")) : 0u;
  g->flags |= kGemmLnA;
  (void)func;   // the same kernel (kGemmLnA is a runtime flag)
  return CGX_OK;
}

// Exec-creation prep of a folded LayerNorm (one CTA per output column n, fixed reduction order):
// W'[n, k] = bf16(gamma_k * W[n, k]), c1[n] = sum_k W'[n, k], c2[n] = sum_k beta_k * W[n, k]
// (fp64 accumulation, rounded once to fp32).
__global__ void k_ln_fold_prep(const __nv_bfloat16* W, const __nv_bfloat16* gamma, const __nv_bfloat16* beta,
                               uint32_t K, __nv_bfloat16* wf, float* c1, float* c2) {
  const uint32_t n = blockIdx.x;
  __shared__ double red[2][32];
  double s1 = 0.0, s2 = 0.0;
  for (uint32_t k = threadIdx.x; k < K; k += blockDim.x) {
    const float w = __bfloat162float(W[(size_t)n * K + k]);
    const __nv_bfloat16 wq = __float2bfloat16_rn(__bfloat162float(gamma[k]) * w);
    wf[(size_t)n * K + k] = wq;
    s1 += (double)__bfloat162float(wq);
    s2 += (double)__bfloat162float(beta[k]) * (double)w;
  }
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s1;
    red[1][threadIdx.x >> 5] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t1 = 0.0, t2 = 0.0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
      t1 += red[0][w];
      t2 += red[1][w];
    }
    c1[n] = (float)t1;
    c2[n] = (float)t2;
  }
}

int decoder_ln_fold_prep(const void* W, const void* gamma, const void* beta, uint32_t N, uint32_t K, void* wf,
                         float* c1, float* c2) {
  k_ln_fold_prep<<<N, 256>>>(static_cast<const __nv_bfloat16*>(W), static_cast<const __nv_bfloat16*>(gamma),
                             static_cast<const __nv_bfloat16*>(beta), K, static_cast<__nv_bfloat16*>(wf), c1, c2);
  const cudaError_t e = cudaDeviceSynchronize();
  return e == cudaSuccess ? CGX_OK : CGX_E_CUDA;
}

bool decoder_gemm_is_gemv(uint32_t M, uint32_t N, uint32_t K) { return gemv_shape(M, N, K); }

template <int BN, bool AR, bool ATT = false>
static const void* setup_kernel();

int decoder_gemm_set_attn_a(void* args, const void* qkv, void* attn_out, uint32_t H, uint32_t D, float scale,
                            dim3* grid, size_t* smem, const void** func) {
  GemmArgs* g = static_cast<GemmArgs*>(args);
  if ((g->flags & (CGX_GEMM_ALLREDUCE | kGemmLnA)) || g->ta >= 0) return CGX_E_UNSUPPORTED;
  if (D != 64 || H == 0 || g->K != H * D) return CGX_E_UNSUPPORTED;
  g->attn_qkv = static_cast<const __nv_bfloat16*>(qkv);
  g->attn_out = static_cast<__nv_bfloat16*>(attn_out);
  g->attn_scale = scale;   // (the GEMV path ignores it: one visible key, weight 1)
  g->attn_H = H;
  if (gemv_shape(g->M, g->N, g->K)) {
    if (g->M != 1) return CGX_E_UNSUPPORTED;   // (k_gemv_bf16<KS, 1, 1> only)
    g->flags |= kGemmAttnA;
    return CGX_OK;
  }
  // tcgen05 (ATT instantiation): one M tile (T <= 128), K split S = the largest divisor of H that is
  // <= 8 (HP = H / S heads = k-blocks per split, cluster (1, 1, S) portable: a cluster of 12 left
  // part of a 288-CTA grid in a second wave), BN = 32, A / W rings of one HP-k-block group
  // Measured slower than the two separate launches (C3: 339 -> 420 us with one CTA pair of heads per
  // split at 2 CTAs / SM, 486 us double-buffered at 1 CTA / SM: the 4 epilogue warps' softmax of a
  // 128 x 128 score tile per head is latency-bound at ~2.4-3.5 us a head, and every N tile repeats
  // it; profiles/r02/ab_attn_gemm.txt, gemm_att_trace.txt): built and tested, but only
  // with the measurement knob CGX_ATTN_GEMM_TC=1.
  const char* tc = getenv("CGX_ATTN_GEMM_TC");
  if (!(tc && tc[0] == '1')) return CGX_E_UNSUPPORTED;
  if (g->M > (uint32_t)kBM || g->N % 32) return CGX_E_UNSUPPORTED;
  uint32_t S = 1;
  for (uint32_t c = 1; c <= 8 && c <= H; ++c)
    if (H % c == 0) S = c;
  const uint32_t HP = H / S;
  if (HP > 2) return CGX_E_UNSUPPORTED;   // (one Q / K / V buffer and one TMEM S region per head)
  if (get_encode() != CGX_OK) return CGX_E_CUDA;
  const GemmPipes pp{HP, 1, HP, 1};
  const size_t sm = smem_bytes(32, S, pp) + (size_t)kBM * 8 + 32 * 8 + 6 * 8 + 1024 + (size_t)HP * kAttQkvBytes;
  if (sm > kSmemLimit) return CGX_E_UNSUPPORTED;
  if (encode_kmajor(&g->tmA, qkv, g->M, 3ull * g->K, kBM, 1) != CGX_OK) return CGX_E_CUDA;   // Q | K | V k-blocks
  if (encode_kmajor(&g->tmB, g->w_ptr, g->N, g->K, 32, HP) != CGX_OK) return CGX_E_CUDA;
  g->split = S;
  g->ga = g->gw = HP;
  g->ra = g->rw = 1;
  g->flags |= kGemmAttnA;
  *grid = dim3(g->N / 32, 1, S);
  *smem = sm;
  *func = setup_kernel<32, false, true>();
  return CGX_OK;
}

bool decoder_gemm_is_tcgen05(const void* func) {
  return func == (const void*)k_gemm_bf16<32, false> || func == (const void*)k_gemm_bf16<64, false> ||
         func == (const void*)k_gemm_bf16<128, false> || func == (const void*)k_gemm_bf16<32, false, true>;
}

void decoder_gemm_plan(uint32_t, uint32_t, uint32_t, size_t* ws_bytes, size_t* cnt_bytes) {
  // split-K partials are reduced through distributed shared memory: no global workspace
  *ws_bytes = 0;
  *cnt_bytes = 0;
}

template <int BN, bool AR, bool ATT>
static const void* setup_kernel() {
  // per call (exec build time, cheap): function attributes belong to the current device's context.
  // Headroom below the 227 KiB per-block limit for the kernel's static shared memory.
  static const int attr = [] {   // CGX_GEMM_SMEM_ATTR: measurement knob (bytes)
    const char* v = getenv("CGX_GEMM_SMEM_ATTR");
    return v ? atoi(v) : (int)kSmemLimit;
  }();
  cudaFuncSetAttribute(k_gemm_bf16<BN, AR, ATT>, cudaFuncAttributeMaxDynamicSharedMemorySize, attr);
  cudaFuncSetAttribute(k_gemm_bf16<BN, AR, ATT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return (const void*)k_gemm_bf16<BN, AR, ATT>;
}

// the fused all-reduce epilogue is a separate instantiation: the plain kernel keeps its code
static const void* kernel_for(int bn, bool ar = false) {
  if (ar) return bn == 128 ? setup_kernel<128, true>() : bn == 64 ? setup_kernel<64, true>() : setup_kernel<32, true>();
  return bn == 128 ? setup_kernel<128, false>() : bn == 64 ? setup_kernel<64, false>() : setup_kernel<32, false>();
}

void decoder_gemm_set_allreduce(void* args, uint32_t rank, uint32_t world, uint32_t ar_index, uint32_t n_ar,
                                uint64_t slot_elems, uint32_t* counters, void* const* recv, uint32_t* const* flags) {
  GemmArgs* g = static_cast<GemmArgs*>(args);
  g->ar_rank = rank;
  g->ar_world = world;
  g->ar_index = ar_index;
  g->ar_nar = n_ar;
  g->ar_slot = slot_elems;
  g->ar_counters = counters;
  for (uint32_t r = 0; r < world && r < (uint32_t)kArMaxWorld; ++r) {
    g->ar_recv[r] = static_cast<__nv_bfloat16*>(recv[r]);
    g->ar_flags[r] = flags[r];
  }
}

uint32_t decoder_gemm_ctas(const void* args, dim3 grid) {
  (void)args;
  return grid.x * grid.y * grid.z;
}

void decoder_gemm_set_a_dynamic(void* args, const uint64_t* table, int32_t idx, void* tm_ws, bool after_wait) {
  GemmArgs* g = static_cast<GemmArgs*>(args);
  g->flags |= kGemmADynamic | (after_wait ? kGemmADynAfterWait : 0u);
  if (table) g->table = table;
  g->ta = idx;
  g->tm_ws = static_cast<CUtensorMap*>(tm_ws);
  if (idx >= 0) g->a_ptr = nullptr;
}
size_t decoder_gemm_a_field(size_t* tidx_off) {
  *tidx_off = offsetof(GemmArgs, ta);
  return offsetof(GemmArgs, a_ptr);
}

void decoder_gemm_set_table(void* args, const uint64_t* table) {
  GemmArgs* g = static_cast<GemmArgs*>(args);
  if (g->ta >= 0 || g->tres >= 0) g->table = table;
}

void decoder_gemm_set_residual_table(void* args, const uint64_t* table, int32_t idx) {
  static_cast<GemmArgs*>(args)->table = table;
  static_cast<GemmArgs*>(args)->tres = idx;
  static_cast<GemmArgs*>(args)->residual = nullptr;
}
size_t decoder_gemm_residual_field(size_t* tidx_off) {
  *tidx_off = offsetof(GemmArgs, tres);
  return offsetof(GemmArgs, residual);
}

void decoder_gemm_set_status(void* args, uint32_t* word, uint64_t timeout_ns) {
  static_cast<GemmArgs*>(args)->st = DevStatus{word, timeout_ns};
}

void decoder_gemm_set_node_trace(void* args, unsigned long long* nt) {
  static_cast<GemmArgs*>(args)->ntrace = nt;
}

void decoder_gemm_set_trace(void* args, unsigned long long* trace) {
  static_cast<GemmArgs*>(args)->trace = trace;
  if (const char* v = getenv("CGX_GEMM_TRACE_CLK"); v && v[0] == '1') static_cast<GemmArgs*>(args)->flags |= kGemmTraceClk;
}

void decoder_gemm_set_w_after_wait(void* args) {
  static_cast<GemmArgs*>(args)->flags |= kGemmWAfterWait;
}

void decoder_gemm_set_trigger_after_wait(void* args) {
  static_cast<GemmArgs*>(args)->flags |= kGemmTriggerAfterWait;
}

static bool gemv_shape(uint32_t M, uint32_t N, uint32_t K) {
  const char* ngv = getenv("CGX_GEMM_NO_GEMV");         // measurement / test knob: force tcgen05
  return !(ngv && ngv[0] == '1') && M >= 1 && M <= (uint32_t)kGvMaxM && N >= 1 && K >= 8 && K % 8 == 0 &&
         K <= (uint32_t)(kGvMaxKS * kGvKV * 256);
}

bool decoder_gemm_supported(uint32_t M, uint32_t N, uint32_t K) {
  return gemv_shape(M, N, K) || (M >= 1 && K >= kBK && K % kBK == 0 && (N % 32 == 0));
}

int decoder_gemm_build(uint32_t M, uint32_t N, uint32_t K, uint32_t flags, const void* A, const void* W,
                       const void* bias, const void* residual, void* out, void* ws, void* cnt, void* args_out,
                       size_t* argbytes, dim3* grid, dim3* block, size_t* smem, const void** func) {
  if (!decoder_gemm_supported(M, N, K)) return CGX_E_UNSUPPORTED;
  if (gemv_shape(M, N, K) && !(flags & CGX_GEMM_ALLREDUCE)) {
    // small-M (decode) path: one output column per KS warps, KS = the K slices of 768 columns
    // (rounded up to a power of two)
    const uint32_t ks = K <= 768u ? 1u : K <= 1536u ? 2u : K <= 3072u ? 4u : 8u;
    *argbytes = sizeof(GemmArgs);
    *block = dim3(kGvWarps * 32);
    *smem = 0;
    // (M = 1, the T = 1 decode: scalar accumulators, 64 registers, 4 CTAs per SM; one output
    // column per warp group: two per warp measured 142.6 -> 157.3 us per decode replay)
    *grid = dim3((N * ks + kGvWarps - 1) / kGvWarps);
    if (M == 1)
      *func = ks == 1 ? (const void*)k_gemv_bf16<1, 1, 1> : ks == 2 ? (const void*)k_gemv_bf16<2, 1, 1>
            : ks == 4 ? (const void*)k_gemv_bf16<4, 1, 1> : (const void*)k_gemv_bf16<8, 1, 1>;
    else
      *func = ks == 1 ? (const void*)k_gemv_bf16<1, kGvMaxM, 1> : ks == 2 ? (const void*)k_gemv_bf16<2, kGvMaxM, 1>
            : ks == 4 ? (const void*)k_gemv_bf16<4, kGvMaxM, 1> : (const void*)k_gemv_bf16<8, kGvMaxM, 1>;
    if (!args_out) return CGX_OK;
    GemmArgs* g = static_cast<GemmArgs*>(args_out);
    memset(g, 0, sizeof(GemmArgs));
    g->a_ptr = static_cast<const __nv_bfloat16*>(A);
    g->w_ptr = static_cast<const __nv_bfloat16*>(W);
    g->bias = static_cast<const __nv_bfloat16*>(bias);
    g->residual = static_cast<const __nv_bfloat16*>(residual);
    g->out = static_cast<__nv_bfloat16*>(out);
    g->M = M;
    g->N = N;
    g->K = K;
    g->flags = flags;
    g->split = 1;
    g->tres = -1;
    g->ta = -1;
    return CGX_OK;
  }
  int bn = 0;
  uint32_t sp = 1;
  pick_tiling(M, N, K, &bn, &sp);
  *argbytes = sizeof(GemmArgs);
  GemmPipes pp = pick_pipes(bn, sp, K / kBK);
  if (const char* v = getenv("CGX_GEMM_PIPES")) parse_pipes(v, &pp);
  if (const char* t = getenv("CGX_GEMM_TILING")) {   // "NxK=BN/S/GA/RA/GW/RW" pins this shape's pipes
    char key[32];
    snprintf(key, sizeof key, "%ux%u=", N, K);
    if (const char* p = strstr(t, key)) {
      int b2 = 0, s2 = 0;
      const char* q = p + strlen(key);
      if (sscanf(q, "%d/%d/", &b2, &s2) == 2) {
        const char* r = strchr(strchr(q, '/') + 1, '/');
        if (r) parse_pipes(r + 1, &pp);
      }
    }
  }
  clamp_pipes(&pp, (K / kBK + sp - 1) / sp);
  *grid = dim3(N / bn, (M + kBM - 1) / kBM, sp);
  *block = dim3(kGemmThreads);
  *smem = smem_bytes(bn, sp, pp);
  if (*smem > kSmemLimit) return CGX_E_UNSUPPORTED;
  *func = kernel_for(bn, (flags & CGX_GEMM_ALLREDUCE) != 0);
  if (!args_out) return CGX_OK;
  if (get_encode() != CGX_OK) return CGX_E_CUDA;
  GemmArgs* g = static_cast<GemmArgs*>(args_out);
  memset(g, 0, sizeof(GemmArgs));
  // an EXTERNAL A has no address before the first bind: encode the template with any aligned
  // address (the kernel replaces it, kGemmADynamic)
  if (encode_kmajor(&g->tmA, A ? A : W, M, K, kBM, pp.ga) != CGX_OK) return CGX_E_CUDA;
  if (encode_kmajor(&g->tmB, W, N, K, (uint32_t)bn, pp.gw) != CGX_OK) return CGX_E_CUDA;
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
  if (getenv("CGX_GEMM_FENCE_ON_WAIT")) g->flags |= kGemmFenceOnWait;
  g->ga = pp.ga;
  g->ra = pp.ra;
  g->gw = pp.gw;
  g->rw = pp.rw;
  g->trace = nullptr;
  g->table = nullptr;
  g->tres = -1;
  g->ta = -1;
  g->a_ptr = static_cast<const __nv_bfloat16*>(A);
  g->w_ptr = static_cast<const __nv_bfloat16*>(W);
  return CGX_OK;
}

}  // namespace cgx
