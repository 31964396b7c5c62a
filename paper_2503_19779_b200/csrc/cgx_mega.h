// Persistent decoder executor (the "megakernel" exec option, cgx_exec_opts.megakernel): a run of
// decoder-chain nodes (LAYERNORM, GEMM_BF16, ATTN_CAUSAL, bf16 ADD) executed by ONE launch of one
// CTA per SM instead of one kernel per node. The host compiles the nodes into STAGES separated by
// grid-wide barriers; every node's output slot is still written exactly as the per-node kernels
// write it (node-local parity applies unchanged). EXTERNAL operands are resolved once at kernel
// start, through the pointer table under INDIRECT ("de-references these
// pointers-to-pointers before performing any computation") or from the by-value ext_ptr array
// that the patch modes rewrite — the rebinding semantics of every arm are those of
// the per-node graph.
//
// Why: at M = 128 the per-node chain is a sequence of ~4-5 us latency
// chains (launch, TMEM allocation, first TMA, MMA issue, epilogue, grid drain) while the weights
// stream in ~2 us per layer. Here TMEM is allocated once, each GEMM's weight slice is TMA-prefetched
// into shared memory one GEMM stage ahead (it is STATIC), and stages hand over through L2 behind a
// ~0.5 us grid barrier.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "cgx_args.h"

namespace cgx {

static constexpr int kMegaMaxExt = 8;          // EXTERNAL operands of a fused range
static constexpr int kMegaThreads = 256;       // 8 warps: 0 TMA producer, 1 MMA issuer, 4-7 epilogue
static constexpr int kMegaMaxRegs = 4;         // row registers of a ROW stage
static constexpr uint32_t kMegaMaxRowOps = 4;  // ops per ROW stage (no register is evicted)
static constexpr uint32_t kMegaMaxSplit = 16;  // K splits of a deferred GEMM (ROW prefetch slots)
static constexpr uint32_t kMegaMaxCols = 2048; // ROW stage row length (256 threads x 4 x 2 chunks)
static constexpr uint32_t kMegaABytes = 128u * 1024u;   // A ring: 2 slots of 4 k-blocks (16 KiB each)
static constexpr uint32_t kMegaASlots = 2;
static constexpr uint32_t kMegaAGroup = 4;              // k-blocks per A slot
static constexpr uint32_t kMegaWBytes = 48u * 1024u;    // per W buffer (2 buffers: one GEMM stage ahead)
static constexpr uint32_t kMegaMaxBN = 64;              // TMEM columns allocated once

enum : uint32_t { kMegaRow = 0, kMegaGemm = 1, kMegaAttn = 2 };
enum : uint32_t { kRowFixup = 0, kRowAdd = 1, kRowLn = 2 };

// An operand: a direct device pointer, an EXTERNAL (index into MegaArgs::ext_*), or — inside a ROW
// stage — a row register holding a value an earlier op of the same stage produced.
struct MegaRef {
  const void* p;
  int32_t ext;    // >= 0: external operand index
  int32_t reg;    // >= 0: row register
};

// One row-local op of a ROW stage (rows are distributed over the CTAs, row r -> CTA r % G, the
// same mapping in every ROW stage, so consecutive row ops need no barrier between them).
//   kRowFixup: out = bf16(epi(sum_{s<S} ws[s][r][:] + bias)), epi = [GELU] [+ residual]: the
//              deferred epilogue of a split-K GEMM stage (the per-node GEMM's exact formula)
//   kRowAdd:   out = bf16(a + b)
//   kRowLn:    out = bf16((x - mean) * rstd * gamma + beta)
struct alignas(16) MegaRowOp {
  uint32_t kind, flags, S, node;   // flags: CGX_GEMM_BIAS / GELU / RESIDUAL (kRowFixup)
  uint32_t pf, col;                // bit x: operand x (a, b, c, d) is fetched from memory / per column
  MegaRef a, b, c, d;              // Fixup: c = bias, d = residual; Add: a + b; Ln: a = x, c = gamma, d = beta
  const float* ws;                 // Fixup: partial tiles [S][rows][cols] fp32
  void* out;                       // bf16 [rows][cols], always written
  int32_t out_reg;                 // register receiving the bf16-rounded row (-1: none)
  float eps;
};

struct alignas(16) MegaStage {
  uint32_t kind, barrier, node;
  uint32_t bar_next;               // the next stage starts with a grid barrier
  int32_t next_gemm;               // index of the next GEMM stage (its W is prefetched at this one), -1
  // ROW
  uint32_t rows, cols, op0, n_ops;
  // GEMM: out[M,N] = epi(A[M,K] W[N,K]^T + bias); tasks = m_tiles x n_tiles x split, K-split
  // slices of kps k-blocks; A through groups of ga k-blocks (3-D box {64, 128, ga}), W through one
  // box {64, bn, kps} per task; deferred = write fp32 partials to ws, a later kFixup applies epi
  uint32_t M, N, K, flags, bn, split, m_tiles, n_tiles, kps, ga, deferred, w_buf;
  uint64_t tmA, tmW;               // device addresses of 64-B aligned CUtensorMaps
  MegaRef bias, res;
  void* out;
  float* ws;
  // ATTN
  uint32_t T, H;
  float scale;
  MegaRef qkv;
  void* aout;
};

// Device records: [stage descriptor (kMegaDescStage B)][kMegaMaxRowOps row ops], one per stage, so a
// stage's whole description is one fixed-size copy with no dependent read.
struct alignas(64) MegaArgs {
  const uint8_t* recs;
  uint32_t n_stages, G;            // G = gridDim.x (one CTA per SM)
  int32_t first_gemm;              // first GEMM stage (its W is prefetched at kernel entry), -1
  const uint64_t* table;           // INDIRECT pointer table (ext_t >= 0)
  const void* ext_ptr[kMegaMaxExt];   // patch modes: the bound pointer (rewritten per bind)
  int32_t ext_t[kMegaMaxExt];         // table index (INDIRECT), -1: ext_ptr
  uint32_t n_ext;
  uint32_t* flags;                 // grid barrier: per-CTA arrival counts (monotonic across replays)
  uint32_t bar_mode, bar_sleep_ns; // barrier variant (measurement knob CGX_MEGA_BAR) and poll back-off
  uint32_t null_work;              // diagnostics (CGX_MEGA_NULL=1): skip every stage body
  uint32_t dbg;                    // diagnostics (CGX_MEGA_DBG bits): skip individual proxy fences
  DevStatus st;                    // barrier spin bound / failure report
  unsigned long long* ntrace;      // CGX_NODE_TRACE=1: [entry min, ready max, exit max] ns
  unsigned long long* strace;      // CGX_MEGA_TRACE: [stage][cta][8] ns stamps (k_mega.cu mtrace)
};
static constexpr uint32_t kDevErrBarrier = 8u;   // a CTA never reached a grid barrier
static constexpr uint32_t kMegaDescStage = 256;   // shared-memory copy of the current stage descriptor
static_assert(sizeof(MegaStage) <= kMegaDescStage && sizeof(MegaStage) % 16 == 0, "stage descriptor size");
static_assert(sizeof(MegaRowOp) % 16 == 0 && sizeof(MegaRowOp) <= 128, "row op descriptor size");
static constexpr uint32_t kMegaRec = kMegaDescStage + kMegaMaxRowOps * (uint32_t)sizeof(MegaRowOp);

const void* kfn_mega();
size_t mega_smem_bytes();

}  // namespace cgx
