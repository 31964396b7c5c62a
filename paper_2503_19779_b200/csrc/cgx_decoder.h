// Decoder-node kernels: LayerNorm, causal attention, tcgen05 bf16 GEMM.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace cgx {
// LayerNorm: one warp per row, registers hold the row (cols <= kLnMaxCols, cols % 8 == 0).
static constexpr uint32_t kLnMaxCols = 2048;
// add: the fused ADD -> LAYERNORM variant (LnArgs::add_b / add_out; tw must be 0)
const void* kfn_layernorm(int tw, bool add, uint32_t cols);
void decoder_ln_launch_dims(uint32_t rows, uint32_t cols, dim3* grid, dim3* block);

// Causal attention on CUDA cores (T <= 1024, D == 64).
const void* kfn_attention();
bool decoder_attn_supported(uint32_t T, uint32_t H, uint32_t D);
void decoder_attn_launch_dims(uint32_t T, uint32_t H, uint32_t D, dim3* grid, dim3* block, size_t* smem);

// tcgen05 GEMM out[M,N] = epi(A[M,K] * W[N,K]^T + bias): TMA tiles, TMEM accumulator.
bool decoder_gemm_supported(uint32_t M, uint32_t N, uint32_t K);
// Builds the by-value parameter block (tensor maps included) into args_out (64-B aligned) when
// args_out != nullptr; always reports its size, launch geometry and kernel handle.
// Split-K workspace and per-tile counters the kernel needs for this shape (0 if unsplit).
void decoder_gemm_plan(uint32_t M, uint32_t N, uint32_t K, size_t* ws_bytes, size_t* cnt_bytes);
int decoder_gemm_build(uint32_t M, uint32_t N, uint32_t K, uint32_t flags, const void* A, const void* W,
                       const void* bias, const void* residual, void* out, void* ws, void* cnt, void* args_out,
                       size_t* argbytes, dim3* grid, dim3* block, size_t* smem, const void** func);
// W / bias written inside the graph: load them only after griddepcontrol.wait.
void decoder_gemm_set_w_after_wait(void* args);
// Make a built GEMM parameter block trigger its PDL dependents only after its wait (T5 node 2).
void decoder_gemm_set_trigger_after_wait(void* args);
// CGX_GEMM_ALLREDUCE: the epilogue's peer all-reduce (regions as for k_allreduce_peer).
void decoder_gemm_set_allreduce(void* args, uint32_t rank, uint32_t world, uint32_t ar_index, uint32_t n_ar,
                                uint64_t slot_elems, uint32_t* counters, void* const* recv, uint32_t* const* flags);
uint32_t decoder_gemm_ctas(const void* args, dim3 grid);
// An EXTERNAL A operand (PI through the TMA descriptor): the kernel builds a per-CTA tensor map
// (tm_ws: decoder_gemm_ctas x 128 B, 128-B aligned device memory) with the replay's A address,
// table[idx] (INDIRECT) or the a_ptr field (idx < 0: patched by the patch modes; its byte offset,
// and that of the idx field, from decoder_gemm_a_field). The small-M path reads a_ptr / table[idx]
// directly.
// after_wait: rebuild the map only after griddepcontrol.wait (EAGER: launches of one node overlap).
void decoder_gemm_set_a_dynamic(void* args, const uint64_t* table, int32_t idx, void* tm_ws, bool after_wait);
size_t decoder_gemm_a_field(size_t* tidx_off);
// Re-point the table of a GEMM reading table entries (T6: graph gi reads table gi).
void decoder_gemm_set_table(void* args, const uint64_t* table);
// An EXTERNAL residual under INDIRECT: the epilogue reads its base pointer from table[idx].
void decoder_gemm_set_residual_table(void* args, const uint64_t* table, int32_t idx);
// Byte offsets of the residual pointer field and its int32 table-index field (patch modes).
size_t decoder_gemm_residual_field(size_t* tidx_off);
// Spin bound / failure word for the fused all-reduce epilogue (DevStatus, cgx_args.h).
void decoder_gemm_set_status(void* args, uint32_t* word, uint64_t timeout_ns);
// Diagnostics: replay-timeline stamps (CGX_NODE_TRACE=1; node_stamp, cgx_debug_node_trace).
void decoder_gemm_set_node_trace(void* args, unsigned long long* nt);
// Diagnostics: per-CTA %globaltimer trace [cta][16] written by the kernel (nullptr = off).
void decoder_gemm_set_trace(void* args, unsigned long long* trace);
// 3-D K-major bf16 operand map {64, rows, K/64}, box {64, box_rows, group}, SW128 (the layout both
// tcgen05 kernels stage: G stacked [box_rows][128 B] tiles), written to tm (128 B, 64-B aligned).
int decoder_encode_kmajor(void* tm, const void* base, uint64_t rows, uint64_t K, uint32_t box_rows, uint32_t group);
// LayerNorm folded into the consumer GEMM (exec option fuse & CGX_FUSE_LN_GEMM): the producer GEMM
// writes per-tile row sums of its bf16 output (stats: [grid.x][M] float2); the consumer streams the
// gamma-scaled weights W' with A = the LN's input h and corrects each output row in its epilogue
// (k_gemm.cu kGemmLnA), and stores the LN output slot. decoder_ln_fold_prep builds W', c1, c2 once
// (synchronous). CGX_E_UNSUPPORTED when the launch cannot (all-reduce epilogue, split shape, smem).
int decoder_gemm_set_stats_out(void* args, void* stats, dim3 grid);
int decoder_gemm_set_ln_a(void* args, dim3 grid, const void* stats, uint32_t ntiles, const void* h, const void* w_fold,
                          const float* c1, const float* c2, const void* gamma, const void* beta, void* ln_out,
                          float eps, size_t* smem, const void** func);
int decoder_ln_fold_prep(const void* W, const void* gamma, const void* beta, uint32_t N, uint32_t K, void* wf,
                         float* c1, float* c2);
bool decoder_gemm_is_tcgen05(const void* func);
// the small-M (GEMV) path serves this shape (M <= 4): a folded LN needs no producer row sums there
bool decoder_gemm_is_gemv(uint32_t M, uint32_t N, uint32_t K);
// Causal attention folded into its GEMM consumer (exec option fuse & CGX_FUSE_ATTN_GEMM, k_gemm.cu
// kGemmAttnA, D = 64, K = H * D): the small-M path at T = M = 1 (A = the v row); the tcgen05 path at
// T <= 128 re-plans the launch (grid, smem, kernel: K split S = H, each split computing its head's
// attention into the A tile). The ATTN output slot is still stored. CGX_E_UNSUPPORTED otherwise.
int decoder_gemm_set_attn_a(void* args, const void* qkv, void* attn_out, uint32_t H, uint32_t D, float scale,
                            dim3* grid, size_t* smem, const void** func);
}  // namespace cgx
