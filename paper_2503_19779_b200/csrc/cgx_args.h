// Kernel argument blocks shared by the runtime (host) and the kernels (device).
// Every chain kernel takes exactly ONE by-value struct, so a node's whole parameter image is one
// contiguous block: SETPARAMS rewrites it with cudaGraphExecKernelNodeSetParams, and the
// parameter-indirection variant differs only in the table index fields ("replaces
// each pointer argument with a pointer-to-pointer").
#pragma once
#include <stdint.h>
#include <cuda_bf16.h>

namespace cgx {

// Device-side failure reporting (include/cgx.h CGX_E_DEVICE): kernels that spin on another agent
// (dataflow counters, peer all-reduce flags) or launch work from the device never trap. On a
// timeout (%globaltimer, timeout_ns) or a failed device launch they store a code into the exec's
// status word (mapped pinned host memory, sys-scope release store), stop waiting and finish; the
// host sees the word at the exec's next cgx_launch, which returns CGX_E_DEVICE from then on.
struct DevStatus {
  uint32_t* word;          // device alias of the exec's mapped host status word (nullptr = none)
  uint64_t timeout_ns;     // spin bound
};
static constexpr uint32_t kDevErrDataflow = 1u;     // dataflow counter never reached its target
static constexpr uint32_t kDevErrPeer = 2u;         // peer all-reduce: a source never published
static constexpr uint32_t kDevErrDevLaunch = 4u;    // device-side cudaGraphLaunch failed

// Operand fetch rule ("de-references these pointers-to-pointers before performing
// any computation"): operand i reads `ptr[i]` when tidx[i] < 0, else `table[tidx[i]]`; the load
// happens once at kernel start into a register (warp-uniform address, one request per warp).
struct ElemArgs {
  const uint64_t* table;   // device pointer table (INDIRECT) or nullptr
  const void* in0;
  const void* in1;
  void* out;
  int32_t t0, t1;          // table index of in0/in1, -1 = direct pointer
  uint32_t flags;          // kFlagTableAfterWait: fetch table entries after griddepcontrol.wait
  uint32_t cols;           // REDUCE_SUM row length
  uint64_t n;              // elements
  float scalar;            // SCALE_IMM
  uint32_t pre;            // bit i: operand i may be loaded BEFORE griddepcontrol.wait (an
                           // EXTERNAL or STATIC slot, never written inside the graph)
  // Dataflow mode (kFlagDataflow; runtime.cu set_dataflow): per-node completion counters replace
  // griddepcontrol.wait, so a node waits for exactly the nodes it depends on.
  uint32_t* df_done;       // per-launch CTA-completion counters of this exec (monotonic)
  uint32_t* df_epoch;      // replay counter of this exec, bumped by its first node
  uint32_t df_self;        // this launch's counter
  uint32_t df_n;           // dependencies
  uint32_t df_dep[4];      // their counters
  uint32_t df_ctas[4];     // their CTA counts: dependency complete <=> done >= epoch * ctas
  unsigned long long* trace;  // diagnostics (CGX_NODE_TRACE=1): [entry min, ready max, exit max] ns
  DevStatus st;            // dataflow spin bound / failure report
};
static constexpr int kDfMaxDeps = 4;
// PDL protocol (see runtime.cu, set_pdl_flags): every chain kernel triggers its dependents at
// entry, so consecutive nodes' prologues cascade; only data nothing in the graph writes (inputs,
// weights, the table under T1) is read before griddepcontrol.wait. The first consumer after a
// root table-writer reads the table after its wait and triggers only then, so no later node can
// start before the root has completed.
static constexpr uint32_t kFlagTableAfterWait = 1u;
static constexpr uint32_t kFlagTriggerAfterWait = 2u;
// Deferred wait (runtime.cu, set_defer_flags): a node whose operands are all EXTERNAL/STATIC and
// whose output no earlier node of the graph reads or writes has no data dependency on any
// predecessor, so it computes and stores BEFORE griddepcontrol.wait and waits only before exiting.
// The wait is kept (at the end) so "node k complete => nodes < k complete" stays transitive for the
// later nodes that rely on it.
static constexpr uint32_t kFlagDeferWait = 4u;
// Dataflow (graph modes, every node a chain kernel): the early-trigger cascade keeps every node of
// the replay launched in order (all CTAs of node k have started before node k+1 is launched), and
// each node, instead of griddepcontrol.wait, spins (one thread, ld.acquire.gpu) until the CTA
// counters of its RAW / WAR / WAW dependencies reach epoch x CTAs, and signals its own counter
// (bar.sync, fence, atomic add) when done. Deadlock-free because a node only ever waits for
// EARLIER nodes, whose CTAs are all resident or finished by the time it runs.
static constexpr uint32_t kFlagDataflow = 8u;
static constexpr uint32_t kFlagEpochBump = 16u;   // first node: CTA 0 bumps the epoch before it triggers
// Dataflow refinements: a dependency on the IMMEDIATELY preceding node is taken with the hardware
// griddepcontrol.wait (cheaper than a counter round trip); only nodes some later node spins on
// signal their counter.
static constexpr uint32_t kFlagDfPdlWait = 32u;
static constexpr uint32_t kFlagDfSignal = 64u;
// Diagnostics only (env CGX_DEBUG_NOOP=1 / 2, scripts/diag_cadence_split.py): return right after
// the trigger (pure launch cascade of the real kernels), or keep the synchronisation but skip the
// memory work.
static constexpr uint32_t kFlagDbgNoop = 1u << 12;
static constexpr uint32_t kFlagDbgNoWork = 1u << 13;
// LayerNorm: gamma and beta are STATIC slots (never written in the graph): load them pre-wait.
static constexpr uint32_t kFlagLnParamsPre = 1u << 14;

// Multi-tensor copy (BASELINE north_star (1)). Static part lives in device
// memory (per exec, written once at capture); the fresh sources travel by value in the params.
struct CopyDesc {
  void* dst;               // placeholder
  uint64_t nbytes;
  uint64_t chunk_begin;    // first global block/chunk index of this tensor
  uint64_t n_chunks;
};
template <int CAP>
struct CopyArgs {
  const CopyDesc* desc;    // [n_tensors]
  const uint32_t* chunk_tensor;  // [n_chunks] owning tensor per chunk (bulk variant only)
  uint32_t n_tensors;
  uint32_t chunk_bytes;
  uint64_t n_chunks;
  const void* src[CAP];
};

// T3 root table writer: pointers by value, one cudaGraphExecKernelNodeSetParams per bind.
template <int CAP>
struct TableWriteArgs {
  uint64_t* table;
  uint32_t n;
  uint32_t pad;
  uint64_t ptr[CAP];
};

// T4 root kernel: read slot (seq % ring) of a mapped pinned staging ring, ack through mapped
// host memory so the host knows when a slot may be overwritten.
struct MappedTableArgs {
  const uint64_t* staging;       // device alias of pinned host ring [ring][n_pad]
  uint64_t* table;
  unsigned long long* seq;       // device counter (replays consumed)
  unsigned long long* ack;       // device alias of pinned host word
  uint32_t n, n_pad, ring, pad;
};

// Decoder nodes.
struct LnArgs {
  const uint64_t* table;
  const void* x; const void* g; const void* b; void* out;
  int32_t tx, pad0;
  uint32_t flags, rows, cols, pad1;
  float eps;
  unsigned long long* ntrace;   // CGX_NODE_TRACE=1: [entry, ready, exit] ns (node_stamp)
  // ADD -> LAYERNORM fused at capture (cgx_exec_opts.fuse & CGX_FUSE_ADD_LN, k_layernorm<TW, true>):
  // the LN input is h = bf16(x + add_b), written to add_out (the ADD node's slot) and normalised
  // from registers. x / tx are then the ADD's first operand.
  const void* add_b;
  void* add_out;
  int32_t tb, pad2;             // table index of an EXTERNAL add_b (-1: direct pointer)
};

// AttnArgs::flags: every warp loads the Q fragments (measurement knob CGX_ATTN_QALL=1, the round-1
// behaviour; by default only the warps owning a key chunk do)
static constexpr uint32_t kAttnQAll = 1u << 8;
struct AttnArgs {
  const void* qkv; void* out;
  uint32_t T, H, D, flags;
  float scale;
  unsigned long long* ntrace;   // CGX_NODE_TRACE=1 (node_stamp)
  unsigned long long* ctrace;   // CGX_CTA_TRACE=1: per-CTA [cta][8] %globaltimer phase stamps (diagnostics)
};

// T5 (FIRST_NODE transport): the first node of the graph carries the bound pointers by value; its
// CTA 0 publishes the table (stores + gpu-scope fence) before triggering the dependent launch, so
// every later node may fetch the table before its wait. ArgsTW<Base, 0> is the plain block.
template <int CAP>
struct TWPart {
  uint64_t* table;
  uint32_t n;
  uint32_t pad;
  uint64_t ptr[CAP];
};
template <typename Base, int CAP>
struct ArgsTW {
  Base a;
  TWPart<CAP> tw;
};
template <typename Base>
struct ArgsTW<Base, 0> {
  Base a;
};
}  // namespace cgx

// Kernel handles exported by the kernel translation units (host functions). `tw` = table-writer
// capacity for the T5 first node (0 = plain kernel; else 8, 64 or 512 pointers).
extern "C++" {
namespace cgx {
// Peer all-reduce (k_allreduce_peer, cgx_chain_set_peers): per-rank region = receive data
// [2 parity][world][slot_elems] bf16, then flags [kArMaxNodes][kArMaxWorld][kArMaxCtas] uint32.
static constexpr int kArMaxWorld = 8;
static constexpr int kArMaxCtas = 256;
static constexpr int kArMaxNodes = 64;
struct PeerArArgs {
  const __nv_bfloat16* in;
  __nv_bfloat16* out;
  uint64_t n;                          // elements (multiple of 8)
  uint64_t slot_elems;                 // elements per receive slot
  uint32_t rank, world, ar_index, n_ar, flags;
  uint32_t* counters;                  // chain-owned [kArMaxNodes][kArMaxCtas] generations
  __nv_bfloat16* recv[kArMaxWorld];    // every rank's receive data (mapped in this process)
  uint32_t* flags_of[kArMaxWorld];     // every rank's flag array
  DevStatus st;                        // spin bound / lost-peer report
};
const void* kfn_allreduce_peer();
// NVLS / multicast all-reduce (cgx_chain_set_multicast, k_allreduce_mc): every rank's region is
// bound to one multicast object at the same offsets: data [max_ar][2 parity][slot] bf16, then the
// arrival counters [max_ar][kArMaxCtas] uint32. uc_* address this rank's copy, mc_* the multicast
// mapping (multimem.* instructions act on every rank's copy through the NVSwitch).
struct McArArgs {
  const __nv_bfloat16* in;
  __nv_bfloat16* out;
  uint64_t n;                          // elements (multiple of 8)
  uint64_t slot_elems;                 // elements per parity slot
  uint32_t world, ar_index, n_ar, pad;
  uint32_t* counters;                  // chain-owned [kArMaxNodes][kArMaxCtas] generations
  __nv_bfloat16* uc_data;              // this node's [2][slot] block, this rank's copy
  __nv_bfloat16* mc_data;              // the same block through the multicast mapping
  uint32_t* uc_flags;                  // [kArMaxCtas] arrival counters of this node, this rank's copy
  uint32_t* mc_flags;                  // the same through the multicast mapping
  DevStatus st;                        // spin bound / lost-peer report
};
const void* kfn_allreduce_mc();
static constexpr int kGatherMax = 64;
struct GatherArgs {
  const void* src[kGatherMax];
  void* dst[kGatherMax];
  uint64_t nbytes[kGatherMax];
  uint32_t n;
};
const void* kfn_gather();
const void* kfn_transpose_bf16(int tw = 0);
const void* kfn_elem(int op, int dtype, int tw = 0);   // ADD/MUL/SCALE_IMM/COPY f32|bf16
const void* kfn_reduce_sum_f32(int tw = 0);
int tw_cap(int n);                                // 8, 64, 512 (0 if n > 512)
const void* kfn_copy(int cap);                    // CAP in {8, 64, 1024}
const void* kfn_copy_bulk(int cap);               // TMA bulk-copy variant
uint32_t copy_block_bytes();                      // block size of the LDG/STG copy kernel
size_t copy_bulk_smem();
uint32_t copy_bulk_chunk();
const void* kfn_table_write(int cap);             // CAP in {8, 64, 512}
const void* kfn_table_mapped();
const void* kfn_empty();
const void* kfn_pdl_nop();
const void* kfn_fill_uniform_f32();
int elem_block_threads();
int elem_tile_vecs();      // 16-B vectors per thread per operand in one elementwise tile
}  // namespace cgx
}
