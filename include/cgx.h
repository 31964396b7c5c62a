/*
 * cgx.h — C ABI of the B200-native CUDA-Graph input-rebinding hot path (arXiv 2503.19779).
 *
 * The calls follow the paper's statement of the problem:
 *   capture a kernel sequence ............ cgx_chain_* + cgx_exec_create   (§2.2)
 *   replace mutable params ............... placeholders / pointer table
 *   refresh them before each replay ...... cgx_bind
 *   replay ............................... cgx_launch
 *   decide per graph whether to deploy ... cgx_profile + cgx_select
 * (P:Lnnn = line of the paper's LaTeX source, PAPER.md; S:Lnnn = SPEC.md.)
 *
 * Conventions
 *  - Every function returns an int status (cgx_status) and never aborts; kernels never trap (a
 *    device-side wait that times out, bound 10 s or env CGX_SPIN_TIMEOUT_MS, is reported through
 *    CGX_E_DEVICE at the exec's next cgx_launch). On a non-OK status
 *    cgx_last_error() returns a thread-local human-readable message (CUDA/NCCL errors carry the
 *    library's own message). Out-parameters are written only on CGX_OK.
 *  - All pointers to tensor data are DEVICE pointers of the chain's device (plain addresses, no
 *    framework types). Host-side arrays (ext_dptrs, attrs, profiles) are read during the call only.
 *  - Ownership: the caller owns external input buffers, static buffers (weights) and any NCCL
 *    communicator. The library owns placeholders, the pointer table and its pinned staging,
 *    internal/output buffers, graphs and execs. Output buffers are static and are overwritten by
 *    the next launch on that chain (PyTorch2-CG semantics).
 *  - Lifetime of inputs: an input bound with cgx_bind must stay valid and unmodified until the
 *    cgx_launch that reads it has completed in stream order. COPY mode stops reading it once the
 *    copy kernel (enqueued by cgx_bind) has run; INDIRECT / SETPARAMS / EAGER read it during the
 *    whole replay (the key semantic difference of parameter indirection).
 *  - Threading: an exec belongs to one stream and one host thread. Execs of the same chain share
 *    the chain's internal buffers, so they must not run concurrently (one stream per chain).
 *    Chains on different devices are independent.
 *  - Sizes are fixed at capture; there are no dynamic shapes.
 */
#ifndef CGX_H_
#define CGX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CGX_ABI_VERSION 1
#define CGX_MAX_IN 4                    /* max inputs per node */
#define CGX_MAX_PROFILE_KERNELS 1024    /* max kernels in one profiled segment */
#define CGX_MAX_PROFILE_DEPS 8192       /* max dependency edges of a profiled segment (model 1) */

typedef struct cgx_chain cgx_chain;     /* a kernel sequence description (slots + nodes) */
typedef struct cgx_exec cgx_exec;       /* one captured+instantiated graph (or eager runner) */

typedef enum {
  CGX_OK = 0,
  CGX_E_INVALID_ARG = 1,      /* null/out-of-range argument, bad slot/node index, bad attr */
  CGX_E_STATE = 2,            /* call not valid now (e.g. launch before the first bind) */
  CGX_E_NOT_ELIGIBLE = 3,     /* host pointer bound (P:L264-265 dangling host pointer hazard),
                                 node writes an EXTERNAL/STATIC slot */
  CGX_E_MISSING_INPUT = 4,    /* bind with the wrong number of inputs */
  CGX_E_SIZE_MISMATCH = 5,    /* node shapes inconsistent with its slots */
  CGX_E_MISALIGNED = 6,       /* bound pointer not 16-byte aligned */
  CGX_E_UNSUPPORTED = 7,      /* op/dtype/mode combination not built */
  CGX_E_OFFSET_NOT_FOUND = 8, /* param-offset discovery: no match (NEXT-2) */
  CGX_E_OFFSET_AMBIGUOUS = 9, /* param-offset discovery: >= 2 matches (NEXT-2) */
  CGX_E_CUDA = 10,            /* CUDA runtime error; message in cgx_last_error() */
  CGX_E_NCCL = 11,            /* NCCL error; message in cgx_last_error() */
  CGX_E_DEVICE = 12           /* a kernel of an earlier replay of this exec reported a device-side
                                 failure instead of trapping (a peer all-reduce or dataflow spin
                                 timed out, a device-side graph launch failed; cgx_stats
                                 device_error has the bits). Sticky for the exec. */
} cgx_status;

typedef enum { CGX_F32 = 0, CGX_BF16 = 1 } cgx_dtype;

/* Slot kinds (P:L601-607 and footnote P:L522-525): EXTERNAL = supplied anew every replay
 * (an application input: rebound); STATIC = captured by address, never rebound (weights,
 * SURVEY reading 4); INTERNAL = produced by an earlier node of the same chain (never copied). */
typedef enum { CGX_SLOT_EXTERNAL = 0, CGX_SLOT_STATIC = 1, CGX_SLOT_INTERNAL = 2 } cgx_slot_kind;

/* Node ops (SPEC opcode algebra, plus the decoder nodes of SURVEY §8(a) a7).
 * Inputs per op (in_slots order) and definitions:
 *   ADD        [a, b]        out[i] = a[i] + b[i]                 f32 or bf16, i < attr.n
 *   MUL        [a, b]        out[i] = a[i] * b[i]
 *   SCALE_IMM  [a]           out[i] = a[i] * attr.scalar (by-value float)
 *   COPY       [a]           out[i] = a[i]
 *   REDUCE_SUM [a]           out[r] = sum_c a[r*cols + c], cols = attr.cols, r < n/cols (f32)
 *   LAYERNORM  [x, g, b]     rows x cols bf16, population variance, attr.eps
 *   GEMM_BF16  [A, W, bias(, residual)]  out[M,N] = epi(A[M,K] W[N,K]^T + bias), flags below
 *   ATTN_CAUSAL [qkv]        qkv [T, 3*H*D] (q|k|v, head-major) -> out [T, H*D], causal softmax
 *   ALLREDUCE_SUM [x]        out = sum over ranks of x (bf16), captured ncclAllReduce
 *   SCALE_T    [a, s]        out[i] = a[i] * s[0], s a 1-element f32 slot: the CGCT rewrite of a
 *                            by-value scalar into a device tensor (NEXT-3) so the
 *                            scalar can be rebound per replay like any input */
typedef enum {
  CGX_OP_ADD = 0, CGX_OP_MUL = 1, CGX_OP_SCALE_IMM = 2, CGX_OP_COPY = 3, CGX_OP_REDUCE_SUM = 4,
  CGX_OP_LAYERNORM = 5, CGX_OP_GEMM_BF16 = 6, CGX_OP_ATTN_CAUSAL = 7, CGX_OP_ALLREDUCE_SUM = 8,
  CGX_OP_SCALE_T = 9,
  /* training-shaped chain, bf16, one rounding each: a - b; a + scalar * b;
     tanh-GELU(a); a * GELU'(b) (a = upstream gradient, b = pre-activation); out[c,r] = in[r,c] for
     a [n / cols, cols] matrix */
  CGX_OP_SUB = 10, CGX_OP_AXPY = 11, CGX_OP_GELU = 12, CGX_OP_GELU_BWD = 13, CGX_OP_TRANSPOSE = 14
} cgx_op;

#define CGX_GEMM_BIAS 1u
#define CGX_GEMM_GELU 2u        /* tanh-approximate GELU after the bias */
#define CGX_GEMM_RESIDUAL 4u    /* + in_slots[3] after the activation */
#define CGX_GEMM_ALLREDUCE 8u   /* row-parallel TP: the epilogue sums the bf16 output tile over the
                                   chain's peer ranks (cgx_chain_set_peers) before storing it — the
                                   GEMM and its all-reduce in ONE kernel; tcgen05 path only */

typedef struct {
  uint64_t n;          /* elementwise/reduce: elements processed (0 = whole first input) */
  float scalar;        /* SCALE_IMM constant; ATTN_CAUSAL softmax scale */
  float eps;           /* LAYERNORM epsilon */
  uint32_t rows, cols; /* LAYERNORM rows x cols; REDUCE_SUM row length (cols) */
  uint32_t M, N, K;    /* GEMM_BF16 */
  uint32_t flags;      /* CGX_GEMM_* */
  uint32_t T, H, D;    /* ATTN_CAUSAL */
} cgx_attr;

/* Execution modes (the arms of BASELINE.json north_star):
 *   EAGER            launch every node from the host with the current pointers (PT2-No-CG)
 *   GRAPH_COPY       placeholders + per-replay multi-tensor copy (PT2-CG baseline)
 *   GRAPH_INDIRECT   parameter indirection: kernels read base pointers from a device pointer
 *                    table patched once per replay
 *   GRAPH_SETPARAMS  rewrite each consuming node's params with cudaGraphExecKernelNodeSetParams
 *                    (comparison arm, "graph management APIs")
 *   GRAPH_STALE      negative control: inputs recorded by value at the first bind and never
 *                    rebound */
typedef enum {
  CGX_MODE_EAGER = 0, CGX_MODE_GRAPH_COPY = 1, CGX_MODE_GRAPH_INDIRECT = 2,
  CGX_MODE_GRAPH_SETPARAMS = 3, CGX_MODE_GRAPH_STALE = 4
} cgx_mode;

/* INDIRECT pointer-table transports (the paper only says "host-to-device
 * copies over the PCIe"):
 *   H2D          T1: cudaMemcpyAsync of pinned staging into the table before cudaGraphLaunch
 *   ROOT_MEMCPY  T2: memcpy node at the graph root from ping-pong pinned staging
 *   ROOT_PARAMS  T3: root table-writer kernel whose by-value params carry the pointers, updated
 *                    with one cudaGraphExecKernelNodeSetParams per bind
 *   ROOT_MAPPED  T4: root kernel reading a mapped pinned staging ring (zero-copy)
 *   FIRST_NODE   T5: no extra node. The first node's by-value params carry the pointers (one
 *                    cudaGraphExecKernelNodeSetParams per bind); its CTA 0 publishes the table
 *                    (store + gpu-scope fence) before it triggers the dependent launch, so every
 *                    later node may fetch table entries before its griddepcontrol.wait. Needs an
 *                    elementwise/reduce/LN first node and <= 512 externals (else UNSUPPORTED).
 *   H2D_PINGPONG T6: two tables and two captured graphs used alternately; the H2D copy of
 *                    replay k+1's pointers (pinned staging -> table) runs on a side stream while
 *                    replay k executes, ordered by events (the paper's "pointer copies over the
 *                    PCIe", with the PCIe latency hidden behind the previous replay).
 *   PRELUDE      T7 (NEXT-1): the consumers are plain direct-pointer kernels (stand-ins for opaque
 *                    vendor kernels) captured as device-updatable nodes; a prelude root
 *                    node dereferences the table (one H2D per replay) and writes every pointer into
 *                    the consumers' parameter buffers with cudaGraphKernelNodeSetParam.
 *   DEVICE       T8 (NEXT-4): as H2D for host binds, but the graph is instantiated for device
 *                    launch, so cgx_device_loop can run many replays with no host work: a
 *                    scheduler kernel copies replay i's pointer set into the table and
 *                    tail-launches the chain graph, then itself. */
typedef enum {
  CGX_XPORT_DEFAULT = 0, CGX_XPORT_H2D = 1, CGX_XPORT_ROOT_MEMCPY = 2, CGX_XPORT_ROOT_PARAMS = 3,
  CGX_XPORT_ROOT_MAPPED = 4, CGX_XPORT_FIRST_NODE = 5, CGX_XPORT_H2D_PINGPONG = 6, CGX_XPORT_PRELUDE = 7,
  CGX_XPORT_DEVICE = 8
} cgx_transport;

typedef enum { CGX_DECIDE_EAGER = 0, CGX_DECIDE_GRAPH_COPY = 1, CGX_DECIDE_GRAPH_INDIRECT = 2 } cgx_decision;

/* Exec options; an all-zero struct means "defaults". */
typedef struct {
  cgx_mode mode;
  cgx_transport transport;  /* INDIRECT only (0 = ROOT_PARAMS) */
  int first_node;           /* node range [first_node, first_node + n_nodes) */
  int n_nodes;              /* 0 = to the end of the chain */
  int no_pdl;               /* 1 = plain stream edges instead of programmatic dependent launch */
  int validate;             /* bind-time residency check: 0 = cached per address (default),
                               1 = every bind, 2 = off (alignment and count are always checked) */
  int copy_impl;            /* GRAPH_COPY: 0 = multi-tensor LDG/STG kernel, 1 = cudaMemcpyAsync per
                               tensor, 2 = multi-tensor TMA bulk-copy kernel */
  int sync_mode;            /* graph modes with PDL, how the captured nodes are ordered:
                               CGX_SYNC_AUTO (0) = GRAPH for every graph mode with PDL (all
                               transports, PRELUDE and DEVICE included); EAGER and no_pdl execs
                               keep their serial stream order; CGX_SYNC_DEFER (1) = one serial stream, deferred
                               griddepcontrol.wait for nodes with no in-graph producer;
                               CGX_SYNC_CHAIN (2) = one serial stream, griddepcontrol.wait in every
                               node; CGX_SYNC_GRAPH (3) = the graph is captured as the chain's
                               data-dependency DAG over `graph_streams` capture streams (PDL +
                               griddepcontrol.wait inside a stream, graph edges across streams);
                               CGX_SYNC_DATAFLOW (4) = one serial stream, per-node completion
                               counters (deferred waits when a node cannot use them) */
  int graph_streams;        /* CGX_SYNC_GRAPH: capture streams (0 = 16, at most 64) */
  int megakernel;           /* 1 = run the node range as ONE persistent launch (one CTA per SM,
                               grid barriers between stages) instead of one kernel per
                               node. Every node must be LAYERNORM, GEMM_BF16 (no ALLREDUCE, A not
                               EXTERNAL, W STATIC), ATTN_CAUSAL or a bf16 ADD, with at most 8
                               EXTERNAL operands; otherwise exec creation fails with
                               CGX_E_UNSUPPORTED. Not with the FIRST_NODE transport or SYNC_DATAFLOW.
                               Every node's output slot is written as in the per-node exec, and the
                               rebinding semantics of every mode are unchanged. 0 = off (default) */
  int fuse;                 /* capture-time fusions (bit mask, 0 = none). CGX_FUSE_ADD_LN runs a
                               bf16 ADD and the LAYERNORM that normalises its output as ONE launch
                               (both output slots written, bit-identical to the two kernels).
                               CGX_FUSE_LN_GEMM folds a LAYERNORM into the GEMM that consumes it
                               (a W^T = rstd (h W'^T) - rstd mean c1 + c2 with W' = gamma-scaled W,
                               prepared once at exec creation): tcgen05 consumers take mean / rstd
                               from per-tile row sums the previous GEMM launch writes (not
                               bit-identical to the LN kernel, within the bf16 tolerance); small-M
                               (GEMV) consumers compute them from their own A loads with the LN
                               kernel's reduction order; the LN output slot is still stored.
                               CGX_FUSE_ATTN_GEMM folds a T = 1 ATTN_CAUSAL (the decode step) into
                               its small-M (GEMV) consumer, which forms A = attention(qkv) itself
                               (one visible key: A = v exactly, bit-identical to the kernel) and stores
                               the ATTN output slot. The exec then has fewer launches
                               than nodes (cgx_stats n_nodes counts nodes, kernels_per_replay
                               launches) */
} cgx_exec_opts;
#define CGX_FUSE_ADD_LN 1
#define CGX_FUSE_LN_GEMM 2
#define CGX_FUSE_ATTN_GEMM 4

typedef enum {
  CGX_SYNC_AUTO = 0, CGX_SYNC_DEFER = 1, CGX_SYNC_CHAIN = 2, CGX_SYNC_GRAPH = 3, CGX_SYNC_DATAFLOW = 4
} cgx_sync_mode;

typedef struct {
  uint64_t bytes_data_rebound;   /* last bind: data bytes copied into placeholders */
  uint64_t bytes_ptr_rebound;    /* last bind: pointer bytes written to the table (8 x N_ext) */
  uint64_t total_bytes_data, total_bytes_ptr;
  uint64_t n_binds, n_launches;
  uint32_t n_setparam_calls;     /* last bind: cudaGraphExecKernelNodeSetParams calls */
  uint32_t n_copy_tensors;       /* last bind: tensors copied */
  uint32_t n_nodes;              /* K: chain nodes in this exec */
  uint32_t n_graph_nodes;        /* nodes in the instantiated graph (incl. a root node) */
  uint32_t n_ext;                /* N_ext of this exec */
  uint32_t kernels_per_replay;   /* library kernels per bind+launch (copy/root/chain) */
  uint32_t mode, transport;
  uint32_t n_deferred;           /* nodes running with the deferred PDL wait */
  uint32_t dataflow;             /* 1: nodes synchronise through dataflow counters */
  uint32_t dag_streams;          /* CGX_SYNC_GRAPH: capture streams holding at least one node */
  uint32_t device_error;         /* device-side failure bits seen so far (0 = none; CGX_E_DEVICE):
                                    1 dataflow timeout, 2 lost peer, 4 device launch failed */
} cgx_stats_t;

/* One segment's slow-path measurements, all microseconds.
 * Estimate models (oracle/selector.py):
 *   model 0 (serial replay): t_graph = G + sum_k (delta + d_k) + F
 *   model 1 (the dependency-DAG replay the runtime deploys): list schedule in chain
 *     order, issue_k = (k+1) delta, start_k = max(issue_k, max_{j in deps(k)} fin_j + lambda),
 *     fin_k = start_k + g_k, S = max_k fin_k, t_graph = max(G, S) + F
 *   t_eager (both): S:L404 recurrence over L and d_k; t_copy = t_graph + c_copy; t_ind = t_graph + c_ind.
 * cgx_profile / cgx_profile_ex fill model 1. */
typedef struct {
  int n_kernels;          /* K */
  int ind_available;      /* 0 -> INDIRECT is not a candidate */
  int use_measured;       /* 1 -> decide on the measured totals, else on the estimates */
  int model;              /* estimate model: 0 = serial replay, 1 = dependency-DAG replay */
  double L_us;            /* host launch cost per kernel (eager) */
  double G_us;            /* host cudaGraphLaunch cost */
  double delta_us;        /* model 0: per-node in-graph overhead; model 1: issue interval per node */
  double c_copy_us;       /* COPY rebinding Δ: its bind+launch loop minus its own launch-only loop (>= 0) */
  double c_ind_us;        /* INDIRECT rebinding Δ, likewise against its own exec (>= 0) */
  double F_us;            /* fixed per-replay overhead term (0 unless set) */
  double t_eager_us, t_copy_us, t_ind_us;   /* measured end-to-end per replay (fresh inputs) */
  double d_us[CGX_MAX_PROFILE_KERNELS];     /* work time per kernel in the EAGER stream (eager model) */
  /* model 1 and measurement details */
  double lambda_us;       /* dependency latency: producer exit -> dependent past its wait (median) */
  double span_us;         /* measured device span of the deployed replay (median, traced exec) */
  double t_copy_base_us, t_ind_base_us;     /* the arms' launch-only loops (same exec, no bind) */
  int n_sets;             /* input sets rotated by the bind loops */
  int n_deps;             /* dependency edges in dep_idx */
  int ind_transport;      /* the INDIRECT candidate measured: ROOT_PARAMS or FIRST_NODE, the faster */
  int reserved2;
  double g_us[CGX_MAX_PROFILE_KERNELS];     /* work time per kernel inside the deployed replay */
  int dep_off[CGX_MAX_PROFILE_KERNELS + 1]; /* deps of kernel k: dep_idx[dep_off[k] .. dep_off[k+1]) */
  int dep_idx[CGX_MAX_PROFILE_DEPS];        /* indices j < k */
} cgx_profile_t;

int cgx_version(void);
const char* cgx_last_error(void);

/* ---- chain description -------------------------------------------------------------------- */
int cgx_chain_create(int device, cgx_chain** out);
/* nelems elements of dtype. STATIC: static_dptr is the caller's device buffer (not copied,
 * must outlive the chain); EXTERNAL/INTERNAL: static_dptr must be NULL. slot_out: slot index.
 * EXTERNAL slots are numbered j = 0.. in declaration order (table order). */
int cgx_chain_add_slot(cgx_chain* c, cgx_slot_kind kind, cgx_dtype dtype, uint64_t nelems,
                       void* static_dptr, int* slot_out);
/* Appends a node. The output slot must be INTERNAL (CGX_E_NOT_ELIGIBLE otherwise). */
int cgx_chain_add_node(cgx_chain* c, cgx_op op, const int* in_slots, int n_in, int out_slot,
                       const cgx_attr* attr, int* node_out);
/* Selector unit: an inclusive node range ("independently for each of the CGs"). */
int cgx_chain_mark_segment(cgx_chain* c, int first_node, int last_node);
/* ncclComm_t (caller-owned) used by ALLREDUCE_SUM nodes. */
int cgx_chain_set_nccl(cgx_chain* c, void* nccl_comm);
int cgx_chain_destroy(cgx_chain* c);

/* ---- capture / bind / replay -------------------------------------------------------------- */
/* Slow path: allocate internals/placeholders/table, capture the nodes (stream capture with
 * programmatic-dependent-launch edges), instantiate and upload. cuda_stream: cudaStream_t. */
int cgx_exec_create(cgx_chain* c, cgx_mode mode, void* cuda_stream, cgx_exec** out);
int cgx_exec_create_ex(cgx_chain* c, const cgx_exec_opts* opts, void* cuda_stream, cgx_exec** out);
/* Per replay: bind the fresh external inputs y_j (device pointers, declaration order).
 * COPY enqueues the copy of every y_j whose address differs from its placeholder (SURVEY
 * reading 1); INDIRECT patches the table (8 x N_ext bytes); SETPARAMS rewrites every node that
 * reads an external; EAGER records the pointers; STALE records them at the first bind only. */
int cgx_bind(cgx_exec* e, const void* const* ext_dptrs, int n_ext);
/* Per replay: cudaGraphLaunch (or K eager launches). CGX_E_STATE if never bound. */
int cgx_launch(cgx_exec* e);
/* NEXT-4: device-launched replays (INDIRECT exec with transport DEVICE). Enqueues on the exec's
 * stream ONE host launch of a scheduler graph that runs n_replays replays on the device: replay i
 * binds pointer set i % n_sets — d_ptr_sets is a caller-owned DEVICE array [n_sets][N_ext] of
 * uint64 input addresses, each 16-B aligned, kept valid (with the buffers it points to) until the
 * stream reaches the end of the loop — by copying it into the pointer table, then tail-launches
 * the chain graph and itself (tail launches run in order, each after the previous completes).
 * Returns immediately; the stream's next work starts after the last replay. n_replays = 0 is a
 * no-op. CGX_E_STATE for other execs; CGX_E_NOT_ELIGIBLE when d_ptr_sets is not device memory. */
int cgx_device_loop(cgx_exec* e, const void* d_ptr_sets, int n_sets, uint64_t n_replays);
/* Library-owned device buffer of a slot (internal: shared per chain; external under COPY: the
 * placeholder). nbytes may be NULL. */
int cgx_output(cgx_exec* e, int slot, void** dptr, uint64_t* nbytes);
int cgx_stats(const cgx_exec* e, cgx_stats_t* out);
/* Pack the library-owned output buffers of `slots` (as cgx_output resolves them, in the given
 * order, each at a 16-byte-aligned offset) into the caller-owned DEVICE buffer `dst` (16-B aligned,
 * `cap` bytes) with one kernel enqueued on the exec's stream, after the launch that wrote them;
 * the caller then reads all results with ONE device-to-host copy. *nbytes_out = packed size
 * (written even on CGX_E_SIZE_MISMATCH). At most 64 slots. Errors: CGX_E_INVALID_ARG (NULL, bad or
 * non-library-owned slot, n > 64), CGX_E_SIZE_MISMATCH (cap too small), CGX_E_MISALIGNED, CGX_E_CUDA. */
int cgx_output_gather(cgx_exec* e, const int* slots, int n, void* dst, uint64_t cap, uint64_t* nbytes_out);
/* Parity hooks: the device pointer table (n entries, host copy; synchronises the stream) and the
 * node indices a SETPARAMS bind rewrites. */
int cgx_debug_read_table(const cgx_exec* e, uint64_t* host_out, int n);
int cgx_debug_setparam_nodes(const cgx_exec* e, int* nodes_out, int cap, int* n_out);
int cgx_exec_destroy(cgx_exec* e);

/* ---- NEXT-2: parameter-offset discovery ("byte-pattern match with the known
 * placeholder pointers") ----------------------------------------------------------- */
/* Unique 8-byte-aligned offset of `pattern` in image[0, image_bytes): CGX_E_OFFSET_NOT_FOUND (no
 * match) or CGX_E_OFFSET_AMBIGUOUS (two or more). Pure host function. */
int cgx_find_param_offset(const void* image, uint64_t image_bytes, uint64_t pattern, uint64_t* offset_out);
/* Copy of the parameter image of the launch at exec position `pos` (min(cap, size) bytes; nbytes_out
 * = size) and, optionally, the size cudaFuncGetParamInfo reports for the kernel's parameter 0. */
int cgx_debug_param_image(const cgx_exec* e, int pos, void* buf, uint64_t cap, uint64_t* nbytes_out,
                          uint64_t* param0_size_out);
/* Byte offsets of the external-pointer fields the runtime patches in launch `pos` (EAGER/SETPARAMS/
 * STALE execs, and the by-value first node of FIRST_NODE). */
int cgx_debug_ext_field_offsets(const cgx_exec* e, int pos, uint64_t* offs, int cap, int* n_out);
/* Diagnostics: run GEMM launch `pos` once alone with per-CTA %globaltimer tracing; host_out gets
 * [cta][16] ns stamps (0 entry, 1 setup done, 2 first stage landed, 3 last MMA issued, 4 stores
 * issued, 5 split partial pushed, 6 all splits arrived, 7 exit, 8 accumulator ready, 9 accumulator
 * in registers, 10 staged; 0 = not reached); n_out = CTA count. */
int cgx_debug_gemm_trace(cgx_exec* e, int pos, uint64_t* host_out, int cap, int* n_out);
/* Diagnostics: replay timeline of an exec created with CGX_NODE_TRACE=1 in the environment (chain
 * kernels only): host_out gets [launch][3] %globaltimer ns = (first CTA entry, first CTA past its
 * input wait, last CTA exit) over the replays since the previous call, which then resets them
 * (an untraced launch keeps entry == ready == UINT64_MAX, exit == 0).
 * CGX_E_STATE when tracing is off. Synchronises the exec's stream. */
int cgx_debug_node_trace(cgx_exec* e, uint64_t* host_out, int cap, int* n_out);
/* Diagnostics: per-CTA phase stamps [cta][8] (%globaltimer ns) of the last replay of ATTN_CAUSAL
   launch `pos`, for an exec created with the environment variable CGX_CTA_TRACE=1 (0 entry, 1 past
   the PDL wait, 2 K/V staged, 3 partials published, 4 exit). host_out may be NULL (count only).
   Returns the CTA count, or CGX_E_INVALID_ARG (not an attention launch) / CGX_E_STATE (no trace). */
int cgx_debug_cta_trace(cgx_exec* e, int pos, uint64_t* host_out, int cap);
/* Diagnostics: the chain node each launch position runs (a fused launch reports its last node;
 * cgx_exec_opts.fuse / megakernel make launches fewer than nodes). *n_out = launch count. */
int cgx_debug_launch_nodes(const cgx_exec* e, int* nodes_out, int cap, int* n_out);
/* Diagnostics: per-stage, per-CTA timeline of a megakernel exec (opts.megakernel = 1) created with
 * CGX_MEGA_TRACE=1: host_out gets [stage][cta][8] %globaltimer ns of the last replay (0 = start
 * after the stage's barrier, 1 = end, 2-6 = phase marks of the stage kind, 7 = barrier arrival;
 * unset marks are 0). Returns the entry count (stages x CTAs x 8; host_out == NULL:
 * only the count), or a negative cgx_status (CGX_E_STATE: not a megakernel exec). Synchronises the
 * exec's stream. */
int cgx_debug_mega_trace(cgx_exec* e, uint64_t* host_out, int cap);

/* ---- selective CUDA graphs ---------------------------------------------------------------- */
/* Slow path: measure one segment (index into the marked segments, or -1 = whole chain) in the
 * three candidate modules (eager, graph+copy, graph+PI) with the given inputs; reps timed
 * iterations after warm-up (SURVEY reading 7). Fills every field of *out (model 1). */
int cgx_profile(cgx_chain* c, int segment, const void* const* ext_dptrs, int n_ext, int reps,
                void* cuda_stream, cgx_profile_t* out);
/* The same, rotating over n_sets input sets (ext_sets: n_sets x n_ext DEVICE pointers, row-major,
 * cgx_bind order): every timed bind binds the next set, so each replay reads fresh inputs; the
 * launch-only bases re-launch the last bound set. The DAG model's g_k / lambda / delta / span come
 * from node-traced replays of a separate INDIRECT exec of the segment (CGX_NODE_TRACE stamps;
 * nodes without stamps, e.g. NCCL, take d_k). Errors as cgx_profile. */
int cgx_profile_ex(cgx_chain* c, int segment, const void* const* ext_sets, int n_sets, int n_ext, int reps,
                   void* cuda_stream, cgx_profile_t* out);
/* Pure host function: per segment argmin over [eager, copy, ind]
 * with strict '<' in that order (ties EAGER > COPY > INDIRECT). est_out (3*n_segments doubles,
 * optional) receives the three estimates/totals used (estimates by the profile's model).
 * CGX_E_INVALID_ARG: n_kernels, model, or (model 1) dep_off / dep_idx out of range. */
int cgx_select(const cgx_profile_t* prof, int n_segments, cgx_decision* out, double* est_out);

/* Slow path (measure candidates with the real inputs, deploy one): choose the
 * dependency-DAG capture's stream count. For each candidates[i] (1..64) an exec with *opts
 * (mode must be a graph mode; sync_mode forced to CGX_SYNC_GRAPH, graph_streams = candidates[i])
 * is created on cuda_stream, replayed reps times (bind + launch each, cycling over the n_sets
 * input sets of ext_sets: n_sets x n_ext DEVICE pointers, row-major, same order as cgx_bind),
 * timed with CUDA events (best of three trials) and destroyed. *best_out = the fastest count;
 * us_out (n_cand doubles, optional) = µs per replay of each candidate. The chain must be ready
 * for exec creation (statics set). Errors: CGX_E_INVALID_ARG on bad arguments or an EAGER mode;
 * any exec-create / bind / launch / CUDA error is returned as is (the candidate exec is freed). */
int cgx_tune_graph_streams(cgx_chain* c, const cgx_exec_opts* opts, void* cuda_stream,
                           const void* const* ext_sets, int n_sets, int n_ext, const int* candidates,
                           int n_cand, int reps, int* best_out, double* us_out);

/* ---- measurement helpers ------------------------------------------------------------------ */
/* Single-dispatch floor: median host µs of cudaGraphLaunch of a 1-node
 * empty-kernel graph and of cudaLaunchKernel of an empty kernel on cuda_stream. */
int cgx_dispatch_floor(void* cuda_stream, int reps, double* graph_launch_us, double* kernel_launch_us);
/* Per-node device µs of a bound exec: replays an instrumented capture of its launches with CUDA
 * event-record nodes between consecutive kernels (median over reps; PDL overlap disabled in the
 * instrumented copy). d_us receives min(cap, K) values; n_out = K. */
int cgx_kernel_times(cgx_exec* e, int reps, double* d_us, int cap, int* n_out);
/* In-graph per-node floor: device µs per replay of a captured graph of n_kernels no-op 1-CTA
 * kernels (with use_pdl: the chain kernels' PDL protocol, trigger at entry then wait). */
int cgx_graph_floor(void* cuda_stream, int n_kernels, int use_pdl, int reps, double* us_per_replay);
/* Stream-ordered copy between any two CUDA-visible addresses (cudaMemcpyAsync, kind inferred):
 * used to read library-owned outputs and to stage end-to-end inputs. */
int cgx_copy(void* dst, const void* src, uint64_t nbytes, void* cuda_stream);
/* Fill a device f32 buffer with the synth.splitmix uniform recipe (k*2^-23 - 1) on device. */
int cgx_fill_uniform_f32(void* dptr, uint64_t n, uint64_t seed, uint64_t stream_id, void* cuda_stream);

/* ---- NCCL bootstrap (ncclComm_t for ALLREDUCE_SUM; caller owns it) ------------------------- */
/* Tensor-parallel all-reduce over peer memory (replaces ncclAllReduce for the
 * chain's ALLREDUCE_SUM nodes once set). Every rank owns one region of cgx_peer_buffer_bytes()
 * bytes of device memory, 256-B aligned and ZERO-FILLED before any exec of the chain is created;
 * `bases[r]` is rank r's region as mapped in THIS process (cudaIpc via cgx_ipc_open across
 * processes, or the plain pointer when ranks share a device). An ALLREDUCE_SUM node then runs a
 * one-shot kernel: each rank pushes its partial into slot `rank` of every region (P2P stores over
 * NVLink), publishes a per-CTA generation flag with sys-scope release, waits for every source, and
 * sums the slots in fixed rank order (bit-identical results on all ranks). Region layout: receive
 * data [max_allreduces][2 parity][world][slot] bf16, then flags [max_allreduces][8][256] uint32 —
 * every all-reduce node (ALLREDUCE_SUM or a GEMM with CGX_GEMM_ALLREDUCE) owns two parity buffers,
 * so any exec may hold any subset of the chain's all-reduces. Requirements: n % 8 == 0,
 * n <= max_elems, world <= 8, the chain's all-reduces <= max_allreduces (1..64), and every rank
 * launches the same all-reduces in the same order (captured graphs order each all-reduce after the
 * previous one). Call before the chain's first exec. Errors: CGX_E_INVALID_ARG,
 * CGX_E_MISALIGNED, CGX_E_STATE; exec creation returns CGX_E_UNSUPPORTED past max_allreduces. */
int cgx_peer_buffer_bytes(int world, uint64_t max_elems, int max_allreduces, uint64_t* bytes);
int cgx_chain_set_peers(cgx_chain* c, int rank, int world, void* const* bases, uint64_t max_elems,
                        int max_allreduces);
/* A dedicated zero-filled device allocation (cudaMalloc + memset, synchronised) and its release:
 * use it for peer regions, so the CUDA IPC handle (which maps the whole allocation) maps exactly
 * the region at offset 0 in the peer process. */
int cgx_device_alloc(int device, uint64_t bytes, void** dptr_out);
int cgx_device_free(void* dptr);
/* CUDA IPC helpers for the multi-process case: a device allocation's 64-byte handle, and mapping /
 * unmapping a peer's allocation in this process. */
int cgx_ipc_handle(void* dptr, void* handle_out /* 64 bytes */);
int cgx_ipc_open(const void* handle /* 64 bytes */, void** dptr_out);
int cgx_ipc_close(void* dptr);
/* NVLS (NVSwitch multicast) all-reduce — SURVEY §8(f) NEXT-4, the in-network reduction that
 * replaces the per-rank pushes of the peer path ("additional kernel launches for inter-GPU
 * collective operations"). Every rank binds one region of cgx_mc_buffer_bytes() (rounded to
 * the size cgx_mc_create returns) to a common multicast object and maps it twice: its own copy (uc)
 * and the multicast address (mc). ALLREDUCE_SUM nodes then run k_allreduce_mc: each rank stores its
 * partial into its own copy, the ranks arrive through one multimem.red on a per-CTA counter, and
 * one multimem.ld_reduce (fp32 accumulation in the switch, one bf16 rounding) returns the sum to
 * every rank. Setup order (multi-process): rank 0 cgx_mc_create(world, bytes, device) and
 * cgx_mc_export_fd; the others cgx_mc_import_fd (the file descriptor passed over a Unix socket);
 * EVERY rank cgx_mc_add_device; a barrier; every rank cgx_mc_bind_map; cgx_chain_set_multicast
 * before capture. cgx_mc_supported reports CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED; without it (or
 * without the driver entry points) the calls return CGX_E_UNSUPPORTED. A lost rank is reported as
 * CGX_E_DEVICE by the next cgx_launch, as for the peer path. cgx_mc_release(uc) unmaps and frees one
 * rank's region (after every exec using it is destroyed). */
int cgx_mc_supported(int device, int* supported);
int cgx_mc_buffer_bytes(uint64_t max_elems, int max_allreduces, uint64_t* bytes);
int cgx_mc_create(int world, uint64_t bytes, int device, uint64_t* handle_out, uint64_t* size_out);
int cgx_mc_export_fd(uint64_t handle, int* fd_out);
int cgx_mc_import_fd(int fd, uint64_t* handle_out);
int cgx_mc_add_device(uint64_t handle, int device);
int cgx_mc_bind_map(uint64_t handle, int device, uint64_t size, void** uc_out, void** mc_out);
int cgx_mc_release(void* uc);
int cgx_chain_set_multicast(cgx_chain* c, int world, void* uc, void* mc, uint64_t max_elems, int max_allreduces);
int cgx_nccl_unique_id(void* id_out /* 128 bytes */);
int cgx_nccl_comm_init(int nranks, int rank, const void* id /* 128 bytes */, int device, void** comm_out);
int cgx_nccl_comm_destroy(void* comm);

#ifdef __cplusplus
}
#endif
#endif /* CGX_H_ */
