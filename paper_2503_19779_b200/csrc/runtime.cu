// cgx runtime: chain description, capture/instantiate/replay, the four rebinding arms, the
// selector, and measurement helpers. Implements include/cgx.h.
//
// Design (B200-first):
//  * One by-value parameter struct per kernel node. A node's parameter image is kept on the host
//    (Launch::args) together with the byte offsets of its external pointer fields, so
//      EAGER      patches the images and launches K kernels from the host,
//      SETPARAMS  patches the images and calls cudaGraphExecKernelNodeSetParams per node,
//      STALE      does that once, at the first bind (recorded by value),
//      COPY       captures placeholder addresses and launches one multi-tensor copy kernel per
//                 bind,
//      INDIRECT   captures table indices; bind patches the device pointer table.
//  * Capture = stream capture on a private stream with programmatic-dependent-launch edges
//    (so NCCL collectives can be captured too); node handles are taken from
//    cudaStreamGetCaptureInfo right after each launch.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/cgx.h"
#include "cgx_args.h"
#include "cgx_decoder.h"
#include "cgx_mega.h"
#include "cgx_prelude.h"

using namespace cgx;

// ============================================================================ errors
static thread_local std::string g_err;
// cgx_profile_ex: the next exec created on this thread stamps the node timeline (as CGX_NODE_TRACE=1)
static thread_local bool g_force_trace = false;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
static int cuda_fail(cudaError_t e, const char* what, int line) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s failed (runtime.cu:%d): %s (%s)", what, line, cudaGetErrorString(e),
           cudaGetErrorName(e));
  g_err = buf;
  return CGX_E_CUDA;
}
#define CK(expr)                                                   \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr, __LINE__);  \
  } while (0)
#define CKS(expr)                                                  \
  do {                                                             \
    int _s = (expr);                                               \
    if (_s != CGX_OK) return _s;                                   \
  } while (0)

extern "C" int cgx_version(void) { return CGX_ABI_VERSION; }
extern "C" const char* cgx_last_error(void) { return g_err.c_str(); }

// ============================================================================ small utilities
namespace {

struct AlignedBuf {  // 64-B aligned byte buffer (CUtensorMap params need 64-B alignment)
  uint8_t* p = nullptr;
  size_t n = 0;
  AlignedBuf() = default;
  explicit AlignedBuf(size_t bytes) { reset(bytes); }
  AlignedBuf(const AlignedBuf&) = delete;
  AlignedBuf& operator=(const AlignedBuf&) = delete;
  AlignedBuf(AlignedBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  AlignedBuf& operator=(AlignedBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    return *this;
  }
  void reset(size_t bytes) {
    free(p);
    n = bytes;
    p = static_cast<uint8_t*>(aligned_alloc(64, ((bytes + 63) / 64) * 64));
    memset(p, 0, n);
  }
  ~AlignedBuf() { free(p); }
};

inline double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

inline uint64_t host_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

}  // namespace

// ============================================================================ chain
struct Slot {
  cgx_slot_kind kind;
  cgx_dtype dtype;
  uint64_t nelems, nbytes;
  void* static_ptr;   // STATIC
  void* buf;          // INTERNAL (chain arena)
  int ext_j;          // EXTERNAL index (declaration order), else -1
};

struct Node {
  cgx_op op;
  int in[CGX_MAX_IN];
  int n_in;
  int out;
  cgx_attr attr;
};

struct cgx_chain {
  int device = 0;
  std::vector<Slot> slots;
  std::vector<Node> nodes;
  std::vector<std::pair<int, int>> segments;
  std::vector<int> ext_slots;   // j -> slot
  void* nccl = nullptr;
  // peer all-reduce (cgx_chain_set_peers): rank, world, every rank's region, generation counters
  int peer_rank = -1, peer_world = 0;
  uint64_t peer_max_elems = 0;
  int peer_max_ar = 0;          // all-reduce nodes the regions have receive buffers for
  std::vector<void*> peer_base;
  uint32_t* peer_counters = nullptr;
  // NVLS / multicast all-reduce (cgx_chain_set_multicast): this rank's copy and the multicast
  // mapping of the region bound to the node's multicast object
  int mc_world = 0;
  void* mc_uc = nullptr;
  void* mc_mc = nullptr;
  uint64_t mc_max_elems = 0;
  int mc_max_ar = 0;
  void* arena = nullptr;        // internal buffers
  bool allocated = false;
  int live_execs = 0;
};

static size_t dtype_size(cgx_dtype d) { return d == CGX_F32 ? 4 : 2; }

// Op families. Elementwise kernels (k_elem_f32 / k_elem_bf16); everything that takes the ElemArgs
// parameter block (elementwise, REDUCE_SUM, TRANSPOSE): table-indexed operands, dataflow flags.
static bool is_elemwise(cgx_op op) {
  return op == CGX_OP_ADD || op == CGX_OP_MUL || op == CGX_OP_SCALE_IMM || op == CGX_OP_COPY || op == CGX_OP_SCALE_T ||
         op == CGX_OP_SUB || op == CGX_OP_AXPY || op == CGX_OP_GELU || op == CGX_OP_GELU_BWD;
}
static bool uses_elem_args(cgx_op op) {
  return is_elemwise(op) || op == CGX_OP_REDUCE_SUM || op == CGX_OP_TRANSPOSE;
}
static bool elem_binary(cgx_op op) {
  return op == CGX_OP_ADD || op == CGX_OP_MUL || op == CGX_OP_SUB || op == CGX_OP_AXPY || op == CGX_OP_GELU_BWD;
}

extern "C" int cgx_chain_create(int device, cgx_chain** out) {
  if (!out) return fail(CGX_E_INVALID_ARG, "cgx_chain_create: out is NULL");
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(CGX_E_INVALID_ARG, "cgx_chain_create: bad device");
  auto* c = new cgx_chain();
  c->device = device;
  *out = c;
  return CGX_OK;
}

extern "C" int cgx_chain_add_slot(cgx_chain* c, cgx_slot_kind kind, cgx_dtype dtype, uint64_t nelems,
                                  void* static_dptr, int* slot_out) {
  if (!c) return fail(CGX_E_INVALID_ARG, "add_slot: chain is NULL");
  if (c->allocated) return fail(CGX_E_STATE, "add_slot: chain already captured");
  if (kind < CGX_SLOT_EXTERNAL || kind > CGX_SLOT_INTERNAL) return fail(CGX_E_INVALID_ARG, "add_slot: kind");
  if (dtype != CGX_F32 && dtype != CGX_BF16) return fail(CGX_E_INVALID_ARG, "add_slot: dtype");
  if (nelems == 0) return fail(CGX_E_INVALID_ARG, "add_slot: nelems == 0");
  if ((kind == CGX_SLOT_STATIC) != (static_dptr != nullptr))
    return fail(CGX_E_INVALID_ARG, "add_slot: static_dptr must be given for STATIC slots only");
  if (static_dptr && (reinterpret_cast<uintptr_t>(static_dptr) & 15))
    return fail(CGX_E_MISALIGNED, "add_slot: static buffer not 16-byte aligned");
  Slot s{kind, dtype, nelems, nelems * dtype_size(dtype), static_dptr, nullptr, -1};
  if (kind == CGX_SLOT_EXTERNAL) {
    s.ext_j = (int)c->ext_slots.size();
    c->ext_slots.push_back((int)c->slots.size());
  }
  c->slots.push_back(s);
  if (slot_out) *slot_out = (int)c->slots.size() - 1;
  return CGX_OK;
}

static int check_node(const cgx_chain* c, const Node& n) {
  auto S = [&](int i) -> const Slot& { return c->slots[n.in[i]]; };
  const Slot& o = c->slots[n.out];
  const cgx_attr& a = n.attr;
  auto need = [&](bool ok, const char* m) { return ok ? CGX_OK : fail(CGX_E_SIZE_MISMATCH, m); };
  switch (n.op) {
    case CGX_OP_SUB:
    case CGX_OP_AXPY:
    case CGX_OP_GELU:
    case CGX_OP_GELU_BWD:
      if (o.dtype != CGX_BF16) return fail(CGX_E_UNSUPPORTED, "sub/axpy/gelu/gelu_bwd: bf16 only");
      [[fallthrough]];
    case CGX_OP_ADD:
    case CGX_OP_MUL:
    case CGX_OP_SCALE_IMM:
    case CGX_OP_COPY: {
      int nin = elem_binary(n.op) ? 2 : 1;
      if (n.n_in != nin) return fail(CGX_E_INVALID_ARG, "elementwise: wrong number of inputs");
      for (int i = 0; i < nin; ++i) {
        if (S(i).dtype != o.dtype) return fail(CGX_E_UNSUPPORTED, "elementwise: mixed dtypes");
        CKS(need(S(i).nelems >= a.n, "elementwise: input shorter than attr.n"));
      }
      return need(o.nelems >= a.n, "elementwise: output shorter than attr.n");
    }
    case CGX_OP_TRANSPOSE:
      if (n.n_in != 1) return fail(CGX_E_INVALID_ARG, "transpose: one input");
      if (S(0).dtype != CGX_BF16 || o.dtype != CGX_BF16) return fail(CGX_E_UNSUPPORTED, "transpose: bf16 only");
      CKS(need(a.cols > 0 && a.n % a.cols == 0, "transpose: n must be rows x cols"));
      return need(S(0).nelems >= a.n && o.nelems >= a.n, "transpose: shape");
    case CGX_OP_SCALE_T:
      if (n.n_in != 2) return fail(CGX_E_INVALID_ARG, "scale_t: inputs a, s");
      if (S(0).dtype != CGX_F32 || S(1).dtype != CGX_F32 || o.dtype != CGX_F32)
        return fail(CGX_E_UNSUPPORTED, "scale_t: f32 only");
      CKS(need(S(0).nelems >= a.n && o.nelems >= a.n, "scale_t: shape"));
      return CGX_OK;
    case CGX_OP_REDUCE_SUM:
      if (n.n_in != 1) return fail(CGX_E_INVALID_ARG, "reduce: one input");
      if (S(0).dtype != CGX_F32 || o.dtype != CGX_F32) return fail(CGX_E_UNSUPPORTED, "reduce: f32 only");
      if (a.cols == 0 || a.cols % 4 || a.n % a.cols) return fail(CGX_E_SIZE_MISMATCH, "reduce: cols must divide n, cols % 4 == 0");
      CKS(need(S(0).nelems >= a.n, "reduce: input shorter than n"));
      return need(o.nelems >= a.n / a.cols, "reduce: output shorter than n/cols");
    case CGX_OP_LAYERNORM:
      if (n.n_in != 3) return fail(CGX_E_INVALID_ARG, "layernorm: inputs x, gamma, beta");
      for (int i = 0; i < 3; ++i)
        if (S(i).dtype != CGX_BF16) return fail(CGX_E_UNSUPPORTED, "layernorm: bf16 only");
      if (o.dtype != CGX_BF16) return fail(CGX_E_UNSUPPORTED, "layernorm: bf16 only");
      CKS(need(a.rows > 0 && a.cols > 0 && a.cols % 8 == 0, "layernorm: rows, cols > 0 and cols % 8 == 0"));
      // k_layernorm keeps the row in registers: 8 x 16 B per lane x 32 lanes = 2048 bf16 columns
      if (a.cols > kLnMaxCols) return fail(CGX_E_UNSUPPORTED, "layernorm: cols > 2048 (row held in one warp's registers)");
      CKS(need(S(0).nelems >= (uint64_t)a.rows * a.cols && o.nelems >= (uint64_t)a.rows * a.cols, "layernorm: shape"));
      return need(S(1).nelems >= a.cols && S(2).nelems >= a.cols, "layernorm: gamma/beta shape");
    case CGX_OP_GEMM_BF16: {
      int nin = (a.flags & CGX_GEMM_RESIDUAL) ? 4 : 3;
      if (n.n_in != nin) return fail(CGX_E_INVALID_ARG, "gemm: inputs A, W, bias(, residual)");
      for (int i = 0; i < nin; ++i)
        if (S(i).dtype != CGX_BF16) return fail(CGX_E_UNSUPPORTED, "gemm: bf16 only");
      CKS(need(S(0).nelems >= (uint64_t)a.M * a.K && S(1).nelems >= (uint64_t)a.N * a.K &&
                   S(2).nelems >= a.N && o.nelems >= (uint64_t)a.M * a.N, "gemm: shape"));
      return decoder_gemm_supported(a.M, a.N, a.K) ? CGX_OK
                                                   : fail(CGX_E_UNSUPPORTED, "gemm: shape not supported by the tcgen05 kernel");
    }
    case CGX_OP_ATTN_CAUSAL:
      if (n.n_in != 1) return fail(CGX_E_INVALID_ARG, "attention: one input qkv");
      if (S(0).dtype != CGX_BF16 || o.dtype != CGX_BF16) return fail(CGX_E_UNSUPPORTED, "attention: bf16 qkv and output only");
      CKS(need(S(0).nelems >= (uint64_t)a.T * 3 * a.H * a.D && o.nelems >= (uint64_t)a.T * a.H * a.D, "attention: shape"));
      return decoder_attn_supported(a.T, a.H, a.D) ? CGX_OK : fail(CGX_E_UNSUPPORTED, "attention: shape");
    case CGX_OP_ALLREDUCE_SUM:
      if (n.n_in != 1) return fail(CGX_E_INVALID_ARG, "allreduce: one input");
      if (S(0).dtype != CGX_BF16 || o.dtype != CGX_BF16) return fail(CGX_E_UNSUPPORTED, "allreduce: bf16 only");
      return need(S(0).nelems >= a.n && o.nelems >= a.n, "allreduce: shape");
  }
  return fail(CGX_E_INVALID_ARG, "unknown op");
}

extern "C" int cgx_chain_add_node(cgx_chain* c, cgx_op op, const int* in_slots, int n_in, int out_slot,
                                  const cgx_attr* attr, int* node_out) {
  if (!c) return fail(CGX_E_INVALID_ARG, "add_node: chain is NULL");
  if (c->allocated) return fail(CGX_E_STATE, "add_node: chain already captured");
  if (n_in < 0 || n_in > CGX_MAX_IN || (n_in > 0 && !in_slots)) return fail(CGX_E_INVALID_ARG, "add_node: inputs");
  if (out_slot < 0 || out_slot >= (int)c->slots.size()) return fail(CGX_E_INVALID_ARG, "add_node: out slot");
  Node n{};
  n.op = op;
  n.n_in = n_in;
  n.out = out_slot;
  if (attr) n.attr = *attr;
  for (int i = 0; i < n_in; ++i) {
    if (in_slots[i] < 0 || in_slots[i] >= (int)c->slots.size()) return fail(CGX_E_INVALID_ARG, "add_node: in slot");
    n.in[i] = in_slots[i];
  }
  if (c->slots[out_slot].kind != CGX_SLOT_INTERNAL)
    return fail(CGX_E_NOT_ELIGIBLE, "add_node: output must be an INTERNAL slot (no writes to inputs/weights)");
  if ((uses_elem_args(op) || op == CGX_OP_ALLREDUCE_SUM) && n.attr.n == 0 && n_in > 0)
    n.attr.n = c->slots[n.in[0]].nelems;
  if (op == CGX_OP_REDUCE_SUM && n.attr.cols == 0) n.attr.cols = 256;
  CKS(check_node(c, n));
  c->nodes.push_back(n);
  if (node_out) *node_out = (int)c->nodes.size() - 1;
  return CGX_OK;
}

extern "C" int cgx_chain_mark_segment(cgx_chain* c, int first, int last) {
  if (!c || first < 0 || last < first || last >= (int)c->nodes.size())
    return fail(CGX_E_INVALID_ARG, "mark_segment: bad range");
  c->segments.push_back({first, last});
  return CGX_OK;
}

extern "C" int cgx_chain_set_nccl(cgx_chain* c, void* comm) {
  if (!c) return fail(CGX_E_INVALID_ARG, "set_nccl: chain is NULL");
  c->nccl = comm;
  return CGX_OK;
}

// Peer all-reduce region of one rank: receive data [max_ar][2 parity][world][slot] bf16 (slots
// 256-B aligned), then the flag array [max_ar][kArMaxWorld][kArMaxCtas] uint32. Every all-reduce
// node owns its two parity buffers, so buffer reuse never depends on which other all-reduces an
// exec runs or in which order execs are launched (node i's parity-p buffer is rewritten at its
// generation g + 2, after every rank has published generation g + 1, i.e. finished reading g).
static uint64_t peer_slot_elems(uint64_t max_elems) { return (max_elems + 127) / 128 * 128; }
static uint64_t peer_node_elems(int world, uint64_t max_elems) {
  return 2ull * (uint64_t)world * peer_slot_elems(max_elems);
}
static uint64_t peer_flag_offset(int world, uint64_t max_elems, int max_ar) {
  return (uint64_t)max_ar * peer_node_elems(world, max_elems) * 2;
}

static bool is_allreduce(const Node& n) {
  return n.op == CGX_OP_ALLREDUCE_SUM || (n.op == CGX_OP_GEMM_BF16 && (n.attr.flags & CGX_GEMM_ALLREDUCE));
}

// Position of node k among the chain's all-reduces (ALLREDUCE_SUM nodes and GEMMs with the fused
// all-reduce), and their total: the generation / parity sequence every rank shares.
static void ar_position(const cgx_chain* c, int k, int* index, int* total) {
  int i = 0, t = 0;
  for (size_t q = 0; q < c->nodes.size(); ++q) {
    const Node& n = c->nodes[q];
    if (is_allreduce(n)) {
      if ((int)q < k) ++i;
      ++t;
    }
  }
  *index = i;
  *total = t;
}

extern "C" int cgx_peer_buffer_bytes(int world, uint64_t max_elems, int max_allreduces, uint64_t* bytes) {
  if (world < 1 || world > kArMaxWorld || !bytes) return fail(CGX_E_INVALID_ARG, "peer_buffer_bytes: world 1..8");
  if (max_allreduces < 1 || max_allreduces > kArMaxNodes)
    return fail(CGX_E_INVALID_ARG, "peer_buffer_bytes: max_allreduces 1..64");
  *bytes = peer_flag_offset(world, max_elems, max_allreduces) +
           sizeof(uint32_t) * (uint64_t)max_allreduces * kArMaxWorld * kArMaxCtas;
  return CGX_OK;
}

extern "C" int cgx_chain_set_peers(cgx_chain* c, int rank, int world, void* const* bases, uint64_t max_elems,
                                   int max_allreduces) {
  if (!c || !bases || world < 1 || world > kArMaxWorld || rank < 0 || rank >= world || max_elems == 0 ||
      max_allreduces < 1 || max_allreduces > kArMaxNodes)
    return fail(CGX_E_INVALID_ARG, "set_peers: bad argument");
  if (c->allocated) return fail(CGX_E_STATE, "set_peers: chain already captured");
  for (int r = 0; r < world; ++r) {
    if (!bases[r]) return fail(CGX_E_INVALID_ARG, "set_peers: NULL region");
    if (reinterpret_cast<uintptr_t>(bases[r]) % 256) return fail(CGX_E_MISALIGNED, "set_peers: region not 256-B aligned");
  }
  CK(cudaSetDevice(c->device));
  if (!c->peer_counters) {
    CK(cudaMalloc(&c->peer_counters, sizeof(uint32_t) * kArMaxNodes * kArMaxCtas));
    CK(cudaMemset(c->peer_counters, 0, sizeof(uint32_t) * kArMaxNodes * kArMaxCtas));
  }
  c->peer_rank = rank;
  c->peer_world = world;
  c->peer_max_elems = max_elems;
  c->peer_max_ar = max_allreduces;
  c->peer_base.assign(bases, bases + world);
  return CGX_OK;
}

// ---------------------------------------------------------------- NVLS multicast regions
// Region of one rank, bound to the node's multicast object at the same offsets on every rank:
// data [max_ar][2 parity][slot] bf16, then (256-B aligned) the arrival counters [max_ar][kArMaxCtas]
// uint32 (k_allreduce_mc). Driver API (virtual memory management + multicast objects) through
// cudaGetDriverEntryPoint: the library links only the runtime.
static uint64_t mc_slot_elems(uint64_t max_elems) { return (max_elems + 127) / 128 * 128; }
static uint64_t mc_flag_offset(uint64_t max_elems, int max_ar) {
  return ((uint64_t)max_ar * 2 * mc_slot_elems(max_elems) * sizeof(uint16_t) + 255) / 256 * 256;
}
template <typename F>
static F drv_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(fn);
}
#define DRV(fnname, ...)                                                                      \
  do {                                                                                        \
    static const auto f_ = drv_fn<decltype(&::fnname)>(#fnname);                              \
    if (!f_) return fail(CGX_E_UNSUPPORTED, #fnname ": driver entry point unavailable");      \
    const CUresult r_ = f_(__VA_ARGS__);                                                      \
    if (r_ != CUDA_SUCCESS) return fail(CGX_E_CUDA, std::string(#fnname " failed: CUresult ") + std::to_string((int)r_)); \
  } while (0)

namespace {
struct McMapping {
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr uc = 0, mcp = 0;
  uint64_t size = 0;
  int device = 0;
};
std::vector<McMapping> g_mc_maps;
std::mutex g_mc_mu;
}  // namespace

// Undo the first `stage` steps of cgx_mc_bind_map (6 = all of them); release_mc also drops this
// process's reference to the multicast object. Returns the first failure.
static int mc_undo(const McMapping& m, int stage, bool release_mc = false) {
  int st = CGX_OK;
  auto step = [&](int r) { if (st == CGX_OK && r != CGX_OK) st = r; };
  auto unmap = [&](CUdeviceptr p) -> int { DRV(cuMemUnmap, p, (size_t)m.size); return CGX_OK; };
  auto vfree = [&](CUdeviceptr p) -> int { DRV(cuMemAddressFree, p, (size_t)m.size); return CGX_OK; };
  auto unbind = [&]() -> int { DRV(cuMulticastUnbind, m.mc, (CUdevice)m.device, (size_t)0, (size_t)m.size); return CGX_OK; };
  auto rel = [&](CUmemGenericAllocationHandle h) -> int { DRV(cuMemRelease, h); return CGX_OK; };
  if (stage >= 6) step(unmap(m.mcp));
  if (stage >= 5) step(vfree(m.mcp));
  if (stage >= 4) step(unmap(m.uc));
  if (stage >= 3) step(vfree(m.uc));
  if (stage >= 2) step(unbind());
  if (stage >= 1) step(rel(m.mem));
  if (release_mc) step(rel(m.mc));
  return st;
}

extern "C" int cgx_mc_supported(int device, int* supported) {
  if (!supported) return fail(CGX_E_INVALID_ARG, "mc_supported: NULL");
  *supported = 0;
  int v = 0;
  DRV(cuDeviceGetAttribute, &v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)device);
  *supported = v;
  return CGX_OK;
}

extern "C" int cgx_mc_buffer_bytes(uint64_t max_elems, int max_allreduces, uint64_t* bytes) {
  if (!bytes || max_elems == 0 || max_allreduces < 1 || max_allreduces > kArMaxNodes)
    return fail(CGX_E_INVALID_ARG, "mc_buffer_bytes: max_elems > 0, max_allreduces 1..64");
  *bytes = mc_flag_offset(max_elems, max_allreduces) + sizeof(uint32_t) * (uint64_t)max_allreduces * kArMaxCtas;
  return CGX_OK;
}

// Multicast object for `world` devices, sized up to the multicast and allocation granularities
// (*size_out: the size every rank binds and maps). Exportable as a POSIX file descriptor.
extern "C" int cgx_mc_create(int world, uint64_t bytes, int device, uint64_t* handle_out, uint64_t* size_out) {
  if (!handle_out || !size_out || world < 1 || world > kArMaxWorld || bytes == 0)
    return fail(CGX_E_INVALID_ARG, "mc_create: bad argument");
  CUmulticastObjectProp mp{};
  mp.numDevices = (unsigned)world;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes;
  size_t g_mc = 0, g_al = 0;
  DRV(cuMulticastGetGranularity, &g_mc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  DRV(cuMemGetAllocationGranularity, &g_al, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  const uint64_t g = std::max<uint64_t>(g_mc, g_al);
  mp.size = (bytes + g - 1) / g * g;
  CUmemGenericAllocationHandle h = 0;
  DRV(cuMulticastCreate, &h, &mp);
  *handle_out = (uint64_t)h;
  *size_out = mp.size;
  return CGX_OK;
}

extern "C" int cgx_mc_export_fd(uint64_t handle, int* fd_out) {
  if (!fd_out) return fail(CGX_E_INVALID_ARG, "mc_export_fd: NULL");
  int fd = -1;
  DRV(cuMemExportToShareableHandle, (void*)&fd, (CUmemGenericAllocationHandle)handle,
      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0ull);
  *fd_out = fd;
  return CGX_OK;
}

extern "C" int cgx_mc_import_fd(int fd, uint64_t* handle_out) {
  if (!handle_out || fd < 0) return fail(CGX_E_INVALID_ARG, "mc_import_fd: bad argument");
  CUmemGenericAllocationHandle h = 0;
  DRV(cuMemImportFromShareableHandle, &h, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  *handle_out = (uint64_t)h;
  return CGX_OK;
}

// Every rank adds its device before ANY rank binds memory (a barrier between the two calls).
extern "C" int cgx_mc_add_device(uint64_t handle, int device) {
  CK(cudaSetDevice(device));
  CK(cudaFree(nullptr));   // (the device's primary context exists before the driver calls)
  DRV(cuMulticastAddDevice, (CUmemGenericAllocationHandle)handle, (CUdevice)device);
  return CGX_OK;
}

// This rank's physical region (size bytes on `device`), bound to the multicast object at offset 0,
// mapped twice: *uc_out = this rank's copy, *mc_out = the multicast address (multimem.* only).
// Zero-filled. Released by cgx_mc_release(uc).
extern "C" int cgx_mc_bind_map(uint64_t handle, int device, uint64_t size, void** uc_out, void** mc_out) {
  if (!uc_out || !mc_out || size == 0) return fail(CGX_E_INVALID_ARG, "mc_bind_map: bad argument");
  CK(cudaSetDevice(device));
  McMapping m;
  m.mc = (CUmemGenericAllocationHandle)handle;
  m.size = size;
  m.device = device;
  // every step acquired is undone if a later one fails (no leaked physical memory, bindings or VA)
  int stage = 0;
  const int st = [&]() -> int {
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    DRV(cuMemCreate, &m.mem, (size_t)size, &ap, 0ull);
    stage = 1;
    DRV(cuMulticastBindMem, m.mc, (size_t)0, m.mem, (size_t)0, (size_t)size, 0ull);
    stage = 2;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    DRV(cuMemAddressReserve, &m.uc, (size_t)size, (size_t)0, (CUdeviceptr)0, 0ull);
    stage = 3;
    DRV(cuMemMap, m.uc, (size_t)size, (size_t)0, m.mem, 0ull);
    stage = 4;
    DRV(cuMemSetAccess, m.uc, (size_t)size, &acc, (size_t)1);
    DRV(cuMemAddressReserve, &m.mcp, (size_t)size, (size_t)0, (CUdeviceptr)0, 0ull);
    stage = 5;
    DRV(cuMemMap, m.mcp, (size_t)size, (size_t)0, m.mc, 0ull);
    stage = 6;
    DRV(cuMemSetAccess, m.mcp, (size_t)size, &acc, (size_t)1);
    CK(cudaMemset(reinterpret_cast<void*>(m.uc), 0, size));
    CK(cudaDeviceSynchronize());
    return CGX_OK;
  }();
  if (st != CGX_OK) {
    const std::string err = g_err;   // (the undo below must not overwrite the first failure)
    mc_undo(m, stage);
    g_err = err;
    return st;
  }
  *uc_out = reinterpret_cast<void*>(m.uc);
  *mc_out = reinterpret_cast<void*>(m.mcp);
  std::lock_guard<std::mutex> lk(g_mc_mu);
  g_mc_maps.push_back(m);
  return CGX_OK;
}

extern "C" int cgx_mc_release(void* uc) {
  McMapping m;
  {
    std::lock_guard<std::mutex> lk(g_mc_mu);
    size_t i = 0;
    while (i < g_mc_maps.size() && reinterpret_cast<void*>(g_mc_maps[i].uc) != uc) ++i;
    if (i == g_mc_maps.size()) return fail(CGX_E_INVALID_ARG, "mc_release: not a cgx_mc_bind_map region");
    m = g_mc_maps[i];
    g_mc_maps.erase(g_mc_maps.begin() + (long)i);
  }
  CK(cudaSetDevice(m.device));
  CK(cudaDeviceSynchronize());
  return mc_undo(m, 6, true);
}

extern "C" int cgx_chain_set_multicast(cgx_chain* c, int world, void* uc, void* mc, uint64_t max_elems,
                                       int max_allreduces) {
  if (!c || !uc || !mc || world < 1 || world > kArMaxWorld || max_elems == 0 || max_allreduces < 1 ||
      max_allreduces > kArMaxNodes)
    return fail(CGX_E_INVALID_ARG, "set_multicast: bad argument");
  if (c->allocated) return fail(CGX_E_STATE, "set_multicast: chain already captured");
  if (reinterpret_cast<uintptr_t>(uc) % 256 || reinterpret_cast<uintptr_t>(mc) % 256)
    return fail(CGX_E_MISALIGNED, "set_multicast: region not 256-B aligned");
  CK(cudaSetDevice(c->device));
  if (!c->peer_counters) {
    CK(cudaMalloc(&c->peer_counters, sizeof(uint32_t) * kArMaxNodes * kArMaxCtas));
    CK(cudaMemset(c->peer_counters, 0, sizeof(uint32_t) * kArMaxNodes * kArMaxCtas));
  }
  c->mc_world = world;
  c->mc_uc = uc;
  c->mc_mc = mc;
  c->mc_max_elems = max_elems;
  c->mc_max_ar = max_allreduces;
  return CGX_OK;
}

// Dedicated zero-filled device allocation (peer regions): its CUDA IPC handle maps exactly this
// buffer at offset 0 in a peer process (a sub-allocation of a caching allocator would not).
extern "C" int cgx_device_alloc(int device, uint64_t bytes, void** dptr_out) {
  if (!dptr_out || bytes == 0) return fail(CGX_E_INVALID_ARG, "device_alloc: bad argument");
  CK(cudaSetDevice(device));
  void* p = nullptr;
  CK(cudaMalloc(&p, bytes));
  const cudaError_t ce = cudaMemset(p, 0, bytes);
  if (ce != cudaSuccess) {
    cudaFree(p);
    return cuda_fail(ce, "device_alloc memset", __LINE__);
  }
  CK(cudaDeviceSynchronize());
  *dptr_out = p;
  return CGX_OK;
}
extern "C" int cgx_device_free(void* dptr) {
  if (!dptr) return CGX_OK;
  CK(cudaFree(dptr));
  return CGX_OK;
}

// CUDA IPC (multi-process TP): export a device allocation's handle (64 bytes) / map a peer's.
extern "C" int cgx_ipc_handle(void* dptr, void* handle_out) {
  if (!dptr || !handle_out) return fail(CGX_E_INVALID_ARG, "ipc_handle: NULL");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, dptr));
  memcpy(handle_out, &h, sizeof(h));
  return CGX_OK;
}
extern "C" int cgx_ipc_open(const void* handle, void** dptr_out) {
  if (!handle || !dptr_out) return fail(CGX_E_INVALID_ARG, "ipc_open: NULL");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  CK(cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return CGX_OK;
}
extern "C" int cgx_ipc_close(void* dptr) {
  if (!dptr) return CGX_OK;
  CK(cudaIpcCloseMemHandle(dptr));
  return CGX_OK;
}

static int chain_allocate(cgx_chain* c) {
  if (c->allocated) return CGX_OK;
  CK(cudaSetDevice(c->device));
  size_t total = 0;
  for (auto& s : c->slots)
    if (s.kind == CGX_SLOT_INTERNAL) total += ceil_div(s.nbytes, 256) * 256;
  if (total) {
    CK(cudaMalloc(&c->arena, total));
    CK(cudaMemset(c->arena, 0, total));
  }
  size_t off = 0;
  for (auto& s : c->slots)
    if (s.kind == CGX_SLOT_INTERNAL) {
      s.buf = static_cast<char*>(c->arena) + off;
      off += ceil_div(s.nbytes, 256) * 256;
    }
  c->allocated = true;
  return CGX_OK;
}

extern "C" int cgx_chain_destroy(cgx_chain* c) {
  if (!c) return CGX_OK;
  if (c->live_execs) return fail(CGX_E_STATE, "chain_destroy: execs still alive");
  if (c->arena) cudaFree(c->arena);
  if (c->peer_counters) cudaFree(c->peer_counters);
  delete c;
  return CGX_OK;
}

// ============================================================================ exec
namespace {

enum LaunchKind { LK_KERNEL = 0, LK_NCCL = 1 };

struct PtrField {  // a pointer-valued field in a node's param image
  size_t off;      // byte offset of the void* field
  size_t tidx_off; // byte offset of the int32 table-index field (or SIZE_MAX)
  int ext_j;       // external index
};

struct Launch {
  LaunchKind kind = LK_KERNEL;
  int node = -1;
  const void* func = nullptr;
  dim3 grid, block;
  size_t smem = 0;
  bool pdl = true;
  AlignedBuf args;
  std::vector<PtrField> ext;  // external operand fields
  size_t tw_ptr_off = 0;      // T5 first node: byte offset of the by-value pointer array (0 = none)
  cudaGraphNode_t gnode[2] = {nullptr, nullptr};
  unsigned cluster_z = 1;                 // thread-block cluster (1, 1, z) (split-K GEMM)
  bool dev_updatable = false;             // T7: consumer patched by the prelude node
  int prio = 0;                           // launch priority (0 = default; CGX_DAG_PRIO experiment)
  bool coop = false;                      // cooperative launch (co-resident grid: the megakernel)
  bool mega = false;                      // the persistent decoder executor (args = MegaArgs)
  int pre_node = -1;                      // capture-time fusion: a node this launch runs first (the ADD
                                          // of an ADD -> LAYERNORM launch, the LN of an LN -> GEMM launch)
  cudaGraphDeviceNode_t dev_node = nullptr;
  // NCCL
  const void* nc_in = nullptr;
  void* nc_out = nullptr;
  size_t nc_count = 0;
};

}  // namespace

struct cgx_exec {
  cgx_chain* c = nullptr;
  cgx_exec_opts o{};
  cudaStream_t s = nullptr;       // replay stream (caller's)
  cudaStream_t cs = nullptr;      // private capture stream
  int first = 0, last = -1;       // node range (inclusive)
  std::vector<Launch> L;
  int n_graphs = 0;
  cudaGraph_t g[2] = {nullptr, nullptr};
  cudaGraphExec_t ge[2] = {nullptr, nullptr};
  uint32_t graph_nodes = 0;
  std::vector<int> ext_read;      // externals read by nodes in range (ordered by j)
  std::vector<const void*> cur;   // currently bound pointers (by j)
  bool bound = false;
  bool stale_frozen = false;
  bool launched_since_bind = true;   // T4: a bind before any launch reuses the pending slot
  uint64_t seq = 0;               // binds so far
  std::unordered_set<uintptr_t> validated;
  cgx_stats_t st{};
  // COPY
  std::vector<void*> ph;          // by j (nullptr if not read)
  void* ph_arena = nullptr;
  CopyDesc* d_desc = nullptr;
  uint32_t* d_chunk = nullptr;
  uint64_t n_chunks = 0;
  uint32_t chunk_bytes = 0;
  int copy_cap = 0;
  const void* copy_fn = nullptr;
  dim3 copy_grid;
  unsigned copy_block = 256;
  size_t copy_smem = 0;
  AlignedBuf copy_args;
  // INDIRECT
  uint64_t* d_table = nullptr;
  uint64_t* d_table2 = nullptr;   // T6: second table (replays alternate between the two)
  void* d_patches = nullptr;      // T7: PreludePatch[n_patches] (device)
  uint32_t n_patches = 0;
  cudaStream_t xs = nullptr;      // T6: side stream carrying the table H2D copies
  cudaEvent_t ev_copy[2] = {nullptr, nullptr};   // T6: H2D into table b done
  cudaEvent_t ev_use[2] = {nullptr, nullptr};    // T6: replay reading table b done
  bool ev_copy_set[2] = {false, false}, ev_use_set[2] = {false, false};
  uint64_t* h_stage = nullptr;    // pinned ring [ring][n_pad]
  uint64_t* d_stage = nullptr;    // device alias (mapped, T4)
  int ring = 0;
  uint32_t n_pad = 0;
  std::vector<cudaEvent_t> ev;
  std::vector<bool> ev_used;
  // GEMM split-K workspace + per-tile counters, shared by the exec's GEMM nodes (they run one
  // after another: a GEMM writes its partials only after its griddepcontrol.wait)
  void* gemm_ws = nullptr;
  void* gemm_cnt = nullptr;
  std::vector<void*> gemm_tm_ws;  // per-CTA A tensor maps of GEMMs with an EXTERNAL A (kGemmADynamic)
  size_t gemm_cnt_off = 0;        // next free counter bytes while building launches
  int t5_pub = 0;                 // T5: position of the table-publishing launch
  unsigned long long* d_trace = nullptr;   // CGX_NODE_TRACE=1: [launch][3] ns stamps
  uint32_t* df_mem = nullptr;     // dataflow: [launches] CTA-completion counters + [1] epoch
  // T8 device loop: scheduler graph (one k_devloop node) + its replay counter
  cudaGraph_t dl_g = nullptr;
  cudaGraphExec_t dl_ge = nullptr;
  cudaGraphNode_t dl_node = nullptr;
  unsigned long long* dl_iter = nullptr;
  bool dataflow = false;
  // CGX_SYNC_GRAPH: dependency-DAG capture streams and per-node completion events
  std::vector<cudaStream_t> dag_s;
  std::vector<cudaEvent_t> dag_ev;
  uint32_t dag_used = 0;          // capture streams that received at least one node
  // T3 / T4 root
  const void* root_fn = nullptr;
  AlignedBuf root_args;
  cudaGraphNode_t root_node[2] = {nullptr, nullptr};
  unsigned long long* d_seq = nullptr;
  volatile unsigned long long* h_ack = nullptr;
  unsigned long long* d_ack = nullptr;
  // device-side failure word (DevStatus, cgx_args.h): mapped pinned host memory written by spinning
  // / device-launching kernels instead of trapping; checked by every cgx_launch
  volatile uint32_t* h_status = nullptr;
  uint32_t* d_status = nullptr;
  uint64_t spin_timeout_ns = 0;
  // megakernel (cgx_mega.h): one device blob = stages | row ops | tensor maps | split-K workspace |
  // grid-barrier counter | stage trace
  std::vector<void*> fuse_bufs;   // CGX_FUSE_LN_GEMM: producer row-sum buffers
  bool mega = false;
  void* mega_mem = nullptr;
  unsigned long long* mega_strace = nullptr;
  uint32_t mega_stages = 0, mega_ctas = 0;
};

static DevStatus dev_status(const cgx_exec* e) { return DevStatus{e->d_status, e->spin_timeout_ns}; }

// Spin bound of the kernels that wait on another agent: 10 s, or CGX_SPIN_TIMEOUT_MS (tests).
static uint64_t spin_timeout_ns() {
  const char* v = getenv("CGX_SPIN_TIMEOUT_MS");
  const long long ms = v ? atoll(v) : 0;
  return (uint64_t)(ms > 0 ? ms : 10000) * 1000000ull;
}

static cgx_transport eff_transport(const cgx_exec_opts& o) {
  return o.transport == CGX_XPORT_DEFAULT ? CGX_XPORT_ROOT_PARAMS : o.transport;
}

template <typename T>
static T* argp(Launch& l) { return reinterpret_cast<T*>(l.args.p); }

// Upper bound on the CTAs of an f32 elementwise / reduction node (the kernels grid-stride beyond
// it). Every CTA of node k must have started before node k+1 can launch, so wide grids slow the
// PDL launch cascade (scripts/launch_microbench.cu: 0.59 us per kernel at 148 CTAs, 0.82 at 512,
// 1.45 at 1184). A dataflow replay is bound by that cascade, so there the grid is capped at one
// CTA per SM (measured C2: 189 us uncapped, 172 us at 148, flat down to 64, 185 us at 16); a
// serial chain is bound by each node's latency and keeps the full-width grid (C2 CHAIN: 249 us
// uncapped, 270 us at 148). Env CGX_CHAIN_MAX_CTAS overrides both (diagnostics).
static uint64_t chain_grid_cap(bool dataflow = false) {
  static const int env = [] {
    const char* v = getenv("CGX_CHAIN_MAX_CTAS");
    return v ? std::max(1, atoi(v)) : 0;
  }();
  if (env) return (uint64_t)env;
  if (!dataflow) return 1ull << 20;
  static const int sms = [] {
    int d = 0, n = 0;
    cudaGetDevice(&d);
    return cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) == cudaSuccess && n > 0 ? n : 148;
  }();
  return (uint64_t)sms;
}

// Build the launch record of one node. Operand addresses are resolved for `mode`:
// EXTERNAL -> placeholder (COPY), table index (INDIRECT), or a patchable field (others).
// T5 (FIRST_NODE): launches 0..t5_pub of an INDIRECT exec take their external operands by value
// (patched like SETPARAMS); launch t5_pub also publishes the table before it triggers its
// dependents. The publisher is the SECOND launch when it can write the table (its publish + fence
// then overlaps the first launch, which it waits for anyway), else the first.
static bool t5_byvalue(const cgx_exec* e, int pos) {
  return e->o.mode == CGX_MODE_GRAPH_INDIRECT &&
         ((eff_transport(e->o) == CGX_XPORT_FIRST_NODE && pos <= e->t5_pub) ||
          eff_transport(e->o) == CGX_XPORT_PRELUDE);
}
static bool tw_capable(cgx_op op) {
  return uses_elem_args(op) || op == CGX_OP_LAYERNORM;
}

template <typename Base>
static void make_args(cgx_exec* e, Launch& l, bool tw) {
  if (!tw) {
    l.args.reset(sizeof(Base));
    return;
  }
  const int n = (int)e->c->ext_slots.size();
  const int cap = tw_cap(n);
  size_t bytes = 0, ptr_off = 0;
  switch (cap) {
    case 8: {
      using T = ArgsTW<Base, 8>;
      bytes = sizeof(T);
      ptr_off = offsetof(T, tw) + offsetof(TWPart<8>, ptr);
      break;
    }
    case 64: {
      using T = ArgsTW<Base, 64>;
      bytes = sizeof(T);
      ptr_off = offsetof(T, tw) + offsetof(TWPart<64>, ptr);
      break;
    }
    default: {
      using T = ArgsTW<Base, 512>;
      bytes = sizeof(T);
      ptr_off = offsetof(T, tw) + offsetof(TWPart<512>, ptr);
      break;
    }
  }
  l.args.reset(bytes);
  TWPart<8>* tw8 = reinterpret_cast<TWPart<8>*>(l.args.p + ptr_off - offsetof(TWPart<8>, ptr));
  tw8->table = e->d_table;
  tw8->n = (uint32_t)n;
  l.tw_ptr_off = ptr_off;
}

static int build_launch(cgx_exec* e, int k, Launch& l, int pre = -1) {
  const int add_k = (pre >= 0 && e->c->nodes[pre].op == CGX_OP_ADD) ? pre : -1;
  const int ln_k = (pre >= 0 && e->c->nodes[pre].op == CGX_OP_LAYERNORM) ? pre : -1;
  cgx_chain* c = e->c;
  const Node& n = c->nodes[k];
  const cgx_mode mode = e->o.mode;
  const int pos = k - e->first;
  l.node = k;
  l.pdl = !e->o.no_pdl;
  auto slot_ptr = [&](int si) -> void* {
    const Slot& s = c->slots[si];
    if (s.kind == CGX_SLOT_STATIC) return s.static_ptr;
    if (s.kind == CGX_SLOT_INTERNAL) return s.buf;
    if (mode == CGX_MODE_GRAPH_COPY) return e->ph[s.ext_j];
    return const_cast<void*>(e->cur[s.ext_j]);   // EAGER/SETPARAMS/STALE: patched at bind
  };
  auto is_ext = [&](int si) { return c->slots[si].kind == CGX_SLOT_EXTERNAL; };
  const bool byvalue = t5_byvalue(e, pos);
  const bool tw = byvalue && pos == e->t5_pub && eff_transport(e->o) == CGX_XPORT_FIRST_NODE;
  const bool indirect = mode == CGX_MODE_GRAPH_INDIRECT && !byvalue;
  const bool patch = mode == CGX_MODE_EAGER || mode == CGX_MODE_GRAPH_SETPARAMS || mode == CGX_MODE_GRAPH_STALE ||
                     byvalue;
  const int twc = tw ? tw_cap((int)c->ext_slots.size()) : 0;
  if (tw && (twc == 0 || !(uses_elem_args(n.op) || n.op == CGX_OP_LAYERNORM)))
    return fail(CGX_E_UNSUPPORTED, "FIRST_NODE transport: first node must be elementwise/reduce/LN, <= 512 externals");

  switch (n.op) {
    case CGX_OP_ADD:
    case CGX_OP_MUL:
    case CGX_OP_SCALE_IMM:
    case CGX_OP_COPY:
    case CGX_OP_SCALE_T:
    case CGX_OP_SUB:
    case CGX_OP_AXPY:
    case CGX_OP_GELU:
    case CGX_OP_GELU_BWD:
    case CGX_OP_TRANSPOSE:
    case CGX_OP_REDUCE_SUM: {
      make_args<ElemArgs>(e, l, tw);
      ElemArgs* a = argp<ElemArgs>(l);
      a->table = indirect ? e->d_table : nullptr;
      a->t0 = a->t1 = -1;
      a->out = slot_ptr(n.out);
      a->n = n.attr.n;
      a->scalar = n.attr.scalar;
      a->cols = n.attr.cols;
      const void** ins[2] = {&a->in0, &a->in1};
      int32_t* tid[2] = {&a->t0, &a->t1};
      for (int i = 0; i < n.n_in && i < 2; ++i) {
        *ins[i] = slot_ptr(n.in[i]);
        if (is_ext(n.in[i])) {
          const int j = c->slots[n.in[i]].ext_j;
          if (indirect) {
            *ins[i] = nullptr;
            *tid[i] = j;
          } else if (patch) {
            l.ext.push_back({(size_t)((uint8_t*)ins[i] - l.args.p), (size_t)((uint8_t*)tid[i] - l.args.p), j});
          }
        }
      }
      if (n.op == CGX_OP_TRANSPOSE) {
        l.func = kfn_transpose_bf16(twc);
        l.block = dim3(256);
        const uint64_t rows = n.attr.n / n.attr.cols;
        const uint64_t tiles = ceil_div(rows, 32) * ceil_div((uint64_t)n.attr.cols, 32);
        l.grid = dim3((unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, 148ull * 8)));
      } else if (n.op == CGX_OP_REDUCE_SUM) {
        l.func = kfn_reduce_sum_f32(twc);
        l.block = dim3(256);
        l.grid = dim3((unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n.attr.n / n.attr.cols, 8), chain_grid_cap())));
      } else {
        const int opi = n.op == CGX_OP_ADD ? 0 : n.op == CGX_OP_MUL ? 1 : n.op == CGX_OP_SCALE_IMM ? 2
                        : n.op == CGX_OP_SCALE_T ? 4 : n.op == CGX_OP_SUB ? 5 : n.op == CGX_OP_AXPY ? 6
                        : n.op == CGX_OP_GELU ? 7 : n.op == CGX_OP_GELU_BWD ? 8 : 3;
        const int dt = c->slots[n.out].dtype == CGX_F32 ? 0 : 1;
        l.func = kfn_elem(opi, dt, twc);
        l.block = dim3(elem_block_threads());
        const uint64_t per_vec = dt == 0 ? 4 : 8;
        const uint64_t nv = n.attr.n / per_vec;
        const uint64_t tiles = ceil_div(nv, (uint64_t)elem_block_threads() * elem_tile_vecs());
        l.grid = dim3((unsigned)std::max<uint64_t>(1, dt == 0 ? std::min<uint64_t>(tiles, chain_grid_cap()) : tiles));
      }
      return CGX_OK;
    }
    case CGX_OP_LAYERNORM: {
      make_args<LnArgs>(e, l, tw);
      LnArgs* a = argp<LnArgs>(l);
      a->table = indirect ? e->d_table : nullptr;
      a->tx = -1;
      a->x = slot_ptr(n.in[0]);
      a->g = slot_ptr(n.in[1]);
      a->b = slot_ptr(n.in[2]);
      a->out = slot_ptr(n.out);
      a->rows = n.attr.rows;
      a->cols = n.attr.cols;
      a->eps = n.attr.eps;
      if (is_ext(n.in[1]) || is_ext(n.in[2])) return fail(CGX_E_UNSUPPORTED, "layernorm: external gamma/beta");
      if (c->slots[n.in[1]].kind == CGX_SLOT_STATIC && c->slots[n.in[2]].kind == CGX_SLOT_STATIC)
        a->flags |= kFlagLnParamsPre;
      if (is_ext(n.in[0])) {
        const int j = c->slots[n.in[0]].ext_j;
        if (indirect) {
          a->x = nullptr;
          a->tx = j;
        } else if (patch) {
          l.ext.push_back({offsetof(LnArgs, x), offsetof(LnArgs, tx), j});
        }
      }
      if (add_k >= 0) {   // the fused ADD -> LAYERNORM pair: x = ADD.in[0], add_b = ADD.in[1]
        const Node& an = c->nodes[add_k];
        a->x = slot_ptr(an.in[0]);
        a->tx = -1;
        a->add_b = slot_ptr(an.in[1]);
        a->tb = -1;
        a->add_out = slot_ptr(an.out);
        const int opnd[2] = {an.in[0], an.in[1]};
        const size_t foff[2] = {offsetof(LnArgs, x), offsetof(LnArgs, add_b)};
        const size_t toff[2] = {offsetof(LnArgs, tx), offsetof(LnArgs, tb)};
        int32_t* tix[2] = {&a->tx, &a->tb};
        const void** pix[2] = {&a->x, &a->add_b};
        for (int i = 0; i < 2; ++i)
          if (is_ext(opnd[i])) {
            const int j = c->slots[opnd[i]].ext_j;
            if (indirect) {
              *pix[i] = nullptr;
              *tix[i] = j;
            } else if (patch) {
              l.ext.push_back({foff[i], toff[i], j});
            }
          }
        l.pre_node = add_k;
      }
      decoder_ln_launch_dims(n.attr.rows, n.attr.cols, &l.grid, &l.block);
      l.func = kfn_layernorm(twc, add_k >= 0, n.attr.cols);
      return CGX_OK;
    }
    case CGX_OP_GEMM_BF16: {
      // EXTERNAL operands. A is read through a TMA tensor map: under COPY it is encoded at capture
      // with the placeholder; under INDIRECT and the patch modes the kernel rebuilds this CTA's copy
      // of the map from table[j] / the patched a_ptr field (tensormap.replace, kGemmADynamic) — PI
      // through the TMA descriptor, no data copy. The residual: table / patched field / placeholder.
      // Weights and bias are STATIC by construction.
      const bool res_ext = (n.attr.flags & CGX_GEMM_RESIDUAL) && is_ext(n.in[3]);
      const bool a_ext = is_ext(n.in[0]) && (indirect || patch);
      for (int i = 1; i < 3; ++i)
        if (is_ext(n.in[i])) return fail(CGX_E_UNSUPPORTED, "gemm: external weights/bias");
      // LN -> GEMM fusion: A is the LayerNorm's INPUT (normalised in the kernel's A prologue)
      void* A = ln_k >= 0 ? slot_ptr(c->nodes[ln_k].in[0]) : slot_ptr(n.in[0]);
      void* W = slot_ptr(n.in[1]);
      void* bias = slot_ptr(n.in[2]);
      void* res = (n.attr.flags & CGX_GEMM_RESIDUAL) ? slot_ptr(n.in[3]) : nullptr;
      size_t argbytes = 0;
      void* cnt_ptr = e->gemm_cnt ? static_cast<char*>(e->gemm_cnt) + e->gemm_cnt_off : nullptr;
      CKS(decoder_gemm_build(n.attr.M, n.attr.N, n.attr.K, n.attr.flags, A, W, bias, res, slot_ptr(n.out),
                             e->gemm_ws, cnt_ptr, nullptr, &argbytes, &l.grid, &l.block, &l.smem, &l.func));
      l.args.reset(argbytes);
      CKS(decoder_gemm_build(n.attr.M, n.attr.N, n.attr.K, n.attr.flags, A, W, bias, res, slot_ptr(n.out),
                             e->gemm_ws, cnt_ptr, l.args.p, &argbytes, &l.grid, &l.block, &l.smem, &l.func));
      {
        size_t w1, c1;
        decoder_gemm_plan(n.attr.M, n.attr.N, n.attr.K, &w1, &c1);
        e->gemm_cnt_off += c1;
      }
      l.cluster_z = l.grid.z;
      // the weight / bias operands are prefetched before griddepcontrol.wait unless a node of the
      // chain writes them (training chain: transposed activations, in-place weight updates)
      {
        bool written = false;
        for (const Node& q : c->nodes)
          if (q.out == n.in[1] || q.out == n.in[2]) written = true;
        if (written) decoder_gemm_set_w_after_wait(l.args.p);
      }
      if (n.attr.flags & CGX_GEMM_ALLREDUCE) {
        if (c->peer_world <= 0) return fail(CGX_E_STATE, "gemm allreduce: no peers (cgx_chain_set_peers)");
        if ((uint64_t)n.attr.M * n.attr.N > c->peer_max_elems || n.attr.N % 8)
          return fail(CGX_E_UNSUPPORTED, "gemm allreduce: M*N <= max_elems and N % 8 == 0");
        if (l.grid.x * l.grid.y * l.grid.z > (unsigned)kArMaxCtas)
          return fail(CGX_E_UNSUPPORTED, "gemm allreduce: more than 256 CTAs");
        int ar_index = 0, n_ar = 0;
        ar_position(c, k, &ar_index, &n_ar);
        if (n_ar > c->peer_max_ar)
          return fail(CGX_E_UNSUPPORTED, "gemm allreduce: more all-reduces than the peer regions hold (max_allreduces)");
        std::vector<void*> recv(c->peer_world);
        std::vector<uint32_t*> flg(c->peer_world);
        for (int r = 0; r < c->peer_world; ++r) {   // this node's [2][world][slot] receive buffers
          recv[r] = static_cast<__nv_bfloat16*>(c->peer_base[r]) +
                    (uint64_t)ar_index * peer_node_elems(c->peer_world, c->peer_max_elems);
          flg[r] = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(c->peer_base[r]) +
                                               peer_flag_offset(c->peer_world, c->peer_max_elems, c->peer_max_ar));
        }
        decoder_gemm_set_allreduce(l.args.p, (uint32_t)c->peer_rank, (uint32_t)c->peer_world, (uint32_t)ar_index,
                                   (uint32_t)n_ar, peer_slot_elems(c->peer_max_elems), c->peer_counters,
                                   recv.data(), flg.data());
        decoder_gemm_set_status(l.args.p, e->d_status, e->spin_timeout_ns);
      }
      if (a_ext) {
        const int j = c->slots[n.in[0]].ext_j;
        const size_t ws_bytes = (size_t)l.grid.x * l.grid.y * l.grid.z * 128;
        void* ws = nullptr;
        CK(cudaMalloc(&ws, ws_bytes));
        e->gemm_tm_ws.push_back(ws);
        const bool late = mode == CGX_MODE_EAGER;
        if (indirect) {
          decoder_gemm_set_a_dynamic(l.args.p, e->d_table, j, ws, late);
        } else {
          decoder_gemm_set_a_dynamic(l.args.p, nullptr, -1, ws, late);
          size_t tidx = 0;
          const size_t off = decoder_gemm_a_field(&tidx);
          l.ext.push_back({off, tidx, j});
        }
      }
      if (res_ext) {
        const int j = c->slots[n.in[3]].ext_j;
        if (indirect) {
          decoder_gemm_set_residual_table(l.args.p, e->d_table, j);
        } else if (patch) {
          size_t tidx = 0;
          const size_t off = decoder_gemm_residual_field(&tidx);
          l.ext.push_back({off, tidx, j});
        }
      }
      return CGX_OK;
    }
    case CGX_OP_ATTN_CAUSAL: {
      if (is_ext(n.in[0])) return fail(CGX_E_UNSUPPORTED, "attention: external qkv");
      l.args.reset(sizeof(AttnArgs));
      AttnArgs* a = argp<AttnArgs>(l);
      a->qkv = slot_ptr(n.in[0]);
      a->out = slot_ptr(n.out);
      a->T = n.attr.T;
      a->H = n.attr.H;
      a->D = n.attr.D;
      a->scale = n.attr.scalar;
      if (const char* qv = getenv("CGX_ATTN_QALL"); qv && qv[0] == '1') a->flags |= kAttnQAll;   // measurement knob
      decoder_attn_launch_dims(n.attr.T, n.attr.H, n.attr.D, &l.grid, &l.block, &l.smem);
      if (const char* cv = getenv("CGX_CTA_TRACE"); cv && cv[0] == '1') {   // diagnostics (cgx_debug_cta_trace)
        void* ctb = nullptr;
        CK(cudaMalloc(&ctb, sizeof(unsigned long long) * 8 * l.grid.x * l.grid.y));
        CK(cudaMemset(ctb, 0, sizeof(unsigned long long) * 8 * l.grid.x * l.grid.y));
        e->fuse_bufs.push_back(ctb);
        a->ctrace = static_cast<unsigned long long*>(ctb);
      }
      l.func = kfn_attention();
      return CGX_OK;
    }
    case CGX_OP_ALLREDUCE_SUM: {
      if (is_ext(n.in[0])) return fail(CGX_E_UNSUPPORTED, "allreduce: external input");
      if (c->mc_world > 0) {
        // one-shot all-reduce through the NVSwitch multicast object (k_allreduce_mc)
        if (n.attr.n % 8 || n.attr.n > c->mc_max_elems)
          return fail(CGX_E_UNSUPPORTED, "allreduce (multicast): n must be a multiple of 8 and <= max_elems");
        int ar_index = 0, n_ar = 0;
        ar_position(c, k, &ar_index, &n_ar);
        if (n_ar > c->mc_max_ar)
          return fail(CGX_E_UNSUPPORTED, "allreduce (multicast): more all-reduces than the region holds (max_allreduces)");
        l.args.reset(sizeof(McArArgs));
        McArArgs* a = argp<McArArgs>(l);
        a->in = static_cast<const __nv_bfloat16*>(slot_ptr(n.in[0]));
        a->out = static_cast<__nv_bfloat16*>(slot_ptr(n.out));
        a->n = n.attr.n;
        a->slot_elems = mc_slot_elems(c->mc_max_elems);
        a->world = (uint32_t)c->mc_world;
        a->ar_index = (uint32_t)ar_index;
        a->n_ar = (uint32_t)n_ar;
        a->counters = c->peer_counters;
        const uint64_t doff = (uint64_t)ar_index * 2 * a->slot_elems * sizeof(uint16_t);
        const uint64_t foff = mc_flag_offset(c->mc_max_elems, c->mc_max_ar) + (uint64_t)ar_index * kArMaxCtas * sizeof(uint32_t);
        a->uc_data = reinterpret_cast<__nv_bfloat16*>(static_cast<uint8_t*>(c->mc_uc) + doff);
        a->mc_data = reinterpret_cast<__nv_bfloat16*>(static_cast<uint8_t*>(c->mc_mc) + doff);
        a->uc_flags = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(c->mc_uc) + foff);
        a->mc_flags = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(c->mc_mc) + foff);
        a->st = dev_status(e);
        const uint64_t nv = n.attr.n / 8;
        l.grid = dim3((unsigned)std::max<uint64_t>(1, std::min<uint64_t>(kArMaxCtas, ceil_div(nv, 256))));
        l.block = dim3(256);
        l.func = kfn_allreduce_mc();
        return CGX_OK;
      }
      if (c->peer_world > 0) {
        // one-shot all-reduce over peer memory (k_allreduce_peer)
        if (n.attr.n % 8 || n.attr.n > c->peer_max_elems)
          return fail(CGX_E_UNSUPPORTED, "allreduce (peer): n must be a multiple of 8 and <= max_elems");
        int ar_index = 0, n_ar = 0;
        ar_position(c, k, &ar_index, &n_ar);
        if (n_ar > c->peer_max_ar)
          return fail(CGX_E_UNSUPPORTED, "allreduce (peer): more all-reduces than the peer regions hold (max_allreduces)");
        l.args.reset(sizeof(PeerArArgs));
        PeerArArgs* a = argp<PeerArArgs>(l);
        a->in = static_cast<const __nv_bfloat16*>(slot_ptr(n.in[0]));
        a->out = static_cast<__nv_bfloat16*>(slot_ptr(n.out));
        a->n = n.attr.n;
        a->slot_elems = peer_slot_elems(c->peer_max_elems);
        a->rank = (uint32_t)c->peer_rank;
        a->world = (uint32_t)c->peer_world;
        a->ar_index = (uint32_t)ar_index;
        a->n_ar = (uint32_t)n_ar;
        a->counters = c->peer_counters;
        for (int r = 0; r < c->peer_world; ++r) {   // this node's [2][world][slot] receive buffers
          a->recv[r] = static_cast<__nv_bfloat16*>(c->peer_base[r]) +
                       (uint64_t)ar_index * peer_node_elems(c->peer_world, c->peer_max_elems);
          a->flags_of[r] = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(c->peer_base[r]) +
                                                      peer_flag_offset(c->peer_world, c->peer_max_elems, c->peer_max_ar));
        }
        a->st = dev_status(e);
        const uint64_t nv = n.attr.n / 8;
        l.grid = dim3((unsigned)std::max<uint64_t>(1, std::min<uint64_t>(kArMaxCtas, ceil_div(nv, 256))));
        l.block = dim3(256);
        l.func = kfn_allreduce_peer();
        return CGX_OK;
      }
      if (!c->nccl) return fail(CGX_E_STATE, "allreduce: no NCCL communicator (cgx_chain_set_nccl)");
      l.kind = LK_NCCL;
      l.nc_in = slot_ptr(n.in[0]);
      l.nc_out = slot_ptr(n.out);
      l.nc_count = n.attr.n;
      return CGX_OK;
    }
  }
  return fail(CGX_E_INVALID_ARG, "build_launch: unknown op");
}

// Pre-wait loads: with every kernel triggering at entry, a kernel may start while ANY earlier node
// of the replay is still running, so only slots nothing inside the graph writes may be read before
// griddepcontrol.wait: EXTERNAL inputs (bound before the replay; COPY placeholders are written by
// the copy kernel, which fully precedes the graph) and STATIC weights.
static void set_prewait_masks(cgx_exec* e) {
  if (e->o.no_pdl || e->mega) return;
  for (auto& l : e->L) {
    if (l.kind != LK_KERNEL) continue;
    const Node& node = e->c->nodes[l.node];
    if (!uses_elem_args(node.op)) continue;
    uint32_t pre = 0;
    for (int j = 0; j < node.n_in && j < 2; ++j) {
      const cgx_slot_kind k = e->c->slots[node.in[j]].kind;
      if (k == CGX_SLOT_EXTERNAL || k == CGX_SLOT_STATIC) pre |= 1u << j;
    }
    argp<ElemArgs>(l)->pre = pre;
  }
}

// How nodes wait for their predecessors in graph modes with PDL (cgx_args.h).
//
// Dataflow (CGX_SYNC_DATAFLOW, every node a chain kernel): node k waits, through per-launch CTA
// counters, for exactly (a) the last earlier writer of each slot it reads (RAW), (b) the last
// earlier writer of its output slot (WAW) and every earlier reader of that slot since then (WAR).
// "Earlier" is within this graph only: a graph launch waits for the previous replay as a whole.
// Waits compose transitively (a node signals only after its own waits returned), so these sets
// suffice. More than kDfMaxDeps dependencies falls back to deferred waits.
//
// Deferred wait (CGX_SYNC_DEFER, or the fallback): inside one graph the early-trigger cascade
// means node k's pre-wait part can overlap ANY earlier, not yet completed node of the same replay.
// So node k may store before its griddepcontrol.wait iff it is an f32 elementwise node whose
// operands are all read pre-wait (EXTERNAL/STATIC) and no earlier node of this graph reads or
// writes its output slot; it still waits before exiting, which keeps "node k complete => nodes < k
// complete" for the nodes after it.
//
// Eager mode keeps plain PDL waits: there the previous iteration's nodes are stream predecessors.
static bool df_capable(const Node& n, cgx_dtype out_dt) {
  if (n.op == CGX_OP_REDUCE_SUM || n.op == CGX_OP_TRANSPOSE) return true;
  if (is_elemwise(n.op) && n.op != CGX_OP_SCALE_T) return true;   // f32 and bf16 elementwise
  return n.op == CGX_OP_SCALE_T && out_dt == CGX_F32;
}

// The chain's data-dependency DAG over the exec's launches, from the slot accesses in chain order
// (RAW: last writer of every input; WAW: last writer of the output; WAR: readers of the output
// since then), plus an artificial edge between consecutive collectives (they run one at a time,
// in chain order, on every rank: NCCL forbids concurrent collectives on one communicator, and the
// peer protocol's spinning kernels must not compete for SMs with each other).
static std::vector<std::vector<int>> chain_deps(const cgx_exec* e) {
  const size_t nl = e->L.size(), ns = e->c->slots.size();
  std::vector<std::vector<int>> deps(nl);
  std::vector<int> last_w(ns, -1);
  std::vector<std::vector<int>> readers(ns);
  int last_ar = -1;
  for (size_t p = 0; p < nl; ++p) {
    auto add = [&](int q) {
      if (q < 0 || q == (int)p) return;
      for (int d : deps[p]) if (d == q) return;
      deps[p].push_back(q);
    };
    // a fused ADD -> LAYERNORM launch performs both nodes' accesses, the ADD's first
    for (int part = 0; part < 2; ++part) {
      const int ni = part == 0 ? e->L[p].pre_node : e->L[p].node;
      if (ni < 0) continue;
      const Node& n = e->c->nodes[ni];
      for (int j = 0; j < n.n_in; ++j) add(last_w[n.in[j]]);
      add(last_w[n.out]);
      for (int r : readers[n.out]) add(r);
      if (is_allreduce(n)) {
        add(last_ar);
        last_ar = (int)p;
      }
      for (int j = 0; j < n.n_in; ++j) readers[n.in[j]].push_back((int)p);
      last_w[n.out] = (int)p;
      readers[n.out].clear();
    }
  }
  return deps;
}

// concurrent[p] = some other launch is neither an ancestor nor a descendant of p in the DAG
// (transitive closure over bitsets; a linear chain has none).
static std::vector<char> concurrent_nodes(const cgx_exec* e) {
  const size_t nl = e->L.size(), w = (nl + 63) / 64;
  const auto deps = chain_deps(e);
  std::vector<uint64_t> anc(nl * w, 0);   // anc[p] includes p itself
  for (size_t p = 0; p < nl; ++p) {
    uint64_t* a = &anc[p * w];
    a[p / 64] |= 1ull << (p % 64);
    for (int d : deps[p])
      for (size_t k = 0; k < w; ++k) a[k] |= anc[(size_t)d * w + k];
  }
  // related[p] = ancestors(p) ∪ descendants(p); descendants via q ∈ desc(p) ⇔ p ∈ anc(q)
  std::vector<uint64_t> rel(anc);
  for (size_t q = 0; q < nl; ++q)
    for (size_t p = 0; p < q; ++p)
      if (anc[q * w + p / 64] >> (p % 64) & 1) rel[p * w + q / 64] |= 1ull << (q % 64);
  std::vector<char> conc(nl, 0);
  for (size_t p = 0; p < nl; ++p) {
    size_t cnt = 0;
    for (size_t k = 0; k < w; ++k) cnt += (size_t)__builtin_popcountll(rel[p * w + k]);
    conc[p] = cnt < nl;
  }
  return conc;
}

static int set_sync_flags(cgx_exec* e) {
  if (e->mega) return CGX_OK;   // one launch: nothing to order
  if (e->o.no_pdl || e->o.mode == CGX_MODE_EAGER || e->o.sync_mode == CGX_SYNC_CHAIN) return CGX_OK;
  if (e->o.sync_mode == CGX_SYNC_GRAPH) {
    // Nodes that can run concurrently with another node of the DAG (neither its ancestor nor its
    // descendant): one CTA per SM for the f32 elementwise / reduction kernels, as in the dataflow
    // replay (C2 at 16 streams: 54.8 us capped vs 56.3 us full width, profiles/r01). A node that
    // runs alone (every other node is ordered with it: C1/C4 are linear chains) keeps the same
    // full-width grid as EAGER — capping it cost up to 1.5x at >= 4 MiB (profiles/r01/c4_sweep.json).
    const std::vector<char> conc = concurrent_nodes(e);
    for (size_t p = 0; p < e->L.size(); ++p) {
      auto& l = e->L[p];
      if (l.kind != LK_KERNEL || !conc[p]) continue;
      const Node& n = e->c->nodes[l.node];
      const bool f32 = e->c->slots[n.out].dtype == CGX_F32 && (n.op <= CGX_OP_COPY || n.op == CGX_OP_SCALE_T);
      if (n.op == CGX_OP_REDUCE_SUM || f32) l.grid.x = (unsigned)std::min<uint64_t>(l.grid.x, chain_grid_cap(true));
    }
    return CGX_OK;
  }
  const size_t ns = e->c->slots.size(), nl = e->L.size();
  if (e->o.sync_mode == CGX_SYNC_DATAFLOW && nl > 0) {
    bool ok = true;
    for (auto& l : e->L) ok = ok && l.kind == LK_KERNEL && df_capable(e->c->nodes[l.node], e->c->slots[e->c->nodes[l.node].out].dtype);
    std::vector<std::vector<uint32_t>> deps(nl);
    if (ok) {
      std::vector<int> last_w(ns, -1);
      std::vector<std::vector<uint32_t>> readers(ns);   // readers since the last writer
      for (size_t p = 0; p < nl && ok; ++p) {
        const Node& n = e->c->nodes[e->L[p].node];
        auto add = [&](int q) {
          if (q < 0) return;
          for (uint32_t d : deps[p]) if (d == (uint32_t)q) return;
          deps[p].push_back((uint32_t)q);
        };
        for (int j = 0; j < n.n_in; ++j) add(last_w[n.in[j]]);
        add(last_w[n.out]);
        for (uint32_t r : readers[n.out]) if (r != p) add((int)r);
        if (deps[p].size() > (size_t)kDfMaxDeps) ok = false;
        for (int j = 0; j < n.n_in; ++j) readers[n.in[j]].push_back((uint32_t)p);
        last_w[n.out] = (int)p;
        readers[n.out].clear();
      }
    }
    if (ok) {
      // narrower grids for the launch-cascade-bound dataflow replay (chain_grid_cap)
      for (auto& l : e->L) {
        const Node& n = e->c->nodes[l.node];
        const bool f32 = e->c->slots[n.out].dtype == CGX_F32;
        if (n.op == CGX_OP_REDUCE_SUM || f32) l.grid.x = (unsigned)std::min<uint64_t>(l.grid.x, chain_grid_cap(true));
      }
      cudaError_t ce = cudaMalloc(&e->df_mem, sizeof(uint32_t) * (nl + 1));
      if (ce == cudaSuccess) ce = cudaMemset(e->df_mem, 0, sizeof(uint32_t) * (nl + 1));
      if (ce != cudaSuccess) return cuda_fail(ce, "dataflow counters", __LINE__);
      // transitive dependency closure (bitsets): a node whose closure is every earlier node takes
      // its immediate predecessor through griddepcontrol.wait (measured: cheaper on a linear chain,
      // C1); a node with independent earlier nodes spins on counters only, because a PDL wait
      // also waits out the in-order retirement of the unrelated grids before it (measured: C2
      // 175 us with counters vs 190 us with PDL waits on the immediate predecessor).
      const size_t words = (nl + 63) / 64;
      std::vector<std::vector<uint64_t>> clo(nl, std::vector<uint64_t>(words, 0));
      std::vector<char> full(nl, 0);
      for (size_t p = 0; p < nl; ++p) {
        for (uint32_t d : deps[p]) {
          clo[p][d / 64] |= 1ull << (d % 64);
          for (size_t w = 0; w < words; ++w) clo[p][w] |= clo[d][w];
        }
        size_t cnt = 0;
        for (size_t w = 0; w < words; ++w) cnt += (size_t)__builtin_popcountll(clo[p][w]);
        full[p] = cnt == p;
      }
      std::vector<char> spun_on(nl, 0);
      for (size_t p = 0; p < nl; ++p) {
        ElemArgs* a = argp<ElemArgs>(e->L[p]);
        a->st = dev_status(e);
        a->df_done = e->df_mem;
        a->df_epoch = e->df_mem + nl;
        a->df_self = (uint32_t)p;
        a->df_n = 0;
        uint32_t f = kFlagDataflow;
        // the first node after a root table-writer waits for the root through PDL
        if (a->flags & kFlagTableAfterWait) f |= kFlagDfPdlWait;
        for (uint32_t d : deps[p]) {
          if (d + 1 == p && full[p]) {  // immediate predecessor of a chain node: hardware wait
            f |= kFlagDfPdlWait;
            continue;
          }
          const Launch& q = e->L[d];
          a->df_dep[a->df_n] = d;
          a->df_ctas[a->df_n] = q.grid.x * q.grid.y * q.grid.z;
          ++a->df_n;
          spun_on[d] = 1;
        }
        a->flags |= f;
      }
      bool any = false;
      for (size_t p = 0; p < nl; ++p)
        if (spun_on[p]) {
          argp<ElemArgs>(e->L[p])->flags |= kFlagDfSignal;
          any = true;
        }
      // the epoch (and its fence before node 0 triggers) is only needed when some node spins
      if (any) argp<ElemArgs>(e->L[0])->flags |= kFlagEpochBump;
      e->dataflow = true;
      return CGX_OK;
    }
  }
  std::vector<char> touched(ns, 0);
  for (auto& l : e->L) {
    const Node& node = e->c->nodes[l.node];
    if (l.kind == LK_KERNEL) {
      const bool elem = node.op <= CGX_OP_COPY || node.op == CGX_OP_SCALE_T;
      const bool f32 = e->c->slots[node.out].dtype == CGX_F32;
      if (elem && f32) {
        const uint32_t need = (node.op == CGX_OP_ADD || node.op == CGX_OP_MUL || node.op == CGX_OP_SCALE_T) ? 3u : 1u;
        ElemArgs* a = argp<ElemArgs>(l);
        if ((a->pre & need) == need && !touched[node.out] && !(a->flags & (kFlagTableAfterWait | kFlagTriggerAfterWait)))
          a->flags |= kFlagDeferWait;
      }
    }
    for (int j = 0; j < node.n_in; ++j) touched[node.in[j]] = 1;
    touched[node.out] = 1;
  }
  return CGX_OK;
}

static int issue(cgx_exec* e, Launch& l, cudaStream_t s) {
  if (l.kind == LK_NCCL) {
    ncclResult_t r = ncclAllReduce(l.nc_in, l.nc_out, l.nc_count, ncclBfloat16, ncclSum,
                                   static_cast<ncclComm_t>(e->c->nccl), s);
    if (r != ncclSuccess) return fail(CGX_E_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
    return CGX_OK;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = l.grid;
  cfg.blockDim = l.block;
  cfg.dynamicSmemBytes = l.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[5];
  unsigned na = 0;
  if (l.coop) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  if (l.prio) {
    attr[na].id = cudaLaunchAttributePriority;
    attr[na].val.priority = l.prio;
    ++na;
  }
  if (l.cluster_z > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = l.cluster_z;
    ++na;
  }
  if (l.pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  int du = -1;
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  if (l.dev_updatable && cudaStreamIsCapturing(s, &cst) == cudaSuccess && cst == cudaStreamCaptureStatusActive) {
    du = (int)na;
    attr[na].id = cudaLaunchAttributeDeviceUpdatableKernelNode;
    attr[na].val.deviceUpdatableKernelNode.deviceUpdatable = 1;
    attr[na].val.deviceUpdatableKernelNode.devNode = nullptr;
    ++na;
  }
  if (na) {
    cfg.attrs = attr;
    cfg.numAttrs = na;
  }
  void* argv[1] = {l.args.p};
  const cudaError_t le = cudaLaunchKernelExC(&cfg, l.func, argv);
  if (le != cudaSuccess) {
    cudaGetLastError();
    return fail(CGX_E_CUDA, std::string("launch of node ") + std::to_string(l.node) + " (op " +
                                std::to_string((int)e->c->nodes[l.node].op) + ", grid " + std::to_string(l.grid.x) + "x" +
                                std::to_string(l.grid.y) + "x" + std::to_string(l.grid.z) + ", block " +
                                std::to_string(l.block.x) + ", smem " + std::to_string(l.smem) + ", cluster " +
                                std::to_string(l.cluster_z) + ", params " + std::to_string(l.args.n) + " B): " +
                                cudaGetErrorString(le));
  }
  if (du >= 0) l.dev_node = attr[du].val.deviceUpdatableKernelNode.devNode;
  return CGX_OK;
}

static int last_captured_node(cudaStream_t cs, cudaGraphNode_t* out) {
  cudaStreamCaptureStatus status;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(cs, &status, nullptr, nullptr, &deps, &nd));
  if (status != cudaStreamCaptureStatusActive || nd != 1)
    return fail(CGX_E_CUDA, "capture: could not identify the captured node");
  *out = deps[0];
  return CGX_OK;
}

// ---------------------------------------------------------------------------- COPY plan
static int setup_copy(cgx_exec* e) {
  cgx_chain* c = e->c;
  const int n_ext = (int)c->ext_slots.size();
  e->ph.assign(n_ext, nullptr);
  size_t total = 0;
  uint64_t data = 0;
  for (int j : e->ext_read) {
    total += ceil_div(c->slots[c->ext_slots[j]].nbytes, 256) * 256;
    data += c->slots[c->ext_slots[j]].nbytes;
  }
  if (total) CK(cudaMalloc(&e->ph_arena, total));
  size_t off = 0;
  for (int j : e->ext_read) {
    e->ph[j] = static_cast<char*>(e->ph_arena) + off;
    off += ceil_div(c->slots[c->ext_slots[j]].nbytes, 256) * 256;
  }
  const int nt = (int)e->ext_read.size();
  if (nt > 1024) return fail(CGX_E_UNSUPPORTED, "COPY: more than 1024 external tensors");
  // LDG/STG kernel: 2 KiB warp-blocks over the concatenated tensors (no lookup table); the TMA
  // bulk variant uses fixed chunks of its shared-memory stage size with a chunk -> tensor map.
  const bool bulk = e->o.copy_impl == 2;
  const uint64_t cb = bulk ? copy_bulk_chunk() : copy_block_bytes();
  e->chunk_bytes = (uint32_t)cb;
  std::vector<CopyDesc> desc(nt);
  std::vector<uint32_t> chunk;
  uint64_t nch = 0;
  for (int t = 0; t < nt; ++t) {
    const Slot& s = c->slots[c->ext_slots[e->ext_read[t]]];
    desc[t].dst = e->ph[e->ext_read[t]];
    desc[t].nbytes = s.nbytes;
    desc[t].chunk_begin = nch;
    desc[t].n_chunks = std::max<uint64_t>(1, ceil_div(s.nbytes, cb));
    nch += desc[t].n_chunks;
    if (bulk)
      for (uint64_t q = 0; q < desc[t].n_chunks; ++q) chunk.push_back((uint32_t)t);
  }
  e->n_chunks = nch;
  if (!bulk && nch >= (1ull << 32)) return fail(CGX_E_UNSUPPORTED, "COPY: more than 8 TiB of inputs");
  if (nt) {
    CK(cudaMalloc(&e->d_desc, sizeof(CopyDesc) * nt));
    CK(cudaMemcpy(e->d_desc, desc.data(), sizeof(CopyDesc) * nt, cudaMemcpyHostToDevice));
  }
  if (bulk && !chunk.empty()) {
    CK(cudaMalloc(&e->d_chunk, sizeof(uint32_t) * chunk.size()));
    CK(cudaMemcpy(e->d_chunk, chunk.data(), sizeof(uint32_t) * chunk.size(), cudaMemcpyHostToDevice));
  }
  e->copy_cap = nt <= 8 ? 8 : nt <= 64 ? 64 : 1024;
  if (bulk) {
    e->copy_fn = kfn_copy_bulk(e->copy_cap);
    e->copy_block = 32;
    e->copy_smem = copy_bulk_smem();
    e->copy_grid = dim3((unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nch, 148)));
  } else {
    // Large copies: 2 CTAs x 256 threads per SM (best sustained HBM rate measured at 3 x 1 GiB);
    // below 256 MiB the ramp dominates, so more CTAs. CGX_COPY_CTAS overrides (measurement knob).
    e->copy_fn = kfn_copy(e->copy_cap);
    e->copy_block = 256;
    e->copy_smem = 0;
    uint64_t ctas = data >= (256ull << 20) ? 148 * 2 : 148 * 8;
    if (const char* env = getenv("CGX_COPY_CTAS")) ctas = std::max<uint64_t>(1, strtoull(env, nullptr, 10));
    e->copy_grid = dim3((unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(nch, 8), ctas)));
  }
  const size_t hdr = offsetof(CopyArgs<8>, src);
  e->copy_args.reset(hdr + sizeof(void*) * e->copy_cap);
  CopyArgs<8>* a = reinterpret_cast<CopyArgs<8>*>(e->copy_args.p);   // header layout is CAP-independent
  a->desc = e->d_desc;
  a->chunk_tensor = e->d_chunk;
  a->n_tensors = (uint32_t)nt;
  a->n_chunks = e->n_chunks;
  a->chunk_bytes = e->chunk_bytes;
  return CGX_OK;
}

// ---------------------------------------------------------------------------- INDIRECT setup
static int setup_table(cgx_exec* e) {
  const int n = (int)e->c->ext_slots.size();
  const int nalloc = std::max(n, 1);
  CK(cudaMalloc(&e->d_table, sizeof(uint64_t) * ((nalloc + 15) / 16) * 16));
  CK(cudaMemset(e->d_table, 0, sizeof(uint64_t) * nalloc));
  const cgx_transport t = eff_transport(e->o);
  e->n_pad = (uint32_t)(((nalloc + 15) / 16) * 16);   // 128-B aligned ring slots
  if (t == CGX_XPORT_H2D || t == CGX_XPORT_ROOT_MEMCPY || t == CGX_XPORT_ROOT_MAPPED || t == CGX_XPORT_PRELUDE ||
      t == CGX_XPORT_DEVICE) {
    e->ring = t == CGX_XPORT_ROOT_MEMCPY ? 2 : 4;
    const unsigned flags = t == CGX_XPORT_ROOT_MAPPED ? cudaHostAllocMapped : cudaHostAllocDefault;
    CK(cudaHostAlloc((void**)&e->h_stage, sizeof(uint64_t) * e->n_pad * e->ring, flags));
    memset(e->h_stage, 0, sizeof(uint64_t) * e->n_pad * e->ring);
    if (t != CGX_XPORT_ROOT_MAPPED) {
      e->ev.resize(e->ring);
      e->ev_used.assign(e->ring, false);
      for (auto& v : e->ev) CK(cudaEventCreateWithFlags(&v, cudaEventDisableTiming));
    } else {
      CK(cudaHostGetDevicePointer((void**)&e->d_stage, e->h_stage, 0));
      unsigned long long* hack = nullptr;
      CK(cudaHostAlloc((void**)&hack, 64, cudaHostAllocMapped));
      *hack = 0;
      e->h_ack = hack;
      CK(cudaHostGetDevicePointer((void**)&e->d_ack, hack, 0));
      CK(cudaMalloc(&e->d_seq, 64));
      CK(cudaMemset(e->d_seq, 0, 64));
    }
  }
  if (t == CGX_XPORT_H2D_PINGPONG) {
    // two tables, two captured graphs; the H2D for replay k+1 runs on a side stream while
    // replay k (reading the other table) executes
    e->ring = 2;
    CK(cudaMalloc(&e->d_table2, sizeof(uint64_t) * e->n_pad));
    CK(cudaMemset(e->d_table2, 0, sizeof(uint64_t) * e->n_pad));
    CK(cudaHostAlloc((void**)&e->h_stage, sizeof(uint64_t) * e->n_pad * 2, cudaHostAllocDefault));
    memset(e->h_stage, 0, sizeof(uint64_t) * e->n_pad * 2);
    CK(cudaStreamCreateWithFlags(&e->xs, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CK(cudaEventCreateWithFlags(&e->ev_copy[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&e->ev_use[b], cudaEventDisableTiming));
    }
  }
  if (t == CGX_XPORT_FIRST_NODE && n > 512)
    return fail(CGX_E_UNSUPPORTED, "FIRST_NODE transport: more than 512 externals");
  if (t == CGX_XPORT_ROOT_PARAMS) {
    if (n > 512) return fail(CGX_E_UNSUPPORTED, "ROOT_PARAMS transport: more than 512 externals");
    const int cap = n <= 8 ? 8 : n <= 64 ? 64 : 512;
    e->root_fn = kfn_table_write(cap);
    e->root_args.reset(offsetof(TableWriteArgs<8>, ptr) + sizeof(uint64_t) * cap);
    auto* a = reinterpret_cast<TableWriteArgs<8>*>(e->root_args.p);
    a->table = e->d_table;
    a->n = (uint32_t)n;
  } else if (t == CGX_XPORT_ROOT_MAPPED) {
    e->root_fn = kfn_table_mapped();
    e->root_args.reset(sizeof(MappedTableArgs));
    auto* a = reinterpret_cast<MappedTableArgs*>(e->root_args.p);
    a->staging = e->d_stage;
    a->table = e->d_table;
    a->seq = e->d_seq;
    a->ack = e->d_ack;
    a->n = (uint32_t)n;
    a->n_pad = e->n_pad;
    a->ring = (uint32_t)e->ring;
  }
  return CGX_OK;
}

// CGX_SYNC_GRAPH: capture the chain as its data-dependency DAG instead of one serial stream.
// Dependencies come from the slot accesses in chain order (RAW: last writer of every input; WAW:
// last writer of the output; WAR: readers of the output since then). Nodes are spread over
// `graph_streams` capture streams: a node joins the stream whose tail is its most recent
// dependency (so that edge is a PDL edge), else an empty stream, else the stream with the oldest
// tail; dependencies on other streams become graph edges (event record/wait during capture).
// Inside a stream every kernel triggers at entry and griddepcontrol.wait's before it reads another
// node's output or writes its own, so any incoming edge (programmatic or not) is honoured, and
// in-stream order makes every earlier node of the stream an ancestor. The first kernel of a
// stream is captured WITHOUT the PDL attribute: its edges from the fork (root table writer,
// T5 publisher) are then full completion edges, so its pre-wait table fetch is safe. Independent
// branches let the graph executor issue launches on several hardware queues at once instead of
// one PDL cascade (scripts/dag_microbench.cu).
static int capture_dag(cgx_exec* e, int gi, cudaStream_t cs, cgx_transport t) {
  const bool indirect = e->o.mode == CGX_MODE_GRAPH_INDIRECT;
  const size_t nl = e->L.size();
  const std::vector<std::vector<int>> deps = chain_deps(e);
  const int S = e->o.graph_streams ? e->o.graph_streams : 16;
  if (e->dag_s.empty()) {
    e->dag_s.assign((size_t)S + 0, nullptr);
    for (auto& st : e->dag_s) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    e->dag_ev.assign(nl + 1 + (size_t)S, nullptr);   // per node, fork, per-stream join
    for (auto& ev : e->dag_ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  // T5: the by-value prefix up to the table publisher runs on the origin stream before the fork.
  // Without a root node (COPY / SETPARAMS / STALE, the H2D and DEVICE transports) the first node
  // is the prefix: a graph whose branches fork from one completed node replays faster than one
  // with many entry nodes (training chain: 345 vs 378-389 us per step; C2 COPY: 2.7 us),
  // measured with scripts/diag_training_arms.py.
  const bool has_root = indirect && (t == CGX_XPORT_ROOT_MEMCPY || t == CGX_XPORT_ROOT_PARAMS ||
                                     t == CGX_XPORT_ROOT_MAPPED || t == CGX_XPORT_PRELUDE);
  int pre = (indirect && t == CGX_XPORT_FIRST_NODE) ? e->t5_pub : -1;
  if (!has_root && pre < 0 && nl > 1) pre = 0;
  // issue order: a topological order of the post-prefix nodes. Default: chain order.
  // CGX_DAG_ORDER=priority: longest remaining path first (list scheduling; weight per node = one
  // launch + its slot bytes at HBM rate); CGX_DAG_ORDER=level: by dependency depth (all first
  // nodes of every branch, then all second nodes, ...). Any topological order gives the same
  // results (every RAW/WAR/WAW hazard is an edge); chain order replays fastest on C2 and the
  // training chain (scripts/diag_dag_order.py, profiles/r01/dag_order.json).
  std::vector<int> order;
  order.reserve(nl);
  std::vector<double> node_cost(nl, 0.0), prio_v(nl, 0.0);
  for (int p = pre + 1; p < (int)nl; ++p) {
    const Node& n = e->c->nodes[e->L[p].node];
    double bytes = (double)e->c->slots[n.out].nbytes;
    for (int j = 0; j < n.n_in; ++j) bytes += (double)e->c->slots[n.in[j]].nbytes;
    node_cost[p] = 1.0 + bytes / (2.0 * 1024 * 1024);
  }
  {
    const char* ov = getenv("CGX_DAG_ORDER");
    const int how = !ov ? 0 : ov[0] == 'p' ? 1 : ov[0] == 'l' ? 2 : 0;
    std::vector<double>& prio = prio_v;
    std::vector<std::vector<int>> succ(nl);
    std::vector<int> indeg(nl, 0);
    for (int p = pre + 1; p < (int)nl; ++p)
      for (int d : deps[p])
        if (d > pre) {
          succ[d].push_back(p);
          ++indeg[p];
        }
    for (int p = (int)nl - 1; p > pre; --p) {
      double m = 0.0;
      for (int q : succ[p]) m = std::max(m, prio[q]);
      prio[p] = node_cost[p] + m;
    }
    std::vector<int> level(nl, 0);
    for (int p = pre + 1; p < (int)nl; ++p)
      for (int d : deps[p])
        if (d > pre) level[p] = std::max(level[p], level[d] + 1);
    std::vector<int> ready;
    for (int p = pre + 1; p < (int)nl; ++p)
      if (indeg[p] == 0) ready.push_back(p);
    while (!ready.empty()) {
      size_t bi = 0;
      for (size_t i = 1; i < ready.size(); ++i) {
        const int a = ready[i], b = ready[bi];
        const bool better = how == 1 ? (prio[a] > prio[b] || (prio[a] == prio[b] && a < b))
                          : how == 2 ? (level[a] < level[b] || (level[a] == level[b] && a < b))
                                     : a < b;
        if (better) bi = i;
      }
      const int p = ready[bi];
      ready[bi] = ready.back();
      ready.pop_back();
      order.push_back(p);
      for (int q : succ[p])
        if (--indeg[q] == 0) ready.push_back(q);
    }
  }
  std::vector<int> pos(nl, -1);
  for (size_t i = 0; i < order.size(); ++i) pos[order[i]] = (int)i;
  // CGX_DAG_PRIO=<MiB> (experiment): nodes moving at least that many slot bytes get the device's
  // greatest launch priority (the graph is instantiated with cudaGraphInstantiateFlagUseNodePriority)
  if (const char* pv = getenv("CGX_DAG_PRIO")) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    const double thr = atof(pv) * 1024.0 * 1024.0;
    for (int p = pre + 1; p < (int)nl; ++p)
      e->L[p].prio = (node_cost[p] - 1.0) * 2.0 * 1024 * 1024 >= thr ? greatest : 0;
  }
  // stream assignment (pure pass, in issue order; tails hold issue positions' nodes). A node
  // continues the stream whose tail is its latest dependency; a node that starts a new branch goes
  // to an empty stream, else the one with the oldest tail. CGX_DAG_ASSIGN=load: the least-loaded
  // stream instead (load = one launch + slot bytes at HBM rate per node) — measured slower on C2
  // (57.4 vs 54.9 us at 16 streams) and the training chain (341.5 vs 335.7 us),
  // profiles/r01/dag_assign.txt.
  std::vector<int> stream_of(nl, -1), tail((size_t)S, -1);
  {
    const char* av = getenv("CGX_DAG_ASSIGN");
    const bool oldest = !(av && av[0] == 'l');
    std::vector<double> load((size_t)S, 0.0);
    for (int p : order) {
      int best = -1, bestd = -1;
      for (int d : deps[p])
        if (stream_of[d] >= 0 && tail[stream_of[d]] == d && pos[d] > bestd) {
          best = stream_of[d];
          bestd = pos[d];
        }
      if (best < 0 && oldest) {
        for (int k = 0; k < S && best < 0; ++k)
          if (tail[k] < 0) best = k;
        if (best < 0) {
          best = 0;
          for (int k = 1; k < S; ++k)
            if (pos[tail[k]] < pos[tail[best]]) best = k;
        }
      } else if (best < 0) {
        best = 0;
        for (int k = 1; k < S; ++k)
          if (load[k] < load[best]) best = k;
      }
      stream_of[p] = best;
      tail[best] = p;
      load[best] += node_cost[p];
    }
  }
  e->dag_used = 0;
  for (int k = 0; k < S; ++k) e->dag_used += tail[k] >= 0 ? 1u : 0u;
  if (e->dag_used <= 1) {
    // a single branch (a linear chain such as C1 or the decoder): capture it on the origin stream
    // without a fork (same graph, no multi-stream capture overhead on the host launch path); the
    // first kernel after a root node still takes a full completion edge
    bool first = true;
    for (int p = 0; p < (int)nl; ++p) {
      Launch& l = e->L[p];
      const bool saved = l.pdl;
      if (first && p > pre) l.pdl = false;
      if (p > pre) first = false;
      const int rc = issue(e, l, cs);
      l.pdl = saved;
      CKS(rc);
      if (l.kind == LK_KERNEL) CKS(last_captured_node(cs, &l.gnode[gi]));
    }
    return CGX_OK;
  }
  for (int p = 0; p <= pre; ++p) {
    Launch& l = e->L[p];
    CKS(issue(e, l, cs));
    if (l.kind == LK_KERNEL) CKS(last_captured_node(cs, &l.gnode[gi]));
  }
  cudaEvent_t fork = e->dag_ev[nl];
  CK(cudaEventRecord(fork, cs));
  for (auto& st : e->dag_s) CK(cudaStreamWaitEvent(st, fork, 0));
  std::vector<char> need_ev(nl, 0), started((size_t)S, 0);
  for (size_t p = 0; p < nl; ++p)
    for (int d : deps[p]) need_ev[d] = 1;
  for (int p : order) {
    const int best = stream_of[p];
    cudaStream_t st = e->dag_s[best];
    for (int d : deps[p])
      if (d > pre && stream_of[d] != best) CK(cudaStreamWaitEvent(st, e->dag_ev[d], 0));
    Launch& l = e->L[p];
    const bool saved = l.pdl;
    if (!started[best]) l.pdl = false;
    started[best] = 1;
    const int rc = issue(e, l, st);
    l.pdl = saved;
    CKS(rc);
    if (l.kind == LK_KERNEL) CKS(last_captured_node(st, &l.gnode[gi]));
    if (need_ev[p]) CK(cudaEventRecord(e->dag_ev[p], st));
  }

  for (int k = 0; k < S; ++k) {
    CK(cudaEventRecord(e->dag_ev[nl + 1 + k], e->dag_s[k]));
    CK(cudaStreamWaitEvent(cs, e->dag_ev[nl + 1 + k], 0));
  }
  return CGX_OK;
}

static int capture_graph(cgx_exec* e, int gi) {
  cudaStream_t cs = e->cs;
  const cgx_transport t = eff_transport(e->o);
  if (e->o.mode == CGX_MODE_GRAPH_INDIRECT && t == CGX_XPORT_H2D_PINGPONG) {
    // graph gi reads table gi: the `table` field is the first member of ElemArgs and LnArgs
    uint64_t* tab = gi == 0 ? e->d_table : e->d_table2;
    for (auto& l : e->L) {
      if (l.mega) {
        argp<MegaArgs>(l)->table = tab;
        continue;
      }
      if (l.kind == LK_KERNEL && (uses_elem_args(e->c->nodes[l.node].op) ||
                                  e->c->nodes[l.node].op == CGX_OP_LAYERNORM))
        memcpy(l.args.p, &tab, sizeof(tab));
      const Node& gn = e->c->nodes[l.node];
      // a GEMM reads the table for an EXTERNAL A (its rebuilt tensor map) and / or residual
      if (l.kind == LK_KERNEL && gn.op == CGX_OP_GEMM_BF16) decoder_gemm_set_table(l.args.p, tab);
    }
  }
  CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  bool after_root = false;
  bool root_is_copy = false;
  if (e->o.mode == CGX_MODE_GRAPH_INDIRECT) {
    const size_t tb = sizeof(uint64_t) * std::max<size_t>(1, e->c->ext_slots.size());
    if (t == CGX_XPORT_ROOT_MEMCPY) {
      CK(cudaMemcpyAsync(e->d_table, e->h_stage + (size_t)gi * e->n_pad, tb, cudaMemcpyHostToDevice, cs));
      after_root = root_is_copy = true;
    } else if (t == CGX_XPORT_PRELUDE) {
      Launch r;
      r.func = kfn_prelude();
      r.grid = dim3(1);
      r.block = dim3(128);
      r.pdl = false;
      r.args.reset(sizeof(PreludeArgs));
      auto* pa = reinterpret_cast<PreludeArgs*>(r.args.p);
      pa->table = e->d_table;
      pa->patches = static_cast<const PreludePatch*>(e->d_patches);
      pa->n_patches = e->n_patches;
      CKS(issue(e, r, cs));
      CKS(last_captured_node(cs, &e->root_node[gi]));
      // consumers start after the prelude's updates (it triggers after a gpu-scope fence)
    } else if (t == CGX_XPORT_ROOT_PARAMS || t == CGX_XPORT_ROOT_MAPPED) {
      Launch r;
      r.func = e->root_fn;
      r.grid = dim3(1);
      r.block = dim3(t == CGX_XPORT_ROOT_MAPPED ? 64 : 128);
      r.pdl = false;
      r.args.reset(e->root_args.n);
      memcpy(r.args.p, e->root_args.p, e->root_args.n);
      CKS(issue(e, r, cs));
      CKS(last_captured_node(cs, &e->root_node[gi]));
      after_root = true;
    }
  }
  if (e->o.sync_mode == CGX_SYNC_GRAPH) {
    CKS(capture_dag(e, gi, cs, t));
  } else {
  bool first_kernel = true;
  for (auto& l : e->L) {
    if (l.kind == LK_KERNEL && first_kernel && after_root) {
      // the first consumer after a root node fetches table entries after its wait
      if (e->o.mode == CGX_MODE_GRAPH_INDIRECT && !l.mega) {   // (the megakernel reads it after its wait)
        const Node& n = e->c->nodes[l.node];
        const uint32_t f = kFlagTableAfterWait | kFlagTriggerAfterWait;
        if (n.op == CGX_OP_LAYERNORM) argp<LnArgs>(l)->flags |= f;
        else if (uses_elem_args(n.op))
          argp<ElemArgs>(l)->flags = (argp<ElemArgs>(l)->flags | f | ((argp<ElemArgs>(l)->flags & kFlagDataflow) ? kFlagDfPdlWait : 0u)) & ~kFlagDeferWait;
        else return fail(CGX_E_UNSUPPORTED, "first node after the root table writer must be elementwise/LN");
      }
      if (root_is_copy) l.pdl = false;
    }
    if (l.kind == LK_KERNEL) first_kernel = false;
    CKS(issue(e, l, cs));
    if (l.kind == LK_KERNEL) CKS(last_captured_node(cs, &l.gnode[gi]));
  }
  }
  CK(cudaStreamEndCapture(cs, &e->g[gi]));
  const bool devl = e->o.mode == CGX_MODE_GRAPH_INDIRECT && t == CGX_XPORT_DEVICE;
  const unsigned long long prio_flag = getenv("CGX_DAG_PRIO") ? cudaGraphInstantiateFlagUseNodePriority : 0ull;
  CK(cudaGraphInstantiateWithFlags(&e->ge[gi], e->g[gi], (devl ? cudaGraphInstantiateFlagDeviceLaunch : 0ull) | prio_flag));
  CK(cudaGraphUpload(e->ge[gi], e->s));
  size_t nn = 0;
  CK(cudaGraphGetNodes(e->g[gi], nullptr, &nn));
  e->graph_nodes = (uint32_t)nn;
  return CGX_OK;
}

static void exec_free(cgx_exec* e) {
  for (int i = 0; i < 2; ++i) {
    if (e->ge[i]) cudaGraphExecDestroy(e->ge[i]);
    if (e->g[i]) cudaGraphDestroy(e->g[i]);
  }
  if (e->cs) cudaStreamDestroy(e->cs);
  if (e->ph_arena) cudaFree(e->ph_arena);
  if (e->gemm_ws) cudaFree(e->gemm_ws);
  if (e->gemm_cnt) cudaFree(e->gemm_cnt);
  for (void* p : e->gemm_tm_ws) cudaFree(p);
  if (e->df_mem) cudaFree(e->df_mem);
  if (e->dl_ge) cudaGraphExecDestroy(e->dl_ge);
  if (e->dl_g) cudaGraphDestroy(e->dl_g);
  if (e->dl_iter) cudaFree(e->dl_iter);
  if (e->d_trace) cudaFree(e->d_trace);
  if (e->mega_mem) cudaFree(e->mega_mem);
  for (void* b : e->fuse_bufs) cudaFree(b);
  if (e->d_desc) cudaFree(e->d_desc);
  if (e->d_chunk) cudaFree(e->d_chunk);
  if (e->d_table) cudaFree(e->d_table);
  if (e->d_table2) cudaFree(e->d_table2);
  if (e->d_patches) cudaFree(e->d_patches);
  if (e->xs) cudaStreamDestroy(e->xs);
  for (int b = 0; b < 2; ++b) {
    if (e->ev_copy[b]) cudaEventDestroy(e->ev_copy[b]);
    if (e->ev_use[b]) cudaEventDestroy(e->ev_use[b]);
  }
  if (e->h_stage) cudaFreeHost(e->h_stage);
  if (e->h_ack) cudaFreeHost((void*)e->h_ack);
  if (e->h_status) cudaFreeHost((void*)e->h_status);
  if (e->d_seq) cudaFree(e->d_seq);
  for (auto& v : e->ev) cudaEventDestroy(v);
  for (auto& v : e->dag_ev) if (v) cudaEventDestroy(v);
  for (auto& v : e->dag_s) if (v) cudaStreamDestroy(v);
  if (e->c) e->c->live_execs--;
  delete e;
}

static void node_trace_reset(cgx_exec* e);

// CGX_FUSE_ADD_LN: node k is a bf16 ADD whose output the next node, a LAYERNORM over the same
// rows x cols, normalises; not the first two nodes of the range (the FIRST_NODE transport's
// by-value prefix keeps one launch per node there)
static bool fusable_add_ln(const cgx_exec* e, int k) {
  const cgx_chain* c = e->c;
  if (k >= e->last || k <= e->first + 1) return false;
  const Node& a = c->nodes[k];
  const Node& l = c->nodes[k + 1];
  if (a.op != CGX_OP_ADD || l.op != CGX_OP_LAYERNORM || l.in[0] != a.out) return false;
  if (c->slots[a.out].dtype != CGX_BF16 || c->slots[a.in[0]].dtype != CGX_BF16 || c->slots[a.in[1]].dtype != CGX_BF16)
    return false;
  return a.attr.n == (uint64_t)l.attr.rows * l.attr.cols && l.attr.cols <= kLnMaxCols && l.attr.cols % 8 == 0;
}

// CGX_FUSE_LN_GEMM: node k is a LAYERNORM whose output only the next node, a GEMM, reads as A; the
// LN input is the output of the previous launch, a tcgen05 GEMM over the same rows x cols (so that
// GEMM can hand over per-tile row sums); gamma / beta STATIC; more than 4 rows (the small-M path
// has no A prologue)
static bool fusable_ln_gemm(const cgx_exec* e, int k) {
  const cgx_chain* c = e->c;
  if (k >= e->last || k <= e->first + 1 || e->L.size() < 2) return false;
  const Node& ln = c->nodes[k];
  const Node& g = c->nodes[k + 1];
  if (ln.op != CGX_OP_LAYERNORM || g.op != CGX_OP_GEMM_BF16 || g.in[0] != ln.out) return false;
  if (g.attr.flags & CGX_GEMM_ALLREDUCE) return false;
  if (g.attr.M != ln.attr.rows || g.attr.K != ln.attr.cols) return false;
  const bool gemv = decoder_gemm_is_gemv(g.attr.M, g.attr.N, g.attr.K);   // computes its own row statistics
  if (c->slots[ln.in[1]].kind != CGX_SLOT_STATIC || c->slots[ln.in[2]].kind != CGX_SLOT_STATIC) return false;
  if (c->slots[g.in[1]].kind != CGX_SLOT_STATIC) return false;   // W' is prepared once from W
  for (int q = e->first; q <= e->last; ++q)   // nothing else reads the LN output (it is still written)
    if (q != k + 1)
      for (int i = 0; i < c->nodes[q].n_in; ++i)
        if (c->nodes[q].in[i] == ln.out) return false;
  if (gemv) return true;   // (the GEMV's K slices hold whole A rows: its own statistics)
  const Launch& prev = e->L[e->L.size() - 2];   // (the slot for node k is already emplaced)
  // (a producer with a fused ATTN in front — the attention-fed O-proj — still writes its row sums)
  if (prev.kind != LK_KERNEL || prev.mega ||
      (prev.pre_node >= 0 && c->nodes[prev.pre_node].op != CGX_OP_ATTN_CAUSAL)) return false;
  const Node& p = c->nodes[prev.node];
  return p.op == CGX_OP_GEMM_BF16 && p.out == ln.in[0] && p.attr.M == ln.attr.rows && p.attr.N == ln.attr.cols &&
         !(p.attr.flags & CGX_GEMM_ALLREDUCE) && decoder_gemm_is_tcgen05(prev.func);
}

// Build the LN (k) -> GEMM (k + 1) pair as ONE launch of the GEMM with the LayerNorm folded into
// it (k_gemm.cu kGemmLnA: gamma-scaled weights W' prepared here once, row correction in the
// epilogue, the LN output slot stored by the same launch), the previous launch (the producer GEMM)
// writing per-tile row sums. *fused = false (and the LN built as a launch of its own) when either
// kernel cannot take the fused role. Requires the GEMM's W / gamma / beta STATIC (prepared once).
static int build_ln_gemm(cgx_exec* e, int k, bool* fused) {
  cgx_chain* c = e->c;
  const Node& ln = c->nodes[k];
  Launch& l = e->L.back();
  Launch& prev = e->L[e->L.size() - 2];
  *fused = false;
  Launch g;
  CKS(build_launch(e, k + 1, g, k));
  const Node& gn = c->nodes[k + 1];
  const bool gemv = decoder_gemm_is_gemv(gn.attr.M, gn.attr.N, gn.attr.K);
  void* stats = nullptr;
  void* wf = nullptr;
  float* cc = nullptr;
  if (!gemv) {   // the producer GEMM's per-tile row sums (the GEMV computes its own statistics)
    CK(cudaMalloc(&stats, sizeof(float) * 2 * (size_t)prev.grid.x * ln.attr.rows));
    e->fuse_bufs.push_back(stats);
  }
  CK(cudaMalloc(&wf, sizeof(uint16_t) * (size_t)gn.attr.N * gn.attr.K));
  e->fuse_bufs.push_back(wf);
  CK(cudaMalloc(reinterpret_cast<void**>(&cc), sizeof(float) * 2 * (size_t)gn.attr.N));
  e->fuse_bufs.push_back(cc);
  CKS(decoder_ln_fold_prep(c->slots[gn.in[1]].static_ptr, c->slots[ln.in[1]].static_ptr, c->slots[ln.in[2]].static_ptr,
                           gn.attr.N, gn.attr.K, wf, cc, cc + gn.attr.N));
  size_t smem = g.smem;
  if ((gemv || decoder_gemm_is_tcgen05(g.func)) &&
      decoder_gemm_set_ln_a(g.args.p, g.grid, stats, prev.grid.x, c->slots[ln.in[0]].buf, wf, cc, cc + gn.attr.N,
                            c->slots[ln.in[1]].static_ptr, c->slots[ln.in[2]].static_ptr, c->slots[ln.out].buf,
                            ln.attr.eps, &smem, &g.func) == CGX_OK &&
      (gemv || decoder_gemm_set_stats_out(prev.args.p, stats, prev.grid) == CGX_OK)) {
    g.smem = smem;
    g.pre_node = k;
    l = std::move(g);
    *fused = true;
    return CGX_OK;
  }
  return build_launch(e, k, l);   // not fusable after all: the LN keeps its own launch
}

// CGX_FUSE_ATTN_GEMM: node k is an ATTN_CAUSAL whose output the next node, a GEMM, reads as A with
// K = H * D: on the small-M (GEMV) path at T = 1 (decode), on the tcgen05 path at T <= 128 (the GEMM
// computes each head's attention in its K split); not the first two nodes of the range (the
// FIRST_NODE transport's by-value prefix keeps one launch per node there). Other readers of the
// attention output are fine: the fused launch still stores it.
static bool fusable_attn_gemm(const cgx_exec* e, int k) {
  const cgx_chain* c = e->c;
  if (k >= e->last || k <= e->first + 1) return false;
  const Node& at = c->nodes[k];
  const Node& g = c->nodes[k + 1];
  if (at.op != CGX_OP_ATTN_CAUSAL || g.op != CGX_OP_GEMM_BF16 || g.in[0] != at.out) return false;
  if (g.attr.flags & CGX_GEMM_ALLREDUCE) return false;
  if (c->slots[at.in[0]].kind == CGX_SLOT_EXTERNAL) return false;
  if (at.attr.D != 64 || g.attr.M != at.attr.T || g.attr.K != at.attr.H * at.attr.D) return false;
  return decoder_gemm_is_gemv(g.attr.M, g.attr.N, g.attr.K) ? at.attr.T == 1 : at.attr.T <= 128;
}

// Build the ATTN (k) -> GEMV (k + 1) pair as ONE launch of the GEMV forming its A operand from the
// attention's qkv input (k_gemm.cu kGemmAttnA) and storing the ATTN output slot. *fused = false
// (the ATTN built as a launch of its own) when the GEMV cannot take the role.
static int build_attn_gemm(cgx_exec* e, int k, bool* fused) {
  cgx_chain* c = e->c;
  const Node& at = c->nodes[k];
  Launch& l = e->L.back();
  *fused = false;
  Launch g;
  CKS(build_launch(e, k + 1, g, k));
  const Slot& qs = c->slots[at.in[0]];
  const void* qkv = qs.kind == CGX_SLOT_STATIC ? qs.static_ptr : qs.buf;
  if (decoder_gemm_set_attn_a(g.args.p, qkv, c->slots[at.out].buf, at.attr.H, at.attr.D, at.attr.scalar, &g.grid,
                              &g.smem, &g.func) == CGX_OK) {
    g.cluster_z = g.grid.z;
    g.pre_node = k;
    l = std::move(g);
    *fused = true;
    return CGX_OK;
  }
  return build_launch(e, k, l);
}

// ---------------------------------------------------------------- megakernel (cgx_mega.h)

// Compile the exec's node range into the stages of ONE persistent launch:
//  * LAYERNORM and bf16 ADD become row ops of a ROW stage (consecutive ones with the same row
//    shape share a stage: row r is handled by CTA r % G in every ROW stage);
//  * a GEMM is one GEMM stage. When the next node is a row op over its output (or the GEMM ends
//    the range, or its weight slice cannot be staged unsplit) it runs DEFERRED: K split S ways into
//    tasks that store fp32 partials, and the next ROW stage opens with a fixup op that sums them in
//    split order and applies the epilogue (bias, GELU, residual, one bf16 rounding). Otherwise S = 1
//    and the epilogue is applied in the GEMM stage;
//  * ATTN_CAUSAL is one ATTN stage.
// Every stage after the first starts with a grid barrier (each stage reads the previous one's
// output, and consecutive stages partition the work differently).
static int build_mega(cgx_exec* e) {
  cgx_chain* c = e->c;
  const cgx_mode mode = e->o.mode;
  const cgx_transport t = eff_transport(e->o);
  if (mode == CGX_MODE_GRAPH_INDIRECT && t == CGX_XPORT_FIRST_NODE)
    return fail(CGX_E_UNSUPPORTED, "megakernel: the FIRST_NODE transport needs an elementwise first node");
  // INDIRECT reads externals through the table; PRELUDE patches the by-value ext_ptr fields like
  // the patch modes do; COPY binds the placeholders by address
  const bool indirect = mode == CGX_MODE_GRAPH_INDIRECT && t != CGX_XPORT_PRELUDE;
  int dev = 0, G = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, dev));
  if (const char* gv = getenv("CGX_MEGA_CTAS")) G = std::max(1, std::min(G, atoi(gv)));   // diagnostics
  std::vector<MegaStage> stages;
  std::vector<MegaRowOp> ops;
  std::vector<int> ext_of(c->ext_slots.size(), -1), ext_js;
  bool ext_overflow = false;
  auto ref = [&](int si) -> MegaRef {
    const Slot& s = c->slots[si];
    MegaRef r{nullptr, -1, -1};
    if (s.kind == CGX_SLOT_STATIC) r.p = s.static_ptr;
    else if (s.kind == CGX_SLOT_INTERNAL) r.p = s.buf;
    else if (mode == CGX_MODE_GRAPH_COPY) r.p = e->ph[s.ext_j];
    else {
      if (ext_of[s.ext_j] < 0) {
        if ((int)ext_js.size() == kMegaMaxExt) ext_overflow = true;
        else {
          ext_of[s.ext_j] = (int)ext_js.size();
          ext_js.push_back(s.ext_j);
        }
      }
      r.ext = ext_of[s.ext_j];
    }
    return r;
  };
  auto bf16 = [&](int si) { return c->slots[si].dtype == CGX_BF16; };
  int cur_row = -1, pending = -1, pending_node = -1, next_reg = 0;
  int reg_slot[kMegaMaxRegs];
  std::unordered_map<int, int> reg_of;
  size_t ws_floats = 0;
  auto new_stage = [&](uint32_t kind, int node) -> int {
    MegaStage st{};
    st.kind = kind;
    st.barrier = stages.empty() ? 0u : 1u;
    st.node = (uint32_t)node;
    st.next_gemm = -1;
    stages.push_back(st);
    cur_row = -1;
    return (int)stages.size() - 1;
  };
  auto row_ref = [&](int si) -> MegaRef {
    auto it = reg_of.find(si);
    if (it != reg_of.end()) return MegaRef{nullptr, -1, it->second};
    return ref(si);
  };
  auto alloc_reg = [&](int si) -> int32_t {
    const int r = next_reg++ % kMegaMaxRegs;
    if (reg_slot[r] >= 0) reg_of.erase(reg_slot[r]);
    reg_slot[r] = si;
    reg_of[si] = r;
    return r;
  };
  std::string why;
  auto open_row = [&](uint32_t rows, uint32_t cols, int node) -> bool {
    const bool same = cur_row >= 0 && stages[cur_row].rows == rows && stages[cur_row].cols == cols;
    if (same && stages[cur_row].n_ops < kMegaMaxRowOps) return true;
    if (cols > kMegaMaxCols || cols % 8 || rows == 0) {
      why = "row shape " + std::to_string(rows) + "x" + std::to_string(cols) + " (cols <= 2048, % 8)";
      return false;
    }
    const int si = new_stage(kMegaRow, node);
    // a full ROW stage continues without a barrier: same rows on the same CTAs, same columns on
    // the same threads, so every value it reads was written by the reading thread itself
    if (same) stages[si].barrier = 0;
    cur_row = si;
    stages[si].rows = rows;
    stages[si].cols = cols;
    stages[si].op0 = (uint32_t)ops.size();
    reg_of.clear();
    for (int& r : reg_slot) r = -1;
    next_reg = 0;
    if (pending >= 0) {   // the deferred GEMM's epilogue opens this stage
      const MegaStage& g = stages[pending];
      if (g.M != rows || g.N != cols) {
        why = "deferred GEMM output shape";
        return false;
      }
      const Node& gn = c->nodes[pending_node];
      MegaRowOp op{};
      op.kind = kRowFixup;
      op.node = (uint32_t)pending_node;
      op.flags = g.flags & (CGX_GEMM_BIAS | CGX_GEMM_GELU | CGX_GEMM_RESIDUAL);
      op.S = g.split;
      op.a = op.b = MegaRef{nullptr, -1, -1};
      op.c = (g.flags & CGX_GEMM_BIAS) ? ref(gn.in[2]) : MegaRef{nullptr, -1, -1};
      op.d = (g.flags & CGX_GEMM_RESIDUAL) ? ref(gn.in[3]) : MegaRef{nullptr, -1, -1};
      op.ws = nullptr;   // set once the workspace is allocated
      op.out = c->slots[gn.out].buf;
      op.out_reg = alloc_reg(gn.out);
      ops.push_back(op);
      stages[si].n_ops++;
      pending = -1;
    }
    return true;
  };
  auto flush_pending = [&](int node) -> bool {
    if (pending < 0) return true;
    return open_row(stages[pending].M, stages[pending].N, node);
  };
  int gemm_count = 0;
  for (int k = e->first; k <= e->last; ++k) {
    const Node& n = c->nodes[k];
    const std::string at = "megakernel: node " + std::to_string(k) + ": ";
    if (!bf16(n.out)) return fail(CGX_E_UNSUPPORTED, at + "output must be bf16");
    switch (n.op) {
      case CGX_OP_LAYERNORM: {
        if (!bf16(n.in[0]) || !bf16(n.in[1]) || !bf16(n.in[2])) return fail(CGX_E_UNSUPPORTED, at + "LN operands must be bf16");
        const uint32_t rows = n.attr.rows, cols = n.attr.cols;
        if (pending >= 0 && (stages[pending].M != rows || stages[pending].N != cols) && !flush_pending(k))
          return fail(CGX_E_UNSUPPORTED, at + why);
        if (!open_row(rows, cols, k)) return fail(CGX_E_UNSUPPORTED, at + why);
        MegaRowOp op{};
        op.kind = kRowLn;
        op.node = (uint32_t)k;
        op.a = row_ref(n.in[0]);
        op.b = MegaRef{nullptr, -1, -1};
        op.c = ref(n.in[1]);
        op.d = ref(n.in[2]);
        op.out = c->slots[n.out].buf;
        op.eps = n.attr.eps;
        op.out_reg = alloc_reg(n.out);
        ops.push_back(op);
        stages[cur_row].n_ops++;
        break;
      }
      case CGX_OP_ADD: {
        if (!bf16(n.in[0]) || !bf16(n.in[1])) return fail(CGX_E_UNSUPPORTED, at + "ADD operands must be bf16");
        const uint64_t ne = n.attr.n;
        uint32_t rows = 0, cols = 0;
        if (pending >= 0 && (uint64_t)stages[pending].M * stages[pending].N == ne) {
          rows = stages[pending].M;
          cols = stages[pending].N;
        } else if (cur_row >= 0 && (uint64_t)stages[cur_row].rows * stages[cur_row].cols == ne) {
          rows = stages[cur_row].rows;
          cols = stages[cur_row].cols;
        } else {
          for (uint32_t cc = kMegaMaxCols; cc >= 8; cc -= 8)
            if (ne % cc == 0) {
              cols = cc;
              break;
            }
          rows = cols ? (uint32_t)(ne / cols) : 0;
        }
        if (pending >= 0 && (stages[pending].M != rows || stages[pending].N != cols) && !flush_pending(k))
          return fail(CGX_E_UNSUPPORTED, at + why);
        if (!open_row(rows, cols, k)) return fail(CGX_E_UNSUPPORTED, at + why);
        MegaRowOp op{};
        op.kind = kRowAdd;
        op.node = (uint32_t)k;
        op.a = row_ref(n.in[0]);
        op.b = row_ref(n.in[1]);
        op.c = op.d = MegaRef{nullptr, -1, -1};
        op.out = c->slots[n.out].buf;
        op.out_reg = alloc_reg(n.out);
        ops.push_back(op);
        stages[cur_row].n_ops++;
        break;
      }
      case CGX_OP_GEMM_BF16: {
        if (!flush_pending(k)) return fail(CGX_E_UNSUPPORTED, at + why);
        const uint32_t M = n.attr.M, N = n.attr.N, K = n.attr.K, fl = n.attr.flags;
        if (fl & CGX_GEMM_ALLREDUCE) return fail(CGX_E_UNSUPPORTED, at + "GEMM with a fused all-reduce");
        if (K % 64 || N % 16 || M == 0) return fail(CGX_E_UNSUPPORTED, at + "GEMM shape (K % 64, N % 16)");
        if (c->slots[n.in[0]].kind == CGX_SLOT_EXTERNAL) return fail(CGX_E_UNSUPPORTED, at + "EXTERNAL A operand");
        if (c->slots[n.in[1]].kind != CGX_SLOT_STATIC) return fail(CGX_E_UNSUPPORTED, at + "W must be STATIC");
        const uint32_t kb = K / 64, m_tiles = (M + 127) / 128;
        auto w_fits = [&](uint32_t bn, uint32_t kps) { return (uint64_t)bn * kps * 128u <= kMegaWBytes; };
        // direct (unsplit) tiling: the widest N tile whose whole-K weight slice fits one W buffer
        uint32_t bn_direct = 0;
        for (uint32_t bn : {64u, 32u, 16u})
          if (N % bn == 0 && w_fits(bn, kb)) {
            bn_direct = bn;
            break;
          }
        bool next_row = false;
        if (k < e->last) {
          const Node& nx = c->nodes[k + 1];
          if (nx.op == CGX_OP_LAYERNORM || nx.op == CGX_OP_ADD)
            for (int i = 0; i < nx.n_in; ++i) next_row = next_row || nx.in[i] == n.out;
        }
        const bool deferred = next_row || k == e->last || bn_direct == 0;
        const int si = new_stage(kMegaGemm, k);
        MegaStage& g = stages[si];
        g.M = M;
        g.N = N;
        g.K = K;
        g.flags = fl & (CGX_GEMM_BIAS | CGX_GEMM_GELU | CGX_GEMM_RESIDUAL);
        g.m_tiles = m_tiles;
        g.deferred = deferred ? 1u : 0u;
        if (deferred) {
          // widest N tile, then the most K splits (<= 16) that keep tasks <= G and the slice staged
          g.bn = N % 64 == 0 ? 64u : N % 32 == 0 ? 32u : 16u;
          g.split = 0;
          for (uint32_t sp = std::min<uint32_t>(kMegaMaxSplit, kb); sp >= 1; --sp)
            if (kb % sp == 0 && (uint64_t)m_tiles * (N / g.bn) * sp <= (uint64_t)G && w_fits(g.bn, kb / sp)) {
              g.split = sp;
              break;
            }
          if (g.split == 0)
            for (uint32_t sp = 1; sp <= std::min<uint32_t>(kMegaMaxSplit, kb); ++sp)   // more tasks than CTAs
              if (kb % sp == 0 && w_fits(g.bn, kb / sp)) {
                g.split = sp;
                break;
              }
          if (g.split == 0) return fail(CGX_E_UNSUPPORTED, at + "no K split stages the weight slice");
          ws_floats = std::max<size_t>(ws_floats, (size_t)g.split * M * N);
          pending = si;
          pending_node = k;
        } else {
          g.bn = bn_direct;
          g.split = 1;
        }
        g.n_tiles = N / g.bn;
        g.kps = kb / g.split;
        g.ga = g.kps % 4 == 0 ? 4u : g.kps % 2 == 0 ? 2u : 1u;
        g.w_buf = (uint32_t)(gemm_count++ % 2);
        g.bias = (fl & CGX_GEMM_BIAS) ? ref(n.in[2]) : MegaRef{nullptr, -1, -1};
        g.res = (fl & CGX_GEMM_RESIDUAL) ? ref(n.in[3]) : MegaRef{nullptr, -1, -1};
        g.out = c->slots[n.out].buf;
        break;
      }
      case CGX_OP_ATTN_CAUSAL: {
        if (!flush_pending(k)) return fail(CGX_E_UNSUPPORTED, at + why);
        if (!bf16(n.in[0])) return fail(CGX_E_UNSUPPORTED, at + "attention operands must be bf16");
        if (n.attr.D != 64 || n.attr.T > 256) return fail(CGX_E_UNSUPPORTED, at + "attention (D == 64, T <= 256)");
        const int si = new_stage(kMegaAttn, k);
        stages[si].T = n.attr.T;
        stages[si].H = n.attr.H;
        stages[si].scale = n.attr.scalar;
        stages[si].qkv = ref(n.in[0]);
        stages[si].aout = c->slots[n.out].buf;
        break;
      }
      default:
        return fail(CGX_E_UNSUPPORTED, at + "op not supported by the megakernel");
    }
  }
  if (!flush_pending(e->last)) return fail(CGX_E_UNSUPPORTED, "megakernel: " + why);
  if (ext_overflow) return fail(CGX_E_UNSUPPORTED, "megakernel: more than 8 EXTERNAL operands");
  for (size_t i = 0; i + 1 < stages.size(); ++i) stages[i].bar_next = stages[i + 1].barrier;
  for (auto& op : ops) {   // operands fetched from memory (not a register of the stage), per column
    const MegaRef* r = &op.a;
    auto present = [](const MegaRef& x) { return x.p != nullptr || x.ext >= 0 || x.reg >= 0; };
    op.pf = op.col = 0;
    for (uint32_t x = 0; x < 4; ++x)
      if (present(r[x]) && r[x].reg < 0) op.pf |= 1u << x;
    if (op.kind == kRowLn) op.col = 0xCu;                  // gamma, beta
    else if (op.kind == kRowFixup) op.col = 0x4u;          // bias
  }
  int first_gemm = -1, prev = -1;
  for (int i = 0; i < (int)stages.size(); ++i)
    if (stages[i].kind == kMegaGemm) {
      if (prev >= 0) stages[prev].next_gemm = i;
      else first_gemm = i;
      prev = i;
    }
  // device blob: stage records | tensor maps (2 per GEMM stage) | ws | barrier words | stage trace
  auto al = [](size_t v, size_t a) { return (v + a - 1) / a * a; };
  const size_t o_st = 0;
  const size_t o_tm = al(o_st + (size_t)kMegaRec * stages.size(), 128);
  const size_t o_ws = al(o_tm + 128 * 2 * stages.size(), 256);
  const size_t o_bar = al(o_ws + sizeof(float) * ws_floats, 256);
  const size_t o_tr = o_bar + 8192;   // per-CTA words [0, 256), spread counters, go word
  const size_t total = o_tr + sizeof(unsigned long long) * 8 * stages.size() * G;
  CK(cudaMalloc(&e->mega_mem, total));
  uint8_t* d = static_cast<uint8_t*>(e->mega_mem);
  std::vector<uint8_t> h(o_bar, 0);
  for (size_t i = 0; i < stages.size(); ++i) {
    MegaStage& g = stages[i];
    if (g.kind != kMegaGemm) continue;
    const Node& gn = c->nodes[g.node];
    uint8_t* tma = h.data() + o_tm + 256 * i;
    if (decoder_encode_kmajor(tma, c->slots[gn.in[0]].buf, g.M, g.K, 128, g.ga) != CGX_OK ||
        decoder_encode_kmajor(tma + 128, c->slots[gn.in[1]].static_ptr, g.N, g.K, g.bn, g.kps) != CGX_OK)
      return fail(CGX_E_CUDA, "megakernel: cuTensorMapEncodeTiled failed (node " + std::to_string(g.node) + ")");
    g.tmA = reinterpret_cast<uint64_t>(d + o_tm + 256 * i);
    g.tmW = g.tmA + 128;
    g.ws = g.deferred ? reinterpret_cast<float*>(d + o_ws) : nullptr;
  }
  for (auto& op : ops)
    if (op.kind == kRowFixup) op.ws = reinterpret_cast<const float*>(d + o_ws);
  for (size_t i = 0; i < stages.size(); ++i) {
    uint8_t* rec = h.data() + o_st + (size_t)kMegaRec * i;
    memcpy(rec, &stages[i], sizeof(MegaStage));
    if (stages[i].kind == kMegaRow)
      for (uint32_t k = 0; k < stages[i].n_ops; ++k)
        memcpy(rec + kMegaDescStage + sizeof(MegaRowOp) * k, &ops[stages[i].op0 + k], sizeof(MegaRowOp));
  }
  CK(cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(d + o_bar, 0, total - o_bar));
  e->mega = true;
  e->mega_strace = reinterpret_cast<unsigned long long*>(d + o_tr);
  e->mega_ctas = (uint32_t)G;
  e->mega_stages = (uint32_t)stages.size();
  Launch l;
  l.kind = LK_KERNEL;
  l.node = e->first;
  l.func = kfn_mega();
  l.grid = dim3((unsigned)G);
  l.block = dim3(kMegaThreads);
  l.smem = mega_smem_bytes();
  l.pdl = !e->o.no_pdl;
  l.coop = getenv("CGX_MEGA_NOCOOP") == nullptr;
  l.mega = true;
  l.args.reset(sizeof(MegaArgs));
  MegaArgs* a = argp<MegaArgs>(l);
  a->recs = d + o_st;
  a->n_stages = (uint32_t)stages.size();
  a->G = (uint32_t)G;
  a->first_gemm = first_gemm;
  a->table = indirect ? e->d_table : nullptr;
  a->n_ext = (uint32_t)ext_js.size();
  for (int i = 0; i < kMegaMaxExt; ++i) {
    a->ext_ptr[i] = nullptr;
    a->ext_t[i] = -1;
  }
  for (size_t i = 0; i < ext_js.size(); ++i) {
    if (indirect) {
      a->ext_t[i] = ext_js[i];
    } else {
      a->ext_ptr[i] = e->cur[ext_js[i]];
      l.ext.push_back({offsetof(MegaArgs, ext_ptr) + sizeof(void*) * i, offsetof(MegaArgs, ext_t) + sizeof(int32_t) * i,
                       ext_js[i]});
    }
  }
  a->flags = reinterpret_cast<uint32_t*>(d + o_bar);
  {
    const char* bm = getenv("CGX_MEGA_BAR");      // measurement knobs: barrier variant / poll back-off
    const char* bs = getenv("CGX_MEGA_BAR_NS");
    a->bar_mode = bm ? (uint32_t)atoi(bm) : 3u;
    a->bar_sleep_ns = bs ? (uint32_t)atoi(bs) : 0u;
    a->null_work = getenv("CGX_MEGA_NULL") ? 1u : 0u;
    a->dbg = getenv("CGX_MEGA_DBG") ? (uint32_t)atoi(getenv("CGX_MEGA_DBG")) : 0u;
  }
  a->st = dev_status(e);
  a->ntrace = nullptr;
  const char* tv = getenv("CGX_MEGA_TRACE");
  a->strace = (tv && tv[0] == '1') ? e->mega_strace : nullptr;
  e->L.clear();
  e->L.push_back(std::move(l));
  return CGX_OK;
}

extern "C" int cgx_exec_create_ex(cgx_chain* c, const cgx_exec_opts* opts, void* stream, cgx_exec** out) {
  if (!c || !out) return fail(CGX_E_INVALID_ARG, "exec_create: NULL argument");
  cgx_exec_opts o{};
  if (opts) o = *opts;
  if (o.mode < CGX_MODE_EAGER || o.mode > CGX_MODE_GRAPH_STALE) return fail(CGX_E_INVALID_ARG, "exec_create: mode");
  if (o.transport < CGX_XPORT_DEFAULT || o.transport > CGX_XPORT_DEVICE)
    return fail(CGX_E_INVALID_ARG, "exec_create: transport");
  if (o.copy_impl < 0 || o.copy_impl > 2) return fail(CGX_E_INVALID_ARG, "exec_create: copy_impl");
  if (o.sync_mode < CGX_SYNC_AUTO || o.sync_mode > CGX_SYNC_DATAFLOW) return fail(CGX_E_INVALID_ARG, "exec_create: sync_mode");
  if (o.graph_streams < 0 || o.graph_streams > 64) return fail(CGX_E_INVALID_ARG, "exec_create: graph_streams (0..64)");
  if (o.megakernel < 0 || o.megakernel > 1) return fail(CGX_E_INVALID_ARG, "exec_create: megakernel (0 or 1)");
  if (o.fuse & ~(CGX_FUSE_ADD_LN | CGX_FUSE_LN_GEMM | CGX_FUSE_ATTN_GEMM))
    return fail(CGX_E_INVALID_ARG, "exec_create: fuse (unknown bits)");
  const int K = (int)c->nodes.size();
  if (K == 0) return fail(CGX_E_STATE, "exec_create: empty chain");
  const int first = o.first_node, last = o.n_nodes ? o.first_node + o.n_nodes - 1 : K - 1;
  if (first < 0 || first >= K || last < first || last >= K) return fail(CGX_E_INVALID_ARG, "exec_create: node range");
  CK(cudaSetDevice(c->device));
  CKS(chain_allocate(c));
  auto* e = new cgx_exec();
  e->c = c;
  c->live_execs++;
  e->o = o;
  // AUTO: graph modes with PDL capture the chain's dependency DAG (CGX_SYNC_GRAPH); without PDL
  // (no_pdl) the serial capture with plain stream edges is kept.
  if (e->o.sync_mode == CGX_SYNC_AUTO)
    e->o.sync_mode = (e->o.mode != CGX_MODE_EAGER && !e->o.no_pdl) ? CGX_SYNC_GRAPH : CGX_SYNC_DATAFLOW;
  e->s = static_cast<cudaStream_t>(stream);
  e->first = first;
  e->last = last;
  const int n_ext = (int)c->ext_slots.size();
  e->cur.assign(n_ext, nullptr);
  std::vector<bool> read(n_ext, false);
  for (int k = first; k <= last; ++k)
    for (int i = 0; i < c->nodes[k].n_in; ++i)
      if (c->slots[c->nodes[k].in[i]].kind == CGX_SLOT_EXTERNAL) read[c->slots[c->nodes[k].in[i]].ext_j] = true;
  for (int j = 0; j < n_ext; ++j)
    if (read[j]) e->ext_read.push_back(j);
  auto bail = [&](int st) { exec_free(e); return st; };
  int st;
  {
    uint32_t* hs = nullptr;
    cudaError_t ce = cudaHostAlloc((void**)&hs, 64, cudaHostAllocMapped);
    if (ce != cudaSuccess) return bail(cuda_fail(ce, "status word", __LINE__));
    *hs = 0;
    e->h_status = hs;
    ce = cudaHostGetDevicePointer((void**)&e->d_status, hs, 0);
    if (ce != cudaSuccess) return bail(cuda_fail(ce, "status word", __LINE__));
    e->spin_timeout_ns = spin_timeout_ns();
  }
  if (o.mode == CGX_MODE_GRAPH_COPY && (st = setup_copy(e)) != CGX_OK) return bail(st);
  if (o.mode == CGX_MODE_GRAPH_INDIRECT && (st = setup_table(e)) != CGX_OK) return bail(st);
  {
    size_t ws = 0, cnt = 0;
    for (int k = first; k <= last; ++k)
      if (c->nodes[k].op == CGX_OP_GEMM_BF16) {
        size_t w1, c1;
        decoder_gemm_plan(c->nodes[k].attr.M, c->nodes[k].attr.N, c->nodes[k].attr.K, &w1, &c1);
        ws = std::max(ws, w1);
        cnt += c1;            // counters are per GEMM node (split counts differ between nodes)
      }
    cudaError_t ce = cudaSuccess;
    if (ws) ce = cudaMalloc(&e->gemm_ws, ws);
    if (ce == cudaSuccess && cnt) ce = cudaMalloc(&e->gemm_cnt, cnt);
    if (ce == cudaSuccess && cnt) ce = cudaMemset(e->gemm_cnt, 0, cnt);
    if (ce != cudaSuccess) return bail(cuda_fail(ce, "gemm workspace", __LINE__));
  }
  if (o.megakernel) {
    if ((st = build_mega(e)) != CGX_OK) return bail(st);
  } else {
    e->t5_pub = (last > first && tw_capable(c->nodes[first + 1].op)) ? 1 : 0;
    e->L.reserve((size_t)(last - first + 1));
    for (int k = first; k <= last; ++k) {
      e->L.emplace_back();
      if ((o.fuse & CGX_FUSE_ADD_LN) && fusable_add_ln(e, k)) {
        if ((st = build_launch(e, k + 1, e->L.back(), k)) != CGX_OK) return bail(st);
        ++k;
      } else if ((o.fuse & CGX_FUSE_LN_GEMM) && fusable_ln_gemm(e, k)) {
        bool fused = false;
        if ((st = build_ln_gemm(e, k, &fused)) != CGX_OK) return bail(st);
        if (fused) ++k;
      } else if ((o.fuse & CGX_FUSE_ATTN_GEMM) && fusable_attn_gemm(e, k)) {
        bool fused = false;
        if ((st = build_attn_gemm(e, k, &fused)) != CGX_OK) return bail(st);
        if (fused) ++k;
      } else if ((st = build_launch(e, k, e->L.back())) != CGX_OK) {
        return bail(st);
      }
    }
  }
  set_prewait_masks(e);
  if ((st = set_sync_flags(e)) != CGX_OK) return bail(st);
  if (const char* dv = getenv("CGX_DEBUG_NOOP"); dv && (dv[0] == '1' || dv[0] == '2') && o.mode != CGX_MODE_EAGER) {
    for (size_t p = 0; p < e->L.size(); ++p)
      if (e->L[p].kind == LK_KERNEL && df_capable(c->nodes[e->L[p].node], c->slots[c->nodes[e->L[p].node].out].dtype))
        argp<ElemArgs>(e->L[p])->flags |= dv[0] == '1' ? kFlagDbgNoop : kFlagDbgNoWork;
  }
  if (const char* tv = getenv("CGX_NODE_TRACE"); g_force_trace || (tv && tv[0] == '1')) {
    const size_t nb = sizeof(unsigned long long) * 3 * e->L.size();
    cudaError_t ce = cudaMalloc(&e->d_trace, nb);
    if (ce != cudaSuccess) return bail(cuda_fail(ce, "node trace", __LINE__));
    node_trace_reset(e);
    for (size_t p = 0; p < e->L.size(); ++p) {
      if (e->L[p].kind != LK_KERNEL) continue;
      const Node& tn = c->nodes[e->L[p].node];
      unsigned long long* nt = e->d_trace + 3 * p;
      if (e->L[p].mega) argp<MegaArgs>(e->L[p])->ntrace = nt;
      else if (uses_elem_args(tn.op)) argp<ElemArgs>(e->L[p])->trace = nt;
      else if (tn.op == CGX_OP_LAYERNORM) argp<LnArgs>(e->L[p])->ntrace = nt;
      else if (tn.op == CGX_OP_ATTN_CAUSAL) argp<AttnArgs>(e->L[p])->ntrace = nt;
      else if (tn.op == CGX_OP_GEMM_BF16) decoder_gemm_set_node_trace(e->L[p].args.p, nt);
    }
  }
  if (o.mode != CGX_MODE_EAGER) {
    cudaError_t ce = cudaStreamCreateWithFlags(&e->cs, cudaStreamNonBlocking);
    if (ce != cudaSuccess) return bail(cuda_fail(ce, "cudaStreamCreate", __LINE__));
    const bool t7 = o.mode == CGX_MODE_GRAPH_INDIRECT && eff_transport(o) == CGX_XPORT_PRELUDE;
    if (t7) {
      uint32_t np = 0;
      for (auto& l : e->L)
        if (l.kind == LK_KERNEL && !l.ext.empty()) {
          l.dev_updatable = true;
          np += (uint32_t)l.ext.size();
        }
      e->n_patches = np;
      cudaError_t pe = cudaMalloc(&e->d_patches, sizeof(PreludePatch) * std::max<uint32_t>(np, 1));
      if (pe != cudaSuccess) return bail(cuda_fail(pe, "prelude patches", __LINE__));
    }
    e->n_graphs = (o.mode == CGX_MODE_GRAPH_INDIRECT && (eff_transport(o) == CGX_XPORT_ROOT_MEMCPY ||
                                                          eff_transport(o) == CGX_XPORT_H2D_PINGPONG))
                      ? 2 : 1;
    for (int gi = 0; gi < e->n_graphs; ++gi)
      if ((st = capture_graph(e, gi)) != CGX_OK) {
        cudaStreamCaptureStatus cst;
        if (cudaStreamIsCapturing(e->cs, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
          cudaGraph_t junk = nullptr;
          cudaStreamEndCapture(e->cs, &junk);
          if (junk) cudaGraphDestroy(junk);
        }
        return bail(st);
      }
    // the DAG's capture streams and events are not referenced by the instantiated graphs
    for (auto& v : e->dag_ev) if (v) cudaEventDestroy(v);
    for (auto& v : e->dag_s) if (v) cudaStreamDestroy(v);
    e->dag_ev.clear();
    e->dag_s.clear();
    if (t7) {
      // patch list: (device node handle, byte offset of the pointer field, pointer cell); the
      // offsets are the fields the runtime itself patches in SETPARAMS mode — the same ones the
      // NEXT-2 byte-pattern discovery finds (tests/test_gpu_next.py)
      std::vector<PreludePatch> pp;
      for (auto& l : e->L)
        if (l.dev_updatable) {
          if (!l.dev_node) return bail(fail(CGX_E_CUDA, "prelude: no device node handle returned by capture"));
          for (auto& f : l.ext) pp.push_back({l.dev_node, (uint32_t)f.off, (uint32_t)f.ext_j});
        }
      cudaError_t pe = pp.empty() ? cudaSuccess
                                  : cudaMemcpy(e->d_patches, pp.data(), sizeof(PreludePatch) * pp.size(),
                                               cudaMemcpyHostToDevice);
      if (pe != cudaSuccess) return bail(cuda_fail(pe, "prelude patch upload", __LINE__));
    }
    cudaError_t se = cudaStreamSynchronize(e->s);
    if (se != cudaSuccess) return bail(cuda_fail(se, "upload sync", __LINE__));
  }
  int kernels = 0;
  for (auto& l : e->L) kernels += l.kind == LK_KERNEL;
  e->st.n_nodes = (uint32_t)(last - first + 1);
  e->st.n_ext = (uint32_t)n_ext;
  e->st.n_graph_nodes = e->graph_nodes;
  e->st.n_deferred = 0;
  for (auto& l : e->L)
    if (l.kind == LK_KERNEL && !l.mega && is_elemwise(e->c->nodes[l.node].op))
      e->st.n_deferred += (argp<ElemArgs>(l)->flags & kFlagDeferWait) ? 1u : 0u;
  e->st.dataflow = e->dataflow ? 1u : 0u;
  e->st.dag_streams = e->dag_used;
  e->st.mode = (uint32_t)o.mode;
  e->st.transport = o.mode == CGX_MODE_GRAPH_INDIRECT ? (uint32_t)eff_transport(o) : 0;
  e->st.kernels_per_replay = (uint32_t)kernels + (o.mode == CGX_MODE_GRAPH_COPY && o.copy_impl != 1 && !e->ext_read.empty()) +
                             ((o.mode == CGX_MODE_GRAPH_INDIRECT && e->root_fn) ? 1 : 0);
  *out = e;
  return CGX_OK;
}

extern "C" int cgx_exec_create(cgx_chain* c, cgx_mode mode, void* stream, cgx_exec** out) {
  cgx_exec_opts o{};
  o.mode = mode;
  return cgx_exec_create_ex(c, &o, stream, out);
}

extern "C" int cgx_exec_destroy(cgx_exec* e) {
  if (!e) return CGX_OK;
  cudaStreamSynchronize(e->s);
  exec_free(e);
  return CGX_OK;
}

// ---------------------------------------------------------------------------- bind
static int validate_ptrs(cgx_exec* e, const void* const* p, int n) {
  for (int j = 0; j < n; ++j) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p[j]);
    if (!a) return fail(CGX_E_MISSING_INPUT, "bind: NULL input " + std::to_string(j));
    if (a & 15) return fail(CGX_E_MISALIGNED, "bind: input " + std::to_string(j) + " not 16-byte aligned");
    if (e->o.validate == 2) continue;
    if (e->o.validate == 0 && e->validated.count(a)) continue;
    cudaPointerAttributes at{};
    cudaError_t ce = cudaPointerGetAttributes(&at, p[j]);
    if (ce != cudaSuccess) {
      cudaGetLastError();
      return fail(CGX_E_NOT_ELIGIBLE, "bind: input " + std::to_string(j) + " is not a CUDA allocation");
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
      return fail(CGX_E_NOT_ELIGIBLE, "bind: input " + std::to_string(j) +
                                          " is host memory (dangling-host-pointer hazard, P:L264-265)");
    if (at.type == cudaMemoryTypeDevice && at.device != e->c->device)
      return fail(CGX_E_NOT_ELIGIBLE, "bind: input " + std::to_string(j) + " lives on another device");
    if (e->o.validate == 0) {
      if (e->validated.size() > 65536) e->validated.clear();
      e->validated.insert(a);
    }
  }
  return CGX_OK;
}

static inline void patch_images(cgx_exec* e) {
  for (auto& l : e->L)
    for (auto& f : l.ext) memcpy(l.args.p + f.off, &e->cur[f.ext_j], sizeof(void*));
}

static int setparams_all(cgx_exec* e, uint32_t* calls) {
  uint32_t n = 0;
  for (auto& l : e->L) {
    if (l.ext.empty()) continue;
    cudaKernelNodeParams kp{};
    kp.func = const_cast<void*>(l.func);
    kp.gridDim = l.grid;
    kp.blockDim = l.block;
    kp.sharedMemBytes = (unsigned)l.smem;
    void* argv[1] = {l.args.p};
    kp.kernelParams = argv;
    for (int gi = 0; gi < e->n_graphs; ++gi) CK(cudaGraphExecKernelNodeSetParams(e->ge[gi], l.gnode[gi], &kp));
    ++n;
  }
  *calls = n;
  return CGX_OK;
}

extern "C" int cgx_bind(cgx_exec* e, const void* const* ext, int n_ext) {
  if (!e) return fail(CGX_E_INVALID_ARG, "bind: exec is NULL");
  const int N = (int)e->c->ext_slots.size();
  if (n_ext != N || (N > 0 && !ext)) return fail(CGX_E_MISSING_INPUT, "bind: expected " + std::to_string(N) + " inputs");
  CKS(validate_ptrs(e, ext, N));
  for (int j = 0; j < N; ++j) e->cur[j] = ext[j];
  e->st.bytes_data_rebound = e->st.bytes_ptr_rebound = 0;
  e->st.n_setparam_calls = e->st.n_copy_tensors = 0;
  const cgx_chain* c = e->c;
  switch (e->o.mode) {
    case CGX_MODE_EAGER:
      patch_images(e);
      break;
    case CGX_MODE_GRAPH_SETPARAMS:
      patch_images(e);
      CKS(setparams_all(e, &e->st.n_setparam_calls));
      break;
    case CGX_MODE_GRAPH_STALE:
      if (!e->stale_frozen) {   // recorded by value at the first bind, never again
        patch_images(e);
        CKS(setparams_all(e, &e->st.n_setparam_calls));
        e->stale_frozen = true;
      }
      break;
    case CGX_MODE_GRAPH_COPY: {
      uint64_t bytes = 0;
      uint32_t nt = 0;
      if (e->o.copy_impl == 1) {
        for (int j : e->ext_read)
          if (ext[j] != e->ph[j]) {
            const uint64_t nb = c->slots[c->ext_slots[j]].nbytes;
            CK(cudaMemcpyAsync(e->ph[j], ext[j], nb, cudaMemcpyDeviceToDevice, e->s));
            bytes += nb;
            ++nt;
          }
      } else if (!e->ext_read.empty()) {
        auto* a = reinterpret_cast<CopyArgs<8>*>(e->copy_args.p);
        const void** src = a->src;
        for (size_t t = 0; t < e->ext_read.size(); ++t) {
          const int j = e->ext_read[t];
          src[t] = ext[j];
          if (ext[j] != e->ph[j]) {
            bytes += c->slots[c->ext_slots[j]].nbytes;
            ++nt;
          }
        }
        if (nt) {
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = e->copy_grid;
          cfg.blockDim = dim3(e->copy_block);
          cfg.dynamicSmemBytes = e->copy_smem;
          cfg.stream = e->s;
          void* argv[1] = {e->copy_args.p};
          CK(cudaLaunchKernelExC(&cfg, e->copy_fn, argv));
        }
      }
      e->st.bytes_data_rebound = bytes;
      e->st.n_copy_tensors = nt;
      break;
    }
    case CGX_MODE_GRAPH_INDIRECT: {
      const cgx_transport t = eff_transport(e->o);
      if (t == CGX_XPORT_FIRST_NODE) {
        patch_images(e);   // by-value operands of launches 0..t5_pub
        Launch& lp = e->L[e->t5_pub];
        memcpy(lp.args.p + lp.tw_ptr_off, ext, sizeof(uint64_t) * N);
        for (int i = 0; i <= e->t5_pub; ++i) {
          Launch& l = e->L[i];
          if (i != e->t5_pub && l.ext.empty()) continue;
          cudaKernelNodeParams kp{};
          kp.func = const_cast<void*>(l.func);
          kp.gridDim = l.grid;
          kp.blockDim = l.block;
          kp.sharedMemBytes = (unsigned)l.smem;
          void* argv[1] = {l.args.p};
          kp.kernelParams = argv;
          CK(cudaGraphExecKernelNodeSetParams(e->ge[0], l.gnode[0], &kp));
          e->st.n_setparam_calls++;
        }
      } else if (t == CGX_XPORT_ROOT_PARAMS) {
        auto* a = reinterpret_cast<TableWriteArgs<8>*>(e->root_args.p);
        memcpy(a->ptr, ext, sizeof(uint64_t) * N);
        cudaKernelNodeParams kp{};
        kp.func = const_cast<void*>(e->root_fn);
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(128);
        void* argv[1] = {e->root_args.p};
        kp.kernelParams = argv;
        CK(cudaGraphExecKernelNodeSetParams(e->ge[0], e->root_node[0], &kp));
      } else if (t == CGX_XPORT_H2D_PINGPONG) {
        const int b = (int)(e->seq % 2);
        if (e->ev_copy_set[b]) CK(cudaEventSynchronize(e->ev_copy[b]));   // staging b free again
        uint64_t* h = e->h_stage + (size_t)b * e->n_pad;
        memcpy(h, ext, sizeof(uint64_t) * N);
        if (e->ev_use_set[b]) CK(cudaStreamWaitEvent(e->xs, e->ev_use[b], 0));   // replay k-2 done
        CK(cudaMemcpyAsync(b == 0 ? e->d_table : e->d_table2, h, sizeof(uint64_t) * N, cudaMemcpyHostToDevice,
                           e->xs));
        CK(cudaEventRecord(e->ev_copy[b], e->xs));
        e->ev_copy_set[b] = true;
      } else if (t == CGX_XPORT_H2D || t == CGX_XPORT_PRELUDE || t == CGX_XPORT_DEVICE) {
        const int slot = (int)(e->seq % e->ring);
        if (e->ev_used[slot]) CK(cudaEventSynchronize(e->ev[slot]));
        uint64_t* h = e->h_stage + (size_t)slot * e->n_pad;
        memcpy(h, ext, sizeof(uint64_t) * N);
        CK(cudaMemcpyAsync(e->d_table, h, sizeof(uint64_t) * N, cudaMemcpyHostToDevice, e->s));
        CK(cudaEventRecord(e->ev[slot], e->s));
        e->ev_used[slot] = true;
      } else if (t == CGX_XPORT_ROOT_MEMCPY) {
        const int b = (int)(e->seq % 2);
        if (e->ev_used[b]) CK(cudaEventSynchronize(e->ev[b]));   // exec b's last replay done
        memcpy(e->h_stage + (size_t)b * e->n_pad, ext, sizeof(uint64_t) * N);
      } else {  // ROOT_MAPPED: replay number r reads ring slot r % ring
        if (!e->launched_since_bind) e->seq--;     // overwrite the not-yet-launched slot
        const uint64_t need = e->seq >= (uint64_t)e->ring ? e->seq - e->ring + 1 : 0;
        if (*e->h_ack < need) {   // slot still owned by an in-flight replay: wait (bounded)
          const double t_start = now_us();
          while (*e->h_ack < need) {
            if (now_us() - t_start > 10e6) return fail(CGX_E_CUDA, "bind: ROOT_MAPPED ring slot not released in 10 s");
          }
        }
        uint64_t* h = e->h_stage + (size_t)(e->seq % e->ring) * e->n_pad;
        volatile uint64_t* vh = h;
        for (int j = 0; j < N; ++j) vh[j] = reinterpret_cast<uint64_t>(ext[j]);
      }
      e->st.bytes_ptr_rebound = 8ull * N;
      break;
    }
  }
  e->st.total_bytes_data += e->st.bytes_data_rebound;
  e->st.total_bytes_ptr += e->st.bytes_ptr_rebound;
  e->st.n_binds++;
  e->bound = true;
  e->seq++;
  e->launched_since_bind = false;
  return CGX_OK;
}

// A kernel of an earlier replay reported a device-side failure (DevStatus): sticky, the exec's
// outputs are no longer trustworthy.
static int check_device_status(const cgx_exec* e) {
  const uint32_t w = e->h_status ? *e->h_status : 0u;
  if (!w) return CGX_OK;
  std::string m = "device-side failure reported by an earlier replay of this exec:";
  if (w & kDevErrPeer) m += " peer all-reduce timed out waiting for a rank (lost peer);";
  if (w & kDevErrDataflow) m += " dataflow dependency counter never reached its target;";
  if (w & kDevErrDevLaunch) m += " device-side cudaGraphLaunch failed;";
  return fail(CGX_E_DEVICE, m);
}

extern "C" int cgx_launch(cgx_exec* e) {
  if (!e) return fail(CGX_E_INVALID_ARG, "launch: exec is NULL");
  if (!e->bound) return fail(CGX_E_STATE, "launch: exec was never bound (cgx_bind first)");
  CKS(check_device_status(e));
  if (e->o.mode == CGX_MODE_EAGER) {
    for (auto& l : e->L) CKS(issue(e, l, e->s));
  } else {
    int gi = 0;
    const bool pingpong = e->o.mode == CGX_MODE_GRAPH_INDIRECT && eff_transport(e->o) == CGX_XPORT_ROOT_MEMCPY;
    const bool t6 = e->o.mode == CGX_MODE_GRAPH_INDIRECT && eff_transport(e->o) == CGX_XPORT_H2D_PINGPONG;
    if (pingpong || t6) gi = (int)((e->seq - 1) % 2);
    if (t6) CK(cudaStreamWaitEvent(e->s, e->ev_copy[gi], 0));
    if (e->o.mode == CGX_MODE_GRAPH_INDIRECT && eff_transport(e->o) == CGX_XPORT_ROOT_MAPPED &&
        e->launched_since_bind) {
      // a launch without a fresh bind consumes the next ring slot: republish the bound pointers
      CKS(cgx_bind(e, e->cur.data(), (int)e->cur.size()));
    }
    CK(cudaGraphLaunch(e->ge[gi], e->s));
    if (pingpong) {
      CK(cudaEventRecord(e->ev[gi], e->s));
      e->ev_used[gi] = true;
    }
    if (t6) {
      CK(cudaEventRecord(e->ev_use[gi], e->s));
      e->ev_use_set[gi] = true;
    }
  }
  e->st.n_launches++;
  e->launched_since_bind = true;
  return CGX_OK;
}

extern "C" int cgx_device_loop(cgx_exec* e, const void* d_ptr_sets, int n_sets, uint64_t n_replays) {
  if (!e) return fail(CGX_E_INVALID_ARG, "device_loop: exec is NULL");
  if (e->o.mode != CGX_MODE_GRAPH_INDIRECT || eff_transport(e->o) != CGX_XPORT_DEVICE)
    return fail(CGX_E_STATE, "device_loop: needs an INDIRECT exec with transport DEVICE");
  if (n_replays == 0) return CGX_OK;
  if (!d_ptr_sets || n_sets <= 0) return fail(CGX_E_INVALID_ARG, "device_loop: no pointer sets");
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, d_ptr_sets) != cudaSuccess || pa.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return fail(CGX_E_NOT_ELIGIBLE, "device_loop: pointer sets must be device memory");
  }
  const uint32_t n_ext = (uint32_t)e->c->ext_slots.size();
  DevLoopArgs a{};
  a.table = e->d_table;
  a.sets = static_cast<const uint64_t*>(d_ptr_sets);
  a.n_replays = n_replays;
  a.chain = e->ge[0];
  a.n_ext = n_ext;
  a.n_sets = (uint32_t)n_sets;
  a.status = e->d_status;
  CKS(check_device_status(e));
  if (!e->dl_ge) {
    CK(cudaMalloc(&e->dl_iter, sizeof(unsigned long long)));
    a.iter = e->dl_iter;
    CK(cudaStreamBeginCapture(e->cs, cudaStreamCaptureModeThreadLocal));
    Launch r;
    r.func = kfn_devloop();
    r.grid = dim3(1);
    r.block = dim3(128);
    r.pdl = false;
    r.args.reset(sizeof(DevLoopArgs));
    memcpy(r.args.p, &a, sizeof(a));
    int st = issue(e, r, e->cs);
    if (st == CGX_OK) st = last_captured_node(e->cs, &e->dl_node);
    if (st != CGX_OK) {
      // leave the exec's capture stream usable: close the capture, drop the partial graph
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(e->cs, &junk);
      if (junk) cudaGraphDestroy(junk);
      return st;
    }
    CK(cudaStreamEndCapture(e->cs, &e->dl_g));
    CK(cudaGraphInstantiateWithFlags(&e->dl_ge, e->dl_g, cudaGraphInstantiateFlagDeviceLaunch));
    CK(cudaGraphUpload(e->dl_ge, e->s));
  }
  a.iter = e->dl_iter;
  cudaKernelNodeParams kp{};
  kp.func = const_cast<void*>(kfn_devloop());
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(128);
  void* argv[1] = {&a};
  kp.kernelParams = argv;
  CK(cudaGraphExecKernelNodeSetParams(e->dl_ge, e->dl_node, &kp));
  CK(cudaMemsetAsync(e->dl_iter, 0, sizeof(unsigned long long), e->s));
  CK(cudaGraphLaunch(e->dl_ge, e->s));
  e->st.n_launches += n_replays;
  e->bound = true;
  e->launched_since_bind = true;
  return CGX_OK;
}

extern "C" int cgx_output(cgx_exec* e, int slot, void** dptr, uint64_t* nbytes) {
  if (!e || !dptr || slot < 0 || slot >= (int)e->c->slots.size()) return fail(CGX_E_INVALID_ARG, "output: bad argument");
  const Slot& s = e->c->slots[slot];
  void* p = nullptr;
  if (s.kind == CGX_SLOT_INTERNAL) p = s.buf;
  else if (s.kind == CGX_SLOT_EXTERNAL && e->o.mode == CGX_MODE_GRAPH_COPY) p = e->ph[s.ext_j];
  else return fail(CGX_E_INVALID_ARG, "output: slot has no library-owned buffer in this exec");
  if (!p) return fail(CGX_E_INVALID_ARG, "output: slot not read by this exec");
  *dptr = p;
  if (nbytes) *nbytes = s.nbytes;
  return CGX_OK;
}

extern "C" int cgx_output_gather(cgx_exec* e, const int* slots, int n, void* dst, uint64_t cap, uint64_t* nbytes_out) {
  if (!e || (n > 0 && (!slots || !dst)) || n < 0) return fail(CGX_E_INVALID_ARG, "output_gather: bad argument");
  if (n > kGatherMax) return fail(CGX_E_INVALID_ARG, "output_gather: more than 64 slots");
  GatherArgs ga{};
  uint64_t off = 0;
  for (int i = 0; i < n; ++i) {
    void* p = nullptr;
    uint64_t nb = 0;
    int st = cgx_output(e, slots[i], &p, &nb);
    if (st != CGX_OK) return st;
    ga.src[i] = p;
    ga.dst[i] = static_cast<uint8_t*>(dst) + off;
    ga.nbytes[i] = nb;
    off += (nb + 15) / 16 * 16;
  }
  ga.n = (uint32_t)n;
  if (nbytes_out) *nbytes_out = off;
  if (off > cap) return fail(CGX_E_SIZE_MISMATCH, "output_gather: destination smaller than the packed outputs");
  if (reinterpret_cast<uintptr_t>(dst) % 16) return fail(CGX_E_MISALIGNED, "output_gather: destination not 16-B aligned");
  if (n == 0) return CGX_OK;
  void* argv[1] = {&ga};
  CK(cudaLaunchKernel(kfn_gather(), dim3(n), dim3(256), argv, 0, e->s));
  return CGX_OK;
}

extern "C" int cgx_stats(const cgx_exec* e, cgx_stats_t* out) {
  if (!e || !out) return fail(CGX_E_INVALID_ARG, "stats: NULL argument");
  *out = e->st;
  out->device_error = e->h_status ? *e->h_status : 0u;
  return CGX_OK;
}

extern "C" int cgx_debug_read_table(const cgx_exec* e, uint64_t* host_out, int n) {
  if (!e || !host_out || n < 0) return fail(CGX_E_INVALID_ARG, "read_table: bad argument");
  if (!e->d_table) return fail(CGX_E_STATE, "read_table: exec has no pointer table (not INDIRECT)");
  if (n > (int)e->c->ext_slots.size()) return fail(CGX_E_INVALID_ARG, "read_table: n > N_ext");
  CK(cudaStreamSynchronize(e->s));
  const uint64_t* tab = e->d_table;
  if (e->d_table2 && e->seq > 0 && (e->seq - 1) % 2 == 1) tab = e->d_table2;   // T6: last bound slot
  if (e->xs) CK(cudaStreamSynchronize(e->xs));
  CK(cudaMemcpy(host_out, tab, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return CGX_OK;
}

// NEXT-2: locate a pointer value inside a kernel's parameter image by
// byte-pattern matching on 8-byte-aligned boundaries.
extern "C" int cgx_find_param_offset(const void* image, uint64_t image_bytes, uint64_t pattern, uint64_t* offset_out) {
  if ((!image && image_bytes) || !offset_out) return fail(CGX_E_INVALID_ARG, "find_param_offset: bad argument");
  const uint8_t* p = static_cast<const uint8_t*>(image);
  int hits = 0;
  uint64_t at = 0;
  for (uint64_t off = 0; off + 8 <= image_bytes; off += 8) {
    uint64_t v;
    memcpy(&v, p + off, 8);
    if (v == pattern) {
      if (++hits == 1) at = off;
    }
  }
  if (hits == 0) return fail(CGX_E_OFFSET_NOT_FOUND, "find_param_offset: pattern not found");
  if (hits > 1) return fail(CGX_E_OFFSET_AMBIGUOUS, "find_param_offset: pattern found " + std::to_string(hits) + " times");
  *offset_out = at;
  return CGX_OK;
}

// The current parameter image of the node at exec position `pos` (what the next launch/replay
// passes), plus its layout from cudaFuncGetParamInfo (param 0 offset/size).
extern "C" int cgx_debug_param_image(const cgx_exec* e, int pos, void* buf, uint64_t cap, uint64_t* nbytes_out,
                                     uint64_t* param0_size_out) {
  if (!e || pos < 0 || pos >= (int)e->L.size() || !nbytes_out) return fail(CGX_E_INVALID_ARG, "param_image: bad argument");
  const Launch& l = e->L[pos];
  if (l.kind != LK_KERNEL) return fail(CGX_E_UNSUPPORTED, "param_image: collective node");
  *nbytes_out = l.args.n;
  if (buf) memcpy(buf, l.args.p, std::min<uint64_t>(cap, l.args.n));
  if (param0_size_out) {
    size_t off = 0, sz = 0;
    CK(cudaFuncGetParamInfo(l.func, 0, &off, &sz));
    *param0_size_out = sz;
  }
  return CGX_OK;
}

static void node_trace_reset(cgx_exec* e) {
  std::vector<unsigned long long> h(3 * e->L.size(), 0);
  for (size_t p = 0; p < e->L.size(); ++p) h[3 * p] = h[3 * p + 1] = ~0ull;
  cudaMemcpy(e->d_trace, h.data(), sizeof(unsigned long long) * h.size(), cudaMemcpyHostToDevice);
}

// Diagnostics (exec created with CGX_NODE_TRACE=1 in the environment): per launch position the
// [first CTA entry, first CTA past its input wait, last CTA exit] %globaltimer ns of the replays
// since the previous call (min / min / max over them), then reset. Synchronises the exec's stream.
extern "C" int cgx_debug_node_trace(cgx_exec* e, uint64_t* host_out, int cap, int* n_out) {
  if (!e || !n_out) return fail(CGX_E_INVALID_ARG, "node_trace: bad argument");
  if (!e->d_trace) return fail(CGX_E_STATE, "node_trace: exec not created with CGX_NODE_TRACE=1");
  CK(cudaStreamSynchronize(e->s));
  const int n = (int)(3 * e->L.size());
  if (host_out) CK(cudaMemcpy(host_out, e->d_trace, sizeof(uint64_t) * std::min(cap, n), cudaMemcpyDeviceToHost));
  node_trace_reset(e);
  *n_out = (int)e->L.size();
  return CGX_OK;
}

// Diagnostics (exec created with CGX_CTA_TRACE=1): per-CTA %globaltimer phase stamps [cta][8] of the
// last replay of launch `pos` (an ATTN_CAUSAL launch: 0 entry, 1 past the PDL wait, 2 K/V staged,
// 3 partials published (0 when one key chunk), 4 exit). Returns the CTA count or a negative status.
extern "C" int cgx_debug_cta_trace(cgx_exec* e, int pos, uint64_t* host_out, int cap) {
  if (!e || pos < 0 || pos >= (int)e->L.size()) return fail(CGX_E_INVALID_ARG, "cta_trace: bad argument");
  Launch& l = e->L[pos];
  if (l.kind != LK_KERNEL || l.mega || e->c->nodes[l.node].op != CGX_OP_ATTN_CAUSAL)
    return fail(CGX_E_INVALID_ARG, "cta_trace: not an attention launch");
  const AttnArgs* a = argp<AttnArgs>(l);
  if (!a->ctrace) return fail(CGX_E_STATE, "cta_trace: exec not created with CGX_CTA_TRACE=1");
  const int ctas = (int)(l.grid.x * l.grid.y);
  if (host_out) {
    CK(cudaStreamSynchronize(e->s));
    CK(cudaMemcpy(host_out, a->ctrace, sizeof(uint64_t) * std::min(cap, 8 * ctas), cudaMemcpyDeviceToHost));
  }
  return ctas;
}

// Diagnostics (megakernel exec created with CGX_MEGA_TRACE=1): [stage][cta][8] %globaltimer ns of
// the last replay (0 start after the stage's barrier, 1 end, 2-6 phase marks, 7 barrier arrival;
// k_mega.cu mtrace). Returns the entry count (host_out == NULL: only the count) or a negative status.
extern "C" int cgx_debug_mega_trace(cgx_exec* e, uint64_t* host_out, int cap) {
  if (!e) return fail(CGX_E_INVALID_ARG, "mega_trace: exec is NULL");
  if (!e->mega) return fail(CGX_E_STATE, "mega_trace: not a megakernel exec");
  const int n = (int)(8 * e->mega_stages * e->mega_ctas);
  if (!host_out) return n;
  CK(cudaStreamSynchronize(e->s));
  CK(cudaMemcpy(host_out, e->mega_strace, sizeof(uint64_t) * std::min(cap, n), cudaMemcpyDeviceToHost));
  return n;
}

// Diagnostics: launch GEMM node `pos` once, alone (no PDL), with per-CTA %globaltimer tracing;
// host_out receives [cta][16] ns timestamps (0 entry, 1 setup done, 2 first stage landed, 3 last MMA
// issued, 4 stores issued, 5 partial pushed, 6 all splits arrived, 7 exit, 8 accumulator ready,
// 9 accumulator in registers, 10 staged).
extern "C" int cgx_debug_gemm_trace(cgx_exec* e, int pos, uint64_t* host_out, int cap, int* n_out) {
  if (!e || pos < 0 || pos >= (int)e->L.size() || !n_out) return fail(CGX_E_INVALID_ARG, "gemm_trace: bad argument");
  Launch& l = e->L[pos];
  if (e->c->nodes[l.node].op != CGX_OP_GEMM_BF16) return fail(CGX_E_INVALID_ARG, "gemm_trace: not a GEMM node");
  const int ctas = (int)(l.grid.x * l.grid.y * l.grid.z);
  unsigned long long* d = nullptr;
  CK(cudaMalloc(&d, sizeof(unsigned long long) * 16 * ctas));
  CK(cudaMemset(d, 0, sizeof(unsigned long long) * 16 * ctas));
  Launch t;
  t.func = l.func;
  t.grid = l.grid;
  t.block = l.block;
  t.smem = l.smem;
  t.cluster_z = l.cluster_z;
  t.pdl = false;
  t.args.reset(l.args.n);
  memcpy(t.args.p, l.args.p, l.args.n);
  decoder_gemm_set_trace(t.args.p, d);
  int st = issue(e, t, e->s);
  if (st == CGX_OK) {
    cudaError_t ce = cudaStreamSynchronize(e->s);
    if (ce == cudaSuccess && host_out)
      ce = cudaMemcpy(host_out, d, sizeof(uint64_t) * std::min(cap, 16 * ctas), cudaMemcpyDeviceToHost);
    if (ce != cudaSuccess) st = cuda_fail(ce, "gemm_trace", __LINE__);
  }
  cudaFree(d);
  *n_out = ctas;
  return st;
}

// Byte offsets of the external-pointer fields the runtime patches in node `pos` (SETPARAMS/EAGER).
extern "C" int cgx_debug_ext_field_offsets(const cgx_exec* e, int pos, uint64_t* offs, int cap, int* n_out) {
  if (!e || pos < 0 || pos >= (int)e->L.size() || !n_out) return fail(CGX_E_INVALID_ARG, "ext_field_offsets: bad argument");
  const Launch& l = e->L[pos];
  int n = 0;
  for (const auto& f : l.ext) {
    if (offs && n < cap) offs[n] = f.off;
    ++n;
  }
  *n_out = n;
  return CGX_OK;
}

extern "C" int cgx_debug_launch_nodes(const cgx_exec* e, int* nodes_out, int cap, int* n_out) {
  if (!e || !n_out) return fail(CGX_E_INVALID_ARG, "launch_nodes: bad argument");
  int n = 0;
  for (const auto& l : e->L) {
    if (nodes_out && n < cap) nodes_out[n] = l.node;
    ++n;
  }
  *n_out = n;
  return CGX_OK;
}

extern "C" int cgx_debug_setparam_nodes(const cgx_exec* e, int* nodes_out, int cap, int* n_out) {
  if (!e || !n_out) return fail(CGX_E_INVALID_ARG, "setparam_nodes: bad argument");
  int n = 0;
  for (auto& l : e->L)
    if (!l.ext.empty()) {
      if (nodes_out && n < cap) nodes_out[n] = l.node;
      ++n;
    }
  *n_out = n;
  return CGX_OK;
}

// ============================================================================ selector
// Estimates and decision: IEEE double, left to right, no contraction (built with
// -ffp-contract=off) so they match oracle/selector.py bit for bit.
static double est_eager(double L, const double* d, int K) {
  double free_t = 0.0;
  for (int k = 1; k <= K; ++k) {
    const double issue_t = (double)k * L;
    const double start = free_t > issue_t ? free_t : issue_t;
    free_t = start + d[k - 1];
  }
  return free_t;
}
static double est_graph(double G, double delta, const double* d, int K, double F) {
  double s = G;
  for (int k = 0; k < K; ++k) s = s + (delta + d[k]);
  return s + F;
}
// model 1: list schedule of the dependency DAG (cgx.h, oracle/selector.py t_graph_dag; same
// operation order, bit-exact)
static double est_graph_dag(const cgx_profile_t& p) {
  std::vector<double> fin((size_t)p.n_kernels);
  double S = 0.0;
  for (int k = 0; k < p.n_kernels; ++k) {
    double start = (double)(k + 1) * p.delta_us;
    for (int e = p.dep_off[k]; e < p.dep_off[k + 1]; ++e) {
      const double c = fin[(size_t)p.dep_idx[e]] + p.lambda_us;
      if (c > start) start = c;
    }
    const double f = start + p.g_us[k];
    fin[(size_t)k] = f;
    if (f > S) S = f;
  }
  return (p.G_us > S ? p.G_us : S) + p.F_us;
}
static bool dag_valid(const cgx_profile_t& p) {
  if (p.dep_off[0] != 0) return false;
  for (int k = 0; k < p.n_kernels; ++k) {
    if (p.dep_off[k + 1] < p.dep_off[k] || p.dep_off[k + 1] > CGX_MAX_PROFILE_DEPS) return false;
    for (int e = p.dep_off[k]; e < p.dep_off[k + 1]; ++e)
      if (p.dep_idx[e] < 0 || p.dep_idx[e] >= k) return false;
  }
  return true;
}

extern "C" int cgx_select(const cgx_profile_t* prof, int n, cgx_decision* out, double* est) {
  if (!prof || !out || n < 0) return fail(CGX_E_INVALID_ARG, "select: bad argument");
  for (int i = 0; i < n; ++i) {
    const cgx_profile_t& p = prof[i];
    if (p.n_kernels < 0 || p.n_kernels > CGX_MAX_PROFILE_KERNELS) return fail(CGX_E_INVALID_ARG, "select: n_kernels");
    if (p.model != 0 && p.model != 1) return fail(CGX_E_INVALID_ARG, "select: model (0 or 1)");
    if (p.model == 1 && !p.use_measured && !dag_valid(p)) return fail(CGX_E_INVALID_ARG, "select: dependency lists");
    double te, tc, ti;
    if (p.use_measured) {
      te = p.t_eager_us;
      tc = p.t_copy_us;
      ti = p.t_ind_us;
    } else {
      const double tg = p.model == 1 ? est_graph_dag(p) : est_graph(p.G_us, p.delta_us, p.d_us, p.n_kernels, p.F_us);
      te = est_eager(p.L_us, p.d_us, p.n_kernels);
      tc = tg + p.c_copy_us;
      ti = tg + p.c_ind_us;
    }
    cgx_decision best = CGX_DECIDE_EAGER;
    double bt = te;
    if (tc < bt) { best = CGX_DECIDE_GRAPH_COPY; bt = tc; }
    if (p.ind_available && ti < bt) { best = CGX_DECIDE_GRAPH_INDIRECT; bt = ti; }
    out[i] = best;
    if (est) { est[3 * i] = te; est[3 * i + 1] = tc; est[3 * i + 2] = ti; }
  }
  return CGX_OK;
}

// profile: below (cgx_profile_ex)
extern "C" int cgx_profile_ex(cgx_chain* c, int segment, const void* const* ext_sets, int n_sets, int n_ext,
                              int reps, void* stream, cgx_profile_t* out);
extern "C" int cgx_profile(cgx_chain* c, int segment, const void* const* ext, int n_ext, int reps, void* stream,
                           cgx_profile_t* out) {
  return cgx_profile_ex(c, segment, ext, 1, n_ext, reps, stream, out);
}

// Slow-path choice of the DAG capture's stream count (candidates are measured with the
// real inputs, then one is deployed). The replay rate of a dependency-DAG graph depends on how
// its branches fall onto capture streams in a way no static rule captured (C2: 14 streams
// 53.3 us, 16 -> 54.9, 12 -> 61.6, 20 -> 57.2; profiles/r01/dag_assign.txt), so each candidate
// exec is built, replayed `reps` times over the given input sets (bind + launch per replay, CUDA
// events on the stream), and the fastest count is returned. Nothing is kept.
extern "C" int cgx_tune_graph_streams(cgx_chain* c, const cgx_exec_opts* opts, void* stream,
                                      const void* const* ext_sets, int n_sets, int n_ext,
                                      const int* candidates, int n_cand, int reps, int* best_out,
                                      double* us_out) {
  if (!c || !opts || !ext_sets || n_sets <= 0 || n_ext < 0 || !candidates || n_cand <= 0 || reps <= 0 ||
      !best_out)
    return fail(CGX_E_INVALID_ARG, "tune_graph_streams: bad argument");
  if (opts->mode == CGX_MODE_EAGER) return fail(CGX_E_INVALID_ARG, "tune_graph_streams: graph modes only");
  for (int ci = 0; ci < n_cand; ++ci)   // every candidate is checked before any is timed
    if (candidates[ci] < 1 || candidates[ci] > 64)
      return fail(CGX_E_INVALID_ARG, "tune_graph_streams: every candidate stream count must be in 1..64");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  struct Ev {
    cudaEvent_t* a;
    cudaEvent_t* b;
    ~Ev() {
      if (*a) cudaEventDestroy(*a);
      if (*b) cudaEventDestroy(*b);
    }
  } ev_guard{&e0, &e1};
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  double best_us = 1e300;
  int best = -1;
  for (int ci = 0; ci < n_cand; ++ci) {
    cgx_exec_opts o = *opts;
    o.sync_mode = CGX_SYNC_GRAPH;
    o.graph_streams = candidates[ci];
    cgx_exec* e = nullptr;
    CKS(cgx_exec_create_ex(c, &o, stream, &e));
    int st = CGX_OK;
    auto run = [&](int n) {
      for (int i = 0; i < n && st == CGX_OK; ++i) {
        st = cgx_bind(e, ext_sets + (size_t)(i % n_sets) * n_ext, n_ext);
        if (st == CGX_OK) st = cgx_launch(e);
      }
    };
    run(std::max(5, reps / 4));                       // warm-up (instantiation upload, L2)
    float ms = 0.f, ms_min = 1e30f;
    for (int t = 0; t < 3 && st == CGX_OK; ++t) {   // best of three trials
      cudaError_t ce = cudaStreamSynchronize(s);
      if (ce == cudaSuccess) ce = cudaEventRecord(e0, s);
      if (ce != cudaSuccess) st = cuda_fail(ce, "tune_graph_streams", __LINE__);
      run(reps);
      if (st == CGX_OK) {
        ce = cudaEventRecord(e1, s);
        if (ce == cudaSuccess) ce = cudaEventSynchronize(e1);
        if (ce == cudaSuccess) ce = cudaEventElapsedTime(&ms, e0, e1);
        if (ce != cudaSuccess) st = cuda_fail(ce, "tune_graph_streams", __LINE__);
        ms_min = std::min(ms_min, ms);
      }
    }
    cgx_exec_destroy(e);
    CKS(st);
    const double us = (double)ms_min * 1e3 / reps;
    if (us_out) us_out[ci] = us;
    if (us < best_us) {
      best_us = us;
      best = candidates[ci];
    }
  }
  *best_out = best;
  return CGX_OK;
}

// ============================================================================ helpers
extern "C" int cgx_dispatch_floor(void* stream, int reps, double* g_us, double* k_us) {
  if (reps <= 0 || !g_us || !k_us) return fail(CGX_E_INVALID_ARG, "dispatch_floor: bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStream_t cs;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  void* noargs[1] = {nullptr};
  CK(cudaLaunchKernel(kfn_empty(), dim3(1), dim3(32), noargs, 0, cs));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamEndCapture(cs, &g));
  CK(cudaGraphInstantiateWithFlags(&ge, g, 0));
  CK(cudaGraphUpload(ge, s));
  std::vector<double> tg, tk;
  for (int r = 0; r < reps + 20; ++r) {
    const double t0 = now_us();
    CK(cudaGraphLaunch(ge, s));
    const double t1 = now_us();
    CK(cudaLaunchKernel(kfn_empty(), dim3(1), dim3(32), noargs, 0, s));
    const double t2 = now_us();
    if (r >= 20) { tg.push_back(t1 - t0); tk.push_back(t2 - t1); }
    if (r % 64 == 63) CK(cudaStreamSynchronize(s));
  }
  CK(cudaStreamSynchronize(s));
  std::sort(tg.begin(), tg.end());
  std::sort(tk.begin(), tk.end());
  *g_us = tg[tg.size() / 2];
  *k_us = tk[tk.size() / 2];
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  return CGX_OK;
}

extern "C" int cgx_graph_floor(void* stream, int n_kernels, int use_pdl, int reps, double* us_per_replay) {
  if (n_kernels <= 0 || reps <= 0 || !us_per_replay) return fail(CGX_E_INVALID_ARG, "graph_floor: bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStream_t cs;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < n_kernels; ++k) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = cs;
    cudaLaunchAttribute attr[1];
    if (use_pdl) {
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
    }
    void* argv[1] = {nullptr};
    CK(cudaLaunchKernelExC(&cfg, use_pdl ? kfn_pdl_nop() : kfn_empty(), argv));
  }
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamEndCapture(cs, &g));
  CK(cudaGraphInstantiateWithFlags(&ge, g, 0));
  CK(cudaGraphUpload(ge, s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 10; ++i) CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(e0, s));
  for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  *us_per_replay = ms * 1e3 / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  return CGX_OK;
}

extern "C" int cgx_copy(void* dst, const void* src, uint64_t nbytes, void* stream) {
  if ((!dst || !src) && nbytes) return fail(CGX_E_INVALID_ARG, "copy: NULL");
  if (nbytes) CK(cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return CGX_OK;
}

extern "C" int cgx_fill_uniform_f32(void* dptr, uint64_t n, uint64_t seed, uint64_t stream_id, void* stream) {
  if (!dptr) return fail(CGX_E_INVALID_ARG, "fill: NULL");
  struct { float* out; uint64_t n; uint64_t base; } a{static_cast<float*>(dptr), n,
                                                      host_mix(seed ^ host_mix(stream_id))};
  void* argv[1] = {&a};
  const unsigned grid = (unsigned)std::min<uint64_t>(std::max<uint64_t>(1, ceil_div(n, 256)), 148 * 16);
  CK(cudaLaunchKernel(kfn_fill_uniform_f32(), dim3(grid), dim3(256), argv, 0, static_cast<cudaStream_t>(stream)));
  return CGX_OK;
}

extern "C" int cgx_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(CGX_E_INVALID_ARG, "nccl_unique_id: NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(CGX_E_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  memcpy(id_out, &id, sizeof(id));
  return CGX_OK;
}

extern "C" int cgx_nccl_comm_init(int nranks, int rank, const void* id, int device, void** comm_out) {
  if (!id || !comm_out || nranks <= 0 || rank < 0 || rank >= nranks) return fail(CGX_E_INVALID_ARG, "nccl_comm_init: bad argument");
  CK(cudaSetDevice(device));
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  ncclResult_t r = ncclCommInitRank(&comm, nranks, uid, rank);
  if (r != ncclSuccess) return fail(CGX_E_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  *comm_out = comm;
  return CGX_OK;
}

extern "C" int cgx_nccl_comm_destroy(void* comm) {
  if (!comm) return CGX_OK;
  ncclResult_t r = ncclCommDestroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return fail(CGX_E_NCCL, std::string("ncclCommDestroy: ") + ncclGetErrorString(r));
  return CGX_OK;
}

// ============================================================================ profiler (slow path)
// P:L413-417 / L630-639: run the candidate modules of one segment, measure, and hand the numbers
// to the pure decision function. Timings follow SURVEY §8(d) and reading 7 (5 warm-up runs, then
// the median of `reps` iterations, three trials for the per-iteration totals).
namespace {
double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v.empty() ? 0.0 : v[v.size() / 2];
}
}  // namespace

// Per-launch device µs: replay an instrumented capture of the exec's launches with an external
// event-record node between consecutive launches (no PDL overlap in this copy), median over reps.
static int kernel_times(cgx_exec* e, int reps, std::vector<double>* out) {
  const int K = (int)e->L.size();
  // every resource is released on every return path (errors included)
  struct Res {
    cudaStream_t cs = nullptr;
    std::vector<cudaEvent_t> ev;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    ~Res() {
      if (ge) cudaGraphExecDestroy(ge);
      if (g) cudaGraphDestroy(g);
      for (auto& v : ev) if (v) cudaEventDestroy(v);
      if (cs) cudaStreamDestroy(cs);
    }
  } r;
  CK(cudaStreamCreateWithFlags(&r.cs, cudaStreamNonBlocking));
  r.ev.assign(K + 1, nullptr);
  for (auto& v : r.ev) CK(cudaEventCreate(&v));
  CK(cudaStreamBeginCapture(r.cs, cudaStreamCaptureModeThreadLocal));
  int st = CGX_OK;
  cudaError_t ce = cudaEventRecordWithFlags(r.ev[0], r.cs, cudaEventRecordExternal);
  if (ce != cudaSuccess) st = cuda_fail(ce, "kernel_times: event record", __LINE__);
  for (int k = 0; k < K && st == CGX_OK; ++k) {
    Launch& l = e->L[k];
    const bool pdl = l.pdl;
    l.pdl = false;
    st = issue(e, l, r.cs);
    l.pdl = pdl;
    if (st != CGX_OK) break;
    ce = cudaEventRecordWithFlags(r.ev[k + 1], r.cs, cudaEventRecordExternal);
    if (ce != cudaSuccess) st = cuda_fail(ce, "kernel_times: event record", __LINE__);
  }
  ce = cudaStreamEndCapture(r.cs, &r.g);
  CKS(st);
  CK(ce);
  CK(cudaGraphInstantiateWithFlags(&r.ge, r.g, 0));
  std::vector<std::vector<double>> dk(K);
  for (int it = 0; it < reps + 2; ++it) {
    CK(cudaGraphLaunch(r.ge, e->s));
    CK(cudaStreamSynchronize(e->s));
    if (it < 2) continue;
    for (int k = 0; k < K; ++k) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, r.ev[k], r.ev[k + 1]));
      dk[k].push_back(ms * 1e3);
    }
  }
  // mean, not median: event timestamps on this part are coarse (~2 us ticks), and the mean of
  // many replays with random phase is an unbiased estimate of a sub-tick duration
  out->resize(K);
  for (int k = 0; k < K; ++k) {
    double sacc = 0.0;
    for (double v : dk[k]) sacc += v;
    (*out)[k] = dk[k].empty() ? 0.0 : sacc / dk[k].size();
  }
  return CGX_OK;
}

extern "C" int cgx_kernel_times(cgx_exec* e, int reps, double* d_us, int cap, int* n_out) {
  if (!e || reps <= 0 || !n_out) return fail(CGX_E_INVALID_ARG, "kernel_times: bad argument");
  if (!e->bound) return fail(CGX_E_STATE, "kernel_times: bind the exec first");
  std::vector<double> v;
  CKS(kernel_times(e, reps, &v));
  for (int k = 0; k < (int)v.size() && k < cap; ++k) d_us[k] = v[k];
  *n_out = (int)v.size();
  return CGX_OK;
}

// n bind+launch (or launch-only) iterations, host wall time per iteration; binds cycle over the
// n_sets input sets (row-major n_sets x n_ext)
static int time_loop(cgx_exec* e, const void* const* sets, int n_sets, int n_ext, bool do_bind, int n, double* us) {
  CK(cudaStreamSynchronize(e->s));
  const double t0 = now_us();
  for (int i = 0; i < n; ++i) {
    if (do_bind) CKS(cgx_bind(e, sets + (size_t)(i % n_sets) * n_ext, n_ext));
    CKS(cgx_launch(e));
  }
  CK(cudaStreamSynchronize(e->s));
  *us = (now_us() - t0) / n;
  return CGX_OK;
}

static int time_loop3(cgx_exec* e, const void* const* sets, int n_sets, int n_ext, bool do_bind, int n, double* us) {
  std::vector<double> v(3);
  for (int t = 0; t < 3; ++t) CKS(time_loop(e, sets, n_sets, n_ext, do_bind, n, &v[t]));
  *us = median(v);
  return CGX_OK;
}

// Node-traced replays of one exec (mode / transport of *base) bound to `ext`: per launch the median
// work time exit - first ready (stamps: cgx_debug_node_trace), plus (dag != NULL) the model-1
// parameters: lambda = median over nodes with dependencies of first-ready_k - max_{j in deps(k)}
// exit_j; delta = the executor's issue interval = median over replays of (last entry - first
// entry) / (K - 1) when the DAG has consecutive launches WITHOUT an edge between them (the
// executor issues them back to back over its streams; their entries are not in chain order), and
// 0 for a linear chain (every entry is gated by its producer, which lambda and the path already
// charge); span = median (last exit - first entry). Untraced launches (NCCL) keep the fallback.
static int traced_times(cgx_chain* c, const cgx_exec_opts& base, void* stream, const void* const* ext, int n_ext,
                        int K, const double* fallback, double* work_out, cgx_profile_t* dag) {
  cgx_exec* et = nullptr;
  g_force_trace = true;
  const int st = cgx_exec_create_ex(c, &base, stream, &et);
  g_force_trace = false;
  if (st != CGX_OK) return st;
  struct G { cgx_exec* e; ~G() { cgx_exec_destroy(e); } } guard{et};
  if ((int)et->L.size() != K) return fail(CGX_E_STATE, "profile: traced exec launch count");
  const auto deps = chain_deps(et);
  if (dag) {
    int ne = 0;
    dag->dep_off[0] = 0;
    for (int k = 0; k < K; ++k) {
      for (int j : deps[k]) {
        if (ne >= CGX_MAX_PROFILE_DEPS) return fail(CGX_E_UNSUPPORTED, "profile: too many dependency edges");
        dag->dep_idx[ne++] = j;
      }
      dag->dep_off[k + 1] = ne;
    }
    dag->n_deps = ne;
  }
  CKS(cgx_bind(et, ext, n_ext));
  for (int i = 0; i < 5; ++i) CKS(cgx_launch(et));
  std::vector<uint64_t> tr(3 * (size_t)K);
  int n_out = 0;
  CKS(cgx_debug_node_trace(et, tr.data(), 3 * K, &n_out));   // reset
  const int R = 21;
  std::vector<std::vector<double>> gk((size_t)K);
  std::vector<double> lam, dl, span;
  auto traced = [&](int k) { return tr[3 * k] != ~0ull && tr[3 * k + 1] != ~0ull && tr[3 * k + 2] != 0; };
  bool independent = false;   // some consecutive pair of launches has no edge between them
  for (int k = 1; k < K && !independent; ++k)
    independent = std::find(deps[k].begin(), deps[k].end(), k - 1) == deps[k].end();
  for (int r = 0; r < R; ++r) {
    CKS(cgx_launch(et));
    CKS(cgx_debug_node_trace(et, tr.data(), 3 * K, &n_out));
    uint64_t e_min = ~0ull, e_max = 0, x_max = 0;
    int n_tr = 0;
    for (int k = 0; k < K; ++k) {
      if (!traced(k)) continue;
      const uint64_t en = tr[3 * k], rd = tr[3 * k + 1], ex = tr[3 * k + 2];
      e_min = std::min(e_min, en);
      x_max = std::max(x_max, ex);
      gk[(size_t)k].push_back(ex > rd ? (double)(ex - rd) * 1e-3 : 0.0);
      uint64_t dep_exit = 0;
      bool any = false;
      for (int j : deps[k])
        if (traced(j)) {
          dep_exit = std::max(dep_exit, (uint64_t)tr[3 * j + 2]);
          any = true;
        }
      if (any) lam.push_back(rd > dep_exit ? (double)(rd - dep_exit) * 1e-3 : 0.0);
      e_max = std::max(e_max, en);
      ++n_tr;
    }
    if (independent && n_tr > 1) dl.push_back((double)(e_max - e_min) * 1e-3 / (n_tr - 1));
    if (x_max > 0) span.push_back((double)(x_max - e_min) * 1e-3);
  }
  for (int k = 0; k < K; ++k) work_out[k] = gk[(size_t)k].empty() ? fallback[k] : median(gk[(size_t)k]);
  if (dag) {
    dag->lambda_us = lam.empty() ? 0.0 : median(lam);
    dag->delta_us = dl.empty() ? 0.0 : median(dl);
    dag->span_us = span.empty() ? 0.0 : median(span);
  }
  return CGX_OK;
}

extern "C" int cgx_profile_ex(cgx_chain* c, int segment, const void* const* sets, int n_sets, int n_ext, int reps,
                              void* stream, cgx_profile_t* out) {
  if (!c || !out || reps <= 0 || n_sets < 1 || n_ext < 0 || (n_ext > 0 && !sets))
    return fail(CGX_E_INVALID_ARG, "profile: bad argument");
  int first = 0, last = (int)c->nodes.size() - 1;
  if (segment >= 0) {
    if (segment >= (int)c->segments.size()) return fail(CGX_E_INVALID_ARG, "profile: segment index");
    first = c->segments[segment].first;
    last = c->segments[segment].second;
  }
  const int K = last - first + 1;
  if (K > CGX_MAX_PROFILE_KERNELS) return fail(CGX_E_UNSUPPORTED, "profile: segment too long");
  cgx_exec_opts o{};
  o.first_node = first;
  o.n_nodes = K;
  cgx_exec *ee = nullptr, *ec = nullptr, *ei = nullptr, *ei5 = nullptr;
  struct Guard {
    cgx_exec** p[4];
    ~Guard() { for (auto q : p) if (*q) cgx_exec_destroy(*q); }
  } guard{{&ee, &ec, &ei, &ei5}};
  o.mode = CGX_MODE_EAGER;
  CKS(cgx_exec_create_ex(c, &o, stream, &ee));
  o.mode = CGX_MODE_GRAPH_COPY;
  CKS(cgx_exec_create_ex(c, &o, stream, &ec));
  o.mode = CGX_MODE_GRAPH_INDIRECT;
  int ind_ok = 1;
  int st = cgx_exec_create_ex(c, &o, stream, &ei);
  if (st == CGX_E_UNSUPPORTED) { ind_ok = 0; ei = nullptr; }
  else if (st != CGX_OK) return st;
  // a second INDIRECT candidate without a root node (FIRST_NODE: the first launches take their
  // operands by value and one of them publishes the table), kept when it replays faster
  cgx_exec_opts o5 = o;
  o5.transport = CGX_XPORT_FIRST_NODE;
  if (ei && cgx_exec_create_ex(c, &o5, stream, &ei5) != CGX_OK) ei5 = nullptr;
  auto* p = new cgx_profile_t{};   // (large: heap, then copied out)
  std::unique_ptr<cgx_profile_t> hold(p);
  p->n_kernels = K;
  p->ind_available = ind_ok;
  p->use_measured = 1;
  p->model = 1;
  p->n_sets = n_sets;
  // warm-up (reading 7: 5 runs)
  double junk = 0;
  CKS(time_loop(ee, sets, n_sets, n_ext, true, 5, &junk));
  CKS(time_loop(ec, sets, n_sets, n_ext, true, 5, &junk));
  if (ei) CKS(time_loop(ei, sets, n_sets, n_ext, true, 5, &junk));
  if (ei5) CKS(time_loop(ei5, sets, n_sets, n_ext, true, 5, &junk));
  // measured end-to-end totals per replay with fresh inputs and each arm's rebinding
  // delta against its OWN launch-only loop (the last bound set stays bound)
  CKS(time_loop3(ee, sets, n_sets, n_ext, true, reps, &p->t_eager_us));
  CKS(time_loop3(ec, sets, n_sets, n_ext, true, reps, &p->t_copy_us));
  CKS(time_loop3(ec, sets, n_sets, n_ext, false, reps, &p->t_copy_base_us));
  cgx_exec_opts o_ind = o;
  if (ei) {
    CKS(time_loop3(ei, sets, n_sets, n_ext, true, reps, &p->t_ind_us));
    CKS(time_loop3(ei, sets, n_sets, n_ext, false, reps, &p->t_ind_base_us));
    if (ei5) {
      double t5 = 0, t5b = 0;
      CKS(time_loop3(ei5, sets, n_sets, n_ext, true, reps, &t5));
      CKS(time_loop3(ei5, sets, n_sets, n_ext, false, reps, &t5b));
      if (t5 < p->t_ind_us) {
        p->t_ind_us = t5;
        p->t_ind_base_us = t5b;
        std::swap(ei, ei5);
        o_ind = o5;
      }
      cgx_exec_destroy(ei5);   // the losing INDIRECT candidate
      ei5 = nullptr;
    }
    p->ind_transport = (int)eff_transport(o_ind);
  } else {
    p->t_ind_us = p->t_ind_base_us = INFINITY;
  }
  p->c_copy_us = std::max(0.0, p->t_copy_us - p->t_copy_base_us);
  p->c_ind_us = ei ? std::max(0.0, p->t_ind_us - p->t_ind_base_us) : INFINITY;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // L: host issue cost per eager kernel; G: host cost of cudaGraphLaunch of the INDIRECT (else
  // COPY) exec — the graph that would be deployed
  cgx_exec* eg = ei ? ei : ec;
  std::vector<double> vl, vg;
  for (int r = 0; r < reps; ++r) {
    CK(cudaStreamSynchronize(s));
    double t0 = now_us();
    CKS(cgx_launch(ee));
    vl.push_back((now_us() - t0) / K);
    CK(cudaStreamSynchronize(s));
    t0 = now_us();
    CKS(cgx_launch(eg));
    vg.push_back(now_us() - t0);
  }
  p->L_us = median(vl);
  p->G_us = median(vg);
  // d_k: each kernel's work time in the EAGER stream (node-traced eager launches: first CTA past
  // its wait -> last CTA exit), the eager recurrence's input; fallback for untraced launches (NCCL):
  // the serialised event-bracketed device time
  std::vector<double> dks;
  CKS(kernel_times(ec, reps, &dks));
  cgx_exec_opts oe = o;
  oe.mode = CGX_MODE_EAGER;
  CKS(traced_times(c, oe, stream, sets, n_ext, K, dks.data(), p->d_us, nullptr));
  p->F_us = 0.0;
  // model 1: the graph that would be deployed (the INDIRECT candidate kept above, else COPY), traced
  cgx_exec_opts og = o_ind;
  if (!ei) og.mode = CGX_MODE_GRAPH_COPY;
  CKS(traced_times(c, og, stream, sets, n_ext, K, dks.data(), p->g_us, p));
  *out = *p;
  return CGX_OK;
}
