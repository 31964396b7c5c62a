"""ctypes binding of include/cgx.h — argument marshalling only.

Every step of the hot path runs inside libcgx.so (hand-written sm_100a kernels + the C++
runtime). There is no Python or CPU fallback: if the library is missing or fails to load, import
fails loudly. Names mirror the C ABI (cgx_chain_create -> chain_create, ...).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcgx.so")

# --------------------------------------------------------------------------- enums (cgx.h)
OK = 0
STATUS = {0: "CGX_OK", 1: "CGX_E_INVALID_ARG", 2: "CGX_E_STATE", 3: "CGX_E_NOT_ELIGIBLE",
          4: "CGX_E_MISSING_INPUT", 5: "CGX_E_SIZE_MISMATCH", 6: "CGX_E_MISALIGNED",
          7: "CGX_E_UNSUPPORTED", 8: "CGX_E_OFFSET_NOT_FOUND", 9: "CGX_E_OFFSET_AMBIGUOUS",
          10: "CGX_E_CUDA", 11: "CGX_E_NCCL", 12: "CGX_E_DEVICE"}
E_INVALID_ARG, E_STATE, E_NOT_ELIGIBLE, E_MISSING_INPUT, E_SIZE_MISMATCH, E_MISALIGNED, \
    E_UNSUPPORTED, E_OFFSET_NOT_FOUND, E_OFFSET_AMBIGUOUS, E_CUDA, E_NCCL, E_DEVICE = range(1, 13)
F32, BF16 = 0, 1
SLOT_EXTERNAL, SLOT_STATIC, SLOT_INTERNAL = 0, 1, 2
OP = {"ADD": 0, "MUL": 1, "SCALE_IMM": 2, "COPY": 3, "REDUCE_SUM": 4, "LAYERNORM": 5,
      "GEMM_BF16": 6, "ATTN_CAUSAL": 7, "ALLREDUCE_SUM": 8, "SCALE_T": 9, "SUB": 10, "AXPY": 11,
      "GELU": 12, "GELU_BWD": 13, "TRANSPOSE": 14}
GEMM_BIAS, GEMM_GELU, GEMM_RESIDUAL, GEMM_ALLREDUCE = 1, 2, 4, 8
MODE = {"EAGER": 0, "COPY": 1, "INDIRECT": 2, "SETPARAMS": 3, "STALE": 4}
XPORT = {"DEFAULT": 0, "H2D": 1, "ROOT_MEMCPY": 2, "ROOT_PARAMS": 3, "ROOT_MAPPED": 4, "FIRST_NODE": 5, "H2D_PINGPONG": 6, "PRELUDE": 7,
         "DEVICE": 8}
XPORT_NAME = {v: k for k, v in XPORT.items() if k != "DEFAULT"}
DECIDE = {0: "EAGER", 1: "GRAPH_COPY", 2: "GRAPH_INDIRECT"}
SYNC = {"AUTO": 0, "DEFER": 1, "CHAIN": 2, "GRAPH": 3, "DATAFLOW": 4}
MAX_PROFILE_KERNELS = 1024
MAX_PROFILE_DEPS = 8192
FUSE_ADD_LN = 1
FUSE_LN_GEMM = 2
FUSE_ATTN_GEMM = 4


class Attr(C.Structure):
    _fields_ = [("n", C.c_uint64), ("scalar", C.c_float), ("eps", C.c_float),
                ("rows", C.c_uint32), ("cols", C.c_uint32), ("M", C.c_uint32), ("N", C.c_uint32),
                ("K", C.c_uint32), ("flags", C.c_uint32), ("T", C.c_uint32), ("H", C.c_uint32),
                ("D", C.c_uint32)]


class ExecOpts(C.Structure):
    _fields_ = [("mode", C.c_int), ("transport", C.c_int), ("first_node", C.c_int),
                ("n_nodes", C.c_int), ("no_pdl", C.c_int), ("validate", C.c_int),
                ("copy_impl", C.c_int), ("sync_mode", C.c_int), ("graph_streams", C.c_int),
                ("megakernel", C.c_int), ("fuse", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("bytes_data_rebound", C.c_uint64), ("bytes_ptr_rebound", C.c_uint64),
                ("total_bytes_data", C.c_uint64), ("total_bytes_ptr", C.c_uint64),
                ("n_binds", C.c_uint64), ("n_launches", C.c_uint64),
                ("n_setparam_calls", C.c_uint32), ("n_copy_tensors", C.c_uint32),
                ("n_nodes", C.c_uint32), ("n_graph_nodes", C.c_uint32), ("n_ext", C.c_uint32),
                ("kernels_per_replay", C.c_uint32), ("mode", C.c_uint32), ("transport", C.c_uint32),
                ("n_deferred", C.c_uint32), ("dataflow", C.c_uint32), ("dag_streams", C.c_uint32),
                ("device_error", C.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Profile(C.Structure):
    _fields_ = [("n_kernels", C.c_int), ("ind_available", C.c_int), ("use_measured", C.c_int),
                ("model", C.c_int), ("L_us", C.c_double), ("G_us", C.c_double),
                ("delta_us", C.c_double), ("c_copy_us", C.c_double), ("c_ind_us", C.c_double),
                ("F_us", C.c_double), ("t_eager_us", C.c_double), ("t_copy_us", C.c_double),
                ("t_ind_us", C.c_double), ("d_us", C.c_double * MAX_PROFILE_KERNELS),
                ("lambda_us", C.c_double), ("span_us", C.c_double), ("t_copy_base_us", C.c_double),
                ("t_ind_base_us", C.c_double), ("n_sets", C.c_int), ("n_deps", C.c_int),
                ("ind_transport", C.c_int), ("reserved2", C.c_int),
                ("g_us", C.c_double * MAX_PROFILE_KERNELS),
                ("dep_off", C.c_int * (MAX_PROFILE_KERNELS + 1)), ("dep_idx", C.c_int * MAX_PROFILE_DEPS)]

    def deps(self):
        return [list(self.dep_idx[self.dep_off[k]:self.dep_off[k + 1]]) for k in range(self.n_kernels)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f not in ("d_us", "g_us", "dep_off", "dep_idx")}
        d["d_us"] = list(self.d_us[: self.n_kernels])
        d["g_us"] = list(self.g_us[: self.n_kernels])
        d["deps"] = self.deps()
        return d

    def oracle_dict(self):
        """The same profile in oracle/selector.py's vocabulary."""
        return dict(L=self.L_us, G=self.G_us, delta=self.delta_us, d=list(self.d_us[: self.n_kernels]),
                    c_copy=self.c_copy_us, c_ind=self.c_ind_us, F=self.F_us, use_measured=bool(self.use_measured),
                    ind_available=bool(self.ind_available), t_eager=self.t_eager_us, t_copy=self.t_copy_us,
                    t_ind=self.t_ind_us, model=self.model, lam=self.lambda_us,
                    g=list(self.g_us[: self.n_kernels]), deps=self.deps())


class CgxError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        super().__init__(f"{fn}: {STATUS.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libcgx.so not built at {LIB_PATH}: run __graft_entry__.build() "
                          "(no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    P, I, U64, VP = C.POINTER, C.c_int, C.c_uint64, C.c_void_p
    sig = {
        "cgx_version": ([], I), "cgx_last_error": ([], C.c_char_p),
        "cgx_chain_create": ([I, P(VP)], I),
        "cgx_chain_add_slot": ([VP, I, I, U64, VP, P(I)], I),
        "cgx_chain_add_node": ([VP, I, P(I), I, I, P(Attr), P(I)], I),
        "cgx_chain_mark_segment": ([VP, I, I], I),
        "cgx_chain_set_nccl": ([VP, VP], I),
        "cgx_chain_destroy": ([VP], I),
        "cgx_exec_create": ([VP, I, VP, P(VP)], I),
        "cgx_exec_create_ex": ([VP, P(ExecOpts), VP, P(VP)], I),
        "cgx_bind": ([VP, P(VP), I], I),
        "cgx_launch": ([VP], I),
        "cgx_output": ([VP, I, P(VP), P(U64)], I),
        "cgx_output_gather": ([VP, P(I), I, VP, U64, P(U64)], I),
        "cgx_stats": ([VP, P(Stats)], I),
        "cgx_debug_read_table": ([VP, P(U64), I], I),
        "cgx_debug_setparam_nodes": ([VP, P(I), I, P(I)], I),
        "cgx_exec_destroy": ([VP], I),
        "cgx_profile": ([VP, I, P(VP), I, I, VP, P(Profile)], I),
        "cgx_profile_ex": ([VP, I, P(VP), I, I, I, VP, P(Profile)], I),
        "cgx_select": ([P(Profile), I, P(I), P(C.c_double)], I),
        "cgx_dispatch_floor": ([VP, I, P(C.c_double), P(C.c_double)], I),
        "cgx_fill_uniform_f32": ([VP, U64, U64, U64, VP], I),
        "cgx_copy": ([VP, VP, U64, VP], I),
        "cgx_graph_floor": ([VP, I, I, I, P(C.c_double)], I),
        "cgx_kernel_times": ([VP, I, P(C.c_double), I, P(I)], I),
        "cgx_find_param_offset": ([VP, U64, U64, P(U64)], I),
        "cgx_debug_param_image": ([VP, I, VP, U64, P(U64), P(U64)], I),
        "cgx_debug_ext_field_offsets": ([VP, I, P(U64), I, P(I)], I),
        "cgx_debug_gemm_trace": ([VP, I, P(U64), I, P(I)], I),
        "cgx_debug_node_trace": ([VP, P(U64), I, P(I)], I),
        "cgx_debug_cta_trace": ([VP, I, P(U64), I], I),
        "cgx_debug_mega_trace": ([VP, P(U64), I], I),
        "cgx_debug_launch_nodes": ([VP, P(I), I, P(I)], I),
        "cgx_device_loop": ([VP, VP, I, U64], I),
        "cgx_nccl_unique_id": ([VP], I),
        "cgx_nccl_comm_init": ([I, I, VP, I, P(VP)], I),
        "cgx_nccl_comm_destroy": ([VP], I),
        "cgx_peer_buffer_bytes": ([I, U64, I, P(U64)], I),
        "cgx_chain_set_peers": ([VP, I, I, P(VP), U64, I], I),
        "cgx_device_alloc": ([I, U64, P(VP)], I), "cgx_device_free": ([VP], I),
        "cgx_ipc_handle": ([VP, VP], I),
        "cgx_ipc_open": ([VP, P(VP)], I),
        "cgx_ipc_close": ([VP], I),
        "cgx_mc_supported": ([I, P(I)], I),
        "cgx_mc_buffer_bytes": ([U64, I, P(U64)], I),
        "cgx_mc_create": ([I, U64, I, P(U64), P(U64)], I),
        "cgx_mc_export_fd": ([U64, P(I)], I),
        "cgx_mc_import_fd": ([I, P(U64)], I),
        "cgx_mc_add_device": ([U64, I], I),
        "cgx_mc_bind_map": ([U64, I, U64, P(VP), P(VP)], I),
        "cgx_mc_release": ([VP], I),
        "cgx_chain_set_multicast": ([VP, I, VP, VP, U64, I], I),
        "cgx_tune_graph_streams": ([VP, P(ExecOpts), VP, VP, I, I, P(C.c_int), I, I, P(C.c_int), P(C.c_double)], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


LIB = _load()
EXPORTED = ("cgx_version", "cgx_last_error", "cgx_chain_create", "cgx_chain_add_slot",
            "cgx_chain_add_node", "cgx_chain_mark_segment", "cgx_chain_set_nccl",
            "cgx_chain_destroy", "cgx_exec_create", "cgx_exec_create_ex", "cgx_bind",
            "cgx_launch", "cgx_output", "cgx_output_gather", "cgx_stats", "cgx_debug_read_table",
            "cgx_debug_setparam_nodes", "cgx_exec_destroy", "cgx_profile", "cgx_profile_ex", "cgx_select",
            "cgx_dispatch_floor", "cgx_fill_uniform_f32", "cgx_copy", "cgx_graph_floor", "cgx_kernel_times", "cgx_find_param_offset",
            "cgx_debug_param_image", "cgx_debug_ext_field_offsets", "cgx_debug_gemm_trace", "cgx_debug_node_trace", "cgx_debug_cta_trace", "cgx_debug_mega_trace", "cgx_debug_launch_nodes", "cgx_device_loop", "cgx_nccl_unique_id",
            "cgx_nccl_comm_init", "cgx_nccl_comm_destroy", "cgx_peer_buffer_bytes", "cgx_chain_set_peers",
            "cgx_device_alloc", "cgx_device_free",
            "cgx_ipc_handle", "cgx_ipc_open", "cgx_ipc_close", "cgx_mc_supported", "cgx_mc_buffer_bytes",
            "cgx_mc_create", "cgx_mc_export_fd", "cgx_mc_import_fd", "cgx_mc_add_device", "cgx_mc_bind_map",
            "cgx_mc_release", "cgx_chain_set_multicast", "cgx_tune_graph_streams")


def _ck(status: int, fn: str):
    if status != OK:
        raise CgxError(status, fn, LIB.cgx_last_error().decode(errors="replace"))


def last_error() -> str:
    return LIB.cgx_last_error().decode(errors="replace")


def version() -> int:
    return LIB.cgx_version()


# --------------------------------------------------------------------------- thin wrappers
def chain_create(device: int = 0) -> int:
    out = C.c_void_p()
    _ck(LIB.cgx_chain_create(device, C.byref(out)), "cgx_chain_create")
    return out.value


def chain_add_slot(chain: int, kind: int, dtype: int, nelems: int, static_dptr: int | None = None) -> int:
    out = C.c_int()
    _ck(LIB.cgx_chain_add_slot(chain, kind, dtype, nelems, static_dptr, C.byref(out)),
        "cgx_chain_add_slot")
    return out.value


def chain_add_node(chain: int, op: int, in_slots, out_slot: int, attr: Attr | None = None) -> int:
    arr = (C.c_int * max(1, len(in_slots)))(*in_slots)
    out = C.c_int()
    _ck(LIB.cgx_chain_add_node(chain, op, arr, len(in_slots), out_slot,
                               C.byref(attr) if attr is not None else None, C.byref(out)),
        "cgx_chain_add_node")
    return out.value


def chain_mark_segment(chain: int, first: int, last: int):
    _ck(LIB.cgx_chain_mark_segment(chain, first, last), "cgx_chain_mark_segment")


def chain_set_nccl(chain: int, comm: int):
    _ck(LIB.cgx_chain_set_nccl(chain, comm), "cgx_chain_set_nccl")


def chain_destroy(chain: int):
    _ck(LIB.cgx_chain_destroy(chain), "cgx_chain_destroy")


def exec_create(chain: int, mode: str, stream: int, transport: str = "DEFAULT", first_node: int = 0,
                n_nodes: int = 0, no_pdl: bool = False, validate: int = 0, copy_impl: int = 0,
                sync: str = "AUTO", graph_streams: int = 0, megakernel: bool = False, fuse: int = 0) -> int:
    """fuse: bit mask of capture-time fusions (FUSE_ADD_LN | FUSE_LN_GEMM | FUSE_ATTN_GEMM)."""
    o = ExecOpts(MODE[mode], XPORT[transport], first_node, n_nodes, int(no_pdl), validate, copy_impl,
                 SYNC[sync], graph_streams, int(megakernel), int(fuse))
    out = C.c_void_p()
    _ck(LIB.cgx_exec_create_ex(chain, C.byref(o), stream, C.byref(out)), "cgx_exec_create_ex")
    return out.value


def tune_graph_streams(chain: int, mode: str, stream: int, ext_sets, candidates=(8, 12, 14, 16, 20, 24, 32),
                       reps: int = 100, transport: str = "DEFAULT", **kw) -> tuple:
    """Slow-path stream-count choice for the DAG capture (cgx_tune_graph_streams): ext_sets is a
    list of input sets (each a list of device pointers in cgx_bind order). Returns
    (best_count, {count: us_per_replay})."""
    n_sets, n_ext = len(ext_sets), len(ext_sets[0]) if ext_sets else 0
    flat = ptr_array([p for row in ext_sets for p in row])
    o = ExecOpts(MODE[mode], XPORT[transport], kw.get("first_node", 0), kw.get("n_nodes", 0),
                 int(kw.get("no_pdl", False)), kw.get("validate", 0), kw.get("copy_impl", 0), SYNC["GRAPH"], 0,
                 int(kw.get("megakernel", False)))
    cand = (C.c_int * len(candidates))(*candidates)
    us = (C.c_double * len(candidates))()
    best = C.c_int()
    _ck(LIB.cgx_tune_graph_streams(chain, C.byref(o), stream, flat, n_sets, n_ext, cand, len(candidates), reps,
                                   C.byref(best), us), "cgx_tune_graph_streams")
    return best.value, {int(c_): us[i] for i, c_ in enumerate(candidates)}


def ptr_array(ptrs):
    return (C.c_void_p * max(1, len(ptrs)))(*ptrs)


def bind(ex: int, ptrs) -> None:
    arr = ptrs if isinstance(ptrs, C.Array) else ptr_array(list(ptrs))
    _ck(LIB.cgx_bind(ex, arr, len(arr) if isinstance(ptrs, C.Array) else len(ptrs)), "cgx_bind")


def launch(ex: int) -> None:
    _ck(LIB.cgx_launch(ex), "cgx_launch")


def output(ex: int, slot: int):
    p, n = C.c_void_p(), C.c_uint64()
    _ck(LIB.cgx_output(ex, slot, C.byref(p), C.byref(n)), "cgx_output")
    return p.value, n.value


def output_gather(ex: int, slots, dst_dptr: int, cap: int) -> int:
    """Pack the output buffers of `slots` into the device buffer dst (16-B aligned offsets) on the
    exec's stream; returns the packed byte count."""
    arr = (C.c_int * max(1, len(slots)))(*slots)
    nb = C.c_uint64()
    _ck(LIB.cgx_output_gather(ex, arr, len(slots), C.c_void_p(dst_dptr), C.c_uint64(cap), C.byref(nb)),
        "cgx_output_gather")
    return nb.value


def stats(ex: int) -> dict:
    s = Stats()
    _ck(LIB.cgx_stats(ex, C.byref(s)), "cgx_stats")
    return s.as_dict()


def debug_read_table(ex: int, n: int) -> list:
    buf = (C.c_uint64 * max(1, n))()
    _ck(LIB.cgx_debug_read_table(ex, buf, n), "cgx_debug_read_table")
    return list(buf[:n])


def debug_setparam_nodes(ex: int) -> list:
    n = C.c_int()
    _ck(LIB.cgx_debug_setparam_nodes(ex, None, 0, C.byref(n)), "cgx_debug_setparam_nodes")
    buf = (C.c_int * max(1, n.value))()
    _ck(LIB.cgx_debug_setparam_nodes(ex, buf, n.value, C.byref(n)), "cgx_debug_setparam_nodes")
    return list(buf[: n.value])


def find_param_offset(image: bytes, pattern: int) -> int:
    buf = C.create_string_buffer(bytes(image), len(image))
    off = C.c_uint64()
    _ck(LIB.cgx_find_param_offset(buf, len(image), pattern & 0xFFFFFFFFFFFFFFFF, C.byref(off)),
        "cgx_find_param_offset")
    return off.value


def param_image(ex: int, pos: int) -> tuple:
    n, p0 = C.c_uint64(), C.c_uint64()
    _ck(LIB.cgx_debug_param_image(ex, pos, None, 0, C.byref(n), C.byref(p0)), "cgx_debug_param_image")
    buf = C.create_string_buffer(n.value)
    _ck(LIB.cgx_debug_param_image(ex, pos, buf, n.value, C.byref(n), C.byref(p0)), "cgx_debug_param_image")
    return buf.raw[: n.value], p0.value


def ext_field_offsets(ex: int, pos: int) -> list:
    n = C.c_int()
    buf = (C.c_uint64 * 16)()
    _ck(LIB.cgx_debug_ext_field_offsets(ex, pos, buf, 16, C.byref(n)), "cgx_debug_ext_field_offsets")
    return list(buf[: n.value])


def gemm_trace(ex: int, pos: int) -> list:
    n = C.c_int()
    buf = (C.c_uint64 * (16 * 4096))()
    _ck(LIB.cgx_debug_gemm_trace(ex, pos, buf, 16 * 4096, C.byref(n)), "cgx_debug_gemm_trace")
    return [list(buf[16 * i: 16 * i + 16]) for i in range(n.value)]


def device_loop(ex: int, d_ptr_sets: int, n_sets: int, n_replays: int) -> None:
    _ck(LIB.cgx_device_loop(ex, d_ptr_sets, n_sets, n_replays), "cgx_device_loop")


def node_trace(ex: int, n_launch: int) -> list:
    """[(entry, ready, exit)] ns per launch position (exec created with CGX_NODE_TRACE=1)."""
    n = C.c_int()
    buf = (C.c_uint64 * (3 * n_launch))()
    _ck(LIB.cgx_debug_node_trace(ex, buf, 3 * n_launch, C.byref(n)), "cgx_debug_node_trace")
    return [tuple(buf[3 * i: 3 * i + 3]) for i in range(n.value)]


def cta_trace(ex: int, pos: int) -> list:
    """[[8 ns stamps] per CTA] of ATTN launch `pos` (exec created with CGX_CTA_TRACE=1)."""
    n = LIB.cgx_debug_cta_trace(ex, pos, None, 0)
    _ck(n if n < 0 else 0, "cgx_debug_cta_trace")
    buf = (C.c_uint64 * (8 * n))()
    _ck(min(0, LIB.cgx_debug_cta_trace(ex, pos, buf, 8 * n)), "cgx_debug_cta_trace")
    return [list(buf[8 * i: 8 * i + 8]) for i in range(n)]


def launch_nodes(ex: int) -> list:
    """Chain node index of every launch position (cgx_debug_launch_nodes)."""
    n = C.c_int()
    _ck(LIB.cgx_debug_launch_nodes(ex, None, 0, C.byref(n)), "cgx_debug_launch_nodes")
    buf = (C.c_int * max(1, n.value))()
    _ck(LIB.cgx_debug_launch_nodes(ex, buf, n.value, C.byref(n)), "cgx_debug_launch_nodes")
    return list(buf[: n.value])


def exec_destroy(ex: int):
    _ck(LIB.cgx_exec_destroy(ex), "cgx_exec_destroy")


def profile(chain: int, segment: int, ptrs, reps: int, stream: int, sets=None) -> Profile:
    """cgx_profile (one input set: ptrs) or cgx_profile_ex (sets: list of pointer lists)."""
    p = Profile()
    if sets:
        n_ext = len(sets[0])
        arr = ptr_array([q for row in sets for q in row])
        _ck(LIB.cgx_profile_ex(chain, segment, arr, len(sets), n_ext, reps, stream, C.byref(p)), "cgx_profile_ex")
        return p
    arr = ptr_array(list(ptrs))
    _ck(LIB.cgx_profile(chain, segment, arr, len(ptrs), reps, stream, C.byref(p)), "cgx_profile")
    return p


def select(profiles) -> tuple:
    n = len(profiles)
    arr = (Profile * max(1, n))(*profiles)
    out = (C.c_int * max(1, n))()
    est = (C.c_double * max(3, 3 * n))()
    _ck(LIB.cgx_select(arr, n, out, est), "cgx_select")
    return list(out[:n]), [tuple(est[3 * i:3 * i + 3]) for i in range(n)]


def dispatch_floor(stream: int, reps: int = 2000) -> tuple:
    g, k = C.c_double(), C.c_double()
    _ck(LIB.cgx_dispatch_floor(stream, reps, C.byref(g), C.byref(k)), "cgx_dispatch_floor")
    return g.value, k.value


def fill_uniform_f32(dptr: int, n: int, seed: int, stream_id: int, stream: int):
    _ck(LIB.cgx_fill_uniform_f32(dptr, n, seed, stream_id, stream), "cgx_fill_uniform_f32")


def kernel_times(ex: int, reps: int = 20) -> list:
    n = C.c_int()
    buf = (C.c_double * 4096)()
    _ck(LIB.cgx_kernel_times(ex, reps, buf, 4096, C.byref(n)), "cgx_kernel_times")
    return list(buf[: n.value])


def graph_floor(stream: int, n_kernels: int, use_pdl: bool = True, reps: int = 200) -> float:
    us = C.c_double()
    _ck(LIB.cgx_graph_floor(stream, n_kernels, int(use_pdl), reps, C.byref(us)), "cgx_graph_floor")
    return us.value


def copy(dst: int, src: int, nbytes: int, stream: int):
    _ck(LIB.cgx_copy(dst, src, nbytes, stream), "cgx_copy")


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _ck(LIB.cgx_nccl_unique_id(buf), "cgx_nccl_unique_id")
    return buf.raw


def nccl_comm_init(nranks: int, rank: int, uid: bytes, device: int) -> int:
    buf = C.create_string_buffer(uid, 128)
    out = C.c_void_p()
    _ck(LIB.cgx_nccl_comm_init(nranks, rank, buf, device, C.byref(out)), "cgx_nccl_comm_init")
    return out.value


def nccl_comm_destroy(comm: int):
    _ck(LIB.cgx_nccl_comm_destroy(comm), "cgx_nccl_comm_destroy")


def peer_buffer_bytes(world: int, max_elems: int, max_allreduces: int = 64) -> int:
    b = C.c_uint64()
    _ck(LIB.cgx_peer_buffer_bytes(world, max_elems, max_allreduces, C.byref(b)), "cgx_peer_buffer_bytes")
    return b.value


def chain_set_peers(chain: int, rank: int, world: int, bases, max_elems: int, max_allreduces: int = 64) -> None:
    arr = (C.c_void_p * world)(*bases)
    _ck(LIB.cgx_chain_set_peers(chain, rank, world, arr, max_elems, max_allreduces), "cgx_chain_set_peers")


def mc_supported(device: int) -> bool:
    v = C.c_int()
    _ck(LIB.cgx_mc_supported(device, C.byref(v)), "cgx_mc_supported")
    return bool(v.value)


def mc_buffer_bytes(max_elems: int, max_allreduces: int = 64) -> int:
    b = C.c_uint64()
    _ck(LIB.cgx_mc_buffer_bytes(max_elems, max_allreduces, C.byref(b)), "cgx_mc_buffer_bytes")
    return b.value


def mc_create(world: int, nbytes: int, device: int) -> tuple:
    """(multicast handle, size every rank binds and maps)."""
    h, sz = C.c_uint64(), C.c_uint64()
    _ck(LIB.cgx_mc_create(world, nbytes, device, C.byref(h), C.byref(sz)), "cgx_mc_create")
    return h.value, sz.value


def mc_export_fd(handle: int) -> int:
    fd = C.c_int()
    _ck(LIB.cgx_mc_export_fd(handle, C.byref(fd)), "cgx_mc_export_fd")
    return fd.value


def mc_import_fd(fd: int) -> int:
    h = C.c_uint64()
    _ck(LIB.cgx_mc_import_fd(fd, C.byref(h)), "cgx_mc_import_fd")
    return h.value


def mc_add_device(handle: int, device: int) -> None:
    _ck(LIB.cgx_mc_add_device(handle, device), "cgx_mc_add_device")


def mc_bind_map(handle: int, device: int, size: int) -> tuple:
    """(this rank's copy, the multicast address) of a zero-filled region bound to `handle`."""
    uc, mc = C.c_void_p(), C.c_void_p()
    _ck(LIB.cgx_mc_bind_map(handle, device, size, C.byref(uc), C.byref(mc)), "cgx_mc_bind_map")
    return uc.value, mc.value


def mc_release(uc: int) -> None:
    _ck(LIB.cgx_mc_release(C.c_void_p(uc)), "cgx_mc_release")


def chain_set_multicast(chain: int, world: int, uc: int, mc: int, max_elems: int, max_allreduces: int = 64) -> None:
    _ck(LIB.cgx_chain_set_multicast(chain, world, C.c_void_p(uc), C.c_void_p(mc), max_elems, max_allreduces),
        "cgx_chain_set_multicast")


def device_alloc(device: int, nbytes: int) -> int:
    """Dedicated zero-filled cudaMalloc allocation (peer regions: IPC maps it at offset 0)."""
    p = C.c_void_p()
    _ck(LIB.cgx_device_alloc(device, nbytes, C.byref(p)), "cgx_device_alloc")
    return p.value


def device_free(dptr: int) -> None:
    _ck(LIB.cgx_device_free(C.c_void_p(dptr)), "cgx_device_free")


def ipc_handle(dptr: int) -> bytes:
    buf = C.create_string_buffer(64)
    _ck(LIB.cgx_ipc_handle(C.c_void_p(dptr), buf), "cgx_ipc_handle")
    return buf.raw


def ipc_open(handle: bytes) -> int:
    p = C.c_void_p()
    _ck(LIB.cgx_ipc_open(C.create_string_buffer(handle, 64), C.byref(p)), "cgx_ipc_open")
    return p.value


def ipc_close(dptr: int) -> None:
    _ck(LIB.cgx_ipc_close(C.c_void_p(dptr)), "cgx_ipc_close")
