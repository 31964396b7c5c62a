"""Marshal a chain description (slots + nodes, e.g. a synth.workloads.ChainSpec) into the C ABI.

Argument marshalling only: torch provides device memory and streams; every node runs in
libcgx.so. A `spec` is duck-typed: `.slots` (name, kind, dtype, nelems), `.nodes` (op, ins, out,
attrs) and `.segments`.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import cgx

_KIND = {"external": cgx.SLOT_EXTERNAL, "static": cgx.SLOT_STATIC, "internal": cgx.SLOT_INTERNAL}
_DT = {"f32": cgx.F32, "bf16": cgx.BF16}
_TDT = {"f32": torch.float32, "bf16": torch.bfloat16}


def make_attr(op: str, attrs: dict) -> cgx.Attr:
    a = cgx.Attr()
    a.n = int(attrs.get("n", 0))
    if op == "ATTN_CAUSAL":
        a.scalar = float(attrs["scale"])
        a.T, a.H, a.D = int(attrs["T"]), int(attrs["H"]), int(attrs["D"])
    else:
        a.scalar = float(attrs.get("scalar", 0.0))
    a.eps = float(attrs.get("eps", 0.0))
    a.rows = int(attrs.get("rows", 0))
    a.cols = int(attrs.get("cols", 0))
    a.M, a.N, a.K = int(attrs.get("M", 0)), int(attrs.get("N", 0)), int(attrs.get("K", 0))
    f = 0
    if attrs.get("bias"):
        f |= cgx.GEMM_BIAS
    if attrs.get("gelu"):
        f |= cgx.GEMM_GELU
    if attrs.get("residual"):
        f |= cgx.GEMM_RESIDUAL
    if attrs.get("allreduce"):
        f |= cgx.GEMM_ALLREDUCE
    a.flags = f
    return a


def host_to_device(values: np.ndarray, dtype: str, device) -> torch.Tensor:
    """Upload synth host values (float32 or bf16 bit patterns) to a device tensor."""
    if dtype == "f32":
        return torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).to(device)
    bits = np.ascontiguousarray(values, dtype=np.uint16).view(np.int16)
    return torch.from_numpy(bits).to(device).view(torch.bfloat16)


def device_to_host(t: torch.Tensor, dtype: str) -> np.ndarray:
    t = t.detach()
    if dtype == "f32":
        return t.float().cpu().numpy()
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


class Chain:
    """A cgx chain built from `spec`, holding its static device tensors alive."""

    def __init__(self, spec, statics: dict, device: int = 0, nccl_comm: int | None = None,
                 peers: tuple | None = None, multicast: tuple | None = None):
        """peers = (rank, world, [region base per rank], max_elems): ALLREDUCE_SUM nodes run the
        peer-memory one-shot all-reduce instead of NCCL (cgx_chain_set_peers); multicast = (world,
        uc, mc, max_elems): they run the NVLS multimem all-reduce (cgx_chain_set_multicast)."""
        self.spec = spec
        self.device = device
        self.handle = cgx.chain_create(device)
        self.statics = statics          # name -> torch tensor (kept alive)
        self.slot = {}
        for s in spec.slots:
            ptr = statics[s.name].data_ptr() if s.kind == "static" else None
            self.slot[s.name] = cgx.chain_add_slot(self.handle, _KIND[s.kind], _DT[s.dtype],
                                                   s.nelems, ptr)
        for n in spec.nodes:
            cgx.chain_add_node(self.handle, cgx.OP[n.op], [self.slot[i] for i in n.ins],
                               self.slot[n.out], make_attr(n.op, n.attrs))
        for f, l in getattr(spec, "segments", []):
            cgx.chain_mark_segment(self.handle, f, l)
        if nccl_comm is not None:
            cgx.chain_set_nccl(self.handle, nccl_comm)
        if peers is not None:
            cgx.chain_set_peers(self.handle, *peers)
        if multicast is not None:
            cgx.chain_set_multicast(self.handle, *multicast)
        self.ext_names = [s.name for s in spec.slots if s.kind == "external"]
        self.execs = []

    def exec(self, mode: str, stream=None, **opts) -> "Exec":
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        e = Exec(self, cgx.exec_create(self.handle, mode, st.cuda_stream, **opts), st)
        self.execs.append(e)
        return e

    def close(self):
        for e in self.execs:
            e.close()
        self.execs = []
        if self.handle:
            cgx.chain_destroy(self.handle)
            self.handle = None


class Exec:
    def __init__(self, chain: Chain, handle: int, stream):
        self.chain, self.handle, self.stream = chain, handle, stream

    def bind_ptrs(self, ptrs):
        cgx.bind(self.handle, ptrs)

    def bind(self, tensors: dict):
        cgx.bind(self.handle, [tensors[n].data_ptr() for n in self.chain.ext_names])

    def launch(self):
        cgx.launch(self.handle)

    def output(self, name: str) -> np.ndarray:
        """Synchronously read a library-owned slot buffer into host memory."""
        s = self.chain.spec.slot(name)
        p, nbytes = cgx.output(self.handle, self.chain.slot[name])
        host = np.empty(nbytes, dtype=np.uint8)
        cgx.copy(host.ctypes.data, p, nbytes, self.stream.cuda_stream)
        self.stream.synchronize()
        return host.view(np.float32 if s.dtype == "f32" else np.uint16)

    def stats(self) -> dict:
        return cgx.stats(self.handle)

    def table(self) -> list:
        return cgx.debug_read_table(self.handle, len(self.chain.ext_names))

    def setparam_nodes(self) -> list:
        return cgx.debug_setparam_nodes(self.handle)

    def close(self):
        if self.handle:
            cgx.exec_destroy(self.handle)
            self.handle = None


def upload_statics(spec, values: dict, device) -> dict:
    return {s.name: host_to_device(values[s.name], s.dtype, device)
            for s in spec.slots if s.kind == "static"}


def upload_externals(spec, values: dict, device) -> dict:
    return {s.name: host_to_device(values[s.name], s.dtype, device)
            for s in spec.slots if s.kind == "external"}
