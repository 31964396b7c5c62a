"""O2/O3 — recorded-by-value capture and the four rebinding semantics.

Memory is a map address -> host array. A captured exec is the node list with every operand
resolved, AT CAPTURE TIME, to a buffer identity ("parameters to kernel are hardcoded
during a graph's capture"; "records kernel parameters by value").

Operand resolution per slot kind (footnote P:L522-525):
  STATIC    the caller's buffer address, never rebound (SURVEY ambiguity 4)
  INTERNAL  an exec-owned buffer the producer writes directly — never copied
  EXTERNAL  depends on the mode:
    COPY       a static data placeholder ph_j. bind copies y_j -> ph_j for
               every j whose address differs from ph_j (ambiguity 1)
    INDIRECT   pointer-to-pointer: cell table[j]; bind writes
               table[j] = addr(y_j) for every external j in declaration order
    SETPARAMS  the address stored in node k's param image; bind rewrites the image of every
               node that reads an external ("graph management APIs"; BJ (3))
    STALE      the capture-time address; bind does nothing (negative control)
A replay then evaluates the frozen node list reading through those resolutions.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from .chain import eval_node, to_host

MODES = ("COPY", "INDIRECT", "SETPARAMS", "STALE")


class Memory:
    """Address space: addr -> array. Addresses are 16-B aligned integers (fake or real)."""

    def __init__(self, base: int = 0x7000_0000_0000):
        self.buf = {}
        self._next = base

    def alloc(self, value, addr: int | None = None) -> int:
        if addr is None:
            addr = self._next
            self._next += ((np.asarray(value).nbytes + 255) // 256 + 1) * 256
        self.buf[addr] = np.array(value, copy=True)
        return addr


@dataclass
class BindResult:
    copies: list = field(default_factory=list)        # COPY: [(j, src, dst, nbytes)]
    table: bytes = b""                                # INDIRECT: 8*N_ext little-endian bytes
    patched_nodes: list = field(default_factory=list)  # SETPARAMS: node indices rewritten
    bytes_data_rebound: int = 0
    bytes_ptr_rebound: int = 0


class CapturedExec:
    """One captured graph of `chain` in `mode` (O2)."""

    def __init__(self, chain, mode: str, mem: Memory, static_addr: dict,
                 capture_ext_addr: list | None = None):
        assert mode in MODES
        self.chain, self.mode, self.mem = chain, mode, mem
        self.ext_names = [s.name for s in chain.externals()]
        self.ext_index = {n: j for j, n in enumerate(self.ext_names)}
        self.static_addr = dict(static_addr)
        self.internal_addr = {}
        for s in chain.internals():
            z = np.zeros(s.nelems, np.float32 if s.dtype == "f32" else np.float64)
            self.internal_addr[s.name] = mem.alloc(z)
        self.placeholder = {}
        if mode == "COPY":
            for s in chain.externals():
                z = np.zeros(s.nelems, np.float32 if s.dtype == "f32" else np.float64)
                self.placeholder[self.ext_index[s.name]] = mem.alloc(z)
        self.table = [0] * len(self.ext_names)
        # per-node recorded external operand addresses (SETPARAMS / STALE param images)
        self.param_image = {}
        for k, node in enumerate(chain.nodes):
            ext_ops = {pos: self.ext_index[nm] for pos, nm in enumerate(node.ins)
                       if nm in self.ext_index}
            if ext_ops:
                init = None
                if capture_ext_addr is not None:
                    init = {pos: capture_ext_addr[j] for pos, j in ext_ops.items()}
                self.param_image[k] = init
        self.bound = mode == "STALE" and capture_ext_addr is not None

    # -------------------------------------------------------------- O3 bind
    def bind(self, ext_addr: list, only=None) -> BindResult:
        """Rebind fresh inputs y_j (given by address) before a replay (O3).

        `only` (COPY mode, tests only) restricts the copy plan to a subset of externals; it
        models an incomplete external classification for the brute-force minimality pin."""
        if len(ext_addr) != len(self.ext_names):
            raise ValueError("MissingInput")          # S:L360 refresh_pointers errors
        r = BindResult()
        if self.mode == "COPY":
            for j, src in enumerate(ext_addr):
                dst = self.placeholder[j]
                if only is not None and j not in only:
                    continue
                if src != dst:                                  # ambiguity 1: address compare
                    n = self.mem.buf[src].nbytes
                    r.copies.append((j, src, dst, n))
                    r.bytes_data_rebound += n
            for j, src, dst, _ in r.copies:
                self.mem.buf[dst] = self.mem.buf[src].copy()    # ph_j <- bytes(y_j)
        elif self.mode == "INDIRECT":
            self.table = list(ext_addr)                         # table[j] <- &y_j
            r.table = struct.pack("<%dQ" % len(ext_addr), *ext_addr)
            r.bytes_ptr_rebound = 8 * len(ext_addr)
        elif self.mode == "SETPARAMS":
            for k in sorted(self.param_image):
                node = self.chain.nodes[k]
                self.param_image[k] = {pos: ext_addr[self.ext_index[nm]]
                                       for pos, nm in enumerate(node.ins) if nm in self.ext_index}
                r.patched_nodes.append(k)
        elif self.mode == "STALE":
            if not self.bound:                                  # capture-time binding only
                for k in self.param_image:
                    node = self.chain.nodes[k]
                    self.param_image[k] = {pos: ext_addr[self.ext_index[nm]]
                                           for pos, nm in enumerate(node.ins)
                                           if nm in self.ext_index}
                self.bound = True
        self._bound_once = True
        return r

    # -------------------------------------------------------------- O2 replay
    def _resolve(self, k: int, pos: int, name: str) -> int:
        s = self.chain.slot(name)
        if s.kind == "static":
            return self.static_addr[name]
        if s.kind == "internal":
            return self.internal_addr[name]
        j = self.ext_index[name]
        if self.mode == "COPY":
            return self.placeholder[j]
        if self.mode == "INDIRECT":
            return self.table[j]
        return self.param_image[k][pos]

    def replay(self) -> dict:
        """Run the frozen node list once; returns name -> value of every INTERNAL slot."""
        dtype_of = lambda name: self.chain.slot(name).dtype  # noqa: E731
        for k, node in enumerate(self.chain.nodes):
            env = {nm: self.mem.buf[self._resolve(k, pos, nm)] for pos, nm in enumerate(node.ins)}
            out = eval_node(self.chain, node, env, dtype_of)
            self.mem.buf[self.internal_addr[node.out]] = out
        return {n: self.mem.buf[a] for n, a in self.internal_addr.items()}


def load_inputs(chain, mem: Memory, ext_values: dict) -> list:
    """Place one replay's external inputs in memory; returns their addresses in slot order."""
    return [mem.alloc(to_host(s, ext_values[s.name])) for s in chain.externals()]


def load_statics(chain, mem: Memory, static_values: dict) -> dict:
    return {s.name: mem.alloc(to_host(s, static_values[s.name]))
            for s in chain.slots if s.kind == "static"}


def copy_plan_bytes(chain) -> int:
    """bytes_copied_per_replay of a COPY exec when every input is fresh."""
    return sum(s.nbytes for s in chain.externals())


def pointer_bytes(chain) -> int:
    """bytes rebound per replay after PI: 8 x #indirected pointers (Table 3)."""
    return 8 * len(chain.externals())


def setparam_nodes(chain) -> list:
    """Nodes a SETPARAMS bind must rewrite: every node that reads an EXTERNAL slot."""
    ext = {s.name for s in chain.externals()}
    return [k for k, n in enumerate(chain.nodes) if any(i in ext for i in n.ins)]
