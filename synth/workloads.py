"""Synthetic workload recipes (chain shapes + seeded values) for configs C1..C5.

Plain data only: slot declarations, node lists and which generator fills each slot. No chain op
is evaluated here. Shapes follow BASELINE.json `configs` as made concrete in SURVEY.md §8(d):
  C1  8-kernel fp32 chain, 3 external inputs of 4096 floats            (SURVEY §8(d) "C1 details")
  C2  200-kernel chain, 64 external lanes of 1 KiB..4 MiB              (SURVEY §8(d) "C2 details")
  C3  GPT-2-small-shaped decoder chain, bf16, T tokens                 ("C3 details")
  C4  C1 with every input of S bytes, window or full kernels           (SURVEY §8(d) "C4 details")
  C5  C3 sharded Megatron-style over p ranks (head padding at p=8)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import splitmix as sm

EXTERNAL, STATIC, INTERNAL = "external", "static", "internal"
OPS = ("ADD", "MUL", "SCALE_IMM", "COPY", "REDUCE_SUM", "LAYERNORM", "GEMM_BF16",
       "ATTN_CAUSAL", "ALLREDUCE_SUM", "SCALE_T")


@dataclass(frozen=True)
class SlotSpec:
    name: str
    kind: str            # EXTERNAL | STATIC | INTERNAL
    dtype: str           # "f32" | "bf16"
    nelems: int
    init: str = "uniform"  # uniform | int | weight | gamma | bias | zero (EXTERNAL/STATIC only)

    @property
    def nbytes(self) -> int:
        return self.nelems * (4 if self.dtype == "f32" else 2)


@dataclass(frozen=True)
class NodeSpec:
    op: str
    ins: tuple
    out: str
    attrs: dict = field(default_factory=dict)


@dataclass
class ChainSpec:
    name: str
    slots: list
    nodes: list
    segments: list = field(default_factory=list)   # [(first, last)] inclusive node ranges

    def index(self, name: str) -> int:
        for i, s in enumerate(self.slots):
            if s.name == name:
                return i
        raise KeyError(name)

    def slot(self, name: str) -> SlotSpec:
        return self.slots[self.index(name)]

    def externals(self) -> list:
        return [s for s in self.slots if s.kind == EXTERNAL]

    def internals(self) -> list:
        return [s for s in self.slots if s.kind == INTERNAL]


# ----------------------------------------------------------------------------- values

def slot_values(chain: ChainSpec, name: str, replay: int = 0, mode: str = "uniform",
                seed: int = sm.SEED) -> np.ndarray:
    """Host values of an EXTERNAL (per replay) or STATIC slot.

    f32 slots -> float32 array; bf16 slots -> uint16 bit patterns.
    mode="int" switches uniform recipes to the integer-exact recipe.
    """
    i = chain.index(name)
    s = chain.slots[i]
    stream = sm.stream_id(i, sm.STATIC_REPLAY if s.kind == STATIC else replay)
    init = s.init
    if mode == "int" and init in ("uniform", "weight", "bias"):
        init = "int"
    if s.dtype == "f32":
        if init == "int":
            return sm.int_f32(seed, stream, s.nelems)
        if init == "zero":
            return np.zeros(s.nelems, np.float32)
        return sm.uniform_f32(seed, stream, s.nelems)
    if init == "int":
        return sm.int_bf16_bits(seed, stream, s.nelems)
    if init == "weight" or init == "bias":
        return sm.uniform_bf16_bits(seed, stream, s.nelems, scale_pow2=-5)
    if init == "gamma":
        return sm.gamma_bf16_bits(seed, stream, s.nelems)
    if init == "zero":
        return np.zeros(s.nelems, np.uint16)
    return sm.uniform_bf16_bits(seed, stream, s.nelems)


# ----------------------------------------------------------------------------- C1 / C4

def c1_chain(nelems: int = 4096, window: int | None = None) -> ChainSpec:
    """t0=ADD(x0,x1) t1=MUL(t0,x2) t2=SCALE(t1,.5) t3=ADD(t2,w) t4=MUL(t3,x0)
    t5=COPY(t4) t6=ADD(t5,x1) out=SCALE(t6,2). With `window`, kernels touch only the first
    `window` elements (C4 window mode); otherwise all `nelems` (C4 full mode / C1)."""
    n = nelems if window is None else min(window, nelems)
    slots = [SlotSpec("x0", EXTERNAL, "f32", nelems), SlotSpec("x1", EXTERNAL, "f32", nelems),
             SlotSpec("x2", EXTERNAL, "f32", nelems), SlotSpec("w", STATIC, "f32", n)]
    for t in ("t0", "t1", "t2", "t3", "t4", "t5", "t6", "out"):
        slots.append(SlotSpec(t, INTERNAL, "f32", n))
    a = {"n": n}
    nodes = [NodeSpec("ADD", ("x0", "x1"), "t0", dict(a)),
             NodeSpec("MUL", ("t0", "x2"), "t1", dict(a)),
             NodeSpec("SCALE_IMM", ("t1",), "t2", dict(a, scalar=0.5)),
             NodeSpec("ADD", ("t2", "w"), "t3", dict(a)),
             NodeSpec("MUL", ("t3", "x0"), "t4", dict(a)),
             NodeSpec("COPY", ("t4",), "t5", dict(a)),
             NodeSpec("ADD", ("t5", "x1"), "t6", dict(a)),
             NodeSpec("SCALE_IMM", ("t6",), "out", dict(a, scalar=2.0))]
    name = "C1" if (nelems == 4096 and window is None) else f"C4_{nelems * 4}B_{'win' if window else 'full'}"
    return ChainSpec(name, slots, nodes, [(0, len(nodes) - 1)])


C4_SIZES = [1024 * 4**k for k in range(11)]   # 1 KiB .. 1 GiB per input


def c4_chain(size_bytes: int, window_mode: bool = True) -> ChainSpec:
    return c1_chain(size_bytes // 4, window=4096 if window_mode else None)


# ----------------------------------------------------------------------------- C2

def c2_lane_bytes(i: int) -> int:
    return 1024 * 2 ** (i % 13)


def c2_chain(n_lanes: int = 64, scale_tail: int = 8, reduce_cols: int = 256) -> ChainSpec:
    """per lane l: t=ADD(x_l,w_l); u=MUL(t,x_l); r=REDUCE_SUM(u as [n/256,256]);
    then SCALE_IMM on the reductions of the last `scale_tail` lanes. 64 lanes -> K = 200."""
    slots, nodes = [], []
    for l in range(n_lanes):
        n = c2_lane_bytes(l) // 4
        slots += [SlotSpec(f"x{l}", EXTERNAL, "f32", n), SlotSpec(f"w{l}", STATIC, "f32", n),
                  SlotSpec(f"t{l}", INTERNAL, "f32", n), SlotSpec(f"u{l}", INTERNAL, "f32", n),
                  SlotSpec(f"r{l}", INTERNAL, "f32", n // reduce_cols)]
        nodes += [NodeSpec("ADD", (f"x{l}", f"w{l}"), f"t{l}", {"n": n}),
                  NodeSpec("MUL", (f"t{l}", f"x{l}"), f"u{l}", {"n": n}),
                  NodeSpec("REDUCE_SUM", (f"u{l}",), f"r{l}", {"n": n, "cols": reduce_cols})]
    for l in range(n_lanes - scale_tail, n_lanes):
        m = c2_lane_bytes(l) // 4 // reduce_cols
        slots.append(SlotSpec(f"s{l}", INTERNAL, "f32", m))
        nodes.append(NodeSpec("SCALE_IMM", (f"r{l}",), f"s{l}", {"n": m, "scalar": 0.25}))
    return ChainSpec("C2" if n_lanes == 64 else f"C2_{n_lanes}", slots, nodes,
                     [(0, len(nodes) - 1)])


# ----------------------------------------------------------------------------- C3 / C5

GPT2 = dict(d=768, heads=12, head_dim=64, d_ff=3072, eps=1e-5)


def c3_chain(T: int = 128, n_layers: int = 12, tp: int = 1, rank: int = 0,
             fuse_residual: bool = False, fuse_allreduce: bool = False) -> ChainSpec:
    """GPT-2-small-shaped decoder chain: per layer LN1, QKV GEMM+bias,
    causal attention, O-proj GEMM+bias, residual ADD, LN2, FC1 GEMM+bias+GELU, FC2 GEMM+bias,
    residual ADD. Only x is EXTERNAL; weights are STATIC (SURVEY ambiguity 4).

    With tp > 1 this is rank `rank`'s shard: QKV and FC1 column-sharded
    (heads / d_ff split p ways; at p=8 the 12 heads are padded to 16 with zero weights,
    SURVEY ambiguity 13), O-proj and FC2 row-sharded with their bias on rank 0 only, each
    followed by ALLREDUCE_SUM. Shard weights are SLICES of the TP=1 weights (see tp_weight).

    fuse_residual (tp == 1 only; SURVEY §8(a) "residual adds may be fused into the GEMM epilogue"):
    the O-proj and FC2 GEMMs take the residual stream as a 4th input and write h1 / h2 directly,
    7 nodes per layer instead of 9 (one bf16 rounding of A W^T + b + residual instead of two)."""
    assert not (fuse_residual and tp > 1), "residual fusion needs the un-reduced sum (TP = 1)"
    # fuse_allreduce (tp > 1, NEXT-4): the O-proj / FC2 GEMMs carry "allreduce" (their epilogue sums
    # the output tile over the ranks through peer memory) instead of separate ALLREDUCE_SUM nodes
    fuse_ar = fuse_allreduce and tp > 1
    d, hd, dff, eps = GPT2["d"], GPT2["head_dim"], GPT2["d_ff"], GPT2["eps"]
    H = GPT2["heads"]
    Hp = H if H % tp == 0 else ((H + tp - 1) // tp) * tp   # 12 -> 16 at tp=8
    hl = Hp // tp                                            # heads per rank
    fl = dff // tp
    slots = [SlotSpec("x", EXTERNAL, "bf16", T * d)]
    nodes = []
    h = "x"
    for l in range(n_layers):
        p = f"L{l}."
        slots += [SlotSpec(p + "ln1_g", STATIC, "bf16", d, "gamma"),
                  SlotSpec(p + "ln1_b", STATIC, "bf16", d, "bias"),
                  SlotSpec(p + "w_qkv", STATIC, "bf16", 3 * hl * hd * d, "weight"),
                  SlotSpec(p + "b_qkv", STATIC, "bf16", 3 * hl * hd, "bias"),
                  SlotSpec(p + "w_o", STATIC, "bf16", d * hl * hd, "weight"),
                  SlotSpec(p + "b_o", STATIC, "bf16", d, "bias"),
                  SlotSpec(p + "ln2_g", STATIC, "bf16", d, "gamma"),
                  SlotSpec(p + "ln2_b", STATIC, "bf16", d, "bias"),
                  SlotSpec(p + "w_fc1", STATIC, "bf16", fl * d, "weight"),
                  SlotSpec(p + "b_fc1", STATIC, "bf16", fl, "bias"),
                  SlotSpec(p + "w_fc2", STATIC, "bf16", d * fl, "weight"),
                  SlotSpec(p + "b_fc2", STATIC, "bf16", d, "bias")]
        for nm, n in (("a", T * d), ("qkv", T * 3 * hl * hd), ("att", T * hl * hd), ("o", T * d),
                      ("h1", T * d), ("a2", T * d), ("f", T * fl), ("g", T * d), ("h2", T * d)):
            slots.append(SlotSpec(p + nm, INTERNAL, "bf16", n))   # (o, g stay when fused: same slot
                                                                    # indices -> same seeded weights)
        # TP: the all-reduced sums get their own slots (not in place), so every rank's partial and
        # the reduced value both stay observable for the node-local parity check
        o_sum, g_sum = (p + "o_sum", p + "g_sum") if tp > 1 and not fuse_ar else (p + "o", p + "g")
        if tp > 1 and not fuse_ar:
            slots += [SlotSpec(o_sum, INTERNAL, "bf16", T * d), SlotSpec(g_sum, INTERNAL, "bf16", T * d)]
        if fuse_residual:
            nodes += [
                NodeSpec("LAYERNORM", (h, p + "ln1_g", p + "ln1_b"), p + "a",
                         {"rows": T, "cols": d, "eps": eps}),
                NodeSpec("GEMM_BF16", (p + "a", p + "w_qkv", p + "b_qkv"), p + "qkv",
                         {"M": T, "N": 3 * hl * hd, "K": d, "bias": True, "gelu": False}),
                NodeSpec("ATTN_CAUSAL", (p + "qkv",), p + "att",
                         {"T": T, "H": hl, "D": hd, "scale": 0.125}),
                NodeSpec("GEMM_BF16", (p + "att", p + "w_o", p + "b_o", h), p + "h1",
                         {"M": T, "N": d, "K": hl * hd, "bias": True, "gelu": False, "residual": True}),
                NodeSpec("LAYERNORM", (p + "h1", p + "ln2_g", p + "ln2_b"), p + "a2",
                         {"rows": T, "cols": d, "eps": eps}),
                NodeSpec("GEMM_BF16", (p + "a2", p + "w_fc1", p + "b_fc1"), p + "f",
                         {"M": T, "N": fl, "K": d, "bias": True, "gelu": True}),
                NodeSpec("GEMM_BF16", (p + "f", p + "w_fc2", p + "b_fc2", p + "h1"), p + "h2",
                         {"M": T, "N": d, "K": fl, "bias": True, "gelu": False, "residual": True}),
            ]
            h = p + "h2"
            continue
        bias_ro = (rank == 0)
        nodes += [
            NodeSpec("LAYERNORM", (h, p + "ln1_g", p + "ln1_b"), p + "a",
                     {"rows": T, "cols": d, "eps": eps}),
            NodeSpec("GEMM_BF16", (p + "a", p + "w_qkv", p + "b_qkv"), p + "qkv",
                     {"M": T, "N": 3 * hl * hd, "K": d, "bias": True, "gelu": False}),
            NodeSpec("ATTN_CAUSAL", (p + "qkv",), p + "att",
                     {"T": T, "H": hl, "D": hd, "scale": 0.125}),
            NodeSpec("GEMM_BF16", (p + "att", p + "w_o", p + "b_o"), p + "o",
                     {"M": T, "N": d, "K": hl * hd, "bias": bias_ro if tp > 1 else True,
                      "gelu": False, "allreduce": fuse_ar}),
        ]
        if tp > 1 and not fuse_ar:
            nodes.append(NodeSpec("ALLREDUCE_SUM", (p + "o",), o_sum, {"n": T * d}))
        nodes += [
            NodeSpec("ADD", (h, o_sum), p + "h1", {"n": T * d}),
            NodeSpec("LAYERNORM", (p + "h1", p + "ln2_g", p + "ln2_b"), p + "a2",
                     {"rows": T, "cols": d, "eps": eps}),
            NodeSpec("GEMM_BF16", (p + "a2", p + "w_fc1", p + "b_fc1"), p + "f",
                     {"M": T, "N": fl, "K": d, "bias": True, "gelu": True}),
            NodeSpec("GEMM_BF16", (p + "f", p + "w_fc2", p + "b_fc2"), p + "g",
                     {"M": T, "N": d, "K": fl, "bias": bias_ro if tp > 1 else True,
                      "gelu": False, "allreduce": fuse_ar}),
        ]
        if tp > 1 and not fuse_ar:
            nodes.append(NodeSpec("ALLREDUCE_SUM", (p + "g",), g_sum, {"n": T * d}))
        nodes.append(NodeSpec("ADD", (p + "h1", g_sum), p + "h2", {"n": T * d}))
        h = p + "h2"
    name = f"C3_T{T}_L{n_layers}" if tp == 1 else f"C5_T{T}_L{n_layers}_tp{tp}_r{rank}"
    if fuse_residual:
        name += "_fused"
    if fuse_ar:
        name += "_arfused"
    return ChainSpec(name, slots, nodes, [(0, len(nodes) - 1)])


# ----------------------------------------------------------------------------- training-shaped (NEXT-4)

def mlp_train_chain(T: int = 128, d: int = 768, dff: int = 3072, n_blocks: int = 6,
                    lr: float = 0.5, stage_x: bool = False) -> ChainSpec:
    """A training step of a stack of GPT-2-shaped MLP blocks (SURVEY §8(f) NEXT-4 "training-shaped
    (fwd+bwd) chain", P:L694 DGPT2-T), bf16, batch T tokens, no biases, MSE loss:

      forward per block l (a_0 = X):  pre_l = a_l W1_l^T;  h_l = GELU(pre_l);  a_{l+1} = h_l W2_l^T
      loss gradient:                  dy = (a_L - target) * 2 / (T d)
      backward per block (l = L-1..0), with dy the gradient w.r.t. a_{l+1}:
        dW2 = dy^T h_l;  dh = dy W2;  dpre = dh * GELU'(pre_l);  dW1 = dpre^T a_l;  da = dpre W1 (l > 0)
      update:                         W <- W - lr dW (in place)

    Every product is a K-major GEMM (out = A B^T): the transposed operands (dy^T, h^T, W2^T, ...)
    come from TRANSPOSE nodes. The weights are INTERNAL slots updated in place every replay; nodes
    [0, 2 n_blocks) form an init segment that copies the STATIC initial weights into them (run once),
    the rest is the training step (segment 1) with X and target EXTERNAL, fresh every step."""
    slots = [SlotSpec("X", EXTERNAL, "bf16", T * d), SlotSpec("target", EXTERNAL, "bf16", T * d),
             SlotSpec("zb_dff", STATIC, "bf16", dff, "zero"), SlotSpec("zb_d", STATIC, "bf16", d, "zero")]
    nodes = []
    for l in range(n_blocks):
        p = f"B{l}."
        slots += [SlotSpec(p + "W1_0", STATIC, "bf16", dff * d, "weight"),
                  SlotSpec(p + "W2_0", STATIC, "bf16", d * dff, "weight"),
                  SlotSpec(p + "W1", INTERNAL, "bf16", dff * d), SlotSpec(p + "W2", INTERNAL, "bf16", d * dff)]
        nodes += [NodeSpec("COPY", (p + "W1_0",), p + "W1", {"n": dff * d}),
                  NodeSpec("COPY", (p + "W2_0",), p + "W2", {"n": d * dff})]
    n_init = len(nodes)
    g = lambda M, N, K: {"M": M, "N": N, "K": K, "bias": False, "gelu": False}  # noqa: E731
    # the first GEMM reads the EXTERNAL X directly as its A operand (PI through the TMA descriptor:
    # the kernel rebuilds its A tensor map from the pointer table). stage_x = True restores the
    # round-1 variant that staged X with a COPY node (a data copy inside the graph), for comparison.
    a = "X"
    if stage_x:
        slots.append(SlotSpec("x_in", INTERNAL, "bf16", T * d))
        nodes.append(NodeSpec("COPY", ("X",), "x_in", {"n": T * d}))
        a = "x_in"
    acts = []
    for l in range(n_blocks):
        p = f"B{l}."
        for nm, n in (("pre", T * dff), ("h", T * dff), ("y", T * d)):
            slots.append(SlotSpec(p + nm, INTERNAL, "bf16", n))
        nodes += [NodeSpec("GEMM_BF16", (a, p + "W1", "zb_dff"), p + "pre", g(T, dff, d)),
                  NodeSpec("GELU", (p + "pre",), p + "h", {"n": T * dff}),
                  NodeSpec("GEMM_BF16", (p + "h", p + "W2", "zb_d"), p + "y", g(T, d, dff))]
        acts.append(a)
        a = p + "y"
    slots += [SlotSpec("r", INTERNAL, "bf16", T * d), SlotSpec("dyL", INTERNAL, "bf16", T * d)]
    nodes += [NodeSpec("SUB", (a, "target"), "r", {"n": T * d}),
              NodeSpec("SCALE_IMM", ("r",), "dyL", {"n": T * d, "scalar": 2.0 / (T * d)})]
    dy = "dyL"
    for l in reversed(range(n_blocks)):
        p = f"B{l}."
        for nm, n in (("dyT", d * T), ("hT", dff * T), ("dW2", d * dff), ("W2T", dff * d), ("dh", T * dff),
                      ("dpre", T * dff), ("dpreT", dff * T), ("aT", d * T), ("dW1", dff * d),
                      ("W1T", d * dff), ("da", T * d)):
            slots.append(SlotSpec(p + nm, INTERNAL, "bf16", n))
        nodes += [NodeSpec("TRANSPOSE", (dy,), p + "dyT", {"n": T * d, "cols": d}),
                  NodeSpec("TRANSPOSE", (p + "h",), p + "hT", {"n": T * dff, "cols": dff}),
                  NodeSpec("GEMM_BF16", (p + "dyT", p + "hT", "zb_dff"), p + "dW2", g(d, dff, T)),
                  NodeSpec("TRANSPOSE", (p + "W2",), p + "W2T", {"n": d * dff, "cols": dff}),
                  NodeSpec("GEMM_BF16", (dy, p + "W2T", "zb_dff"), p + "dh", g(T, dff, d)),
                  NodeSpec("GELU_BWD", (p + "dh", p + "pre"), p + "dpre", {"n": T * dff}),
                  NodeSpec("TRANSPOSE", (p + "dpre",), p + "dpreT", {"n": T * dff, "cols": dff}),
                  NodeSpec("TRANSPOSE", (acts[l],), p + "aT", {"n": T * d, "cols": d}),
                  NodeSpec("GEMM_BF16", (p + "dpreT", p + "aT", "zb_d"), p + "dW1", g(dff, d, T))]
        if l > 0:
            nodes += [NodeSpec("TRANSPOSE", (p + "W1",), p + "W1T", {"n": dff * d, "cols": d}),
                      NodeSpec("GEMM_BF16", (p + "dpre", p + "W1T", "zb_d"), p + "da", g(T, d, dff))]
            dy = p + "da"
        nodes += [NodeSpec("AXPY", (p + "W2", p + "dW2"), p + "W2", {"n": d * dff, "scalar": -lr}),
                  NodeSpec("AXPY", (p + "W1", p + "dW1"), p + "W1", {"n": dff * d, "scalar": -lr})]
    return ChainSpec(f"MLPT_T{T}_B{n_blocks}", slots, nodes, [(0, n_init - 1), (n_init, len(nodes) - 1)])


def tp_weight(full: ChainSpec, name: str, tp: int, rank: int, values: np.ndarray) -> np.ndarray:
    """Slice the TP=1 value array of weight slot `name` (bf16 bits) into rank `rank`'s shard.

    Layouts (row-major, nn.Linear [out, in]): w_qkv [3*H*64, 768] with rows q|k|v, head-major;
    w_o [768, H*64]; w_fc1 [3072, 768]; w_fc2 [768, 3072]. Padded heads get zero rows/cols."""
    d, hd, dff, H = GPT2["d"], GPT2["head_dim"], GPT2["d_ff"], GPT2["heads"]
    Hp = H if H % tp == 0 else ((H + tp - 1) // tp) * tp
    hl = Hp // tp
    fl = dff // tp
    base = name.split(".", 1)[1]
    v = np.asarray(values)
    if base in ("w_qkv", "b_qkv"):
        cols = d if base == "w_qkv" else 1
        w = v.reshape(3, H, hd, cols)
        pad = np.zeros((3, Hp, hd, cols), v.dtype)
        pad[:, :H] = w
        return pad[:, rank * hl:(rank + 1) * hl].reshape(-1).copy()
    if base == "w_o":
        w = v.reshape(d, H * hd)
        pad = np.zeros((d, Hp * hd), v.dtype)
        pad[:, :H * hd] = w
        return pad[:, rank * hl * hd:(rank + 1) * hl * hd].reshape(-1).copy()
    if base in ("w_fc1", "b_fc1"):
        cols = d if base == "w_fc1" else 1
        return v.reshape(dff, cols)[rank * fl:(rank + 1) * fl].reshape(-1).copy()
    if base == "w_fc2":
        return v.reshape(d, dff)[:, rank * fl:(rank + 1) * fl].reshape(-1).copy()
    return v.copy()   # LN params and O/FC2 biases are replicated


def static_values(chain: ChainSpec, mode: str = "uniform", tp: int = 1, rank: int = 0,
                  full: ChainSpec | None = None) -> dict:
    """name -> host values for every STATIC slot (TP shards sliced from the TP=1 chain)."""
    out = {}
    for s in chain.slots:
        if s.kind != STATIC:
            continue
        if tp == 1:
            out[s.name] = slot_values(chain, s.name, mode=mode)
        else:
            assert full is not None
            out[s.name] = tp_weight(full, s.name, tp, rank, slot_values(full, s.name, mode=mode))
    return out


def external_values(chain: ChainSpec, replay: int, mode: str = "uniform") -> dict:
    return {s.name: slot_values(chain, s.name, replay, mode) for s in chain.externals()}
