"""O1 — eager chain evaluator (SPEC interpreter `run_eager` S:L116-124).

Evaluates the nodes of a synth.workloads.ChainSpec in list order on host arrays. This is the
"module without CG" semantics: each node reads the CURRENT value of its inputs (P:L63, L169 —
eager launches with the current pointers, nothing recorded by value).
"""
from __future__ import annotations

import numpy as np

from . import ops
from .numerics import bits_to_f64


def to_host(spec_slot, values):
    """Slot values in the oracle's representation: float32 for f32, float64 bf16-values for bf16
    (input bf16 arrive as uint16 bit patterns from synth)."""
    if spec_slot.dtype == "f32":
        return np.asarray(values, dtype=np.float32)
    v = np.asarray(values)
    return bits_to_f64(v) if v.dtype == np.uint16 else v.astype(np.float64)


def eval_node(chain, node, env, dtype_of):
    """Apply one node; `env` maps slot name -> current host value."""
    op, ins, at = node.op, node.ins, node.attrs
    dt = dtype_of(node.out)
    if op == "ADD":
        return ops.add(env[ins[0]], env[ins[1]], at, dt)
    if op == "MUL":
        return ops.mul(env[ins[0]], env[ins[1]], at, dt)
    if op == "SCALE_IMM":
        return ops.scale_imm(env[ins[0]], at, dt)
    if op == "COPY":
        return ops.copy(env[ins[0]], at, dt)
    if op == "SCALE_T":
        return ops.scale_t(env[ins[0]], env[ins[1]], at, dt)
    if op == "REDUCE_SUM":
        return ops.reduce_sum(env[ins[0]], at, dt)
    if op == "LAYERNORM":
        return ops.layernorm(env[ins[0]], env[ins[1]], env[ins[2]], at)
    if op == "GEMM_BF16":
        res = env[ins[3]] if len(ins) > 3 else None
        return ops.gemm_bf16(env[ins[0]], env[ins[1]], env[ins[2]], at, residual=res)
    if op == "ATTN_CAUSAL":
        return ops.attn_causal(env[ins[0]], at)
    if op == "SUB":
        return ops.sub(env[ins[0]], env[ins[1]], at, dt)
    if op == "AXPY":
        return ops.axpy(env[ins[0]], env[ins[1]], at, dt)
    if op == "GELU":
        return ops.gelu(env[ins[0]], at, dt)
    if op == "GELU_BWD":
        return ops.gelu_bwd(env[ins[0]], env[ins[1]], at, dt)
    if op == "TRANSPOSE":
        return ops.transpose(env[ins[0]], at, dt)
    raise ValueError(f"eval_node: op {op} needs the multi-rank evaluator")


def eval_chain(chain, ext: dict, static: dict, state: dict | None = None, nodes: tuple | None = None) -> dict:
    """Eager evaluation: returns name -> value for every slot after running all nodes once.
    `ext` / `static` map slot names to values as produced by synth (uint16 for bf16).
    `state`: values of INTERNAL slots carried over from a previous step (the training chain's
    weights, updated in place every replay); `nodes`: an inclusive node range (first, last)."""
    env = {}
    for name, v in (state or {}).items():
        env[name] = np.array(v, copy=True)
    for s in chain.slots:
        if s.kind == "external":
            env[s.name] = to_host(s, ext[s.name])
        elif s.kind == "static":
            env[s.name] = to_host(s, static[s.name])
    dtype_of = lambda name: chain.slot(name).dtype  # noqa: E731
    first, last = nodes if nodes is not None else (0, len(chain.nodes) - 1)
    for node in chain.nodes[first:last + 1]:
        env[node.out] = eval_node(chain, node, env, dtype_of)
    return env


def eval_chain_tp(chains: list, ext: list, static: list) -> list:
    """Lockstep evaluation of p rank-chains with identical node structure; ALLREDUCE_SUM nodes
    sum the p partials (ops.allreduce_sum) and hand the result to every rank."""
    envs = []
    for c, e, st in zip(chains, ext, static):
        env = {}
        for s in c.slots:
            if s.kind == "external":
                env[s.name] = to_host(s, e[s.name])
            elif s.kind == "static":
                env[s.name] = to_host(s, st[s.name])
        envs.append(env)
    for k in range(len(chains[0].nodes)):
        nodes = [c.nodes[k] for c in chains]
        if nodes[0].op == "ALLREDUCE_SUM":
            red = ops.allreduce_sum([env[nodes[0].ins[0]] for env in envs])
            for env in envs:
                env[nodes[0].out] = red.copy()
            continue
        if nodes[0].op == "GEMM_BF16" and nodes[0].attrs.get("allreduce"):
            # the GEMM with its all-reduce fused: each rank's bf16 output tile, then ALLREDUCE_SUM
            parts = [eval_node(c, node, env, lambda name, c=c: c.slot(name).dtype)
                     for c, env, node in zip(chains, envs, nodes)]
            red = ops.allreduce_sum(parts)
            for env in envs:
                env[nodes[0].out] = red.copy()
            continue
        for c, env, node in zip(chains, envs, nodes):
            env[node.out] = eval_node(c, node, env, lambda name, c=c: c.slot(name).dtype)
    return envs
