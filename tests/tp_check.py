"""Node-local, element-wise parity of a tensor-parallel chain (SURVEY §8(c) tolerances; VERDICT r1
"What's weak" 1): every node of every rank is re-evaluated by the oracle from the GPU's OWN node
inputs on that rank, so an error cannot hide behind compounding or behind a norm:

* per-rank nodes (LN, column-/row-parallel GEMM shard, attention, residual ADD): the oracle op on
  this rank's GPU inputs, per element |g - o| <= 2e-2 |o| + 2e-2 rms(o) (a dropped 64-wide K-tile of
  a 384-deep shard GEMM is ~0.4 |o|, far outside);
* ALLREDUCE_SUM: the oracle sum of EVERY rank's GPU input partial (f64, one bf16 rounding);
* a GEMM with the all-reduce fused: per rank the oracle GEMM of its own GPU inputs rounded to bf16,
  then summed over ranks (oracle.ops.allreduce_sum), compared with the all-reduced GPU output;
* every rank's all-reduced output bit-identical across ranks.
"""
import numpy as np

from oracle import ops
from oracle.numerics import bits_to_f64


def close(g_bits, o, what=""):
    g = bits_to_f64(g_bits)
    o = np.asarray(o, dtype=np.float64)
    rms = np.sqrt(np.mean(o ** 2)) if o.size else 0.0
    bad = np.abs(g - o) > 2e-2 * np.abs(o) + 2e-2 * rms
    assert not bad.any(), f"{what}: {bad.sum()} of {bad.size} outside tolerance; " \
                          f"max err {np.max(np.abs(g - o)):.4g}, rms {rms:.4g}"


def _env(spec, st, ext, got):
    env = {}
    for s in spec.slots:
        if s.kind == "external":
            env[s.name] = bits_to_f64(ext[s.name])
        elif s.kind == "static":
            env[s.name] = bits_to_f64(st[s.name])
        else:
            env[s.name] = bits_to_f64(got[s.name])
    return env


def _local(node, env):
    a = node.attrs
    if node.op == "LAYERNORM":
        return ops.layernorm(env[node.ins[0]], env[node.ins[1]], env[node.ins[2]], a)
    if node.op == "GEMM_BF16":
        res = env[node.ins[3]] if len(node.ins) > 3 else None
        return ops.gemm_bf16(env[node.ins[0]], env[node.ins[1]], env[node.ins[2]], a, res)
    if node.op == "ATTN_CAUSAL":
        return ops.attn_causal(env[node.ins[0]], a)
    if node.op == "ADD":
        return ops.add(env[node.ins[0]], env[node.ins[1]], a, "bf16")
    if node.op == "COPY":
        return ops.copy(env[node.ins[0]], a, "bf16")
    raise AssertionError(node.op)


def check_tp_node_local(specs, statics, exts, gots, ctx=""):
    """specs/statics/exts/gots: per rank (gots: slot name -> GPU bf16 bits of every INTERNAL slot).
    Returns the number of node outputs checked."""
    p = len(specs)
    envs = [_env(specs[r], statics[r], exts[r], gots[r]) for r in range(p)]
    checked = 0
    for k, node0 in enumerate(specs[0].nodes):
        nodes = [specs[r].nodes[k] for r in range(p)]
        fused = node0.op == "GEMM_BF16" and node0.attrs.get("allreduce")
        if node0.op == "ALLREDUCE_SUM" or fused:
            if fused:
                parts = [_local(nodes[r], envs[r]) for r in range(p)]       # bf16-rounded partials
            else:
                parts = [envs[r][nodes[r].ins[0]] for r in range(p)]        # the GPU's own partials
            ref = ops.allreduce_sum(parts)
            for r in range(p):
                close(gots[r][nodes[r].out], ref, f"{ctx} rank {r} node {k} {node0.op}{' +AR' if fused else ''}")
                assert np.array_equal(gots[r][nodes[r].out], gots[0][nodes[0].out]), (ctx, r, k)
        else:
            for r in range(p):
                close(gots[r][nodes[r].out], _local(nodes[r], envs[r]), f"{ctx} rank {r} node {k} {node0.op}")
        checked += p
    return checked
