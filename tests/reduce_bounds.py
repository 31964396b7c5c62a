"""Shared parity rule for fp32 reductions (SURVEY §8(c) ambiguity 12, DESIGN reading 9): the
oracle sums in float64, the GPU in a fixed tree, so a REDUCE_SUM output r must satisfy
|g - o| <= 1e-5 * sum_c |x[r, c]|; a SCALE_IMM of a reduction scales that bound by |scalar|.
Every other fp32 node is compared bit for bit."""
import numpy as np


def _producer(spec, name):
    return [n for n in spec.nodes if n.out == name][0]


def reduce_bound(spec, env, name):
    """Per-element bound for `name` if a reduction (or a scaled reduction) produces it, else None."""
    prod = _producer(spec, name)
    scale = 1.0
    if prod.op == "SCALE_IMM":
        src = [n for n in spec.nodes if n.out == prod.ins[0]]
        if not src or src[0].op != "REDUCE_SUM":
            return None
        scale = abs(prod.attrs["scalar"])
        prod = src[0]
    if prod.op != "REDUCE_SUM":
        return None
    cols = prod.attrs.get("cols", 256)
    x = np.asarray(env[prod.ins[0]], dtype=np.float64)
    n = prod.attrs.get("n") or x.size
    return scale * 1e-5 * np.abs(x[:n]).reshape(-1, cols).sum(axis=1)


def assert_output(spec, env, name, got, ctx=None):
    """got (GPU) vs env[name] (oracle): the reduction bound where it applies, else bit-exact."""
    o = env[name]
    b = reduce_bound(spec, env, name)
    if b is None:
        assert np.array_equal(got, o), (ctx, name)
    else:
        d = np.abs(np.asarray(got, dtype=np.float64)[: b.size] - np.asarray(o, dtype=np.float64)[: b.size])
        assert np.all(d <= b), (ctx, name, float(np.max(d - b)))
