"""Generator and workload-shape checks (no GPU)."""
import numpy as np
import ml_dtypes

from synth import splitmix as sm
from synth import workloads as wl


def test_splitmix_reference_value():
    # splitmix64 from state 0: first output 0xE220A8397B1DCDAF (Steele/Vigna reference)
    assert int(sm._mix(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_values_exact_and_deterministic():
    a = sm.uniform_f32(sm.SEED, 5, 10000)
    assert np.array_equal(a, sm.uniform_f32(sm.SEED, 5, 10000))
    assert a.min() >= -1 and a.max() < 1
    assert np.array_equal((a.astype(np.float64) + 1) * 2**23 % 1, np.zeros(10000))
    b = sm.bf16_bits_to_f32(sm.uniform_bf16_bits(sm.SEED, 6, 5000))
    assert np.array_equal(b.astype(ml_dtypes.bfloat16).astype(np.float32), b)
    assert set(np.unique(sm.int_f32(sm.SEED, 7, 1000)).tolist()) == {-2, -1, 0, 1, 2}
    g = sm.bf16_bits_to_f32(sm.gamma_bf16_bits(sm.SEED, 8, 1000))
    assert g.min() >= 0.9375 and g.max() < 1.06


def test_config_shapes():
    c1 = wl.c1_chain()
    assert len(c1.nodes) == 8 and [s.nelems for s in c1.externals()] == [4096] * 3
    c2 = wl.c2_chain()
    assert len(c2.nodes) == 200 and len(c2.externals()) == 64
    assert sum(s.nbytes for s in c2.externals()) == 37_743_616
    assert len(wl.c3_chain().nodes) == 108
    assert len(wl.c3_chain(tp=8).nodes) == 132
    assert [len(wl.c4_chain(s).externals()) for s in wl.C4_SIZES] == [3] * 11
    assert wl.C4_SIZES[0] == 1024 and wl.C4_SIZES[-1] == 2**30


def test_tp_shards_partition_weights():
    full = wl.c3_chain(T=4, n_layers=1)
    for tp in (2, 4, 8):
        parts = [wl.c3_chain(T=4, n_layers=1, tp=tp, rank=r) for r in range(tp)]
        for nm in ("L0.w_fc1", "L0.w_qkv", "L0.w_o"):
            v = wl.slot_values(full, nm)
            shards = [wl.tp_weight(full, nm, tp, r, v) for r in range(tp)]
            assert all(s.size == p.slot(nm).nelems for s, p in zip(shards, parts))
            nz = sum(int(np.count_nonzero(s)) for s in shards)
            assert nz == int(np.count_nonzero(v))          # padding adds only zeros
