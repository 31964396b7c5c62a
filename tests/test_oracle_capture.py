"""Pins for oracle/chain.py and oracle/capture.py (O1-O3), no GPU.

What pins them: replay == eager for every non-stale arm over >= 100 random
replays, the staleness witness (criterion 1 S:L554), copy-byte
accounting (Table 3), copy minimality and a brute-force
enumeration of rebinding subsets on a tiny chain.
"""
import itertools
import struct

import numpy as np
import pytest

from oracle import capture as cap
from oracle.chain import eval_chain
from synth import workloads as wl
from synth.workloads import EXTERNAL, INTERNAL, STATIC, ChainSpec, NodeSpec, SlotSpec


def _run_arm(chain, mode, replays, mode_vals="uniform"):
    mem = cap.Memory()
    st = wl.static_values(chain, mode=mode_vals)
    saddr = cap.load_statics(chain, mem, st)
    first = cap.load_inputs(chain, mem, wl.external_values(chain, 0, mode_vals))
    ex = cap.CapturedExec(chain, mode, mem, saddr,
                          capture_ext_addr=first if mode == "STALE" else None)
    outs = []
    for r in range(replays):
        addrs = first if r == 0 else cap.load_inputs(chain, mem, wl.external_values(chain, r, mode_vals))
        res = ex.bind(addrs)
        outs.append(({k: v.copy() for k, v in ex.replay().items()}, res))
    return outs, st


def _eager(chain, r, st, mode_vals="uniform"):
    return eval_chain(chain, wl.external_values(chain, r, mode_vals), st)


@pytest.mark.parametrize("mode", ["COPY", "INDIRECT", "SETPARAMS"])
def test_replay_equals_eager_c1_100_replays(mode):
    chain = wl.c1_chain(nelems=64)   # small C1 for 100 replays
    outs, st = _run_arm(chain, mode, 100)
    for r, (o, _) in enumerate(outs):
        env = _eager(chain, r, st)
        for s in chain.internals():
            assert np.array_equal(o[s.name], env[s.name]), (mode, r, s.name)


def test_stale_diverges_and_equals_capture_time_eager():
    chain = wl.c1_chain()
    outs, st = _run_arm(chain, "STALE", 4)
    env0 = _eager(chain, 0, st)
    for r, (o, _) in enumerate(outs):
        assert np.array_equal(o["out"], env0["out"])          # frozen capture-time inputs
        if r > 0:
            assert not np.array_equal(o["out"], _eager(chain, r, st)["out"])   # witness


def test_c2_replay_equals_eager_all_arms():
    chain = wl.c2_chain(n_lanes=16)
    for mode in ("COPY", "INDIRECT", "SETPARAMS"):
        outs, st = _run_arm(chain, mode, 2)
        for r, (o, _) in enumerate(outs):
            env = _eager(chain, r, st)
            for s in chain.internals():
                assert np.array_equal(o[s.name], env[s.name])


def test_copy_bytes_and_minimality():
    chain = wl.c1_chain()
    outs, _ = _run_arm(chain, "COPY", 3)
    for o, res in outs:
        assert res.bytes_data_rebound == 3 * 4096 * 4
        internal = {s.name for s in chain.internals()}
        assert len(res.copies) == 3 and all(j < 3 for j, *_ in res.copies)
        assert not internal & {chain.externals()[j].name for j, *_ in res.copies}


def test_spec_copy_bytes_three_mib():
    # 3 external tensors of 1 MB each -> bytes_copied_per_replay = 3,145,728
    slots = [SlotSpec(f"x{i}", EXTERNAL, "f32", 2**18) for i in range(3)] + \
            [SlotSpec("t", INTERNAL, "f32", 2**18), SlotSpec("u", INTERNAL, "f32", 2**18)]
    nodes = [NodeSpec("ADD", ("x0", "x1"), "t"), NodeSpec("MUL", ("t", "x2"), "u")]
    c = ChainSpec("spec3", slots, nodes)
    assert cap.copy_plan_bytes(c) == 3_145_728
    assert cap.pointer_bytes(c) == 24


@pytest.mark.parametrize("name,before,n_ptr,after", [
    ("DR-I", 3 * 2**30, 1, 8),         # P:L828 3.0 GB -> 8.0 B
    ("XLNET-I", 8 * 1024, 2, 16),      # P:L825 8.0 KB -> 16.0 B
    ("ALNET", 2 * 3 * 224 * 224 * 2, 1, 8),    # P:L831 588.0 KB -> 8.0 B (bs 2, 16-bit image)
    ("DNET", 64 * 3 * 224 * 224 * 2, 1, 8),    # P:L834 18.4 MB -> 8.0 B (bs 64)
    ("LCNET", 256 * 3 * 224 * 224 * 2, 1, 8),  # P:L833 73.5 MB -> 8.0 B (bs 256)
])
def test_table3_pointer_bytes(name, before, n_ptr, after):
    per = before // n_ptr // 2
    slots = [SlotSpec(f"x{i}", EXTERNAL, "bf16", per) for i in range(n_ptr)]
    slots += [SlotSpec("w", STATIC, "bf16", 1), SlotSpec("y", INTERNAL, "bf16", 1)]
    nodes = [NodeSpec("ADD", (f"x{i}", "w"), "y", {"n": 1}) for i in range(n_ptr)]
    c = ChainSpec(name, slots, nodes)
    assert cap.copy_plan_bytes(c) == before
    assert cap.pointer_bytes(c) == after


def test_table3_after_bytes_are_multiples_of_8():
    after = [16, 336, 24, 184, 232, 136, 120, 16, 8, 8, 16, 16, 24, 8, 8, 312, 24, 8, 32, 16,
             16, 56, 136, 136, 136]   # Table 3, all 25 rows
    assert len(after) == 25 and all(a % 8 == 0 for a in after)


def test_table_bytes_are_the_addresses():
    chain = wl.c1_chain(nelems=16)
    mem = cap.Memory()
    saddr = cap.load_statics(chain, mem, wl.static_values(chain))
    ex = cap.CapturedExec(chain, "INDIRECT", mem, saddr)
    addrs = [0x7F00_0000_1000, 0x7F00_0000_2000, 0x7F00_0000_3000]
    res = ex.bind(addrs)
    assert res.table == struct.pack("<3Q", *addrs) and res.bytes_ptr_rebound == 24


def test_setparam_nodes_per_config():
    assert cap.setparam_nodes(wl.c1_chain()) == [0, 1, 4, 6]        # C1 4 nodes
    assert len(cap.setparam_nodes(wl.c2_chain())) == 128            # C2: 2 per lane
    c3 = wl.c3_chain(T=4, n_layers=2)
    assert len(cap.setparam_nodes(c3)) == 2                         # C3: LN1 + residual


def test_bind_same_address_copies_nothing():
    chain = wl.c1_chain(nelems=16)
    mem = cap.Memory()
    saddr = cap.load_statics(chain, mem, wl.static_values(chain))
    ex = cap.CapturedExec(chain, "COPY", mem, saddr)
    res = ex.bind([ex.placeholder[j] for j in range(3)])            # ambiguity 1
    assert res.bytes_data_rebound == 0 and res.copies == []


def test_missing_input():
    chain = wl.c1_chain(nelems=16)
    mem = cap.Memory()
    ex = cap.CapturedExec(chain, "INDIRECT", mem, cap.load_statics(chain, mem, wl.static_values(chain)))
    with pytest.raises(ValueError):
        ex.bind([1, 2])


def test_bruteforce_rebinding_subsets():
    """Enumerate all 2^N subsets S of externals to rebind on a tiny chain with one declared but
    unread external. Replay == eager for every fresh input iff S contains every READ external."""
    slots = [SlotSpec(f"x{i}", EXTERNAL, "f32", 8) for i in range(4)] + \
            [SlotSpec("w", STATIC, "f32", 8)] + \
            [SlotSpec(n, INTERNAL, "f32", 8) for n in ("a", "b", "c")]
    nodes = [NodeSpec("ADD", ("x0", "w"), "a"), NodeSpec("MUL", ("a", "x2"), "b"),
             NodeSpec("ADD", ("b", "x1"), "c")]
    c = ChainSpec("tiny", slots, nodes)
    read = {0, 1, 2}                                              # x3 is never read
    st = wl.static_values(c)
    for k in range(5):
        for S in itertools.combinations(range(4), k):
            mem = cap.Memory()
            ex = cap.CapturedExec(c, "COPY", mem, cap.load_statics(c, mem, st))
            ok = True
            for r in range(3):
                addrs = cap.load_inputs(c, mem, wl.external_values(c, r))
                ex.bind(addrs, only=set(S))
                out = ex.replay()["c"]
                ok &= np.array_equal(out, eval_chain(c, wl.external_values(c, r), st)["c"])
            assert ok == read.issubset(S), S
