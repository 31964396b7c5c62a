"""Oracle pins driven by the values the paper and the SPEC print (tests/golden/, each cited):
Table 3's byte reductions and the SPEC's worked examples. No value here comes from the
CUDA path or from the oracle itself."""
import json
import os

import numpy as np
import pytest

from oracle import capture as cap
from oracle import ops
from oracle import selector as sel
from synth.workloads import EXTERNAL, INTERNAL, STATIC, ChainSpec, NodeSpec, SlotSpec

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_table3_after_bytes_are_whole_pointers():
    t3 = _load("paper_table3_bytes.json")
    assert len(t3["rows"]) == 25
    for app, _before, after, _graphs in t3["rows"]:
        assert after % 8 == 0 and after > 0, app          # 8 B per rebound pointer


@pytest.mark.parametrize("case", _load("paper_table3_bytes.json")["worked"], ids=lambda c: c["app"])
def test_table3_worked_rows(case):
    n = case["n_pointers"]
    per = case["before_bytes"] // n // 2
    slots = [SlotSpec(f"x{i}", EXTERNAL, "bf16", per) for i in range(n)]
    slots += [SlotSpec("w", STATIC, "bf16", 1), SlotSpec("y", INTERNAL, "bf16", 1)]
    nodes = [NodeSpec("ADD", (f"x{i}", "w"), "y", {"n": 1}) for i in range(n)]
    c = ChainSpec(case["app"], slots, nodes)
    assert cap.copy_plan_bytes(c) == case["before_bytes"]
    assert cap.pointer_bytes(c) == case["after_bytes"]


def test_spec_scale_by_scalar():
    g = _load("spec_worked_examples.json")["scale_by_scalar"]
    out = ops.scale_imm(np.array(g["x"], np.float32), {"scalar": g["s"]})
    assert out.tolist() == g["out"]


@pytest.mark.parametrize("case", _load("spec_worked_examples.json")["eager_recurrence"], ids=lambda c: c["cite"])
def test_spec_eager_recurrence(case):
    if "durations_us" in case:
        assert sel.t_eager(case["launch_us"], case["durations_us"]) == case["total_us"]
    else:
        d = [case["sum_durations_us"] / case["n_kernels"]] * case["n_kernels"]
        t = sel.t_eager(case["launch_us"], d)
        assert abs(t - case["total_us"]) / case["total_us"] <= case["rel_tol"]


def test_spec_graph_cost_and_copy_bytes():
    g = _load("spec_worked_examples.json")
    gc = g["graph_cost"]
    assert sel.t_graph(gc["graph_launch_us"], gc["delta_us"], gc["durations_us"], F=gc["fixed_us"]) == gc["total_us"]
    cb = g["copy_bytes"]
    n = cb["bytes_each"] // 4
    slots = [SlotSpec(f"x{i}", EXTERNAL, "f32", n) for i in range(cb["n_inputs"])] + \
            [SlotSpec("t", INTERNAL, "f32", n), SlotSpec("u", INTERNAL, "f32", n)]
    nodes = [NodeSpec("ADD", ("x0", "x1"), "t"), NodeSpec("MUL", ("t", "x2"), "u")]
    assert cap.copy_plan_bytes(ChainSpec("spec", slots, nodes)) == cb["total"]
