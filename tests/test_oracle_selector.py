"""Pins for oracle/selector.py (O4), no GPU.

SPEC worked examples, the paper's named cases (EOS P:L738/L790, tiny tensors
P:L642-644, VM 4 of 21 P:L848), never-worse, and a brute force over all 3^S
per-segment policies under the additive model.
"""
import itertools
import random

import pytest
from hypothesis import given, settings
from hypothesis import strategies as hs

from oracle import selector as sel
from oracle.selector import EAGER, GRAPH_COPY, GRAPH_INDIRECT


def test_spec_eager_examples():
    assert sel.t_eager(10.0, [100.0]) == 110.0
    assert sel.t_eager(5.0, [100.0] * 10) == 1005.0


def test_dalle2_analog_launch_bound():
    # S:L407 / P:L171: 740 kernels, 3.4 ms device, 14 ms end-to-end -> ~75% launch-bound
    L = 14000.0 / 740
    d = [3400.0 / 740] * 740
    t = sel.t_eager(L, d)
    assert abs(t - 14000.0) / 14000.0 <= 0.02
    assert 1 - sum(d) / t >= 0.73


def test_spec_replay_closed_form():
    # 7.5 + 2 x (0.5 + 10) + 2 = 30.5 us (zero-copy graph, one output rebuild of 2 us)
    assert sel.t_graph(7.5, 0.5, [10.0, 10.0], F=2.0) == 30.5


def _prof(L=5.0, G=7.5, delta=0.5, d=(10.0,), c_copy=0.0, c_ind=0.0, **kw):
    p = dict(L=L, G=G, delta=delta, d=list(d), c_copy=c_copy, c_ind=c_ind)
    p.update(kw)
    return p


def test_eos_like_picks_eager():
    # short kernels, replay overhead ~50%; graph 1.29x slower than eager -> disable
    p = dict(use_measured=True, t_eager=100.0, t_copy=129.0, t_ind=129.0)
    assert sel.select([p]) == [EAGER]


def test_tiny_tensor_prefers_copy_over_pi():
    # P:L642-644 / S:L462: H2D pointer copy costs more than the small D2D data copy
    p = _prof(L=8.0, d=[2.0] * 20, c_copy=1.0, c_ind=3.0)
    assert sel.select([p]) == [GRAPH_COPY]


def test_large_copy_prefers_pi():
    # DR-I-like 3 GB copy vs an 8-byte pointer write
    p = _prof(L=8.0, d=[2.0] * 20, c_copy=3 * 2**30 / 2000e3, c_ind=3.0)
    assert sel.select([p]) == [GRAPH_INDIRECT]


def test_ind_unavailable_drops_candidate():
    p = _prof(L=8.0, d=[2.0] * 20, c_copy=50.0, c_ind=1.0, ind_available=False)
    assert sel.select([p]) == [GRAPH_COPY]


def test_ties_follow_fixed_order():
    assert sel.decide(1.0, 1.0, 1.0) == EAGER
    assert sel.decide(2.0, 1.0, 1.0) == GRAPH_COPY
    assert sel.decide(2.0, 2.0, 1.0) == GRAPH_INDIRECT


def test_vm_analog_4_of_21():
    # VM exposes 21 candidate CGs, 4 enabled, 17 disabled
    profs = []
    for s in range(21):
        good = s % 5 == 0 and s < 20
        profs.append(dict(use_measured=True, t_eager=100.0,
                          t_copy=80.0 if good else 120.0, t_ind=85.0 if good else 125.0))
    dec = sel.select(profs)
    assert sum(1 for x in dec if x != EAGER) == 4 and dec.count(EAGER) == 17


def test_deploy_iff_benefit_exceeds_rebinding_cost():
    """North-star wording: graph deployed iff t_eager - t_graph > rebinding cost (PI off)."""
    rnd = random.Random(1)
    for _ in range(2000):
        p = _prof(L=rnd.uniform(1, 10), G=rnd.uniform(1, 10), delta=rnd.uniform(0, 2),
                  d=[rnd.uniform(0.5, 30) for _ in range(rnd.randint(1, 30))],
                  c_copy=rnd.uniform(0, 200), c_ind=1e9, ind_available=False)
        te = sel.t_eager(p["L"], p["d"])
        tg = sel.t_graph(p["G"], p["delta"], p["d"])
        assert (sel.select([p])[0] == GRAPH_COPY) == (te - tg > p["c_copy"] and te > tg + p["c_copy"])


@settings(max_examples=300, deadline=None)
@given(hs.lists(hs.tuples(hs.floats(0, 1e4), hs.floats(0, 1e4), hs.floats(0, 1e4)),
                min_size=1, max_size=6))
def test_never_worse_and_bruteforce_policies(segs):
    """Per-segment argmin == global optimum over all 3^S policies (additive model); the chosen
    total is never worse than all-eager or all-graph."""
    profs = [dict(use_measured=True, t_eager=a, t_copy=b, t_ind=c) for a, b, c in segs]
    dec = sel.select(profs)
    chosen = sum(segs[i][d] for i, d in enumerate(dec))
    best = min(sum(segs[i][pol[i]] for i in range(len(segs)))
               for pol in itertools.product(range(3), repeat=len(segs)))
    assert chosen == best
    assert chosen <= sum(a for a, _, _ in segs) and chosen <= sum(b for _, b, _ in segs)
    for i, d in enumerate(dec):                 # tie order: first minimal candidate
        assert d == min(range(3), key=lambda k: (segs[i][k], k))


def test_estimate_path_matches_manual_sums():
    p = _prof(L=3.0, G=4.0, delta=0.25, d=[1.5, 2.5, 3.0], c_copy=2.0, c_ind=0.5)
    te, tc, ti = sel.estimates(p)
    assert te == 9.0 + 3.0                       # issue_3 = 9, GPU idle before each start
    assert tc == 4.0 + 1.75 + 2.75 + 3.25 + 2.0
    assert ti == 4.0 + 1.75 + 2.75 + 3.25 + 0.5
