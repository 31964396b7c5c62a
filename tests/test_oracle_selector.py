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


# ---- model 1: the dependency-DAG replay (oracle/selector.py t_graph_dag)

def _paths_ending(deps, k):
    """Every path p_1 -> ... -> p_m = k of the DAG (brute force, tiny DAGs)."""
    if not deps[k]:
        return [[k]]
    out = [[k]]
    for j in deps[k]:
        out += [p + [k] for p in _paths_ending(deps, j)]
    return out


def _span_by_paths(delta, lam, g, deps):
    """Closed form of the list schedule: fin_k = max over paths ending at k of
    issue_{p_1} + sum_i g_{p_i} + (m - 1) lam (each max in the recurrence picks the issue time or
    one predecessor), S = max_k fin_k. Independent of the recurrence's code path."""
    best = 0.0
    for k in range(len(g)):
        for p in _paths_ending(deps, k):
            v = (p[0] + 1) * delta + sum(g[i] for i in p) + (len(p) - 1) * lam
            best = max(best, v)
    return best


def _random_dag(rnd, K):
    return [sorted(rnd.sample(range(k), rnd.randint(0, min(k, 3)))) if k else [] for k in range(K)]


def test_dag_model_equals_path_enumeration():
    rnd = random.Random(7)
    for _ in range(400):
        K = rnd.randint(1, 7)
        deps = _random_dag(rnd, K)
        g = [rnd.uniform(0, 10) for _ in range(K)]
        delta, lam = rnd.uniform(0, 3), rnd.uniform(0, 3)
        S = _span_by_paths(delta, lam, g, deps)
        assert abs(sel.t_graph_dag(0.0, delta, lam, g, deps) - S) <= 1e-9 * max(1.0, S)
        G = rnd.uniform(0, 40)
        assert abs(sel.t_graph_dag(G, delta, lam, g, deps, F=1.5) - (max(G, S) + 1.5)) <= 1e-9 * max(1.0, S)


def test_dag_model_linear_chain_is_the_serial_form():
    # a linear chain with lam == delta and no host bound: sum_k (delta + g_k) + F, the serial
    # replay form of S:L413 (with G = 0); S:L417's example numbers
    g = [10.0, 10.0]
    assert sel.t_graph_dag(0.0, 0.5, 0.5, g, [[], [0]], F=2.0) == sel.t_graph(0.0, 0.5, g, F=2.0) == 23.0
    rnd = random.Random(3)
    for _ in range(100):
        K = rnd.randint(1, 40)
        g = [rnd.uniform(0, 5) for _ in range(K)]
        d = rnd.uniform(0, 2)
        chain = [[]] + [[k - 1] for k in range(1, K)]
        assert abs(sel.t_graph_dag(0.0, d, d, g, chain) - sel.t_graph(0.0, d, g)) <= 1e-9 * K * 10


def test_dag_model_independent_nodes_are_issue_bound():
    # no dependencies: every node starts at its issue time; the span is max_k (k+1) delta + g_k
    g = [5.0, 0.1, 0.1, 0.1]
    assert sel.t_graph_dag(0.0, 1.0, 9.0, g, [[], [], [], []]) == 6.0
    assert sel.t_graph_dag(0.0, 1.0, 9.0, [0.1, 0.1, 0.1, 5.0], [[], [], [], []]) == 9.0


def test_dag_estimates_dispatch():
    p = _prof(L=3.0, G=4.0, delta=0.25, d=[1.5, 2.5, 3.0], c_copy=2.0, c_ind=0.5,
              model=1, lam=1.0, g=[1.0, 2.0, 3.0], deps=[[], [0], [0]])
    te, tc, ti = sel.estimates(p)
    S = max(0.25 + 1.0, 1.25 + 1.0 + 2.0, 1.25 + 1.0 + 3.0)
    assert te == 12.0 and tc == max(4.0, S) + 2.0 and ti == max(4.0, S) + 0.5
