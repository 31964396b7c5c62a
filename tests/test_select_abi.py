"""cgx_select (pure host function of the C ABI) == oracle/selector.py bit for bit, on random
multi-segment profiles, in both decision modes (measured totals / analytical estimates)."""
import random

import pytest
from hypothesis import given, settings
from hypothesis import strategies as hs

from oracle import selector as sel


@pytest.fixture(scope="module")
def cgx():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx as c
    return c


def _mk(cgx, d):
    p = cgx.Profile()
    p.n_kernels = len(d["d"])
    p.ind_available = int(d["ind_available"])
    p.use_measured = int(d["use_measured"])
    p.model = d.get("model", 0)
    for k in ("L", "G", "delta", "c_copy", "c_ind", "F"):
        setattr(p, k + "_us", d[k])
    p.t_eager_us, p.t_copy_us, p.t_ind_us = d["t_eager"], d["t_copy"], d["t_ind"]
    for i, x in enumerate(d["d"]):
        p.d_us[i] = x
    if p.model == 1:
        p.lambda_us = d["lam"]
        off = 0
        p.dep_off[0] = 0
        for k, dk in enumerate(d["deps"]):
            p.g_us[k] = d["g"][k]
            for j in dk:
                p.dep_idx[off] = j
                off += 1
            p.dep_off[k + 1] = off
        p.n_deps = off
    return p


fl = hs.floats(0.0, 1e5, allow_nan=False, allow_infinity=False)


@settings(max_examples=200, deadline=None)
@given(hs.lists(hs.fixed_dictionaries({
    "L": fl, "G": fl, "delta": hs.floats(-5.0, 50.0), "c_copy": fl, "c_ind": fl, "F": fl,
    "t_eager": fl, "t_copy": fl, "t_ind": fl, "ind_available": hs.booleans(),
    "use_measured": hs.booleans(), "d": hs.lists(fl, min_size=0, max_size=40)}), min_size=1, max_size=8))
def test_select_matches_oracle(cgx, profs):
    dec, est = cgx.select([_mk(cgx, d) for d in profs])
    assert dec == sel.select(profs)
    for d, e in zip(profs, est):
        if d["use_measured"]:
            assert e == (d["t_eager"], d["t_copy"], d["t_ind"])
        else:
            assert e == sel.estimates(d)                 # bit-exact doubles


def test_select_ties_and_unavailable(cgx):
    base = dict(L=1.0, G=1.0, delta=0.0, c_copy=0.0, c_ind=0.0, F=0.0, d=[1.0], ind_available=True,
                use_measured=True)
    for te, tc, ti, want in ((5, 5, 5, 0), (6, 5, 5, 1), (6, 6, 5, 2), (6, 7, 1, 2)):
        d = dict(base, t_eager=te, t_copy=tc, t_ind=ti)
        assert cgx.select([_mk(cgx, d)])[0] == [want] == sel.select([d])
    d = dict(base, t_eager=9.0, t_copy=8.0, t_ind=1.0, ind_available=False)
    assert cgx.select([_mk(cgx, d)])[0] == [1] == sel.select([d])


def test_select_rejects_bad_input(cgx):
    p = cgx.Profile()
    p.n_kernels = cgx.MAX_PROFILE_KERNELS + 1
    with pytest.raises(cgx.CgxError):
        cgx.select([p])
    rnd = random.Random(3)
    ps = [_mk(cgx, dict(L=rnd.random(), G=1, delta=0, c_copy=1, c_ind=2, F=0, t_eager=0, t_copy=0, t_ind=0,
                        ind_available=True, use_measured=False, d=[rnd.random() for _ in range(5)]))
          for _ in range(3)]
    assert len(cgx.select(ps)[0]) == 3


@settings(max_examples=200, deadline=None)
@given(hs.data())
def test_select_dag_model_matches_oracle(cgx, data):
    """Model 1 (dependency-DAG replay list schedule): cgx_select's estimates == oracle bit for bit."""
    profs = []
    for _ in range(data.draw(hs.integers(1, 5))):
        K = data.draw(hs.integers(0, 30))
        deps = [sorted(set(data.draw(hs.lists(hs.integers(0, k - 1), max_size=4)))) if k else [] for k in range(K)]
        profs.append(dict(L=data.draw(fl), G=data.draw(fl), delta=data.draw(hs.floats(0.0, 50.0)),
                          c_copy=data.draw(fl), c_ind=data.draw(fl), F=data.draw(fl), t_eager=0.0, t_copy=0.0,
                          t_ind=0.0, ind_available=data.draw(hs.booleans()), use_measured=False, model=1,
                          d=[data.draw(fl) for _ in range(K)], g=[data.draw(fl) for _ in range(K)],
                          lam=data.draw(hs.floats(0.0, 50.0)), deps=deps))
    dec, est = cgx.select([_mk(cgx, d) for d in profs])
    assert dec == sel.select(profs)
    for d, e in zip(profs, est):
        assert e == sel.estimates(d)


def test_select_rejects_bad_dag(cgx):
    d = dict(L=1.0, G=1.0, delta=0.1, c_copy=0.0, c_ind=0.0, F=0.0, t_eager=0.0, t_copy=0.0, t_ind=0.0,
             ind_available=True, use_measured=False, model=1, d=[1.0, 1.0], g=[1.0, 1.0], lam=0.0,
             deps=[[], [0]])
    p = _mk(cgx, d)
    p.dep_idx[0] = 1                     # a dependency on itself (not an earlier node)
    with pytest.raises(cgx.CgxError):
        cgx.select([p])
    p = _mk(cgx, d)
    p.model = 2
    with pytest.raises(cgx.CgxError):
        cgx.select([p])
