"""Selective CUDA graphs per segment ("independently for each of the CGs"; SURVEY §8(a)
a10): a chain split into segments, each profiled and decided on its own, then executed with a
DIFFERENT mode per segment (the deployed module of P:L639) — outputs must equal eager."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import selector as osel  # noqa: E402
from oracle.chain import eval_chain  # noqa: E402
from synth import workloads as wl  # noqa: E402
from reduce_bounds import assert_output  # noqa: E402


@pytest.fixture(scope="module")
def rt():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx, runner
    return cgx, runner


def _spec():
    spec = wl.c2_chain(n_lanes=16, scale_tail=4)
    K = len(spec.nodes)
    spec.segments = [(0, 23), (24, 47), (48, K - 1)]
    return spec


def test_profile_and_select_per_segment(rt):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = _spec()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    t = runner.upload_externals(spec, wl.external_values(spec, 0), dev)
    ptrs = [t[n].data_ptr() for n in chain.ext_names]
    sh = torch.cuda.current_stream().cuda_stream
    profs = [cgx.profile(chain.handle, s, ptrs, 20, sh) for s in range(len(spec.segments))]
    dec, est = cgx.select(profs)
    py = []
    for p in profs:
        d = p.as_dict()
        assert d["n_kernels"] == spec.segments[profs.index(p)][1] - spec.segments[profs.index(p)][0] + 1
        py.append(p.oracle_dict())
        assert d["c_copy_us"] >= 0 and d["c_ind_us"] >= 0 and d["delta_us"] >= 0 and d["lambda_us"] >= 0
    assert dec == osel.select(py)                      # bit-exact decisions per segment
    for p in profs:                                    # the estimate path too (model 1), bit for bit
        p.use_measured = 0
    dec_e, est_e = cgx.select(profs)
    for p, e in zip(profs, est_e):
        assert e == osel.estimates(p.oracle_dict())
    chain.close()


@pytest.mark.parametrize("modes", [("EAGER", "INDIRECT", "COPY"), ("INDIRECT", "EAGER", "SETPARAMS"),
                                   ("COPY", "COPY", "INDIRECT")])
def test_mixed_modes_per_segment_equal_eager(rt, modes):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = _spec()
    st = wl.static_values(spec)
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    execs = [chain.exec(m, first_node=f, n_nodes=l - f + 1) for m, (f, l) in zip(modes, spec.segments)]
    finals = [s.name for s in spec.internals() if not any(s.name in n.ins for n in spec.nodes)]
    keep = []
    for r in range(3):
        vals = wl.external_values(spec, r)
        tt = runner.upload_externals(spec, vals, dev)
        keep.append(tt)
        for ex in execs:                               # the deployed program: segment by segment
            ex.bind(tt)
            ex.launch()
        env = eval_chain(spec, vals, st)
        for nm in finals:
            assert_output(spec, env, nm, execs[-1].output(nm), (modes, r))
        # elementwise intermediates are exact
        for l in range(16):
            assert np.array_equal(execs[-1].output(f"t{l}"), env[f"t{l}"])
    chain.close()
