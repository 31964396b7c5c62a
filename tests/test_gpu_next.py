"""GPU coverage of the NEXT rows:
  NEXT-1  prelude-kernel PI for opaque consumers (device-updatable nodes + cudaGraphKernelNodeSetParam)
  NEXT-2  parameter-offset discovery (see also test_gpu_chain.py::test_param_offset_discovery_...)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.chain import eval_chain  # noqa: E402
from synth import workloads as wl  # noqa: E402
from reduce_bounds import assert_output  # noqa: E402


@pytest.fixture(scope="module")
def rt():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx, runner
    return cgx, runner


def _finals(spec):
    return [s.name for s in spec.internals() if not any(s.name in n.ins for n in spec.nodes)]


@pytest.mark.parametrize("which", ["C1", "C2_26"])
def test_prelude_indirection_parity(rt, which):
    """the prelude dereferences the pointer cells and patches every opaque
    consumer's parameter buffer; outputs equal eager on fresh inputs every replay."""
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c1_chain() if which == "C1" else wl.c2_chain(n_lanes=26)
    st = wl.static_values(spec)
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec("INDIRECT", transport="PRELUDE")
    keep = []
    for r in range(6):
        vals = wl.external_values(spec, r)
        t = runner.upload_externals(spec, vals, dev)
        keep.append(t)
        ex.bind(t)
        ex.launch()
        env = eval_chain(spec, vals, st)
        for nm in _finals(spec):
            assert_output(spec, env, nm, ex.output(nm), r)
        assert ex.table() == [t[n].data_ptr() for n in chain.ext_names]
    s = ex.stats()
    assert s["bytes_ptr_rebound"] == 8 * len(chain.ext_names) and s["bytes_data_rebound"] == 0
    chain.close()


def test_prelude_rotating_inputs_back_to_back(rt):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()
    st = wl.static_values(spec)
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec("INDIRECT", transport="PRELUDE")
    sets = [runner.upload_externals(spec, wl.external_values(spec, r), dev) for r in range(3)]
    refs = [eval_chain(spec, wl.external_values(spec, r), st)["out"] for r in range(3)]
    snaps = []
    sh = torch.cuda.current_stream().cuda_stream
    for i in range(200):
        ex.bind(sets[i % 3])
        ex.launch()
        if i % 9 == 0:
            p, nb = cgx.output(ex.handle, chain.slot["out"])
            buf = torch.empty(nb, dtype=torch.uint8, device=dev)
            cgx.copy(buf.data_ptr(), p, nb, sh)
            snaps.append((i, buf))
    torch.cuda.synchronize()
    for i, buf in snaps:
        assert np.array_equal(buf.cpu().numpy().view(np.float32), refs[i % 3]), i
    chain.close()
