"""NVLS (NVSwitch multicast) all-reduce: ALLREDUCE_SUM nodes through
k_allreduce_mc (each rank stores its partial into its own copy of a region bound to a multicast
object, arrives with multimem.red, reads the sum with multimem.ld_reduce).

Where multicast objects can be created (an NVSwitch box whose fabric the process can reach), the
world-1 tests run the real path on one device — the multicast object, its binding and two mappings
(driver VMM API), the multimem instructions through the switch, the generation / parity protocol
over many replays — where the reduction is over one rank (the identity); the world > 1 path runs in
test_multigpu_multicast_tp (torchrun, one process per GPU, the object's file descriptor passed over
a Unix socket). This pool's containers refuse cuMulticastCreate, so all of them skip here."""
import numpy as np
import pytest
import torch

from oracle.numerics import bf16_bits, bits_to_f64
from synth import workloads as wl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rt():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx, runner
    if not cgx.mc_supported(0):
        pytest.skip("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0 on this device")
    from paper_2503_19779_b200 import tp as _tp
    try:   # the attribute alone is not enough: the NVSwitch fabric must be reachable from here
        _tp.MulticastRegion(1, 0, 4096, torch.device("cuda:0")).close()
    except cgx.CgxError as exn:
        pytest.skip(f"multicast objects unavailable in this environment ({exn}); on this pool's containers "
                    "cuMulticastCreate returns CUDA_ERROR_INVALID_VALUE for every handle type and device "
                    "count although CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 1 (profiles/r02/multicast_probe.txt)")
    return cgx, runner


def test_mc_region_layout(rt):
    """The region holds the per-node parity slots and the arrival counters; mc_create rounds the
    size up to the multicast granularity; bind/map yields two distinct 256-B aligned addresses."""
    cgx, runner = rt
    from paper_2503_19779_b200 import tp
    nb = cgx.mc_buffer_bytes(4096, 4)
    assert nb >= 4 * 2 * 4096 * 2 + 4 * 256 * 4
    r = tp.MulticastRegion(1, 0, 4096, torch.device("cuda:0"), max_allreduces=4)
    try:
        assert r.size >= nb and r.uc % 256 == 0 and r.mc % 256 == 0 and r.uc != r.mc
    finally:
        r.close()


@pytest.mark.parametrize("n", [8, 4096, 98304])
@pytest.mark.parametrize("mode", ["INDIRECT", "EAGER", "SETPARAMS"])
def test_mc_allreduce_world1_bit_exact(rt, n, mode):
    """Two chained all-reduces (s = AR(x); s2 = AR(s + x)) over 6 replays with fresh inputs: every
    output equals the one-rank sum bit for bit (the switch's fp32 accumulation of one bf16 value,
    one rounding) — exercising the generation counters and both parity slots."""
    cgx, runner = rt
    from paper_2503_19779_b200 import tp
    from test_gpu_peer_allreduce import _ar_spec
    spec = _ar_spec(n)
    dev = torch.device("cuda:0")
    r = tp.MulticastRegion(1, 0, max(n, 4096), dev)
    try:
        chain = runner.Chain(spec, {}, 0, multicast=r.multicast())
        ex = chain.exec(mode)
        for rep in range(6):
            x = wl.slot_values(spec, "x", rep, "int")
            t = runner.upload_externals(spec, {"x": x}, dev)
            ex.bind(t)
            ex.launch()
            xv = bits_to_f64(x)
            assert np.array_equal(ex.output("s"), bf16_bits(xv)), rep
            assert np.array_equal(ex.output("s2"), bf16_bits(xv + xv)), rep
        chain.close()
    finally:
        r.close()


@pytest.mark.parametrize("tp_", [2, 4])
def test_mc_tp_shard_world1_matches_nccl(rt, tp_):
    """Rank 0's TP shard of the decoder (T = 128, 2 layers) with its all-reduces through a one-device
    multicast object: bit-identical to the same shard with a one-rank NCCL communicator (both the
    identity), node-local parity against the oracle, INDIRECT and EAGER bit-identical."""
    cgx, runner = rt
    from paper_2503_19779_b200 import cgx as c
    from paper_2503_19779_b200 import tp
    from test_gpu_decoder import _node_local_check
    full = wl.c3_chain(T=128, n_layers=2)
    spec = wl.c3_chain(T=128, n_layers=2, tp=tp_, rank=0)
    st = wl.static_values(spec, tp=tp_, rank=0, full=full)
    dev = torch.device("cuda:0")
    comm = c.nccl_comm_init(1, 0, c.nccl_unique_id(), 0)
    r = tp.MulticastRegion(1, 0, 128 * 768, dev)
    try:
        outs = {}
        for kind in ("mc", "nccl"):
            for mode in ("INDIRECT", "EAGER"):
                chain = (runner.Chain(spec, runner.upload_statics(spec, st, dev), multicast=r.multicast())
                         if kind == "mc" else
                         runner.Chain(spec, runner.upload_statics(spec, st, dev), nccl_comm=comm))
                ex = chain.exec(mode)
                got = []
                for rep in range(2):
                    t = runner.upload_externals(spec, wl.external_values(spec, rep), dev)
                    ex.bind(t)
                    ex.launch()
                    got.append({s_.name: ex.output(s_.name) for s_ in spec.internals()})
                chain.close()
                outs[(kind, mode)] = got
        for rep in range(2):
            _node_local_check(spec, st, wl.external_values(spec, rep), outs[("mc", "INDIRECT")][rep], one_rank=True)
            for k in outs[("mc", "INDIRECT")][rep]:
                ref = outs[("nccl", "INDIRECT")][rep][k]
                assert np.array_equal(outs[("mc", "INDIRECT")][rep][k], ref), k
                assert np.array_equal(outs[("mc", "EAGER")][rep][k], ref), k
    finally:
        r.close()
        c.nccl_comm_destroy(comm)


@pytest.mark.parametrize("tp_", [2, 4, 8])
def test_multigpu_multicast_tp(rt, tp_, tmp_path):
    """C5 at TP = 2 / 4 / 8 with the NVLS all-reduce, one torchrun process per GPU: node-local
    element-wise parity of every node of every rank (tests/tp_check.py), ranks identical."""
    if torch.cuda.device_count() < tp_:
        pytest.skip(f"needs {tp_} GPUs")
    from test_gpu_peer_allreduce import _torchrun_tp
    _torchrun_tp(tp_, "mc", 2, tmp_path, one_gpu=False)
