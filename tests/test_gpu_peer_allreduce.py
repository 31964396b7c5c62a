"""Peer-memory one-shot all-reduce (cgx_chain_set_peers, k_allreduce_peer).

This box has one GPU, so the ranks are emulated inside one process on one device: each rank is its
own chain (its TP shard of the decoder) with its own region, every rank's region is passed to every
chain as its "peer" pointer, and the ranks' graphs are launched on separate streams so their
all-reduce kernels run concurrently and meet through the flags exactly as they would over NVLink
(the kernel code path — remote stores, sys-scope release/acquire flags, fixed-order sums — is the
same; only the link differs). Results must be bit-identical across ranks and match the lockstep
TP oracle (integer mode: exact; uniform values: the decoder tolerance)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.chain import eval_chain, eval_chain_tp  # noqa: E402
from oracle.numerics import bf16_bits, bits_to_f64  # noqa: E402
from synth import workloads as wl  # noqa: E402
from synth.workloads import ChainSpec, NodeSpec, SlotSpec  # noqa: E402
from tp_check import check_tp_node_local  # noqa: E402


@pytest.fixture(scope="module")
def rt():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx, runner
    return cgx, runner


def _regions(cgx, world, max_elems, dev):
    nb = cgx.peer_buffer_bytes(world, max_elems)
    return [torch.zeros(nb + 256, dtype=torch.uint8, device=dev) for _ in range(world)]


def _base(t):
    return (t.data_ptr() + 255) // 256 * 256


def _ar_spec(n):
    slots = [SlotSpec("x", "external", "bf16", n), SlotSpec("a", "internal", "bf16", n),
             SlotSpec("s", "internal", "bf16", n), SlotSpec("y", "internal", "bf16", n),
             SlotSpec("s2", "internal", "bf16", n)]
    nodes = [NodeSpec("COPY", ("x",), "a", {"n": n}), NodeSpec("ALLREDUCE_SUM", ("a",), "s", {"n": n}),
             NodeSpec("ADD", ("s", "a"), "y", {"n": n}), NodeSpec("ALLREDUCE_SUM", ("y",), "s2", {"n": n})]
    return ChainSpec("ar", slots, nodes, [(0, 3)])


def _run_ranks(rt, specs, statics, exts_per_replay, world, max_elems, mode="INDIRECT", transport="DEFAULT"):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    regs = _regions(cgx, world, max_elems, dev)
    bases = [_base(t) for t in regs]
    chains = [runner.Chain(specs[r], runner.upload_statics(specs[r], statics[r], dev),
                           peers=(r, world, bases, max_elems)) for r in range(world)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(world)]
    exs = [chains[r].exec(mode, stream=streams[r], transport=transport) for r in range(world)]
    outs, keep = [], []
    for ext in exts_per_replay:
        ts = [runner.upload_externals(specs[r], ext[r], dev) for r in range(world)]
        keep.append(ts)
        torch.cuda.synchronize()
        for r in range(world):
            exs[r].bind(ts[r])
        for r in range(world):                      # all ranks' replays in flight together
            exs[r].launch()
        torch.cuda.synchronize()
        outs.append([{s.name: exs[r].output(s.name) for s in specs[r].internals()} for r in range(world)])
    for ch in chains:
        ch.close()
    return outs


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("n", [8, 4096, 98304])
def test_allreduce_integer_exact(rt, world, n):
    spec = _ar_spec(n)
    specs = [spec] * world
    exts = [[{"x": wl.slot_values(spec, "x", 10 * rep + r, "int")} for r in range(world)] for rep in range(5)]
    outs = _run_ranks(rt, specs, [{}] * world, exts, world, max(n, 4096))
    for rep in range(5):
        parts = [bits_to_f64(exts[rep][r]["x"]) for r in range(world)]
        s = sum(parts)
        y = [s + p for p in parts]
        s2 = sum(y)
        for r in range(world):
            assert np.array_equal(outs[rep][r]["s"], bf16_bits(s)), (rep, r)
            assert np.array_equal(outs[rep][r]["s2"], bf16_bits(s2)), (rep, r)


@pytest.mark.parametrize("tp", [2, 4])
@pytest.mark.parametrize("mode,transport", [("INDIRECT", "FIRST_NODE"), ("COPY", "DEFAULT"), ("EAGER", "DEFAULT")])
def test_tp_decoder_peer_allreduce(rt, monkeypatch, tp, mode, transport):
    """C5 (TP decoder, 2 layers, T=128) with the peer all-reduce: every rank's output identical, and
    equal to the lockstep TP oracle within the decoder tolerance."""
    # The virtual ranks share ONE GPU: a rank's all-reduce spins until every rank's partial has
    # arrived, so every rank's GEMMs must still find room beside the spinning CTAs. Split-K GEMMs
    # launch as thread-block clusters, which need several free SMs of one GPC at once; with the
    # S = 3 shard tilings EAGER at TP = 4 could not place a rank's cluster and tripped the bounded
    # spin on every run. Unsplit BN = 32 tilings (no clusters) keep the emulation schedulable; on
    # an NVSwitch box each rank has its own GPU (test_multigpu_tp_chain runs the default tilings).
    hl, fl = 12 // tp, 3072 // tp
    shapes = {(3 * hl * 64, 768), (768, hl * 64), (fl, 768), (768, fl)}
    monkeypatch.setenv("CGX_GEMM_TILING", ",".join(f"{n}x{k}=32/1" for n, k in shapes))
    full = wl.c3_chain(T=128, n_layers=2)
    specs = [wl.c3_chain(T=128, n_layers=2, tp=tp, rank=r) for r in range(tp)]
    statics = [wl.static_values(specs[r], tp=tp, rank=r, full=full) for r in range(tp)]
    exts = [[wl.external_values(specs[r], rep) for r in range(tp)] for rep in range(3)]
    outs = _run_ranks(rt, specs, statics, exts, tp, 128 * 768, mode, transport)
    last = specs[0].nodes[-1].out
    for rep in range(3):
        for r in range(1, tp):
            assert np.array_equal(outs[rep][r][last], outs[rep][0][last]), (rep, r)
        # every node of every rank, element-wise, from the GPU's own node inputs (shard GEMMs included)
        assert check_tp_node_local(specs, statics, exts[rep], outs[rep], f"tp{tp} {mode} rep {rep}") == \
            tp * len(specs[0].nodes)
        ref = eval_chain_tp(specs, exts[rep], statics)[0][last]
        g = bits_to_f64(outs[rep][0][last])
        assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 2e-2
        tp1 = eval_chain(full, wl.external_values(full, rep), wl.static_values(full))[last]
        assert np.linalg.norm(g - tp1) / np.linalg.norm(tp1) <= 2e-2


def test_set_peers_errors(rt):
    cgx, runner = rt
    spec = _ar_spec(4096)
    ch = runner.Chain(spec, {}, 0)
    with pytest.raises(cgx.CgxError):
        cgx.chain_set_peers(ch.handle, 2, 2, [256, 512], 4096)          # rank out of range
    with pytest.raises(cgx.CgxError):
        cgx.chain_set_peers(ch.handle, 0, 2, [256 + 16, 512], 4096)     # misaligned region
    ch.close()


def _torchrun_tp(tp, allreduce, layers, tmp_path, one_gpu):
    """Run scripts/bench_tp.py under torchrun with `tp` ranks (each on its own GPU, or all on GPU 0
    when one_gpu), dump every rank's internals and check them node-local against the oracle."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    if one_gpu:
        env["CGX_TP_DEVICE"] = "0"
    dump = str(tmp_path / f"tp{tp}_{allreduce}")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(tp),
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(root, "scripts", "bench_tp.py"), "--allreduce", allreduce, "--layers",
                        str(layers), "--steps", "5", "--check", "--dump", dump],
                       env=env, capture_output=True, text=True, timeout=400)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and line, r.stdout[-2000:] + r.stderr[-2000:]
    res = json.loads(line[-1])["us_per_replay_max_over_ranks"]
    assert res["ranks_identical"]
    assert max(res["check_rel_err_per_rank"]) <= 2e-2
    full = wl.c3_chain(T=128, n_layers=layers)
    specs = [wl.c3_chain(T=128, n_layers=layers, tp=tp, rank=k, fuse_allreduce=allreduce == "fused")
             for k in range(tp)]
    statics = [wl.static_values(wl.c3_chain(T=128, n_layers=layers, tp=tp, rank=k), tp=tp, rank=k, full=full)
               for k in range(tp)]
    exts = [wl.external_values(specs[k], 0) for k in range(tp)]
    gots = []
    for k in range(tp):
        z = np.load(os.path.join(dump, f"rank{k}.npz"))
        gots.append({nm: z[nm] for nm in z.files})
    assert check_tp_node_local(specs, statics, exts, gots, f"torchrun tp{tp} {allreduce}") == tp * len(specs[0].nodes)
    return res


@pytest.mark.parametrize("allreduce", ["peer", "fused"])
def test_multiprocess_ipc_peer_allreduce(rt, allreduce, tmp_path):
    """Two processes (torchrun) on this one GPU: regions exchanged as CUDA IPC handles through a
    gloo process group (tp.PeerRegions, dedicated allocations), TP=2 decoder layer with the peer
    all-reduce. The ranks time-share the device, so only the results are checked: every node of
    every rank element-wise against the oracle fed that rank's GPU inputs, ranks identical."""
    _torchrun_tp(2, allreduce, 1, tmp_path, one_gpu=True)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (NCCL ranks on separate devices)")
@pytest.mark.parametrize("tp", [2, 4, 8])
@pytest.mark.parametrize("allreduce", ["nccl", "peer", "fused"])
def test_multigpu_tp_chain(rt, tp, allreduce, tmp_path):
    """C5 on real ranks: TP = 2/4/8 decoder (2 layers, T = 128), one
    process per GPU, ALLREDUCE_SUM as a captured ncclAllReduce over NVLink (or the peer / fused
    peer all-reduce over IPC-mapped regions); node-local element-wise parity on every rank."""
    if torch.cuda.device_count() < tp:
        pytest.skip(f"needs {tp} GPUs")
    _torchrun_tp(tp, allreduce, 2, tmp_path, one_gpu=False)


@pytest.mark.parametrize("tp", [2, 4])
@pytest.mark.parametrize("mode,transport", [("INDIRECT", "FIRST_NODE"), ("SETPARAMS", "DEFAULT"), ("EAGER", "DEFAULT")])
def test_tp_decoder_gemm_fused_allreduce(rt, monkeypatch, tp, mode, transport):
    """The row-parallel GEMMs (O-proj, FC2) with the all-reduce fused into their epilogue
    (CGX_GEMM_ALLREDUCE: one kernel computes the partial tile, pushes it to every rank and sums):
    bit-identical to the chain with separate peer ALLREDUCE_SUM nodes, identical across ranks,
    and within the decoder tolerance of the TP oracle. Small row-parallel tilings keep every
    virtual rank's all-reducing GEMM resident on the one shared GPU."""
    # every GEMM of every virtual rank on an unsplit BN = 32 tiling (<= 48 CTAs each): the ranks share
    # ONE GPU here, and an all-reducing GEMM spins until every rank's GEMM for the same tile has
    # arrived, so all of them must be able to be resident at once (on an NVSwitch box each rank has
    # its own GPU). Larger footprints can starve a rank and trip the bounded spin.
    hl, fl = 12 // tp, 3072 // tp
    shapes = {(3 * hl * 64, 768), (768, hl * 64), (fl, 768), (768, fl)}
    monkeypatch.setenv("CGX_GEMM_TILING", ",".join(f"{n}x{k}=32/1" for n, k in shapes))
    full = wl.c3_chain(T=128, n_layers=2)
    specs_f = [wl.c3_chain(T=128, n_layers=2, tp=tp, rank=r, fuse_allreduce=True) for r in range(tp)]
    specs_u = [wl.c3_chain(T=128, n_layers=2, tp=tp, rank=r) for r in range(tp)]
    assert len(specs_f[0].nodes) + 4 == len(specs_u[0].nodes)
    statics = [wl.static_values(specs_u[r], tp=tp, rank=r, full=full) for r in range(tp)]
    exts = [[wl.external_values(specs_u[r], rep) for r in range(tp)] for rep in range(3)]
    outs_f = _run_ranks(rt, specs_f, statics, exts, tp, 128 * 768, mode, transport)
    outs_u = _run_ranks(rt, specs_u, statics, exts, tp, 128 * 768, mode, transport)
    last = specs_f[0].nodes[-1].out
    for rep in range(3):
        for r in range(tp):
            assert np.array_equal(outs_f[rep][r][last], outs_u[rep][r][last]), (rep, r)
            assert np.array_equal(outs_f[rep][r][last], outs_f[rep][0][last]), (rep, r)
        check_tp_node_local(specs_f, statics, exts[rep], outs_f[rep], f"tp{tp} fused {mode} rep {rep}")
        ref = eval_chain_tp(specs_f, exts[rep], statics)[0][last]
        g = bits_to_f64(outs_f[rep][0][last])
        assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 2e-2


def test_lost_peer_reports_device_error(rt, monkeypatch):
    """A rank whose peer never arrives must not hang or trap the context: the
    spinning all-reduce gives up after the spin bound (CGX_SPIN_TIMEOUT_MS), stores kDevErrPeer in
    the exec's status word, and the exec's next cgx_launch returns CGX_E_DEVICE (sticky); the CUDA
    context stays usable for other work."""
    cgx, runner = rt
    monkeypatch.setenv("CGX_SPIN_TIMEOUT_MS", "300")
    n = 4096
    dev = torch.device("cuda:0")
    regs = _regions(cgx, 2, n, dev)
    spec = _ar_spec(n)
    chain = runner.Chain(spec, {}, peers=(0, 2, [_base(t) for t in regs], n))   # rank 1 never runs
    ex = chain.exec("INDIRECT")
    x = runner.upload_externals(spec, wl.external_values(spec, 0), dev)
    ex.bind(x)
    ex.launch()                                  # returns at once; the kernel gives up after ~0.3 s
    torch.cuda.synchronize()
    assert ex.stats()["device_error"] == 2
    ex.bind(x)
    with pytest.raises(cgx.CgxError) as ei:
        ex.launch()
    assert ei.value.status == cgx.E_DEVICE and "lost peer" in str(ei.value)
    with pytest.raises(cgx.CgxError):
        ex.launch()                              # sticky
    chain.close()
    y = torch.ones(16, device=dev) * 2           # the context is still healthy
    assert float(y.sum().item()) == 32.0
