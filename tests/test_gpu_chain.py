"""GPU parity of the chain path (C1, C2, C4 shapes) through the C ABI against the CPU oracle.

Bar (SURVEY §8(c) tolerances): bit-exact for copies, pointer tables, fp32 elementwise outputs
and across GPU arms; |g - o| <= 1e-5 * sum|x| for fp32 row reductions.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import capture as ocap  # noqa: E402
from oracle.chain import eval_chain  # noqa: E402
from synth import splitmix as sm  # noqa: E402
from synth import workloads as wl  # noqa: E402
from reduce_bounds import assert_output  # noqa: E402
from synth.workloads import ChainSpec, NodeSpec, SlotSpec  # noqa: E402

ARMS = [("EAGER", "DEFAULT"), ("COPY", "DEFAULT"), ("SETPARAMS", "DEFAULT"),
        ("INDIRECT", "H2D"), ("INDIRECT", "ROOT_MEMCPY"), ("INDIRECT", "ROOT_PARAMS"),
        ("INDIRECT", "ROOT_MAPPED"), ("INDIRECT", "FIRST_NODE"), ("INDIRECT", "H2D_PINGPONG")]


@pytest.fixture(scope="module")
def rt():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx, runner
    assert torch.cuda.is_available()
    return cgx, runner


def _check_reduce(got, ref, u):
    cols = 256
    bound = 1e-5 * np.abs(u.astype(np.float64)).reshape(-1, cols).sum(axis=1)
    assert np.all(np.abs(got.astype(np.float64) - ref.astype(np.float64)) <= bound)


def _compare(spec, got: dict, env: dict):
    for s in spec.internals():
        g, o = got[s.name], env[s.name]
        if s.dtype == "bf16":
            from oracle.numerics import bf16_bits
            o = bf16_bits(o)
        producer = [n for n in spec.nodes if n.out == s.name][0]
        if producer.op == "REDUCE_SUM":
            _check_reduce(g, o, env[producer.ins[0]])
        elif producer.op == "SCALE_IMM" and any(n.out == producer.ins[0] and n.op == "REDUCE_SUM"
                                                for n in spec.nodes):
            red = [n for n in spec.nodes if n.out == producer.ins[0]][0]
            bound = abs(producer.attrs["scalar"]) * 1e-5 * np.abs(
                env[red.ins[0]].astype(np.float64)).reshape(-1, 256).sum(axis=1)
            assert np.all(np.abs(g.astype(np.float64) - o.astype(np.float64)) <= bound)
        else:
            assert np.array_equal(g, o), s.name


def _run(rt, spec, mode, transport, replays, st_vals, dev, mode_vals="uniform", keep=False):
    cgx, runner = rt
    chain = runner.Chain(spec, runner.upload_statics(spec, st_vals, dev))
    ex = chain.exec(mode, transport=transport)
    outs, inputs, statss = [], [], []
    for r in range(replays):
        ext = wl.external_values(spec, r, mode_vals)
        t = runner.upload_externals(spec, ext, dev)
        inputs.append(t)            # keep every replay's buffers alive (fresh addresses)
        ex.bind(t)
        ex.launch()
        outs.append({s.name: ex.output(s.name) for s in spec.internals()})
        statss.append(ex.stats())
        if mode == "INDIRECT":
            assert ex.table() == [t[n].data_ptr() for n in chain.ext_names]   # O3 table, bit-exact
    res = (outs, statss, ex.setparam_nodes())
    chain.close()
    return res


@pytest.mark.parametrize("mode,transport", ARMS)
def test_c1_arms_bitexact(rt, mode, transport):
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()
    st = wl.static_values(spec)
    outs, stats, spn = _run(rt, spec, mode, transport, 10, st, dev)
    for r, got in enumerate(outs):
        env = eval_chain(spec, wl.external_values(spec, r), st)
        _compare(spec, got, env)
    s = stats[-1]
    if mode == "COPY":
        assert s["bytes_data_rebound"] == ocap.copy_plan_bytes(spec) == 3 * 4096 * 4
        assert s["n_copy_tensors"] == 3
    if mode == "INDIRECT":
        assert s["bytes_ptr_rebound"] == ocap.pointer_bytes(spec) == 24
        assert s["bytes_data_rebound"] == 0
    if mode == "SETPARAMS":
        assert s["n_setparam_calls"] == 4
    if mode in ("SETPARAMS", "EAGER"):
        assert spn == ocap.setparam_nodes(spec)


def test_stale_negative_control(rt):
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()
    st = wl.static_values(spec)
    outs, _, _ = _run(rt, spec, "STALE", "DEFAULT", 4, st, dev)
    env0 = eval_chain(spec, wl.external_values(spec, 0), st)
    for r, got in enumerate(outs):
        assert np.array_equal(got["out"], env0["out"])
        if r:
            assert not np.array_equal(got["out"], eval_chain(spec, wl.external_values(spec, r), st)["out"])


@pytest.mark.parametrize("mode,transport", [("EAGER", "DEFAULT"), ("COPY", "DEFAULT"),
                                            ("INDIRECT", "ROOT_PARAMS"), ("INDIRECT", "H2D"),
                                            ("INDIRECT", "FIRST_NODE"), ("SETPARAMS", "DEFAULT")])
def test_c2_parity_and_cross_arm_identity(rt, mode, transport):
    dev = torch.device("cuda:0")
    spec = wl.c2_chain()
    st = wl.static_values(spec)
    outs, stats, spn = _run(rt, spec, mode, transport, 2, st, dev)
    for r, got in enumerate(outs):
        env = eval_chain(spec, wl.external_values(spec, r), st)
        _compare(spec, got, env)
    if mode == "COPY":
        assert stats[-1]["bytes_data_rebound"] == 37_743_616
    if mode == "INDIRECT":
        assert stats[-1]["bytes_ptr_rebound"] == 512
    if mode == "SETPARAMS":
        assert stats[-1]["n_setparam_calls"] == 128 and spn == ocap.setparam_nodes(spec)
    # cross-arm identity: compare against the EAGER arm bit for bit
    ref, _, _ = _run(rt, spec, "EAGER", "DEFAULT", 2, st, dev)
    for a, b in zip(outs, ref):
        for k in a:
            assert np.array_equal(a[k], b[k]), k


def test_c2_integer_mode_exact(rt):
    dev = torch.device("cuda:0")
    spec = wl.c2_chain(n_lanes=13)
    st = wl.static_values(spec, mode="int")
    outs, _, _ = _run(rt, spec, "INDIRECT", "ROOT_PARAMS", 2, st, dev, mode_vals="int")
    for r, got in enumerate(outs):
        env = eval_chain(spec, wl.external_values(spec, r, "int"), st)
        for s in spec.internals():
            assert np.array_equal(got[s.name], env[s.name]), s.name


@pytest.mark.parametrize("size", [1024, 4096, 65536, 1 << 20, 16 << 20])
@pytest.mark.parametrize("window", [True, False])
def test_c4_points(rt, size, window):
    dev = torch.device("cuda:0")
    spec = wl.c4_chain(size, window_mode=window)
    st = wl.static_values(spec)
    for mode in ("COPY", "INDIRECT"):
        outs, stats, _ = _run(rt, spec, mode, "DEFAULT", 2, st, dev)
        for r, got in enumerate(outs):
            env = eval_chain(spec, wl.external_values(spec, r), st)
            _compare(spec, got, env)
        if mode == "COPY":
            assert stats[-1]["bytes_data_rebound"] == 3 * size


def test_c4_1gib_window_copy_and_indirect(rt):
    """BASELINE C4 at its largest point, in the launch configuration bench.py times: 3 inputs of
    1 GiB (device generator, bit-exact with synth), window kernels. COPY placeholders must equal
    the bound inputs byte for byte (compared on the device), and both arms' outputs must equal the
    oracle, which evaluates the same chain on the 4096-element window (counter-based generator:
    the window of a 1 GiB input IS the C1-sized input of the same slot and replay)."""
    cgx, runner = rt
    dev = torch.device("cuda:0")
    S = 1 << 30
    spec, ref_spec = wl.c4_chain(S, window_mode=True), wl.c1_chain()
    st = wl.static_values(spec)
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    sh = torch.cuda.current_stream().cuda_stream
    scratch = torch.empty(S // 4, dtype=torch.float32, device=dev)
    for mode in ("COPY", "INDIRECT"):
        ex = chain.exec(mode)
        for r in range(2):
            ts = {}
            for s_ in spec.externals():
                t = torch.empty(s_.nelems, dtype=torch.float32, device=dev)
                cgx.fill_uniform_f32(t.data_ptr(), s_.nelems, sm.SEED, sm.stream_id(spec.index(s_.name), r), sh)
                ts[s_.name] = t
            ex.bind(ts)
            ex.launch()
            env = eval_chain(ref_spec, wl.external_values(ref_spec, r), st)
            assert np.array_equal(ex.output("out"), env["out"]), (mode, r)
            if mode == "COPY":
                assert ex.stats()["bytes_data_rebound"] == 3 * S
                for s_ in spec.externals():
                    p, nb = cgx.output(ex.handle, chain.slot[s_.name])
                    assert nb == S
                    cgx.copy(scratch.data_ptr(), p, nb, sh)
                    assert torch.equal(scratch, ts[s_.name]), s_.name
            del ts
        ex.close()
    chain.close()


def _ragged_chain(n, cols):
    slots = [SlotSpec("x", "external", "f32", n), SlotSpec("y", "external", "f32", n + 7),
             SlotSpec("w", "static", "f32", n), SlotSpec("a", "internal", "f32", n),
             SlotSpec("b", "internal", "f32", n), SlotSpec("c", "internal", "f32", n),
             SlotSpec("r", "internal", "f32", n // cols)]
    nodes = [NodeSpec("ADD", ("x", "y"), "a", {"n": n}), NodeSpec("MUL", ("a", "w"), "b", {"n": n}),
             NodeSpec("SCALE_IMM", ("b",), "c", {"n": n, "scalar": -1.75}),
             NodeSpec("REDUCE_SUM", ("c",), "r", {"n": n, "cols": cols})]
    return ChainSpec("ragged", slots, nodes, [(0, 3)])


@pytest.mark.parametrize("n,cols", [(4, 4), (1003 * 4, 4), (5 * 1000, 1000), (3 * 4100, 4100),
                                    (2 * 257 * 4, 1028)])
def test_ragged_sizes(rt, n, cols):
    dev = torch.device("cuda:0")
    spec = _ragged_chain(n, cols)
    st = wl.static_values(spec)
    for mode, xp in (("EAGER", "DEFAULT"), ("INDIRECT", "DEFAULT"), ("INDIRECT", "FIRST_NODE"),
                     ("COPY", "DEFAULT")):
        outs, _, _ = _run(rt, spec, mode, xp, 2, st, dev)
        for r, got in enumerate(outs):
            env = eval_chain(spec, wl.external_values(spec, r), st)
            for k in ("a", "b", "c"):
                assert np.array_equal(got[k], env[k]), k
            bound = 1e-5 * np.abs(env["c"].astype(np.float64)).reshape(-1, cols).sum(axis=1)
            assert np.all(np.abs(got["r"].astype(np.float64) - env["r"]) <= bound)


def test_elementwise_tail_not_multiple_of_4(rt):
    dev = torch.device("cuda:0")
    n = 4096 + 3
    slots = [SlotSpec("x", "external", "f32", n), SlotSpec("w", "static", "f32", n),
             SlotSpec("a", "internal", "f32", n), SlotSpec("b", "internal", "f32", n)]
    nodes = [NodeSpec("ADD", ("x", "w"), "a", {"n": n}), NodeSpec("COPY", ("a",), "b", {"n": n})]
    spec = ChainSpec("tail", slots, nodes, [(0, 1)])
    st = wl.static_values(spec)
    outs, _, _ = _run(rt, spec, "INDIRECT", "DEFAULT", 2, st, dev)
    for r, got in enumerate(outs):
        env = eval_chain(spec, wl.external_values(spec, r), st)
        assert np.array_equal(got["a"], env["a"]) and np.array_equal(got["b"], env["b"])


def test_bind_errors(rt):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    ex = chain.exec("INDIRECT")
    with pytest.raises(cgx.CgxError) as e:
        ex.launch()
    assert e.value.status == cgx.E_STATE
    t = runner.upload_externals(spec, wl.external_values(spec, 0), dev)
    ptrs = [t[n].data_ptr() for n in chain.ext_names]
    with pytest.raises(cgx.CgxError) as e:
        ex.bind_ptrs(ptrs[:2])
    assert e.value.status == cgx.E_MISSING_INPUT
    with pytest.raises(cgx.CgxError) as e:
        ex.bind_ptrs([ptrs[0] + 4, ptrs[1], ptrs[2]])
    assert e.value.status == cgx.E_MISALIGNED
    host = torch.zeros(4096, dtype=torch.float32).pin_memory()
    with pytest.raises(cgx.CgxError) as e:
        ex.bind_ptrs([host.data_ptr(), ptrs[1], ptrs[2]])
    assert e.value.status == cgx.E_NOT_ELIGIBLE
    import numpy as _np
    pageable = _np.zeros(4096 + 16, _np.float32)
    addr = (pageable.ctypes.data + 15) // 16 * 16
    with pytest.raises(cgx.CgxError) as e:
        ex.bind_ptrs([addr, ptrs[1], ptrs[2]])
    assert e.value.status == cgx.E_NOT_ELIGIBLE
    ex.bind_ptrs(ptrs)
    ex.launch()
    chain.close()


def test_output_must_be_internal(rt):
    cgx, _ = rt
    c = cgx.chain_create(0)
    x = cgx.chain_add_slot(c, cgx.SLOT_EXTERNAL, cgx.F32, 64)
    y = cgx.chain_add_slot(c, cgx.SLOT_EXTERNAL, cgx.F32, 64)
    with pytest.raises(cgx.CgxError) as e:
        cgx.chain_add_node(c, cgx.OP["COPY"], [x], y)
    assert e.value.status == cgx.E_NOT_ELIGIBLE
    cgx.chain_destroy(c)


def test_output_gather_packs_outputs(rt):
    """cgx_output_gather == the individual outputs, byte for byte, at 16-B aligned offsets."""
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c2_chain()
    st = wl.static_values(spec)
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec("INDIRECT", transport="FIRST_NODE")
    t = runner.upload_externals(spec, wl.external_values(spec, 0), dev)
    ex.bind(t)
    ex.launch()
    names = [s.name for s in spec.internals()][-72:]
    slots = [chain.slot[n] for n in names]
    buf = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
    with pytest.raises(cgx.CgxError):
        cgx.output_gather(ex.handle, slots[:64], buf.data_ptr(), 16)           # too small
    with pytest.raises(cgx.CgxError):
        cgx.output_gather(ex.handle, slots + slots, buf.data_ptr(), buf.numel())  # > 64 slots
    nb = cgx.output_gather(ex.handle, slots[:64], buf.data_ptr(), buf.numel())
    torch.cuda.synchronize()
    host = buf[:nb].cpu().numpy()
    off = 0
    for n in names[:64]:
        ref = ex.output(n).view(np.uint8)
        assert np.array_equal(host[off:off + ref.size], ref), n
        off += (ref.size + 15) // 16 * 16
    assert off == nb
    chain.close()


def test_copy_placeholder_rebind_copies_nothing(rt):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    ex = chain.exec("COPY")
    phs = [cgx.output(ex.handle, chain.slot[n])[0] for n in chain.ext_names]
    ex.bind_ptrs(phs)                    # SURVEY reading 1: same address -> nothing copied
    assert ex.stats()["bytes_data_rebound"] == 0
    chain.close()


def test_device_generator_matches_synth(rt):
    cgx, _ = rt
    n = 1 << 20
    t = torch.empty(n, dtype=torch.float32, device="cuda:0")
    cgx.fill_uniform_f32(t.data_ptr(), n, sm.SEED, 12345, torch.cuda.current_stream().cuda_stream)
    assert np.array_equal(t.cpu().numpy(), sm.uniform_f32(sm.SEED, 12345, n))


def test_dispatch_floor(rt):
    cgx, _ = rt
    g, k = cgx.dispatch_floor(torch.cuda.current_stream().cuda_stream, 500)
    assert 0 < g < 100 and 0 < k < 100


def test_profile_select_matches_oracle(rt):
    cgx, runner = rt
    from oracle import selector as sel
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    t = runner.upload_externals(spec, wl.external_values(spec, 0), dev)
    ptrs = [t[n].data_ptr() for n in chain.ext_names]
    sets = []
    for r in range(4):                       # rotating fresh input sets (cgx_profile_ex)
        tr = runner.upload_externals(spec, wl.external_values(spec, r), dev)
        sets.append(tr)
    p = cgx.profile(chain.handle, -1, ptrs, 50, torch.cuda.current_stream().cuda_stream,
                    sets=[[tr[n].data_ptr() for n in chain.ext_names] for tr in sets])
    d = p.as_dict()
    assert d["n_kernels"] == 8 and d["ind_available"] == 1 and d["model"] == 1 and d["n_sets"] == 4
    assert all(x > 0 for x in d["d_us"]) and d["t_eager_us"] > 0
    # every profile field is physical (negative delta / c_ind)
    assert d["c_copy_us"] >= 0 and d["c_ind_us"] >= 0 and d["delta_us"] >= 0 and d["lambda_us"] >= 0
    assert all(x >= 0 for x in d["g_us"]) and d["span_us"] > 0
    assert d["deps"] == [[]] + [[k - 1] for k in range(1, 8)]          # C1 is a linear chain
    dec, est = cgx.select([p])
    prof = p.oracle_dict()
    assert dec == sel.select([prof])
    p.use_measured = 0
    dec2, est2 = cgx.select([p])
    prof["use_measured"] = False
    assert est2[0] == sel.estimates(prof) and dec2 == sel.select([prof])
    chain.close()


@pytest.mark.parametrize("impl", [0, 1, 2])
def test_copy_impls_placeholders_bitexact(rt, impl):
    """Every COPY implementation leaves placeholders byte-identical to the bound inputs, including
    ragged tails (n*4 bytes not a multiple of 16) and tensors spanning many chunks."""
    cgx, runner = rt
    dev = torch.device("cuda:0")
    sizes = [1, 3, 4099, 8191, 65536 + 5, (1 << 20) + 3, 3 << 20]
    slots = [SlotSpec(f"x{i}", "external", "f32", n) for i, n in enumerate(sizes)]
    slots += [SlotSpec(f"y{i}", "internal", "f32", n) for i, n in enumerate(sizes)]
    nodes = [NodeSpec("COPY", (f"x{i}",), f"y{i}", {"n": n}) for i, n in enumerate(sizes)]
    spec = ChainSpec("copies", slots, nodes, [(0, len(nodes) - 1)])
    chain = runner.Chain(spec, {})
    ex = chain.exec("COPY", copy_impl=impl)
    for r in range(3):
        vals = wl.external_values(spec, r)
        t = runner.upload_externals(spec, vals, dev)
        ex.bind(t)
        ex.launch()
        for i in range(len(sizes)):
            assert np.array_equal(ex.output(f"x{i}"), vals[f"x{i}"]), (impl, i)   # placeholder
            assert np.array_equal(ex.output(f"y{i}"), vals[f"x{i}"]), (impl, i)
        assert ex.stats()["bytes_data_rebound"] == 4 * sum(sizes)
    chain.close()


def test_kernel_times_and_graph_floor(rt):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    ex = chain.exec("INDIRECT", transport="FIRST_NODE")
    t = runner.upload_externals(spec, wl.external_values(spec, 0), dev)
    with pytest.raises(cgx.CgxError):
        cgx.kernel_times(ex.handle, 5)          # not bound yet
    ex.bind(t)
    ex.launch()
    d = cgx.kernel_times(ex.handle, 5)
    assert len(d) == 8 and all(0 < x < 1000 for x in d)
    sh = torch.cuda.current_stream().cuda_stream
    f1, f200 = cgx.graph_floor(sh, 1, True, 50), cgx.graph_floor(sh, 200, True, 20)
    assert 0 < f1 < f200 < 10000
    chain.close()


@pytest.mark.parametrize("transport", ["FIRST_NODE", "ROOT_PARAMS", "H2D", "ROOT_MAPPED", "H2D_PINGPONG",
                                       "ROOT_MEMCPY"])
def test_indirect_stress_rotating_inputs(rt, transport):
    """Back-to-back replays (no host sync in between) rotating 3 resident input sets: every
    replay must read ITS table (a stale or half-published table would mix sets)."""
    cgx, runner = rt
    dev = torch.device("cuda:0")
    for spec, reps in ((wl.c1_chain(), 300), (wl.c2_chain(n_lanes=26), 60)):
        st = wl.static_values(spec)
        chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
        ex = chain.exec("INDIRECT", transport=transport)
        sets = [runner.upload_externals(spec, wl.external_values(spec, r), dev) for r in range(3)]
        finals = [s.name for s in spec.internals() if not any(s.name in n.ins for n in spec.nodes)]
        ref = [eval_chain(spec, wl.external_values(spec, r), st) for r in range(3)]
        snap = {}
        for i in range(reps):
            ex.bind(sets[i % 3])
            ex.launch()
            if i % 7 == 0 or i >= reps - 3:                 # copy finals out without syncing the host
                for nm in finals:
                    p, nb = cgx.output(ex.handle, chain.slot[nm])
                    buf = torch.empty(nb, dtype=torch.uint8, device=dev)
                    cgx.copy(buf.data_ptr(), p, nb, torch.cuda.current_stream().cuda_stream)
                    snap.setdefault(i, {})[nm] = buf
        torch.cuda.synchronize()
        for i, d in snap.items():
            for nm, buf in d.items():
                got = buf.cpu().numpy().view(np.float32)
                assert_output(spec, ref[i % 3], nm, got, (transport, i))
        chain.close()


def test_scalar_staleness_and_cgct_rewrite(rt):
    """NEXT-3 (S:L554 criterion 1): a by-value scalar captured in a
    graph goes stale when the application changes it; rewritten as a 1-element device tensor
    slot (SCALE_T) bound per replay, the graph tracks the new value bit-exactly."""
    cgx, runner = rt
    dev = torch.device("cuda:0")
    n = 4096
    temps = [8.0, 0.125, 3.0, -2.5]
    # naive: the scalar is a by-value node attribute, frozen at capture
    naive = ChainSpec("naive", [SlotSpec("q", "external", "f32", n), SlotSpec("o", "internal", "f32", n)],
                      [NodeSpec("SCALE_IMM", ("q",), "o", {"n": n, "scalar": temps[0]})], [(0, 0)])
    chain = runner.Chain(naive, {})
    ex = chain.exec("INDIRECT")
    stale = False
    for r, tmp in enumerate(temps):
        vals = wl.external_values(naive, r)
        t = runner.upload_externals(naive, vals, dev)
        ex.bind(t)
        ex.launch()
        eager_ref = vals["q"] * np.float32(tmp)            # what the program means at replay r
        stale |= not np.array_equal(ex.output("o"), eager_ref)
    assert stale                                            # witness: replays used the old scalar
    chain.close()
    # CGCT rewrite: the scalar becomes an EXTERNAL 1-element slot, rebound like any input
    fixed = ChainSpec("cgct", [SlotSpec("q", "external", "f32", n), SlotSpec("s", "external", "f32", 1),
                               SlotSpec("o", "internal", "f32", n)],
                      [NodeSpec("SCALE_T", ("q", "s"), "o", {"n": n})], [(0, 0)])
    for mode, xp in (("INDIRECT", "FIRST_NODE"), ("INDIRECT", "ROOT_PARAMS"), ("COPY", "DEFAULT"),
                     ("SETPARAMS", "DEFAULT"), ("EAGER", "DEFAULT")):
        chain = runner.Chain(fixed, {})
        ex = chain.exec(mode, transport=xp)
        keep = []
        for r, tmp in enumerate(temps * 3):
            vals = wl.external_values(fixed, r)
            vals["s"] = np.array([tmp], np.float32)
            t = runner.upload_externals(fixed, vals, dev)
            keep.append(t)
            ex.bind(t)
            ex.launch()
            assert np.array_equal(ex.output("o"), eval_chain(fixed, vals, {})["o"]), (mode, r)
        chain.close()


def test_param_offset_discovery_on_live_node_images(rt):
    """NEXT-2: pattern-match each bound input pointer in the parameter image of every
    node that reads it; the offset found is the field the runtime patches (and the kernel reads, as
    the parity tests prove), and cudaFuncGetParamInfo's size matches the image."""
    cgx, runner = rt
    from oracle import offsets as ooff
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    ex = chain.exec("SETPARAMS")
    t = runner.upload_externals(spec, wl.external_values(spec, 0), dev)
    ex.bind(t)
    ptr = {n: t[n].data_ptr() for n in chain.ext_names}
    for pos, node in enumerate(spec.nodes):
        img, p0 = cgx.param_image(ex.handle, pos)
        assert p0 == len(img)
        want = sorted(cgx.ext_field_offsets(ex.handle, pos))
        found = []
        for nm in dict.fromkeys(i for i in node.ins if i in ptr):
            found.append(cgx.find_param_offset(img, ptr[nm]))
            assert found[-1] == ooff.find_param_offset(img, ptr[nm])
        assert sorted(found) == want, (pos, found, want)
    chain.close()
