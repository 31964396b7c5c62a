"""The C-ABI library builds, loads and exports every symbol include/cgx.h declares (no GPU, no
compute calls). Also checks the product path never imports the oracle and vice versa."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx
    return cgx


def declared():
    src = open(os.path.join(ROOT, "include", "cgx.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(cgx_\w+)\(", src, re.M)))


def test_header_symbols_exported(lib):
    names = declared()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cgx_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(lib.EXPORTED) == set(names)


def test_version_and_pure_select_on_cpu(lib):
    assert lib.version() == 1
    # cgx_select is a pure host function: callable without a GPU
    p = lib.Profile()
    p.n_kernels, p.ind_available, p.use_measured = 2, 1, 0
    p.L_us, p.G_us, p.delta_us, p.c_copy_us, p.c_ind_us = 10.0, 7.5, 0.5, 3.0, 1.0
    p.d_us[0], p.d_us[1] = 2.0, 2.0
    dec, est = lib.select([p])
    from oracle import selector as sel
    pe = dict(L=10.0, G=7.5, delta=0.5, d=[2.0, 2.0], c_copy=3.0, c_ind=1.0)
    assert est[0] == sel.estimates(pe)
    assert dec[0] == sel.select([pe])[0]


def test_no_cpu_device_without_gpu(lib):
    import ctypes as C
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    out = C.c_void_p()
    st = lib.LIB.cgx_chain_create(0, C.byref(out))
    assert st != 0    # no CUDA device here: fails loudly instead of falling back


def test_product_and_oracle_are_independent():
    for d, forbidden in (("paper_2503_19779_b200", "oracle"), ("oracle", "paper_2503_19779_b200")):
        for dirpath, _, files in os.walk(os.path.join(ROOT, d)):
            for f in files:
                if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                    txt = open(os.path.join(dirpath, f)).read()
                    assert not re.search(rf"^\s*(from|import)\s+{forbidden}\b", txt, re.M), (f, forbidden)


def test_peer_buffer_bytes_host_only():
    """cgx_peer_buffer_bytes is pure host arithmetic: receive data [max_ar][2][world][slot] bf16
    (slots rounded up to 128 elements: every all-reduce node owns two parity buffers) followed by
    the flag array [max_ar][8][256] uint32."""
    from paper_2503_19779_b200 import cgx
    for world, n, nar in ((1, 8, 1), (2, 98304, 24), (8, 1000, 64)):
        slot = (n + 127) // 128 * 128
        assert cgx.peer_buffer_bytes(world, n, nar) == nar * 2 * world * slot * 2 + 4 * nar * 8 * 256
    assert cgx.peer_buffer_bytes(2, 8) == cgx.peer_buffer_bytes(2, 8, 64)
    for bad in (0, 9):
        with pytest.raises(cgx.CgxError):
            cgx.peer_buffer_bytes(bad, 1024)
    for bad_ar in (0, 65):
        with pytest.raises(cgx.CgxError):
            cgx.peer_buffer_bytes(2, 1024, bad_ar)


def test_bench_reference_arm_contract_on_cpu():
    """bench.py --impl reference (the oracle timed on host cores) prints the contract's JSON line."""
    import json
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "3"], capture_output=True, text=True, timeout=240, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["unit"] == "iters/s" and d["higher_is_better"] is True


def test_tune_graph_streams_argument_checks_on_cpu(lib):
    """cgx_tune_graph_streams rejects bad arguments before touching the device (include/cgx.h)."""
    import ctypes as C
    c = lib
    opts = c.ExecOpts(c.MODE["INDIRECT"], c.XPORT["ROOT_PARAMS"], 0, 0, 0, 0, 0, c.SYNC["GRAPH"], 0)
    cand = (C.c_int * 1)(16)
    best = C.c_int()
    sets = c.ptr_array([0])
    # NULL chain, no candidates, zero reps: all CGX_E_INVALID_ARG with a message
    assert c.LIB.cgx_tune_graph_streams(None, C.byref(opts), None, sets, 1, 1, cand, 1, 10, C.byref(best),
                                        None) == c.E_INVALID_ARG
    assert "tune_graph_streams" in c.last_error()
    fake_chain = C.c_void_p(0x1000)   # never dereferenced: the checks below fail first
    assert c.LIB.cgx_tune_graph_streams(fake_chain, C.byref(opts), None, sets, 1, 1, cand, 0, 10, C.byref(best),
                                        None) == c.E_INVALID_ARG
    assert c.LIB.cgx_tune_graph_streams(fake_chain, C.byref(opts), None, sets, 1, 1, cand, 1, 0, C.byref(best),
                                        None) == c.E_INVALID_ARG
    eager = c.ExecOpts(c.MODE["EAGER"], 0, 0, 0, 0, 0, 0, 0, 0)
    assert c.LIB.cgx_tune_graph_streams(fake_chain, C.byref(eager), None, sets, 1, 1, cand, 1, 10, C.byref(best),
                                        None) == c.E_INVALID_ARG


def test_tune_graph_streams_rejects_out_of_range_candidates_on_cpu(lib):
    """Every candidate stream count is validated (1..64) before any candidate is built or timed
    (0 used to build the default 16 streams and could be returned as the best)."""
    import ctypes as C
    c = lib
    opts = c.ExecOpts(c.MODE["INDIRECT"], c.XPORT["ROOT_PARAMS"], 0, 0, 0, 0, 0, c.SYNC["GRAPH"], 0)
    best = C.c_int(-7)
    sets = c.ptr_array([0])
    fake_chain = C.c_void_p(0x1000)   # never dereferenced: the candidate check fails first
    for bad in ((16, 0), (65,), (8, 16, -1)):
        cand = (C.c_int * len(bad))(*bad)
        assert c.LIB.cgx_tune_graph_streams(fake_chain, C.byref(opts), None, sets, 1, 1, cand, len(bad), 10,
                                            C.byref(best), None) == c.E_INVALID_ARG
        assert "1..64" in c.last_error() and best.value == -7
