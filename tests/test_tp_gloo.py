"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 paths:
  * the NCCL unique-id bootstrap over a torch process group (paper_2503_19779_b200.tp);
  * the tensor-parallel partitioning of the decoder chain: each rank evaluates its
    shard with the oracle, ALLREDUCE_SUM nodes sum partials with a gloo all_reduce, and the result
    equals the single-process lockstep evaluation exactly and the TP=1 chain within tolerance.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import chain as och
from oracle import ops
from oracle.numerics import bits_to_f64
from synth import workloads as wl

T, L = 4, 1


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_eval(spec, ext, st):
    env = {}
    for s in spec.slots:
        if s.kind == "external":
            env[s.name] = och.to_host(s, ext[s.name])
        elif s.kind == "static":
            env[s.name] = och.to_host(s, st[s.name])
    for node in spec.nodes:
        if node.op == "ALLREDUCE_SUM":
            t = torch.from_numpy(np.asarray(env[node.ins[0]], dtype=np.float64).copy())
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            env[node.out] = ops.allreduce_sum([t.numpy()])
        else:
            env[node.out] = och.eval_node(spec, node, env, lambda n: spec.slot(n).dtype)
    return env


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_19779_b200 import tp
        uid = tp.broadcast_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        full = wl.c3_chain(T=T, n_layers=L)
        spec = wl.c3_chain(T=T, n_layers=L, tp=world, rank=rank)
        st = wl.static_values(spec, tp=world, rank=rank, full=full)
        ext = wl.external_values(spec, 0)
        env = _rank_eval(spec, ext, st)
        last = spec.nodes[-1].out
        q.put((rank, len(set(ids)) == 1 and len(uid) == 128, env[last]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_tp_two_ranks_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    assert all(ok for _, ok, _ in res)
    outs = [o for _, _, o in res]
    assert np.array_equal(outs[0], outs[1])                  # replicated output after all-reduce
    # equals the single-process lockstep evaluation exactly
    full = wl.c3_chain(T=T, n_layers=L)
    chains = [wl.c3_chain(T=T, n_layers=L, tp=world, rank=r) for r in range(world)]
    sts = [wl.static_values(c, tp=world, rank=r, full=full) for r, c in enumerate(chains)]
    exts = [wl.external_values(c, 0) for c in chains]
    envs = och.eval_chain_tp(chains, exts, sts)
    assert np.array_equal(envs[0][chains[0].nodes[-1].out], outs[0])
    # and the TP=1 chain within the bf16 end-to-end tolerance (Megatron column/row identity)
    ref = och.eval_chain(full, wl.external_values(full, 0), wl.static_values(full))[full.nodes[-1].out]
    assert np.linalg.norm(outs[0] - ref) / np.linalg.norm(ref) <= 2e-2


@pytest.mark.parametrize("tp", [4, 8])
def test_tp_lockstep_matches_tp1(tp):
    """TP = 4 and TP = 8 (12 heads padded to 16) in the single-process lockstep evaluator."""
    full = wl.c3_chain(T=T, n_layers=L)
    chains = [wl.c3_chain(T=T, n_layers=L, tp=tp, rank=r) for r in range(tp)]
    sts = [wl.static_values(c, tp=tp, rank=r, full=full) for r, c in enumerate(chains)]
    exts = [wl.external_values(c, 0) for c in chains]
    envs = och.eval_chain_tp(chains, exts, sts)
    out = envs[0][chains[0].nodes[-1].out]
    for e in envs[1:]:
        assert np.array_equal(e[chains[0].nodes[-1].out], out)
    ref = och.eval_chain(full, wl.external_values(full, 0), wl.static_values(full))[full.nodes[-1].out]
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= 2e-2


def _fd_worker(rank, world, port, q):
    """tp.share_fd over a world-2 gloo group: rank 0's descriptor of a temp file is duplicated into
    rank 1, which reads the file's content through it (the NVLS multicast object's handle travels
    the same way, tp.MulticastRegion)."""
    import tempfile
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2503_19779_b200 import tp
        fd = None
        if rank == 0:
            f = tempfile.TemporaryFile()
            f.write(b"cgx-multicast-handle")
            f.flush()
            fd = os.dup(f.fileno())
        got = tp.share_fd(fd, rank, world)
        os.lseek(got, 0, os.SEEK_SET)
        data = os.read(got, 64)
        os.close(got)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, data))
    except Exception as exn:  # noqa: BLE001
        q.put((rank, repr(exn)))


def test_share_fd_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_fd_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: b"cgx-multicast-handle", 1: b"cgx-multicast-handle"}, res
