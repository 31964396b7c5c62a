"""C5 — tensor-parallel decoder step with captured NCCL all-reduce.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 scripts/bench_tp.py [--layers 12] [--T 128]

Each rank builds its Megatron shard of the GPT-2-small chain (column-parallel QKV/FC1, row-parallel
O/FC2, two ALLREDUCE_SUM nodes per layer), bootstraps an NCCL communicator through the torch
process group (paper_2503_19779_b200.tp), captures the chain INCLUDING the ncclAllReduce calls into
its graph, and replays it with a fresh (replicated) x every step. Per-replay µs is the device time
of each rank's stream, max over ranks. With --check the rank outputs are compared with the
single-process lockstep oracle (1 layer).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--T", type=int, default=128)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--dump", default="", help="directory: every rank saves the GPU value of every INTERNAL "
                    "slot after one INDIRECT replay with input set 0 (rank{r}.npz) for node-local parity")
    ap.add_argument("--allreduce", choices=("nccl", "peer", "fused", "mc"), default="nccl",
                    help="ALLREDUCE_SUM nodes: captured ncclAllReduce, the peer-memory one-shot kernel "
                         "over CUDA IPC-mapped regions (tp.PeerRegions), that all-reduce fused into "
                         "the row-parallel GEMM epilogues (CGX_GEMM_ALLREDUCE), or the NVLS multimem "
                         "all-reduce through an NVSwitch multicast object (tp.MulticastRegion)")
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CGX_TP_DEVICE pins every rank to one GPU (functional runs of the peer path on a 1-GPU box:
    # the ranks' kernels then time-share the device, so the timings mean nothing)
    if os.environ.get("CGX_TP_DEVICE") is not None:
        local = int(os.environ["CGX_TP_DEVICE"])
    torch.cuda.set_device(local)
    use_nccl_pg = world > 1 and args.allreduce == "nccl"   # peer modes: gloo carries the IPC handles
    dist.init_process_group("nccl" if use_nccl_pg else "gloo",
                            device_id=torch.device("cuda", local) if use_nccl_pg else None)
    from paper_2503_19779_b200 import build
    if rank == 0:
        build.build()
    dist.barrier()
    from paper_2503_19779_b200 import cgx, runner, tp
    from synth import workloads as wl

    dev = torch.device("cuda", local)
    comm = tp.nccl_bootstrap(local) if args.allreduce == "nccl" else None
    full = wl.c3_chain(T=args.T, n_layers=args.layers)
    spec = (wl.c3_chain(T=args.T, n_layers=args.layers, tp=world, rank=rank,
                        fuse_allreduce=args.allreduce == "fused") if world > 1 else full)
    st = wl.static_values(spec, tp=world, rank=rank, full=full) if world > 1 else wl.static_values(spec)
    regions = tp.PeerRegions(world, rank, args.T * 768, dev) if args.allreduce in ("peer", "fused") else None
    mcr = tp.MulticastRegion(world, rank, args.T * 768, dev) if args.allreduce == "mc" else None
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev), device=local, nccl_comm=comm,
                         peers=regions.peers() if regions else None, multicast=mcr.multicast() if mcr else None)
    stream = torch.cuda.Stream(device=dev)
    xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
    ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
    LIB = cgx.LIB
    res = {}
    for name, mode, xp in (("indirect_first_node", "INDIRECT", "FIRST_NODE"), ("copy", "COPY", "DEFAULT"),
                           ("eager", "EAGER", "DEFAULT")):
        ex = chain.exec(mode, stream=stream, transport=xp)
        for i in range(5):
            LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
            LIB.cgx_launch(ex.handle)
        stream.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = args.steps if mode != "EAGER" else max(20, args.steps // 10)
        e0.record(stream)
        for i in range(n):
            LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
            LIB.cgx_launch(ex.handle)
        e1.record(stream)
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e3 / n], dtype=torch.float64)
        if world > 1:
            if use_nccl_pg:
                t = t.to(dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = float(t.item())
        if args.dump and name == "indirect_first_node":
            LIB.cgx_bind(ex.handle, ptrs[0], 1)
            LIB.cgx_launch(ex.handle)
            os.makedirs(args.dump, exist_ok=True)
            np.savez(os.path.join(args.dump, f"rank{rank}.npz"),
                     **{s.name: ex.output(s.name) for s in spec.internals()})
        if args.check and name == "indirect_first_node":
            LIB.cgx_bind(ex.handle, ptrs[0], 1)
            LIB.cgx_launch(ex.handle)
            got = ex.output(spec.nodes[-1].out)
            gathered = [None] * world
            dist.all_gather_object(gathered, got)
            if rank == 0:
                from oracle import chain as och
                from oracle.numerics import bits_to_f64
                chains = [wl.c3_chain(T=args.T, n_layers=args.layers, tp=world, rank=r) if world > 1 else full
                          for r in range(world)]
                sts = [wl.static_values(c, tp=world, rank=r, full=full) if world > 1 else wl.static_values(c)
                       for r, c in enumerate(chains)]
                exts = [wl.external_values(c, 0) for c in chains]
                envs = och.eval_chain_tp(chains, exts, sts) if world > 1 else [och.eval_chain(full, exts[0], sts[0])]
                o = envs[0][spec.nodes[-1].out]
                errs = [float(np.linalg.norm(bits_to_f64(g) - o) / np.linalg.norm(o)) for g in gathered]
                res["check_rel_err_per_rank"] = errs
                res["ranks_identical"] = all(np.array_equal(g, gathered[0]) for g in gathered)
        ex.close()
    if rank == 0:
        res["tokens_per_s_indirect"] = args.T * 1e6 / res["indirect_first_node"]
        print(json.dumps({"config": f"C5 TP={world} T={args.T} layers={args.layers} allreduce={args.allreduce}",
                          "us_per_replay_max_over_ranks": res}))
    chain.close()
    if comm is not None:
        cgx.nccl_comm_destroy(comm)
    if regions is not None:
        dist.barrier()                  # no rank unmaps a region a peer may still write
        regions.close()
    if mcr is not None:
        dist.barrier()                  # no rank releases its copy while a peer's multimem op may reach it
        mcr.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
