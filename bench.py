#!/usr/bin/env python
"""bench.py — per-replay rebinding µs and chain iters/s (graph+indirection vs copy vs eager).

Workload (BASELINE.json configs[1]): the 200-kernel elementwise/reduction chain
with 64 external fp32 inputs of 1 KiB..4 MiB (37.7 MB), batch-1 inference-style replay with a
FRESH input set bound every step. A step = one replay of the hot path as deployed: cgx_bind of the
step's 64 input pointers (pointer table patched once) + cgx_launch (one
cudaGraphLaunch of the captured 200-kernel graph). `value` = replays/s over all ranks.

Also measured in the same run (rank 0): every arm's per-replay time and rebinding Δ (COPY,
INDIRECT T1-T4, SETPARAMS, EAGER; Δ = T_iter(arm) - T_iter(graph replay with no rebinding)),
host API µs vs the single-dispatch floor, graph span vs Σ kernel device time, the selector's
decision, the copy kernel at the C4 1 GiB point (HBM roofline), the end-to-end number through the
public API with host<->device copies, and the CPU oracle baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
Under torchrun each rank replays its own graph on its own GPU (independent replicas, no
data-path collective: "scaling": "weak").
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "per-replay rebinding µs and chain iters/s (graph+indirection vs copy vs eager)"
WORKLOAD = ("C2: 200-kernel fp32 elementwise/reduction chain, 64 external inputs of 1 KiB-4 MiB "
            "(37,743,616 B), batch-1 replay with fresh inputs every step")
N_SETS = 8   # rotating input sets: 8 x 37.7 MB = 302 MB > 126 MB L2
MAIN_TRANSPORT = "ROOT_PARAMS"   # INDIRECT pointer-table transport of the deployed arm (fastest DAG replay, r01)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="only the timed hot-path loop")
    ap.add_argument("--graph-streams", type=int, default=0,
                    help="DAG capture streams of the deployed exec (0: measured choice, cgx_tune_graph_streams)")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    return ap.parse_args()


# ------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_ids):
        self.gpu_ids = gpu_ids
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(map(str, self.gpu_ids)), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------------------------- helpers
def final_outputs(spec):
    used = {i for n in spec.nodes for i in n.ins}
    return [s for s in spec.internals() if s.name not in used]


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def cpu_info():
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model


def run_oracle_replays(spec, budget_s: float, max_replays: int = 1000):
    """Time the CPU oracle (INDIRECT capture model: bind + replay with fresh inputs), one thread."""
    from threadpoolctl import threadpool_limits

    from oracle import capture as ocap
    from synth import workloads as wl
    with threadpool_limits(limits=1):
        mem = ocap.Memory()
        saddr = ocap.load_statics(spec, mem, wl.static_values(spec))
        ex = ocap.CapturedExec(spec, "INDIRECT", mem, saddr)
        inputs = [ocap.load_inputs(spec, mem, wl.external_values(spec, r)) for r in range(2)]
        n, t0 = 0, time.perf_counter()
        while n < max_replays:
            ex.bind(inputs[n % 2])
            ex.replay()
            n += 1
            if time.perf_counter() - t0 >= budget_s:
                break
        dt = time.perf_counter() - t0
    return n, dt


def run_oracle_timings():
    """SURVEY §8(d) 'Oracle timing' column: the CPU oracle, one thread, on bounded samples of the
    other configs (C2's is `cpu_baseline`). Seconds of wall time."""
    from threadpoolctl import threadpool_limits

    from oracle import capture as ocap
    from oracle.chain import eval_chain, eval_chain_tp
    from synth import workloads as wl
    out = {}
    with threadpool_limits(limits=1):
        # C1: 10 replays x {COPY, INDIRECT, SETPARAMS} plus the STALE control
        spec = wl.c1_chain()
        t0 = time.perf_counter()
        for mode in ("COPY", "INDIRECT", "SETPARAMS", "STALE"):
            mem = ocap.Memory()
            saddr = ocap.load_statics(spec, mem, wl.static_values(spec))
            inputs = [ocap.load_inputs(spec, mem, wl.external_values(spec, r)) for r in range(10)]
            ex = ocap.CapturedExec(spec, mode, mem, saddr, inputs[0] if mode == "STALE" else None)
            for r in range(10):
                if mode != "STALE":
                    ex.bind(inputs[r])
                ex.replay()
        out["C1_10_replays_x4_arms_s"] = time.perf_counter() - t0
        # C3: one step of the 12-layer decoder (f64 NumPy)
        spec = wl.c3_chain(T=128, n_layers=12)
        st, ext = wl.static_values(spec), wl.external_values(spec, 0)
        t0 = time.perf_counter()
        eval_chain(spec, ext, st)
        out["C3_one_step_12_layers_s"] = time.perf_counter() - t0
        # C4: the window chain at every sweep point up to 64 MiB (the kernels read the window)
        t0 = time.perf_counter()
        for S in [1024 * 4 ** k for k in range(9)]:
            spec = wl.c4_chain(S, window_mode=True)
            eval_chain(spec, wl.external_values(spec, 0), wl.static_values(spec))
        out["C4_window_points_to_64MiB_s"] = time.perf_counter() - t0
        # C5: TP = 2 lockstep ranks (partials + their reduction), 1 layer
        full = wl.c3_chain(T=128, n_layers=1)
        chains = [wl.c3_chain(T=128, n_layers=1, tp=2, rank=r) for r in range(2)]
        stats = [wl.static_values(c, tp=2, rank=r, full=full) for r, c in enumerate(chains)]
        exts = [wl.external_values(c, 0) for c in chains]
        t0 = time.perf_counter()
        eval_chain_tp(chains, exts, stats)
        out["C5_tp2_one_layer_s"] = time.perf_counter() - t0
    out["cores"] = 1
    out["host"] = cpu_info()
    return out


# ------------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import workloads as wl
    spec = wl.c2_chain()
    for _ in range(args.warmup):
        run_oracle_replays(spec, 1e9, max_replays=1)
    n, dt = run_oracle_replays(spec, 1e9, max_replays=max(1, args.steps))
    v = n / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s",
            "n_gpus": args.gpus, "steps": n, "warmup": args.warmup, "ms_per_step": 1e3 * dt / n,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "arm": "oracle INDIRECT capture model (NumPy, CPU)",
                       "parallelism": "rank 0 only"},
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": 1, "kind": "oracle",
                             "sample": f"{n} C2 replays (bind + replay, fresh inputs), 1 thread, "
                                       f"{cpu_info()}"},
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- launcher
def self_launch(args) -> int | None:
    """`python bench.py --gpus N` outside torchrun (WORLD_SIZE unset, N > 1): start N ranks of this
    script with torch.distributed.run on 127.0.0.1 (one process per GPU) and return their exit
    code; rank 0 prints the JSON line. Under torchrun (WORLD_SIZE set) nothing happens."""
    if args.gpus <= 1 or os.environ.get("WORLD_SIZE") is not None:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


# ------------------------------------------------------------------------------- ours
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # (the host thread is not pinned: the clock sampler's nvidia-smi subprocess and the CPU oracle
    # would inherit a one-core affinity and compete with the launch loop on that core)
    # functional checks of the multi-rank path on a one-GPU box (never a measurement):
    # CGX_BENCH_DEVICE pins every rank to one device, CGX_BENCH_PG=gloo avoids NCCL's one-rank-per-GPU rule
    if os.environ.get("CGX_BENCH_DEVICE") is not None:
        local = int(os.environ["CGX_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    pg_gloo = os.environ.get("CGX_BENCH_PG") == "gloo"
    if world > 1:
        if pg_gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2503_19779_b200 import build
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    from paper_2503_19779_b200 import cgx, runner
    from synth import splitmix as sm
    from synth import workloads as wl

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream
    spec = wl.c2_chain()
    statics = runner.upload_statics(spec, wl.static_values(spec), dev)
    chain = runner.Chain(spec, statics, device=local)
    ext = spec.externals()
    # rotating input sets generated on device with the synth recipe (stream (slot<<20)|set)
    sets, set_ptrs = [], []
    for r in range(N_SETS):
        ts = []
        for s in ext:
            t = torch.empty(s.nelems, dtype=torch.float32, device=dev)
            cgx.fill_uniform_f32(t.data_ptr(), s.nelems, sm.SEED,
                                 sm.stream_id(spec.index(s.name), r + 1000 * rank), sh)
            ts.append(t)
        sets.append(ts)
        set_ptrs.append(cgx.ptr_array([t.data_ptr() for t in ts]))
    torch.cuda.synchronize(dev)
    n_ext = len(ext)
    LIB = cgx.LIB

    def loop(handle, n, bind=True, start=0):
        for i in range(n):
            if bind:
                st = LIB.cgx_bind(handle, set_ptrs[(start + i) % N_SETS], n_ext)
                if st:
                    raise cgx.CgxError(st, "cgx_bind", cgx.last_error())
            st = LIB.cgx_launch(handle)
            if st:
                raise cgx.CgxError(st, "cgx_launch", cgx.last_error())

    def timed(handle, n, bind=True):
        """device-timeline µs per iteration over n back-to-back iterations (events on `stream`)."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            loop(handle, n, bind)
            e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e3 / n

    main_arm = ("INDIRECT", MAIN_TRANSPORT)
    # slow path (like the selector's profiling): the DAG capture's stream count is
    # measured on this workload's inputs and the fastest deployed (cgx_tune_graph_streams)
    tune_us = None
    if args.graph_streams:
        best_streams = args.graph_streams
    else:
        best_streams, tune_us = cgx.tune_graph_streams(
            chain.handle, main_arm[0], stream.cuda_stream, [[t.data_ptr() for t in ts] for ts in sets],
            candidates=(8, 12, 14, 16, 20, 24, 32), reps=100, transport=main_arm[1])
    ex_main = chain.exec(main_arm[0], stream=stream, transport=main_arm[1], validate=0, graph_streams=best_streams)
    h = ex_main.handle
    loop(h, max(3, args.warmup))
    stream.synchronize()

    # ---------------------------------------------------------------- timed hot-path loop
    clocks = ClockSampler([local] if world == 1 else list(range(world))) if rank == 0 else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    if clocks:
        clocks.start()
        time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    with torch.cuda.stream(stream):
        e0.record(stream)
        loop(h, args.steps)
        e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    el_ms = e0.elapsed_time(e1)
    t = torch.tensor([el_ms], dtype=torch.float64, device="cpu" if pg_gloo else dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * args.steps / (max_ms / 1e3)
    stats_main = ex_main.stats()

    e2e = None
    if not args.no_extras:
        if world > 1:
            dist.barrier()
        e2e = run_e2e_all(torch, cgx, wl, spec, chain, stream, dev, world)
    # C5 (BASELINE configs[4]): the TP = N decoder step with captured all-reduces, every rank
    c5 = None
    if world > 1 and not args.no_extras:
        dist.barrier()
        c5 = bench_tp_leg(torch, dist, cgx, runner, wl, dev, local, rank, world, pg_gloo)
    extras = {}
    if rank == 0 and not args.no_extras:
        extras = run_extras(args, torch, cgx, runner, wl, sm, spec, chain, stream, sets, set_ptrs,
                            timed, loop, ex_main, dev)
    if world > 1:
        dist.barrier()
    if rank != 0:
        chain.close()
        if world > 1:
            dist.destroy_process_group()
        return

    line = {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "arm": f"GRAPH_INDIRECT (pointer table, {MAIN_TRANSPORT} transport)",
                   "kernels_per_replay": stats_main["kernels_per_replay"],
                   "graph_streams": best_streams,
                   "graph_streams_tuning_us": ({str(k): round(v, 2) for k, v in tune_us.items()} if tune_us
                                               else "fixed by --graph-streams"),
                   "l2": f"rotating {N_SETS} input sets ({N_SETS * 37743616 / 1e6:.0f} MB > 126 MB L2)",
                   "parallelism": f"independent replicas x{world}"},
        "gpu_launches": args.steps * stats_main["kernels_per_replay"],
        "clocks": clk,
        "wall_s_timed_region": wall,
    }
    line.update(extras)
    if e2e is not None:
        line["e2e"] = e2e
    if c5 is not None:
        line["c5_tp"] = c5
    print(json.dumps(line), flush=True)
    chain.close()
    if world > 1:
        dist.destroy_process_group()


def bench_tp_leg(torch, dist, cgx, runner, wl, dev, local, rank, world, pg_gloo):
    """C5: the GPT-2-small decoder (12 layers, T = 128) Megatron-sharded
    TP = world ways, one process per GPU, replayed as each rank's captured graph with a fresh
    (replicated) x bound every step. Variants: ALLREDUCE_SUM as a captured ncclAllReduce (NVLink /
    NVSwitch), and the row-parallel GEMMs with the peer all-reduce fused into their epilogue over
    CUDA-IPC-mapped regions. µs per replay = device time on each rank's stream, MAX over ranks;
    tokens/s = T / that. A third variant runs the all-reduces through an NVSwitch multicast object
    (NVLS, multimem.ld_reduce) where the driver grants one. Never fatal: a failing variant is
    reported as its error string."""
    from paper_2503_19779_b200 import tp
    T, L = 128, 12
    out = {"tp": world, "workload": f"C5: GPT-2-small decoder, {L} layers, T={T}, bf16, TP={world} "
                                     "(column-parallel QKV/FC1, row-parallel O/FC2, 2 all-reduces per layer)"}
    full = wl.c3_chain(T=T, n_layers=L)
    stream = torch.cuda.Stream(device=dev)

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if pg_gloo else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for name, kind in (("nccl", "nccl"), ("peer_fused", "fused"), ("nvls", "mc")):
        comm = regions = mcr = chain = None
        res = {}
        try:
            spec = wl.c3_chain(T=T, n_layers=L, tp=world, rank=rank, fuse_allreduce=kind == "fused")
            st = wl.static_values(wl.c3_chain(T=T, n_layers=L, tp=world, rank=rank), tp=world, rank=rank, full=full)
            if kind == "nccl":
                if pg_gloo:
                    raise RuntimeError("NCCL ranks need one GPU each (CGX_BENCH_PG=gloo run)")
                comm = tp.nccl_bootstrap(local)
            elif kind == "mc":   # NVLS: multimem all-reduce through an NVSwitch multicast object
                ok = cgx.mc_supported(local)
                t_ok = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64, device="cpu" if pg_gloo else dev)
                dist.all_reduce(t_ok, op=dist.ReduceOp.MIN)
                if t_ok.item() < 1.0:
                    raise RuntimeError("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0 on some rank")
                mcr = tp.MulticastRegion(world, rank, T * 768, dev, max_allreduces=2 * L)
            else:
                regions = tp.PeerRegions(world, rank, T * 768, dev, max_allreduces=2 * L)
            chain = runner.Chain(spec, runner.upload_statics(spec, st, dev), device=local, nccl_comm=comm,
                                 peers=regions.peers() if regions else None,
                                 multicast=mcr.multicast() if mcr else None)
            xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
            ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
            ex = chain.exec("INDIRECT", stream=stream, transport="FIRST_NODE")
            n = 200
            for i in range(10):
                cgx.bind(ex.handle, [xs[i % 4].data_ptr()])
                cgx.launch(ex.handle)
            stream.synchronize()
            best = 1e30
            for _ in range(3):
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for i in range(n):
                    if cgx.LIB.cgx_bind(ex.handle, ptrs[i % 4], 1) or cgx.LIB.cgx_launch(ex.handle):
                        raise cgx.CgxError(1, "bind/launch", cgx.last_error())
                e1.record(stream)
                e1.synchronize()
                best = min(best, max_over_ranks(e0.elapsed_time(e1) * 1e3 / n))
            res = {"us_per_replay_max_over_ranks": best, "tokens_per_s": T * 1e6 / best,
                   "kernels_per_replay": ex.stats()["kernels_per_replay"]}
            ex.close()
        except Exception as exn:  # noqa: BLE001
            res = {"error": f"{type(exn).__name__}: {exn}"[:400]}
        finally:
            if chain is not None:
                chain.close()
            try:
                dist.barrier()
            except Exception:  # noqa: BLE001
                pass
            if comm is not None:
                cgx.nccl_comm_destroy(comm)
            if regions is not None:
                regions.close()
            if mcr is not None:
                mcr.close()
        out[name] = res
    return out


def run_e2e_all(torch, cgx, wl, spec, chain, stream, dev, world):
    """End to end through the public API on EVERY rank at once (pinned H2D inputs + D2H results);
    the whole-job value is all ranks' steps over the max-over-ranks elapsed time."""
    LIB = cgx.LIB
    sh = stream.cuda_stream
    n_ext = len(spec.externals())
    main_transport = MAIN_TRANSPORT
    # ---------------- end to end through the public API (pinned H2D inputs + D2H result)
    # Inputs live packed in one pinned host arena per step and are copied (two halves, two copy
    # streams) into a triple-buffered device arena, overlapping the replays; the 64 final outputs
    # are packed on the device (cgx_output_gather) and read back with one D2H copy, and the host
    # waits for every step's results before the clock stops.
    outs = final_outputs(spec)
    exts = spec.externals()
    offs, tot = [], 0
    for s_ in exts:
        offs.append(tot)
        tot += (s_.nbytes + 255) // 256 * 256
    NB = 3                                     # triple-buffered pinned/device arenas
    host_arena = []
    for r in range(NB):
        vals = wl.external_values(spec, r % 2)
        h = torch.zeros(tot, dtype=torch.uint8).pin_memory()
        hv = h.numpy()
        for s_, o in zip(exts, offs):
            hv[o:o + s_.nbytes] = vals[s_.name].view("u1")
        host_arena.append(h)
    dev_arena = [torch.empty(tot, dtype=torch.uint8, device=dev) for _ in range(NB)]
    arena_ptrs = [cgx.ptr_array([d.data_ptr() + o for o in offs]) for d in dev_arena]
    out_slots = [chain.slot[s_.name] for s_ in outs]
    out_cap = sum((s_.nbytes + 15) // 16 * 16 for s_ in outs)
    host_out = [torch.empty(out_cap, dtype=torch.uint8).pin_memory() for _ in range(NB)]
    dev_out = [torch.empty(out_cap, dtype=torch.uint8, device=dev) for _ in range(NB)]
    ex2 = chain.exec("INDIRECT", stream=stream, transport=main_transport)
    out_bytes = cgx.output_gather(ex2.handle, out_slots, dev_out[0].data_ptr(), out_cap)
    torch.cuda.synchronize(dev)
    # the H2D of a step is split in two halves on two copy streams (one 37.7 MB copy measured
    # 42-54 GB/s run to run, two concurrent halves a steady ~53.6 GB/s: scripts/diag_h2d.py)
    cstreams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    half = (tot // 2) // 256 * 256
    ev_h2d = [[torch.cuda.Event() for _ in range(2)] for _ in range(NB)]
    ev_free = [torch.cuda.Event() for _ in range(NB)]
    h2 = ex2.handle

    def issue_h2d(i):
        b = i % NB
        for k, cs_ in enumerate(cstreams):
            if i >= NB:
                cs_.wait_event(ev_free[b])     # step i - NB has released arena b
            lo, hi = (0, half) if k == 0 else (half, tot)
            cgx.copy(dev_arena[b].data_ptr() + lo, host_arena[b].data_ptr() + lo, hi - lo, cs_.cuda_stream)
            ev_h2d[b][k].record(cs_)

    def issue_compute(i):
        b = i % NB
        for ev_ in ev_h2d[b]:
            stream.wait_event(ev_)
        st_ = LIB.cgx_bind(h2, arena_ptrs[b], n_ext)
        if st_ == 0:
            st_ = LIB.cgx_launch(h2)
        if st_:
            raise cgx.CgxError(st_, "e2e", cgx.last_error())
        # the 64 results: packed on the device by one gather kernel, read with ONE D2H copy
        cgx.output_gather(h2, out_slots, dev_out[b].data_ptr(), out_cap)
        cgx.copy(host_out[b].data_ptr(), dev_out[b].data_ptr(), out_bytes, sh)
        ev_free[b].record(stream)

    def run_e2e(n):
        # step i: H2D of its inputs (issued two steps ahead on the copy stream), bind + replay,
        # D2H of its 64 results; the host waits for step i-1's results after issuing step i, and
        # for the last step's before the clock stops: every step's result reaches host memory
        torch.cuda.synchronize(dev)
        t0w = time.perf_counter()
        for j in range(min(NB - 1, n)):
            issue_h2d(j)
        for i in range(n):
            issue_compute(i)
            if i + NB - 1 < n:
                issue_h2d(i + NB - 1)
            if i >= 1:
                ev_free[(i - 1) % NB].synchronize()
        ev_free[(n - 1) % NB].synchronize()
        torch.cuda.synchronize(dev)
        return time.perf_counter() - t0w

    run_e2e(10)
    n_e2e = 400
    e2e_dt = run_e2e(n_e2e)
    if world > 1:                               # whole job: every rank's steps / max over ranks
        import torch.distributed as dist
        tt = torch.tensor([e2e_dt], dtype=torch.float64,
                          device="cpu" if os.environ.get("CGX_BENCH_PG") == "gloo" else dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_dt = float(tt.item()) / world
    res = {"value": n_e2e / e2e_dt, "unit": "iters/s",
                  "h2d_bytes_per_step": sum(s_.nbytes for s_ in exts),
                  "d2h_bytes_per_step": out_bytes,
                  "h2d_GBps": sum(s_.nbytes for s_ in exts) * n_e2e / e2e_dt / 1e9,
                  "note": "public API (cgx_copy H2D of the step's 64 inputs from one pinned arena on a "
                          "copy stream, cgx_bind + cgx_launch, cgx_output_gather of the 64 final "
                          "outputs + ONE cgx_copy D2H, "
                          "host waits for every step's result); triple-buffered: the H2D of step "
                          "i+2 (two halves on two copy streams) overlaps replay i; PCIe Gen5 x16 H2D ceiling on this box ~54 GB/s "
                          "(scripts/diag_h2d.py)"}
    ex2.close()
    return res



def run_extras(args, torch, cgx, runner, wl, sm, spec, chain, stream, sets, set_ptrs, timed, loop,
               ex_main, dev):
    sh = stream.cuda_stream
    main_transport = MAIN_TRANSPORT
    deployed_streams = ex_main.stats()["dag_streams"] or 16   # the main exec's DAG capture streams
    out = {}
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
    n_ext = len(spec.externals())
    LIB = cgx.LIB

    # ---------------- arms: per-replay device time and rebinding Δ
    # Headline base (SURVEY §8(d) literal): the SAME exec relaunched without binding (same pointers),
    # interleaved with bind+launch pairs on it. Its inputs stay L2-warm while the rebinding replays
    # read fresh (cold) inputs, so Δ also charges each arm the cold-input reads of its replay — for
    # INDIRECT (whose graph reads the fresh inputs directly) that makes Δ an over-estimate; COPY's
    # graph reads placeholders its copy kernel just wrote. Also reported: Δ against a cold base of
    # N_SETS COPY execs (one input set each) launched round-robin without binding; with the
    # dependency-DAG capture that base is slower than an INDIRECT replay (exec switching).
    M = 2000
    arms = {}
    ex_copy = chain.exec("COPY", stream=stream)
    loop(ex_copy.handle, 20)
    base_warm = min(timed(ex_copy.handle, M, bind=False) for _ in range(3))
    cold = [chain.exec("COPY", stream=stream) for _ in range(N_SETS)]
    for i, exc in enumerate(cold):
        LIB.cgx_bind(exc.handle, set_ptrs[i], n_ext)
        LIB.cgx_launch(exc.handle)
    stream.synchronize()

    def timed_rr(n):
        e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        with torch.cuda.stream(stream):
            e0_.record(stream)
            for i in range(n):
                LIB.cgx_launch(cold[i % N_SETS].handle)
            e1_.record(stream)
        e1_.synchronize()
        return e0_.elapsed_time(e1_) * 1e3 / n
    timed_rr(50)
    base = min(timed_rr(M) for _ in range(3))
    arms["graph_no_rebind_cold_copy_rr"] = {"us_per_replay": base,
                                            "base": f"cold: {N_SETS} COPY execs round-robin, no bind"}
    arms["graph_no_rebind_warm_copy"] = {"us_per_replay": base_warm, "base": "warm: one COPY exec, same inputs"}
    for name, (mode, xp) in {"copy": ("COPY", "DEFAULT"), "indirect_h2d": ("INDIRECT", "H2D"),
                             "indirect_root_memcpy": ("INDIRECT", "ROOT_MEMCPY"),
                             "indirect_root_params": ("INDIRECT", "ROOT_PARAMS"),
                             "indirect_root_mapped": ("INDIRECT", "ROOT_MAPPED"),
                             "indirect_first_node": ("INDIRECT", "FIRST_NODE"),
                             "indirect_h2d_pingpong": ("INDIRECT", "H2D_PINGPONG"),
                             "indirect_prelude": ("INDIRECT", "PRELUDE"),
                             "setparams": ("SETPARAMS", "DEFAULT")}.items():
        ex = ex_copy if mode == "COPY" else chain.exec(mode, stream=stream, transport=xp)
        loop(ex.handle, 20)
        # base (same exec, no bind) and arm interleaved, 5 pairs: the median pair difference
        # cancels slow drift; the cold round-robin COPY base is interleaved the same way
        pairs, pairs_c = [], []
        for _ in range(5):
            b_ = timed(ex.handle, M // 2, bind=False)
            a_ = timed(ex.handle, M // 2)
            c_ = timed_rr(M // 4)
            pairs.append((a_, b_))
            pairs_c.append((a_, c_))
        us = statistics.median(a_ for a_, _ in pairs)
        us_base = statistics.median(b_ for _, b_ in pairs)
        delta = statistics.median(a_ - b_ for a_, b_ in pairs)
        noise = statistics.pstdev(a_ - b_ for a_, b_ in pairs)
        delta_c = statistics.median(a_ - c_ for a_, c_ in pairs_c)
        host = []
        for i in range(200):
            stream.synchronize()
            t0 = time.perf_counter()
            LIB.cgx_bind(ex.handle, set_ptrs[i % N_SETS], n_ext)
            LIB.cgx_launch(ex.handle)
            host.append((time.perf_counter() - t0) * 1e6)
        stream.synchronize()
        arms[name] = {"us_per_replay": us, "us_per_replay_no_rebind_same_exec": us_base,
                      "rebind_delta_us": delta, "rebind_delta_noise_us": noise,
                      "rebind_delta_vs_cold_copy_base_us": delta_c,
                      "host_bind_launch_us": statistics.median(host)}
        if ex is not ex_copy:
            ex.close()
    for exc in cold:
        exc.close()
    # node ordering inside the replay: the dependency-DAG capture (deployed, GRAPH) at
    # several stream counts vs the serial captures (dataflow counters, deferred PDL waits, plain
    # PDL chain), same INDIRECT exec otherwise
    sync_cmp = {}
    for sm_, ns_ in (("GRAPH", 16), ("GRAPH", 8), ("GRAPH", 4), ("GRAPH", 32), ("DATAFLOW", 0), ("DEFER", 0),
                     ("CHAIN", 0)):
        ex = chain.exec("INDIRECT", stream=stream, transport=main_transport, sync=sm_, graph_streams=ns_)
        loop(ex.handle, 20)
        key = f"{sm_}_{ns_}" if sm_ == "GRAPH" else sm_
        sync_cmp[key] = {"us_per_replay": min(timed(ex.handle, M) for _ in range(3)),
                         "dataflow": ex.stats()["dataflow"], "n_deferred": ex.stats()["n_deferred"],
                         "dag_streams": ex.stats()["dag_streams"]}
        ex.close()
    out["sync_modes"] = sync_cmp
    # NEXT-4: device-launched replays (transport DEVICE): one host call runs M replays; the host
    # thread's CPU time per replay vs the host-driven loop on the same exec
    try:
        exd = chain.exec("INDIRECT", stream=stream, transport="DEVICE")
        tab = torch.tensor([[t.data_ptr() for t in ts] for ts in sets], dtype=torch.int64, device=dev)
        loop(exd.handle, 20)
        host_us = min(timed(exd.handle, M) for _ in range(3))
        stream.synchronize()
        c0 = time.process_time()
        loop(exd.handle, M)
        c_host = (time.process_time() - c0) * 1e6 / M
        stream.synchronize()

        def dl():
            e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            with torch.cuda.stream(stream):
                e0_.record(stream)
                c0_ = time.process_time()
                cgx.device_loop(exd.handle, tab.data_ptr(), N_SETS, M)
                c1_ = time.process_time()
                e1_.record(stream)
            e1_.synchronize()
            return e0_.elapsed_time(e1_) * 1e3 / M, (c1_ - c0_) * 1e6 / M
        dl()
        dev_us, c_dev = min(dl() for _ in range(3))
        out["device_loop"] = {"us_per_replay_device_loop": dev_us, "us_per_replay_host_loop_same_exec": host_us,
                              "host_cpu_us_per_replay_device_loop": c_dev,
                              "host_cpu_us_per_replay_host_loop": c_host,
                              "note": "NEXT-4: cgx_device_loop (scheduler kernel binds set i and tail-launches "
                                      "the chain graph); host CPU = process time of the issuing thread"}
        exd.close()
    except Exception as exn:  # noqa: BLE001
        out["device_loop"] = {"error": str(exn)}
    ex_e = chain.exec("EAGER", stream=stream)
    loop(ex_e.handle, 3)
    us_e = min(timed(ex_e.handle, 100) for _ in range(3))
    arms["eager"] = {"us_per_replay": us_e}
    ex_e.close()
    main_ind = "indirect_" + MAIN_TRANSPORT.lower()          # the deployed transport is the headline
    best_ind = min((k for k in arms if k.startswith("indirect")), key=lambda k: arms[k]["rebind_delta_us"])
    d_copy = arms["copy"]["rebind_delta_us"]
    d_ind = arms[main_ind]["rebind_delta_us"]
    # a Δ within the pair-to-pair noise is unresolved: the ratio is then a lower bound, computed
    # with Δ_indirect raised to that noise (reported, never a division by ~0)
    ind_res = max(d_ind, arms[main_ind]["rebind_delta_noise_us"], 0.05)
    out["arms"] = arms
    out["rebinding_us"] = {"copy": d_copy, "indirect": d_ind, "indirect_transport": main_ind,
                           "setparams": arms["setparams"]["rebind_delta_us"],
                           "copy_over_indirect": d_copy / ind_res,
                           "copy_over_indirect_is_lower_bound": ind_res > d_ind,
                           "indirect_noise_us": arms[main_ind]["rebind_delta_noise_us"],
                           "lowest_indirect": {"transport": best_ind, "delta_us": arms[best_ind]["rebind_delta_us"]},
                           "definition": "T_iter(bind+launch, fresh inputs from 8 rotating sets) - "
                                         "T_iter(launch only, same exec, same pointers), device timeline, "
                                         "median of 5 interleaved pairs of 1000 replays (DESIGN reading 14)",
                           "vs_cold_copy_base": {"copy": arms["copy"]["rebind_delta_vs_cold_copy_base_us"],
                                                 "indirect": arms[main_ind]["rebind_delta_vs_cold_copy_base_us"]}}
    g_floor, k_floor = cgx.dispatch_floor(sh, 2000)
    out["dispatch_floor"] = {"graph_launch_us": g_floor, "kernel_launch_us": k_floor,
                             "bind_launch_over_floor": arms[main_ind]["host_bind_launch_us"] / g_floor}

    # ---------------- selector profile (slow path)
    # cgx_profile_ex over the 8 rotating input sets: each arm's delta against its own launch-only
    # loop, the dependency-DAG estimate model (cgx.h model 1), estimates vs measured totals
    prof = cgx.profile(chain.handle, -1, None, 30, sh, sets=[[ps[i] for i in range(n_ext)] for ps in set_ptrs])
    pd = prof.as_dict()
    dec, est = cgx.select([prof])
    prof.use_measured = 0
    dec_e, est_e = cgx.select([prof])
    meas = (pd["t_eager_us"], pd["t_copy_us"], pd["t_ind_us"])
    out["selector"] = {"decision": cgx.DECIDE[dec[0]], "decision_estimates": cgx.DECIDE[dec_e[0]],
                       "t_eager_us": pd["t_eager_us"], "t_copy_us": pd["t_copy_us"], "t_ind_us": pd["t_ind_us"],
                       "t_copy_base_us": pd["t_copy_base_us"], "t_ind_base_us": pd["t_ind_base_us"],
                       "L_us": pd["L_us"], "G_us": pd["G_us"], "c_copy_us": pd["c_copy_us"],
                       "c_ind_us": pd["c_ind_us"], "model": "dependency-DAG list schedule (cgx.h model 1)",
                       "delta_issue_us": pd["delta_us"], "lambda_us": pd["lambda_us"],
                       "span_traced_us": pd["span_us"], "n_sets": pd["n_sets"], "n_deps": pd["n_deps"],
                       "estimates_us": list(est_e[0]),
                       "estimate_rel_err": [(e - m) / m for e, m in zip(est_e[0], meas)]}

    # ---------------- Σ kernel device time vs replay (span <= 1.5 x Σ)
    # Kernel durations come from CUPTI activity records (torch.profiler) of a replay of the same
    # graph captured WITHOUT programmatic dependent launch, so each kernel's duration is its own
    # execution (with PDL a kernel is resident early and its record includes the wait).
    rep_us = arms["indirect_first_node"]["us_per_replay"]
    per_name, sum_cupti = {}, None
    ex_np = chain.exec("INDIRECT", stream=stream, transport=main_transport, no_pdl=True)
    loop(ex_np.handle, 5)
    stream.synchronize()
    try:
        from torch.profiler import ProfilerActivity, profile as tprof
        with tprof(activities=[ProfilerActivity.CUDA]) as tp:
            loop(ex_np.handle, 10)
            stream.synchronize()
        tot = 0.0
        for ev in tp.key_averages():
            if "k_" in ev.key and "cgx" in ev.key:
                t_ = getattr(ev, "device_time_total", None)
                if t_ is None:
                    t_ = getattr(ev, "cuda_time_total", 0.0)
                tot += t_
                per_name[ev.key] = {"us_per_replay": t_ / 10, "launches_per_replay": ev.count / 10}
        sum_cupti = tot / 10
    except Exception as exn:  # noqa: BLE001
        per_name = {"error": str(exn)}
    us_nopdl = timed(ex_np.handle, 1000)
    ex_np.close()
    floor200 = cgx.graph_floor(sh, 200, True, 300)
    out["graph_span_over_sum_kernel"] = {
        "replay_us": rep_us, "replay_us_no_pdl": us_nopdl, "sum_kernel_us": sum_cupti,
        "ratio": (rep_us / sum_cupti) if sum_cupti else None,
        "graph_floor_200_noop_kernels_us": floor200,
        "per_kernel": per_name,
        "note": "Σ = CUPTI kernel durations of the same INDIRECT graph captured without PDL; "
                "replay_us = deployed replay (with PDL); floor = 200 no-op 1-CTA kernels, same PDL "
                "protocol"}

    # ---------------- roofline of the dominant kernel (by share of Σ kernel time)
    # Its launches (same kernel, same shapes, same INDIRECT operand fetch) are captured alone in a
    # graph without PDL and timed with CUDA events on the replay stream over 200 replays:
    # avg launch duration = replay span / launches (includes each node's in-graph dispatch).
    from synth.workloads import ChainSpec as _CS
    name_op = {"k_elem_f32<0": "ADD", "k_elem_f32<1": "MUL", "k_reduce_sum_f32": "REDUCE_SUM",
               "k_elem_f32<2": "SCALE_IMM"}
    dom_op = "ADD"
    if isinstance(per_name, dict) and per_name and "error" not in per_name:
        best = max(per_name.items(), key=lambda kv: kv[1]["us_per_replay"])[0]
        for k_, v_ in name_op.items():
            if k_ in best:
                dom_op = v_
    share = None
    if sum_cupti:
        share = sum(v["us_per_replay"] for k_, v in per_name.items()
                    if any(k2 in k_ for k2, o in name_op.items() if o == dom_op)) / sum_cupti

    def algo_bytes(node):
        n = node.attrs["n"]
        if node.op in ("ADD", "MUL"):
            return 3 * 4 * n
        if node.op in ("SCALE_IMM", "COPY"):
            return 2 * 4 * n
        return 4 * n + 4 * n // node.attrs.get("cols", 256)

    def sub_roofline(nodes, overlapped=False):
        used = {i for n in nodes for i in n.ins} | {n.out for n in nodes}
        slots = [s_ for s_ in spec.slots if s_.name in used]
        sub = _CS("dom", slots, nodes, [(0, len(nodes) - 1)])
        sch = runner.Chain(sub, {k_: v for k_, v in chain.statics.items() if k_ in used}, device=dev.index or 0)
        exs = sch.exec("INDIRECT", stream=stream, transport=MAIN_TRANSPORT if overlapped else "ROOT_PARAMS",
                       no_pdl=not overlapped, graph_streams=deployed_streams if overlapped else 0)
        idx = [spec.externals().index(s_) for s_ in sub.externals()]
        arrs = [cgx.ptr_array([set_ptrs[r][i] for i in idx]) for r in range(N_SETS)]
        nx = len(idx)
        for i in range(5):
            LIB.cgx_bind(exs.handle, arrs[i % N_SETS], nx)
            LIB.cgx_launch(exs.handle)
        best_ = 1e30
        for _ in range(3):
            e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            e0_.record(stream)
            for i in range(200):
                LIB.cgx_bind(exs.handle, arrs[i % N_SETS], nx)
                LIB.cgx_launch(exs.handle)
            e1_.record(stream)
            e1_.synchronize()
            best_ = min(best_, e0_.elapsed_time(e1_) * 1e3 / 200)
        exs.close()
        sch.close()
        # the root writer node (1 CTA, ~the graph floor) is part of the span: subtract it
        has_root = (not overlapped) or MAIN_TRANSPORT.startswith("ROOT")    # FIRST_NODE / H2D: no root node
        root = cgx.graph_floor(sh, 1, False, 200) if has_root else 0.0
        per_launch = max(1e-3, (best_ - root) / len(nodes))
        byts = sum(algo_bytes(n) for n in nodes) / len(nodes)
        return per_launch, byts

    dom_nodes = [n for n in spec.nodes if n.op == dom_op]
    us_l, by_l = sub_roofline(dom_nodes)
    # the same measurement per lane size: the latency floor at small sizes vs HBM at 4 MiB
    by_size = []
    for nsz in sorted({n.attrs["n"] for n in dom_nodes}):
        grp = [n for n in dom_nodes if n.attrs["n"] == nsz]
        u_, b_ = sub_roofline(grp)
        by_size.append({"bytes_per_launch": b_, "launches": len(grp), "us_per_launch": u_,
                        "GBps": b_ / (u_ * 1e-6) / 1e9})
    big = [n for n in dom_nodes if n.attrs["n"] == (4 << 20) // 4]
    us_b, by_b = sub_roofline(big) if big else (None, None)
    achieved = by_l / (us_l * 1e-6) / 1e9
    # the same launches captured the way the replay deploys them (PDL early trigger, dataflow sync:
    # the independent lanes overlap): throughput of this kernel class in the deployed regime
    us_o, by_o = sub_roofline(dom_nodes, overlapped=True)
    kname = {"ADD": "k_elem_f32<0>", "MUL": "k_elem_f32<1>", "REDUCE_SUM": "k_reduce_sum_f32",
             "SCALE_IMM": "k_elem_f32<2>"}[dom_op]
    traffic = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tj.get(kname)
    except (OSError, ValueError):
        pass
    achieved_dep = by_o / (us_o * 1e-6) / 1e9
    # per-launch durations of this kernel INSIDE the deployed C2 replay: the deployed
    # exec rebuilt with node-timeline stamps (CGX_NODE_TRACE=1: first CTA entry, last CTA past its
    # PDL wait, last CTA exit per launch), 50 replays with rotating inputs; work = exit - ready
    node_trace = None
    try:
        os.environ["CGX_NODE_TRACE"] = "1"
        ex_tr = chain.exec("INDIRECT", stream=stream, transport=MAIN_TRANSPORT, graph_streams=deployed_streams)
        os.environ.pop("CGX_NODE_TRACE", None)
        K_ = len(spec.nodes)
        for i in range(10):
            LIB.cgx_bind(ex_tr.handle, set_ptrs[i % N_SETS], n_ext)
            LIB.cgx_launch(ex_tr.handle)
        cgx.node_trace(ex_tr.handle, K_)
        pos = [k for k, n in enumerate(spec.nodes) if n.op == dom_op]
        work, resident, bsum, wsum = [], [], 0.0, 0.0
        for i in range(50):
            LIB.cgx_bind(ex_tr.handle, set_ptrs[i % N_SETS], n_ext)
            LIB.cgx_launch(ex_tr.handle)
            tr = cgx.node_trace(ex_tr.handle, K_)
            for k in pos:
                en, rd, xt = tr[k]
                w_ = max(1, xt - rd) * 1e-3
                work.append(w_)
                resident.append(max(1, xt - en) * 1e-3)
                bsum += algo_bytes(spec.nodes[k])
                wsum += w_
        ex_tr.close()
        ach_w = bsum / (wsum * 1e-6) / 1e9
        dram = traffic
        node_trace = {"launches_sampled": len(work), "median_work_us": statistics.median(work),
                      "median_resident_us": statistics.median(resident),
                      "achieved_GBps_work": ach_w, "frac_work": ach_w / hbm,
                      "dram_bytes_per_launch": dram,
                      "dram_GBps_work": (dram * len(pos) * 50 / (wsum * 1e-6) / 1e9) if dram else None,
                      "dram_frac_work": (dram * len(pos) * 50 / (wsum * 1e-6) / 1e9 / hbm) if dram else None,
                      "timing": "node-timeline stamps (%globaltimer) of every launch of this kernel inside the "
                                "deployed INDIRECT replay (dependency DAG, PDL), 50 replays with rotating inputs: "
                                "work = last CTA exit - last CTA past its griddepcontrol.wait; achieved = sum of "
                                "algorithmic bytes / sum of work times (launches overlap, so this is per-launch, "
                                "not class throughput); dram_* use the ncu DRAM bytes per launch (traffic)"}
    except Exception as exn:  # noqa: BLE001
        os.environ.pop("CGX_NODE_TRACE", None)
        node_trace = {"error": str(exn)}
    out["roofline"] = {"bound": "hbm", "achieved": achieved_dep, "peak": hbm, "unit": "GB/s",
                       "frac": achieved_dep / hbm, "traffic": traffic, "kernel": kname,
                       "share_of_sum_kernel_time": share, "launches_per_replay": len(dom_nodes),
                       "algorithmic_bytes_per_launch": by_o, "avg_launch_us": us_o,
                       "timing": "CUDA events on the replay stream around 200 replays of a graph holding "
                                 "only this kernel's 64 launches, captured the way the replay deploys them "
                                 f"(dependency DAG over the deployed {deployed_streams} streams, PDL, INDIRECT operands): span / launches. "
                                 "Independent launches overlap, so this is the kernel's sustained per-launch "
                                 "time in the deployed regime (class throughput), not one launch's duration",
                       "serial_no_pdl": {"avg_launch_us": us_l, "achieved_GBps": achieved, "frac": achieved / hbm,
                                         "timing": "the same launches serialised in a graph without PDL: span "
                                                   "minus one root node, divided by launches (each includes the "
                                                   "in-graph launch gap)"},
                       "largest_lanes_4MiB": ({"avg_launch_us": us_b, "algorithmic_bytes_per_launch": by_b,
                                               "achieved_GBps": by_b / (us_b * 1e-6) / 1e9} if big else None),
                       "by_lane_size_serial": by_size,
                       "deployed_node_trace": node_trace,
                       "peak_source": peak_src}
    ex_copy.close()

    # ---------------- C3: GPT-2-small decoder chain (T = 128, 12 layers), tcgen05 GEMM nodes
    try:
        out["decoder_c3"] = bench_decoder(torch, cgx, runner, wl, stream, dev, peaks)
    except Exception as exn:  # noqa: BLE001
        out["decoder_c3"] = {"error": str(exn)}
    # ---------------- NEXT-4: training-shaped chain (fwd + bwd + SGD of 6 GPT-2 MLP blocks)
    try:
        out["training_chain"] = bench_training(torch, cgx, runner, wl, stream, dev)
    except Exception as exn:  # noqa: BLE001
        out["training_chain"] = {"error": str(exn)}

    # ---------------- copy kernel at the C4 1 GiB point (HBM roofline target >= 80%)
    try:
        S = 1 << 30
        c4 = wl.c4_chain(S, window_mode=True)
        c4_chain = runner.Chain(c4, runner.upload_statics(c4, wl.static_values(c4), dev))
        exc = c4_chain.exec("COPY", stream=stream)
        srcs = []
        for s in c4.externals():
            t = torch.empty(S // 4, dtype=torch.float32, device=dev)
            cgx.fill_uniform_f32(t.data_ptr(), S // 4, sm.SEED, sm.stream_id(c4.index(s.name), 0), sh)
            srcs.append(t)
        arr = cgx.ptr_array([t.data_ptr() for t in srcs])
        ds = []
        for i in range(12):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            with torch.cuda.stream(stream):
                a.record(stream)
                LIB.cgx_bind(exc.handle, arr, 3)
                b.record(stream)
            b.synchronize()
            if i >= 2:
                ds.append(a.elapsed_time(b) * 1e-3)
        dt = statistics.median(ds)
        gbs = 2 * 3 * S / dt / 1e9
        out["copy_kernel"] = {"workload": "C4 1 GiB x 3 inputs, COPY arm rebinding (multi-tensor copy)",
                              "bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                              "frac": gbs / hbm, "frac_of_8TBps_nominal": gbs / 8000.0,
                              "us": dt * 1e6, "algorithmic_bytes": 6 * S, "peak_source": peak_src}
        c4_chain.close()
        del srcs
        torch.cuda.empty_cache()
    except Exception as exn:  # noqa: BLE001
        out["copy_kernel"] = {"error": str(exn)}

    # ---------------- CPU oracle baseline (bounded sample) and the other configs' oracle timings
    try:
        out["oracle_timings"] = run_oracle_timings()
    except Exception as exn:  # noqa: BLE001
        out["oracle_timings"] = {"error": str(exn)}
    n, dt = run_oracle_replays(spec, args.cpu_budget_s)
    out["cpu_baseline"] = {"value": n / dt, "unit": "iters/s", "cores": 1, "kind": "oracle",
                           "sample": f"{n} C2 replays (INDIRECT bind + replay, NumPy f32/f64, "
                                     f"threadpoolctl 1 thread) on {os.cpu_count()}-core host "
                                     f"{cpu_info()}"}
    return out


def bench_training(torch, cgx, runner, wl, stream, dev):
    """Training-shaped chain: one step = forward + loss gradient + backward +
    in-place SGD of 6 GPT-2-shaped MLP blocks (T=128, bf16), fresh X / target every step. Per arm:
    µs per step and the rebinding Δ against the same exec without binding."""
    spec = wl.mlp_train_chain(n_blocks=6)
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    f0, l0 = spec.segments[0]
    f1, l1 = spec.segments[1]
    sets = [runner.upload_externals(spec, wl.external_values(spec, r), dev) for r in range(4)]
    ptrs = [cgx.ptr_array([t[n].data_ptr() for n in chain.ext_names]) for t in sets]
    LIB = cgx.LIB
    init = chain.exec("EAGER", stream=stream, first_node=f0, n_nodes=l0 - f0 + 1)
    LIB.cgx_bind(init.handle, ptrs[0], 2)
    LIB.cgx_launch(init.handle)

    def timed(h, n, bind=True):
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            e0.record(stream)
            for i in range(n):
                if bind:
                    LIB.cgx_bind(h, ptrs[i % 4], 2)
                LIB.cgx_launch(h)
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / n)
        return best
    res = {"workload": "6 GPT-2 MLP blocks (d 768, d_ff 3072, T 128, bf16): forward, MSE gradient, backward "
                       "(TRANSPOSE + tcgen05 GEMMs + GELU_BWD), in-place SGD; fresh X / target per step",
           "kernels_per_step": l1 - f1 + 1, "us_per_step": {}, "rebind_delta_us": {}}
    # slow path: the DAG capture's stream count measured on this chain (as for C2)
    best_s, tune = cgx.tune_graph_streams(chain.handle, "INDIRECT", stream.cuda_stream,
                                          [[t[n].data_ptr() for n in chain.ext_names] for t in sets],
                                          candidates=(8, 12, 16, 20, 24, 32), reps=30, transport="ROOT_PARAMS",
                                          first_node=f1, n_nodes=l1 - f1 + 1)
    res["graph_streams"] = best_s
    res["graph_streams_tuning_us"] = {str(k): round(v, 1) for k, v in tune.items()}
    for name, mode, xp in (("indirect_root_params", "INDIRECT", "ROOT_PARAMS"), ("copy", "COPY", "DEFAULT"),
                           ("setparams", "SETPARAMS", "DEFAULT"), ("eager", "EAGER", "DEFAULT")):
        ex = chain.exec(mode, stream=stream, transport=xp, first_node=f1, n_nodes=l1 - f1 + 1,
                        graph_streams=best_s if mode != "EAGER" else 0)
        for i in range(5):
            LIB.cgx_bind(ex.handle, ptrs[i % 4], 2)
            LIB.cgx_launch(ex.handle)
        n = 100 if mode != "EAGER" else 30
        us = timed(ex.handle, n)
        res["us_per_step"][name] = us
        if mode != "EAGER":
            res["rebind_delta_us"][name] = us - timed(ex.handle, n, bind=False)
        ex.close()
    res["steps_per_s_indirect"] = 1e6 / res["us_per_step"]["indirect_root_params"]
    chain.close()
    return res


def bench_decoder(torch, cgx, runner, wl, stream, dev, peaks):
    """C3: per-replay µs per arm, tokens/s, per-GEMM device time vs rooflines."""
    T, L = 128, 12
    spec = wl.c3_chain(T=T, n_layers=L)
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
    ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
    LIB = cgx.LIB

    def timed(h, n, bind=True):
        for i in range(5):
            if bind:
                LIB.cgx_bind(h, ptrs[i % 4], 1)
            LIB.cgx_launch(h)
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            e0.record(stream)
            for i in range(n):
                if bind and LIB.cgx_bind(h, ptrs[i % 4], 1):
                    raise cgx.CgxError(1, "bind", cgx.last_error())
                if LIB.cgx_launch(h):
                    raise cgx.CgxError(1, "launch", cgx.last_error())
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / n)
        return best
    res = {"workload": "C3: GPT-2-small decoder, 12 layers, T=128, bf16, 108 kernels, fresh x per replay"}
    exc = chain.exec("COPY", stream=stream)
    timed(exc.handle, 5)
    base = timed(exc.handle, 300, bind=False)
    arms = {"graph_no_rebind": base}
    for name, mode, xp in (("copy", "COPY", "DEFAULT"), ("indirect_first_node", "INDIRECT", "FIRST_NODE"),
                           ("indirect_root_params", "INDIRECT", "ROOT_PARAMS"),
                           ("setparams", "SETPARAMS", "DEFAULT"), ("eager", "EAGER", "DEFAULT")):
        ex = exc if mode == "COPY" else chain.exec(mode, stream=stream, transport=xp)
        arms[name] = timed(ex.handle, 300 if mode != "EAGER" else 50)
        if ex is not exc:
            ex.close()
    # capture-time ADD -> LAYERNORM fusion (cgx_exec_opts.fuse): 85 launches for the
    # 108 nodes, every node output still written (bit-identical, test_c3_fused_add_layernorm)
    for name, xp in (("indirect_first_node_fused_add_ln", "FIRST_NODE"), ("indirect_root_params_fused_add_ln", "ROOT_PARAMS")):
        try:
            exf = chain.exec("INDIRECT", stream=stream, transport=xp, fuse=cgx.FUSE_ADD_LN)
            arms[name] = timed(exf.handle, 300)
            exf.close()
        except Exception as exn:  # noqa: BLE001
            arms[name] = str(exn)
    # the same chain as ONE persistent launch (exec option megakernel): measured beside
    # the per-node graph, not deployed (it replays slower: grid barriers ~1.8 us x 84 stages)
    try:
        exm = chain.exec("INDIRECT", stream=stream, megakernel=True)
        arms["megakernel_indirect"] = timed(exm.handle, 300)
        exm.close()
    except Exception as exn:  # noqa: BLE001
        arms["megakernel_indirect"] = str(exn)
    exc.close()
    res["us_per_replay"] = arms
    res["tokens_per_s_indirect"] = T * 1e6 / arms["indirect_first_node"]
    # the T = 1 decode variant (SURVEY §8(a) a7 "T=1 uses swap-AB or CUDA cores"): small-M GEMV path
    try:
        dspec = wl.c3_chain(T=1, n_layers=L)
        dchain = runner.Chain(dspec, runner.upload_statics(dspec, wl.static_values(dspec), dev))
        dxs = [runner.host_to_device(wl.slot_values(dspec, "x", r), "bf16", dev) for r in range(4)]
        dptrs = [cgx.ptr_array([x.data_ptr()]) for x in dxs]
        dex = dchain.exec("INDIRECT", stream=stream, transport="FIRST_NODE")
        for i in range(20):
            LIB.cgx_bind(dex.handle, dptrs[i % 4], 1)
            LIB.cgx_launch(dex.handle)
        best_d = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            e0.record(stream)
            for i in range(300):
                LIB.cgx_bind(dex.handle, dptrs[i % 4], 1)
                LIB.cgx_launch(dex.handle)
            e1.record(stream)
            e1.synchronize()
            best_d = min(best_d, e0.elapsed_time(e1) * 1e3 / 300)
        # the same decode chain with capture-time fusions (85 launches each): ADD -> LAYERNORM, and
        # LAYERNORM folded into its GEMV consumer (the GEMV computes the row statistics itself)
        best_f = {}
        for nm_, fz in (("fused_add_ln", cgx.FUSE_ADD_LN), ("ln_folded", cgx.FUSE_LN_GEMM)):
            dexf = dchain.exec("INDIRECT", stream=stream, transport="FIRST_NODE", fuse=fz)
            for i in range(20):
                LIB.cgx_bind(dexf.handle, dptrs[i % 4], 1)
                LIB.cgx_launch(dexf.handle)
            bf_ = 1e30
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                stream.synchronize()
                e0.record(stream)
                for i in range(300):
                    LIB.cgx_bind(dexf.handle, dptrs[i % 4], 1)
                    LIB.cgx_launch(dexf.handle)
                e1.record(stream)
                e1.synchronize()
                bf_ = min(bf_, e0.elapsed_time(e1) * 1e3 / 300)
            best_f[nm_] = bf_
            dexf.close()
        dchain.close()
        # the fused-residual decode chain (84 nodes) with the LayerNorms folded (61 launches)
        rspec = wl.c3_chain(T=1, n_layers=L, fuse_residual=True)
        rchain = runner.Chain(rspec, runner.upload_statics(rspec, wl.static_values(rspec), dev))
        rxs = [runner.host_to_device(wl.slot_values(rspec, "x", r), "bf16", dev) for r in range(4)]
        rptrs = [cgx.ptr_array([x.data_ptr()]) for x in rxs]
        # (+ the T = 1 attention folded into its O-proj GEMV, fuse = CGX_FUSE_ATTN_GEMM: 50 launches)
        best_rf, launches_rf = {}, {}
        for nm_, fz in (("ln", cgx.FUSE_LN_GEMM), ("ln_attn", cgx.FUSE_LN_GEMM | cgx.FUSE_ATTN_GEMM)):
            rex = rchain.exec("INDIRECT", stream=stream, transport="FIRST_NODE", fuse=fz)
            for i in range(20):
                LIB.cgx_bind(rex.handle, rptrs[i % 4], 1)
                LIB.cgx_launch(rex.handle)
            bf_ = 1e30
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                stream.synchronize()
                e0.record(stream)
                for i in range(300):
                    LIB.cgx_bind(rex.handle, rptrs[i % 4], 1)
                    LIB.cgx_launch(rex.handle)
                e1.record(stream)
                e1.synchronize()
                bf_ = min(bf_, e0.elapsed_time(e1) * 1e3 / 300)
            best_rf[nm_], launches_rf[nm_] = bf_, rex.stats()["kernels_per_replay"]
            rex.close()
        best_r, r_launches = best_rf["ln"], launches_rf["ln"]
        best_ra = best_rf["ln_attn"]
        rchain.close()
        res["decode_t1"] = {"kernels_per_replay": len(dspec.nodes), "us_per_replay": best_d,
                            "us_per_replay_fused_add_ln": best_f["fused_add_ln"],
                            "us_per_replay_ln_folded": best_f["ln_folded"],
                            "tokens_per_s": 1e6 / best_d,
                            "weight_GBps": 12 * 14.16e6 / (best_d * 1e-6) / 1e9,
                            "fused_residual_ln_folded": {"kernels_per_replay": r_launches, "us_per_replay": best_r,
                                                         "tokens_per_s": 1e6 / best_r,
                                                         "weight_GBps": 12 * 14.16e6 / (best_r * 1e-6) / 1e9},
                            "fused_residual_ln_attn_folded": {"kernels_per_replay": launches_rf["ln_attn"],
                                                              "us_per_replay": best_ra, "tokens_per_s": 1e6 / best_ra,
                                                              "weight_GBps": 12 * 14.16e6 / (best_ra * 1e-6) / 1e9,
                                                              "hbm_frac": 12 * 14.16e6 / (best_ra * 1e-6) / 1e9 / peaks.get("hbm_gbs", 6650.0)},
                            "note": "12 layers, T = 1: GEMM nodes on the small-M weight-stream path "
                                    "(k_gemv_bf16); 170 MB of weights per replay"}
    except Exception as exn:  # noqa: BLE001
        res["decode_t1"] = {"error": str(exn)}
    # the same decoder with the residual adds fused into the O-proj / FC2 GEMM epilogues (SURVEY
    # §8(a) allows it): 84 kernels instead of 108
    try:
        fspec = wl.c3_chain(T=T, n_layers=L, fuse_residual=True)
        fchain = runner.Chain(fspec, runner.upload_statics(fspec, wl.static_values(fspec), dev))
        fex = fchain.exec("INDIRECT", stream=stream, transport="FIRST_NODE")
        fus = timed(fex.handle, 300)
        res["fused_residual"] = {"kernels_per_replay": len(fspec.nodes), "us_per_replay": fus,
                                 "tokens_per_s": T * 1e6 / fus}
        # + LayerNorm folded into its consumer GEMM (fuse = CGX_FUSE_LN_GEMM): 61 launches
        fexl = fchain.exec("INDIRECT", stream=stream, transport="FIRST_NODE", fuse=cgx.FUSE_LN_GEMM)
        ful = timed(fexl.handle, 300)
        res["fused_residual"]["ln_folded"] = {"kernels_per_replay": fexl.stats()["kernels_per_replay"] - 0,
                                              "us_per_replay": ful, "tokens_per_s": T * 1e6 / ful}
        res["best"] = {"arm": "fused residual + LayerNorm folded into its consumer GEMM (INDIRECT, FIRST_NODE)",
                       "us_per_replay": ful, "tokens_per_s": T * 1e6 / ful}
        fexl.close()
        fchain.close()
    except Exception as exn:  # noqa: BLE001
        res["fused_residual"] = {"error": str(exn)}
    res["rebind_delta_us"] = {k: arms[k] - base for k in ("copy", "indirect_first_node", "indirect_root_params", "setparams")}
    bf16_peak = peaks.get("bf16_tflops", 1590.0)
    hbm = peaks.get("hbm_gbs", 6650.0)
    # per-kernel durations: CUPTI records of the same chain captured WITHOUT PDL (with PDL a kernel
    # is resident early and its record includes the wait)
    ex_np = chain.exec("INDIRECT", stream=stream, transport="FIRST_NODE", no_pdl=True)
    arms["indirect_first_node_no_pdl"] = timed(ex_np.handle, 200)
    per = {}
    try:
        from torch.profiler import ProfilerActivity, profile as tprof
        with tprof(activities=[ProfilerActivity.CUDA]) as tp:
            for i in range(5):
                LIB.cgx_bind(ex_np.handle, ptrs[i % 4], 1)
                LIB.cgx_launch(ex_np.handle)
            stream.synchronize()
        for ev in tp.key_averages():
            t_ = getattr(ev, "device_time_total", None)
            if t_ is None:
                t_ = getattr(ev, "cuda_time_total", 0.0)
            if "cgx" in ev.key:
                per[ev.key] = {"launches_per_replay": ev.count / 5, "us_per_launch": t_ / max(1, ev.count),
                               "us_per_replay": t_ / 5}
    except Exception as exn:  # noqa: BLE001
        per = {"error": str(exn)}
    ex_np.close()
    res["per_kernel_cupti_no_pdl"] = per
    g_us = sum(v["us_per_replay"] for k, v in per.items() if "k_gemm" in k) if "error" not in per else None
    fl = 0.0
    wb = 0.0
    for node in spec.nodes:
        if node.op == "GEMM_BF16":
            a_ = node.attrs
            fl += 2.0 * a_["M"] * a_["N"] * a_["K"]
            wb += 2.0 * a_["N"] * a_["K"]
    if g_us:
        res["gemm"] = {"launches_per_replay": sum(1 for n in spec.nodes if n.op == "GEMM_BF16"),
                       "sum_us": g_us, "TFLOPs": fl / (g_us * 1e-6) / 1e12,
                       "frac_of_bf16_peak": fl / (g_us * 1e-6) / 1e12 / bf16_peak,
                       "weight_GBps": wb / (g_us * 1e-6) / 1e9, "frac_of_hbm": wb / (g_us * 1e-6) / 1e9 / hbm,
                       "bound": "latency (M = 128: weight-streaming roofline 14.2 MB/layer at HBM speed "
                                "is ~2.2 us/layer; each GEMM node runs ~5-8 us)",
                       "timing": "CUPTI kernel durations, no-PDL capture of the same chain"}
    # the same GEMM nodes timed INSIDE the deployed replay (node-timeline stamps, 20 replays):
    # work = last CTA exit - first CTA past its griddepcontrol.wait (the per-node hand-over gap is
    # reported separately: first ready - the previous node's last exit)
    try:
        os.environ["CGX_NODE_TRACE"] = "1"
        ext_ = chain.exec("INDIRECT", stream=stream, transport="FIRST_NODE")
        os.environ.pop("CGX_NODE_TRACE", None)
        K_ = len(spec.nodes)
        for i in range(10):
            LIB.cgx_bind(ext_.handle, ptrs[i % 4], 1)
            LIB.cgx_launch(ext_.handle)
        cgx.node_trace(ext_.handle, K_)
        per_op = {}
        for i in range(20):
            LIB.cgx_bind(ext_.handle, ptrs[i % 4], 1)
            LIB.cgx_launch(ext_.handle)
            tr = cgx.node_trace(ext_.handle, K_)
            for k, n in enumerate(spec.nodes):
                key = n.op if n.op != "GEMM_BF16" else f"GEMM {n.attrs['N']}x{n.attrs['K']}"
                d_ = per_op.setdefault(key, {"work": [], "gap": []})
                d_["work"].append((tr[k][2] - tr[k][1]) * 1e-3)
                if k > 0:
                    d_["gap"].append((tr[k][1] - tr[k - 1][2]) * 1e-3)
        ext_.close()
        g_work = sum(statistics.median(v["work"]) * sum(1 for n in spec.nodes if n.op == "GEMM_BF16" and
                     f"GEMM {n.attrs['N']}x{n.attrs['K']}" == k_) for k_, v in per_op.items() if k_.startswith("GEMM"))
        res["deployed_node_trace"] = {
            "per_op_median_us": {k_: {"work": statistics.median(v["work"]),
                                      "gap": statistics.median(v["gap"]) if v["gap"] else None}
                                 for k_, v in per_op.items()},
            "gemm_work_sum_us": g_work, "gemm_weight_GBps_work": wb / (g_work * 1e-6) / 1e9,
            "gemm_frac_of_hbm_work": wb / (g_work * 1e-6) / 1e9 / hbm,
            "timing": "node-timeline stamps inside the deployed INDIRECT replay (FIRST_NODE), 20 replays; "
                      "work = last CTA exit - first CTA past its wait, gap = first ready - previous exit"}
    except Exception as exn:  # noqa: BLE001
        os.environ.pop("CGX_NODE_TRACE", None)
        res["deployed_node_trace"] = {"error": str(exn)}
    chain.close()
    return res


if __name__ == "__main__":
    main()
