"""Pick the decoder GEMM tilings on the real objective: the deployed C3 replay (12 layers, T=128,
INDIRECT / FIRST_NODE, PDL) in µs, one subprocess per CGX_GEMM_TILING candidate.

    python scripts/diag_c3_tiling.py            # sweep the candidate table below
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import torch
    from paper_2503_19779_b200 import cgx, runner
    from synth import workloads as wl
    dev = torch.device("cuda:0")
    spec = wl.c3_chain(T=128, n_layers=12)
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
    ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
    stream = torch.cuda.current_stream()
    ex = chain.exec("INDIRECT", stream=stream, transport="FIRST_NODE")
    L = cgx.LIB
    for i in range(20):
        L.cgx_bind(ex.handle, ptrs[i % 4], 1)
        L.cgx_launch(ex.handle)
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        e0.record(stream)
        for i in range(200):
            L.cgx_bind(ex.handle, ptrs[i % 4], 1)
            L.cgx_launch(ex.handle)
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / 200)
    print(json.dumps({"us_per_replay": best}))
    ex.close()
    chain.close()
    sys.exit(0)

SHAPES = {"qkv": "2304x768", "o": "768x768", "fc1": "3072x768", "fc2": "768x3072"}
CANDS = {
    "qkv": ["32/1", "32/2", "64/3", "64/4"],
    "o": ["32/3", "32/4", "64/6", "64/8"],
    "fc1": ["32/1", "64/1", "64/4", "32/2"],
    "fc2": ["32/8", "64/6", "64/8", "32/4"],
}


def run(tiling):
    env = dict(os.environ)
    if tiling:
        env["CGX_GEMM_TILING"] = tiling
    r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True, timeout=240)
    try:
        return json.loads(r.stdout.strip().splitlines()[-1])["us_per_replay"]
    except (IndexError, ValueError, KeyError):
        return None


def main():
    base = run(None)
    print(json.dumps({"tiling": "model", "us": base}), flush=True)
    # coordinate descent from the first candidate of each shape
    cur = {k: v[0] for k, v in CANDS.items()}
    for rnd in range(2):
        for k in SHAPES:
            res = {}
            for c in CANDS[k]:
                t = dict(cur, **{k: c})
                s = ",".join(f"{SHAPES[kk]}={vv}" for kk, vv in t.items())
                res[c] = run(s)
                print(json.dumps({"round": rnd, "shape": k, "cand": c, "tiling": s, "us": res[c]}), flush=True)
            ok = {c: u for c, u in res.items() if u}
            if ok:
                cur[k] = min(ok, key=ok.get)
    print(json.dumps({"best": cur}))


if __name__ == "__main__":
    main()
