"""Host<->device copy bandwidth on the box (the e2e leg's ceiling): pinned H2D / D2H GB/s vs size,
one copy at a time and split over 2 / 4 concurrent streams."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

dev = torch.device("cuda:0")
res = {}
for mb in (1, 4, 16, 37.7, 128, 512):
    n = int(mb * (1 << 20)) // 256 * 256
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    row = {}
    for nst in (1, 2, 4):
        streams = [torch.cuda.Stream(device=dev) for _ in range(nst)]
        chunk = (n // nst) // 256 * 256
        for direction in ("h2d", "d2h"):
            best = 0.0
            for _ in range(5):
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                for i, s in enumerate(streams):
                    s.wait_event(e0)
                    lo = i * chunk
                    hi = n if i == nst - 1 else lo + chunk
                    with torch.cuda.stream(s):
                        if direction == "h2d":
                            d[lo:hi].copy_(h[lo:hi], non_blocking=True)
                        else:
                            h[lo:hi].copy_(d[lo:hi], non_blocking=True)
                for s in streams:
                    torch.cuda.current_stream().wait_stream(s)
                e1.record()
                e1.synchronize()
                best = max(best, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
            row[f"{direction}_streams{nst}_GBps"] = round(best, 1)
    res[f"{mb}MB"] = row
    print(json.dumps({f"{mb}MB": row}), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/h2d.json", "w"), indent=1)
