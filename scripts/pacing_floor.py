"""Back-to-back replays of tiny graphs (cgx_graph_floor: n no-op kernels, PDL on/off, 20,000
replays between two events): per-replay µs vs n. Shows the launch front end's pacing quantum
(replays of tiny graphs take whole multiples of ~2.05 us)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx  # noqa: E402

stream = torch.cuda.Stream()
res = {}
for pdl in (0, 1):
    for n in (1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 24, 32):
        us = cgx.graph_floor(stream.cuda_stream, n, bool(pdl), 20000)
        res[f"pdl{pdl}_n{n}"] = us
        print(f"pdl={pdl} kernels={n:3d}  {us:8.3f} us per replay  ({us / 2.048:6.2f} x 2.048 us)", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/pacing_floor.json", "w"), indent=1)
