"""The tcgen05 GEMM kernel on a large, compute-bound shape (evidence of tensor-pipe throughput when
the shape allows it; the decoder's M = 128 nodes are latency-bound): out[M,N] = A[M,K] W[N,K]^T in
bf16 through the C ABI (one GEMM node), device time per launch from CUDA events, TFLOP/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth.workloads import ChainSpec, NodeSpec, SlotSpec  # noqa: E402

dev = torch.device("cuda:0")
for (M, N, K) in ((4096, 4096, 4096), (8192, 8192, 4096)):
    for bn in ("32", "64", "128"):
        os.environ["CGX_GEMM_TILING"] = f"{N}x{K}={bn}/1"
        slots = [SlotSpec("a", "internal", "bf16", M * K), SlotSpec("w", "static", "bf16", N * K, "weight"),
                 SlotSpec("b", "static", "bf16", N, "bias"), SlotSpec("y", "internal", "bf16", M * N)]
        spec = ChainSpec("big", slots, [NodeSpec("GEMM_BF16", ("a", "w", "b"), "y",
                                                 {"M": M, "N": N, "K": K, "bias": False, "gelu": False})], [(0, 0)])
        statics = {"w": torch.randn(N * K, device=dev).to(torch.bfloat16) * 0.02,
                   "b": torch.zeros(N, device=dev, dtype=torch.bfloat16)}
        chain = runner.Chain(spec, statics)
        ex = chain.exec("EAGER")
        ex.bind_ptrs([])                     # no EXTERNAL slot
        for _ in range(3):
            cgx.launch(ex.handle)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            cgx.launch(ex.handle)
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / n
        print(json.dumps({"M": M, "N": N, "K": K, "BN": int(bn), "us": us, "TFLOPs": 2 * M * N * K / (us * 1e-6) / 1e12}),
              flush=True)
        chain.close()
