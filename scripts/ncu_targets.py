"""Short, deterministic launch sequences for `ncu --set full` captures (one GPU, no warm-up loop).

  python scripts/ncu_targets.py replay   # one C2 INDIRECT (FIRST_NODE) replay: 200 kernels
  python scripts/ncu_targets.py copy     # one COPY-arm bind at the C4 1 GiB point (copy kernel)
  python scripts/ncu_targets.py gemm     # one C3 (T=128, 1 layer) INDIRECT replay (tcgen05 GEMMs)
  python scripts/ncu_targets.py mega     # one C3 (T=128, 12 layers) megakernel launch (persistent executor)
  python scripts/ncu_targets.py gemm_fold  # one C3 (T=128, 2 layers, fused residual) replay with the
                                           # LayerNorms folded into their consumer GEMMs
  python scripts/ncu_targets.py replay_nopdl  # one C2 INDIRECT replay captured without PDL (the
                                              # roofline's sub-graph configuration)
  python scripts/ncu_targets.py decode     # one T = 1 decode replay (2 layers, fused residual, LN and
                                           # attention folded into their GEMV consumers)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import splitmix as sm  # noqa: E402
from synth import workloads as wl  # noqa: E402


def fill(spec, dev, sh, rep=0):
    ts = []
    for s in spec.externals():
        if s.dtype == "f32":
            t = torch.empty(s.nelems, dtype=torch.float32, device=dev)
            cgx.fill_uniform_f32(t.data_ptr(), s.nelems, sm.SEED, sm.stream_id(spec.index(s.name), rep), sh)
        else:
            t = runner.host_to_device(wl.slot_values(spec, s.name, rep), "bf16", dev)
        ts.append(t)
    return ts


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "replay"
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    if what == "copy":
        S = 1 << 30
        spec = wl.c4_chain(S, window_mode=True)
        mode, xp = "COPY", "DEFAULT"
    elif what == "gemm":
        spec = wl.c3_chain(T=128, n_layers=1)
        mode, xp = "INDIRECT", "FIRST_NODE"
    elif what == "gemm_fold":
        spec = wl.c3_chain(T=128, n_layers=2, fuse_residual=True)
        mode, xp = "INDIRECT", "FIRST_NODE"
    elif what == "decode":
        spec = wl.c3_chain(T=1, n_layers=2, fuse_residual=True)
        mode, xp = "INDIRECT", "FIRST_NODE"
    elif what == "mega":
        spec = wl.c3_chain(T=128, n_layers=12)
        mode, xp = "INDIRECT", "ROOT_PARAMS"
    else:
        spec = wl.c2_chain()
        mode, xp = "INDIRECT", "FIRST_NODE"
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    ex = chain.exec(mode, transport=xp, no_pdl=(what == "replay_nopdl"), megakernel=(what == "mega"),
                    fuse=cgx.FUSE_LN_GEMM if what == "gemm_fold" else
                    cgx.FUSE_LN_GEMM | cgx.FUSE_ATTN_GEMM if what == "decode" else 0)
    ts = fill(spec, dev, sh)
    torch.cuda.synchronize()
    ex.bind_ptrs([t.data_ptr() for t in ts])
    if what != "copy":
        ex.launch()
    torch.cuda.synchronize()
    chain.close()


if __name__ == "__main__":
    main()
