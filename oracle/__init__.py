"""CPU oracle for the CUDA-Graph input-rebinding hot path of arXiv 2503.19779.

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import anything under `oracle/`. The product path
(`paper_2503_19779_b200/`) never imports it, and this package never imports the product path;
the two share only the seeded generators in `synth/`.

Plain, slow, obviously-correct NumPy (float64 unless the method fixes fp32), single-threaded.
Each function cites the PAPER.md (`P:Lnnn`) / SPEC.md (`S:Lnnn`) passage or the SURVEY.md §8(c)
reading it follows. Modules:
  numerics  bf16 round-to-nearest-even from float64 (single rounding)
  ops       O1: per-node definitions (ADD, MUL, SCALE_IMM, COPY, REDUCE_SUM, LAYERNORM,
            GEMM_BF16, ATTN_CAUSAL, ALLREDUCE_SUM)
  chain     O1: eager chain evaluator (and lockstep TP evaluator for ALLREDUCE_SUM)
  capture   O2/O3: recorded-by-value capture and the COPY / INDIRECT / SETPARAMS / STALE
            rebinding semantics
  selector  O4: eager recurrence, graph cost, three-way argmin with fixed tie-break

Parity status: every function is pinned by `-m "not gpu"` tests in tests/test_oracle_*.py
against closed forms, library routines, paper/SPEC worked examples or brute force, except the
absolute microsecond values the selector consumes on B200 ("parity unpinned": the paper
reports none, SURVEY §8(c) last row).
"""
