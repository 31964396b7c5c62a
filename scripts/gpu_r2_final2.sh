#!/bin/bash
# round-2 final evidence run (after the decode attention fold, attention Q-load / merge changes and
# the O-proj S = 3 tiling): full GPU suite, smoke, bench (ours + reference), ncu launch list, ncu
# --set full of the C2 lanes, the C3 GEMMs + attention (LN-folded chain) and the decode GEMVs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; tail -c 300 gpurun_out/bench_ours.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --graph-profiling node -k regex:"k_elem_f32|k_reduce" \
  -s 36 -c 3 -o gpurun_out/ncu_c2 -f python scripts/ncu_targets.py replay > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --graph-profiling node -k regex:"k_gemm|k_attention" -c 6 \
  -o gpurun_out/ncu_fold -f python scripts/ncu_targets.py gemm_fold > gpurun_out/ncu_fold.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --graph-profiling node -k regex:"k_gemv" -c 4 \
  -o gpurun_out/ncu_decode -f python scripts/ncu_targets.py decode > gpurun_out/ncu_decode.log 2>&1
ls -la gpurun_out/*.ncu-rep
