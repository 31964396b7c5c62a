#!/bin/bash
# round-2 measurement call: bench (ours + reference), ncu launch list, ncu --set full captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; tail -c 400 gpurun_out/bench_ours.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --graph-profiling node -k regex:"k_elem_f32|k_reduce" \
  -s 36 -c 3 -o gpurun_out/ncu_c2 -f python scripts/ncu_targets.py replay > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --graph-profiling node -k regex:k_gemm -c 4 \
  -o gpurun_out/ncu_gemm -f python scripts/ncu_targets.py gemm > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --graph-profiling node -k regex:k_mega -c 1 \
  -o gpurun_out/ncu_mega -f python scripts/ncu_targets.py mega > gpurun_out/ncu_mega.log 2>&1
ls -la gpurun_out/*.ncu-rep
