#!/bin/bash
# one GPU call: bench (ours + reference), launch list under ncu
set -x
cd $GRAFT_REPO_ROOT
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err
tail -c 3000 gpurun_out/bench_ours.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-extras > gpurun_out/bench_ncu.log 2>&1
ls -la gpurun_out
