#!/bin/bash
# Round-1 evidence run: GPU tests, bench (ours + reference), launch list under ncu, ncu --set full
# captures (C2 lanes, copy kernel, one C3 layer: GEMMs / attention / LN), C4 selector sweep, PI
# latency sweep, launch-cadence microbenchmark, cadence decomposition, H2D ceiling. Every step has
# its own timeout.
cd $GRAFT_REPO_ROOT
nproc > gpurun_out/nproc.txt
timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_final.txt
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 120 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_final.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/bench_ncu_final.log 2>&1
timeout 200 ncu --set full --import-source on --clock-control none --graph-profiling node -k regex:"k_elem_f32|k_reduce" -s 36 -c 3 -o gpurun_out/ncu_c2_final -f python scripts/ncu_targets.py replay > /dev/null 2>&1
timeout 200 ncu --set full --import-source on --clock-control none -k regex:k_copy -c 1 -o gpurun_out/ncu_copy_final -f python scripts/ncu_targets.py copy > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none --graph-profiling node -k regex:"k_attention|k_layernorm|k_elem_bf16|k_gemm" -c 9 -o gpurun_out/ncu_c3layer_final -f python scripts/ncu_targets.py gemm > /dev/null 2>&1
timeout 240 python scripts/c4_sweep.py window full > gpurun_out/c4_final.log 2>&1
timeout 120 python scripts/pi_sweep.py > gpurun_out/pi_sweep_final.log 2>&1
[ -x scripts/launch_microbench ] && timeout 120 ./scripts/launch_microbench > gpurun_out/launch_microbench.txt 2>&1
[ -x scripts/dag_microbench ] && timeout 120 ./scripts/dag_microbench > gpurun_out/dag_microbench.txt 2>&1
timeout 600 python scripts/diag_cadence_split.py graph > gpurun_out/dag_sweep.txt 2>&1
timeout 300 python scripts/diag_cadence_split.py > gpurun_out/cadence_split.txt 2>&1
timeout 120 python scripts/diag_h2d.py > gpurun_out/h2d.txt 2>&1
timeout 300 python scripts/diag_decode.py > gpurun_out/decode.txt 2>&1
timeout 300 python scripts/diag_devloop.py > gpurun_out/devloop.txt 2>&1
timeout 300 python scripts/diag_training_arms.py > gpurun_out/training_arms.txt 2>&1
timeout 300 python scripts/diag_concurrent_graphs.py > gpurun_out/concurrent_graphs.txt 2>&1
timeout 200 ncu --graph-profiling graph --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv python scripts/ncu_targets.py replay > gpurun_out/ncu_graph_replay.csv 2>&1
ls -la gpurun_out | tail -30
