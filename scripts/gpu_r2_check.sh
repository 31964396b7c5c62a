cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python scripts/sweep_c3_knobs.py "" "CGX_LN_WARPS=4" > gpurun_out/c3_knobs2.txt 2>&1; cat gpurun_out/c3_knobs2.txt
timeout 1500 python scripts/c4_sweep.py --sweeps 3 > gpurun_out/c4_sweep.log 2>&1; tail -1 gpurun_out/c4_sweep.log | cut -c1-1500
CGX_BENCH_DEVICE=0 CGX_BENCH_PG=gloo timeout 600 python bench.py --gpus 2 --steps 50 --warmup 5 --no-extras > gpurun_out/bench_2rank.txt 2>&1; tail -c 1500 gpurun_out/bench_2rank.txt
