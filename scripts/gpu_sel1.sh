cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_chain.py tests/test_gpu_segments.py -q -x -p no:cacheprovider -k "profile or segment" > gpurun_out/pytest_sel.txt 2>&1; tail -15 gpurun_out/pytest_sel.txt
timeout 1500 python scripts/c4_sweep.py --sweeps 3 > gpurun_out/c4_sweep.log 2>&1; tail -2 gpurun_out/c4_sweep.log
