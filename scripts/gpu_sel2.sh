cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_chain.py tests/test_gpu_segments.py -q -x -p no:cacheprovider -k "profile or segment" > gpurun_out/pytest_sel.txt 2>&1; tail -15 gpurun_out/pytest_sel.txt
timeout 1500 python scripts/c4_sweep.py --sweeps 3 > gpurun_out/c4_sweep.log 2>&1; tail -1 gpurun_out/c4_sweep.log
timeout 900 python scripts/sweep_c3_knobs.py "" "CGX_ATTN_WARPS=8" "CGX_LN_WARPS=1" "CGX_LN_WARPS=2" "CGX_LN_WARPS=8" "CGX_ATTN_WARPS=8;CGX_LN_WARPS=2" > gpurun_out/c3_knobs.txt 2>&1; cat gpurun_out/c3_knobs.txt
