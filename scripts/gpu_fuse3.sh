cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_decoder.py -q -x -p no:cacheprovider -k "fused_ln_gemm" > gpurun_out/pytest_fuse3.txt 2>&1; tail -25 gpurun_out/pytest_fuse3.txt
timeout 300 python scripts/sweep_c3_knobs.py "" > gpurun_out/c3_fuse4.txt 2>&1; cat gpurun_out/c3_fuse4.txt
timeout 300 python scripts/diag_c3_timeline.py 128 12 --ln-gemm > gpurun_out/c3_tl_lngemm.txt 2>&1; grep -A12 "^op" gpurun_out/c3_tl_lngemm.txt; head -3 gpurun_out/c3_tl_lngemm.txt
