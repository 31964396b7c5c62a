cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_decoder.py -q -x -p no:cacheprovider -k "fused_ln_gemm" > gpurun_out/pytest_fuse2.txt 2>&1; tail -25 gpurun_out/pytest_fuse2.txt
