cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_decoder.py -q -x -p no:cacheprovider -k "fused_ln_gemm or decode_fused_ln_gemv or small_m or t1_decode" > gpurun_out/pytest_fuse6.txt 2>&1; tail -25 gpurun_out/pytest_fuse6.txt
