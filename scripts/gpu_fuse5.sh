cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=5000
timeout 1200 python -m pytest tests/test_gpu_decoder.py tests/test_gpu_training.py tests/test_gpu_peer_allreduce.py -q -x -p no:cacheprovider > gpurun_out/pytest_fuse5.txt 2>&1; tail -3 gpurun_out/pytest_fuse5.txt
timeout 300 python scripts/diag_c3_timeline.py 128 12 --ln-gemm > gpurun_out/c3_tl_lngemm.txt 2>&1; grep -A12 "^op" gpurun_out/c3_tl_lngemm.txt; head -1 gpurun_out/c3_tl_lngemm.txt
