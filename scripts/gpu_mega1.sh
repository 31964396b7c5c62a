cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=3000
timeout 180 python scripts/diag_mega.py 128 1 > gpurun_out/mega_d1.txt 2>&1; echo "rc=$?" >> gpurun_out/mega_d1.txt; tail -20 gpurun_out/mega_d1.txt
timeout 180 python scripts/diag_mega.py 128 12 > gpurun_out/mega_d12.txt 2>&1; echo "rc=$?" >> gpurun_out/mega_d12.txt; tail -20 gpurun_out/mega_d12.txt
timeout 600 python -m pytest tests/test_gpu_mega.py -q -x -p no:cacheprovider > gpurun_out/pytest_mega.txt 2>&1; tail -30 gpurun_out/pytest_mega.txt
