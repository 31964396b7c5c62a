cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=3000
timeout 600 python -m pytest tests/test_gpu_mega.py -q -x -p no:cacheprovider > gpurun_out/pytest_mega.txt 2>&1; tail -5 gpurun_out/pytest_mega.txt
for cfg in "1 0" "0 0" "0 300"; do
  set -- $cfg
  echo "=== bar_mode $1 sleep $2"
  CGX_MEGA_BAR=$1 CGX_MEGA_BAR_NS=$2 timeout 120 python scripts/diag_mega.py 128 12 2>&1 | grep -E "span|mega_us|stage   [0-9] "
done
