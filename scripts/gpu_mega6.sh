cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=3000
timeout 300 python -m pytest tests/test_gpu_mega.py -q -x -p no:cacheprovider 2>&1 | tail -3
for m in 1 3 35; do
  echo "=== bar_mode $m"
  CGX_MEGA_BAR=$m timeout 120 python scripts/diag_mega.py 128 12 2>&1 | grep -E "span|mega_us|stage   [0-8] " | cut -c1-250
done
CGX_MEGA_BAR=3 timeout 300 python -m pytest tests/test_gpu_mega.py -q -x -p no:cacheprovider -k c3_chain 2>&1 | tail -1
