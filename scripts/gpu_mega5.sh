cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=3000
for m in 1 33 17 49 48; do
  echo "=== bar_mode $m"
  CGX_MEGA_BAR=$m timeout 120 python scripts/diag_mega.py 128 12 2>&1 | grep -E "span|mega_us|stage   [1-4] " | cut -c1-250
  CGX_MEGA_BAR=$m timeout 300 python -m pytest tests/test_gpu_mega.py -q -x -p no:cacheprovider -k "c3_chain" 2>&1 | tail -1
done
