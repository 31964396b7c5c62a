cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=3000
for m in 1 3 19 35 51; do
  echo "=== NULL bar_mode $m"
  CGX_MEGA_NULL=1 CGX_MEGA_BAR=$m timeout 120 python scripts/diag_mega.py 128 12 2>&1 | grep -E "span|stage   [1-3] " | cut -c1-200
done
echo "=== work bar_mode 3"
CGX_MEGA_BAR=3 timeout 120 python scripts/diag_mega.py 128 12 2>&1 | grep -E "span|stage   [0-8] " | cut -c1-250
