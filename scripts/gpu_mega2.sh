cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=3000
for cfg in "0 0" "0 200" "1 0" "1 100" "2 0" "2 100" "0 500"; do
  set -- $cfg
  echo "=== bar_mode $1 sleep $2" 
  CGX_MEGA_BAR=$1 CGX_MEGA_BAR_NS=$2 timeout 120 python scripts/diag_mega.py 128 12 2>&1 | grep -E "span|mega_us|stage   [1-4] "
done
