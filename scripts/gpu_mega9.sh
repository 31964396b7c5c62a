cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=3000 CGX_MEGA_BAR=3
for ns in 0 200 1000; do
  echo "=== sleep $ns"
  CGX_MEGA_BAR_NS=$ns timeout 120 python scripts/diag_mega.py 128 12 2>&1 | grep -E "span|stage   [0-7] " | cut -c1-250
done
