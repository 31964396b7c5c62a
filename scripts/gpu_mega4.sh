cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CGX_SPIN_TIMEOUT_MS=3000
timeout 120 python scripts/diag_mega.py 128 12 2>&1 | grep -E "span|mega_us|stage   [0-9] " | cut -c1-300
