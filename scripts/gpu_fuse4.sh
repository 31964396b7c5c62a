cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python scripts/sweep_c3_knobs.py "" "CGX_GEMM_LN_RUNTIME=1" 2>&1
done
