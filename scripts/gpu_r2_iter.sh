cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python scripts/sweep_gemm_groups.py "" > gpurun_out/r2_sweep_final.txt 2>&1; cat gpurun_out/r2_sweep_final.txt
