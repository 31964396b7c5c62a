cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decoder.py -q -x -p no:cacheprovider -k "layernorm or c3_decoder_chain or fused_add" > gpurun_out/pytest_ln3.txt 2>&1; tail -3 gpurun_out/pytest_ln3.txt
timeout 300 python scripts/sweep_c3_knobs.py "" > gpurun_out/c3_ln3.txt 2>&1; cat gpurun_out/c3_ln3.txt
