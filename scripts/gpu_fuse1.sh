cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decoder.py -q -x -p no:cacheprovider -k "fused_add_layernorm or c3_decoder_chain or layernorm" > gpurun_out/pytest_fuse.txt 2>&1; tail -15 gpurun_out/pytest_fuse.txt
timeout 300 python scripts/sweep_c3_knobs.py "" > gpurun_out/c3_fuse.txt 2>&1; cat gpurun_out/c3_fuse.txt
