cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decoder.py -m gpu -q -x -k "attn or decode or fused_ln" 2>&1 | tail -3
timeout 300 python scripts/diag_decode_fuse.py > gpurun_out/decode_attn_fuse.txt 2>&1; cat gpurun_out/decode_attn_fuse.txt | tail -8
timeout 300 python scripts/diag_c3_timeline.py 1 12 --fuse --ln-gemm --attn-gemm > gpurun_out/c3_tl_decode_attn.txt 2>&1; head -1 gpurun_out/c3_tl_decode_attn.txt; tail -8 gpurun_out/c3_tl_decode_attn.txt
