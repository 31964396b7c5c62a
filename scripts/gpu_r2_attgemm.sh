cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decoder.py -m gpu -q -x -k "fused_attn_gemm" 2>&1 | tail -25
timeout 300 python scripts/ab_attn_gemm.py 128 > gpurun_out/ab_attn_gemm.txt 2>&1; tail -3 gpurun_out/ab_attn_gemm.txt
timeout 300 python scripts/diag_gemm.py --fused --attn > gpurun_out/gemm_att_trace.txt 2>&1; grep -A18 "768x768" gpurun_out/gemm_att_trace.txt | head -19
timeout 300 python scripts/diag_c3_timeline.py 128 12 --fuse --ln-gemm --attn-gemm > gpurun_out/c3_tl_attn_gemm.txt 2>&1; head -1 gpurun_out/c3_tl_attn_gemm.txt; tail -7 gpurun_out/c3_tl_attn_gemm.txt
