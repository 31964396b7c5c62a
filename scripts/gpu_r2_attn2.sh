cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decoder.py tests/test_gpu_mega.py -m gpu -q -x 2>&1 | tail -3
timeout 300 python scripts/diag_attn_cta.py > gpurun_out/attn_cta_bulk.txt 2>&1; tail -14 gpurun_out/attn_cta_bulk.txt
timeout 300 python scripts/diag_c3_timeline.py 128 12 --fuse --ln-gemm > gpurun_out/c3_tl_attn_bulk.txt 2>&1; head -1 gpurun_out/c3_tl_attn_bulk.txt; tail -8 gpurun_out/c3_tl_attn_bulk.txt
