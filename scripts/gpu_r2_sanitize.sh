#!/bin/bash
# compute-sanitizer over the round-2 decoder changes: K-split GEMV (+ folded LN, named barriers),
# the staged split-K GEMM epilogue with relaxed cluster arrives, attention single-chunk tiles
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/memcheck
K='test_fused_ln_gemv_k_slices or test_c3_decode_fused_ln_gemv or test_c3_fused_ln_gemm or test_gemm_split_tilings_integer_exact or test_gemm_small_m_paths or test_attention'
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_decoder.py -x -q -m gpu -k "$K" -p no:cacheprovider > gpurun_out/memcheck/r2b_memcheck.txt 2>&1
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest tests/test_gpu_decoder.py -x -q -m gpu -k "test_fused_ln_gemv_k_slices or test_c3_fused_ln_gemm or test_attention" -p no:cacheprovider > gpurun_out/memcheck/r2b_racecheck.txt 2>&1
tail -3 gpurun_out/memcheck/r2b_memcheck.txt; tail -3 gpurun_out/memcheck/r2b_racecheck.txt
