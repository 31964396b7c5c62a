cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/memcheck_r2
export CGX_SPIN_TIMEOUT_MS=20000
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_decoder.py -q -x -p no:cacheprovider -k "fused_ln_gemm and 1- or decode_fused_ln_gemv or fused_add_layernorm and 1" > gpurun_out/memcheck_r2/fusion_memcheck.txt 2>&1; echo "fusion memcheck rc=$?" | tee -a gpurun_out/memcheck_r2/fusion_memcheck.txt; tail -4 gpurun_out/memcheck_r2/fusion_memcheck.txt
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python -m pytest tests/test_gpu_decoder.py -q -x -p no:cacheprovider -k "fused_ln_gemm and 128-1" > gpurun_out/memcheck_r2/fusion_racecheck.txt 2>&1; echo "fusion racecheck rc=$?" | tee -a gpurun_out/memcheck_r2/fusion_racecheck.txt; tail -4 gpurun_out/memcheck_r2/fusion_racecheck.txt
