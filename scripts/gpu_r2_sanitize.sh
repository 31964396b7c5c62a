cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/memcheck_r2
export CGX_SPIN_TIMEOUT_MS=20000
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_mega.py -q -x -p no:cacheprovider -k "c3_chain and 1-False or token_counts or gemm_shapes" > gpurun_out/memcheck_r2/mega_memcheck.txt 2>&1; echo "mega memcheck rc=$?" | tee -a gpurun_out/memcheck_r2/mega_memcheck.txt; tail -4 gpurun_out/memcheck_r2/mega_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python -m pytest tests/test_gpu_mega.py -q -x -p no:cacheprovider -k "c3_chain and 1-False" > gpurun_out/memcheck_r2/mega_racecheck.txt 2>&1; echo "mega racecheck rc=$?" | tee -a gpurun_out/memcheck_r2/mega_racecheck.txt; tail -4 gpurun_out/memcheck_r2/mega_racecheck.txt
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_chain.py tests/test_gpu_segments.py -q -x -p no:cacheprovider -k "profile or segment" > gpurun_out/memcheck_r2/selector_memcheck.txt 2>&1; echo "selector memcheck rc=$?" | tee -a gpurun_out/memcheck_r2/selector_memcheck.txt; tail -4 gpurun_out/memcheck_r2/selector_memcheck.txt
timeout 600 python -m pytest tests/test_gpu_chain.py tests/test_gpu_segments.py -q -x -p no:cacheprovider -k "profile or segment" 2>&1 | tail -2
timeout 1500 python scripts/c4_sweep.py --sweeps 3 > gpurun_out/c4_sweep.log 2>&1; tail -1 gpurun_out/c4_sweep.log | cut -c1-1200
