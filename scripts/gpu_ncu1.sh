#!/bin/bash
# ncu --set full captures of: the C3 tcgen05 GEMMs (1 layer), the C2 replay's largest-lane ADD/MUL/REDUCE,
# and the COPY-arm copy kernel at 1 GiB. Reports land in gpurun_out/.
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none --graph-profiling node -k regex:k_gemm -c 4 \
  -o gpurun_out/ncu_gemm -f python scripts/ncu_targets.py gemm > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --graph-profiling node -k regex:"k_elem_f32|k_reduce" \
  -s 36 -c 3 -o gpurun_out/ncu_c2 -f python scripts/ncu_targets.py replay > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_copy -c 1 \
  -o gpurun_out/ncu_copy -f python scripts/ncu_targets.py copy > gpurun_out/ncu_copy.log 2>&1
ls -la gpurun_out/*.ncu-rep
