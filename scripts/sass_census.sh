#!/bin/bash
# SASS census of the tensor-core / TMA kernels (profiles/r02/sass_census.txt)
cd "$(dirname "$0")/.." && python -c "from paper_2503_19779_b200 import build; build.build()"
for o in k_gemm k_mega k_chain k_decoder; do
  echo "== $o.o"
  cuobjdump -sass build/cgx/$o.o | awk '/Function :/ {fn=$3} /UTCHMMA|UTCQMMA|UTMALDG|UTMASTG|UBLKCP|LDTM|STTM|UTCBAR|UTCATOMSWS|UTMAPF|HMMA/ {match($0, /(UTCHMMA|UTCQMMA|UTMALDG|UTMASTG|UBLKCP|LDTM|STTM|UTCBAR|UTCATOMSWS|UTMAPF|HMMA)[A-Z0-9._]*/); print fn, substr($0, RSTART, RLENGTH)}' | sort | uniq -c
done
