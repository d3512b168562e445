#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py -> gpurun_out/sanitizer/
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_cases.py ida > /dev/null 2>&1  # warm-up (page-in)
for c in ${CASES:-alloc_cluster2 alloc_cluster16 umma ida sweep denoise}; do
  for t in memcheck racecheck synccheck; do
    extra=""
    [ "$t" = "memcheck" ] && extra="--leak-check no"
    timeout 900 $CS --tool $t $extra --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/sanitizer/${c}_${t}.log 2>&1
    echo "$c $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard|case ok' gpurun_out/sanitizer/${c}_${t}.log | tr '\n' ' ')"
  done
done
