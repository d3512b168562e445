#!/bin/bash
# ncu --set full (with source) of the cfg2 sweep's CTA allocator (all plans in one launch)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
O=gpurun_out/${TAG:-allocta}
mkdir -p $O
timeout 300 python tools/prof_sweep.py > $O/plain.log 2>&1 && \
timeout 600 ncu --clock-control none --import-source on --set full -k regex:alloc_ -s 1 -c 1 \
  -o $O/alloc_cta -f python tools/prof_sweep.py > $O/ncu.log 2>&1
echo "rc=$?"
ncu -i $O/alloc_cta.ncu-rep --page raw --csv > $O/alloc_cta_raw.csv 2>/dev/null
