#!/bin/bash
# ncu --set full of cfg3's B = 8 gather + decode pass and its class allocator
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
O=gpurun_out/${TAG:-cfg3}
mkdir -p $O
timeout 300 python tools/cfg_time.py 3 > $O/plain.log 2>&1 && \
timeout 600 ncu --clock-control none --import-source on --set full -k regex:"sense8" -s 3 -c 1 \
  -o $O/cfg3 -f python tools/cfg_time.py 3 > $O/ncu.log 2>&1
echo "rc=$?"
ncu -i $O/cfg3.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
