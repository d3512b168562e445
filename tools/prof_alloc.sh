#!/bin/bash
# ncu --set full (with source) of the class allocator on cfg4 (64 x 1024 blocks, BBV) and cfg3
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
O=gpurun_out/${TAG:-alloc}
mkdir -p $O
for c in 4 3; do
  timeout 300 python tools/cfg_time.py $c > $O/cfg${c}_plain.log 2>&1 && \
  timeout 600 ncu --clock-control none --import-source on --set full -k regex:alloc_class -s 3 -c 1 \
    -o $O/alloc_cfg$c -f python tools/cfg_time.py $c > $O/cfg${c}_ncu.log 2>&1
  echo "cfg$c rc=$?"
  ncu -i $O/alloc_cfg$c.ncu-rep --page raw --csv > $O/alloc_cfg${c}_raw.csv 2>/dev/null
done
