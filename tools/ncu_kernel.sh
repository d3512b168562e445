#!/bin/bash
# ncu --set full (with SASS source counters) of one launch of each kernel regex in $KERNELS
# while running $SCRIPT (default tools/prof_sweep.py) -> gpurun_out/$TAG/<name>_{details,raw,sass}.csv
TAG=${TAG:-kern}
SCRIPT=${SCRIPT:-tools/prof_sweep.py}
KERNELS=${KERNELS:-sense16_kernel alloc_cta}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python $SCRIPT > $O/plain.log 2>&1 || { echo "plain run failed"; tail $O/plain.log; exit 1; }
for k in $KERNELS; do
  timeout 900 ncu --clock-control none --import-source on --set full -k regex:$k -s ${SKIP:-1} -c 1 \
    -o $O/$k -f python $SCRIPT > $O/${k}_ncu.log 2>&1
  echo "$k ncu rc=$?"
  ncu -i $O/$k.ncu-rep --page details --csv > $O/${k}_details.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page source --csv --print-source sass > $O/${k}_sass.csv 2>/dev/null
done
ls -la $O
