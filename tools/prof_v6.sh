#!/bin/bash
# r02 v6: ncu --set full (with source) of the current IDA step and the sweep's DD phase-1 and
# payload passes; each ncu run after its own command exited 0 without ncu.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
O=gpurun_out/${TAG:-v6}
mkdir -p $O
timeout 300 python tools/ida_time.py cfg4 --no-check > $O/ida_plain.log 2>&1 && \
timeout 900 ncu --clock-control none --import-source on --set full -k regex:ida_mma_kernel -s 3 -c 1 \
  -o $O/ida -f python tools/ida_time.py cfg4 --no-check > $O/ida_ncu.log 2>&1
echo "ida rc=$?"
timeout 300 python tools/prof_sweep.py > $O/sweep_plain.log 2>&1 && \
timeout 900 ncu --clock-control none --import-source on --set full -k regex:"sense16_kernel|sense16_multi" -s 2 -c 2 \
  -o $O/sweep -f python tools/prof_sweep.py > $O/sweep_ncu.log 2>&1
echo "sweep rc=$?"
for k in ida sweep; do
  ncu -i $O/$k.ncu-rep --page details --csv > $O/${k}_details.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page source --csv --print-source sass > $O/${k}_sass.csv 2>/dev/null
done
ls -la $O
