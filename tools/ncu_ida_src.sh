#!/bin/bash
# ncu --set full of one IDA step launch (cfg4) with per-source-line SASS counts
TAG=${TAG:-ida}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 300 python tools/ida_time.py cfg4 --no-check > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --clock-control none --import-source on --set full -k regex:ida_mma_kernel -s ${SKIP:-3} -c 1 \
  -o gpurun_out/${TAG}_ida -f python tools/ida_time.py cfg4 --no-check > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}_ida.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_ida.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_src.csv 2>/dev/null
ls -la gpurun_out
