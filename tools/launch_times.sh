#!/bin/bash
# Per-kernel launch list (ncu duration + instructions) of tools/prof_step.py MODE, after a clean plain run.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
MODE=${1:-all}
timeout 300 python tools/prof_step.py $MODE > gpurun_out/p.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python tools/prof_step.py $MODE > gpurun_out/ncu.log 2>&1
echo "prof exit $?"
tail -2 gpurun_out/p.log
