#!/bin/bash
# r01 v5 evidence: launch list of the bench step (sweep), ncu --set full of the hot kernels
# (each after its command ran clean without ncu), exported to CSV under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
NCU="ncu --clock-control none --import-source on"
run() {  # name, ncu filter args..., -- command
  local name=$1; shift
  local filt=()
  while [ "$1" != "--" ]; do filt+=("$1"); shift; done; shift
  timeout 300 "$@" > gpurun_out/${name}_plain.log 2>&1 && \
  timeout 900 $NCU --set full "${filt[@]}" -o gpurun_out/${name} -f "$@" > gpurun_out/${name}_ncu.log 2>&1
  echo "$name rc=$?"
  ncu -i gpurun_out/${name}.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
}
# 1. launch list of one sweep step (all kernels, durations)
timeout 300 python tools/prof_sweep.py > gpurun_out/ll_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/v5_launches.csv python tools/prof_sweep.py > gpurun_out/ll_ncu.log 2>&1
echo "launches rc=$?"
# 2. full captures (second sweep step: warm)
run v5_sweepw -k regex:sense16_kernel -s 4 -c 1 -- python tools/prof_sweep.py
run v5_fused -k regex:sense16_kernel -s 5 -c 3 -- python tools/prof_sweep.py
run v5_alloc_cta -k regex:alloc_cta -s 3 -c 1 -- python tools/prof_sweep.py
run v5_ida -k regex:ida_mma_kernel -s 3 -c 1 -- python tools/prof_step.py ida
run v5_alloc5 -k regex:alloc_class -s 1 -c 1 -- python tools/prof_cfg.py 5
run v5_sense8 -k regex:sense8_kernel -s 1 -c 1 -- python tools/prof_cfg.py 3
