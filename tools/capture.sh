#!/bin/bash
# r01 evidence (TAG=v8, v9, ...): full bench line, launch list of the bench command, ncu --set full of the
# multi-plan payload kernel (each ncu run only after its command exited 0 without ncu).
TAG=${TAG:-v9}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?"
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-config-sweep > gpurun_out/${TAG}_bl_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-config-sweep \
  > gpurun_out/${TAG}_bl_ncu.log 2>&1
echo "bench launches rc=$?"
timeout 300 python tools/prof_sweep.py > gpurun_out/${TAG}_ll_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/prof_sweep.py > gpurun_out/${TAG}_ll_ncu.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --clock-control none --import-source on --set full -k regex:sense16_multi -s 1 -c 1 \
  -o gpurun_out/${TAG}_multi -f python tools/prof_sweep.py > gpurun_out/${TAG}_multi_ncu.log 2>&1
echo "multi rc=$?"
ncu -i gpurun_out/${TAG}_multi.ncu-rep --page details --csv > gpurun_out/${TAG}_multi_details.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_multi.ncu-rep --page raw --csv > gpurun_out/${TAG}_multi_raw.csv 2>/dev/null
