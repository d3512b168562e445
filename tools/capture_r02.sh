#!/bin/bash
# r02 evidence (TAG=r02_vN): GPU suite, smoke, full bench line, reference arm, ncu launch list of
# the bench command, ncu --set full of the IDA step and of the sweep's multi-plan payload pass
# (each ncu run only after its command exited 0 without ncu).
TAG=${TAG:-r02}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi -L > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" | tee -a $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-config-sweep > $O/bl_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-config-sweep \
  > $O/bl_ncu.log 2>&1
echo "launches rc=$?"
timeout 300 python tools/ida_time.py cfg4 --no-check > $O/ida_plain.log 2>&1 && \
timeout 900 ncu --clock-control none --import-source on --set full -k regex:ida_mma_kernel -s 3 -c 1 \
  -o $O/ida -f python tools/ida_time.py cfg4 --no-check > $O/ida_ncu.log 2>&1
echo "ida ncu rc=$?"
timeout 300 python tools/prof_sweep.py > $O/sweep_plain.log 2>&1 && \
timeout 900 ncu --clock-control none --import-source on --set full -k regex:sense16_multi -s 1 -c 1 \
  -o $O/multi -f python tools/prof_sweep.py > $O/multi_ncu.log 2>&1
echo "multi ncu rc=$?"
timeout 900 ncu --clock-control none --import-source on --set full -k regex:sense16_kernel -s 1 -c 1 \
  -o $O/weights -f python tools/prof_sweep.py > $O/weights_ncu.log 2>&1
echo "weights ncu rc=$?"
timeout 900 ncu --clock-control none --import-source on --set full -k regex:alloc_warp -s 1 -c 1 \
  -o $O/alloc -f python tools/prof_sweep.py > $O/alloc_ncu.log 2>&1
echo "alloc ncu rc=$?"
for k in ida multi weights alloc; do
  ncu -i $O/$k.ncu-rep --page details --csv > $O/${k}_details.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page source --csv --print-source sass > $O/${k}_sass.csv 2>/dev/null
done
ls -la $O
