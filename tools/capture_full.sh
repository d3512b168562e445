#!/bin/bash
# ncu --set full captures of the hot kernels (cfg2 fused step at 1 stream: DD weights, warp
# allocator, fused gather+decode x 3 subrates; cfg4 IDA step), each only after the same
# command ran clean without ncu; then a plain bench run.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 300 python tools/prof_step.py fused > gpurun_out/p_fused.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:sense16_kernel|alloc_warp" -s 12 -c 9 -o gpurun_out/full_fused -f \
  python tools/prof_step.py fused > gpurun_out/ncu_fused.log 2>&1
echo "fused capture exit $?"
if [ -z "${NO_IDA:-}" ]; then
timeout 300 python tools/prof_step.py ida > gpurun_out/p_ida.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ida_mma_kernel -s 3 -c 1 \
  -o gpurun_out/full_ida -f python tools/prof_step.py ida > gpurun_out/ncu_ida.log 2>&1
echo "ida capture exit $?"
fi
if [ -z "${NO_BENCH:-}" ]; then
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench exit $?"
fi
