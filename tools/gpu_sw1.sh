cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sweep_time.py > gpurun_out/sw1_time.log 2>&1; echo "rc=$?" >> gpurun_out/sw1_time.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sweep or dd or DD or guard or race" > gpurun_out/sw1_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sw1_tests.log
