cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tensor_core" > gpurun_out/tc3_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tc3_tests.log
TAG=tc3 bash tools/ncu_tc.sh
