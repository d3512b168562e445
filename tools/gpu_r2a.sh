cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/ida_time.py cfg4 > gpurun_out/r2a_cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_cfg4.log
timeout 900 python -m pytest tests -m gpu -x -q -k "ida or recon or IDA or sharded or damp or race or tensor_core" > gpurun_out/r2a_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_tests.log
