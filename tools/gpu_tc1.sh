cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/ida_time.py cfg4 > gpurun_out/tc1_cfg4.log 2>&1; echo "tc rc=$?" >> gpurun_out/tc1_cfg4.log
ABCS_IDA_TC=0 timeout 300 python tools/ida_time.py cfg4 --no-check > gpurun_out/tc1_cfg4_f32.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "ida or recon or IDA or sharded or damp or race" > gpurun_out/tc1_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tc1_tests.log
