cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ABCS_IDA_TC=1 timeout 300 python tools/ida_time.py cfg4 > gpurun_out/tc2_cfg4.log 2>&1; echo "tc rc=$?" >> gpurun_out/tc2_cfg4.log
