# cfg4 / cfg5 IDA batch (CUDA graph) vs the number of sub-batch chains (ABCS_IDA_SPLIT), alternating
for r in 1 2; do for k in 1 2 3 4; do echo "cfg4 chains=$k $(ABCS_IDA_SPLIT=$k python tools/ida_time.py cfg4 --no-check 2>&1 | grep 'CUDA graph')"; done; done
for k in 1 2 4; do echo "cfg5 chains=$k $(ABCS_IDA_SPLIT=$k python tools/ida_time.py cfg5 --no-check 2>&1 | grep 'CUDA graph')"; done
