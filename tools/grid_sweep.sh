# cfg2 sweep step vs the number of batch chunks over the 3 pipe streams (ABCS_SWEEP_CHUNKS), alternating
for r in 1 2 3; do for v in 3 4 6 2; do echo "chunks=$v $(ABCS_SWEEP_CHUNKS=$v python tools/sweep_time.py 2>/dev/null | head -1)"; done; done
