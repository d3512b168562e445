# A/B of the fixup grid (CTAs per SM) on the pipelined cfg2 sweep step, alternating
for r in 1 2 3 4; do for v in 1 8; do echo "per_sm=$v $(ABCS_FIXUP_PER_SM=$v python tools/sweep_time.py | grep step)"; done; done
