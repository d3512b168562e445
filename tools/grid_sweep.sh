# cfg2 sweep step vs pipe stream priorities (ABCS_PIPE_PRIO), alternating
for r in 1 2 3; do for v in 0 1 2; do echo "prio=$v $(ABCS_PIPE_PRIO=$v python tools/sweep_time.py 2>/dev/null | head -1)"; done; done
