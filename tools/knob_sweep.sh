# cfg2 sweep step over the launch knobs (payload-pass rounds x other run kernels' rounds), 2 passes
for r in 1 2; do for m in 2 3 4; do for g in 2 3; do
  echo "multi=$m grid=$g $(ABCS_MULTI_WAVES=$m ABCS_GRID_WAVES=$g python tools/sweep_time.py 2>/dev/null | head -1)"
done; done; done
