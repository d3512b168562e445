# cfg2 sweep step vs the grid-stride cap of the other run kernels (ABCS_GRID_WAVES), alternating
for r in 1 2 3; do for v in 2 1 3; do echo "grid_waves=$v $(ABCS_GRID_WAVES=$v python tools/sweep_time.py 2>/dev/null | head -1)"; done; done
