# cfg4/cfg5 sense+decode batch time vs the run kernels' grid-stride cap (ABCS_GRID_WAVES)
for r in 1 2; do for c in 5 4 3; do for v in 2 3 4 0; do echo "cfg$c grid_waves=$v $(ABCS_GRID_WAVES=$v python tools/cfg_time.py $c 2>/dev/null | head -1)"; done; done; done
