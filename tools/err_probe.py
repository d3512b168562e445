"""Measure the device DCT error vs the fp64 reference and the DD near-threshold rate."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np, torch
import paper_2001_09632_b200 as p
import oracle as o
chk = o.best_available()
imgs = p.synth_images(p.SynthSpec(512, 512, 20, 5.0, 2), 0, 8)
for num, den in ((1, 10), (3, 10), (1, 2)):
    b = p.sense_batch(imgs, p.SensingConfig(16, 1, 1, p.Algorithm.ZZ))  # full rate: all 256 coefficients
    worst, near, tot = 0.0, 0, 0
    T = p.dd_threshold(512, num, den)
    ph1 = 16 * 16 * num // (2 * den)
    for i in range(8):
        h = imgs[i].cpu().numpy()
        want = chk.sense(h, 16, 1, 1, 0)["coeffs"]
        got = b.payload[i].cpu().numpy().astype(np.float64)
        worst = max(worst, float(np.max(np.abs(got - want))))
        w = want.reshape(-1, 256)[:, :ph1]
        near += int(np.sum(np.abs(np.abs(w) - T) < 2e-2))
        tot += w.size
    print(f"subrate {num}/{den}: max |coef err| {worst:.3e}; near-band(2e-2) fraction {near / tot:.2e} ({near} of {tot})")
