"""SSIM of 1024 decoded 512^2 images against their sources (the bench's metrics row), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2001_09632_b200 as p  # noqa: E402

imgs = p.synth_images(p.SynthSpec(512, 512, 20, 5.0, 2), 0, 1024)
b, x = p.sense_decode_batch(imgs, p.SensingConfig(16, 3, 10, p.Algorithm.DD))
for _ in range(2):
    q = p.quality_batch(imgs, x, want=("ssim",))
torch.cuda.synchronize()
print("ok", float(q["ssim"].mean()))
