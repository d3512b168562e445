"""cfg2 sweep step timing (1024 x 512^2, DD {0.1,0.3,0.5}): step ms and per-kernel ms on a serialised
pass. python tools/sweep_time.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2001_09632_b200 as p  # noqa: E402

imgs = p.synth_images(p.SynthSpec(512, 512, 20, 5.0, 2), 0, 1024)
cfgs = [p.SensingConfig(16, n, d, p.Algorithm.DD) for n, d in ((1, 10), (3, 10), (1, 2))]
outs = p.sense_decode_sweep(imgs, cfgs)
bs, xs = [o[0] for o in outs], [o[1] for o in outs]
for _ in range(3):
    p.sense_decode_sweep(imgs, cfgs, outs=bs, image_outs=xs)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
s.record()
for _ in range(reps):
    p.sense_decode_sweep(imgs, cfgs, outs=bs, image_outs=xs)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
print(f"step {ms:.3f} ms  {3 * 1024 * 512 * 512 / ms / 1e3:.0f} MP/s")
ctx = p.Context.get()
ctx.set_pipeline_streams(1)
ctx.kernel_timing(True)
for _ in range(reps):
    p.sense_decode_sweep(imgs, cfgs, outs=bs, image_outs=xs)
torch.cuda.synchronize()
for k, (cnt, tot, _) in ctx.kernel_times().items():
    print(f"  {k:24s} {tot / reps:.4f} ms/step ({cnt // reps} launches)")
