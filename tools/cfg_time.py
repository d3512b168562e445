"""Per-kernel device time of one BASELINE config's sense+decode: python tools/cfg_time.py {1,3,4,5}"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2001_09632_b200 as p  # noqa: E402

CFGS = {"1": (256, 256, 1, 16, 1, 4, p.Algorithm.BBV, 20, 5.0, 1, False),
        "3": (1080, 1920, 256, 8, 1, 5, p.Algorithm.BBV, 20, 5.0, 3, True),
        "4": (512, 512, 64, 16, 3, 10, p.Algorithm.BBV, 20, 5.0, 4, False),
        "5": (4096, 4096, 16, 16, 1, 4, p.Algorithm.DD, 200, 8.0, 5, False)}
H, W, n, B, num, den, algo, ell, sig, seed, video = CFGS[sys.argv[1]]
imgs = p.synth_images(p.SynthSpec(H, W, ell, sig, seed, video=video), 0, n)
cfg = p.SensingConfig(B, num, den, algo)
plan = p.sense_plan(cfg, H, W)
b, x = p.sense_decode_batch(imgs, cfg, plan)
for _ in range(3):
    p.sense_decode_batch(imgs, cfg, plan, out=b, image_out=x)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    p.sense_decode_batch(imgs, cfg, plan, out=b, image_out=x)
e.record()
torch.cuda.synchronize()
print(f"cfg{sys.argv[1]}: {s.elapsed_time(e) / 10:.4f} ms per batch")
ctx = p.Context.get()
ctx.set_pipeline_streams(1)
ctx.kernel_timing(True)
for _ in range(10):
    p.sense_decode_batch(imgs, cfg, plan, out=b, image_out=x)
torch.cuda.synchronize()
for k, (cnt, tot, _) in ctx.kernel_times().items():
    print(f"  {k:24s} {tot / 10:.4f} ms ({cnt // 10} launches)")
