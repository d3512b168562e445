"""Per-kernel device times (ctx kernel timing) of sense+decode for BASELINE configs 3/4/5 and the cfg2 step."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2001_09632_b200 as p  # noqa: E402

CFGS = {"3": (1080, 1920, 256, 8, 1, 5, p.Algorithm.BBV, 20, 5.0, 3, True),
        "4": (512, 512, 64, 16, 3, 10, p.Algorithm.BBV, 20, 5.0, 4, False),
        "5": (4096, 4096, 16, 16, 1, 4, p.Algorithm.DD, 200, 8.0, 5, False)}
ctx = p.Context.get()
ctx.set_pipeline_streams(1)
out = {}
for key in sys.argv[1:] or ["3", "4", "5"]:
    H, W, n, B, num, den, algo, ell, sig, seed, video = CFGS[key]
    imgs = p.synth_images(p.SynthSpec(H, W, ell, sig, seed, video=video), 0, n)
    cfg = p.SensingConfig(B, num, den, algo)
    for _ in range(3):
        p.sense_decode_batch(imgs, cfg)
    torch.cuda.synchronize()
    ctx.kernel_timing(True)
    for _ in range(5):
        p.sense_decode_batch(imgs, cfg)
    torch.cuda.synchronize()
    t = ctx.kernel_times()
    ctx.kernel_timing(False)
    out["cfg" + key] = {k: {"launches_per_call": v[0] / 5, "ms_per_call": round(v[1] / 5, 4)} for k, v in t.items()}
print(json.dumps(out, indent=1))
