"""One warm cfg2 sweep step (3 subrates through abcs_sense_decode_sweep_batch), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2001_09632_b200 as p  # noqa: E402

imgs = p.synth_images(p.SynthSpec(512, 512, 20, 5.0, 2), 0, 1024)
p.Context.get().set_pipeline_streams(int(os.environ.get("PROF_STREAMS", "1")))
cfgs = [p.SensingConfig(16, num, den, p.Algorithm.DD) for num, den in ((1, 10), (3, 10), (1, 2))]
for rep in range(2):
    p.sense_decode_sweep(imgs, cfgs)
torch.cuda.synchronize()
print("ok")
