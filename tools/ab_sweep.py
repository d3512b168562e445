"""A/B timing of the cfg2 sweep step: python tools/ab_sweep.py ROOT_A ROOT_B [reps]; each ROOT holds a
built paper_2001_09632_b200 package. Alternates A and B in separate processes, 3 rounds each."""
import subprocess
import sys

code = r'''
import sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2001_09632_b200 as p
imgs = p.synth_images(p.SynthSpec(512, 512, 20, 5.0, 2), 0, 1024)
cfgs = [p.SensingConfig(16, n, d, p.Algorithm.DD) for n, d in ((1, 10), (3, 10), (1, 2))]
outs = p.sense_decode_sweep(imgs, cfgs)
bs, xs = [o[0] for o in outs], [o[1] for o in outs]
for _ in range(3):
    p.sense_decode_sweep(imgs, cfgs, outs=bs, image_outs=xs)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
s.record()
for _ in range(reps):
    p.sense_decode_sweep(imgs, cfgs, outs=bs, image_outs=xs)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
ctx = p.Context.get()
ctx.set_pipeline_streams(1)
ctx.kernel_timing(True)
for _ in range(reps):
    p.sense_decode_sweep(imgs, cfgs, outs=bs, image_outs=xs)
torch.cuda.synchronize()
kt = ctx.kernel_times()
print(f"step {ms:.4f} ms " + " ".join(f"{k}={t / c * 1e3:.1f}us" for k, (c, t, _) in kt.items()))
'''
for rnd in range(3):
    for tag, root in (("A", sys.argv[1]), ("B", sys.argv[2])):
        out = subprocess.run([sys.executable, "-c", code, root], capture_output=True, text=True)
        print(tag, out.stdout.strip() or out.stderr[-500:], flush=True)
