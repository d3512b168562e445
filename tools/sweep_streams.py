"""cfg2 sweep step under different host-side conditions (pipeline streams, per-step events)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2001_09632_b200 as p  # noqa: E402
imgs = p.synth_images(p.SynthSpec(512, 512, 20, 5.0, 2), 0, 1024)
cfgs = [p.SensingConfig(16, n, d, p.Algorithm.DD) for n, d in ((1, 10), (3, 10), (1, 2))]
outs = p.sense_decode_sweep(imgs, cfgs)
bs, xs = [o[0] for o in outs], [o[1] for o in outs]
ctx = p.Context.get()
stream = torch.cuda.current_stream()
for ns, use_ev, reps in ((3, False, 20), (3, True, 20), (3, False, 10), (3, True, 10), (1, False, 20), (3, False, 20)):
    ctx.set_pipeline_streams(ns)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(reps)]
    for _ in range(3):
        p.sense_decode_sweep(imgs, cfgs, outs=bs, image_outs=xs)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for k in range(reps):
        if use_ev:
            ev[k][0].record(stream)
        p.sense_decode_sweep(imgs, cfgs, outs=bs, image_outs=xs)
        if use_ev:
            for x in ev[k][1:]:
                x.record(stream)
    e.record()
    torch.cuda.synchronize()
    print(ns, use_ev, reps, round(s.elapsed_time(e) / reps, 4))
