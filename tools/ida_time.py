"""cfg4 IDA timing for kernel iteration: per-launch ida_step time (library CUDA events) and the
batch rate, plus parity of the final image against the oracle on 2 images.
python tools/ida_time.py [cfg4|cfg5] [--no-check]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2001_09632_b200 as p  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "cfg4"
nimg = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--n=")), "0"))
if which == "cfg4":
    H, n, ell, sig, seed, algo, num, den, iters = 512, 64, 20, 5.0, 4, p.Algorithm.BBV, 3, 10, 10
else:
    H, n, ell, sig, seed, algo, num, den, iters = 4096, 16, 200, 8.0, 5, p.Algorithm.DD, 1, 4, 5
n = nimg or n
imgs = p.synth_images(p.SynthSpec(H, H, ell, sig, seed), 0, n)
b = p.sense_batch(imgs, p.SensingConfig(16, num, den, algo))
rc = p.ReconConfig(p.ReconMethod.Ida, iterations=iters)
out = torch.empty((n, H, H), dtype=torch.float32, device=imgs.device)
for _ in range(3):
    p.ida_batch(b, rc, out=out, trace=False, check=False)
torch.cuda.synchronize()
ctx = p.Context.get()
ctx.kernel_timing(True)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
s.record()
for _ in range(reps):
    p.ida_batch(b, rc, out=out, trace=False, check=False)
e.record()
torch.cuda.synchronize()
kt = ctx.kernel_times()
ctx.kernel_timing(False)
ms = s.elapsed_time(e) / reps
K = b.plan.coeffs_per_image
per_iter = n * (8 * H * H + 12 * K)
for k, (cnt, tot, _) in kt.items():
    avg = tot / cnt
    extra = f"  {per_iter / avg / 1e6:.0f} GB/s ({per_iter / avg / 1e6 / 6547:.3f} of HBM)" if k == "ida_step" else ""
    print(f"{k:14s} launches {cnt:4d}  avg {avg * 1e3:8.1f} us{extra}")
print(f"batch {ms:.3f} ms  {n * iters / ms * 1e3:.0f} it/s (kernel timing on: plain launches)")
s.record()
for _ in range(reps):
    p.ida_batch(b, rc, out=out, trace=False, check=False)
e.record()
torch.cuda.synchronize()
ms2 = s.elapsed_time(e) / reps
print(f"batch {ms2:.3f} ms  {n * iters / ms2 * 1e3:.0f} it/s (default: CUDA graph unless ABCS_NO_GRAPHS=1)")
if "--no-check" not in sys.argv:
    import oracle as o
    chk = o.best_available()
    out2, tr, _ = p.ida_batch(b, rc, reference=imgs)
    for i in range(2):
        host = imgs[i].cpu().numpy()
        want = chk.sense(host, 16, num, den, int(algo))
        assert np.array_equal(b.counts[i].cpu().numpy().astype(np.int64), want["counts"].astype(np.int64))
        xr, trr = chk.reconstruct_ida(b.plan.rows, b.plan.cols, 16, want["counts"], want["coeffs"], iters, ref=host)
        d = np.max(np.abs(out2[i].cpu().numpy() - xr))
        print(f"image {i}: max |x - ref| = {d:.2e}; psnr {tr[i, -1, 3]:.4f} vs {trr[-1, 3]:.4f}")
