"""Device-path throughput of every BASELINE config (cfg1..cfg5) on one GPU, with the
algorithmic-bytes roofline fraction. Inputs resident in HBM. One line each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2001_09632_b200 as p  # noqa: E402

HBM = 6536.0
ctx = p.Context.get()
ctx.set_pipeline_streams(1)  # serial: per-kernel times add up to the call


def breakdown(fn):
    ctx.kernel_timing(True)
    fn()
    t = ctx.kernel_times()
    ctx.kernel_timing(False)
    return {k: round(v[1], 4) for k, v in t.items()}


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def sense_decode(name, H, W, n, B, num, den, algo, ell, sig, seed, video=False):
    spec = p.SynthSpec(H, W, ell, sig, seed, video=video)
    imgs = p.synth_images(spec, 0, n)
    cfg = p.SensingConfig(B, num, den, algo)
    plan = p.sense_plan(cfg, H, W)
    b, out = p.sense_decode_batch(imgs, cfg, plan)
    ms = timed(lambda: p.sense_decode_batch(imgs, cfg, plan, out=b, image_out=out))
    N, K, S, nB = H * W, plan.coeffs_per_image, plan.side_per_image, plan.n_blocks
    Nc = plan.rows * B * plan.cols * B
    alg = n * (N + 8 * K + 4 * nB + 4 * S + 4 * Nc)
    kt = breakdown(lambda: p.sense_decode_batch(imgs, cfg, plan, out=b, image_out=out))
    print(json.dumps({"cfg": name, "ms": round(ms, 4), "MP_s": round(n * N / ms / 1e3, 1),
                      "hbm_frac": round(alg / (ms / 1e3) / 1e9 / HBM, 4), "kernels_ms": kt}), flush=True)
    return b


def ida(name, b, iters):
    rc = p.ReconConfig(p.ReconMethod.Ida, iterations=iters)
    out = torch.empty((b.n, b.plan.rows * b.plan.block, b.plan.cols * b.plan.block), device="cuda")
    ms = timed(lambda: p.ida_batch(b, rc, out=out, trace=False, check=False), reps=3, warm=1)
    Nc = out.shape[1] * out.shape[2]
    K = b.plan.coeffs_per_image
    alg = b.n * ((8 * Nc + 12 * K) * iters + 8 * K + 4 * Nc)
    kt = breakdown(lambda: p.ida_batch(b, rc, out=out, trace=False, check=False))
    print(json.dumps({"cfg": name + " IDA", "ms": round(ms, 3), "it_s": round(b.n * iters / ms * 1e3, 1),
                      "hbm_frac": round(alg / (ms / 1e3) / 1e9 / HBM, 4), "kernels_ms": kt}), flush=True)


which = sys.argv[1:] or ["1", "2", "3", "4", "5"]
if "1" in which:
    sense_decode("cfg1 256^2 B16 BBV0.25", 256, 256, 1, 16, 1, 4, p.Algorithm.BBV, 20, 5.0, 1)
if "2" in which:
    for num, den in ((1, 10), (3, 10), (1, 2)):
        sense_decode(f"cfg2 1024x512^2 B16 DD{num}/{den}", 512, 512, 1024, 16, num, den, p.Algorithm.DD, 20, 5.0, 2)
if "3" in which:
    sense_decode("cfg3 256x1080p B8 BBV0.2", 1080, 1920, 256, 8, 1, 5, p.Algorithm.BBV, 20, 5.0, 3, video=True)
if "4" in which:
    b = sense_decode("cfg4 64x512^2 B16 BBV0.3", 512, 512, 64, 16, 3, 10, p.Algorithm.BBV, 20, 5.0, 4)
    ida("cfg4", b, 10)
if "5" in which:
    b = sense_decode("cfg5 16x4096^2 B16 DD0.25 (per GPU of 8)", 4096, 4096, 16, 16, 1, 4, p.Algorithm.DD, 200, 8.0, 5)
    ida("cfg5", b, 5)
