"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck): one per hot kernel.
python tools/sanitize_cases.py CASE   with CASE in
  alloc_cluster2 / alloc_cluster16  BBV allocation by the cluster allocator (DSMEM, cluster barriers)
  umma                              tcgen05 / TMEM gather + decode (ABCS_UMMA=1)
  ida                               fused IDA step (TMA window, fp32 denoiser + block phase), B=16 and B=8
  sweep                             the sweep's multi-plan payload pass (sense16_multi_kernel) + DD phase 1
  denoise                           standalone denoiser, DAMP (divergence probe), container, metrics, block DCT
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
case = sys.argv[1]
if case.startswith("alloc_cluster"):
    os.environ["ABCS_ALLOC_CLUSTER"] = case[len("alloc_cluster"):]
if case == "umma":
    os.environ["ABCS_UMMA"] = "1"
import torch  # noqa: E402

import paper_2001_09632_b200 as p  # noqa: E402

if case.startswith("alloc_cluster"):
    imgs = p.synth_images(p.SynthSpec(256, 384, 20, 5.0, 3), 0, 2)
    for algo, num, den in ((p.Algorithm.BBV, 3, 10), (p.Algorithm.DD, 1, 4)):
        b = p.sense_batch(imgs, p.SensingConfig(16, num, den, algo))
elif case == "umma":
    imgs = p.synth_images(p.SynthSpec(128, 256, 20, 5.0, 2), 0, 2)
    for num, den in ((1, 10), (1, 2)):
        b, x = p.sense_decode_batch(imgs, p.SensingConfig(16, num, den, p.Algorithm.DD))
        p.decode_batch(b)
elif case == "ida":
    for B, H, W in ((16, 128, 192), (8, 96, 128)):
        imgs = p.synth_images(p.SynthSpec(H, W, 20, 5.0, 4), 0, 2)
        b = p.sense_batch(imgs, p.SensingConfig(B, 3, 10, p.Algorithm.BBV))
        p.ida_batch(b, p.ReconConfig(p.ReconMethod.Ida, iterations=2), reference=imgs)
elif case == "sweep":
    imgs = p.synth_images(p.SynthSpec(128, 128, 20, 5.0, 2), 0, 3)
    cfgs = [p.SensingConfig(16, n, d, p.Algorithm.DD) for n, d in ((1, 10), (3, 10), (1, 2))]
    p.sense_decode_sweep(imgs, cfgs)
elif case == "denoise":
    imgs = p.synth_images(p.SynthSpec(64, 64, 20, 5.0, 5), 0, 1)
    b = p.sense_batch(imgs, p.SensingConfig(16, 1, 4, p.Algorithm.BBV))
    p.recon_batch(b, p.ReconConfig(p.ReconMethod.Damp, 2), trace=False, check=False)
    p.denoise(p.DenoiserSpec("dct_threshold"), imgs[0].cpu().numpy().astype(float), 20.0)
    p.unpack_containers(p.pack_containers(b), b.plan)
    x = p.decode_batch(b)
    p.quality_batch(imgs, x, ("mse", "psnr", "ssim"))
    p.block_dct_batch(torch.rand(3, 16, 16, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
print("case ok:", case)
