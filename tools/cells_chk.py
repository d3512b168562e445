import sys, torch; sys.path.insert(0, '.')
import paper_2001_09632_b200 as p
imgs = p.synth_images(p.SynthSpec(512, 512, 20, 5.0, 2), 0, 1024)
cfgs = [p.SensingConfig(16, a, b, p.Algorithm.DD) for a, b in ((1, 10), (3, 10), (1, 2))]
h = imgs.cpu().pin_memory()
cells = p.bench_cells_host(h, cfgs, chunk=64)
got = p.sense_decode_sweep(imgs, cfgs)
for j, (b, x) in enumerate(got):
    q = p.quality_batch(imgs, x)
    print(j, float(cells["psnr"][j].mean()), float(q["psnr"].mean()), float(q["psnr"][0]), float(cells["psnr"][j][0]),
          [bool(torch.equal(cells[k][j], q[k].cpu())) for k in ("mse", "psnr", "ssim")])
