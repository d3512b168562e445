#!/usr/bin/env python3
"""Regenerates tests/golden/* from the REFERENCE library itself (oracle/_ref,
compiled from /root/reference/proj/core/src by oracle/Makefile). Run in the
build container (the reference is not on the GPU box):

    make -C oracle && python tests/golden/make_golden.py

Inputs are stored in the fixtures, so they do not depend on our generator.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as o  # noqa: E402
import paper_2001_09632_b200 as p  # noqa: E402

SENSE_CASES = [  # (H, W, B, num, den, algo, seed)
    (256, 256, 16, 1, 4, 1, 1),    # cfg1 shape
    (64, 64, 16, 1, 10, 2, 2), (64, 64, 16, 3, 10, 2, 2), (64, 64, 16, 1, 2, 2, 2),  # cfg2 shapes
    (72, 96, 8, 1, 5, 1, 3),       # cfg3 shape (B=8, L=5)
    (64, 64, 16, 3, 10, 1, 4),     # cfg4 shape
    (64, 64, 16, 1, 4, 2, 5),      # cfg5 shape
    (64, 64, 16, 1, 4, 0, 6),      # zz
    (64, 64, 16, 1, 1, 1, 7),      # bbv full-rate fallback
    (64, 64, 16, 1, 40, 1, 8),     # bbv C_F > B fallback
    (64, 64, 16, 1, 600, 2, 9),    # dd phase1 = 0 fallback
    (70, 90, 16, 1, 3, 1, 10),     # ragged (cropped) image
    (64, 64, 32, 1, 4, 2, 11),     # B = 32
]
SYNTH = [(256, 256, 20, 5.0, 1, 0), (64, 64, 200, 8.0, 5, 0), (54, 96, 20, 5.0, 3, 1)]


def main():
    ref = o.Reference()
    rng = np.random.default_rng(20010963)
    out = {}
    for i, (H, W, B, num, den, algo, seed) in enumerate(SENSE_CASES):
        img = p.synth_images_host(p.SynthSpec(H, W, 20, 5.0, seed), 0, 1)[0]
        r = ref.sense(img, B, num, den, algo)
        out[f"s{i}_img"] = img
        out[f"s{i}_cfg"] = np.array([H, W, B, num, den, algo])
        out[f"s{i}_counts"] = r["counts"]
        out[f"s{i}_coeffs"] = r["coeffs"]
        out[f"s{i}_side"] = r["side"]
        out[f"s{i}_meta"] = np.array([r["algorithm"], r["threshold"], r["target"], r["actual"]], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "sense_cases.npz"), **out)

    al = {}
    for i in range(300):
        m = int(rng.integers(1, 64))
        kind = i % 3
        w = (rng.integers(0, 8, m) if kind == 0 else rng.integers(0, 20000, m) if kind == 1
             else rng.integers(0, 3, m) * int(rng.integers(1, 100))).astype(np.float64)
        caps = np.full(m, int(rng.integers(1, 300)), np.int32)
        budget = int(rng.integers(0, int(caps.sum()) + 1))
        al[f"a{i}_w"], al[f"a{i}_caps"] = w, caps
        al[f"a{i}_budget"] = np.array([budget])
        al[f"a{i}_out"] = ref.allocate(w, budget, caps)
    np.savez_compressed(os.path.join(HERE, "alloc_cases.npz"), **al)

    img = p.synth_images_host(p.SynthSpec(64, 64, 20, 5.0, 4), 0, 1)[0]
    ms = ref.sense(img, 16, 3, 10, 1)
    x, tr = ref.reconstruct_ida(4, 4, 16, ms["counts"], ms["coeffs"], 5, ref=img)
    field = rng.normal(128, 40, (32, 48))
    np.savez_compressed(os.path.join(HERE, "recon_case.npz"), img=img, counts=ms["counts"], coeffs=ms["coeffs"],
                        ida_x=x, ida_trace=tr, decode=ref.decode(4, 4, 16, ms["counts"], ms["coeffs"]),
                        field=field, den0=ref.denoise(field, 0.0), den20=ref.denoise(field, 20.0))

    with open(os.path.join(HERE, "synth_hashes.txt"), "w") as f:
        for (h, w, e, s, seed, v) in SYNTH:
            d = hashlib.sha256(p.synth_images_host(p.SynthSpec(h, w, e, s, seed, bool(v)), 0, 2).tobytes()).hexdigest()
            f.write(f"{h}x{w}-{e}-{s}-{seed}-{v} {d}\n")


CONTAINER_CASES = [  # (H, W, B, num, den, algo, seed): zz, bbv (with side data), dd, ragged, B = 8
    (64, 64, 16, 1, 4, 0, 21), (64, 64, 16, 1, 4, 1, 22), (64, 64, 16, 3, 10, 2, 23), (70, 90, 16, 1, 3, 1, 24),
    (48, 40, 8, 1, 5, 1, 25)]


def main_containers():
    """tests/golden/container_cases.npz: write_measurement_set bytes of reference sense() results."""
    import tempfile
    ref = o.Reference()
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for i, (H, W, B, num, den, algo, seed) in enumerate(CONTAINER_CASES):
            img = p.synth_images_host(p.SynthSpec(H, W, 20, 5.0, seed), 0, 1)[0]
            r = ref.sense(img, B, num, den, algo)
            ms = dict(height=H, width=W, block=B, algorithm=r["algorithm"], cr_num=num, cr_den=den,
                      threshold=r["threshold"], counts=r["counts"], coeffs=r["coeffs"], side=r["side"])
            path = os.path.join(d, f"c{i}.abcs")
            ref.write_container(ms, path)
            with open(path, "rb") as f:
                out[f"c{i}_bytes"] = np.frombuffer(f.read(), np.uint8)
            out[f"c{i}_hdr"] = np.array([H, W, B, r["algorithm"], num, den, r["threshold"]], dtype=np.float64)
            out[f"c{i}_counts"] = r["counts"]
            out[f"c{i}_coeffs"] = r["coeffs"]
            out[f"c{i}_side"] = r["side"]
    np.savez_compressed(os.path.join(HERE, "container_cases.npz"), **out)


FAMILY_CASES = [  # (name, method, iters, lambda, seed, denoiser, sigma_scale, damping)
    ("ista", 1, 4, 0.05, 42, 0, 25.0, 2.0), ("amp", 2, 3, 0.5, 42, 0, 25.0, 2.0),
    ("damp_dct", 3, 3, 1.0, 42, 0, 25.0, 2.0), ("dampd_dct", 4, 3, 1.0, 7, 0, 25.0, 3.0),
    ("damp_blur", 3, 3, 1.0, 42, 1, 25.0, 2.0), ("ida_blur", 5, 3, 1.0, 42, 1, 5.0, 2.0),
    ("ida_identity", 5, 2, 1.0, 42, 2, 25.0, 2.0)]


def main_family():
    """tests/golden/family_cases.npz: the rest of the reconstruction family from the reference
    (recon.cpp:133-259, denoise.cpp:14-128) and std::mt19937_64 outputs for the probe."""
    ref = o.Reference()
    rng = np.random.default_rng(2001)
    out = {}
    img = p.synth_images_host(p.SynthSpec(64, 64, 20, 5.0, 41), 0, 1)[0]
    ms = ref.sense(img, 16, 1, 4, 1)
    out["img"], out["counts"], out["coeffs"] = img, ms["counts"], ms["coeffs"]
    for name, method, iters, lam, seed, den, scale, damping in FAMILY_CASES:
        x, tr = ref.reconstruct(4, 4, 16, ms["counts"], ms["coeffs"], method, iters, damping=damping, lam=lam,
                                seed=seed, denoiser=den, sigma_scale=scale, ref=img)
        out[f"{name}_x"], out[f"{name}_trace"] = x, tr
    img8 = p.synth_images_host(p.SynthSpec(48, 40, 20, 5.0, 42), 0, 1)[0]
    ms8 = ref.sense(img8, 8, 1, 5, 1)
    out["img8"], out["counts8"], out["coeffs8"] = img8, ms8["counts"], ms8["coeffs"]
    out["amp8_x"], out["amp8_trace"] = ref.reconstruct(6, 5, 8, ms8["counts"], ms8["coeffs"], 2, 3, lam=0.5, ref=img8)
    field = rng.normal(128, 40, (40, 56))
    out["field"] = field
    for sig in (0.0, 7.0, 60.0, 400.0):
        out[f"blur_{int(sig)}"] = ref.denoise2(field, sig, denoiser=1, sigma_scale=25.0)
    out["div"] = np.array([ref.divergence(field, 20.0, 0.3, 99, denoiser=0),
                           ref.divergence(field, 80.0, 0.5, 12345, denoiser=1, sigma_scale=25.0)])
    for seed in (0, 42, 0x9E3779B97F4A7C15):
        out[f"mt_{seed:x}"] = ref.mt19937_64(seed, 2000)
    # THB / THI (metrics.cpp:126-225): (H, W, B, num, den) incl. a ragged crop and a flat image (all-zero AC ties)
    for i, (H, W, B, num, den, seed) in enumerate([(64, 80, 16, 1, 4, 51), (56, 48, 8, 1, 5, 52),
                                                   (100, 90, 16, 3, 10, 53), (64, 64, 32, 1, 2, 54)]):
        im = p.synth_images_host(p.SynthSpec(H, W, 12, 5.0, seed), 0, 1)[0]
        out[f"th{i}_img"], out[f"th{i}_cfg"] = im, np.array([B, num, den])
        for g in (0, 1):
            out[f"th{i}_x{g}"], out[f"th{i}_c{g}"] = ref.threshold_decode(im, B, num, den, bool(g))
    flat = np.full((32, 32), 77, np.uint8)
    out["thflat_img"] = flat
    for g in (0, 1):
        out[f"thflat_x{g}"], out[f"thflat_c{g}"] = ref.threshold_decode(flat, 16, 1, 2, bool(g))
    np.savez_compressed(os.path.join(HERE, "family_cases.npz"), **out)


if __name__ == "__main__":
    if "--containers" in sys.argv:
        main_containers()
    elif "--family" in sys.argv:
        main_family()
    else:
        main()
        main_containers()
        main_family()
