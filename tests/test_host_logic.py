"""CPU-only checks of the product's host logic and C-ABI library (no GPU compute):
plan derivations, parse_ratio, dd_threshold, zigzag tables, generated DCT
tables, the x87-emulating allocator keys and the synthetic generator."""
import ctypes as C
import hashlib
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, synth

import paper_2001_09632_b200 as p
from paper_2001_09632_b200 import _lib

HEADER = os.path.join(ROOT, "include", "abcs_b200.h")


def test_library_exports_every_header_symbol():
    text = open(HEADER).read()
    declared = set(re.findall(r"^\s*(?:int|double|int64_t|size_t|const char\*)\s+(abcs_\w+)\s*\(", text, re.M))
    assert len(declared) >= 18
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(r"\bT " + name + r"\b", out), name
    assert lib.abcs_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_ctx_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = _lib.load().abcs_ctx_create(0, C.byref(h))
    assert st == _lib.CUDA
    with pytest.raises(p.CudaError):
        p.sense(np.zeros((32, 32), np.uint8), p.SensingConfig(16, 1, 4, p.Algorithm.ZZ))


@pytest.mark.parametrize("text", ["0.1", "1/10", "0.25", "3/12", ".5", "2.", "1", "0.333333333", "1/3",
                                  "0", "abc", "1/0", "0.1234567890", "", "/", "12345678901/3"])
def test_parse_ratio_matches_reference(ref, text):
    import oracle as o
    try:
        want = ref.parse_ratio(text)
    except o.OracleError:
        with pytest.raises(ValueError):
            p.SensingConfig.parse_ratio(text)
        return
    assert p.SensingConfig.parse_ratio(text) == want


def test_dd_threshold_matches_reference(ref):
    for h in (100, 256, 383, 384, 512, 1080):
        for num, den in ((1, 1), (1, 2), (1, 3), (3, 10), (10, 33), (1, 4), (1, 5), (1, 9), (1, 10), (1, 20), (100, 333)):
            assert p.dd_threshold(h, num, den) == ref.dd_threshold(h, num, den)


def test_zigzag_matches_reference(ref):
    for B in (1, 2, 3, 8, 16, 32, 33):
        assert np.array_equal(p.zigzag_order(B).index, ref.zigzag(B))


PLAN_CASES = [(256, 256, 16, 1, 4, 1), (512, 512, 16, 1, 10, 2), (512, 512, 16, 3, 10, 2), (512, 512, 16, 1, 2, 2),
              (1080, 1920, 8, 1, 5, 1), (512, 512, 16, 3, 10, 1), (4096, 4096, 16, 1, 4, 2), (64, 64, 16, 1, 1, 1),
              (64, 64, 16, 1, 40, 1), (64, 64, 16, 1, 600, 2), (70, 90, 16, 1, 3, 1), (64, 64, 16, 1, 300, 0),
              (100, 60, 32, 7, 9, 2), (64, 64, 2, 1, 2, 1), (8, 64, 16, 1, 4, 1)]


@pytest.mark.parametrize("case", PLAN_CASES)
def test_plan_matches_reference(ref, case):
    """The plan's derived quantities equal what the reference's sense() produces."""
    import oracle as o
    H, W, B, num, den, algo = case
    img = synth(H, W, seed=1)[0] if H * W <= 1 << 22 else np.zeros((H, W), np.uint8)
    cfg = p.SensingConfig(B, num, den, p.Algorithm(algo))
    try:
        want = ref.sense(img, B, num, den, algo) if H * W <= 1 << 22 else None
    except o.OracleError as e:
        with pytest.raises(ValueError):
            p.sense_plan(cfg, H, W)
        assert e.code == 1
        return
    plan = p.sense_plan(cfg, H, W)
    assert plan.rows == H // B and plan.cols == W // B
    if want is None:
        assert plan.coeffs_per_image == 2 * plan.n_blocks * plan.dd_phase1
        return
    assert plan.algorithm_used == want["algorithm"]
    assert plan.threshold == want["threshold"]
    assert plan.coeffs_per_image == len(want["coeffs"])
    assert plan.side_per_image == len(want["side"])
    assert plan.target == want["target"] and plan.budget_actual == want["actual"]


def test_generated_dct_header_is_current():
    r = subprocess.run(["python", os.path.join(ROOT, "tools", "gen_dct.py"), "--check"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout


def test_generated_basis_is_the_reference_basis(port):
    """fp64 tables in dct_gen.cuh equal the oracle's (reference-pinned) basis bit for bit."""
    text = open(os.path.join(ROOT, "paper_2001_09632_b200", "csrc", "dct_gen.cuh")).read()
    for B in (8, 16, 32):
        body = re.search(r"static constexpr double kBasis%d\[\d+\] = \{(.*?)\};" % B, text, re.S).group(1)
        vals = np.array([float.fromhex(t) for t in re.findall(r"-?0x[0-9a-fp.+-]+", body)])
        assert np.array_equal(vals, port.basis(B))
        zz = re.search(r"static constexpr unsigned short kZigzag%d\[\d+\] = \{(.*?)\};" % B, text, re.S).group(1)
        assert np.array_equal(np.array([int(t) for t in re.findall(r"\d+", zz)]), port.zigzag(B))


def test_fp32_butterflies_host_build(tmp_path):
    """The generated even/odd DCTs, built for the host, match the fp64 reference transform."""
    src = tmp_path / "chk.cpp"
    src.write_text(r'''
#include <cmath>
#include <cstdio>
#include <cstdlib>
#define ABCS_DCT_QUAL static inline
#include "dct_gen.cuh"
template <int B> double chk(void (*f)(const float*, float*), void (*g)(const float*, float*), const double* Cb) {
  double e = 0; srand(1);
  for (int t = 0; t < 2000; ++t) { float x[B], y[B], xr[B];
    for (int i = 0; i < B; ++i) x[i] = rand() % 256;
    f(x, y); for (int k = 0; k < B; ++k) { double s = 0; for (int n = 0; n < B; ++n) s += Cb[k*B+n]*x[n]; e = fmax(e, fabs(s - y[k])); }
    g(y, xr); for (int n = 0; n < B; ++n) e = fmax(e, fabs(xr[n] - x[n])); }
  return e; }
int main() { printf("%g %g %g\n", chk<8>(abcs_gen::dct8_fwd, abcs_gen::dct8_inv, abcs_gen::kBasis8),
  chk<16>(abcs_gen::dct16_fwd, abcs_gen::dct16_inv, abcs_gen::kBasis16),
  chk<32>(abcs_gen::dct32_fwd, abcs_gen::dct32_inv, abcs_gen::kBasis32)); }
''')
    exe = tmp_path / "chk"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_2001_09632_b200", "csrc"),
                    str(src), "-o", str(exe)], check=True)
    errs = [float(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert max(errs) < 2e-4, errs


def test_allocator_keys_emulate_x87(tmp_path):
    """alloc_keys.h (the device allocator's ranking) equals x87 long double on 600k cases."""
    exe = tmp_path / "akc"
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "paper_2001_09632_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "alloc_keys_check.c"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "600000"], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout


def test_synth_host_deterministic_and_pinned():
    a = p.synth_images_host(p.SynthSpec(64, 96, 20, 5.0, 9), 3, 2)
    b = p.synth_images_host(p.SynthSpec(64, 96, 20, 5.0, 9), 3, 2)
    assert np.array_equal(a, b)
    c = p.synth_images_host(p.SynthSpec(64, 96, 20, 5.0, 9), 4, 1)
    assert np.array_equal(a[1], c[0])
    golden = os.path.join(ROOT, "tests", "golden", "synth_hashes.txt")
    got = {f"{h}x{w}-{e}-{s}-{seed}-{v}": hashlib.sha256(
        p.synth_images_host(p.SynthSpec(h, w, e, s, seed, bool(v)), 0, 2).tobytes()).hexdigest()
        for (h, w, e, s, seed, v) in ((256, 256, 20, 5.0, 1, 0), (64, 64, 200, 8.0, 5, 0), (54, 96, 20, 5.0, 3, 1))}
    want = dict(line.split() for line in open(golden).read().splitlines() if line.strip())
    assert got == want


def test_video_frames_are_shifted_copies():
    a = synth(54, 96, n=3, seed=3, sigma=0.0, video=True)
    # noise-free frames differ only by an integer translation with edge replication
    assert a.shape == (3, 54, 96)
    assert not np.array_equal(a[0], a[1]) or not np.array_equal(a[1], a[2])


def test_unsupported_configs_fail_loudly():
    with pytest.raises(ValueError):
        p.sense_plan(p.SensingConfig(1, 1, 4, p.Algorithm.BBV), 64, 64)
    with pytest.raises(ValueError):
        p.SensingConfig(16, 0, 4).validate()
    cfg = p.ReconConfig(method=p.ReconMethod.Ida, denoiser=p.DenoiserSpec("blur"))
    with pytest.raises(p.UnsupportedError):
        cfg._ida_c()
