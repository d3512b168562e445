"""The C oracle against the golden vectors produced by the reference library
itself (tests/golden/make_golden.py). This pins the oracle on any machine,
including the GPU box where /root/reference does not exist."""
import os

import numpy as np
import pytest

from conftest import ROOT

G = os.path.join(ROOT, "tests", "golden")


def load(name):
    return np.load(os.path.join(G, name))


def test_sense_cases(port):
    z = load("sense_cases.npz")
    n = len([k for k in z.files if k.endswith("_cfg")])
    assert n >= 12
    for i in range(n):
        H, W, B, num, den, algo = (int(v) for v in z[f"s{i}_cfg"])
        r = port.sense(z[f"s{i}_img"], B, num, den, algo)
        meta = z[f"s{i}_meta"]
        assert r["algorithm"] == int(meta[0]) and r["threshold"] == meta[1]
        assert (r["target"], r["actual"]) == (int(meta[2]), int(meta[3]))
        assert np.array_equal(r["counts"], z[f"s{i}_counts"]), i
        assert np.array_equal(r["coeffs"], z[f"s{i}_coeffs"]), i
        assert np.array_equal(r["side"], z[f"s{i}_side"]), i


def test_alloc_cases(port):
    z = load("alloc_cases.npz")
    n = len([k for k in z.files if k.endswith("_w")])
    for i in range(n):
        got = port.allocate(z[f"a{i}_w"], int(z[f"a{i}_budget"][0]), z[f"a{i}_caps"])
        assert np.array_equal(got, z[f"a{i}_out"]), i


def test_recon_case(port):
    z = load("recon_case.npz")
    assert np.array_equal(port.decode(4, 4, 16, z["counts"], z["coeffs"]), z["decode"])
    x, tr = port.reconstruct_ida(4, 4, 16, z["counts"], z["coeffs"], 5, ref=z["img"])
    assert np.array_equal(x, z["ida_x"])
    assert np.array_equal(tr, z["ida_trace"])
    assert np.array_equal(port.denoise(z["field"], 0.0), z["den0"])
    assert np.array_equal(port.denoise(z["field"], 20.0), z["den20"])


def test_oracle_synth_matches_golden_hashes():
    """The oracle-side input generator (used by bench.py's reference arm, which must not load the
    product library) produces the pinned bytes."""
    import hashlib
    import oracle as o
    got = {f"{h}x{w}-{e}-{s}-{seed}-{v}": hashlib.sha256(o.synth_images(h, w, e, s, seed, 0, 2, bool(v)).tobytes())
           .hexdigest() for (h, w, e, s, seed, v) in ((256, 256, 20, 5.0, 1, 0), (64, 64, 200, 8.0, 5, 0),
                                                      (54, 96, 20, 5.0, 3, 1))}
    want = dict(line.split() for line in open(os.path.join(G, "synth_hashes.txt")).read().splitlines() if line.strip())
    assert got == want
