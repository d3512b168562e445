"""Pins the C restatement (oracle/abcs_oracle.c) to the reference library itself
(oracle/_ref, compiled from /root/reference/proj/core/src): bit-exact on every
hot-path routine, on seeded synthetic scenes, the reference's own test scenes
(synth.cpp make_test_image) and adversarial allocator vectors."""
import numpy as np
import pytest

from conftest import synth

CASES = [  # (H, W, B, num, den, algo)
    (256, 256, 16, 1, 4, 1), (64, 64, 16, 1, 4, 1), (96, 80, 8, 1, 5, 1), (64, 48, 16, 3, 10, 1),
    (64, 64, 16, 1, 10, 2), (64, 64, 16, 3, 10, 2), (64, 64, 16, 1, 2, 2), (40, 72, 8, 1, 4, 2),
    (64, 64, 32, 1, 4, 2), (64, 64, 16, 1, 4, 0), (64, 64, 16, 1, 1, 1), (64, 64, 16, 1, 40, 1),
    (64, 64, 16, 1, 600, 2), (70, 90, 16, 1, 3, 1), (392, 64, 16, 1, 4, 2), (64, 64, 2, 1, 2, 1),
    (64, 64, 16, 1, 300, 0),
]


@pytest.mark.parametrize("case", CASES)
def test_sense_bit_exact(port, ref, case):
    H, W, B, num, den, algo = case
    import oracle as o
    img = synth(H, W, seed=H * 7 + W)[0]
    try:
        a = ref.sense(img, B, num, den, algo)
    except o.OracleError as e:  # error behaviour must match too
        with pytest.raises(o.OracleError) as eb:
            port.sense(img, B, num, den, algo)
        assert eb.value.code == e.code
        return
    b = port.sense(img, B, num, den, algo)
    assert a["algorithm"] == b["algorithm"]
    assert a["threshold"] == b["threshold"]
    assert np.array_equal(a["counts"], b["counts"])
    assert np.array_equal(a["coeffs"], b["coeffs"])
    assert np.array_equal(a["side"], b["side"])
    assert (a["target"], a["actual"]) == (b["target"], b["actual"])


def test_sense_threshold_override(port, ref):
    img = synth(64, 64, seed=3)[0]
    for thr in (0.0, 7.5, 123.0):
        a = ref.sense(img, 16, 1, 4, 2, threshold=thr)
        b = port.sense(img, 16, 1, 4, 2, threshold=thr)
        assert a["threshold"] == b["threshold"] == thr
        assert np.array_equal(a["counts"], b["counts"])


@pytest.mark.parametrize("bad", [(64, 64, 1, 1, 4, 1), (64, 64, 16, 0, 4, 1), (64, 64, 16, 5, 4, 1),
                                 (8, 64, 16, 1, 4, 1), (300, 300, 256, 1, 4, 1)])
def test_sense_errors_match(port, ref, bad):
    import oracle as o
    H, W, B, num, den, algo = bad
    img = synth(H, W)[0]
    with pytest.raises(o.OracleError) as ea:
        ref.sense(img, B, num, den, algo)
    with pytest.raises(o.OracleError) as eb:
        port.sense(img, B, num, den, algo)
    assert ea.value.code == eb.value.code


def test_reference_scenes(port, ref):
    import ctypes as C
    for name in ("blobs", "edges", "mixed", "texture"):
        img = np.zeros((128, 128), np.uint8)
        assert ref.lib.ref_make_test_image(name.encode(), 128, img.ctypes.data_as(C.c_void_p)) == 0
        for algo, num, den in ((1, 1, 4), (2, 1, 10), (2, 1, 2)):
            a = ref.sense(img, 16, num, den, algo)
            b = port.sense(img, 16, num, den, algo)
            assert np.array_equal(a["counts"], b["counts"]) and np.array_equal(a["coeffs"], b["coeffs"])


def test_dct_tables(port, ref, rng):
    for B in (2, 3, 8, 16, 32):
        assert np.array_equal(ref.zigzag(B), port.zigzag(B))
        for _ in range(5):
            x = rng.integers(0, 256, B * B).astype(np.float64)
            assert np.array_equal(ref.dct2(x, B), port.dct2(x, B))
            y = rng.normal(0, 50, B * B)
            assert np.array_equal(ref.idct2(y, B), port.idct2(y, B))


def adversarial_vectors(rng, n):
    for i in range(n):
        m = int(rng.integers(1, 40))
        kind = i % 4
        if kind == 0:
            w = rng.integers(0, 8, m).astype(np.float64)
        elif kind == 1:
            w = rng.integers(0, 3, m).astype(np.float64) * rng.integers(1, 1000)
        elif kind == 2:
            w = rng.integers(0, 20000, m).astype(np.float64)
        else:
            w = np.zeros(m)
        cap = int(rng.integers(1, 300))
        caps = np.full(m, cap, np.int32)
        if i % 7 == 0:
            caps = rng.integers(0, 300, m).astype(np.int32)
        budget = int(rng.integers(0, int(caps.sum()) + 1))
        yield w, budget, caps


def test_allocator_bit_exact(port, ref, rng):
    for w, budget, caps in adversarial_vectors(rng, 3000):
        assert np.array_equal(ref.allocate(w, budget, caps), port.allocate(w, budget, caps))


def test_allocator_spec_examples(port, ref):
    # SPEC.md worked examples (sensing module): proportional splits and cap redistribution
    assert list(ref.allocate([10, 20, 30, 40], 900, [1024] * 4)) == [90, 180, 270, 360]
    assert list(ref.allocate([1, 0, 0, 0], 2000, [1024] * 4)) == [1024, 326, 325, 325]
    assert list(ref.allocate([5, 3, 2, 0], 40, [246] * 4)) == [20, 12, 8, 0]
    for args in (([10, 20, 30, 40], 900, [1024] * 4), ([1, 0, 0, 0], 2000, [1024] * 4)):
        assert np.array_equal(ref.allocate(*args), port.allocate(*args))


def test_bbv_measure(port, ref):
    for (H, W, B, num, den) in ((256, 256, 16, 1, 4), (96, 80, 8, 1, 5), (64, 64, 16, 1, 1), (64, 64, 4, 1, 1)):
        img = synth(H, W, seed=H + W)[0]
        a, b = ref.bbv_measure(img, B, num, den), port.bbv_measure(img, B, num, den)
        for k in ("stride", "offset", "per_side", "phase1_total"):
            assert a[k] == b[k]
        assert np.array_equal(a["variation"], b["variation"]) and np.array_equal(a["side"], b["side"])


def test_decode_forward_denoise(port, ref, rng):
    img = synth(64, 96, seed=11)[0]
    ms = ref.sense(img, 16, 3, 10, 1)
    rows, cols = 4, 6
    assert np.array_equal(ref.decode(rows, cols, 16, ms["counts"], ms["coeffs"]),
                          port.decode(rows, cols, 16, ms["counts"], ms["coeffs"]))
    field = rng.normal(128, 40, (64, 96))
    assert np.array_equal(ref.forward(rows, cols, 16, ms["counts"], field),
                          port.forward(rows, cols, 16, ms["counts"], field))
    for thr in (0.0, 5.0, 40.0):
        assert np.array_equal(ref.denoise(field, thr), port.denoise(field, thr))


def test_ida_bit_exact(port, ref):
    img = synth(64, 64, seed=5)[0]
    for B, num, den, algo in ((16, 3, 10, 1), (8, 1, 4, 2)):
        ms = ref.sense(img, B, num, den, algo)
        rows, cols = 64 // B, 64 // B
        xa, ta = ref.reconstruct_ida(rows, cols, B, ms["counts"], ms["coeffs"], 4, ref=img)
        xb, tb = port.reconstruct_ida(rows, cols, B, ms["counts"], ms["coeffs"], 4, ref=img)
        assert np.array_equal(xa, xb)
        assert np.array_equal(ta, tb)


def test_ida_divergence_and_validation(port, ref):
    import oracle as o
    img = synth(32, 32, seed=2)[0]
    ms = ref.sense(img, 16, 1, 4, 1)
    for it, dmp in ((0, 2.0), (3, 0.5)):
        with pytest.raises(o.OracleError) as ea:
            ref.reconstruct_ida(2, 2, 16, ms["counts"], ms["coeffs"], it, damping=dmp)
        with pytest.raises(o.OracleError) as eb:
            port.reconstruct_ida(2, 2, 16, ms["counts"], ms["coeffs"], it, damping=dmp)
        assert ea.value.code == eb.value.code == 1
    huge = ms["coeffs"] * 1e7
    with pytest.raises(o.OracleError) as ea:
        ref.reconstruct_ida(2, 2, 16, ms["counts"], huge, 3)
    with pytest.raises(o.OracleError) as eb:
        port.reconstruct_ida(2, 2, 16, ms["counts"], huge, 3)
    assert ea.value.code == eb.value.code == 3 and ea.value.iteration == eb.value.iteration


def test_quality_metrics(port, ref, rng):
    """metrics.cpp:63-125: mse / psnr / ssim restated in the C port."""
    for H, W in ((11, 11), (40, 53), (96, 64)):
        a = rng.integers(0, 256, (H, W)).astype(np.float64)
        b = np.clip(a + rng.normal(0, 7, a.shape), -20, 280)
        m0, p0, s0 = ref.quality(a, b)
        m1, p1, s1 = port.quality(a, b)
        assert m1 == pytest.approx(m0, rel=1e-12) and p1 == p0 and s1 == s0
    assert ref.quality(a, a)[1] == float("inf") and port.quality(a, a)[1] == float("inf")
