"""The .abcs v1 container (container.cpp:58-149): device pack/unpack vs
fixtures written by the reference itself (tests/golden/container_cases.npz, made by
tests/golden/make_golden.py), the oracle's restatement of the layout, and the reader's
FormatError cases."""
import ctypes as C
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "container_cases.npz")


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


@pytest.fixture(scope="module")
def p(torch):
    import paper_2001_09632_b200 as p
    return p


def cases():
    z = np.load(GOLDEN)
    i = 0
    while f"c{i}_bytes" in z.files:
        H, W, B, algo, num, den, thr = z[f"c{i}_hdr"]
        yield dict(height=int(H), width=int(W), block=int(B), algorithm=int(algo), cr_num=int(num), cr_den=int(den),
                   threshold=float(thr), counts=z[f"c{i}_counts"], coeffs=z[f"c{i}_coeffs"], side=z[f"c{i}_side"],
                   bytes=z[f"c{i}_bytes"].tobytes())
        i += 1


def corrupt_variants(good: bytes, block: int):
    """(name, bytes) the reference reader rejects with FormatError (container.cpp:95-149)."""
    yield "truncated", good[:-3]
    yield "bad magic", b"ABCX" + good[4:]
    yield "trailing bytes", good + b"\0"
    v = bytearray(good)
    v[4] = 2
    yield "version", bytes(v)
    v = bytearray(good)
    v[37:39] = (block * block + 1).to_bytes(2, "little")
    yield "count > B^2", bytes(v)
    v = bytearray(good)
    v[16] = 3
    yield "algorithm id", bytes(v)


def test_oracle_layout_matches_reference_fixtures(port):
    import oracle
    for c in cases():
        got = oracle.container_bytes(c["height"], c["width"], c["block"], c["algorithm"], c["cr_num"], c["cr_den"],
                                     c["threshold"], c["counts"], c["coeffs"], c["side"])
        assert got == c["bytes"]


def test_reference_writer_and_reader(ref, tmp_path):
    for i, c in enumerate(cases()):
        path = tmp_path / f"r{i}.abcs"
        ref.write_container(c, path)
        assert path.read_bytes() == c["bytes"]
        back = ref.read_container(path)
        assert np.array_equal(back["counts"], c["counts"])
        assert np.array_equal(back["coeffs"], c["coeffs"].astype(np.float32).astype(np.float64))
        for name, bad in corrupt_variants(c["bytes"], c["block"]):
            (tmp_path / "bad.abcs").write_bytes(bad)
            with pytest.raises(Exception) as e:
                ref.read_container(tmp_path / "bad.abcs")
            assert "[2]" in str(e.value), name  # FormatError


def test_host_parse_layout_and_errors():
    from paper_2001_09632_b200 import _lib
    lib = _lib.load()
    for c in cases():
        buf = np.frombuffer(c["bytes"], np.uint8)
        plan = _lib.SensePlanC()
        assert lib.abcs_container_parse(buf.ctypes.data, buf.size, C.byref(plan)) == _lib.OK
        assert (plan.height, plan.width, plan.block) == (c["height"], c["width"], c["block"])
        assert plan.coeffs_per_image == len(c["coeffs"]) and plan.side_per_image == len(c["side"])
        assert plan.n_blocks == len(c["counts"]) and lib.abcs_container_size(C.byref(plan)) == buf.size
        for name, bad in corrupt_variants(c["bytes"], c["block"]):
            b = np.frombuffer(bad, np.uint8)
            assert lib.abcs_container_parse(b.ctypes.data, b.size, C.byref(plan)) == _lib.FORMAT, name


@pytest.mark.gpu
def test_device_write_read_match_reference_bytes(p, torch, tmp_path):
    for i, c in enumerate(cases()):
        ms = p.MeasurementSet(c["height"], c["width"], c["block"], p.Algorithm(c["algorithm"]), c["cr_num"],
                              c["cr_den"], c["threshold"], c["counts"].astype(np.uint16),
                              c["coeffs"].astype(np.float32), c["side"].astype(np.float32))
        path = tmp_path / f"d{i}.abcs"
        p.write_measurement_set(ms, path)
        assert path.read_bytes() == c["bytes"]
        (tmp_path / "ref.abcs").write_bytes(c["bytes"])
        back = p.read_measurement_set(tmp_path / "ref.abcs")
        assert (back.height, back.width, back.block, int(back.algorithm)) == (c["height"], c["width"], c["block"],
                                                                              c["algorithm"])
        assert (back.cr_num, back.cr_den, back.threshold) == (c["cr_num"], c["cr_den"], c["threshold"])
        assert np.array_equal(back.counts, c["counts"])
        assert np.array_equal(back.coeffs, c["coeffs"].astype(np.float32))
        assert np.array_equal(back.side, c["side"].astype(np.float32))
        for name, bad in corrupt_variants(c["bytes"], c["block"]):
            (tmp_path / "bad.abcs").write_bytes(bad)
            with pytest.raises(p.FormatError):
                p.read_measurement_set(tmp_path / "bad.abcs")


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(16, 3, 10, 2), (16, 1, 4, 1), (8, 1, 5, 1), (16, 1, 10, 0)])
def test_batch_pack_unpack_round_trip(p, torch, cfg):
    import oracle
    B, num, den, algo = cfg
    imgs = p.synth_images(p.SynthSpec(96, 128, 12, 5.0, 31), 0, 5)
    b = p.sense_batch(imgs, p.SensingConfig(B, num, den, p.Algorithm(algo)))
    data = p.pack_containers(b)
    size = p.container_size(b.plan)
    host = data.cpu().numpy()
    for i in range(b.n):
        want = oracle.container_bytes(b.plan.height, b.plan.width, b.plan.block, b.plan.algorithm_used, num, den,
                                      b.plan.threshold, b.counts[i].cpu().numpy(), b.payload[i].cpu().numpy(),
                                      b.side[i].cpu().numpy() if b.side is not None else [])
        assert host[i, :size].tobytes() == want
    back, infos = p.unpack_containers(data, b.plan)
    assert torch.equal(back.counts, b.counts) and torch.equal(back.payload, b.payload)
    if b.side is not None:
        assert torch.equal(back.side, b.side)
    assert all(inf[1:3] == (num, den) for inf in infos)
    bad = data.clone()
    bad[2, 37:39] = torch.tensor([255, 255], dtype=torch.uint8)      # one container's count > B^2
    with pytest.raises(p.FormatError):
        p.unpack_containers(bad, b.plan)
