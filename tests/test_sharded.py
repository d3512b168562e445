"""Intra-image sharding (paper_2001_09632_b200/sharded.py).

CPU: the sharded allocation protocol (phases + collectives) over gloo with world size 2 and
several shards per rank, with each shard's phases computed by an exact pure-Python model of
the kernel phases (test-only). The result must equal the reference allocation
(largest_remainder_allocate, sensing.cpp:110-177, via the C port) of the whole vector.
GPU: the device phases (abcs_allocate_shard_step) and the sharded sense + decode of whole
images against the single-GPU path, bit for bit, as k shards in one process."""
import os
import socket
import sys
from fractions import Fraction

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rn64(q: Fraction) -> Fraction:
    """Round a non-negative rational to the nearest 64-bit-mantissa binary float (ties to even):
    the x87 long double the reference computes share in (sensing.cpp:144-148)."""
    if q == 0:
        return q
    e = q.numerator.bit_length() - q.denominator.bit_length()
    if Fraction(2) ** e > q:
        e -= 1
    scale = Fraction(2) ** (63 - e)
    m = q * scale
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return Fraction(fl) / scale


class ModelShard:
    """Exact model of one shard's kernel phases (alloc_shard_kernel) for the protocol test."""

    def __init__(self, w, wmax, cap, base):
        self.w = np.minimum(np.asarray(w, np.int64), wmax)
        self.raw = np.asarray(w, np.int64)
        self.nb, self.wmax, self.cap, self.base = len(w), wmax, cap, base
        self.a = np.zeros(self.nb, np.int64)

    def _out(self, vals):
        import torch
        out = torch.zeros(self.wmax + 3, dtype=torch.int64)
        out[:len(vals)] = torch.tensor([int(v) for v in vals], dtype=torch.int64)
        return out

    def phase(self, k, inp=None, remaining=0, prefix=0, counts=None, offsets=None):
        import torch
        act = self.a < self.cap
        if k == 0:
            self.a[:] = 0
            return self._out([int((self.raw > self.wmax).any())])
        if k == 1:
            h = np.bincount(self.w[act], minlength=self.wmax + 1)
            return torch.tensor(list(h) + [int(self.w[act].sum()), int(act.sum())], dtype=torch.int64)
        if k == 2:
            g = inp.tolist()
            T0, n_act = g[self.wmax + 1], g[self.wmax + 2]
            uniform = T0 == 0
            T = n_act if uniform else T0
            self.cls = {}
            handed = 0
            for c in range(self.wmax + 1):
                if g[c]:
                    s = rn64(Fraction(remaining * (1 if uniform else c), T))
                    whole = s.numerator // s.denominator
                    self.cls[c] = (whole, s - whole)
                    handed += g[c] * whole
            left = remaining - handed
            self.sel_all = left > 0 and left >= n_act
            self.none = left <= 0
            self.thr, self.need, self.all_eq = None, 0, False
            if not self.sel_all and not self.none:
                fr = sorted({f for _, f in self.cls.values()}, reverse=True)
                above = 0
                for f in fr:
                    eq = sum(g[c] for c, (_, ff) in self.cls.items() if ff == f)
                    if above < left <= above + eq:
                        self.thr, self.need, self.all_eq = f, left - above, left - above == eq
                        break
                    above += eq
            ties = 0
            if not self.sel_all and not self.none and not self.all_eq:
                ties = sum(1 for i in range(self.nb) if act[i] and self.cls[self.w[i]][1] == self.thr)
            return self._out([ties])
        if k == 3:
            taken = 0
            tie = prefix
            for i in range(self.nb):
                if not act[i]:
                    continue
                whole, f = self.cls[self.w[i]]
                if self.sel_all:
                    sel = True
                elif self.none:
                    sel = False
                elif f > self.thr:
                    sel = True
                elif f == self.thr:
                    sel = self.all_eq or tie < self.need
                    tie += 1
                else:
                    sel = False
                t = min(whole + int(sel), self.cap - self.a[i])
                self.a[i] += t
                taken += t
            return self._out([taken, int((self.a < self.cap).sum())])
        c = self.base + self.a
        counts[:] = torch.from_numpy(c.astype(np.int32))
        if offsets is not None:
            offsets[:] = torch.from_numpy((prefix + np.cumsum(c) - c).astype(np.int32))
        return self._out([int(c.sum())])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [  # (n blocks, wmax, cap, base, budget fraction, seed)
    (97, 12, 30, 2, 0.6, 1),      # DD-like small weights: big exact-tie groups across shards
    (64, 0, 5, 0, 0.5, 2),        # all weights zero: uniform shares
    (150, 400, 9, 0, 0.97, 3),    # many capping rounds
    (40, 7, 200, 1, 0.0, 4),      # budget 0
]


def _worker(rank, world, port, out_dir, n_local):
    import torch
    import torch.distributed as dist

    from paper_2001_09632_b200.sharded import ShardComm, allocate_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = ShardComm(n_local)
        for ci, (n, wmax, cap, base, frac, seed) in enumerate(CASES):
            rng = np.random.default_rng(seed)
            w = rng.integers(0, wmax + 1, n)
            budget = int(frac * cap * n)
            cuts = [n * k // comm.n_shards for k in range(comm.n_shards + 1)]
            mine = range(comm.first, comm.first + n_local)
            shards = [ModelShard(w[cuts[g]:cuts[g + 1]], wmax, cap, base) for g in mine]
            counts = [torch.zeros(s.nb, dtype=torch.int32) for s in shards]
            offs = [torch.zeros(s.nb, dtype=torch.int32) for s in shards]
            allocate_sharded(shards, comm, budget, counts, offs)
            np.save(os.path.join(out_dir, f"c{ci}_r{rank}.npy"),
                    np.stack([np.concatenate([c.numpy() for c in counts]), np.concatenate([o.numpy() for o in offs])]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_local", [1, 2])
def test_sharded_allocation_protocol_gloo(tmp_path, n_local):
    import torch.multiprocessing as mp

    import oracle
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), n_local), nprocs=world, join=True,
                       start_method="spawn")
    port = oracle.CPort()
    for ci, (n, wmax, cap, base, frac, seed) in enumerate(CASES):
        rng = np.random.default_rng(seed)
        w = rng.integers(0, wmax + 1, n)
        budget = int(frac * cap * n)
        got = np.concatenate([np.load(tmp_path / f"c{ci}_r{r}.npy") for r in range(world)], axis=1)
        want = base + np.asarray(port.allocate(w.astype(np.float64), budget, np.full(n, cap, np.int32)))
        assert np.array_equal(got[0], want), ci
        assert np.array_equal(got[1], np.cumsum(want) - want), ci


def _halo_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2001_09632_b200.sharded import ShardComm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = ShardComm(2)
        full = torch.arange(4 * 16 * 5, dtype=torch.float32).reshape(4 * 16, 5)   # 4 shards of 16 rows
        mine = [full[16 * g:16 * (g + 1)].clone() for g in range(comm.first, comm.first + 2)]
        res = comm.halo(mine, 4)
        z = torch.full((4, 5), -1.0)
        np.save(os.path.join(out_dir, f"h{rank}.npy"),
                np.stack([torch.stack([a if a is not None else z, b if b is not None else z]).numpy()
                          for a, b in res]))
    finally:
        dist.destroy_process_group()


def test_halo_exchange_gloo(tmp_path):
    """ShardComm.halo across 2 ranks x 2 shards: each strip gets its neighbours' edge rows."""
    import torch.multiprocessing as mp
    mp.start_processes(_halo_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    full = np.arange(4 * 16 * 5, dtype=np.float32).reshape(64, 5)
    got = np.concatenate([np.load(tmp_path / f"h{r}.npy") for r in range(2)])   # (4 shards, 2, 4, 5)
    for g in range(4):
        above = full[16 * g - 4:16 * g] if g > 0 else np.full((4, 5), -1.0)
        below = full[16 * (g + 1):16 * (g + 1) + 4] if g < 3 else np.full((4, 5), -1.0)
        assert np.array_equal(got[g, 0], above) and np.array_equal(got[g, 1], below), g


def test_rn64_rounding():
    assert rn64(Fraction(1, 3)) == Fraction(round(Fraction(2 ** 65, 3)), 2 ** 65)
    assert rn64(Fraction(7)) == 7
    assert rn64(Fraction(2 ** 64 + 1)) == 2 ** 64  # 65 significant bits round to even


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_device_shard_allocation(k, checker):
    """The device phases, k shards in one process: equal to the reference allocator
    (largest_remainder_allocate, sensing.cpp:110-177) through the oracle."""
    import torch

    import paper_2001_09632_b200 as p
    from paper_2001_09632_b200.sharded import DeviceShard, ShardComm, allocate_sharded
    rng = np.random.default_rng(10 + k)
    for n, wmax, cap, frac in [(4096, 64, 192, 0.4), (65536, 32, 224, 0.14), (3000, 2000, 40, 0.9), (500, 3, 7, 1.0)]:
        w = rng.integers(0, wmax + 1, n).astype(np.int64)
        budget = int(frac * cap * n)
        comm = ShardComm(k)
        cuts = [n * j // k for j in range(k + 1)]
        wt = torch.from_numpy(w.astype(np.int32)).cuda()
        shards = [DeviceShard(wt[cuts[j]:cuts[j + 1]], wmax, cap, 0) for j in range(k)]
        counts = [torch.empty(s.nb, dtype=torch.uint16, device="cuda") for s in shards]
        offs = [torch.empty(s.nb, dtype=torch.int32, device="cuda") for s in shards]
        allocate_sharded(shards, comm, budget, counts, offs)
        got = np.concatenate([c.cpu().numpy().view(np.uint16).astype(np.int64) for c in counts])
        want = checker.allocate(w.astype(np.float64), budget, np.full(n, cap, np.int32))
        assert np.array_equal(got, np.asarray(want, dtype=np.int64)), (n, k)
        assert np.array_equal(np.concatenate([o.cpu().numpy() for o in offs]), np.cumsum(got) - got)


@pytest.mark.gpu
@pytest.mark.parametrize("H,W,num,den,k", [(2048, 2048, 1, 4, 4), (1024, 1536, 3, 10, 3), (1000, 1000, 1, 2, 2),
                                           (512, 512, 1, 4, 1)])
def test_sharded_sense_decode_equals_whole_image(H, W, num, den, k, checker):
    """DD sense + decode of one image split into k block-row strips: counts, offsets, payload
    slices and decoded rows equal the single-GPU sense_decode_batch of the whole image, and the
    reference (oracle): counts bit-exact, payload within the fp32 bound, pixels within 1e-3."""
    import torch

    import paper_2001_09632_b200 as p
    from paper_2001_09632_b200.sharded import ShardComm, sense_decode_sharded, split_rows
    img = p.synth_images(p.SynthSpec(H, W, 30, 6.0, 21), 0, 1)
    cfg = p.SensingConfig(16, num, den, p.Algorithm.DD)
    b, x = p.sense_decode_batch(img, cfg)
    rows = b.plan.rows
    cuts = split_rows(rows, k)
    strips = [img[0, cuts[j] * 16:cuts[j + 1] * 16].contiguous() for j in range(k)]
    res = sense_decode_sharded(strips, cuts[:-1], cfg, H, W, ShardComm(k))
    cols = b.plan.cols
    for j, r in enumerate(res):
        sl = slice(cuts[j] * cols, cuts[j + 1] * cols)
        assert torch.equal(r.counts.view(torch.int16), b.counts[0, sl].view(torch.int16))
        assert torch.equal(r.offsets, b.offsets[0, sl])
        assert torch.equal(r.payload, b.payload[0, r.payload_offset:r.payload_offset + r.payload.numel()])
        assert torch.equal(r.decoded, x[0, cuts[j] * 16:cuts[j + 1] * 16])
    host = img[0].cpu().numpy()
    want = checker.sense(host, 16, num, den, 2)
    got_counts = np.concatenate([r.counts.cpu().numpy().view(np.uint16) for r in res]).astype(np.int64)
    assert np.array_equal(got_counts, want["counts"].astype(np.int64))
    got_pay = np.concatenate([r.payload.cpu().numpy() for r in res]).astype(np.float64)
    assert np.max(np.abs(got_pay - want["coeffs"])) <= 2e-3
    ref = checker.decode(rows, cols, 16, want["counts"], want["coeffs"])
    assert np.max(np.abs(torch.cat([r.decoded for r in res]).cpu().numpy() - ref)) <= 1e-3


@pytest.mark.gpu
def test_sharded_sense_zz():
    import torch

    import paper_2001_09632_b200 as p
    from paper_2001_09632_b200.sharded import ShardComm, sense_decode_sharded, split_rows
    img = p.synth_images(p.SynthSpec(512, 768, 10, 5.0, 3), 0, 1)
    cfg = p.SensingConfig(16, 1, 4, p.Algorithm.ZZ)
    b, x = p.sense_decode_batch(img, cfg)
    cuts = split_rows(b.plan.rows, 3)
    strips = [img[0, cuts[j] * 16:cuts[j + 1] * 16].contiguous() for j in range(3)]
    res = sense_decode_sharded(strips, cuts[:-1], cfg, 512, 768, ShardComm(3))
    assert torch.equal(torch.cat([r.counts.view(torch.int16) for r in res]), b.counts[0].view(torch.int16))
    assert torch.equal(torch.cat([r.decoded for r in res]), x[0])


@pytest.mark.gpu
@pytest.mark.parametrize("H,W,B,num,den,k", [(1024, 1024, 16, 3, 10, 3), (1080, 1920, 8, 1, 5, 4),
                                             (1000, 1480, 16, 1, 4, 2)])
def test_sharded_sense_bbv(H, W, B, num, den, k, checker):
    """BBV on strips (bottom probes read the next strip's first row): weights, side values,
    counts, payload and decoded rows equal the whole-image sense and the reference (oracle)."""
    import torch

    import paper_2001_09632_b200 as p
    from paper_2001_09632_b200.sharded import ShardComm, sense_decode_sharded, split_rows
    img = p.synth_images(p.SynthSpec(H, W, 25, 5.0, 13), 0, 1)
    cfg = p.SensingConfig(B, num, den, p.Algorithm.BBV)
    b, x = p.sense_decode_batch(img, cfg)
    assert b.plan.algorithm_used == p.Algorithm.BBV
    cuts = split_rows(b.plan.rows, k)
    strips = [img[0, cuts[j] * B:cuts[j + 1] * B].contiguous() for j in range(k)]
    res = sense_decode_sharded(strips, cuts[:-1], cfg, H, W, ShardComm(k))
    cols = b.plan.cols
    for j, r in enumerate(res):
        sl = slice(cuts[j] * cols, cuts[j + 1] * cols)
        assert torch.equal(r.counts.view(torch.int16), b.counts[0, sl].view(torch.int16)), j
        assert torch.equal(r.offsets, b.offsets[0, sl]), j
        assert torch.equal(r.payload, b.payload[0, r.payload_offset:r.payload_offset + r.payload.numel()]), j
        assert torch.equal(r.side, b.side[0, r.side_offset:r.side_offset + r.side.numel()]), j
        assert torch.equal(r.decoded, x[0, cuts[j] * B:cuts[j + 1] * B]), j
    assert sum(r.side.numel() for r in res) == b.side.shape[1]
    want = checker.sense(img[0].cpu().numpy(), B, num, den, 1)
    assert np.array_equal(np.concatenate([r.counts.cpu().numpy().view(np.uint16) for r in res]).astype(np.int64),
                          want["counts"].astype(np.int64))
    assert np.array_equal(np.concatenate([r.side.cpu().numpy() for r in res]).astype(np.float64), want["side"])
    ref = checker.decode(b.plan.rows, cols, B, want["counts"], want["coeffs"])
    assert np.max(np.abs(torch.cat([r.decoded for r in res]).cpu().numpy() - ref)) <= 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("H,W,k", [(1024, 768, 3), (512, 512, 2)])
def test_sharded_ida_matches_whole_image(H, W, k, checker):
    """IDA (dct_threshold) on k block-row strips with halo exchange and sigma all-reduce: the
    estimate matches the reference's reconstruct (oracle) and the single-GPU reconstruct of the
    whole image (1e-3 bar, PSNR 0.01 dB)."""
    import torch

    import paper_2001_09632_b200 as p
    from paper_2001_09632_b200.sharded import ShardComm, ida_sharded, sense_decode_sharded, split_rows
    img = p.synth_images(p.SynthSpec(H, W, 30, 6.0, 8), 0, 1)
    cfg = p.SensingConfig(16, 1, 4, p.Algorithm.DD)
    b = p.sense_batch(img, cfg)
    rc = p.ReconConfig(p.ReconMethod.Ida, iterations=6)
    whole, _, _ = p.ida_batch(b, rc, trace=False, check=True)
    cuts = split_rows(b.plan.rows, k)
    strips = [img[0, cuts[j] * 16:cuts[j + 1] * 16].contiguous() for j in range(k)]
    comm = ShardComm(k)
    parts = sense_decode_sharded(strips, cuts[:-1], cfg, H, W, comm, decode=False)
    xs = ida_sharded(parts, W, 16, comm, iterations=6)
    got = torch.cat(xs)
    diff = float((got - whole[0]).abs().max())
    assert diff <= 1e-3, diff
    ref = img[0].double()
    mse = lambda x: float(((x.double() - ref) ** 2).mean())  # noqa: E731
    assert abs(10 * np.log10(255 ** 2 / mse(got)) - 10 * np.log10(255 ** 2 / mse(whole[0]))) <= 0.01
    host = img[0].cpu().numpy()
    want = checker.sense(host, 16, 1, 4, 2)
    xr, _ = checker.reconstruct_ida(b.plan.rows, b.plan.cols, 16, want["counts"], want["coeffs"], 6, ref=host)
    assert float(np.max(np.abs(got.cpu().numpy() - xr))) <= 1e-3
    psnr_ref = 10 * np.log10(255 ** 2 / np.mean((xr - host.astype(np.float64)) ** 2))
    assert abs(10 * np.log10(255 ** 2 / mse(got)) - psnr_ref) <= 0.01


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 2])
def test_device_shard_allocation_crowded_buckets(k, checker):
    """The round threshold search by key buckets (> 64 weight classes, alloc.cu
    class_round_select): shares far below one unit put every class's key in the lowest buckets
    (65-256 classes ranked pairwise inside one bucket, or > 256 -> the radix fallback), and capped
    multi-round vectors, against the reference allocator (sensing.cpp:110-177)."""
    import torch

    from paper_2001_09632_b200.sharded import DeviceShard, ShardComm, allocate_sharded
    rng = np.random.default_rng(77 + k)
    cases = [(np.repeat(np.arange(1, 1001), 4), 1000, 255, 1),      # > 256 classes in bucket 0
             (np.repeat(np.arange(1, 1001), 4), 1000, 255, 5),      # ~170 classes per bucket
             (np.repeat(np.arange(1, 1001), 4), 1000, 255, 50),
             (np.repeat(np.arange(1, 201), 3), 200, 255, 7),
             (rng.integers(65, 4000, 4096), 4000, 120, 4096 * 40),  # capped rounds
             ((np.arange(600) % 150 + 1) * 64, 150 * 64, 200, 12345)]  # shares with equal fractions
    for w, wmax, cap, budget in cases:
        w = np.asarray(w, dtype=np.int64)
        n = w.size
        comm = ShardComm(k)
        cuts = [n * j // k for j in range(k + 1)]
        wt = torch.from_numpy(w.astype(np.int32)).cuda()
        shards = [DeviceShard(wt[cuts[j]:cuts[j + 1]], wmax, cap, 0) for j in range(k)]
        counts = [torch.empty(s.nb, dtype=torch.uint16, device="cuda") for s in shards]
        offs = [torch.empty(s.nb, dtype=torch.int32, device="cuda") for s in shards]
        allocate_sharded(shards, comm, budget, counts, offs)
        got = np.concatenate([c.cpu().numpy().view(np.uint16).astype(np.int64) for c in counts])
        want = checker.allocate(w.astype(np.float64), budget, np.full(n, cap, np.int32))
        assert np.array_equal(got, np.asarray(want, dtype=np.int64)), (n, budget, k)
