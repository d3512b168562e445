"""Intra-image sharding: one image's block rows split over GPUs (last tier).

The batch path shards whole images and needs no collective. An image too large for one GPU, or a
single image that should use several, is split into horizontal strips of whole block rows
(shards, in block order). Everything of `sense` + `decode_idct` is per block, except the
allocation (largest_remainder_allocate, sensing.cpp:110-177), which ranks all blocks of the image.
That is the path's only exchange. Per allocation round:

    phase 1  active-weight histogram, sum of weights, active count   -> all-reduce (sum)
    phase 2  class table + threshold from the global histogram (identical everywhere);
             the shard's exact-tie blocks                           -> all-gather (prefix)
    phase 3  apply + clamp with the lower shards' tie count          -> all-reduce (taken, open)

followed by one all-gather of the shard totals for the payload offsets. The phases are the
device kernels behind `abcs_allocate_shard_step` (csrc/alloc.cu), so every shard's counts and
payload are bit-identical to the single-GPU sense of the whole image
(tests/test_sharded.py).

A process may hold several shards (`ShardComm(n_local)`): their collectives are summed locally
before the torch.distributed collective across processes (one rank per GPU, NCCL), so the
same code runs as 1 process x k shards on one GPU (the GPU tests) or as k ranks x 1 shard.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .abcs import (Algorithm, Context, LogicError, SensingConfig, UnsupportedError, _check, _ptr, _stream_ptr,
                   _torch, sense_plan)


class ShardComm:
    """Collectives over the shards of one image: n_local shards in this process, the same number
    in every rank of torch.distributed (if initialised with world size > 1); rank r holds global
    shards [r * n_local, (r + 1) * n_local)."""

    def __init__(self, n_local: int = 1, device=None, group=None):
        torch = _torch_any()
        self.n_local = int(n_local)
        self.group = group
        dist = torch.distributed
        self.dist = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        self.world = dist.get_world_size(group) if self.dist else 1
        self.rank = dist.get_rank(group) if self.dist else 0
        if device is None and self.dist and dist.get_backend(group) == "nccl":
            device = torch.device("cuda", torch.cuda.current_device())  # NCCL collectives need device tensors
        self.device = device

    @property
    def n_shards(self) -> int:
        return self.world * self.n_local

    @property
    def first(self) -> int:
        return self.rank * self.n_local

    def allreduce(self, parts):
        """Elementwise sum of one int64 tensor per local shard over all shards."""
        acc = parts[0].clone()
        for t in parts[1:]:
            acc += t
        if self.dist:
            _torch_any().distributed.all_reduce(acc, group=self.group)
        return acc

    def allgather(self, vals: Sequence[int]) -> List[int]:
        """One integer per local shard -> the list over all shards in global order."""
        if not self.dist:
            return [int(v) for v in vals]
        torch = _torch_any()
        t = torch.tensor([int(v) for v in vals], dtype=torch.int64, device=self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        torch.distributed.all_gather(out, t, group=self.group)
        return [int(x) for o in out for x in o.tolist()]


    def halo(self, fields, rows: int):
        """fields: one (h_j, W) tensor per local shard (global order). Returns per local shard
        (above, below): the last `rows` rows of the previous shard and the first `rows` of the
        next (None at the image's top / bottom). Across ranks: paired send/recv with rank +- 1."""
        n = len(fields)
        above = [fields[j - 1][-rows:] if j > 0 else None for j in range(n)]
        below = [fields[j + 1][:rows] if j + 1 < n else None for j in range(n)]
        if self.dist:
            torch = _torch_any()
            dist = torch.distributed
            ops, bufs = [], {}
            if self.rank > 0:
                bufs["up"] = torch.empty_like(fields[0][:rows])
                ops.append(dist.P2POp(dist.isend, fields[0][:rows].contiguous(), self.rank - 1, self.group))
                ops.append(dist.P2POp(dist.irecv, bufs["up"], self.rank - 1, self.group))
            if self.rank + 1 < self.world:
                bufs["down"] = torch.empty_like(fields[-1][-rows:])
                ops.append(dist.P2POp(dist.isend, fields[-1][-rows:].contiguous(), self.rank + 1, self.group))
                ops.append(dist.P2POp(dist.irecv, bufs["down"], self.rank + 1, self.group))
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
            if "up" in bufs:
                above[0] = bufs["up"]
            if "down" in bufs:
                below[-1] = bufs["down"]
        return list(zip(above, below))


def _torch_any():
    import torch
    return torch


class DeviceShard:
    """One shard's allocation state on the device (abcs_allocate_shard_step)."""

    def __init__(self, weights, wmax: int, cap: int, base: int):
        torch = _torch()
        self.w = weights.contiguous()
        self.nb = int(self.w.numel())
        self.wmax, self.cap, self.base = int(wmax), int(cap), int(base)
        lib = _lib.load()
        dev = self.w.device
        nbytes = lib.abcs_allocate_shard_scratch_bytes(self.nb, self.wmax)
        if nbytes == 0:
            raise ValueError("bad shard geometry")
        self.scratch = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
        self.out = torch.zeros(self.wmax + 3, dtype=torch.int64, device=dev)
        self.ctx = Context.get(dev.index)

    def phase(self, k: int, inp=None, remaining: int = 0, prefix: int = 0, counts=None, offsets=None):
        torch = _torch()
        _check(_lib.load().abcs_allocate_shard_step(
            self.ctx.handle, k, _ptr(self.w), self.nb, self.wmax, self.cap, self.base, self.scratch.data_ptr(),
            self.out.data_ptr(), _ptr(inp), int(remaining), int(prefix), _ptr(counts), _ptr(offsets),
            _stream_ptr(torch)))
        return self.out


def allocate_sharded(shards: Sequence, comm: ShardComm, budget: int, counts: Sequence, offsets: Sequence):
    """largest_remainder_allocate of one weight vector held as `shards` (this process's
    DeviceShard-like objects, in global order) -> counts[i] (u16) and offsets[i] (int32, global
    payload offsets; entries may be None) of each local shard. Returns the local shard totals."""
    nb_total = sum(comm.allgather([s.nb for s in shards]))
    cap = shards[0].cap
    if budget < 0 or budget > cap * nb_total or cap < 0 or cap > 65535:
        raise ValueError("allocate: budget exceeds the capacity of the blocks")
    bad = comm.allreduce([s.phase(0)[:1] for s in shards])
    if int(bad[0]):
        raise LogicError("allocate: a weight exceeds the declared bound")
    remaining = int(budget)
    taken_local = [0] * len(shards)
    rounds = 0
    while remaining > 0:
        rounds += 1
        if rounds > nb_total + 1:
            raise LogicError("allocate: no progress")
        hist = comm.allreduce([s.phase(1) for s in shards])            # exchange 1
        ties = comm.allgather([int(s.phase(2, inp=hist, remaining=remaining)[0]) for s in shards])  # exchange 2
        parts = []
        for j, s in enumerate(shards):
            g = comm.first + j
            out = s.phase(3, prefix=sum(ties[:g]))[:2].clone()
            taken_local[j] += int(out[0])
            parts.append(out)
        tk = comm.allreduce(parts)                                      # exchange 3
        remaining -= int(tk[0])
        if remaining > 0 and int(tk[1]) == 0:
            raise LogicError("allocate: capacity exhausted before budget placed")
    totals_local = [s.base * s.nb + t for s, t in zip(shards, taken_local)]
    totals = comm.allgather(totals_local)                               # payload offsets
    for j, s in enumerate(shards):
        g = comm.first + j
        s.phase(4, prefix=sum(totals[:g]), counts=counts[j], offsets=offsets[j])
    return totals_local


@dataclass
class ShardSense:
    """One shard's sense + decode: block rows [row0, row0 + rows) of the image."""
    row0: int
    rows: int
    counts: object        # (rows * cols,) uint16, the image's counts of these blocks
    offsets: object       # (rows * cols,) int32, offsets into the image's payload
    payload_offset: int   # where this shard's payload slice starts in the image's payload
    payload: object       # (its total,) float32: the image's payload[payload_offset : + total]
    decoded: Optional[object]  # (rows * B, cols * B) float32
    side: Optional[object] = None  # BBV: this shard's boundary values, side[side_offset : + len]
    side_offset: int = 0


def split_rows(rows: int, n_shards: int) -> List[int]:
    """Block-row starts of n_shards balanced strips (the last entry is `rows`)."""
    return [rows * k // n_shards for k in range(n_shards + 1)]


def sense_decode_sharded(strips: Sequence, row0s: Sequence[int], cfg: SensingConfig, height: int, width: int,
                         comm: ShardComm, decode: bool = True) -> List[ShardSense]:
    """sense (+ decode_idct) of one height x width image whose block rows are split over shards.
    strips[j]: this process's shard j as a (rows_j * B, W) uint8 CUDA tensor holding block rows
    [row0s[j], row0s[j] + rows_j) of the image; shards in global order across ranks. DD, BBV and
    ZZ sensing (after the reference's fallbacks) are supported; BBV's bottom-side probes of a
    strip's last block row read the next strip's first pixel row (a 1-row halo exchange)."""
    torch = _torch()
    plan = sense_plan(cfg, height, width)
    B, cols = plan.block, plan.cols
    if plan.algorithm_used not in (Algorithm.DD, Algorithm.ZZ, Algorithm.BBV):
        raise UnsupportedError("sharded sense: unsupported algorithm")
    lib = _lib.load()
    rows_total = plan.rows
    below_rows = comm.halo(list(strips), 1) if plan.algorithm_used == Algorithm.BBV else None
    shards, counts, offsets, strip_plans, sides = [], [], [], [], []
    for strip, r0 in zip(strips, row0s):
        if strip.dtype != torch.uint8 or strip.dim() != 2 or not strip.is_cuda or strip.shape[1] != width:
            raise ValueError("strips must be (rows * B, W) uint8 CUDA tensors")
        rows = strip.shape[0] // B
        sp = _lib.SensePlanC.from_buffer_copy(plan)  # the image's plan on the strip's block rows
        sp.rows, sp.height, sp.n_blocks = rows, rows * B, rows * cols
        strip_plans.append((sp, r0, rows))
        dev = strip.device
        counts.append(torch.empty(rows * cols, dtype=torch.uint16, device=dev))
        offsets.append(torch.empty(rows * cols, dtype=torch.int32, device=dev))
        if plan.algorithm_used == Algorithm.DD:
            w = torch.empty(rows * cols, dtype=torch.int32, device=dev)
            _check(lib.abcs_sense_weights_batch(Context.get(dev.index).handle, C.byref(sp), strip.data_ptr(),
                                                strip.numel(), width, 1, w.data_ptr(), None, _stream_ptr(torch)))
            shards.append(DeviceShard(w, plan.dd_phase1, plan.cap, plan.count_base))
        elif plan.algorithm_used == Algorithm.BBV:
            # side values of these blocks: valid probes x (top, left per block; right per block row;
            # bottom per block of the image's last block row), contiguous in block-major order
            valid = plan.bbv_valid_probes
            last = r0 + rows == rows_total
            n_side = valid * (2 * rows * cols + rows + (cols if last else 0))
            side = torch.empty(max(n_side, 1), dtype=torch.float32, device=dev)[:n_side]
            below = below_rows[len(sides)][1]
            ext = strip if last else torch.cat([strip, below[:1]]).contiguous()
            w = torch.empty(rows * cols, dtype=torch.int32, device=dev)
            _check(lib.abcs_bbv_weights_strip(Context.get(dev.index).handle, C.byref(sp), ext.data_ptr(),
                                              ext.numel(), width, 0 if last else 1, w.data_ptr(), _ptr(side),
                                              _stream_ptr(torch)))
            sides.append((side, valid * (2 * r0 * cols + r0)))
            shards.append(DeviceShard(w, 4 * valid * 255, plan.cap, plan.count_base))
    if plan.algorithm_used in (Algorithm.DD, Algorithm.BBV):
        totals_local = allocate_sharded(shards, comm, plan.alloc_budget, counts, offsets)
    else:  # ZZ: floor(M / n_B) per block, +1 for the first M mod n_B blocks (sensing.cpp:181-190)
        totals_local = []
        for c, o, (sp, r0, rows) in zip(counts, offsets, strip_plans):
            g = np.arange(r0 * cols, (r0 + rows) * cols, dtype=np.int64)
            cnt = np.minimum(plan.zz_per_block + (g < plan.zz_extra), B * B).astype(np.uint16)
            c.copy_(torch.from_numpy(cnt.view(np.int16)).view(torch.uint16))
            totals_local.append(int(cnt.sum(dtype=np.int64)))
        totals = comm.allgather(totals_local)
        for j, (c, o) in enumerate(zip(counts, offsets)):
            pre = sum(totals[:comm.first + j])
            cnt = c.view(torch.int16).to(torch.int64) & 0xFFFF
            o.copy_((torch.cumsum(cnt, 0) - cnt + pre).to(torch.int32))
    out = []
    for strip, c, o, tot, (sp, r0, rows) in zip(strips, counts, offsets, totals_local, strip_plans):
        dev = strip.device
        pay = torch.empty(max(tot, 1), dtype=torch.float32, device=dev)[:tot]
        pre = int(o[0]) if rows * cols else 0
        local_off = o - pre
        dec = torch.empty((rows * B, cols * B), dtype=torch.float32, device=dev) if decode else None
        _check(lib.abcs_gather_decode_batch(Context.get(dev.index).handle, rows, cols, B, strip.data_ptr(),
                                            strip.numel(), width, 1, _ptr(c), local_off.data_ptr(), _ptr(pay),
                                            max(tot, 1), _ptr(dec), rows * B * cols * B, cols * B,
                                            _stream_ptr(torch)))
        sd, so = sides[len(out)] if sides else (None, 0)
        out.append(ShardSense(r0, rows, c, o, pre, pay, dec, sd, so))
    return out


def ida_sharded(parts: Sequence[ShardSense], width: int, block: int, comm: ShardComm, iterations: int = 10,
                damping: float = 2.0, k: float = 2.7):
    """reconstruct() with method Ida (recon.cpp:199-259, dct_threshold denoiser) of one image
    whose block rows are split over shards: `parts` are this process's ShardSense results of
    sense_decode_sharded (global order). Per iteration the exchanges are the 4-row halo of the
    pseudo field (denoiser tiles at stride 4 straddle the strip boundaries) and the all-reduce
    of ||z||^2 for sigma = ||z|| / sqrt(M) (recon.cpp:81-93); divergence is agreed by all shards.
    Returns this process's clamped estimate strips."""
    torch = _torch()
    lib = _lib.load()
    B = block
    Wc = (width // B) * B
    cols = Wc // B
    geo = []
    for r in parts:
        dev = r.counts.device
        ctx = Context.get(dev.index).handle
        off = (r.offsets - r.payload_offset).contiguous()
        geo.append((ctx, r.rows, r.counts, off, r.payload.contiguous(), dev))
    st = _stream_ptr(torch)

    def adjoint(g, v):  # A* v: the strip's IDCT of its prefixes (operators.cpp:51-76)
        ctx, rows, cnt, off, y, dev = g
        out = torch.empty((rows * B, Wc), dtype=torch.float32, device=dev)
        _check(lib.abcs_decode_batch(ctx, rows, cols, B, _ptr(cnt), _ptr(off), _ptr(v), max(v.numel(), 1), 1,
                                     out.data_ptr(), out.numel(), Wc, None, None, st))
        return out

    def forward(g, x):  # A x (operators.cpp:23-48)
        ctx, rows, cnt, off, y, dev = g
        out = torch.empty(y.numel(), dtype=torch.float32, device=dev)
        _check(lib.abcs_forward_batch(ctx, rows, cols, B, _ptr(cnt), _ptr(off), x.data_ptr(), x.numel(), Wc, 1,
                                      _ptr(out), max(out.numel(), 1), st))
        return out

    def gsum(vals):  # fp64 sum over all shards
        return float(comm.allreduce([torch.tensor([v], dtype=torch.float64, device=g[5])
                                     for v, g in zip(vals, geo)])[0])

    M = float(sum(comm.allgather([g[4].numel() for g in geo])))
    if M <= 0:
        raise ValueError("reconstruct: no measurements")
    # warm start (recon.cpp:119-131): x0 = A* y, z0 = y - A x0, sigma0 = ||y|| / sqrt(M)
    xs = [adjoint(g, g[4]) for g in geo]
    zs = [g[4] - forward(g, x) for g, x in zip(geo, xs)]
    sigma = (gsum([float(torch.sum(g[4].double() ** 2)) for g in geo]) / M) ** 0.5
    ons = 1.0 / damping
    for it in range(1, iterations + 1):
        pseudo = [x + adjoint(g, z) for g, x, z in zip(geo, xs, zs)]       # recon.cpp:75-79
        new_x = []
        for (above, below), ps, g in zip(comm.halo(pseudo, 4), pseudo, geo):
            ext = torch.cat([t for t in (above, ps, below) if t is not None]).contiguous()
            den = torch.empty_like(ext)
            sig = (C.c_double * 1)(sigma)
            _check(lib.abcs_denoise_dct_batch(g[0], ext.data_ptr(), ext.shape[0], Wc, ext.numel(), 1, sig, k, 8,
                                              den.data_ptr(), st))
            top = 0 if above is None else above.shape[0]
            new_x.append(den[top:top + ps.shape[0]])
        xs = new_x
        zs = [(g[4] - forward(g, x)) + ons * z for g, x, z in zip(geo, xs, zs)]  # finish_step, recon.cpp:81-93
        sigma = (gsum([float(torch.sum(z.double() ** 2)) for z in zs]) / M) ** 0.5
        bad = gsum([float((~torch.isfinite(x)).any() | (x.abs() > 1e6).any() | (~torch.isfinite(z)).any())
                    for x, z in zip(xs, zs)])
        if bad:
            from .abcs import DivergenceError
            raise DivergenceError(f"reconstruct: diverged at iteration {it}", it)
    return [x.clamp(0.0, 255.0) for x in xs]                               # recon.cpp:255-257
