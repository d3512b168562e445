"""Host-side mirror of the reference's abcs:: C++ API (proj/core/include/abcs/*.hpp)
over the B200 C ABI (include/abcs_b200.h).

Same names, argument meaning and error behaviour as the reference:
  std::invalid_argument -> ValueError, abcs::FormatError -> FormatError,
  abcs::DivergenceError -> DivergenceError (.iteration), std::logic_error -> LogicError.
Configurations the device path does not implement raise UnsupportedError;
nothing here computes on the CPU (the oracle under oracle/ is test-only).

Single-image calls (sense, decode_idct, reconstruct, ...) take/return numpy
arrays like the reference's PixelImage/vector<double>; the *_batch calls take
and return torch CUDA tensors so batches stay resident in HBM.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import IdaConfigC, SensePlanC, SensingConfigC, SynthSpecC


# ---- errors (recon.hpp:22-30, image.hpp:12-15) -------------------------------------
class FormatError(RuntimeError):
    pass


class DivergenceError(RuntimeError):
    def __init__(self, what: str, iteration: int):
        super().__init__(what)
        self.iteration = iteration


class LogicError(RuntimeError):
    pass


class UnsupportedError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


def _check(status: int, iteration: int = 0) -> None:
    if status == _lib.OK:
        return
    msg = _lib.last_error()
    if status == _lib.INVALID:
        raise ValueError(msg)
    if status == _lib.FORMAT:
        raise FormatError(msg)
    if status == _lib.DIVERGENCE:
        raise DivergenceError(msg, iteration)
    if status == _lib.LOGIC:
        raise LogicError(msg)
    if status == _lib.UNSUPPORTED:
        raise UnsupportedError(msg)
    raise CudaError(msg)


# ---- enums (sensing.hpp:12, recon.hpp:14) --------------------------------------------
class Algorithm(enum.IntEnum):
    ZZ = 0
    BBV = 1
    DD = 2


class ReconMethod(enum.IntEnum):
    Idct = 0
    Ista = 1
    Amp = 2
    Damp = 3
    DampD = 4
    Ida = 5


_ALGO_NAMES = {Algorithm.ZZ: "zz", Algorithm.BBV: "bbv", Algorithm.DD: "dd"}
_METHOD_NAMES = {ReconMethod.Idct: "idct", ReconMethod.Ista: "ista", ReconMethod.Amp: "amp",
                 ReconMethod.Damp: "damp", ReconMethod.DampD: "dampd", ReconMethod.Ida: "ida"}


def algorithm_name(a: Algorithm) -> str:
    return _ALGO_NAMES.get(Algorithm(a), "?")


def algorithm_from_name(name: str) -> Optional[Algorithm]:
    for k, v in _ALGO_NAMES.items():
        if v == name:
            return k
    return None


def recon_method_name(m: ReconMethod) -> str:
    return _METHOD_NAMES.get(ReconMethod(m), "?")


def recon_method_from_name(name: str) -> Optional[ReconMethod]:
    for k, v in _METHOD_NAMES.items():
        if v == name:
            return k
    return None


# ---- grid (image.hpp:35-46, image.cpp:106-116) ---------------------------------------
@dataclass(frozen=True)
class BlockGrid:
    block: int = 0
    rows: int = 0
    cols: int = 0

    def count(self) -> int:
        return self.rows * self.cols

    def cropped_height(self) -> int:
        return self.rows * self.block

    def cropped_width(self) -> int:
        return self.cols * self.block

    def pixel_count(self) -> int:
        return self.count() * self.block * self.block


def make_grid(height: int, width: int, block: int) -> BlockGrid:
    if block < 2:
        raise ValueError("block size must be >= 2")
    if block > height or block > width:
        raise ValueError("block size exceeds image dimensions")
    return BlockGrid(block, height // block, width // block)


# ---- SensingConfig (sensing.hpp:20-40) -----------------------------------------------
@dataclass
class SensingConfig:
    block: int = 32
    cr_num: int = 1
    cr_den: int = 1
    algorithm: Algorithm = Algorithm.ZZ
    threshold: Optional[float] = None

    def cr(self) -> float:
        return self.cr_num / self.cr_den

    def cf(self) -> float:
        return self.cr_den / self.cr_num

    def cf_floor(self) -> int:
        return self.cr_den // self.cr_num

    def validate(self) -> None:
        if self.block < 2 or self.block > 255:
            raise ValueError("block size must be in [2, 255]")
        if self.cr_num == 0 or self.cr_den == 0:
            raise ValueError("C_R must be positive")
        if self.cr_num > self.cr_den:
            raise ValueError("C_R must be in (0, 1]")
        if self.threshold is not None and self.threshold < 0:
            raise ValueError("threshold must be >= 0")

    def target_measurements(self, total_pixels: int) -> int:
        return (self.cr_num * total_pixels) // self.cr_den

    @staticmethod
    def parse_ratio(text: str) -> Tuple[int, int]:
        num, den = C.c_uint32(), C.c_uint32()
        _check(_lib.load().abcs_parse_ratio(text.encode(), C.byref(num), C.byref(den)))
        return num.value, den.value

    def set_cr(self, num_or_text, den: Optional[int] = None) -> "SensingConfig":
        if den is None:
            self.cr_num, self.cr_den = self.parse_ratio(str(num_or_text))
        else:
            import math
            g = math.gcd(int(num_or_text), int(den))
            if g == 0:
                raise ValueError("C_R must be positive")
            self.cr_num, self.cr_den = int(num_or_text) // g, int(den) // g
        return self

    def _c(self) -> SensingConfigC:
        c = SensingConfigC()
        c.block = self.block
        c.cr_num = self.cr_num
        c.cr_den = self.cr_den
        c.algorithm = int(self.algorithm)
        c.has_threshold = 1 if self.threshold is not None else 0
        c.threshold = float(self.threshold) if self.threshold is not None else 0.0
        return c


def sense_plan(cfg: SensingConfig, height: int, width: int) -> SensePlanC:
    """Every derivation abcs::sense makes from (config, size) — host logic, no GPU."""
    plan = SensePlanC()
    c = cfg._c()
    _check(_lib.load().abcs_sense_plan_init(C.byref(c), int(height), int(width), C.byref(plan)))
    return plan


def dd_threshold(image_height: int, cr_num: int, cr_den: int) -> float:
    return _lib.load().abcs_dd_threshold(int(image_height), int(cr_num), int(cr_den))


@dataclass
class ZigzagOrder:
    block: int
    index: np.ndarray
    rank: np.ndarray


def zigzag_order(block: int) -> ZigzagOrder:
    idx = np.zeros(block * block, dtype=np.int32)
    _check(_lib.load().abcs_zigzag_order(block, idx.ctypes.data))
    rank = np.zeros_like(idx)
    rank[idx] = np.arange(idx.size, dtype=np.int32)
    return ZigzagOrder(block, idx, rank)


# ---- MeasurementSet (sensing.hpp:74-88) ----------------------------------------------
@dataclass
class MeasurementSet:
    height: int = 0
    width: int = 0
    block: int = 0
    algorithm: Algorithm = Algorithm.ZZ
    cr_num: int = 1
    cr_den: int = 1
    threshold: float = 0.0
    counts: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint16))
    coeffs: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    side: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    def grid(self) -> BlockGrid:
        return make_grid(self.height, self.width, self.block)

    def total_coeffs(self) -> int:
        return int(np.asarray(self.counts, dtype=np.int64).sum())


@dataclass
class BudgetSummary:
    target: int = 0
    actual: int = 0


def measurement_budget(ms: MeasurementSet) -> BudgetSummary:
    """sensing.cpp:472-487"""
    g = ms.grid()
    target = (ms.cr_num * g.pixel_count()) // ms.cr_den
    actual = ms.total_coeffs()
    if ms.algorithm == Algorithm.BBV:
        L = ms.cr_den // ms.cr_num
        if 1 <= L <= g.block:
            per_side = g.block // L
            extent = g.cropped_height() + g.cropped_width()
            actual += 2 * per_side * g.count() + (extent + L - 1) // L
    return BudgetSummary(target, actual)


# ---- device plumbing -------------------------------------------------------------------
class Context:
    """One abcs_ctx per CUDA device (thread-safe lazily created singletons)."""

    _ctxs = {}

    def __init__(self, device: int):
        self.device = device
        self.handle = C.c_void_p()
        _check(_lib.load().abcs_ctx_create(device, C.byref(self.handle)))

    @classmethod
    def get(cls, device: Optional[int] = None) -> "Context":
        import torch
        if device is None:
            device = torch.cuda.current_device()
        ctx = cls._ctxs.get(device)
        if ctx is None:
            ctx = cls(device)
            cls._ctxs[device] = ctx
        return ctx

    def launches(self) -> int:
        return int(_lib.load().abcs_ctx_launch_count(self.handle))

    def set_pipeline_streams(self, streams: int) -> None:
        """Chunked batch pipelining width (1..3; 1 serialises the kernels of a batch call)."""
        _check(_lib.load().abcs_ctx_set_pipeline_streams(self.handle, int(streams)))

    def kernel_timing(self, enable: bool) -> None:
        """Start (clearing) or stop per-kernel CUDA-event timing on this context."""
        _check(_lib.load().abcs_ctx_kernel_timing(self.handle, 1 if enable else 0))

    def kernel_times(self) -> dict:
        """{kernel name: (launches, total_ms, max_ms)} recorded since kernel_timing(True); synchronizes."""
        cap = 64
        buf = (_lib.KernelTimeC * cap)()
        cnt = C.c_int32()
        _check(_lib.load().abcs_ctx_kernel_times(self.handle, buf, cap, C.byref(cnt)))
        return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms), float(buf[i].max_ms))
                for i in range(min(cnt.value, cap))}


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise CudaError("no CUDA device: the ABCS path runs on B200 only (no CPU fallback)")
    return torch


def _stream_ptr(torch) -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _as_u8_image(img) -> np.ndarray:
    a = np.asarray(img)
    if a.ndim != 2:
        raise ValueError("image must be 2-D (height, width)")
    if a.dtype == np.uint8:
        return np.ascontiguousarray(a)
    f = a.astype(np.float64)
    if not np.all(np.isfinite(f)) or np.any(f != np.round(f)) or f.min() < 0 or f.max() > 255:
        raise ValueError("device sensing requires integer pixel values in [0, 255] (8-bit images)")
    return np.ascontiguousarray(f.astype(np.uint8))


# ---- batched device API ---------------------------------------------------------------
@dataclass
class MeasurementBatch:
    """n MeasurementSets of one image size, resident on the GPU."""
    plan: SensePlanC
    cfg: SensingConfig
    counts: "object"   # torch.uint16 (n, n_blocks)
    offsets: "object"  # torch.int32 (n, n_blocks)
    payload: "object"  # torch.float32 (n, K)
    side: "object"     # torch.float32 (n, S) or None

    @property
    def n(self) -> int:
        return self.counts.shape[0]

    def grid(self) -> BlockGrid:
        return BlockGrid(self.plan.block, self.plan.rows, self.plan.cols)

    def to_host(self, i: int) -> MeasurementSet:
        p = self.plan
        return MeasurementSet(
            height=p.height, width=p.width, block=p.block, algorithm=Algorithm(p.algorithm_used),
            cr_num=p.cr_num, cr_den=p.cr_den, threshold=p.threshold,
            counts=self.counts[i].cpu().numpy().astype(np.uint16),
            coeffs=self.payload[i].cpu().numpy(),
            side=(self.side[i].cpu().numpy() if self.side is not None else np.zeros(0, np.float32)))


def sense_batch(images, cfg: SensingConfig, plan: Optional[SensePlanC] = None,
                out: Optional[MeasurementBatch] = None) -> MeasurementBatch:
    """abcs::sense on a (n, H, W) uint8 CUDA tensor (sensing.cpp:418-470)."""
    torch = _torch()
    if images.dtype != torch.uint8 or images.dim() != 3 or not images.is_cuda:
        raise ValueError("images must be a (n, H, W) uint8 CUDA tensor")
    n, H, W = images.shape
    if plan is None:
        plan = sense_plan(cfg, H, W)
    dev = images.device
    if out is None:
        K, S, NB = plan.coeffs_per_image, plan.side_per_image, plan.n_blocks
        out = MeasurementBatch(
            plan=plan, cfg=cfg,
            counts=torch.empty((n, NB), dtype=torch.uint16, device=dev),
            offsets=torch.empty((n, NB), dtype=torch.int32, device=dev),
            payload=torch.empty((n, max(K, 1)), dtype=torch.float32, device=dev)[:, :K],
            side=torch.empty((n, S), dtype=torch.float32, device=dev) if S > 0 else None)
    images = images.contiguous()
    ctx = Context.get(dev.index)
    _check(_lib.load().abcs_sense_batch(
        ctx.handle, C.byref(plan), images.data_ptr(), H * W, W, n, _ptr(out.counts), _ptr(out.offsets),
        _ptr(out.payload), _ptr(out.side), _stream_ptr(torch)))
    return out


def sense_decode_batch(images, cfg: SensingConfig, plan: Optional[SensePlanC] = None,
                       out: Optional[MeasurementBatch] = None, image_out=None):
    """sense then decode_idct on a (n, H, W) uint8 CUDA tensor in one fused pass over the
    payload; returns (MeasurementBatch, (n, Hc, Wc) float32 decoded images)."""
    torch = _torch()
    if images.dtype != torch.uint8 or images.dim() != 3 or not images.is_cuda:
        raise ValueError("images must be a (n, H, W) uint8 CUDA tensor")
    n, H, W = images.shape
    if plan is None:
        plan = sense_plan(cfg, H, W)
    dev = images.device
    if out is None:
        K, S, NB = plan.coeffs_per_image, plan.side_per_image, plan.n_blocks
        out = MeasurementBatch(
            plan=plan, cfg=cfg,
            counts=torch.empty((n, NB), dtype=torch.uint16, device=dev),
            offsets=torch.empty((n, NB), dtype=torch.int32, device=dev),
            payload=torch.empty((n, max(K, 1)), dtype=torch.float32, device=dev)[:, :K],
            side=torch.empty((n, S), dtype=torch.float32, device=dev) if S > 0 else None)
    Hc, Wc = plan.rows * plan.block, plan.cols * plan.block
    if image_out is None:
        image_out = torch.empty((n, Hc, Wc), dtype=torch.float32, device=dev)
    images = images.contiguous()
    ctx = Context.get(dev.index)
    _check(_lib.load().abcs_sense_decode_batch(
        ctx.handle, C.byref(plan), images.data_ptr(), H * W, W, n, _ptr(out.counts), _ptr(out.offsets),
        _ptr(out.payload), _ptr(out.side), image_out.data_ptr(), Hc * Wc, Wc, _stream_ptr(torch)))
    return out, image_out


def sense_decode_sweep(images, cfgs, outs=None, image_outs=None):
    """sense_decode_batch of the same (n, H, W) uint8 CUDA images under each config of cfgs
    (a subrate sweep, as the reference bench's --crs loop, tools/abcs_main.cpp:215-260).
    DD B=16 sweeps share DD phase 1's forward transform; each config's outputs are identical
    to its own sense_decode_batch call. Returns [(MeasurementBatch, decoded images)]."""
    torch = _torch()
    if images.dtype != torch.uint8 or images.dim() != 3 or not images.is_cuda:
        raise ValueError("images must be a (n, H, W) uint8 CUDA tensor")
    cfgs = list(cfgs)
    if not cfgs:
        return []
    n, H, W = images.shape
    dev = images.device
    plans = [sense_plan(c, H, W) for c in cfgs]
    Hc, Wc = plans[0].rows * plans[0].block, plans[0].cols * plans[0].block
    if any(q.rows * q.block != Hc or q.cols * q.block != Wc for q in plans):
        raise ValueError("sweep configs must crop the images to the same grid")
    if outs is None:
        outs = []
        for c, q in zip(cfgs, plans):
            K, S, NB = q.coeffs_per_image, q.side_per_image, q.n_blocks
            outs.append(MeasurementBatch(
                plan=q, cfg=c,
                counts=torch.empty((n, NB), dtype=torch.uint16, device=dev),
                offsets=torch.empty((n, NB), dtype=torch.int32, device=dev),
                payload=torch.empty((n, max(K, 1)), dtype=torch.float32, device=dev)[:, :K],
                side=torch.empty((n, S), dtype=torch.float32, device=dev) if S > 0 else None))
    if image_outs is None:
        image_outs = [torch.empty((n, Hc, Wc), dtype=torch.float32, device=dev) for _ in cfgs]
    images = images.contiguous()
    m = len(cfgs)
    parr = (SensePlanC * m)(*plans)
    arr = lambda xs: (C.c_void_p * m)(*[_ptr(x) for x in xs])  # noqa: E731
    ctx = Context.get(dev.index)
    _check(_lib.load().abcs_sense_decode_sweep_batch(
        ctx.handle, parr, m, images.data_ptr(), H * W, W, n, arr([o.counts for o in outs]),
        arr([o.offsets for o in outs]), arr([o.payload for o in outs]), arr([o.side for o in outs]),
        arr(image_outs), Hc * Wc, Wc, _stream_ptr(torch)))
    return list(zip(outs, image_outs))


def bench_cells_host(images, cfgs, device=0, chunk=64, ssim=True):
    """The reference bench step (tools/abcs_main.cpp:226-258) from HOST images: sense + IDCT
    decode under each config, then mse/psnr/ssim of every decoded image against the input
    cropped to the block grid (metrics.cpp:63-125). images: (n, H, W) uint8 CPU tensor (pin it
    for full PCIe rate). Only the cells come back: dict of (len(cfgs), n) float64 tensors."""
    torch = _torch()
    if images.dtype != torch.uint8 or images.dim() != 3 or images.is_cuda:
        raise ValueError("images must be a (n, H, W) uint8 CPU tensor")
    cfgs = list(cfgs)
    n, H, W = images.shape
    plans = [sense_plan(c, H, W) for c in cfgs]
    m = len(plans)
    images = images.contiguous()
    cells = {k: torch.empty((m, n), dtype=torch.float64) for k in (("mse", "psnr", "ssim") if ssim else ("mse", "psnr"))}
    ctx = Context.get(device)
    _check(_lib.load().abcs_bench_cells_host(
        ctx.handle, (SensePlanC * m)(*plans), m, images.data_ptr(), n, cells["mse"].data_ptr(),
        cells["psnr"].data_ptr(), cells["ssim"].data_ptr() if ssim else None, chunk))
    return cells


def block_dct_batch(blocks, inverse: bool = False):
    """BlockDct::forward / inverse (dct.cpp:9-79) on a (n, B, B) float64 device tensor, any B >= 1:
    fp64, bit-identical to the reference (abcs_block_dct_f64)."""
    torch = _torch()
    if blocks.dim() != 3 or blocks.shape[1] != blocks.shape[2] or blocks.dtype != torch.float64:
        raise ValueError("block_dct_batch: expects (n, B, B) float64")
    x = blocks.contiguous()
    out = torch.empty_like(x)
    _check(_lib.load().abcs_block_dct_f64(Context.get(x.device.index).handle, x.shape[1], 1 if inverse else 0,
                                          _ptr(x), _ptr(out), x.shape[0], _stream_ptr(torch)))
    return out


def dct2(block, size: int) -> np.ndarray:
    """abcs::dct2 (dct.hpp:30): one size x size block (row-major values), on the device."""
    torch = _torch()
    b = torch.as_tensor(np.asarray(block, np.float64).reshape(1, size, size), device="cuda")
    return block_dct_batch(b).reshape(-1).cpu().numpy()


def idct2(coeffs, size: int) -> np.ndarray:
    """abcs::idct2 (dct.hpp:31)."""
    torch = _torch()
    b = torch.as_tensor(np.asarray(coeffs, np.float64).reshape(1, size, size), device="cuda")
    return block_dct_batch(b, inverse=True).reshape(-1).cpu().numpy()


def decode_batch(batch: MeasurementBatch, out=None):
    """decode_idct on every set of the batch -> (n, Hc, Wc) float32 CUDA tensor."""
    torch = _torch()
    p = batch.plan
    Hc, Wc = p.rows * p.block, p.cols * p.block
    if out is None:
        out = torch.empty((batch.n, Hc, Wc), dtype=torch.float32, device=batch.counts.device)
    ctx = Context.get(batch.counts.device.index)
    _check(_lib.load().abcs_decode_batch(
        ctx.handle, p.rows, p.cols, p.block, _ptr(batch.counts), _ptr(batch.offsets), _ptr(batch.payload),
        batch.payload.stride(0) if batch.payload.numel() else p.coeffs_per_image, batch.n,
        out.data_ptr(), Hc * Wc, Wc, None, None, _stream_ptr(torch)))
    return out


@dataclass
class TraceRow:
    iteration: int = 0
    residual_norm: float = 0.0
    sigma: float = 0.0
    psnr_db: float = float("nan")


@dataclass
class DenoiserSpec:
    name: str = "dct_threshold"
    params: dict = field(default_factory=dict)

    def param(self, key: str, fallback: float) -> float:
        return float(self.params.get(key, fallback))


@dataclass
class ReconConfig:
    method: ReconMethod = ReconMethod.Idct
    iterations: int = 15
    damping: float = 2.0
    denoiser: DenoiserSpec = field(default_factory=DenoiserSpec)
    lambda_: float = 1.0
    seed: int = 42

    def validate(self) -> None:
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")
        if self.damping < 1.0:
            raise ValueError("damping factor D_F must be >= 1")
        if self.lambda_ < 0.0:
            raise ValueError("lambda must be >= 0")

    def _ida_c(self) -> IdaConfigC:
        if self.denoiser.name != "dct_threshold":
            raise UnsupportedError(f"device IDA implements the dct_threshold denoiser, not '{self.denoiser.name}'")
        c = IdaConfigC()
        c.iterations = self.iterations
        c.denoiser_block = int(self.denoiser.param("block", 8.0))
        c.damping = self.damping
        c.k = self.denoiser.param("k", 2.7)
        return c


def ida_batch(batch: MeasurementBatch, cfg: ReconConfig, reference=None, out=None, trace: bool = True,
              check: bool = True):
    """reconstruct(method=Ida) on every set: returns (images (n,Hc,Wc) f32, trace (n,T,4) f64 | None,
    diverged (n,2) int32). With check=True, synchronizes and raises DivergenceError."""
    torch = _torch()
    cfg.validate()
    p = batch.plan
    Hc, Wc = p.rows * p.block, p.cols * p.block
    dev = batch.counts.device
    if out is None:
        out = torch.empty((batch.n, Hc, Wc), dtype=torch.float32, device=dev)
    tr = torch.empty((batch.n, cfg.iterations + 1, 4), dtype=torch.float64, device=dev) if trace else None
    div = torch.zeros((batch.n, 2), dtype=torch.int32, device=dev)
    ref_ptr, ref_stride, ref_pitch = None, 0, 0
    if reference is not None:
        if reference.dtype != torch.uint8 or reference.dim() != 3:
            raise ValueError("reference must be a (n, H, W) uint8 CUDA tensor")
        if reference.shape[1] < Hc or reference.shape[2] < Wc:
            raise ValueError("reconstruct: reference smaller than decoded image")
        reference = reference.contiguous()
        ref_ptr, ref_stride, ref_pitch = reference.data_ptr(), reference.shape[1] * reference.shape[2], reference.shape[2]
    c = cfg._ida_c()
    ctx = Context.get(dev.index)
    _check(_lib.load().abcs_ida_batch(
        ctx.handle, p.rows, p.cols, p.block, _ptr(batch.counts), _ptr(batch.offsets), _ptr(batch.payload),
        batch.payload.stride(0) if batch.payload.numel() else p.coeffs_per_image, batch.n, C.byref(c),
        ref_ptr, ref_stride, ref_pitch, out.data_ptr(), Hc * Wc, Wc, _ptr(tr), div.data_ptr(), _stream_ptr(torch)))
    if check:
        h = div.cpu().numpy()
        first = C.c_int32()
        st = _lib.load().abcs_ida_check(h.ctypes.data, batch.n, C.byref(first))
        if st != _lib.OK:
            _check(st, iteration=int(h[first.value, 0]))
    return out, tr, div


_DENOISERS = {"dct_threshold": 0, "blur": 1, "identity": 2}


def _recon_c(cfg: "ReconConfig", method=None, denoiser: "DenoiserSpec" = None):
    d = cfg.denoiser if denoiser is None else denoiser
    if d.name not in _DENOISERS:
        raise ValueError(f"unknown denoiser: '{d.name}'")
    c = _lib.ReconConfigC()
    c.method = int(cfg.method if method is None else method)
    c.iterations = cfg.iterations
    c.damping = cfg.damping
    c.lambda_ = cfg.lambda_
    c.seed = cfg.seed
    c.denoiser = _DENOISERS[d.name]
    c.denoiser_block = int(d.param("block", 8.0))
    c.k = d.param("k", 2.7)
    c.sigma_scale = d.param("sigma_scale", 25.0)
    return c


def recon_batch(batch: MeasurementBatch, cfg: ReconConfig, reference=None, out=None, trace: bool = True,
                check: bool = True):
    """reconstruct() for every set with any method (Ista/Amp/Damp/DampD/Ida with any denoiser):
    (images (n,Hc,Wc) f32, trace (n,T,4) f64 | None, diverged (n,2) int32)."""
    torch = _torch()
    cfg.validate()
    p = batch.plan
    Hc, Wc = p.rows * p.block, p.cols * p.block
    dev = batch.counts.device
    if out is None:
        out = torch.empty((batch.n, Hc, Wc), dtype=torch.float32, device=dev)
    tr = torch.empty((batch.n, cfg.iterations + 1, 4), dtype=torch.float64, device=dev) if trace else None
    div = torch.zeros((batch.n, 2), dtype=torch.int32, device=dev)
    ref_ptr, ref_stride, ref_pitch = None, 0, 0
    if reference is not None:
        if reference.dtype != torch.uint8 or reference.dim() != 3:
            raise ValueError("reference must be a (n, H, W) uint8 CUDA tensor")
        if reference.shape[1] < Hc or reference.shape[2] < Wc:
            raise ValueError("reconstruct: reference smaller than decoded image")
        reference = reference.contiguous()
        ref_ptr, ref_stride, ref_pitch = reference.data_ptr(), reference.shape[1] * reference.shape[2], reference.shape[2]
    c = _recon_c(cfg)
    _check(_lib.load().abcs_reconstruct_batch(
        Context.get(dev.index).handle, p.rows, p.cols, p.block, _ptr(batch.counts), _ptr(batch.offsets),
        _ptr(batch.payload), batch.payload.stride(0) if batch.payload.numel() else p.coeffs_per_image, batch.n,
        C.byref(c), ref_ptr, ref_stride, ref_pitch, out.data_ptr(), Hc * Wc, Wc, _ptr(tr), div.data_ptr(),
        _stream_ptr(torch)))
    if check:
        h = div.cpu().numpy()
        first = C.c_int32()
        st = _lib.load().abcs_ida_check(h.ctypes.data, batch.n, C.byref(first))
        if st != _lib.OK:
            _check(st, iteration=int(h[first.value, 0]))
    return out, tr, div


# ---- single-image API (reference signatures) -------------------------------------------
def _batch_from_host(ms: MeasurementSet, coeffs=None) -> MeasurementBatch:
    torch = _torch()
    g = ms.grid()
    counts = np.ascontiguousarray(np.asarray(ms.counts, dtype=np.uint16))
    if counts.size != g.count():
        raise ValueError("SensingOperator: counts/grid mismatch")
    if np.any(counts.astype(np.int64) > g.block * g.block):
        raise ValueError("SensingOperator: count exceeds B^2")
    y = np.ascontiguousarray(np.asarray(ms.coeffs if coeffs is None else coeffs, dtype=np.float32))
    plan = SensePlanC()
    plan.height, plan.width, plan.block = ms.height, ms.width, ms.block
    plan.rows, plan.cols, plan.n_blocks = g.rows, g.cols, g.count()
    plan.algorithm = plan.algorithm_used = int(ms.algorithm)
    plan.cr_num, plan.cr_den, plan.threshold = ms.cr_num, ms.cr_den, ms.threshold
    plan.coeffs_per_image = y.size
    dev = torch.device("cuda", torch.cuda.current_device())
    ct = torch.from_numpy(counts.view(np.int16)).to(dev).view(torch.uint16).reshape(1, -1)
    off = np.zeros(counts.size, dtype=np.int32)
    if counts.size > 1:
        off[1:] = np.cumsum(counts.astype(np.int64))[:-1]
    ot = torch.from_numpy(off).to(dev).reshape(1, -1)
    yt = torch.from_numpy(y).to(dev).reshape(1, -1)
    return MeasurementBatch(plan=plan, cfg=SensingConfig(ms.block, ms.cr_num, ms.cr_den, Algorithm(ms.algorithm)),
                            counts=ct, offsets=ot, payload=yt, side=None)


def sense(img, cfg: SensingConfig, warning: Optional[List[str]] = None) -> MeasurementSet:
    """abcs::sense (sensing.hpp:98-99). `warning`, if a list, receives the fallback notes."""
    torch = _torch()
    cfg.validate()
    a = _as_u8_image(img)
    plan = sense_plan(cfg, a.shape[0], a.shape[1])
    if warning is not None:
        if plan.algorithm == Algorithm.ZZ and plan.zz_last_zero:
            warning.append("C_R is so low that some blocks receive zero coefficients")
        if plan.fallback == 1:
            warning.append("full-rate sensing leaves nothing to adapt; reverting to non-adaptive zz")
        elif plan.fallback == 2:
            warning.append(f"floor(C_F) = {cfg.cf_floor()} exceeds block size {cfg.block}; "
                           "reverting to non-adaptive zz")
        elif plan.fallback == 3:
            warning.append("phase-1 budget floor(B^2/(2 C_F)) is zero at this C_R; reverting to non-adaptive zz")
    dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.from_numpy(a).to(dev).reshape(1, *a.shape)
    b = sense_batch(t, cfg, plan)
    ms = b.to_host(0)
    ms.cr_num, ms.cr_den = cfg.cr_num, cfg.cr_den
    return ms


def sense_zz(img, cfg: SensingConfig) -> MeasurementSet:
    c = SensingConfig(cfg.block, cfg.cr_num, cfg.cr_den, Algorithm.ZZ, cfg.threshold)
    return sense(img, c)


def sense_dd(img, cfg: SensingConfig) -> MeasurementSet:
    plan = sense_plan(SensingConfig(cfg.block, cfg.cr_num, cfg.cr_den, Algorithm.DD, cfg.threshold), *np.shape(img))
    if plan.dd_phase1 == 0:
        raise UnsupportedError("sense_dd with a zero phase-1 budget (the reference divides by zero-size phases)")
    return sense(img, SensingConfig(cfg.block, cfg.cr_num, cfg.cr_den, Algorithm.DD, cfg.threshold))


@dataclass
class BbvParams:
    stride: int = 0
    offset: int = 0
    per_side: int = 0
    phase1_total: int = 0
    variation: np.ndarray = field(default_factory=lambda: np.zeros(0))
    side_values: np.ndarray = field(default_factory=lambda: np.zeros(0))


def bbv_measure(img, cfg: SensingConfig) -> BbvParams:
    """abcs::bbv_measure (sensing.cpp:239-296) via the device phase-1 kernel."""
    torch = _torch()
    cfg.validate()
    a = _as_u8_image(img)
    H, W = a.shape
    g = make_grid(H, W, cfg.block)
    L = cfg.cf_floor()
    out = BbvParams(stride=L, offset=L // 2, per_side=0 if L > g.block else g.block // L,
                    variation=np.zeros(g.count()))
    if out.per_side == 0:
        return out
    extent = g.cropped_height() + g.cropped_width()
    out.phase1_total = 2 * out.per_side * g.count() + (extent + L - 1) // L
    plan = SensePlanC()
    plan.height, plan.width, plan.block = H, W, g.block
    plan.rows, plan.cols, plan.n_blocks = g.rows, g.cols, g.count()
    plan.algorithm = plan.algorithm_used = int(Algorithm.BBV)
    plan.bbv_stride, plan.bbv_offset, plan.bbv_per_side = L, L // 2, out.per_side
    valid = sum(1 for j in range(out.per_side) if not ((L // 2 + j * L) < 1 or (L // 2 + j * L) + 1 > g.block))
    plan.bbv_valid_probes = valid
    plan.side_per_image = valid * (2 * g.count() + g.cols + g.rows)
    dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.from_numpy(a).to(dev)
    w = torch.empty(g.count(), dtype=torch.int32, device=dev)
    side = torch.empty(max(plan.side_per_image, 1), dtype=torch.float32, device=dev)
    _check(_lib.load().abcs_sense_weights_batch(Context.get(dev.index).handle, C.byref(plan), t.data_ptr(),
                                                H * W, W, 1, w.data_ptr(), side.data_ptr(), _stream_ptr(torch)))
    out.variation = w.cpu().numpy().astype(np.float64)
    out.side_values = side[:plan.side_per_image].cpu().numpy().astype(np.float64)
    return out


def largest_remainder_allocate(weights: Sequence[float], budget: int, caps: Sequence[int]) -> np.ndarray:
    """abcs::largest_remainder_allocate (sensing.cpp:110-177), bit-exact on device.
    Weights must be integer valued (< 2^32): the reference's x87 ranking is emulated exactly for those."""
    torch = _torch()
    w = np.asarray(weights, dtype=np.float64)
    cp = np.asarray(caps, dtype=np.int64)
    if cp.size != w.size:
        raise ValueError("allocate: weights/caps size mismatch")
    if budget < 0:
        raise ValueError("allocate: negative budget")
    if np.any(w < 0) or not np.all(np.isfinite(w)):
        raise ValueError("allocate: weights must be finite and >= 0")
    if np.any(cp < 0):
        raise ValueError("allocate: negative cap")
    if budget > int(cp.sum()):
        raise ValueError("allocate: budget exceeds capacity")
    if np.any(w != np.floor(w)) or np.any(w >= 2.0 ** 32) or np.any(cp > 65535):
        raise UnsupportedError("device allocator takes integer weights < 2^32 and caps <= 65535")
    n = w.size
    if n == 0:
        return np.zeros(0, dtype=np.int32)
    dev = torch.device("cuda", torch.cuda.current_device())
    wt = torch.from_numpy(w.astype(np.uint32).view(np.int32)).to(dev)
    ct = torch.from_numpy(cp.astype(np.int32)).to(dev)
    counts = torch.empty(n, dtype=torch.int16, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _check(_lib.load().abcs_allocate_batch(Context.get(dev.index).handle, wt.data_ptr(), n, 1, int(budget),
                                           ct.data_ptr(), 0, 0, counts.data_ptr(), None, status.data_ptr(),
                                           _stream_ptr(torch)))
    st = int(status.item())
    if st != _lib.OK:
        raise {1: ValueError, 5: LogicError}.get(st, RuntimeError)(
            "allocate: budget exceeds capacity" if st == 1 else "allocate: capacity exhausted before budget placed")
    return counts.cpu().numpy().view(np.uint16).astype(np.int32)


@dataclass
class AllocationPlan:
    block_size: int = 0
    phase1_is_dct: bool = False
    phase1: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    phase2: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    target: int = 0
    shared_overhead: int = 0

    def actual(self) -> int:
        return int(self.shared_overhead + self.phase1.sum() + self.phase2.sum())

    def coeff_count(self, i: int) -> int:
        return int((self.phase1[i] if self.phase1_is_dct else 0) + self.phase2[i])


def allocate_bbv(bbv: BbvParams, total_budget: int, n_blocks: int, block: int) -> AllocationPlan:
    """sensing.cpp:298-321"""
    if len(bbv.variation) != n_blocks:
        raise ValueError("allocate_bbv: variation/block count mismatch")
    if total_budget <= bbv.phase1_total:
        raise ValueError("allocate_bbv: measurement budget does not cover the phase-1 probes (M <= M_BBV)")
    per_block = 2 * bbv.per_side
    cap = block * block - per_block
    if cap < 0:
        raise ValueError("allocate_bbv: probes exceed block capacity")
    phase2 = largest_remainder_allocate(bbv.variation, total_budget - bbv.phase1_total, [cap] * n_blocks)
    return AllocationPlan(block_size=block, phase1_is_dct=False,
                          phase1=np.full(n_blocks, per_block, dtype=np.int32), phase2=phase2,
                          target=total_budget, shared_overhead=bbv.phase1_total - per_block * n_blocks)


class SensingOperator:
    """operators.hpp:18-48 — matrix-free block DCT + zigzag-prefix selection, on device."""

    def __init__(self, grid: BlockGrid, counts):
        self._grid = grid
        self.counts = np.asarray(counts, dtype=np.uint16)
        if self.counts.size != grid.count():
            raise ValueError("SensingOperator: counts/grid mismatch")
        if np.any(self.counts.astype(np.int64) > grid.block * grid.block):
            raise ValueError("SensingOperator: count exceeds B^2")
        self._m = int(self.counts.astype(np.int64).sum())

    @classmethod
    def from_ms(cls, ms: MeasurementSet) -> "SensingOperator":
        return cls(ms.grid(), ms.counts)

    def grid(self) -> BlockGrid:
        return self._grid

    def measurements(self) -> int:
        return self._m

    def field_size(self) -> int:
        return self._grid.pixel_count()

    def field_height(self) -> int:
        return self._grid.cropped_height()

    def field_width(self) -> int:
        return self._grid.cropped_width()

    def _ms(self, y=None) -> MeasurementSet:
        g = self._grid
        return MeasurementSet(height=g.cropped_height(), width=g.cropped_width(), block=g.block,
                              counts=self.counts, coeffs=np.zeros(self._m, np.float32) if y is None else y)

    def forward(self, field_values) -> np.ndarray:
        torch = _torch()
        f = np.ascontiguousarray(np.asarray(field_values, dtype=np.float32).reshape(-1))
        if f.size != self.field_size():
            raise ValueError("forward: field size mismatch")
        b = _batch_from_host(self._ms())
        g = self._grid
        dev = b.counts.device
        ft = torch.from_numpy(f).to(dev)
        y = torch.empty(max(self._m, 1), dtype=torch.float32, device=dev)
        _check(_lib.load().abcs_forward_batch(Context.get(dev.index).handle, g.rows, g.cols, g.block,
                                              _ptr(b.counts), _ptr(b.offsets), ft.data_ptr(), f.size,
                                              g.cropped_width(), 1, y.data_ptr(), self._m, _stream_ptr(torch)))
        return y[:self._m].cpu().numpy()

    def adjoint(self, y) -> np.ndarray:
        yy = np.asarray(y, dtype=np.float32).reshape(-1)
        if yy.size != self._m:
            raise ValueError("adjoint: measurement vector length mismatch")
        b = _batch_from_host(self._ms(yy))
        return decode_batch(b)[0].cpu().numpy().reshape(-1)


def decode_idct(ms: MeasurementSet) -> np.ndarray:
    """recon.cpp:109-117 — (Hc, Wc) float32, unclamped."""
    if ms.total_coeffs() != len(ms.coeffs):
        raise FormatError("decode: payload length does not match counts")
    b = _batch_from_host(ms)
    return decode_batch(b)[0].cpu().numpy()


@dataclass
class ReconResult:
    image: np.ndarray
    trace: List[TraceRow]


def reconstruct(ms: MeasurementSet, cfg: ReconConfig, reference=None) -> ReconResult:
    """recon.cpp:199-259 for methods Idct and Ida."""
    torch = _torch()
    cfg.validate()
    g = ms.grid()
    ref_t = None
    if reference is not None:
        r = _as_u8_image(reference)
        if r.shape[0] < g.cropped_height() or r.shape[1] < g.cropped_width():
            raise ValueError("reconstruct: reference smaller than decoded image")
        ref_t = torch.from_numpy(np.ascontiguousarray(r)).cuda().reshape(1, *r.shape)
    if cfg.method == ReconMethod.Idct:
        img = decode_idct(ms)
        trace = []
        if ref_t is not None:  # psnr vs the cropped reference (recon.cpp:217-221, metrics.cpp:63-77)
            xt = torch.from_numpy(np.ascontiguousarray(img)).to(ref_t.device)
            out = torch.empty(1, dtype=torch.float64, device=ref_t.device)
            _check(_lib.load().abcs_psnr_batch(Context.get(ref_t.device.index).handle, ref_t.data_ptr(),
                                               ref_t[0].numel(), ref_t.shape[2], xt.data_ptr(), xt.numel(),
                                               g.cropped_width(), g.cropped_height(), g.cropped_width(), 1,
                                               out.data_ptr(), _stream_ptr(torch)))
            trace.append(TraceRow(0, 0.0, 0.0, float(out.item())))
        return ReconResult(img, trace)
    if ms.total_coeffs() != len(ms.coeffs):
        raise ValueError("init_state: measurement vector length mismatch")
    b = _batch_from_host(ms)
    out, tr, _ = recon_batch(b, cfg, reference=ref_t, trace=True, check=True)
    rows = [TraceRow(int(r[0]), float(r[1]), float(r[2]), float(r[3])) for r in tr[0].cpu().numpy()]
    return ReconResult(out[0].cpu().numpy(), rows)


@dataclass
class ReconState:
    """recon.hpp:46-51 — x (pixel field, flat f32), z (residual), sigma, iteration."""
    x: np.ndarray
    z: np.ndarray
    sigma: float = 0.0
    iteration: int = 0


def init_state(op: "SensingOperator", y, warm: bool) -> ReconState:
    """recon.cpp:119-131 via abcs_ida_init_state (x0 = A* y or 0, z0 = y - A x0, sigma0 = ||y||/sqrt(M))."""
    torch = _torch()
    yy = np.ascontiguousarray(np.asarray(y, dtype=np.float32).reshape(-1))
    if yy.size != op.measurements():
        raise ValueError("init_state: measurement vector length mismatch")
    b = _batch_from_host(op._ms(yy))
    g = op.grid()
    dev = b.counts.device
    x = torch.empty(op.field_size(), dtype=torch.float32, device=dev)
    z = torch.empty(max(yy.size, 1), dtype=torch.float32, device=dev)
    sig = torch.zeros(1, dtype=torch.float64, device=dev)
    _check(_lib.load().abcs_ida_init_state(Context.get(dev.index).handle, g.rows, g.cols, g.block, _ptr(b.counts),
                                           _ptr(b.offsets), _ptr(b.payload), yy.size, 1, 1 if warm else 0,
                                           x.data_ptr(), z.data_ptr(), sig.data_ptr(), _stream_ptr(torch)))
    return ReconState(x.cpu().numpy(), z[:yy.size].cpu().numpy(), float(sig.item()), 0)


def _step(state: ReconState, op: "SensingOperator", y, cfg: "ReconConfig", method: ReconMethod) -> None:
    """One ista/amp/damp step on the explicit state via abcs_recon_step_state; raises DivergenceError
    like finish_step/check_finite (recon.cpp:81-93, 53-73) after updating the state."""
    torch = _torch()
    yy = np.ascontiguousarray(np.asarray(y, dtype=np.float32).reshape(-1))
    if yy.size != op.measurements() or np.size(state.z) != yy.size or np.size(state.x) != op.field_size():
        raise ValueError("step: state / measurement size mismatch")
    b = _batch_from_host(op._ms(yy))
    g = op.grid()
    dev = b.counts.device
    x = torch.from_numpy(np.ascontiguousarray(np.asarray(state.x, dtype=np.float32).reshape(-1))).to(dev)
    z = torch.from_numpy(np.ascontiguousarray(np.asarray(state.z, dtype=np.float32).reshape(-1))).to(dev)
    sig = torch.tensor([float(state.sigma)], dtype=torch.float64, device=dev)
    div = torch.zeros(2, dtype=torch.int32, device=dev)
    c = _recon_c(cfg, method)
    c.iterations = 1
    _check(_lib.load().abcs_recon_step_state(Context.get(dev.index).handle, g.rows, g.cols, g.block, _ptr(b.counts),
                                             _ptr(b.offsets), _ptr(b.payload), yy.size, 1, C.byref(c), x.data_ptr(),
                                             z.data_ptr(), sig.data_ptr(), state.iteration, div.data_ptr(),
                                             _stream_ptr(torch)))
    state.x = x.cpu().numpy()
    state.z = z.cpu().numpy()
    state.sigma = float(sig.item())
    state.iteration += 1
    d = div.cpu().numpy()
    if d[0] > 0:
        what = {1: "non-finite estimate", 2: "|x| > 1e6"}.get(int(d[1]), "non-finite residual")
        raise DivergenceError(f"solver diverged ({what}) at iteration {int(d[0])}", int(d[0]))


def ista_step(state: ReconState, op: "SensingOperator", y, lam: float) -> None:
    """recon.cpp:133-142"""
    _step(state, op, y, ReconConfig(ReconMethod.Ista, 1, 2.0, DenoiserSpec(), lam), ReconMethod.Ista)


def amp_step(state: ReconState, op: "SensingOperator", y, lam: float) -> None:
    """recon.cpp:144-168"""
    _step(state, op, y, ReconConfig(ReconMethod.Amp, 1, 2.0, DenoiserSpec(), lam), ReconMethod.Amp)


def damp_step(state: ReconState, op: "SensingOperator", y, denoiser: DenoiserSpec, variant: ReconMethod,
              damping: float, seed: int = 42) -> None:
    """recon.cpp:170-197 for variants Damp, DampD and Ida, any denoiser."""
    if variant not in (ReconMethod.Damp, ReconMethod.DampD, ReconMethod.Ida):
        raise ValueError("damp_step: variant must be damp, dampd or ida")
    if damping < 1.0:
        raise ValueError("damping factor D_F must be >= 1")
    _step(state, op, y, ReconConfig(variant, 1, damping, denoiser, 1.0, seed), variant)


def divergence(spec: DenoiserSpec, field_values, sigma: float, epsilon: float, seed: int) -> float:
    """denoise.cpp:111-128 on the device (std::mt19937_64 Rademacher probe)."""
    torch = _torch()
    if epsilon <= 0:
        raise ValueError("divergence: epsilon must be > 0")
    f = np.ascontiguousarray(np.asarray(field_values, dtype=np.float32))
    H, W = f.shape
    dev = torch.device("cuda", torch.cuda.current_device())
    ft = torch.from_numpy(f).to(dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    c = _recon_c(ReconConfig(), None, spec)
    s_ = (C.c_double * 1)(sigma)
    e_ = (C.c_double * 1)(epsilon)
    _check(_lib.load().abcs_divergence_batch(Context.get(dev.index).handle, ft.data_ptr(), H, W, 1, s_, e_, seed,
                                             C.byref(c), out.data_ptr(), _stream_ptr(torch)))
    return float(out.item())


def rademacher_probe(seed: int, n: int):
    """std::mt19937_64(seed)'s first n outputs mapped (bit 0) to +1/-1 (denoise.cpp:115-116), on the device."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(n, dtype=torch.float32, device=dev)
    _check(_lib.load().abcs_rademacher_probe(Context.get(dev.index).handle, seed, n, out.data_ptr(),
                                             _stream_ptr(torch)))
    return out


def denoise(spec: DenoiserSpec, field_values, sigma: float) -> np.ndarray:
    """denoise.cpp:96-109 (dct_threshold on device; identity passes through)."""
    torch = _torch()
    if sigma < 0:
        raise ValueError("denoise: sigma must be >= 0")
    f = np.ascontiguousarray(np.asarray(field_values, dtype=np.float32))
    if spec.name == "identity":
        return f.copy()
    if spec.name not in ("dct_threshold", "blur"):
        raise ValueError(f"unknown denoiser: '{spec.name}'")
    H, W = f.shape
    ft = torch.from_numpy(f).cuda()
    out = torch.empty_like(ft)
    s = (C.c_double * 1)(sigma)
    c = _recon_c(ReconConfig(), None, spec)
    _check(_lib.load().abcs_denoise_batch(Context.get().handle, ft.data_ptr(), H, W, H * W, 1, s, C.byref(c),
                                          out.data_ptr(), _stream_ptr(torch)))
    return out.cpu().numpy()


# ---- quality metrics (metrics.hpp; metrics.cpp:63-130) ---------------------------------
@dataclass
class QualityReport:
    psnr_db: float = 0.0
    ssim: float = 0.0
    mse: float = 0.0


def quality_batch(refs, images, want=("mse", "psnr", "ssim")):
    """Per-image (mse, psnr, ssim) of f32 images (n,H,W) against u8 references (n,H',W') >= (H,W)
    (references are cropped to the images), on the device. Returns a dict of float64 tensors."""
    torch = _torch()
    n, H, W = images.shape
    dev = images.device
    out = {k: torch.empty(n, dtype=torch.float64, device=dev) for k in want}
    im = images.contiguous()
    _check(_lib.load().abcs_quality_batch(Context.get(dev.index).handle, refs.data_ptr(), refs.stride(0),
                                          refs.stride(1), im.data_ptr(), im.stride(0), im.stride(1), H, W, n,
                                          _ptr(out.get("mse")), _ptr(out.get("psnr")), _ptr(out.get("ssim")),
                                          _stream_ptr(torch)))
    return out


def _pair(ref, test):
    torch = _torch()
    r = _as_u8_image(ref)
    t = np.ascontiguousarray(np.asarray(test, dtype=np.float32))
    if r.shape != t.shape:
        raise ValueError("metric: image dimensions differ")
    dev = torch.device("cuda", torch.cuda.current_device())
    return torch.from_numpy(np.ascontiguousarray(r)).to(dev)[None], torch.from_numpy(t).to(dev)[None]


def quality(ref, test) -> QualityReport:
    """abcs::quality (metrics.cpp:118-125); `ref` must hold 8-bit integer values (the device path)."""
    r, t = _pair(ref, test)
    q = quality_batch(r, t)
    return QualityReport(float(q["psnr"][0]), float(q["ssim"][0]), float(q["mse"][0]))


def mse(ref, test) -> float:
    r, t = _pair(ref, test)
    return float(quality_batch(r, t, ("mse",))["mse"][0])


def psnr(ref, test) -> float:
    r, t = _pair(ref, test)
    return float(quality_batch(r, t, ("psnr",))["psnr"][0])


def ssim(ref, test) -> float:
    r, t = _pair(ref, test)
    if r.shape[1] < 11 or r.shape[2] < 11:
        raise ValueError("ssim: images smaller than the 11x11 window")
    return float(quality_batch(r, t, ("ssim",))["ssim"][0])


# ---- THB / THI full-sensing oracles (metrics.hpp:27-38, metrics.cpp:126-225) ------------
@dataclass
class ThresholdDecode:
    image: np.ndarray  # float64, cropped grid
    counts: np.ndarray  # int32 retained coefficients per block


def threshold_decode_batch(images, cfg: SensingConfig, global_: bool):
    """thb (global_=False) / thi (global_=True) for (n, H, W) uint8 CUDA images:
    (decoded (n, Hc, Wc) float64 tensor, counts (n, n_blocks) int32 tensor), bit-identical to the reference."""
    torch = _torch()
    cfg.validate()
    n, H, W = images.shape
    g = make_grid(H, W, cfg.block)
    dev = images.device
    im = images.contiguous()
    out = torch.empty((n, g.cropped_height(), g.cropped_width()), dtype=torch.float64, device=dev)
    counts = torch.empty((n, g.count()), dtype=torch.int32, device=dev)
    c = cfg._c()
    _check(_lib.load().abcs_threshold_decode_batch(Context.get(dev.index).handle, C.byref(c), im.data_ptr(), H * W,
                                                   W, H, W, n, 1 if global_ else 0, counts.data_ptr(),
                                                   out.data_ptr(), out.stride(0), out.stride(1), _stream_ptr(torch)))
    return out, counts


def _threshold(img, cfg: SensingConfig, global_: bool) -> ThresholdDecode:
    torch = _torch()
    a = _as_u8_image(img)
    t = torch.from_numpy(a).to(torch.device("cuda", torch.cuda.current_device()))[None]
    out, counts = threshold_decode_batch(t, cfg, global_)
    return ThresholdDecode(out[0].cpu().numpy(), counts[0].cpu().numpy())


def thb(img, cfg: SensingConfig) -> ThresholdDecode:
    """abcs::thb: per-block top-|c| with balanced counts (metrics.cpp:178-193)."""
    return _threshold(img, cfg, False)


def thi(img, cfg: SensingConfig) -> ThresholdDecode:
    """abcs::thi: image-wide top-|c| (metrics.cpp:162-177)."""
    return _threshold(img, cfg, True)


# ---- .abcs v1 container (container.hpp:8-14, container.cpp:58-149) --------------------
def container_size(plan: SensePlanC) -> int:
    return int(_lib.load().abcs_container_size(C.byref(plan)))


def pack_containers(batch: MeasurementBatch, out=None):
    """write_measurement_set's bytes for every set of the batch: (n, stride) uint8 CUDA tensor
    (stride = size rounded up to 4; row i[:container_size(plan)] is container i)."""
    torch = _torch()
    plan = batch.plan
    size = container_size(plan)
    stride = (size + 3) // 4 * 4
    dev = batch.counts.device
    if out is None:
        out = torch.empty((batch.n, stride), dtype=torch.uint8, device=dev)
    _check(_lib.load().abcs_container_pack_batch(Context.get(dev.index).handle, C.byref(plan), _ptr(batch.counts),
                                                 _ptr(batch.payload), _ptr(batch.side), batch.n, out.data_ptr(),
                                                 out.stride(0), _stream_ptr(torch)))
    return out


def unpack_containers(data, plan: SensePlanC):
    """read_measurement_set on the device for n containers of one layout: (MeasurementBatch,
    [per-container (algorithm, cr_num, cr_den, threshold)]). Raises FormatError naming the
    first invalid container."""
    torch = _torch()
    n = data.shape[0]
    dev = data.device
    K, S, nB = plan.coeffs_per_image, plan.side_per_image, plan.n_blocks
    counts = torch.empty((n, nB), dtype=torch.int16, device=dev).view(torch.uint16)
    payload = torch.empty((n, max(K, 1)), dtype=torch.float32, device=dev)
    side = torch.empty((n, max(S, 1)), dtype=torch.float32, device=dev) if S else None
    info = torch.empty((n, C.sizeof(_lib.ContainerInfoC)), dtype=torch.uint8, device=dev)
    _check(_lib.load().abcs_container_unpack_batch(Context.get(dev.index).handle, C.byref(plan), data.data_ptr(),
                                                   data.stride(0), n, counts.data_ptr(), payload.data_ptr(),
                                                   _ptr(side), info.data_ptr(), _stream_ptr(torch)))
    raw = info.cpu().numpy()
    infos = [_lib.ContainerInfoC.from_buffer_copy(raw[i].tobytes()) for i in range(n)]
    for i, inf in enumerate(infos):
        if inf.status != _lib.OK:
            raise FormatError(f"container {i}: invalid (header does not match the batch layout, "
                              f"count > B^2, payload or side length mismatch)")
    batch = MeasurementBatch(plan=plan, cfg=SensingConfig(plan.block, plan.cr_num, plan.cr_den,
                                                          Algorithm(plan.algorithm_used)),
                             counts=counts, offsets=None, payload=payload[:, :K], side=side)
    return batch, [(Algorithm(i.algorithm), i.cr_num, i.cr_den, i.threshold) for i in infos]


def write_measurement_set(ms: MeasurementSet, path) -> None:
    """abcs::write_measurement_set (container.cpp:58-93): packed on the device."""
    torch = _torch()
    if ms.block < 2 or ms.block * ms.block > 65535:
        raise ValueError("container: block size must fit u16 counts")
    g = ms.grid()
    if np.size(ms.counts) != g.count():
        raise ValueError("container: count table does not match grid")
    if ms.total_coeffs() != np.size(ms.coeffs):
        raise ValueError("container: payload length does not match counts")
    b = _batch_from_host(ms)
    side = np.ascontiguousarray(np.asarray(ms.side, dtype=np.float32).reshape(-1))
    b.plan.side_per_image = side.size
    b.side = torch.from_numpy(side).to(b.counts.device).reshape(1, -1) if side.size else None
    size = container_size(b.plan)
    data = pack_containers(b)[0, :size].cpu().numpy()
    with open(path, "wb") as f:
        f.write(data.tobytes())


def read_measurement_set(path) -> MeasurementSet:
    """abcs::read_measurement_set (container.cpp:95-149): parsed and unpacked on the device."""
    torch = _torch()
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError:
        raise FormatError(f"cannot open container: {path}")
    plan = SensePlanC()
    buf = np.frombuffer(raw, dtype=np.uint8)
    _check(_lib.load().abcs_container_parse(buf.ctypes.data if buf.size else None, buf.size, C.byref(plan)))
    stride = (buf.size + 3) // 4 * 4
    padded = np.zeros((1, stride), np.uint8)
    padded[0, :buf.size] = buf
    dev = torch.device("cuda", torch.cuda.current_device())
    batch, infos = unpack_containers(torch.from_numpy(padded).to(dev), plan)
    algo, num, den, thr = infos[0]
    return MeasurementSet(height=plan.height, width=plan.width, block=plan.block, algorithm=algo, cr_num=num,
                          cr_den=den, threshold=thr, counts=batch.counts[0].cpu().numpy().astype(np.uint16),
                          coeffs=batch.payload[0].cpu().numpy(),
                          side=(batch.side[0].cpu().numpy() if batch.side is not None else np.zeros(0, np.float32)))


# ---- synthetic inputs ---------------------------------------------
@dataclass
class SynthSpec:
    height: int
    width: int
    n_ellipses: int = 20
    noise_sigma: float = 5.0
    seed: int = 1
    video: bool = False
    max_shift: int = 8

    def _c(self) -> SynthSpecC:
        c = SynthSpecC()
        c.height, c.width, c.n_ellipses = self.height, self.width, self.n_ellipses
        c.video, c.max_shift = int(self.video), self.max_shift
        c.noise_sigma, c.seed = self.noise_sigma, self.seed
        return c


def synth_images(spec: SynthSpec, first: int, n: int, device=None):
    """(n, H, W) uint8 CUDA tensor generated on the device."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    out = torch.empty((n, spec.height, spec.width), dtype=torch.uint8, device=dev)
    c = spec._c()
    _check(_lib.load().abcs_synth_generate(Context.get(dev.index).handle, C.byref(c), first, n, out.data_ptr(),
                                           spec.height * spec.width, _stream_ptr(torch)))
    return out


def synth_images_host(spec: SynthSpec, first: int, n: int) -> np.ndarray:
    """Same bytes as synth_images, generated on the host (inputs for CPU baselines/oracle)."""
    out = np.empty((n, spec.height, spec.width), dtype=np.uint8)
    c = spec._c()
    _check(_lib.load().abcs_synth_generate_host(C.byref(c), first, n, out.ctypes.data))
    return out
