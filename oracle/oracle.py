"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU oracles.

Two interchangeable checkers with one Python interface:
  * CPort     — oracle/abcs_oracle.c, our plain-C restatement of the reference
                hot path (always buildable: gcc only);
  * Reference — the UNMODIFIED reference library compiled from
                /root/reference/proj/core/src by oracle/Makefile into
                oracle/_ref/libabcs_ref.so (present when the reference was
                available at build time; the .so travels to the GPU box).
Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl
reference) may import this module — never the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libabcs_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libabcs_ref.so")

P = C.c_void_p


def build() -> None:
    subprocess.run(["make", "-C", HERE, "-s"], check=True, capture_output=True)


def _load(path):
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


class OracleError(RuntimeError):
    def __init__(self, code, msg, iteration=0):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.iteration = iteration


def _u8(img):
    a = np.ascontiguousarray(np.asarray(img, dtype=np.uint8))
    assert a.ndim == 2
    return a


class CPort:
    """oracle/abcs_oracle.c"""

    name = "port"

    def __init__(self):
        lib = _load(PORT_SO)
        lib.o_last_error.restype = C.c_char_p
        lib.o_dd_threshold.restype = C.c_double
        lib.o_psnr.restype = C.c_double
        self.lib = lib

    def _err(self, st, it=0):
        if st != 0:
            raise OracleError(st, self.lib.o_last_error().decode(), it)

    def basis(self, B):
        out = np.zeros(B * B)
        self.lib.o_basis(B, out.ctypes.data_as(P))
        return out

    def zigzag(self, B):
        out = np.zeros(B * B, np.int32)
        self.lib.o_zigzag(B, out.ctypes.data_as(P))
        return out

    def dct2(self, block, B):
        b = np.ascontiguousarray(block, dtype=np.float64).reshape(-1)
        out = np.zeros(B * B)
        self.lib.o_dct_forward(self.basis(B).ctypes.data_as(P), B, b.ctypes.data_as(P), out.ctypes.data_as(P))
        return out

    def idct2(self, coef, B):
        b = np.ascontiguousarray(coef, dtype=np.float64).reshape(-1)
        out = np.zeros(B * B)
        self.lib.o_dct_inverse(self.basis(B).ctypes.data_as(P), B, b.ctypes.data_as(P), out.ctypes.data_as(P))
        return out

    def allocate(self, weights, budget, caps):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        c = np.ascontiguousarray(caps, dtype=np.int32)
        out = np.zeros(w.size, np.int32)
        self._err(self.lib.o_largest_remainder(w.ctypes.data_as(P), w.size, C.c_longlong(budget),
                                               c.ctypes.data_as(P), out.ctypes.data_as(P)))
        return out

    def dd_threshold(self, h, num, den):
        return self.lib.o_dd_threshold(h, C.c_uint32(num), C.c_uint32(den))

    def sense(self, img, block, num, den, algo, threshold=None):
        a = _u8(img)
        H, W = a.shape
        nb = (H // block) * (W // block) if block <= min(H, W) and block >= 2 else 1
        counts = np.zeros(max(nb, 1), np.uint16)
        coeffs = np.zeros(max(nb, 1) * block * block)
        side = np.zeros(max(nb, 1) * 4 * block + 16)
        info = np.zeros(8, np.int64)
        thr = C.c_double()
        self._err(self.lib.o_sense(a.ctypes.data_as(P), H, W, block, C.c_uint32(num), C.c_uint32(den), algo,
                                   1 if threshold is not None else 0, C.c_double(threshold or 0.0),
                                   counts.ctypes.data_as(P), coeffs.ctypes.data_as(P), side.ctypes.data_as(P),
                                   info.ctypes.data_as(P), C.byref(thr)))
        return dict(counts=counts[:nb], coeffs=coeffs[:info[1]], side=side[:info[2]], algorithm=int(info[0]),
                    threshold=thr.value, fallback=int(info[3]), rows=int(info[4]), cols=int(info[5]),
                    target=int(info[6]), actual=int(info[7]))

    def bbv_measure(self, img, block, num, den):
        a = _u8(img)
        H, W = a.shape
        nb = (H // block) * (W // block)
        params = np.zeros(5, np.int64)
        var = np.zeros(nb)
        side = np.zeros(nb * 4 * block + 16)
        self._err(self.lib.o_bbv_measure(a.ctypes.data_as(P), H, W, block, C.c_uint32(num), C.c_uint32(den),
                                         params.ctypes.data_as(P), var.ctypes.data_as(P), side.ctypes.data_as(P)))
        return dict(stride=int(params[0]), offset=int(params[1]), per_side=int(params[2]),
                    phase1_total=int(params[3]), variation=var, side=side[:params[4]])

    def decode(self, rows, cols, B, counts, coeffs):
        c = np.ascontiguousarray(counts, dtype=np.uint16)
        y = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros((rows * B, cols * B))
        self._err(self.lib.o_decode(rows, cols, B, c.ctypes.data_as(P), y.ctypes.data_as(P), C.c_longlong(y.size),
                                    out.ctypes.data_as(P)))
        return out

    def forward(self, rows, cols, B, counts, field):
        c = np.ascontiguousarray(counts, dtype=np.uint16)
        f = np.ascontiguousarray(field, dtype=np.float64)
        y = np.zeros(int(c.astype(np.int64).sum()))
        self._err(self.lib.o_forward(rows, cols, B, c.ctypes.data_as(P), f.ctypes.data_as(P), y.ctypes.data_as(P)))
        return y

    def denoise(self, field, threshold, block=8):
        f = np.ascontiguousarray(field, dtype=np.float64)
        out = np.zeros_like(f)
        self._err(self.lib.o_denoise_dct(f.ctypes.data_as(P), f.shape[0], f.shape[1], C.c_double(threshold), block,
                                         out.ctypes.data_as(P)))
        return out

    def quality(self, ref, test):
        """(mse, psnr, ssim) -- metrics.cpp:63-125 restated (o_psnr, o_ssim)."""
        a = np.ascontiguousarray(ref, dtype=np.float64)
        b = np.ascontiguousarray(test, dtype=np.float64)
        self.lib.o_psnr.restype = C.c_double
        self.lib.o_ssim.restype = C.c_double
        mse = float(np.mean((a - b) ** 2))
        ps = self.lib.o_psnr(a.ctypes.data_as(P), b.ctypes.data_as(P), C.c_longlong(a.size))
        ss = self.lib.o_ssim(a.ctypes.data_as(P), b.ctypes.data_as(P), a.shape[0], a.shape[1])
        return mse, ps, ss

    def reconstruct_ida(self, rows, cols, B, counts, coeffs, iters, damping=2.0, k=2.7, dblock=8, ref=None):
        c = np.ascontiguousarray(counts, dtype=np.uint16)
        y = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros((rows * B, cols * B))
        trace = np.zeros((iters + 1, 4))
        div = C.c_int(0)
        r = None if ref is None else _u8(ref)
        st = self.lib.o_reconstruct_ida(rows, cols, B, c.ctypes.data_as(P), y.ctypes.data_as(P),
                                        C.c_longlong(y.size), iters, C.c_double(damping), C.c_double(k), dblock,
                                        None if r is None else r.ctypes.data_as(P),
                                        0 if r is None else r.shape[0], 0 if r is None else r.shape[1],
                                        out.ctypes.data_as(P), trace.ctypes.data_as(P), C.byref(div))
        self._err(st, div.value)
        return out, trace


def container_bytes(height, width, block, algorithm, cr_num, cr_den, threshold, counts, coeffs, side) -> bytes:
    """write_measurement_set's byte image (container.cpp:58-93): little-endian, packed;
    coefficients and side data narrowed to f32 (container.cpp:83,85)."""
    import struct
    c = np.asarray(counts, dtype="<u2")
    out = [b"ABCS", struct.pack("<HIIHBIIdI", 1, height, width, block, algorithm, cr_num, cr_den, threshold, c.size),
           c.tobytes(), np.asarray(coeffs, dtype="<f4").tobytes(), struct.pack("<I", np.size(side)),
           np.asarray(side, dtype="<f4").tobytes()]
    return b"".join(out)


class Reference:
    """oracle/_ref/libabcs_ref.so — the reference library itself (ref_capi.cpp shims)."""

    name = "reference"

    @staticmethod
    def available() -> bool:
        if not os.path.exists(REF_SO):
            try:
                build()
            except Exception:
                return False
        return os.path.exists(REF_SO)

    def __init__(self):
        if not self.available():
            raise FileNotFoundError(REF_SO)
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_dd_threshold.restype = C.c_double
        lib.ref_ms_warning.restype = C.c_char_p
        lib.ref_ms_make.restype = P
        lib.ref_ms_free.argtypes = [P]
        for fn in ("ref_ms_info", "ref_ms_counts", "ref_ms_coeffs", "ref_ms_side", "ref_decode", "ref_ms_warning"):
            getattr(lib, fn).argtypes = None
        self.lib = lib

    def _err(self, st, it=0):
        if st != 0:
            raise OracleError(st, self.lib.ref_last_error().decode(), it)

    def _ms_to_dict(self, h):
        info = np.zeros(11, np.int64)
        thr = C.c_double()
        self.lib.ref_ms_info(P(h), info.ctypes.data_as(P), C.byref(thr))
        counts = np.zeros(info[6], np.uint16)
        coeffs = np.zeros(info[7])
        side = np.zeros(info[8])
        self.lib.ref_ms_counts(P(h), counts.ctypes.data_as(P))
        self.lib.ref_ms_coeffs(P(h), coeffs.ctypes.data_as(P))
        self.lib.ref_ms_side(P(h), side.ctypes.data_as(P))
        self.lib.ref_ms_warning.argtypes = [P]
        warn = self.lib.ref_ms_warning(P(h)).decode()
        B = int(info[2])
        return dict(counts=counts, coeffs=coeffs, side=side, algorithm=int(info[3]), threshold=thr.value,
                    rows=int(info[0]) // B, cols=int(info[1]) // B, target=int(info[9]), actual=int(info[10]),
                    warning=warn, cr_num=int(info[4]), cr_den=int(info[5]))

    def zigzag(self, B):
        out = np.zeros(B * B, np.int32)
        self.lib.ref_zigzag(B, out.ctypes.data_as(P))
        return out

    def dct2(self, block, B):
        b = np.ascontiguousarray(block, dtype=np.float64).reshape(-1)
        out = np.zeros(B * B)
        self.lib.ref_dct2(b.ctypes.data_as(P), B, out.ctypes.data_as(P))
        return out

    def idct2(self, coef, B):
        b = np.ascontiguousarray(coef, dtype=np.float64).reshape(-1)
        out = np.zeros(B * B)
        self.lib.ref_idct2(b.ctypes.data_as(P), B, out.ctypes.data_as(P))
        return out

    def allocate(self, weights, budget, caps):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        c = np.ascontiguousarray(caps, dtype=np.int32)
        out = np.zeros(w.size, np.int32)
        self._err(self.lib.ref_allocate(w.ctypes.data_as(P), w.size, C.c_longlong(budget), c.ctypes.data_as(P),
                                        out.ctypes.data_as(P)))
        return out

    def dd_threshold(self, h, num, den):
        return self.lib.ref_dd_threshold(h, C.c_uint32(num), C.c_uint32(den))

    def parse_ratio(self, text):
        n, d = C.c_uint32(), C.c_uint32()
        self._err(self.lib.ref_parse_ratio(text.encode(), C.byref(n), C.byref(d)))
        return n.value, d.value

    def sense(self, img, block, num, den, algo, threshold=None):
        a = _u8(img)
        H, W = a.shape
        h = P()
        self._err(self.lib.ref_sense(a.ctypes.data_as(P), H, W, block, C.c_uint32(num), C.c_uint32(den), algo,
                                     1 if threshold is not None else 0, C.c_double(threshold or 0.0), C.byref(h)))
        try:
            return self._ms_to_dict(h.value)
        finally:
            self.lib.ref_ms_free(h)

    def bbv_measure(self, img, block, num, den):
        a = _u8(img)
        H, W = a.shape
        nb = (H // block) * (W // block)
        params = np.zeros(5, np.int64)
        var = np.zeros(nb)
        side = np.zeros(nb * 4 * block + 16)
        self._err(self.lib.ref_bbv_measure(a.ctypes.data_as(P), H, W, block, C.c_uint32(num), C.c_uint32(den),
                                           params.ctypes.data_as(P), var.ctypes.data_as(P), side.ctypes.data_as(P),
                                           C.c_longlong(side.size)))
        return dict(stride=int(params[0]), offset=int(params[1]), per_side=int(params[2]),
                    phase1_total=int(params[3]), variation=var, side=side[:params[4]])

    def _make(self, rows, cols, B, counts, coeffs):
        c = np.ascontiguousarray(counts, dtype=np.uint16)
        y = np.ascontiguousarray(coeffs, dtype=np.float64)
        return self.lib.ref_ms_make(rows * B, cols * B, B, 0, C.c_uint32(1), C.c_uint32(1), C.c_double(0.0),
                                    c.ctypes.data_as(P), c.size, y.ctypes.data_as(P), C.c_longlong(y.size))

    def reconstruct(self, rows, cols, B, counts, coeffs, method, iters, damping=2.0, lam=1.0, seed=42, denoiser=0,
                    k=2.7, dblock=8, sigma_scale=25.0, ref=None):
        """abcs::reconstruct with every ReconConfig field -> (image, trace rows)."""
        h = self._make(rows, cols, B, counts, coeffs)
        try:
            out = np.zeros((rows * B, cols * B))
            trace = np.zeros((iters + 1, 4))
            nrows, div = C.c_int(), C.c_int(0)
            r = None if ref is None else _u8(ref)
            self.lib.ref_reconstruct2.argtypes = [P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_ulonglong,
                                                  C.c_int, C.c_double, C.c_double, C.c_double, P, C.c_int, C.c_int,
                                                  P, P, P, P]
            st = self.lib.ref_reconstruct2(h, int(method), iters, damping, lam, seed, denoiser, k, float(dblock),
                                           sigma_scale, None if r is None else r.ctypes.data_as(P),
                                           0 if r is None else r.shape[0], 0 if r is None else r.shape[1],
                                           out.ctypes.data_as(P), trace.ctypes.data_as(P), C.byref(nrows),
                                           C.byref(div))
            self._err(st, div.value)
            return out, trace[:nrows.value]
        finally:
            self.lib.ref_ms_free(h)

    def denoise2(self, field, sigma, denoiser=0, k=2.7, dblock=8, sigma_scale=25.0):
        f = np.ascontiguousarray(field, dtype=np.float64)
        out = np.zeros_like(f)
        self.lib.ref_denoise2.argtypes = [P, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                          C.c_double, P]
        self._err(self.lib.ref_denoise2(f.ctypes.data_as(P), f.shape[0], f.shape[1], sigma, denoiser, k,
                                        float(dblock), sigma_scale, out.ctypes.data_as(P)))
        return out

    def divergence(self, field, sigma, eps, seed, denoiser=0, k=2.7, dblock=8, sigma_scale=25.0):
        f = np.ascontiguousarray(field, dtype=np.float64)
        out = C.c_double()
        self.lib.ref_divergence.argtypes = [P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_ulonglong, C.c_int,
                                            C.c_double, C.c_double, C.c_double, P]
        self._err(self.lib.ref_divergence(f.ctypes.data_as(P), f.shape[0], f.shape[1], sigma, eps, seed, denoiser, k,
                                          float(dblock), sigma_scale, C.byref(out)))
        return out.value

    def threshold_decode(self, img, B, num, den, global_):
        """abcs::thb (global_=False) / abcs::thi -> (decoded image, counts)."""
        a = _u8(img)
        rows, cols = a.shape[0] // B, a.shape[1] // B
        out = np.zeros((rows * B, cols * B))
        counts = np.zeros(rows * cols, np.int32)
        self.lib.ref_threshold_decode.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_int, P, P]
        self._err(self.lib.ref_threshold_decode(a.ctypes.data_as(P), a.shape[0], a.shape[1], B, num, den,
                                                1 if global_ else 0, out.ctypes.data_as(P),
                                                counts.ctypes.data_as(P)))
        return out, counts

    def mt19937_64(self, seed, n):
        out = np.zeros(n, np.uint64)
        self.lib.ref_mt19937_64.argtypes = [C.c_ulonglong, C.c_longlong, P]
        self.lib.ref_mt19937_64(seed, n, out.ctypes.data_as(P))
        return out

    def quality(self, ref, test):
        """abcs::quality -> (mse, psnr, ssim)."""
        a = np.ascontiguousarray(ref, dtype=np.float64)
        b = np.ascontiguousarray(test, dtype=np.float64)
        m, p_, s_ = C.c_double(), C.c_double(), C.c_double()
        self.lib.ref_quality.argtypes = [P, P, C.c_int, C.c_int, P, P, P]
        self._err(self.lib.ref_quality(a.ctypes.data_as(P), b.ctypes.data_as(P), a.shape[0], a.shape[1],
                                       C.byref(m), C.byref(p_), C.byref(s_)))
        return m.value, p_.value, s_.value

    def write_container(self, ms, path):
        """abcs::write_measurement_set on a MeasurementSet given as a dict (sense()'s layout)."""
        c = np.ascontiguousarray(ms["counts"], dtype=np.uint16)
        y = np.ascontiguousarray(ms["coeffs"], dtype=np.float64)
        sd = np.ascontiguousarray(ms.get("side", np.zeros(0)), dtype=np.float64)
        h = self.lib.ref_ms_make(ms["height"], ms["width"], ms["block"], int(ms["algorithm"]),
                                 C.c_uint32(ms["cr_num"]), C.c_uint32(ms["cr_den"]), C.c_double(ms["threshold"]),
                                 c.ctypes.data_as(P), c.size, y.ctypes.data_as(P), C.c_longlong(y.size))
        try:
            self.lib.ref_ms_set_side.argtypes = [P, P, C.c_longlong]
            self.lib.ref_ms_set_side(h, sd.ctypes.data_as(P), sd.size)
            self.lib.ref_container_write.argtypes = [P, C.c_char_p]
            self._err(self.lib.ref_container_write(h, str(path).encode()))
        finally:
            self.lib.ref_ms_free(h)

    def read_container(self, path):
        """abcs::read_measurement_set -> dict (counts, coeffs, side, header fields)."""
        h = P()
        self.lib.ref_container_read.argtypes = [C.c_char_p, C.POINTER(P)]
        self._err(self.lib.ref_container_read(str(path).encode(), C.byref(h)))
        try:
            return self._ms_dict(h)
        finally:
            self.lib.ref_ms_free(h)

    def _ms_dict(self, h):
        info = (C.c_longlong * 11)()
        thr = C.c_double()
        self.lib.ref_ms_info(h, info, C.byref(thr))
        counts = np.zeros(info[6], np.uint16)
        coeffs = np.zeros(info[7])
        side = np.zeros(info[8])
        self.lib.ref_ms_counts(h, counts.ctypes.data_as(P))
        self.lib.ref_ms_coeffs(h, coeffs.ctypes.data_as(P))
        self.lib.ref_ms_side(h, side.ctypes.data_as(P))
        return {"height": info[0], "width": info[1], "block": info[2], "algorithm": info[3], "cr_num": info[4],
                "cr_den": info[5], "threshold": thr.value, "counts": counts, "coeffs": coeffs, "side": side}

    def decode(self, rows, cols, B, counts, coeffs):
        h = self._make(rows, cols, B, counts, coeffs)
        try:
            out = np.zeros((rows * B, cols * B))
            self.lib.ref_decode.argtypes = [P, P]
            self._err(self.lib.ref_decode(h, out.ctypes.data_as(P)))
            return out
        finally:
            self.lib.ref_ms_free(h)

    def forward(self, rows, cols, B, counts, field):
        h = self._make(rows, cols, B, counts, np.zeros(int(np.asarray(counts, np.int64).sum())))
        try:
            f = np.ascontiguousarray(field, dtype=np.float64)
            y = np.zeros(int(np.asarray(counts, np.int64).sum()))
            self.lib.ref_op_forward.argtypes = [P, P, P]
            self._err(self.lib.ref_op_forward(h, f.ctypes.data_as(P), y.ctypes.data_as(P)))
            return y
        finally:
            self.lib.ref_ms_free(h)

    def denoise(self, field, threshold, block=8):
        # denoise(spec, field, sigma) thresholds at k*sigma: pass k=1, sigma=threshold
        f = np.ascontiguousarray(field, dtype=np.float64)
        out = np.zeros_like(f)
        self._err(self.lib.ref_denoise(f.ctypes.data_as(P), f.shape[0], f.shape[1], C.c_double(threshold),
                                       C.c_double(1.0), C.c_double(block), out.ctypes.data_as(P)))
        return out

    def reconstruct_ida(self, rows, cols, B, counts, coeffs, iters, damping=2.0, k=2.7, dblock=8, ref=None):
        h = self._make(rows, cols, B, counts, coeffs)
        try:
            out = np.zeros((rows * B, cols * B))
            trace = np.zeros((iters + 1, 4))
            nrows, div = C.c_int(), C.c_int(0)
            r = None if ref is None else _u8(ref)
            self.lib.ref_reconstruct.argtypes = [P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, P,
                                                 C.c_int, C.c_int, P, P, P, P]
            st = self.lib.ref_reconstruct(h, 5, iters, damping, k, float(dblock),
                                          None if r is None else r.ctypes.data_as(P),
                                          0 if r is None else r.shape[0], 0 if r is None else r.shape[1],
                                          out.ctypes.data_as(P), trace.ctypes.data_as(P), C.byref(nrows), C.byref(div))
            self._err(st, div.value)
            return out, trace
        finally:
            self.lib.ref_ms_free(h)

    def sense_reconstruct_batch(self, imgs, block, num, den, algo, method=0, iters=1, threads=1, out=None):
        a = np.ascontiguousarray(imgs, dtype=np.uint8)
        n, H, W = a.shape
        self.lib.ref_sense_reconstruct_batch.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint32,
                                                         C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int, P]
        self._err(self.lib.ref_sense_reconstruct_batch(a.ctypes.data_as(P), n, H, W, block, num, den, algo, method,
                                                       iters, threads, None if out is None else out.ctypes.data_as(P)))


def synth_images(height, width, ellipses, sigma, seed, first, n, video=False, threads=None):
    """The BASELINE seeded inputs (csrc/synth_gen.h host path compiled into the oracle library by
    oracle/synth_inputs.c): the same bytes as the product's generator, without loading it."""
    lib = _load(PORT_SO)
    lib.o_synth_images.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.c_int32,
                                   C.c_int64, C.c_int32, P, C.c_int32]
    out = np.empty((n, height, width), dtype=np.uint8)
    if threads is None:
        threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    st = lib.o_synth_images(height, width, ellipses, float(sigma), seed, int(bool(video)), first, n,
                            out.ctypes.data_as(P), threads)
    if st != 0:
        raise OracleError(st, "o_synth_images failed")
    return out


def reference_bench_phases(imgs, block, num, den, algo, method, iters, threads):
    """Wall seconds (sense, reconstruct) of the reference library over a batch on `threads` host
    threads (ref_bench_phases in ref_capi.cpp). method: 0 Idct, 5 Ida (recon.hpp:15)."""
    lib = C.CDLL(REF_SO)
    lib.ref_bench_phases.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_int,
                                     C.c_int, C.c_int, C.c_int, P, P]
    a = np.ascontiguousarray(imgs, dtype=np.uint8)
    n, H, W = a.shape
    ts, tr = C.c_double(0.0), C.c_double(0.0)
    st = lib.ref_bench_phases(a.ctypes.data_as(P), n, H, W, block, num, den, algo, method, iters, threads,
                              C.byref(ts), C.byref(tr))
    if st != 0:
        raise OracleError(st, "ref_bench_phases failed")
    return ts.value, tr.value


def best_available():
    """The reference library when it was built here, else the C port."""
    return Reference() if Reference.available() else CPort()
