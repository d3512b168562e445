"""ctypes binding of libabcs_b200.so (the C ABI in include/abcs_b200.h).

The library is built in-tree by `make -C paper_2001_09632_b200` (done by
__graft_entry__.build()). If it is missing, `load()` tries that build once and
otherwise raises: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ABCS_LIB_OVERRIDE") or os.path.join(HERE, "libabcs_b200.so")

OK, INVALID, FORMAT, DIVERGENCE, CUDA, LOGIC, UNSUPPORTED = range(7)


class SensingConfigC(C.Structure):
    _fields_ = [
        ("block", C.c_int32),
        ("cr_num", C.c_uint32),
        ("cr_den", C.c_uint32),
        ("algorithm", C.c_int32),
        ("has_threshold", C.c_int32),
        ("reserved", C.c_int32),
        ("threshold", C.c_double),
    ]


class SensePlanC(C.Structure):
    _fields_ = [
        ("height", C.c_int32), ("width", C.c_int32), ("block", C.c_int32),
        ("rows", C.c_int32), ("cols", C.c_int32), ("n_blocks", C.c_int32),
        ("algorithm", C.c_int32), ("algorithm_used", C.c_int32),
        ("fallback", C.c_int32), ("zz_last_zero", C.c_int32),
        ("cr_num", C.c_uint32), ("cr_den", C.c_uint32),
        ("threshold", C.c_double),
        ("target", C.c_int64), ("coeffs_per_image", C.c_int64),
        ("side_per_image", C.c_int64), ("budget_actual", C.c_int64),
        ("bbv_stride", C.c_int64), ("bbv_offset", C.c_int32), ("bbv_per_side", C.c_int32),
        ("bbv_phase1_total", C.c_int64), ("bbv_valid_probes", C.c_int32),
        ("dd_phase1", C.c_int32), ("cap", C.c_int32), ("count_base", C.c_int32),
        ("alloc_budget", C.c_int64), ("zz_per_block", C.c_int64), ("zz_extra", C.c_int64),
    ]


class IdaConfigC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("denoiser_block", C.c_int32),
        ("damping", C.c_double),
        ("k", C.c_double),
    ]


class SynthSpecC(C.Structure):
    _fields_ = [
        ("height", C.c_int32), ("width", C.c_int32), ("n_ellipses", C.c_int32),
        ("video", C.c_int32), ("max_shift", C.c_int32), ("reserved", C.c_int32),
        ("noise_sigma", C.c_double), ("seed", C.c_uint64),
    ]


class ReconConfigC(C.Structure):
    _fields_ = [("method", C.c_int32), ("iterations", C.c_int32), ("damping", C.c_double), ("lambda_", C.c_double),
                ("seed", C.c_uint64), ("denoiser", C.c_int32), ("denoiser_block", C.c_int32), ("k", C.c_double),
                ("sigma_scale", C.c_double)]


class ContainerInfoC(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("cr_num", C.c_uint32), ("cr_den", C.c_uint32), ("status", C.c_int32),
                ("threshold", C.c_double)]


class KernelTimeC(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_int64), ("total_ms", C.c_double), ("max_ms", C.c_double)]


P = C.c_void_p
I32, I64, U32, U64, D = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double

# name -> (restype, argtypes); also the export list the CPU tests check against the header
SIGNATURES = {
    "abcs_abi_version": (C.c_int, []),
    "abcs_last_error": (C.c_char_p, []),
    "abcs_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "abcs_ctx_destroy": (C.c_int, [P]),
    "abcs_ctx_launch_count": (I64, [P]),
    "abcs_ctx_kernel_timing": (C.c_int, [P, I32]),
    "abcs_ctx_set_pipeline_streams": (C.c_int, [P, I32]),
    "abcs_ctx_kernel_times": (C.c_int, [P, C.POINTER(KernelTimeC), I32, C.POINTER(I32)]),
    "abcs_parse_ratio": (C.c_int, [C.c_char_p, C.POINTER(U32), C.POINTER(U32)]),
    "abcs_dd_threshold": (D, [I32, U32, U32]),
    "abcs_zigzag_order": (C.c_int, [I32, P]),
    "abcs_sense_plan_init": (C.c_int, [C.POINTER(SensingConfigC), I32, I32, C.POINTER(SensePlanC)]),
    "abcs_synth_generate_host": (C.c_int, [C.POINTER(SynthSpecC), I64, I32, P]),
    "abcs_sense_batch": (C.c_int, [P, C.POINTER(SensePlanC), P, I64, I32, I32, P, P, P, P, P]),
    "abcs_sense_decode_batch": (C.c_int, [P, C.POINTER(SensePlanC), P, I64, I32, I32, P, P, P, P, P, I64, I32, P]),
    "abcs_bbv_weights_strip": (C.c_int, [P, C.POINTER(SensePlanC), P, I64, I32, I32, P, P, P]),
    "abcs_gather_decode_batch": (C.c_int, [P, I32, I32, I32, P, I64, I32, I32, P, P, P, I64, P, I64, I32, P]),
    "abcs_allocate_shard_scratch_bytes": (C.c_size_t, [I32, I32]),
    "abcs_allocate_shard_step": (C.c_int, [P, I32, P, I32, I32, I32, I32, P, P, P, I64, I64, P, P, P]),
    "abcs_sense_decode_sweep_batch": (C.c_int, [P, C.POINTER(SensePlanC), I32, P, I64, I32, I32, P, P, P, P, P, I64,
                                                I32, P]),
    "abcs_sense_weights_batch": (C.c_int, [P, C.POINTER(SensePlanC), P, I64, I32, I32, P, P, P]),
    "abcs_allocate_batch": (C.c_int, [P, P, I32, I32, I64, P, I32, I32, P, P, P, P]),
    "abcs_allocate_small_batch": (C.c_int, [P, P, I32, I32, I64, I32, I32, I32, P, P, P, P]),
    "abcs_decode_batch": (C.c_int, [P, I32, I32, I32, P, P, P, I64, I32, P, I64, I32, P, P, P]),
    "abcs_forward_batch": (C.c_int, [P, I32, I32, I32, P, P, P, I64, I32, I32, P, I64, P]),
    "abcs_block_dct_f64": (C.c_int, [P, I32, I32, P, P, I64, P]),
    "abcs_denoise_dct_batch": (C.c_int, [P, P, I32, I32, I64, I32, P, D, I32, P, P]),
    "abcs_ida_batch": (C.c_int, [P, I32, I32, I32, P, P, P, I64, I32, C.POINTER(IdaConfigC),
                                 P, I64, I32, P, I64, I32, P, P, P]),
    "abcs_ida_check": (C.c_int, [P, I32, C.POINTER(I32)]),
    "abcs_reconstruct_batch": (C.c_int, [P, I32, I32, I32, P, P, P, I64, I32, C.POINTER(ReconConfigC),
                                         P, I64, I32, P, I64, I32, P, P, P]),
    "abcs_recon_step_state": (C.c_int, [P, I32, I32, I32, P, P, P, I64, I32, C.POINTER(ReconConfigC), P, P, P, I32,
                                        P, P]),
    "abcs_denoise_batch": (C.c_int, [P, P, I32, I32, I64, I32, P, C.POINTER(ReconConfigC), P, P]),
    "abcs_divergence_batch": (C.c_int, [P, P, I32, I32, I32, P, P, U64, C.POINTER(ReconConfigC), P, P]),
    "abcs_rademacher_probe": (C.c_int, [P, U64, I64, P, P]),
    "abcs_threshold_decode_batch": (C.c_int, [P, C.POINTER(SensingConfigC), P, I64, I32, I32, I32, I32, I32, P, P,
                                              I64, I32, P]),
    "abcs_container_size": (I64, [C.POINTER(SensePlanC)]),
    "abcs_container_pack_batch": (C.c_int, [P, C.POINTER(SensePlanC), P, P, P, I32, P, I64, P]),
    "abcs_container_unpack_batch": (C.c_int, [P, C.POINTER(SensePlanC), P, I64, I32, P, P, P, P, P]),
    "abcs_container_parse": (C.c_int, [P, I64, C.POINTER(SensePlanC)]),
    "abcs_quality_batch": (C.c_int, [P, P, I64, I32, P, I64, I32, I32, I32, I32, P, P, P, P]),
    "abcs_ssim_batch": (C.c_int, [P, P, I64, I32, P, I64, I32, I32, I32, I32, P, P]),
    "abcs_psnr_batch": (C.c_int, [P, P, I64, I32, P, I64, I32, I32, I32, I32, P, P]),
    "abcs_ida_init_state": (C.c_int, [P, I32, I32, I32, P, P, P, I64, I32, I32, P, P, P, P]),
    "abcs_ida_step_state": (C.c_int, [P, I32, I32, I32, P, P, P, I64, I32, C.POINTER(IdaConfigC), P, P, P, I32,
                                      P, P]),
    "abcs_synth_generate": (C.c_int, [P, C.POINTER(SynthSpecC), I64, I32, P, I64, P]),
    "abcs_sense_decode_host": (C.c_int, [P, C.POINTER(SensePlanC), P, I32, P, P, P, I32]),
    "abcs_sense_decode_sweep_host": (C.c_int, [P, C.POINTER(SensePlanC), I32, P, I32, P, I32]),
    "abcs_bench_cells_host": (C.c_int, [P, C.POINTER(SensePlanC), I32, P, I32, P, P, P, I32]),
}

_lib = None
_lock = threading.Lock()


def build(quiet: bool = True) -> None:
    """Compile libabcs_b200.so for sm_100a in-tree (nvcc; no GPU needed)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("building libabcs_b200.so failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])


def load() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            build()
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing and could not be built; no CPU fallback exists")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    return load().abcs_last_error().decode(errors="replace")
