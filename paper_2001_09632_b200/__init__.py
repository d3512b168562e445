"""B200-native ABCS hot path (adaptive block compressive sensing, arXiv 2001.09632).

sm_100a CUDA kernels behind the C ABI in include/abcs_b200.h (libabcs_b200.so,
built in-tree); `abcs` mirrors the reference's abcs:: C++ API on top of it.
"""
from .abcs import *  # noqa: F401,F403
from .abcs import (Algorithm, AllocationPlan, BbvParams, BlockGrid, BudgetSummary, Context, CudaError,  # noqa: F401
                   DenoiserSpec, DivergenceError, FormatError, LogicError, MeasurementBatch, MeasurementSet,
                   ReconConfig, ReconMethod, ReconResult, SensingConfig, SensingOperator, SynthSpec, TraceRow,
                   UnsupportedError, allocate_bbv, bbv_measure, dd_threshold, decode_batch, decode_idct, denoise,
                   ida_batch, largest_remainder_allocate, make_grid, measurement_budget, reconstruct, sense,
                   sense_batch, sense_decode_batch, sense_decode_sweep, sense_dd, sense_plan, sense_zz, synth_images, synth_images_host, zigzag_order)

__all__ = [n for n in dir() if not n.startswith("_")]
