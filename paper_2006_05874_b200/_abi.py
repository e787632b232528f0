"""ctypes mirror of include/ihs_gpu.h (struct layouts and enums only).

Kept in one place so the product wrapper (`ihs.py`) and the test-side oracle
binding (`oracle/oracle.py`) describe the C boundary identically.
"""
from __future__ import annotations

import ctypes as C

# ihs_status (errors.hpp:15-40 mapping)
IHS_OK = 0
IHS_INVALID_INPUT = 1
IHS_OUT_OF_VALIDITY_RANGE = 2
IHS_SKETCH_TOO_LARGE = 3
IHS_NUMERICAL_BREAKDOWN = 4
IHS_CUDA_ERROR = 5
IHS_NCCL_ERROR = 6
IHS_INTERNAL_ERROR = 7

SKETCH_GAUSSIAN = 0
SKETCH_SRHT = 1
MODE_POLYAK_THEN_GRADIENT = 0
MODE_GRADIENT_ONLY = 1
STEP_POLYAK = 0
STEP_GRADIENT = 1
STEP_RESKETCH = 2
FACTOR_WOODBURY_INNER = 0
FACTOR_DIRECT_GRAM = 1
FIXED_GRADIENT = 0
FIXED_POLYAK = 1


class Counters(C.Structure):
    _fields_ = [("sketch", C.c_uint64), ("factor", C.c_uint64), ("solve", C.c_uint64), ("matvec", C.c_uint64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class Tuning(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("lam", "Lam", "mu_gd", "c_gd", "mu_p", "beta_p", "c_p")]

    def as_dict(self):
        return {k: float(getattr(self, k)) for k, _ in self._fields_}


SketchOverrideFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_uint64, C.POINTER(C.c_double))


class SolverConfigC(C.Structure):
    _fields_ = [
        ("rho", C.c_double),
        ("eta", C.c_double),
        ("sketch_kind", C.c_int32),
        ("mode", C.c_int32),
        ("m_initial", C.c_int64),
        ("eps", C.c_double),
        ("max_iters", C.c_int64),
        ("max_sketch", C.c_int64),
        ("seed", C.c_uint64),
        ("enforce_validity", C.c_int32),
        ("recompute_r_after_resketch", C.c_int32),
        ("record_iterates", C.c_int32),
        ("has_tuning_override", C.c_int32),
        ("tuning_override", Tuning),
        ("warm_start", C.POINTER(C.c_double)),
        ("sketch_override", SketchOverrideFn),
        ("sketch_override_user", C.c_void_p),
    ]


class IterationRecordC(C.Structure):
    _fields_ = [("t", C.c_int64), ("m", C.c_int64), ("r", C.c_double), ("r_prev", C.c_double),
                ("branch", C.c_int32), ("_pad", C.c_int32)]


class PhaseTimes(C.Structure):
    _fields_ = [("sketch_ms", C.c_double), ("factor_ms", C.c_double), ("gradient_ms", C.c_double),
                ("solve_ms", C.c_double), ("n_sketch", C.c_int64), ("n_factor", C.c_int64),
                ("n_gradient", C.c_int64), ("n_solve", C.c_int64), ("kernel_launches", C.c_int64),
                ("total_ms", C.c_double), ("gradient_bytes", C.c_double), ("sketch_bytes", C.c_double),
                ("sketch_flops", C.c_double), ("alloc_ms", C.c_double), ("host_rng_ms", C.c_double),
                ("sketch_kernel_ms", C.c_double), ("n_sketch_kernel", C.c_int64),
                ("gradient_kernel_ms", C.c_double), ("n_gradient_kernel", C.c_int64),
                ("n_srht_l2", C.c_int64), ("n_srht_compact", C.c_int64), ("n_srht_two_kernel", C.c_int64)]

    def as_dict(self):
        return {k: (float if t is C.c_double else int)(getattr(self, k)) for k, t in self._fields_}


class SolveReportC(C.Structure):
    _fields_ = [
        ("x", C.POINTER(C.c_double)),
        ("iterations", C.c_int64),
        ("rejections", C.c_int64),
        ("final_m", C.c_int64),
        ("r1", C.c_double),
        ("r_final", C.c_double),
        ("converged", C.c_int32),
        ("sketch_exhausted", C.c_int32),
        ("log", C.POINTER(IterationRecordC)),
        ("log_capacity", C.c_int64),
        ("log_size", C.c_int64),
        ("iterates", C.POINTER(C.c_double)),
        ("iterates_capacity", C.c_int64),
        ("iterates_size", C.c_int64),
        ("counters", Counters),
        ("wall_seconds", C.c_double),
        ("tuning", Tuning),
        ("recompute_r_after_resketch", C.c_int32),
        ("_pad", C.c_int32),
        ("times", PhaseTimes),
        ("dual_final", C.POINTER(C.c_double)),
    ]


class CgReportC(C.Structure):
    """ihs_cg_report: CgResult / PcgResult (baselines.hpp:16-36)."""
    _fields_ = [
        ("x", C.POINTER(C.c_double)),
        ("residuals", C.POINTER(C.c_double)),
        ("residuals_capacity", C.c_int64),
        ("residuals_size", C.c_int64),
        ("iterations", C.c_int64),
        ("converged", C.c_int32),
        ("m_capped", C.c_int32),
        ("m", C.c_int64),
        ("setup_flops", C.c_uint64),
        ("counters", Counters),
        ("wall_seconds", C.c_double),
        ("device_ms", C.c_double),
        ("kernel_launches", C.c_int64),
        ("times", PhaseTimes),
    ]


class GpuOptions(C.Structure):
    _fields_ = [("device", C.c_int32), ("world_size", C.c_int32), ("rank", C.c_int32), ("_pad", C.c_int32),
                ("nccl_comm", C.c_void_p), ("n_global", C.c_int64), ("row_offset", C.c_int64)]


class SynthSpec(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int64), ("spectrum", C.c_int32), ("_pad", C.c_int32),
                ("decay", C.c_double), ("noise_std", C.c_double), ("outlier_frac", C.c_double),
                ("outlier_scale", C.c_double), ("data_seed", C.c_uint64), ("threads", C.c_int32),
                ("_pad2", C.c_int32)]


def dptr(a):
    """double* of a C-contiguous float64 numpy array (None -> NULL)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))
