"""Loader for the in-tree sm_100a library ``libihs_b200.so``.

There is no CPU fallback: if the shared library is missing the import of the
product API fails loudly (build it with ``make -C paper_2006_05874_b200`` or
``python -c "import __graft_entry__ as g; g.build()"``).
"""
from __future__ import annotations

import ctypes as C
import pathlib

from . import _abi as abi

PKG_DIR = pathlib.Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libihs_b200.so"

_lib = None


class LibraryMissing(ImportError):
    pass


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise LibraryMissing(f"{LIB_PATH} not built; run `make -C {PKG_DIR}` (no CPU fallback exists)")
    L = C.CDLL(str(LIB_PATH))
    P = C.POINTER
    d = P(C.c_double)
    vp = C.c_void_p
    i32, i64, u64 = C.c_int32, C.c_int64, C.c_uint64
    sigs = {
        "ihs_gpu_last_error": (C.c_char_p, []),
        "ihs_gpu_version": (C.c_char_p, []),
        "ihs_gpu_kernel_launch_count": (i64, []),
        "ihs_gpu_device_count": (C.c_int, []),
        "ihs_rates_from_bounds": (C.c_int, [C.c_double, C.c_double, P(abi.Tuning)]),
        "ihs_gaussian_targets": (C.c_int, [C.c_double, C.c_double, C.c_int, d, d]),
        "ihs_srht_targets": (C.c_int, [C.c_double, d, d]),
        "ihs_derive_seed": (u64, [u64, u64]),
        "ihs_next_pow2": (i64, [i64]),
        "ihs_solver_config_default": (None, [P(abi.SolverConfigC)]),
        "ihs_gpu_problem_create": (C.c_int, [d, i64, i64, i64, d, C.c_double, i32, P(abi.GpuOptions), P(vp)]),
        "ihs_gpu_problem_destroy": (None, [vp]),
        "ihs_gpu_problem_rows": (i64, [vp]),
        "ihs_gpu_problem_cols": (i64, [vp]),
        "ihs_gpu_problem_upload": (C.c_int, [vp, d, i64, d]),
        "ihs_gpu_problem_set_phase_timing": (C.c_int, [vp, C.c_int32]),
        "ihs_gpu_gradient": (C.c_int, [vp, d, d, P(abi.Counters)]),
        "ihs_gpu_sketch": (C.c_int, [vp, i32, i64, u64, d, P(abi.Counters)]),
        "ihs_gpu_fwht": (C.c_int, [d, i64]),
        "ihs_gpu_sketch_matrix": (C.c_int, [d, i64, i64, i64, i32, i64, u64, d, P(abi.Counters)]),
        "ihs_gpu_rademacher_bits": (C.c_int, [u64, i64, P(C.c_uint32)]),
        "ihs_gpu_fill_gaussian": (C.c_int, [u64, i64, i64, C.c_double, d]),
        "ihs_gpu_fill_gaussian_window": (C.c_int, [u64, i64, i64, C.c_double, i32, i64, d]),
        "ihs_gpu_mt19937_64": (C.c_int, [u64, i64, P(C.c_uint64)]),
        "ihs_sample_without_replacement": (C.c_int, [u64, i64, i64, P(C.c_int64)]),
        "ihs_gpu_system_factorize": (C.c_int, [d, i64, i64, i64, C.c_double, i32, P(abi.Counters), P(vp)]),
        "ihs_gpu_system_destroy": (None, [vp]),
        "ihs_gpu_system_kind": (i32, [vp]),
        "ihs_gpu_system_m": (i64, [vp]),
        "ihs_gpu_system_d": (i64, [vp]),
        "ihs_gpu_system_factor_flops": (u64, [vp]),
        "ihs_gpu_system_flops_per_solve": (u64, [vp]),
        "ihs_gpu_system_solve": (C.c_int, [vp, d, d, P(abi.Counters)]),
        "ihs_newton_decrement": (C.c_int, [d, d, i64, d]),
        "ihs_gpu_adaptive_solve": (C.c_int, [vp, P(abi.SolverConfigC), P(abi.SolveReportC)]),
        "ihs_gpu_solve_underdetermined": (C.c_int, [vp, P(abi.SolverConfigC), P(abi.SolveReportC)]),
        "ihs_gpu_prediction_error": (C.c_int, [vp, d, d, d]),
        "ihs_gpu_fixed_sketch_ihs": (C.c_int, [vp, vp, P(abi.Tuning), i64, i32, d, d]),
        "ihs_synth_generate": (C.c_int, [P(abi.SynthSpec), i64, i64, d, i64, d, d]),
        "ihs_gpu_shard_rows": (C.c_int, [i64, i32, i32, P(i64), P(i64)]),
        "ihs_gpu_nccl_unique_id": (C.c_int, [P(C.c_uint8)]),
        "ihs_gpu_nccl_comm_create": (C.c_int, [P(C.c_uint8), i32, i32, i32, P(vp)]),
        "ihs_gpu_nccl_comm_destroy": (None, [vp]),
        "ihs_gpu_emu_comm_create": (C.c_int, [i32, i32, P(vp)]),
        "ihs_gpu_comm_selftest": (C.c_int, [vp, i32, i64, P(i64)]),
        "ihs_gpu_thread_generated_draws": (i64, []),
        "ihs_gpu_thread_upload_doublings": (i64, []),
        "ihs_gpu_thread_upload_gram_rows": (i64, []),
        "ihs_gpu_sketch_sharded_emulated": (C.c_int, [vp, i32, i64, u64, i32, d]),
        "ihs_pcg_sketch_size": (C.c_int, [i64, i64, i32, C.c_double, P(i64), P(i32)]),
        "ihs_gpu_problem_set_nu": (C.c_int, [vp, C.c_double]),
        "ihs_gpu_problem_upload_async": (C.c_int, [vp, d, i64, d]),
        "ihs_gpu_direct_solve": (C.c_int, [vp, d]),
        "ihs_gpu_cg_solve": (C.c_int, [vp, C.c_double, i64, d, P(abi.CgReportC)]),
        "ihs_gpu_pcg_solve_with": (C.c_int, [vp, d, i64, i64, C.c_double, i64, d, P(abi.CgReportC)]),
        "ihs_gpu_pcg_solve": (C.c_int, [vp, i32, u64, C.c_double, C.c_double, i64, d, P(abi.CgReportC)]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return _lib


EXPORTED_SYMBOLS = (
    "ihs_gpu_last_error", "ihs_gpu_version", "ihs_gpu_kernel_launch_count", "ihs_gpu_device_count",
    "ihs_rates_from_bounds", "ihs_gaussian_targets", "ihs_srht_targets", "ihs_derive_seed", "ihs_next_pow2",
    "ihs_solver_config_default", "ihs_gpu_problem_create", "ihs_gpu_problem_destroy", "ihs_gpu_problem_rows",
    "ihs_gpu_problem_cols", "ihs_gpu_problem_upload", "ihs_gpu_problem_set_phase_timing", "ihs_gpu_gradient", "ihs_gpu_sketch", "ihs_gpu_fwht",
    "ihs_gpu_sketch_matrix", "ihs_gpu_rademacher_bits", "ihs_gpu_fill_gaussian", "ihs_gpu_mt19937_64",
    "ihs_sample_without_replacement", "ihs_gpu_system_factorize", "ihs_gpu_system_destroy", "ihs_gpu_system_kind",
    "ihs_gpu_system_m", "ihs_gpu_system_d", "ihs_gpu_system_factor_flops", "ihs_gpu_system_flops_per_solve",
    "ihs_gpu_system_solve", "ihs_newton_decrement", "ihs_gpu_adaptive_solve", "ihs_gpu_solve_underdetermined", "ihs_gpu_prediction_error", "ihs_gpu_fixed_sketch_ihs",
    "ihs_synth_generate", "ihs_gpu_shard_rows", "ihs_gpu_nccl_unique_id", "ihs_gpu_nccl_comm_create",
    "ihs_gpu_nccl_comm_destroy", "ihs_gpu_emu_comm_create", "ihs_gpu_comm_selftest", "ihs_gpu_thread_generated_draws", "ihs_gpu_thread_upload_doublings", "ihs_gpu_thread_upload_gram_rows", "ihs_gpu_sketch_sharded_emulated", "ihs_pcg_sketch_size", "ihs_gpu_cg_solve",
    "ihs_gpu_pcg_solve_with", "ihs_gpu_pcg_solve", "ihs_gpu_problem_set_nu", "ihs_gpu_direct_solve",
    "ihs_gpu_problem_upload_async", "ihs_gpu_fill_gaussian_window",
)
