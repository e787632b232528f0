"""ctypes binding of the CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module. It restates the reference
hot path (see ihs_oracle.hpp); the product never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib
import subprocess

import numpy as np

from paper_2006_05874_b200 import _abi as abi

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "libihs_oracle.so"
# the reference's own headers compiled against oracle/eigen_stub (oracle/Makefile `ref`; see ref_capi.cpp):
# same entry points with the prefix ihs_ref_, loaded by oracle/ref.py through this very module
REF_LIB_PATH = HERE / "_ref" / "libihs_ref.so"
_PREFIX = "ihs_oracle_"

_STATUS_EXC = {}


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


def build(force: bool = False) -> pathlib.Path:
    if force or not LIB_PATH.exists():
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


class _Prefixed:
    """Maps the ihs_oracle_* names used below onto a library exporting them under another prefix."""

    def __init__(self, cdll, prefix):
        self._cdll = cdll
        self._prefix = prefix

    def __getattr__(self, name):
        if name.startswith("ihs_oracle_"):
            name = self._prefix + name[len("ihs_oracle_"):]
        return getattr(self._cdll, name)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if _PREFIX == "ihs_oracle_":
            build()
            L = C.CDLL(str(LIB_PATH))
        else:
            if not REF_LIB_PATH.exists():
                raise OSError(f"{REF_LIB_PATH} not built (make -C {HERE} ref; needs /root/reference)")
            L = _Prefixed(C.CDLL(str(REF_LIB_PATH)), _PREFIX)
        P = C.POINTER
        d = P(C.c_double)
        L.ihs_oracle_last_error.restype = C.c_char_p
        L.ihs_oracle_derive_seed.restype = C.c_uint64
        L.ihs_oracle_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ihs_oracle_mt_raw.argtypes = [C.c_uint64, C.c_int64, P(C.c_uint64)]
        L.ihs_oracle_rademacher.argtypes = [C.c_uint64, C.c_int64, d]
        L.ihs_oracle_sample_wor.argtypes = [C.c_uint64, C.c_int64, C.c_int64, P(C.c_int64)]
        L.ihs_oracle_fill_gaussian.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_double, d]
        L.ihs_oracle_fwht.argtypes = [d, C.c_int64]
        L.ihs_oracle_next_pow2.restype = C.c_int64
        L.ihs_oracle_next_pow2.argtypes = [C.c_int64]
        L.ihs_oracle_sketch.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_uint64, d,
                                        P(abi.Counters)]
        L.ihs_oracle_gradient.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, d, C.c_double, d, d, P(abi.Counters)]
        L.ihs_oracle_system_solve.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, C.c_double, d, d, P(C.c_int32),
                                              P(C.c_uint64), P(C.c_uint64), P(abi.Counters)]
        L.ihs_oracle_newton_decrement.argtypes = [d, d, C.c_int64, d]
        L.ihs_oracle_rates_from_bounds.argtypes = [C.c_double, C.c_double, P(abi.Tuning)]
        L.ihs_oracle_gaussian_targets.argtypes = [C.c_double, C.c_double, C.c_int, d, d]
        L.ihs_oracle_srht_targets.argtypes = [C.c_double, d, d]
        L.ihs_oracle_test_support_data.argtypes = [C.c_uint64, C.c_int64, C.c_int64, d, C.c_int64, d]
        L.ihs_oracle_solve_underdetermined.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, d, C.c_double,
                                                       C.POINTER(abi.SolverConfigC), C.POINTER(abi.SolveReportC)]
        L.ihs_oracle_adaptive_solve.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, d, C.c_double,
                                                P(abi.SolverConfigC), P(abi.SolveReportC)]
        L.ihs_oracle_fixed_sketch_ihs.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, d, C.c_double, d, C.c_int64,
                                                  P(abi.Tuning), C.c_int64, C.c_int32, d, d]
        L.ihs_oracle_direct_solve.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, d, C.c_double, d]
        L.ihs_oracle_prediction_error.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, d, C.c_double, d, d, d]
        L.ihs_oracle_synth.argtypes = [P(abi.SynthSpec), d, d, d]
        L.ihs_oracle_cg.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, d, C.c_double, C.c_int32, d, C.c_int64,
                                    C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_double, C.c_int64, d,
                                    P(abi.CgReportC)]
        L.ihs_oracle_pcg_sketch_size.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_double, P(C.c_int64),
                                                 P(C.c_int32)]
        if not hasattr(L, "ihs_oracle_time_sketch"):  # the reference build (oracle/ref.py) has no timing hooks
            _lib = L
            return _lib
        L.ihs_oracle_time_sketch.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_uint64, d,
                                             P(abi.Counters)]
        L.ihs_oracle_time_fill_gaussian.argtypes = [C.c_uint64, C.c_int64, C.c_int64, d]
        L.ihs_oracle_time_gradient.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, d, C.c_double, d, C.c_int32, d,
                                               P(abi.Counters)]
        L.ihs_oracle_time_system.argtypes = [d, C.c_int64, C.c_int64, C.c_int64, C.c_double, d, C.c_int32, d, d,
                                             P(abi.Counters)]
        _lib = L
    return _lib


def _check(status):
    if status != 0:
        raise OracleError(status, lib().ihs_oracle_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _fortran(A):
    return np.asfortranarray(A, dtype=np.float64)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ----------------------------------------------------------------- rng.hpp
def derive_seed(seed: int, tag: int) -> int:
    return int(lib().ihs_oracle_derive_seed(seed, tag))


def mt_raw(stream_seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().ihs_oracle_mt_raw(stream_seed, count, out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def rademacher(stream_seed: int, n: int) -> np.ndarray:
    out = np.empty(n)
    lib().ihs_oracle_rademacher(stream_seed, n, _dp(out))
    return out


def sample_without_replacement(stream_seed: int, n: int, m: int) -> np.ndarray:
    out = np.empty(m, dtype=np.int64)
    lib().ihs_oracle_sample_wor(stream_seed, n, m, out.ctypes.data_as(C.POINTER(C.c_int64)))
    return out


def fill_gaussian(stream_seed: int, rows: int, cols: int, stddev: float = 1.0) -> np.ndarray:
    out = np.empty((rows, cols), order="F")
    lib().ihs_oracle_fill_gaussian(stream_seed, rows, cols, stddev, _dp(out))
    return out


# ----------------------------------------------------------------- sketch.hpp
def next_pow2(n: int) -> int:
    return int(lib().ihs_oracle_next_pow2(n))


def fwht_inplace(v: np.ndarray) -> np.ndarray:
    v = _f64(v).copy()
    _check(lib().ihs_oracle_fwht(_dp(v), v.size))
    return v


def sketch(A, kind: int, m: int, seed: int, counters: abi.Counters | None = None) -> np.ndarray:
    A = _fortran(A)
    n, d = A.shape
    SA = np.empty((m, d), order="F")
    c = counters if counters is not None else abi.Counters()
    _check(lib().ihs_oracle_sketch(_dp(A), n, d, n, kind, m, seed, _dp(SA), C.byref(c)))
    return SA


def srht_sketch(A, m, seed, counters=None):
    return sketch(A, abi.SKETCH_SRHT, m, seed, counters)


def gaussian_sketch(A, m, seed, counters=None):
    return sketch(A, abi.SKETCH_GAUSSIAN, m, seed, counters)


# ----------------------------------------------------------------- problem / system
def gradient(A, b, nu, x, counters=None):
    A = _fortran(A)
    n, d = A.shape
    b = _f64(b)
    x = _f64(x)
    g = np.empty(d)
    c = counters if counters is not None else abi.Counters()
    _check(lib().ihs_oracle_gradient(_dp(A), n, d, n, _dp(b), nu, _dp(x), _dp(g), C.byref(c)))
    return g


def system_solve(SA, nu, g=None, counters=None):
    SA = _fortran(SA)
    m, d = SA.shape
    kind = C.c_int32()
    ff = C.c_uint64()
    fps = C.c_uint64()
    c = counters if counters is not None else abi.Counters()
    z = np.empty(d) if g is not None else None
    gg = _f64(g) if g is not None else None
    _check(lib().ihs_oracle_system_solve(_dp(SA), m, d, m, nu, _dp(gg) if gg is not None else None,
                                         _dp(z) if z is not None else None, C.byref(kind), C.byref(ff),
                                         C.byref(fps), C.byref(c)))
    return z, int(kind.value), int(ff.value), int(fps.value)


def newton_decrement(g, gt):
    r = C.c_double()
    g = _f64(g)
    gt = _f64(gt)
    _check(lib().ihs_oracle_newton_decrement(_dp(g), _dp(gt), g.size, C.byref(r)))
    return r.value


def rates_from_bounds(lam, Lam):
    t = abi.Tuning()
    _check(lib().ihs_oracle_rates_from_bounds(lam, Lam, C.byref(t)))
    return t


def gaussian_targets(rho, eta, enforce_validity=True):
    a, b = C.c_double(), C.c_double()
    _check(lib().ihs_oracle_gaussian_targets(rho, eta, int(enforce_validity), C.byref(a), C.byref(b)))
    return a.value, b.value


def srht_targets(rho):
    a, b = C.c_double(), C.c_double()
    _check(lib().ihs_oracle_srht_targets(rho, C.byref(a), C.byref(b)))
    return a.value, b.value


def adaptive_solve(A, b, nu, cfg: abi.SolverConfigC, log_capacity=4096, iterates_capacity=0):
    """Returns (x, report-struct, log list). cfg is an abi.SolverConfigC."""
    A = _fortran(A)
    n, d = A.shape
    b = _f64(b)
    x = np.empty(d)
    rep = abi.SolveReportC()
    rep.x = _dp(x)
    logbuf = (abi.IterationRecordC * log_capacity)()
    rep.log = logbuf
    rep.log_capacity = log_capacity
    its = None
    if iterates_capacity:
        its = np.empty((iterates_capacity, d))
        rep.iterates = _dp(its)
        rep.iterates_capacity = iterates_capacity
    _check(lib().ihs_oracle_adaptive_solve(_dp(A), n, d, n, _dp(b), nu, C.byref(cfg), C.byref(rep)))
    log = [(int(e.t), int(e.m), float(e.r), float(e.r_prev), int(e.branch))
           for e in logbuf[: min(rep.log_size, log_capacity)]]
    if its is not None:
        its = its[: rep.iterates_size]
    return x, rep, log, its


def test_support_data(seed, rows, cols, vlen=0):
    """proj/tests/support.hpp:32-47: (random_matrix(rows, cols, gen), random_vector(vlen, gen)) from
    one std::mt19937_64(seed), the reference tests' own data."""
    M = np.empty((rows, cols), order="F")
    v = np.empty(vlen)
    _check(lib().ihs_oracle_test_support_data(seed, rows, cols, _dp(M), vlen, _dp(v) if vlen else None))
    return M, v


def solve_underdetermined(A, b, nu, cfg: abi.SolverConfigC, log_capacity=4096, iterates_capacity=0):
    """dual.hpp:13-33. Returns (x, z (dual_final), report-struct, log list, dual iterates)."""
    A = _fortran(A)
    n, d = A.shape
    b = _f64(b)
    x = np.empty(d)
    z = np.empty(n)
    rep = abi.SolveReportC()
    rep.x = _dp(x)
    rep.dual_final = _dp(z)
    logbuf = (abi.IterationRecordC * log_capacity)()
    rep.log = logbuf
    rep.log_capacity = log_capacity
    its = None
    if iterates_capacity:
        its = np.empty((iterates_capacity, n))
        rep.iterates = _dp(its)
        rep.iterates_capacity = iterates_capacity
    _check(lib().ihs_oracle_solve_underdetermined(_dp(A), n, d, n, _dp(b), nu, C.byref(cfg), C.byref(rep)))
    log = [(int(e.t), int(e.m), float(e.r), float(e.r_prev), int(e.branch))
           for e in logbuf[: min(rep.log_size, log_capacity)]]
    if its is not None:
        its = its[: rep.iterates_size]
    return x, z, rep, log, its


def fixed_sketch_ihs(A, b, nu, SA, tuning: abi.Tuning, T, mode, x_start=None):
    A = _fortran(A)
    n, d = A.shape
    SA = _fortran(SA)
    out = np.empty((T + 1, d))
    xs = _f64(x_start) if x_start is not None else None
    _check(lib().ihs_oracle_fixed_sketch_ihs(_dp(A), n, d, n, _dp(_f64(b)), nu, _dp(SA), SA.shape[0],
                                             C.byref(tuning), T, mode, _dp(xs) if xs is not None else None,
                                             _dp(out)))
    return out


def direct_solve(A, b, nu):
    A = _fortran(A)
    n, d = A.shape
    x = np.empty(d)
    _check(lib().ihs_oracle_direct_solve(_dp(A), n, d, n, _dp(_f64(b)), nu, _dp(x)))
    return x


def prediction_error(A, b, nu, x, xs):
    A = _fortran(A)
    n, d = A.shape
    out = C.c_double()
    _check(lib().ihs_oracle_prediction_error(_dp(A), n, d, n, _dp(_f64(b)), nu, _dp(_f64(x)), _dp(_f64(xs)),
                                             C.byref(out)))
    return out.value


def synth(n, d, spectrum=0, decay=0.95, noise_std=0.01, outlier_frac=0.0, outlier_scale=100.0, data_seed=0):
    spec = abi.SynthSpec(n=n, d=d, spectrum=spectrum, decay=decay, noise_std=noise_std, outlier_frac=outlier_frac,
                         outlier_scale=outlier_scale, data_seed=data_seed)
    A = np.empty((n, d), order="F")
    b = np.empty(n)
    xt = np.empty(d)
    _check(lib().ihs_oracle_synth(C.byref(spec), _dp(A), _dp(b), _dp(xt)))
    return A, b, xt


def default_config(**kw) -> abi.SolverConfigC:
    """SolverConfig defaults (solver.hpp:28-57)."""
    c = abi.SolverConfigC()
    c.rho = 0.1
    c.eta = 0.01
    c.sketch_kind = abi.SKETCH_GAUSSIAN
    c.mode = abi.MODE_POLYAK_THEN_GRADIENT
    c.m_initial = 1
    c.eps = 1e-10
    c.max_iters = 500
    c.max_sketch = 0
    c.seed = 0
    c.enforce_validity = 1
    c.recompute_r_after_resketch = 1
    c.record_iterates = 0
    c.has_tuning_override = 0
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def _cg(method, A, b, nu, tol, max_iters, x0=None, SA=None, kind=0, seed=0, rho=0.5):
    A = _fortran(A)
    n, d = A.shape
    b = _f64(b)
    x = np.empty(d)
    cap = max_iters + 1
    res = np.empty(cap)
    rep = abi.CgReportC()
    rep.x = _dp(x)
    rep.residuals = _dp(res)
    rep.residuals_capacity = cap
    SAf = _fortran(SA) if SA is not None else None
    x0 = _f64(x0) if x0 is not None else None
    _check(lib().ihs_oracle_cg(_dp(A), n, d, n, _dp(b), nu, method, _dp(SAf) if SAf is not None else None,
                               SAf.shape[0] if SAf is not None else 0, SAf.shape[0] if SAf is not None else 0,
                               kind, seed, rho, tol, max_iters, _dp(x0) if x0 is not None else None, C.byref(rep)))
    return x, res[: min(rep.residuals_size, cap)].copy(), rep


def cg_solve(A, b, nu, tol, max_iters, x0=None):
    """baselines.hpp:40-92. Returns (x, residuals, report-struct)."""
    return _cg(0, A, b, nu, tol, max_iters, x0)


def pcg_solve_with(A, b, nu, SA, tol, max_iters, x0=None):
    """baselines.hpp:98-165."""
    return _cg(1, A, b, nu, tol, max_iters, x0, SA=SA)


def pcg_solve(A, b, nu, kind, seed, rho, tol, max_iters, x0=None):
    """baselines.hpp:190-200."""
    return _cg(2, A, b, nu, tol, max_iters, x0, kind=kind, seed=seed, rho=rho)


def pcg_sketch_size(n, d, kind, rho):
    """baselines.hpp:170-187 -> (m, capped)."""
    m, c = C.c_int64(), C.c_int32()
    _check(lib().ihs_oracle_pcg_sketch_size(n, d, kind, rho, C.byref(m), C.byref(c)))
    return m.value, bool(c.value)


# ----------------------------------------------------------------- host phase timings (bench.py cpu_baseline)
def time_sketch(A, kind, m, seed):
    """Seconds of one apply_sketch (sketch.hpp:110-117) on A (inputs prepared outside the timer), counters."""
    A = _fortran(A)
    n, d = A.shape
    t = C.c_double()
    c = abi.Counters()
    _check(lib().ihs_oracle_time_sketch(_dp(A), n, d, n, kind, m, seed, C.byref(t), C.byref(c)))
    return t.value, c


def time_fill_gaussian(stream_seed, rows, cols):
    t = C.c_double()
    _check(lib().ihs_oracle_time_fill_gaussian(stream_seed, rows, cols, C.byref(t)))
    return t.value


def time_gradient(A, b, nu, x, reps=1):
    """Seconds of `reps` gradient calls (problem.hpp:59-69) on a problem built outside the timer, counters."""
    A = _fortran(A)
    n, d = A.shape
    t = C.c_double()
    c = abi.Counters()
    _check(lib().ihs_oracle_time_gradient(_dp(A), n, d, n, _dp(_f64(b)), nu, _dp(_f64(x)), reps, C.byref(t),
                                          C.byref(c)))
    return t.value, c


def time_system(SA, nu, g, solves=1):
    """(seconds of SketchedSystem::factorize, seconds of `solves` solves, counters) (sketched_system.hpp)."""
    SA = _fortran(SA)
    m, d = SA.shape
    tf, ts = C.c_double(), C.c_double()
    c = abi.Counters()
    _check(lib().ihs_oracle_time_system(_dp(SA), m, d, m, nu, _dp(_f64(g)), solves, C.byref(tf), C.byref(ts),
                                        C.byref(c)))
    return tf.value, ts.value, c
