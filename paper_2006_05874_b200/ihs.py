"""Python mirror of the reference solver API (proj/include/ihs/*.hpp).

Same names, argument meaning and error behaviour as the reference C++ API,
implemented over the C-ABI of ``libihs_b200.so`` (include/ihs_gpu.h). Every
numerical call runs on the B200; host code here only marshals arguments.

    reference (C++)                          here
    ProblemInstance(A, b, nu, orientation)   ProblemInstance(A, b, nu, orientation)   problem.hpp:20-55
    gradient(p, x, counters)                 gradient(p, x, counters)                 problem.hpp:59-69
    fwht_inplace(v)                          fwht_inplace(v)                          sketch.hpp:33-49
    gaussian_sketch / srht_sketch / apply_sketch                                      sketch.hpp:58-117
    SketchedSystem::factorize / solve        SketchedSystem.factorize / .solve        sketched_system.hpp:23-66
    newton_decrement(g, g_tilde)             newton_decrement(g, g_tilde)             sketched_system.hpp:95-101
    rates_from_bounds / gaussian_targets / srht_targets                                tuning.hpp:25-63
    adaptive_solve(p, cfg) -> SolveReport    adaptive_solve(p, cfg)                   solver.hpp:242-250
    fixed_sketch_ihs(p, sys, tp, T, mode)    fixed_sketch_ihs(...)                    solver.hpp:258-276
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _abi as abi
from ._lib import lib


# ------------------------------------------------------------------ errors.hpp:9-57
class Error(RuntimeError):
    pass


class InvalidInput(Error):
    pass


class OutOfValidityRange(Error):
    pass


class SketchTooLarge(Error):
    pass


class NumericalBreakdown(Error):
    pass


class ParseError(Error):
    """Text-format parse failure; remembers the 1-based line number (errors.hpp:42-51)."""

    def __init__(self, what: str, line: int):
        super().__init__(f"{what} (line {line})")
        self.line = line


class ShapeError(Error):
    """Rows of a parsed dataset disagree on width (errors.hpp:53-57)."""


class DeviceError(Error):
    """CUDA / NCCL failure (no reference counterpart)."""


_EXC = {
    abi.IHS_INVALID_INPUT: InvalidInput,
    abi.IHS_OUT_OF_VALIDITY_RANGE: OutOfValidityRange,
    abi.IHS_SKETCH_TOO_LARGE: SketchTooLarge,
    abi.IHS_NUMERICAL_BREAKDOWN: NumericalBreakdown,
    abi.IHS_CUDA_ERROR: DeviceError,
    abi.IHS_NCCL_ERROR: DeviceError,
    abi.IHS_INTERNAL_ERROR: Error,
}


def _check(status: int):
    if status != abi.IHS_OK:
        msg = lib().ihs_gpu_last_error().decode(errors="replace")
        raise _EXC.get(status, Error)(msg)


# ------------------------------------------------------------------ enums
class SketchKind(enum.IntEnum):  # sketch.hpp:16
    Gaussian = abi.SKETCH_GAUSSIAN
    SRHT = abi.SKETCH_SRHT


class SolveMode(enum.IntEnum):  # solver.hpp:19-22
    PolyakThenGradient = abi.MODE_POLYAK_THEN_GRADIENT
    GradientOnly = abi.MODE_GRADIENT_ONLY


class StepKind(enum.IntEnum):  # solver.hpp:24
    Polyak = abi.STEP_POLYAK
    Gradient = abi.STEP_GRADIENT
    Resketch = abi.STEP_RESKETCH


class FactorKind(enum.IntEnum):  # sketched_system.hpp:12
    WoodburyInner = abi.FACTOR_WOODBURY_INNER
    DirectGram = abi.FACTOR_DIRECT_GRAM


class Orientation(enum.IntEnum):  # problem.hpp:13
    Overdetermined = 0
    Underdetermined = 1


class FixedMode(enum.IntEnum):  # solver.hpp:252
    Gradient = abi.FIXED_GRADIENT
    Polyak = abi.FIXED_POLYAK


# ------------------------------------------------------------------ types.hpp:18-33
@dataclass
class CostCounters:
    sketch: int = 0
    factor: int = 0
    solve: int = 0
    matvec: int = 0

    def total(self) -> int:
        return self.sketch + self.factor + self.solve + self.matvec

    def _c(self) -> abi.Counters:
        return abi.Counters(self.sketch, self.factor, self.solve, self.matvec)

    def _absorb(self, c: abi.Counters):
        self.sketch, self.factor, self.solve, self.matvec = int(c.sketch), int(c.factor), int(c.solve), int(c.matvec)


class _CounterArg:
    """Pass a CostCounters through the C-ABI and copy the result back."""

    def __init__(self, counters: Optional[CostCounters]):
        self.counters = counters
        self.c = counters._c() if counters is not None else None

    def ptr(self):
        return C.byref(self.c) if self.c is not None else None

    def done(self):
        if self.counters is not None:
            self.counters._absorb(self.c)


# ------------------------------------------------------------------ tuning.hpp:13-63
@dataclass
class TuningParams:
    lam: float = 1.0
    Lam: float = 1.0
    mu_gd: float = 1.0
    c_gd: float = 0.0
    mu_p: float = 1.0
    beta_p: float = 0.0
    c_p: float = 0.0

    def _c(self) -> abi.Tuning:
        return abi.Tuning(self.lam, self.Lam, self.mu_gd, self.c_gd, self.mu_p, self.beta_p, self.c_p)

    @staticmethod
    def _from(t: abi.Tuning) -> "TuningParams":
        return TuningParams(**t.as_dict())


def rates_from_bounds(lam: float, Lam: float) -> TuningParams:
    t = abi.Tuning()
    _check(lib().ihs_rates_from_bounds(lam, Lam, C.byref(t)))
    return TuningParams._from(t)


def gaussian_targets(rho: float, eta: float, enforce_validity: bool = True):
    a, b = C.c_double(), C.c_double()
    _check(lib().ihs_gaussian_targets(rho, eta, int(enforce_validity), C.byref(a), C.byref(b)))
    return a.value, b.value


def srht_targets(rho: float):
    a, b = C.c_double(), C.c_double()
    _check(lib().ihs_srht_targets(rho, C.byref(a), C.byref(b)))
    return a.value, b.value


# ------------------------------------------------------------------ rng.hpp
def derive_seed(seed: int, tag: int) -> int:
    return int(lib().ihs_derive_seed(seed, tag))


def next_pow2(n: int) -> int:
    return int(lib().ihs_next_pow2(n))


def rademacher_bits(stream_seed: int, n: int) -> np.ndarray:
    """Sign bits of rademacher(n, mt19937_64(stream_seed)) generated on the GPU."""
    out = np.zeros((n + 31) // 32, dtype=np.uint32)
    _check(lib().ihs_gpu_rademacher_bits(stream_seed, n, out.ctypes.data_as(C.POINTER(C.c_uint32))))
    return out


def rademacher(stream_seed: int, n: int) -> np.ndarray:
    bits = rademacher_bits(stream_seed, n)
    b = np.unpackbits(bits.view(np.uint8), bitorder="little")[:n]
    return np.where(b == 1, 1.0, -1.0)


def fill_gaussian(stream_seed: int, rows: int, cols: int, stddev: float = 1.0) -> np.ndarray:
    out = np.empty((rows, cols), order="F")
    _check(lib().ihs_gpu_fill_gaussian(stream_seed, rows, cols, stddev, abi.dptr(out)))
    return out


def fill_gaussian_window(stream_seed: int, first: int, count: int, stddev: float = 1.0, streamed: bool = False,
                         block: int = 1 << 20) -> np.ndarray:
    """Normals [first, first + count) of fill_gaussian's stream (a row shard's window of S); streamed uses the
    chunked generator of tall Gaussian sketches."""
    out = np.empty(count)
    _check(lib().ihs_gpu_fill_gaussian_window(stream_seed, first, count, stddev, int(bool(streamed)), block,
                                              abi.dptr(out)))
    return out


def mt19937_64(stream_seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    _check(lib().ihs_gpu_mt19937_64(stream_seed, count, out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return out


def sample_without_replacement(stream_seed: int, n: int, m: int) -> np.ndarray:
    out = np.empty(m, dtype=np.int64)
    _check(lib().ihs_sample_without_replacement(stream_seed, n, m, out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


# ------------------------------------------------------------------ problem.hpp
def _fortran(A) -> np.ndarray:
    A = np.asarray(A, dtype=np.float64)
    if A.ndim != 2:
        raise InvalidInput("expected a matrix")
    return np.asfortranarray(A)


def _vec(x, n=None) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
    if n is not None and x.size != n:
        raise InvalidInput("dimension mismatch")
    return x


def shard_rows(n_global: int, world_size: int, rank: int):
    """(row0, rows) of rank's shard: rows [r*n_loc, (r+1)*n_loc) of the padded index space."""
    r0, rows = C.c_int64(), C.c_int64()
    _check(lib().ihs_gpu_shard_rows(n_global, world_size, rank, C.byref(r0), C.byref(rows)))
    return int(r0.value), int(rows.value)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().ihs_gpu_nccl_unique_id(buf))
    return bytes(buf)


class NcclComm:
    """NCCL communicator owned by the library (the id travels over torch.distributed)."""

    def __init__(self, uid: bytes, world_size: int, rank: int, device: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(lib().ihs_gpu_nccl_comm_create(buf, world_size, rank, device, C.byref(h)))
        self.handle = h

    def close(self):
        """Destroy the communicator now (ncclCommDestroy); also done on garbage collection."""
        h = getattr(self, "handle", None)
        if h:
            lib().ihs_gpu_nccl_comm_destroy(h)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001  (interpreter shutdown: the library wrapper may already be gone)
            pass


def comm_selftest(comm, device: int = 0, count: int = 4099) -> int:
    """Run the sharded path's three collectives (all-reduce sum, all-gather, all-to-all) on exact fp64 patterns
    through `comm` (NcclComm or EmuComm); returns this rank's wrong elements (0 on success)."""
    bad = C.c_int64(-1)
    _check(lib().ihs_gpu_comm_selftest(comm.handle, device, count, C.byref(bad)))
    return int(bad.value)


class EmuComm:
    """One rank's communicator of an EMULATED group (ihs_gpu_emu_comm_create): world_size ranks of this process,
    each driven by its own host thread, run the library's real row-sharded code on one device; collectives are
    host barriers plus device copies. Use EmuComm.group(world_size) and one thread per rank."""

    def __init__(self, handle, group):
        self.handle = handle
        self._group = group  # keeps the sibling handles alive together

    @staticmethod
    def group(world_size: int, device: int = 0):
        arr = (C.c_void_p * world_size)()
        _check(lib().ihs_gpu_emu_comm_create(world_size, device, arr))
        grp = _EmuGroup([arr[r] for r in range(world_size)])
        return [EmuComm(C.c_void_p(arr[r]), grp) for r in range(world_size)]


class _EmuGroup:
    def __init__(self, handles):
        self.handles = handles

    def __del__(self):
        for h in self.handles:
            if h:
                lib().ihs_gpu_nccl_comm_destroy(h)
        self.handles = []


class ProblemInstance:
    """A regularized least-squares instance, uploaded to the device once.

    minimize_x 1/2 ||A x - b||^2 + nu^2/2 ||x||^2 (problem.hpp:15-55).
    For a row-sharded problem pass the local rows (see shard_rows) together
    with world_size, rank, comm (NcclComm) and n_global.
    """

    def __init__(self, A, b, nu: float, orientation: Orientation = Orientation.Overdetermined, device: int = 0,
                 world_size: int = 1, rank: int = 0, comm: Optional["NcclComm"] = None, n_global: Optional[int] = None):
        self._A = _fortran(A)
        self._b = _vec(b)
        self._nu = float(nu)
        self._orientation = Orientation(orientation)
        self._comm = comm
        n, d = self._A.shape
        if self._b.size != n and n >= 1 and d >= 1 and self._nu > 0:
            raise InvalidInput("ProblemInstance: size of b must match rows of A")
        if world_size > 1:
            row0, _ = shard_rows(n_global, world_size, rank)
            opts = abi.GpuOptions(device=device, world_size=world_size, rank=rank,
                                  nccl_comm=comm.handle if comm is not None else None, n_global=n_global,
                                  row_offset=row0)
        else:
            opts = abi.GpuOptions(device=device, world_size=1, rank=0, nccl_comm=None, n_global=n, row_offset=0)
        h = C.c_void_p()
        _check(lib().ihs_gpu_problem_create(abi.dptr(self._A) if self._A.size else None, n, d, max(n, 1),
                                            abi.dptr(self._b) if self._b.size else None, self._nu,
                                            int(self._orientation), C.byref(opts), C.byref(h)))
        self._h = h

    @staticmethod
    def make(A, b, nu: float) -> "ProblemInstance":
        A = _fortran(A)
        o = Orientation.Overdetermined if A.shape[0] >= A.shape[1] else Orientation.Underdetermined
        return ProblemInstance(A, b, nu, o)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # (module globals are already cleared at interpreter shutdown)
            lib().ihs_gpu_problem_destroy(h)
            self._h = None

    def A(self):
        return self._A

    def b(self):
        return self._b

    def nu(self):
        return self._nu

    def orientation(self):
        return self._orientation

    def rows(self):
        return self._A.shape[0]

    def cols(self):
        return self._A.shape[1]

    @property
    def handle(self):
        return self._h

    def set_phase_timing(self, enabled: bool):
        """Per-phase CUDA-event timing of adaptive solves (SolveReport.device_times); default on."""
        _check(lib().ihs_gpu_problem_set_phase_timing(self._h, 1 if enabled else 0))

    def set_nu(self, nu: float):
        """Change nu in place, A staying resident on the device (the regularization path's A-resident
        sweep; bench.hpp:131-171 rebuilds the instance per nu instead)."""
        _check(lib().ihs_gpu_problem_set_nu(self._h, float(nu)))
        self._nu = float(nu)

    def upload(self, A=None, b=None):
        """Re-upload A and/or b (same shape) to the device."""
        Af = _fortran(A) if A is not None else None
        bf = _vec(b, self.rows()) if b is not None else None
        _check(lib().ihs_gpu_problem_upload(self._h, abi.dptr(Af), self.rows(), abi.dptr(bf)))

    def upload_async(self, A=None, b=None):
        """Re-upload A and/or b without waiting: the next solve's A-independent work (sketch RNG) overlaps the
        copy. A and b must be contiguous float64 (column-major A; pinned for a true overlap) and stay alive
        and unchanged until the next call on this instance returns."""
        Af = _fortran(A) if A is not None else None
        bf = _vec(b, self.rows()) if b is not None else None
        def copied(orig, used):  # a conversion copy would die before the transfer reads it
            return orig is not None and np.asarray(orig).__array_interface__["data"][0] != used.ctypes.data
        if copied(A, Af) or copied(b, bf):
            raise InvalidInput("upload_async: A must be Fortran-ordered float64 and b contiguous float64")
        self._pending_upload = (Af, bf)  # keep the host buffers alive until the next call
        _check(lib().ihs_gpu_problem_upload_async(self._h, abi.dptr(Af), self.rows(), abi.dptr(bf)))


def gradient(p: ProblemInstance, x, counters: Optional[CostCounters] = None) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    if x.size != p.cols():
        raise InvalidInput("gradient: dimension mismatch")
    x = np.ascontiguousarray(x)
    g = np.empty(p.cols())
    ca = _CounterArg(counters)
    _check(lib().ihs_gpu_gradient(p.handle, abi.dptr(x), abi.dptr(g), ca.ptr()))
    ca.done()
    return g


def direct_solve(p: ProblemInstance) -> np.ndarray:
    """Exact ridge minimizer (problem.hpp:73-82) on the device: DMMA Gram of the resident A, Cholesky,
    iterative refinement with the fused gradient; the kernel form through the dual when d > n."""
    x = np.empty(p.cols())
    _check(lib().ihs_gpu_direct_solve(p.handle, abi.dptr(x)))
    return x


def prediction_error(p: ProblemInstance, x, x_star) -> float:
    """1/2 ||A (x - x*)||^2 + nu^2/2 ||x - x*||^2 (problem.hpp:104-109), on the device."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
    xs = np.ascontiguousarray(np.asarray(x_star, dtype=np.float64).reshape(-1))
    if x.size != p.cols() or xs.size != p.cols():
        raise InvalidInput("prediction_error: dimension mismatch")
    out = C.c_double()
    _check(lib().ihs_gpu_prediction_error(p.handle, abi.dptr(x), abi.dptr(xs), C.byref(out)))
    return float(out.value)


# ------------------------------------------------------------------ sketch.hpp
def fwht_inplace(v: np.ndarray) -> np.ndarray:
    """In-place normalized FWHT on the device (sketch.hpp:33-49)."""
    if not (isinstance(v, np.ndarray) and v.dtype == np.float64 and v.flags.c_contiguous):
        raise InvalidInput("fwht_inplace: expected a contiguous float64 vector")
    _check(lib().ihs_gpu_fwht(abi.dptr(v) if v.size else None, v.size))
    return v


@dataclass
class SketchConfig:  # sketch.hpp:20-24
    kind: SketchKind = SketchKind.Gaussian
    m: int = 1
    seed: int = 0


def _sketch(A, kind: int, m: int, seed: int, counters: Optional[CostCounters]) -> np.ndarray:
    ca = _CounterArg(counters)
    if isinstance(A, ProblemInstance):
        if m < 1:
            raise InvalidInput(("srht_sketch" if kind == abi.SKETCH_SRHT else "gaussian_sketch") + ": m must be >= 1")
        SA = np.empty((m, A.cols()), order="F")
        _check(lib().ihs_gpu_sketch(A.handle, kind, m, seed, abi.dptr(SA), ca.ptr()))
    else:
        Af = _fortran(A)
        n, d = Af.shape
        SA = np.empty((max(m, 0), d), order="F")
        _check(lib().ihs_gpu_sketch_matrix(abi.dptr(Af), n, d, max(n, 1), kind, m, seed,
                                           abi.dptr(SA) if SA.size else None, ca.ptr()))
    ca.done()
    return SA


def gaussian_sketch(A, m: int, seed: int, counters: Optional[CostCounters] = None) -> np.ndarray:
    return _sketch(A, abi.SKETCH_GAUSSIAN, m, seed, counters)


def srht_sketch(A, m: int, seed: int, counters: Optional[CostCounters] = None) -> np.ndarray:
    return _sketch(A, abi.SKETCH_SRHT, m, seed, counters)


def srht_sketch_sharded_emulated(p: ProblemInstance, m: int, seed: int, shards: int) -> np.ndarray:
    """SRHT through the row-sharded decomposition run on one device (test vehicle)."""
    SA = np.empty((m, p.cols()), order="F")
    _check(lib().ihs_gpu_sketch_sharded_emulated(p.handle, abi.SKETCH_SRHT, m, seed, shards, abi.dptr(SA)))
    return SA


def apply_sketch(A, cfg: SketchConfig, counters: Optional[CostCounters] = None) -> np.ndarray:
    if cfg.kind not in (SketchKind.Gaussian, SketchKind.SRHT):
        raise InvalidInput("apply_sketch: unknown sketch kind")
    return _sketch(A, int(cfg.kind), cfg.m, cfg.seed, counters)


# ------------------------------------------------------------------ sketched_system.hpp
class SketchedSystem:
    """Cached device factorization of H_S = (SA)^T SA + nu^2 I (sketched_system.hpp:23-101)."""

    def __init__(self):
        raise TypeError("use SketchedSystem.factorize")

    @classmethod
    def factorize(cls, SA, nu: float, counters: Optional[CostCounters] = None, device: int = 0) -> "SketchedSystem":
        self = object.__new__(cls)
        self._h = None
        SAf = _fortran(SA)
        m, d = SAf.shape
        self._SA = SAf
        self._nu = float(nu)
        ca = _CounterArg(counters)
        h = C.c_void_p()
        _check(lib().ihs_gpu_system_factorize(abi.dptr(SAf) if SAf.size else None, m, d, max(m, 1), self._nu, device,
                                              ca.ptr(), C.byref(h)))
        ca.done()
        self._h = h
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().ihs_gpu_system_destroy(h)
            self._h = None

    def m(self):
        return self._SA.shape[0]

    def d(self):
        return self._SA.shape[1]

    def nu(self):
        return self._nu

    def kind(self) -> FactorKind:
        return FactorKind(lib().ihs_gpu_system_kind(self._h))

    def SA(self):
        return self._SA

    def factor_flops(self) -> int:
        return int(lib().ihs_gpu_system_factor_flops(self._h))

    def flops_per_solve(self) -> int:
        return int(lib().ihs_gpu_system_flops_per_solve(self._h))

    def solve(self, g, counters: Optional[CostCounters] = None) -> np.ndarray:
        g = np.asarray(g, dtype=np.float64).reshape(-1)
        if g.size != self.d():
            raise InvalidInput("SketchedSystem::solve: dimension mismatch")
        g = np.ascontiguousarray(g)
        z = np.empty(self.d())
        ca = _CounterArg(counters)
        _check(lib().ihs_gpu_system_solve(self._h, abi.dptr(g), abi.dptr(z), ca.ptr()))
        ca.done()
        return z

    @property
    def handle(self):
        return self._h


def newton_decrement(g, g_tilde) -> float:
    g = _vec(g)
    gt = _vec(g_tilde)
    if g.size != gt.size:
        raise InvalidInput("newton_decrement: dimension mismatch")
    r = C.c_double()
    _check(lib().ihs_newton_decrement(abi.dptr(g), abi.dptr(gt), g.size, C.byref(r)))
    return r.value


# ------------------------------------------------------------------ solver.hpp
@dataclass
class SolverConfig:  # solver.hpp:28-57
    rho: float = 0.1
    eta: float = 0.01
    sketch_kind: SketchKind = SketchKind.Gaussian
    m_initial: int = 1
    eps: float = 1e-10
    max_iters: int = 500
    max_sketch: Optional[int] = None
    mode: SolveMode = SolveMode.PolyakThenGradient
    seed: int = 0
    enforce_validity: bool = True
    recompute_r_after_resketch: bool = True
    record_iterates: bool = False
    warm_start: Optional[np.ndarray] = None
    tuning_override: Optional[TuningParams] = None
    sketch_override: Optional[Callable] = None  # (A, m, sub_seed) -> SA (m x d)

    def _c(self, A_for_override=None):
        c = abi.SolverConfigC()
        lib().ihs_solver_config_default(C.byref(c))
        c.rho, c.eta = self.rho, self.eta
        c.sketch_kind = int(self.sketch_kind)
        c.mode = int(self.mode)
        c.m_initial = self.m_initial
        c.eps = self.eps
        c.max_iters = self.max_iters
        c.max_sketch = self.max_sketch if self.max_sketch is not None else 0
        c.seed = self.seed
        c.enforce_validity = int(self.enforce_validity)
        c.recompute_r_after_resketch = int(self.recompute_r_after_resketch)
        c.record_iterates = int(self.record_iterates)
        keep = []
        if self.warm_start is not None:
            ws = _vec(self.warm_start)
            keep.append(ws)
            c.warm_start = abi.dptr(ws)
        if self.tuning_override is not None:
            c.has_tuning_override = 1
            c.tuning_override = self.tuning_override._c()
        if self.sketch_override is not None:
            fn = self.sketch_override

            def tramp(user, m, sub_seed, out):
                try:
                    SA = np.asarray(fn(A_for_override, int(m), int(sub_seed)), dtype=np.float64)
                    d = A_for_override.shape[1]
                    if SA.shape != (m, d):
                        return 1
                    dst = np.ctypeslib.as_array(out, shape=(m * d,))
                    dst[:] = np.asfortranarray(SA).reshape(-1, order="F")
                    return 0
                except Exception:  # noqa: BLE001 - surfaced as InvalidInput by the C side
                    return 1

            cb = abi.SketchOverrideFn(tramp)
            keep.append(cb)
            c.sketch_override = cb
        return c, keep


@dataclass
class IterationRecord:  # solver.hpp:62-68
    t: int
    m: int
    r: float
    r_prev: float
    branch: StepKind


@dataclass
class SolveReport:  # solver.hpp:70-87
    x: np.ndarray
    iterations: int = 1
    rejections: int = 0
    final_m: int = 0
    r1: float = 0.0
    r_final: float = 0.0
    converged: bool = False
    sketch_exhausted: bool = False
    log: List[IterationRecord] = field(default_factory=list)
    iterates: List[np.ndarray] = field(default_factory=list)
    counters: CostCounters = field(default_factory=CostCounters)
    wall_seconds: float = 0.0
    tuning: TuningParams = field(default_factory=TuningParams)
    recompute_r_after_resketch: bool = True
    device_times: dict = field(default_factory=dict)
    dual_final: Optional[np.ndarray] = None  # underdetermined solves (solver.hpp:82)


def _run_solve(fn, p: ProblemInstance, cfg: SolverConfig, dim: int, sketch_matrix, out_dim: int,
               log_capacity: int, dual: bool) -> SolveReport:
    c, keep = cfg._c(sketch_matrix)
    x = np.empty(out_dim)
    rep = abi.SolveReportC()
    rep.x = abi.dptr(x)
    z = None
    if dual:
        z = np.empty(dim)
        rep.dual_final = abi.dptr(z)
    logbuf = (abi.IterationRecordC * log_capacity)()
    rep.log = logbuf
    rep.log_capacity = log_capacity
    its = None
    if cfg.record_iterates:
        cap = cfg.max_iters + 1
        its = np.empty((cap, dim))
        rep.iterates = abi.dptr(its)
        rep.iterates_capacity = cap
    _check(fn(p.handle, C.byref(c), C.byref(rep)))
    del keep
    out = SolveReport(x=x)
    if z is not None:
        out.dual_final = z
    out.iterations, out.rejections, out.final_m = int(rep.iterations), int(rep.rejections), int(rep.final_m)
    out.r1, out.r_final = float(rep.r1), float(rep.r_final)
    out.converged, out.sketch_exhausted = bool(rep.converged), bool(rep.sketch_exhausted)
    out.log = [IterationRecord(int(e.t), int(e.m), float(e.r), float(e.r_prev), StepKind(int(e.branch)))
               for e in logbuf[: min(rep.log_size, log_capacity)]]
    if its is not None:
        out.iterates = [its[i].copy() for i in range(min(rep.iterates_size, its.shape[0]))]
    out.counters._absorb(rep.counters)
    out.wall_seconds = float(rep.wall_seconds)
    out.tuning = TuningParams._from(rep.tuning)
    out.recompute_r_after_resketch = bool(rep.recompute_r_after_resketch)
    out.device_times = rep.times.as_dict()
    return out


def adaptive_solve(p: ProblemInstance, cfg: SolverConfig, log_capacity: int = 1 << 14) -> SolveReport:
    """Adaptive Polyak-IHS (solver.hpp:242-250) on the device-resident problem."""
    if p.orientation() != Orientation.Overdetermined:
        raise InvalidInput("adaptive_solve: expects an overdetermined instance (use solve_underdetermined for d > n)")
    return _run_solve(lib().ihs_gpu_adaptive_solve, p, cfg, p.cols(), p.A(), p.cols(), log_capacity, False)


def solve_underdetermined(p: ProblemInstance, cfg: SolverConfig, log_capacity: int = 1 << 14) -> SolveReport:
    """Underdetermined case through the dual (dual.hpp:13-33): adaptive IHS on the ridge problem in A^T with
    gradient A(A^T z) - b + nu^2 z (SRHT pads d); x = A^T z_T, dual_final = z_T, iterates hold the dual trace."""
    if p.orientation() != Orientation.Underdetermined:
        raise InvalidInput("solve_underdetermined: expects an underdetermined instance")
    return _run_solve(lib().ihs_gpu_solve_underdetermined, p, cfg, p.rows(), np.asfortranarray(p.A().T), p.cols(),
                      log_capacity, True)


def fixed_sketch_ihs(p: ProblemInstance, sys: SketchedSystem, tp: TuningParams, T: int, mode: FixedMode,
                     x_start=None) -> List[np.ndarray]:
    """T fixed-sketch heavy-ball steps (solver.hpp:258-276); returns T+1 iterates."""
    d = p.cols()
    out = np.empty((T + 1, d))
    xs = _vec(x_start, d) if x_start is not None else None
    t = tp._c()
    _check(lib().ihs_gpu_fixed_sketch_ihs(p.handle, sys.handle, C.byref(t), T, int(mode), abi.dptr(xs),
                                          abi.dptr(out)))
    return [out[i].copy() for i in range(T + 1)]


# ------------------------------------------------------------------ baselines.hpp
@dataclass
class CgResult:
    """CgResult / PcgResult (baselines.hpp:16-36); m, m_capped, setup_flops stay 0 for plain CG."""
    x: np.ndarray
    iterations: int = 0
    residuals: List[float] = field(default_factory=list)
    converged: bool = False
    m: int = 0
    m_capped: bool = False
    setup_flops: int = 0
    counters: CostCounters = field(default_factory=CostCounters)
    wall_seconds: float = 0.0
    device_ms: float = 0.0
    kernel_launches: int = 0
    device_times: dict = field(default_factory=dict)


PcgResult = CgResult


def _run_cg(fn, p: ProblemInstance, max_iters: int, x0, *args) -> CgResult:
    d = p.cols()
    x = np.empty(d)
    cap = max(0, int(max_iters)) + 1
    res = np.empty(cap)
    rep = abi.CgReportC()
    rep.x = abi.dptr(x)
    rep.residuals = abi.dptr(res)
    rep.residuals_capacity = cap
    xs = _vec(x0, d) if x0 is not None else None
    _check(fn(p.handle, *args, abi.dptr(xs), C.byref(rep)))
    out = CgResult(x=x, iterations=int(rep.iterations), residuals=res[: min(rep.residuals_size, cap)].tolist(),
                   converged=bool(rep.converged), m=int(rep.m), m_capped=bool(rep.m_capped),
                   setup_flops=int(rep.setup_flops), wall_seconds=float(rep.wall_seconds),
                   device_ms=float(rep.device_ms), kernel_launches=int(rep.kernel_launches),
                   device_times=rep.times.as_dict())
    out.counters._absorb(rep.counters)
    return out


def cg_solve(p: ProblemInstance, tol: float, max_iters: int, x0=None) -> CgResult:
    """CG on the regularized normal equations (baselines.hpp:40-92), H p as one pass over the resident A."""
    if x0 is not None and np.asarray(x0).size != p.cols():
        raise InvalidInput("cg_solve: dimension mismatch")
    return _run_cg(lib().ihs_gpu_cg_solve, p, max_iters, x0, float(tol), int(max_iters))


def pcg_solve_with(p: ProblemInstance, SA, tol: float, max_iters: int, x0=None) -> CgResult:
    """CG preconditioned by the Cholesky factor of SA^T SA + nu^2 I (baselines.hpp:98-165)."""
    SA = _fortran(SA)
    if SA.ndim != 2 or SA.shape[1] != p.cols():
        raise InvalidInput("pcg_solve: dimension mismatch")
    if x0 is not None and np.asarray(x0).size != p.cols():
        raise InvalidInput("pcg_solve: dimension mismatch")
    return _run_cg(lib().ihs_gpu_pcg_solve_with, p, max_iters, x0, abi.dptr(SA), SA.shape[0], SA.shape[0],
                   float(tol), int(max_iters))


def pcg_sketch_size(n: int, d: int, kind: SketchKind, rho: float):
    """baselines.hpp:170-187 -> (m, capped)."""
    m, c = C.c_int64(), C.c_int32()
    _check(lib().ihs_pcg_sketch_size(int(n), int(d), int(kind), float(rho), C.byref(m), C.byref(c)))
    return int(m.value), bool(c.value)


def pcg_solve(p: ProblemInstance, kind: SketchKind, seed: int, rho: float, tol: float, max_iters: int,
              x0=None) -> CgResult:
    """Sketch-preconditioned CG with the prescribed sketch size (baselines.hpp:190-200); the sketch, Gram,
    Cholesky and inverse all run on the device."""
    if x0 is not None and np.asarray(x0).size != p.cols():
        raise InvalidInput("pcg_solve: dimension mismatch")
    return _run_cg(lib().ihs_gpu_pcg_solve, p, max_iters, x0, int(kind), int(seed), float(rho), float(tol),
                   int(max_iters))


# ------------------------------------------------------------------ synthetic data
def synth_generate(n: int, d: int, spectrum: int = 0, decay: float = 0.95, noise_std: float = 0.01,
                   outlier_frac: float = 0.0, outlier_scale: float = 100.0, data_seed: int = 0, threads: int = 0,
                   row0: int = 0, rows: Optional[int] = None, A_out=None, b_out=None):
    """SURVEY §8(d) generator (host, threaded). Returns (A, b, x_true)."""
    rows = n - row0 if rows is None else rows
    spec = abi.SynthSpec(n=n, d=d, spectrum=spectrum, decay=decay, noise_std=noise_std, outlier_frac=outlier_frac,
                         outlier_scale=outlier_scale, data_seed=data_seed, threads=threads)
    A = A_out if A_out is not None else np.empty((rows, d), order="F")
    b = b_out if b_out is not None else np.empty(rows)
    xt = np.empty(d)
    _check(lib().ihs_synth_generate(C.byref(spec), row0, rows, abi.dptr(A), rows, abi.dptr(b), abi.dptr(xt)))
    return A, b, xt


def thread_generated_draws() -> int:
    """MT19937-64 draws this thread's Gaussian sketches generated so far (a row shard's generation work)."""
    return int(lib().ihs_gpu_thread_generated_draws())


def thread_upload_doublings() -> int:
    """Doublings this thread's adaptive solves sketched behind a chunked asynchronous upload (diagnostic)."""
    return int(lib().ihs_gpu_thread_upload_doublings())


def thread_upload_gram_rows() -> int:
    """Rows of sketched Gram matrices this thread's solves enqueued behind a chunked upload (diagnostic)."""
    return int(lib().ihs_gpu_thread_upload_gram_rows())


def kernel_launch_count() -> int:
    return int(lib().ihs_gpu_kernel_launch_count())


def device_count() -> int:
    return int(lib().ihs_gpu_device_count())
