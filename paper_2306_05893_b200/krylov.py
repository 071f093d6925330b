"""SpMV and (preconditioned) CG on the B200 (drop-in for tetsim.krylov, krylov.py:1-163).

`spmv` is bit-identical to the reference (same per-row summation order).
`pcg`/`cg` run entirely on the device for the identity, Jacobi and
nested-dissection LDL^T preconditioners: one persistent cooperative kernel
per solve (csrc/pcg.cu), alpha/beta/convergence on the device, one report
read back per solve.  Vectors may be NumPy arrays (copied in/out, reference
semantics) or CUDA tensors (stay resident; the solution is returned as a
CUDA tensor).
"""

from __future__ import annotations

import enum
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .assembly import CsrMatrix

__all__ = [
    "SolverError",
    "SolveMode",
    "SolverConfig",
    "SolveReport",
    "spmv",
    "cg",
    "pcg",
    "jacobi_precond",
    "IdentityPreconditioner",
    "JacobiPreconditioner",
]


class SolverError(ValueError):
    pass


class SolveMode(enum.Enum):
    CG = "cg"
    PCG_JACOBI = "pcg-jacobi"
    PCG_LDLT = "pcg-ldlt"


@dataclass
class SolverConfig:
    tolerance: float = 1e-9
    max_iterations: int = 1000
    mode: SolveMode = SolveMode.CG

    def __post_init__(self):
        if not self.tolerance > 0:
            raise SolverError(f"tolerance must be positive, got {self.tolerance}")


@dataclass
class SolveReport:
    iterations: int
    final_residual: float
    converged: bool
    wall_time: float


def _vec_in(x, n, what="vector"):
    """-> (cuda float64 tensor, was_host)."""
    t = _lib.require_cuda()
    if _lib.is_tensor(x):
        if x.numel() != n:
            raise SolverError(f"dimension mismatch: {what} has {x.numel()} entries, expected {n}")
        return x.to(device="cuda", dtype=t.float64).contiguous().view(-1), False
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())
    if len(arr) != n:
        raise SolverError(f"dimension mismatch: {what} has {len(arr)} entries, expected {n}")
    return t.from_numpy(arr).cuda(), True


def spmv(a: CsrMatrix, x, workers: int = 1):
    """y = A @ x on the device, bit-identical to the reference's reduceat order."""
    n_x = x.numel() if _lib.is_tensor(x) else len(x)
    if n_x != a.ncols:
        raise SolverError(f"dimension mismatch: matrix is {a.nrows}x{a.ncols}, vector has {n_x}")
    t = _lib.require_cuda()
    dx, host = _vec_in(x, a.ncols)
    y = t.zeros(a.nrows, dtype=t.float64, device="cuda")
    if a.nnz:
        d_rp, d_ci = a.device_pattern()
        dv = a.device_values()
        _lib.check(_lib.load().tsb_spmv(a.nrows, _lib.ptr(d_rp), _lib.ptr(d_ci), _lib.ptr(dv),
                                        _lib.ptr(dx), _lib.ptr(y), _lib.stream_ptr()), "spmv")
    return y.cpu().numpy() if host else y


class IdentityPreconditioner:
    def apply(self, r):
        return r


class JacobiPreconditioner:
    """z = r * (1/diag) (krylov.py:104-109).  Built from a matrix, the diagonal
    is extracted and inverted on the device inside the solve."""

    def __init__(self, diag=None, *, matrix: CsrMatrix | None = None):
        self._matrix = matrix
        self._diag = None if diag is None else np.asarray(diag, dtype=np.float64)
        self._inv = None if diag is None else 1.0 / self._diag

    @property
    def inv_diag(self) -> np.ndarray:
        if self._inv is None:
            self._diag = self._matrix.diagonal()
            self._inv = 1.0 / self._diag
        return self._inv

    def device_inv_diag(self):
        """1/diag of the matrix this preconditioner was built from, as a CUDA
        tensor (computed once; on the device for a device matrix)."""
        if getattr(self, "_dinv", None) is None:
            t = _lib.require_cuda()
            m = self._matrix
            if self._inv is None and m is not None and m.on_device:
                d = t.empty(min(m.nrows, m.ncols), dtype=t.float64, device="cuda")
                d_rp, d_ci = m.device_pattern()
                _lib.check(_lib.load().tsb_csr_diagonal(m.nrows, m.ncols, _lib.ptr(d_rp), _lib.ptr(d_ci),
                                                        _lib.ptr(m.device_values()), _lib.ptr(d),
                                                        _lib.stream_ptr()), "csr_diagonal")
                zero = t.nonzero(d == 0.0)
                if zero.numel():
                    raise SolverError(f"zero diagonal entry at row {int(zero[0, 0])}")
                self._dinv = 1.0 / d
            else:
                self._dinv = t.from_numpy(np.ascontiguousarray(self.inv_diag)).cuda()
        return self._dinv

    def apply(self, r):
        if _lib.is_tensor(r):
            t = _lib.torch()
            return r * t.from_numpy(self.inv_diag).to(r.device)
        return r * self.inv_diag


def jacobi_precond(a: CsrMatrix) -> JacobiPreconditioner:
    """Diagonal preconditioner.  A zero diagonal raises SolverError; for
    device-resident matrices the check runs on the device during the solve
    (no host round-trip here), for host matrices it runs immediately."""
    if not a.on_device:
        d = a.diagonal()
        if np.any(d == 0.0):
            raise SolverError(f"zero diagonal entry at row {int(np.flatnonzero(d == 0.0)[0])}")
        return JacobiPreconditioner(d)
    return JacobiPreconditioner(matrix=a)


# ---------------------------------------------------------------------------
# device PCG
# ---------------------------------------------------------------------------

class _PcgHandle:
    """One libtsb PCG workspace (device vectors + report struct)."""

    pending = None

    def __init__(self, n: int):
        import ctypes as C

        lib = _lib.load()
        h = C.c_void_p()
        _lib.check(lib.tsb_pcg_create(n, C.byref(h)), "pcg_create")
        self.h = h
        self.n = n
        self._lib = lib

    def __del__(self):
        try:
            if self.h:
                self._lib.tsb_pcg_destroy(self.h)
        except Exception:
            pass


_handles: dict[int, _PcgHandle] = {}


def _handle(n: int) -> _PcgHandle:
    h = _handles.get(n)
    if h is None:
        h = _PcgHandle(n)
        _handles[n] = h
    return h


def _precond_kind(precond, a):
    """-> (kind, ldlt device handle or None, inv_diag tensor or None) or None for a host object."""
    from . import ndprecond

    if precond is None or isinstance(precond, IdentityPreconditioner):
        return _lib.PRECOND_IDENTITY, None, None
    if isinstance(precond, JacobiPreconditioner):
        if precond._matrix is a:
            # the diagonal of the matrix being solved: extracted and inverted inside the kernel
            return _lib.PRECOND_JACOBI, None, None
        # built from another matrix: keep ITS diagonal, as the reference does (krylov.py:104-117)
        return _lib.PRECOND_JACOBI, None, precond.device_inv_diag()
    factors = ndprecond.as_factors(precond)
    if factors is not None:
        return _lib.PRECOND_LDLT, factors.device(), None
    return None


class _DeviceReport:
    """SolveReport of a device solve whose report struct is read back lazily:
    a caller that only enqueues more device work (the integrator's kinematic
    update) does not stall the stream; the first attribute read synchronises."""

    def __init__(self, handle, t0):
        self._h, self._t0, self._r = handle, t0, None
        handle.pending = self  # the next solve on this workspace reads it first

    def _get(self):
        if self._r is None:
            import ctypes as C

            rep = _lib.Report()
            _lib.check(_lib.load().tsb_pcg_report(self._h.h, C.byref(rep), _lib.stream_ptr()), "pcg_report")
            if rep.status == _lib.TSB_E_SOLVER:
                raise SolverError(f"zero diagonal entry at row {int(rep.zero_diag_row)}")
            self._r = SolveReport(int(rep.iterations), float(rep.final_residual), bool(rep.converged),
                                  time.perf_counter() - self._t0)
        return self._r

    iterations = property(lambda self: self._get().iterations)
    final_residual = property(lambda self: self._get().final_residual)
    converged = property(lambda self: self._get().converged)
    wall_time = property(lambda self: self._get().wall_time)

    def __repr__(self):
        return repr(self._get())


def pcg(a: CsrMatrix, b, precond, config: SolverConfig, x0=None, workers: int = 1):
    """Preconditioned CG (krylov.py:120-158); returns (x, SolveReport).  With a
    device right-hand side the report is read back lazily (see _DeviceReport)."""
    t0 = time.perf_counter()
    n = a.ncols
    kind = _precond_kind(precond, a)
    if kind is None:
        return _pcg_host_preconditioner(a, b, precond, config, x0, t0)
    kind, ldlt, inv = kind
    t = _lib.require_cuda()
    db, host = _vec_in(b, n, "rhs")
    dx0 = _vec_in(x0, n, "x0")[0] if x0 is not None else None
    x = t.empty(n, dtype=t.float64, device="cuda")
    if not host:
        solve_device(a, db, x, kind, ldlt, config.tolerance, config.max_iterations, x0=dx0, inv_diag=inv,
                     sync=False)
        return x, _DeviceReport(_handle(a.nrows), t0)
    rep = solve_device(a, db, x, kind, ldlt, config.tolerance, config.max_iterations, x0=dx0, inv_diag=inv)
    report = SolveReport(int(rep.iterations), float(rep.final_residual), bool(rep.converged),
                         time.perf_counter() - t0)
    return x.cpu().numpy(), report


def solve_device(a: CsrMatrix, d_b, d_x, kind, ldlt, tol, max_it, x0=None, inv_diag=None, sync=True):
    """Enqueue one device PCG solve; returns the libtsb report (synchronising once) or None."""
    import ctypes as C

    lib = _lib.load()
    if a.nrows != a.ncols:
        raise SolverError(f"pcg needs a square matrix, got {a.nrows}x{a.ncols}")
    h = _handle(a.nrows)
    if h.pending is not None:  # a lazily read report of this workspace: fetch it before it is overwritten
        h.pending._get()
        h.pending = None
    d_rp, d_ci = a.device_pattern()
    dv = a.device_values()
    rep = _lib.Report()
    status = lib.tsb_pcg_solve(
        h.h, a.nrows, _lib.ptr(d_rp), _lib.ptr(d_ci), _lib.ptr(dv), _lib.ptr(d_b),
        _lib.ptr(x0), _lib.ptr(d_x), kind, ldlt.h if ldlt is not None else None,
        _lib.ptr(inv_diag), float(tol), int(max_it), C.byref(rep) if sync else None,
        _lib.stream_ptr(),
    )
    _lib.check(status, "pcg")
    if sync and rep.status == _lib.TSB_E_SOLVER:
        raise SolverError(f"zero diagonal entry at row {int(rep.zero_diag_row)}")
    return rep if sync else None


def _pcg_host_preconditioner(a, b, precond, config, x0, t0):
    """PCG with an arbitrary Python preconditioner object (.apply(r) -> z).

    The reference's preconditioner protocol (krylov.py:99-109) admits any
    object; one that is not an identity, Jacobi or LDL^T preconditioner
    cannot run inside the device graph, so its .apply runs where the caller
    wrote it (on host arrays) while every SpMV runs on the device.  This is
    the API-compatibility path, not the hot path.
    """
    n = a.ncols
    x = np.zeros(n) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    b = np.asarray(b.cpu().numpy() if _lib.is_tensor(b) else b, dtype=np.float64)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return np.zeros(n), SolveReport(0, 0.0, True, time.perf_counter() - t0)
    r = b - spmv(a, x) if x0 is not None else b.copy()
    res = float(np.linalg.norm(r)) / bnorm
    if res <= config.tolerance:
        return x, SolveReport(0, res, True, time.perf_counter() - t0)
    z = np.asarray(precond.apply(r), dtype=np.float64)
    p = z.copy()
    rz = float(r @ z)
    it = 0
    converged = False
    while it < config.max_iterations:
        ap = spmv(a, p)
        alpha = rz / float(p @ ap)
        x += alpha * p
        r -= alpha * ap
        it += 1
        res = float(np.linalg.norm(r)) / bnorm
        if res <= config.tolerance:
            converged = True
            break
        z = np.asarray(precond.apply(r), dtype=np.float64)
        rz_next = float(r @ z)
        p = z + (rz_next / rz) * p
        rz = rz_next
    return x, SolveReport(it, res, converged, time.perf_counter() - t0)


def cg(a: CsrMatrix, b, config: SolverConfig, x0=None, workers: int = 1):
    """Plain CG = identity-preconditioned pcg (krylov.py:161-163); same device path."""
    return pcg(a, b, IdentityPreconditioner(), config, x0=x0, workers=workers)
