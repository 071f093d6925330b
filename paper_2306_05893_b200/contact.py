"""Plane-contact stage on the B200 (drop-in for tetsim.contact, contact.py:1-257).

Free motion (the device implicit step), constraint resolution and motion
correction, with the reference's API and semantics:

  detect_plane_contacts   ordered compaction of the nodes below the plane
                          (tsb_plane_contacts)
  build_compliance        W = J A^-1 J^T column by column through the given
                          solve, then J S symmetrised (tsb_compliance_from_columns)
  projected_gauss_seidel  one-warp PGS in constraint order (tsb_pgs)
  correct_motion          a = a_free - S lambda, kinematics (tsb_contact_correct,
                          tsb_advance)

PlaneContactPipeline.step additionally takes LDL^T factors directly
(`apply_inverse=factors`, an LdlFactors or a ready AsyncPreconditioner):
then the compliance needs only lower sweeps and one upper sweep,

    W = J A^-1 J^T = Y^T D^-1 Y,  Y = L^-1 P J^T;   S lambda = P^T L^-T D^-1 (Y lambda)

(the same matrix as the reference's m full applies, mathematically).  Any
other callable is used exactly as the reference uses it, one column at a time.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

from . import _lib
from .integrator import BackwardEulerIntegrator, SimState, StepResult

logger = logging.getLogger(__name__)

__all__ = [
    "ContactError",
    "ConstraintSet",
    "detect_plane_contacts",
    "build_compliance",
    "projected_gauss_seidel",
    "correct_motion",
    "ContactStepInfo",
    "PlaneContactPipeline",
    "BILATERAL",
    "UNILATERAL",
]

BILATERAL = "bilateral"
UNILATERAL = "unilateral"


class ContactError(RuntimeError):
    pass


@dataclass
class ConstraintSet:
    """Sparse constraint Jacobian (one CSR row per constraint) + violations (contact.py:48-86)."""

    ndof: int
    indptr: np.ndarray
    col_ind: np.ndarray
    coeffs: np.ndarray
    violation: np.ndarray
    types: list

    @property
    def nconstraints(self) -> int:
        return len(self.violation)

    def row_dense(self, i: int) -> np.ndarray:
        row = np.zeros(self.ndof)
        lo, hi = self.indptr[i], self.indptr[i + 1]
        row[self.col_ind[lo:hi]] = self.coeffs[lo:hi]
        return row

    def matvec(self, x) -> np.ndarray:
        x = _host(x)
        out = np.empty(self.nconstraints)
        for i in range(self.nconstraints):
            lo, hi = self.indptr[i], self.indptr[i + 1]
            out[i] = self.coeffs[lo:hi] @ x[self.col_ind[lo:hi]]
        return out

    def rmatvec(self, lam) -> np.ndarray:
        lam = _host(lam)
        out = np.zeros(self.ndof)
        for i in range(self.nconstraints):
            lo, hi = self.indptr[i], self.indptr[i + 1]
            out[self.col_ind[lo:hi]] += lam[i] * self.coeffs[lo:hi]
        return out

    def device(self):
        """(indptr int64, col_ind int32, coeffs f64, violation f64, unilateral u8) on the device."""
        t = _lib.torch()

        def up(a, dt):  # at least one element, so every pointer is valid
            a = np.asarray(a, dtype=dt)
            return t.from_numpy(np.ascontiguousarray(a if len(a) else np.zeros(1, dtype=dt))).cuda()

        unilateral = np.array([kind == UNILATERAL for kind in self.types], dtype=np.uint8)
        return (up(self.indptr, np.int64), up(self.col_ind, np.int32), up(self.coeffs, np.float64),
                up(self.violation, np.float64), up(unilateral, np.uint8))


def _host(a):
    return a.detach().cpu().numpy() if _lib.is_tensor(a) else np.asarray(a)


def _dev(a, dtype=None):
    t = _lib.torch()
    dtype = dtype or t.float64
    if _lib.is_tensor(a):
        return a.to(device="cuda", dtype=dtype).contiguous()
    return _lib.to_device(np.asarray(a)).to(dtype=dtype)


def _check(st, what):
    _lib.check(st, what)


def _plane_scan(positions, plane_z, with_nodes=True):
    t = _lib.require_cuda()
    pos = _dev(positions).reshape(-1)
    n_nodes = pos.numel() // 3
    nodes = t.empty(max(n_nodes, 1), dtype=t.int32, device="cuda") if with_nodes else None
    pen = t.empty(max(n_nodes, 1), dtype=t.float64, device="cuda") if with_nodes else None
    out = t.zeros(2, dtype=t.float64, device="cuda")
    cnt = t.zeros(1, dtype=t.int64, device="cuda")
    _check(_lib.load().tsb_plane_contacts(n_nodes, _lib.ptr(pos), float(plane_z), _lib.ptr(nodes), _lib.ptr(pen),
                                          _lib.ptr(cnt), _lib.ptr(out), _lib.stream_ptr()), "plane_contacts")
    return nodes, pen, cnt, out


def detect_plane_contacts(positions, plane_z: float) -> ConstraintSet:
    """Unilateral contacts for nodes below z = plane_z (contact.py:89-106), on the device."""
    nodes, pen, cnt, _ = _plane_scan(positions, plane_z)
    m = int(cnt.item())
    nd = nodes[:m].cpu().numpy().astype(np.int64)
    n_nodes = (positions.numel() if _lib.is_tensor(positions) else np.asarray(positions).size) // 3
    return ConstraintSet(ndof=3 * n_nodes, indptr=np.arange(m + 1, dtype=np.int64), col_ind=3 * nd + 2,
                         coeffs=np.full(m, -1.0), violation=pen[:m].cpu().numpy(), types=[UNILATERAL] * m)


def _compliance_from_columns(constraints, s_cols, scale=1.0):
    t = _lib.torch()
    m, n = constraints.nconstraints, constraints.ndof
    ip, ci, co, _, _ = constraints.device()
    W = t.empty((m, m), dtype=t.float64, device="cuda")
    _check(_lib.load().tsb_compliance_from_columns(m, n, _lib.ptr(ip), _lib.ptr(ci), _lib.ptr(co), _lib.ptr(s_cols),
                                                   float(scale), _lib.ptr(W), _lib.stream_ptr()), "compliance")
    return W


def build_compliance(constraints: ConstraintSet, solve_fn):
    """W = J A^-1 J^T, one solve per constraint column (contact.py:109-125).
    `solve_fn(rhs)` receives the dense column J^T e_i (NumPy, as the reference
    passes it); returns (W, S) as NumPy arrays, W symmetrised by averaging."""
    m, n = constraints.nconstraints, constraints.ndof
    if m == 0:
        return np.empty((0, 0)), np.empty((n, 0))
    t = _lib.require_cuda()
    S = t.empty((m, n), dtype=t.float64, device="cuda")  # column i = row i (column-major n x m)
    for i in range(m):
        S[i] = _dev(solve_fn(constraints.row_dense(i)))
    W = _compliance_from_columns(constraints, S)
    return W.cpu().numpy(), S.t().cpu().numpy()


def _pgs_device(W, rhs, unilateral, tol, max_sweeps):
    t = _lib.torch()
    m = len(rhs) if not _lib.is_tensor(rhs) else rhs.numel()
    lam = t.zeros(max(m, 1), dtype=t.float64, device="cuda")
    info = t.zeros(3, dtype=t.float64, device="cuda")
    if m:
        _check(_lib.load().tsb_pgs(m, _lib.ptr(W), _lib.ptr(rhs), _lib.ptr(unilateral), float(tol), int(max_sweeps),
                                   _lib.ptr(lam), _lib.ptr(info), _lib.stream_ptr()), "pgs")
    return lam[:m], info


def projected_gauss_seidel(w, rhs, types, tol: float = 1e-12, max_sweeps: int = 500) -> np.ndarray:
    """Solve W lambda = rhs with lambda >= 0 on unilateral rows (contact.py:128-166), on the device."""
    m = len(rhs)
    if m == 0:
        return np.zeros(0)
    t = _lib.require_cuda()
    uni = t.from_numpy(np.array([x == UNILATERAL for x in types], dtype=np.uint8)).cuda()
    lam, info = _pgs_device(_dev(w).contiguous(), _dev(rhs), uni, tol, max_sweeps)
    if info[2].item():
        logger.warning("dropping %d constraint(s) with zero compliance diagonal", int(info[2].item()))
    return lam.cpu().numpy()


def _advance(acc, state, dt, fixed_nodes):
    """a[pinned] = 0, v' = v + h a, x' = x + h v', pinned keep (tsb_advance)."""
    t = _lib.torch()
    n = acc.numel()
    fixed = np.zeros(n, dtype=np.uint8)
    fixed[(3 * np.asarray(fixed_nodes, dtype=np.int64)[:, None] + np.arange(3)).ravel()] = 1
    fd = t.from_numpy(fixed).cuda()
    v0, x0 = _dev(state.velocities).reshape(-1), _dev(state.positions).reshape(-1)
    a1, v1, x1 = (t.empty(n, dtype=t.float64, device="cuda") for _ in range(3))
    flags = t.zeros(4, dtype=t.int32, device="cuda")
    _check(_lib.load().tsb_advance(n, _lib.ptr(acc), _lib.ptr(v0), _lib.ptr(x0), _lib.ptr(fd), float(dt),
                                   _lib.ptr(a1), _lib.ptr(v1), _lib.ptr(x1), _lib.ptr(flags), _lib.stream_ptr()),
           "advance")
    return a1, v1, x1


def _like(ref, dev):
    out = dev.reshape(-1, 3)
    return out if _lib.is_tensor(ref) else out.cpu().numpy()


def _corrected(free, state, acc_dev, dt, fixed_nodes):
    a1, v1, x1 = _advance(acc_dev, state, dt, fixed_nodes)
    return StepResult(
        positions=_like(state.positions, x1), velocities=_like(state.velocities, v1),
        accelerations=_like(free.accelerations, a1), f_int=free.f_int, f_ext=free.f_ext,
        matrix=free.matrix, rhs=free.rhs, report=free.report, pattern_rebuilt=free.pattern_rebuilt,
        assembly_time=free.assembly_time, solve_time=free.solve_time)


def correct_motion(free: StepResult, state: SimState, constraints: ConstraintSet, lam, s_cols, dt: float,
                   fixed_nodes) -> StepResult:
    """a_corr = a_free - S lambda and the kinematic update (contact.py:169-195)."""
    t = _lib.require_cuda()
    n = constraints.ndof
    lam_d = _dev(lam).reshape(-1)
    m = lam_d.numel()
    delta = t.zeros(n, dtype=t.float64, device="cuda")
    lib = _lib.load()
    if m:
        S = _dev(s_cols).reshape(n, m).t().contiguous()  # column-major n x m
        _check(lib.tsb_gemv_cols(n, m, _lib.ptr(S), _lib.ptr(lam_d), _lib.ptr(delta), _lib.stream_ptr()), "gemv")
    acc = t.empty(n, dtype=t.float64, device="cuda")
    _check(lib.tsb_contact_correct(n, _lib.ptr(_dev(free.accelerations).reshape(-1)), _lib.ptr(delta), None,
                                   _lib.ptr(acc), _lib.stream_ptr()), "correct")
    return _corrected(free, state, acc, dt, fixed_nodes)


@dataclass
class ContactStepInfo:
    result: StepResult
    ncontacts: int
    complementarity_residual: float
    max_penetration: float


def _factors_of(obj):
    from .ndprecond import AsyncPreconditioner, LdlFactors

    if isinstance(obj, LdlFactors):
        return obj
    if isinstance(obj, AsyncPreconditioner) and obj.factors is not None:
        return obj.factors
    return None


class PlaneContactPipeline:
    """Free motion / constraint resolution / motion correction per step (contact.py:204-257)."""

    def __init__(self, integrator: BackwardEulerIntegrator, plane_z: float):
        self.integrator = integrator
        self.plane_z = plane_z
        self.last = {}

    def step(self, state: SimState, solve, apply_inverse=None) -> ContactStepInfo:
        integ = self.integrator
        free = integ.compute_step(state, solve)
        constraints = detect_plane_contacts(free.positions, self.plane_z)
        m = constraints.nconstraints
        if m == 0:
            integ.commit(state, free)
            return ContactStepInfo(free, 0, 0.0, self._max_penetration(state))
        h = integ.config.dt
        factors = _factors_of(apply_inverse)
        if factors is not None:
            lam, info, acc = self._resolve_with_factors(free, constraints, factors, h)
        else:
            from .ndprecond import AsyncPreconditioner

            if isinstance(apply_inverse, AsyncPreconditioner):
                # not ready yet: the reference falls back to solving each column (contact.py:109-125)
                apply_inverse = None
            if apply_inverse is None:
                def apply_inverse(rhs):
                    x, report = solve(free.matrix, rhs)
                    if not report.converged:
                        raise ContactError(f"compliance solve stalled at residual {report.final_residual:g}")
                    return x
            try:
                lam, info, acc = self._resolve_with_columns(free, constraints, apply_inverse, h)
            except ContactError:
                logger.warning("compliance solve failed; committing free motion", exc_info=True)
                integ.commit(state, free)
                return ContactStepInfo(free, m, float("nan"), self._max_penetration(state))
        if info[2].item():
            logger.warning("dropping %d constraint(s) with zero compliance diagonal", int(info[2].item()))
        corrected = _corrected(free, state, acc, h, integ.mesh.fixed_nodes)
        integ.commit(state, corrected)
        self.last = {"lam": lam, "sweeps": info[0]}
        return ContactStepInfo(corrected, m, float(info[1].item()), self._max_penetration(state))

    def _resolve_with_columns(self, free, cs, apply_inverse, h):
        """Reference path: one apply_inverse per column (contact.py:109-125)."""
        t = _lib.torch()
        m, n = cs.nconstraints, cs.ndof
        _, _, _, viol, uni = cs.device()
        S = t.empty((m, n), dtype=t.float64, device="cuda")
        for i in range(m):
            S[i] = _dev(apply_inverse(cs.row_dense(i))).reshape(-1)
        W = _compliance_from_columns(cs, S, scale=h * h)
        lam, info = _pgs_device(W, viol, uni, 1e-12, 500)
        lib = _lib.load()
        delta = t.empty(n, dtype=t.float64, device="cuda")
        _check(lib.tsb_gemv_cols(n, m, _lib.ptr(S), _lib.ptr(lam), _lib.ptr(delta), _lib.stream_ptr()), "gemv")
        acc = t.empty(n, dtype=t.float64, device="cuda")
        _check(lib.tsb_contact_correct(n, _lib.ptr(_dev(free.accelerations).reshape(-1)), _lib.ptr(delta), None,
                                       _lib.ptr(acc), _lib.stream_ptr()), "correct")
        return lam, info, acc

    def _resolve_with_factors(self, free, cs, factors, h):
        """W = Y^T D^-1 Y with Y = L^-1 P J^T; S lambda = P^T L^-T D^-1 (Y lambda)."""
        t = _lib.torch()
        dev = factors.device()
        m, n = cs.nconstraints, cs.ndof
        ip, ci, co, viol, uni = cs.device()
        iperm = getattr(factors, "_iperm_dev", None)
        if iperm is None:
            iperm = t.from_numpy(np.argsort(np.asarray(factors.plan.perm)).astype(np.int32)).cuda()
            factors._iperm_dev = iperm
        lib = _lib.load()
        sp = _lib.stream_ptr()
        R = t.empty((m, n), dtype=t.float64, device="cuda")
        _check(lib.tsb_contact_rhs(m, _lib.ptr(ip), _lib.ptr(ci), _lib.ptr(co), _lib.ptr(iperm), n, _lib.ptr(R), sp),
               "contact_rhs")
        Y = t.empty((m, n), dtype=t.float64, device="cuda")
        dev.lower_multi(R, Y)  # multi-RHS lower sweeps (permuted order)
        W = t.empty((m, m), dtype=t.float64, device="cuda")
        part = t.empty(max(int(lib.tsb_gram_scratch(n, m)), 1), dtype=t.float64, device="cuda")
        _check(lib.tsb_gram(n, m, _lib.ptr(Y), _lib.ptr(dev.t["d"]), float(h * h), _lib.ptr(part), _lib.ptr(W), sp),
               "gram")
        lam, info = _pgs_device(W, viol, uni, 1e-12, 500)
        u = t.empty(n, dtype=t.float64, device="cuda")
        _check(lib.tsb_gemv_cols(n, m, _lib.ptr(Y), _lib.ptr(lam), _lib.ptr(u), sp), "gemv")
        z = t.empty(n, dtype=t.float64, device="cuda")
        dev.run("upper_scaled", u, z)
        acc = t.empty(n, dtype=t.float64, device="cuda")
        _check(lib.tsb_contact_correct(n, _lib.ptr(_dev(free.accelerations).reshape(-1)), _lib.ptr(z),
                                       _lib.ptr(iperm), _lib.ptr(acc), sp), "correct")
        self.last_w = W
        return lam, info, acc

    def _max_penetration(self, state: SimState) -> float:
        _, _, _, out = _plane_scan(state.positions, self.plane_z, with_nodes=False)
        return float(out[0].item())
