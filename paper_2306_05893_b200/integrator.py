"""Backward-Euler step on the B200 (drop-in for tetsim.integrator, integrator.py:1-236).

`assemble_system` is one fused device pass (element kernel -> CSR block
gather -> nodal gather + rhs) into a fixed pattern built once from the mesh
topology; `compute_step` keeps A, b, the solve and the kinematic update on
the device.  States may hold NumPy arrays (host buffers: uploaded at the
start of the step, results downloaded at the end -- the reference-facing
path) or CUDA tensors (fully device-resident).

System: A = (1 + h alpha) M + h (h + beta) K,
        b = f_ext - f(x_t) - (h + beta) K v_t - alpha M v_t,  pinned rows identity / zero.
"""

from __future__ import annotations

import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._plan import AssemblyPlan, device_topology_pattern
from .assembly import CsrMatrix, build_pattern, TripletStream
from .krylov import SolveReport
from .mesh import Mesh
from .models import lumped_mass

__all__ = [
    "IntegratorError",
    "StepError",
    "IntegratorConfig",
    "SimState",
    "StepResult",
    "BackwardEulerIntegrator",
]


class IntegratorError(ValueError):
    pass


class StepError(RuntimeError):
    """Linear solve failed during a step; carries the solver report."""

    def __init__(self, message: str, report: SolveReport):
        super().__init__(message)
        self.report = report


@dataclass
class IntegratorConfig:
    dt: float
    rayleigh_mass: float = 0.0
    rayleigh_stiffness: float = 0.0
    gravity: tuple = (0.0, 0.0, -9.81)
    newton_iterations: int = 1

    def __post_init__(self):
        if not self.dt > 0:
            raise IntegratorError(f"dt must be positive, got {self.dt}")
        if self.rayleigh_mass < 0 or self.rayleigh_stiffness < 0:
            raise IntegratorError("Rayleigh coefficients must be non-negative")
        if self.newton_iterations < 1:
            raise IntegratorError("newton_iterations must be >= 1")


def _copy(a):
    return a.clone() if _lib.is_tensor(a) else a.copy()


@dataclass
class SimState:
    """Nodal kinematics (NumPy arrays or CUDA tensors) plus last step's forces."""

    positions: object      # (n, 3)
    velocities: object     # (n, 3)
    accelerations: object  # (n, 3)
    f_int: object          # (3n,)
    f_ext: object          # (3n,)
    time: float = 0.0

    @classmethod
    def rest(cls, mesh: Mesh, device: bool = False) -> "SimState":
        n = mesh.node_count
        st = cls(mesh.nodes.copy(), np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(3 * n), np.zeros(3 * n))
        return st.to_device() if device else st

    @property
    def on_device(self) -> bool:
        return _lib.is_tensor(self.positions)

    def to_device(self) -> "SimState":
        t = _lib.require_cuda()
        cv = lambda a: t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()  # noqa: E731
        if self.on_device:
            return self
        return SimState(cv(self.positions), cv(self.velocities), cv(self.accelerations),
                        cv(self.f_int), cv(self.f_ext), self.time)

    def to_host(self) -> "SimState":
        if not self.on_device:
            return self
        cv = lambda a: a.detach().cpu().numpy()  # noqa: E731
        return SimState(cv(self.positions), cv(self.velocities), cv(self.accelerations),
                        cv(self.f_int), cv(self.f_ext), self.time)

    def copy(self) -> "SimState":
        return SimState(_copy(self.positions), _copy(self.velocities), _copy(self.accelerations),
                        _copy(self.f_int), _copy(self.f_ext), self.time)


@dataclass
class StepResult:
    positions: object
    velocities: object
    accelerations: object
    f_int: object
    f_ext: object
    matrix: CsrMatrix
    rhs: object
    report: SolveReport
    pattern_rebuilt: bool
    assembly_time: float
    solve_time: float


class _DeviceAssembler:
    """Pattern owner of the device path (stands in for MatrixAssembler on the
    integrator: `pattern_rebuilds`, `force_rebuild`, lazily a `mapping`)."""

    def __init__(self, mesh: Mesh):
        self.mesh = mesh
        self.n = mesh.ndof
        self.fixed_dofs = mesh.fixed_dofs()
        self.pattern = None
        self.pattern_rebuilds = 0
        self.force_rebuild = False
        self._mapping = None

    def ensure(self) -> bool:
        if self.pattern is None or self.force_rebuild:
            self.pattern = device_topology_pattern(self.mesh)  # csrc/pattern.cu
            self.pattern_rebuilds += 1
            self._mapping = None
            return True
        return False

    @property
    def mapping(self):
        """Reference CompressionMapping of the fused mass+stiffness stream (built on demand)."""
        if self._mapping is None and self.pattern is not None:
            el = self.mesh.elements
            gdof = (3 * el[:, :, None] + np.arange(3)).reshape(len(el), 12)
            st = TripletStream()
            st.begin_pass()
            st.add_block(gdof.ravel(), gdof.ravel(), np.zeros(gdof.size))
            st.add_block(np.repeat(gdof, 12, axis=1).ravel(), np.tile(gdof, (1, 12)).ravel(),
                         np.zeros(144 * len(el)))
            st.end_pass()
            _, self._mapping = build_pattern(st, self.n, self.fixed_dofs)
        return self._mapping


class BackwardEulerIntegrator:
    """Owns the device plan (mesh layout, pattern, gather lists) and the mass data."""

    def __init__(self, mesh: Mesh, model, config: IntegratorConfig, workers: int = 1):
        self.mesh = mesh
        self.model = model
        self.config = config
        self.workers = workers
        self.fixed_dofs = mesh.fixed_dofs()
        self.assembler = _DeviceAssembler(mesh)
        self.mass_diag = lumped_mass(mesh, model.params)
        share = model.params.density * mesh.signed_volumes() / 4.0
        self._mass_share = share
        self._gravity_force = (self.mass_diag.reshape(-1, 3) * np.asarray(config.gravity)).ravel()
        self._plan: AssemblyPlan | None = None
        self._law = getattr(model, "law", "corotational")

    @property
    def _mass_vals(self) -> np.ndarray:
        return np.repeat(self._mass_share, 12)

    def _coefficients(self):
        h = self.config.dt
        return 1.0 + h * self.config.rayleigh_mass, h * (h + self.config.rayleigh_stiffness)

    def _ensure_plan(self) -> bool:
        rebuilt = self.assembler.ensure()
        if rebuilt or self._plan is None:
            self._plan = AssemblyPlan(
                self.model.precomp, pattern=self.assembler.pattern, mass_share=self._mass_share,
                mass_diag=self.mass_diag, gravity=self._gravity_force, fixed_dof=self.fixed_dofs,
                n_nodes=self.mesh.node_count,
            )
        return rebuilt

    # -- device core ------------------------------------------------------
    def _assemble_device(self, x, v, f_ext_state, outs=None):
        """Enqueue the fused assembly; returns (A, b, f_int, f_ext, rebuilt) as device objects
        (`outs` = preallocated (b, f_int, f_ext) device views, else fresh tensors)."""
        t = _lib.torch()
        rebuilt = self._ensure_plan()
        plan = self._plan
        pat = self.assembler.pattern
        n = self.mesh.ndof
        cfg = self.config
        key = (cfg.dt, cfg.rayleigh_stiffness, cfg.rayleigh_mass, self._law)
        co = self._co.get(key) if hasattr(self, "_co") else None
        if co is None:  # per-step coefficients (integrator.py:135-143), built once per config
            cm, ck = self._coefficients()
            co = plan.coeffs(h=cfg.dt, beta=cfg.rayleigh_stiffness, alpha=cfg.rayleigh_mass, cm=cm, ck=ck,
                             law=self._law, want_matrix=True)
            self._co = {key: co}
        nnz = len(pat["col_ind"])
        buf = t.empty(nnz + (n if outs is not None else 4 * n), dtype=t.float64, device="cuda")  # one allocation
        values, kv = buf[:nnz], buf[nnz:nnz + n]
        if outs is not None:
            b, f_int, f_ext = outs
        else:
            b, f_int, f_ext = buf[nnz + n:nnz + 2 * n], buf[nnz + 2 * n:nnz + 3 * n], buf[nnz + 3 * n:]
        plan.run(co, x, v, f_ext_state, values, b, f_int, kv, f_ext)  # zeroes the status words first
        a = CsrMatrix(n, n, pat["row_ptr"], pat["col_ind"], values)
        return a, b, f_int, f_ext, rebuilt

    @staticmethod
    def _flat_dev(a):
        t = _lib.torch()
        if _lib.is_tensor(a):
            return a.reshape(-1).to(dtype=t.float64).contiguous()
        return t.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))).cuda()

    def _raise_model_flags(self, flags):
        from .models import ModelError

        if int(flags[0]):
            raise ModelError("non-finite positions")

    # -- reference API ----------------------------------------------------
    def assemble_system(self, state: SimState):
        """One fused mass-and-stiffness pass on the device; returns (A, b, info)."""
        t0 = time.perf_counter()
        host = not state.on_device
        x = self._flat_dev(state.positions)
        v = self._flat_dev(state.velocities)
        fe = self._flat_dev(state.f_ext)
        a, b, f_int, f_ext, rebuilt = self._assemble_device(x, v, fe)
        flags = self._plan.flags.cpu()
        self._raise_model_flags(flags)
        if host:
            b, f_int, f_ext = b.cpu().numpy(), f_int.cpu().numpy(), f_ext.cpu().numpy()
        info = {"pattern_rebuilt": rebuilt, "assembly_time": time.perf_counter() - t0,
                "f_int": f_int, "f_ext": f_ext}
        return a, b, info

    def compute_step(self, state: SimState, solve) -> StepResult:
        """One implicit step without committing it (integrator.py:171-221).

        `solve(A, b) -> (x, SolveReport)`.  Solvers marked `accepts_device`
        receive b as a CUDA tensor; others get a NumPy array as in the reference.
        """
        t = _lib.torch()
        cfg = self.config
        h = cfg.dt
        host = not state.on_device
        n = self.mesh.ndof
        stage = None
        if host:  # H2D of (x, v, f_ext) into one device buffer, one D2H of the six results
            stage = self._host_stage(n)
            d_in = stage["d_in"]
            for k, arr in enumerate((state.positions, state.velocities, state.f_ext)):
                # results of an earlier step are views of pinned memory: straight DMA; user arrays stage
                a_ = np.ascontiguousarray(np.asarray(arr, dtype=np.float64)).reshape(-1)
                src = t.from_numpy(a_ if a_.flags.writeable else a_.copy())
                d_in[k * n:(k + 1) * n].copy_(src, non_blocking=True)
            x0, v0, fe_state = d_in[:n], d_in[n:2 * n], d_in[2 * n:]
        else:
            x0 = self._flat_dev(state.positions)
            v0 = self._flat_dev(state.velocities)
            fe_state = self._flat_dev(state.f_ext)
        dev_solve = bool(getattr(solve, "accepts_device", False))
        ev = getattr(self, "_ev", None)
        if ev is None:
            ev = self._ev = [t.cuda.Event(enable_timing=True) for _ in range(3)]
        ent = self._out_buffer(n) if host else None
        try:
            return self._step_body(state, solve, host, n, h, stage, ent, x0, v0, fe_state, dev_solve, ev)
        except BaseException:
            if ent is not None:
                _release_buffer(ent)  # no result views were handed out
            raise

    def _step_body(self, state, solve, host, n, h, stage, ent, x0, v0, fe_state, dev_solve, ev):
        t = _lib.torch()
        cfg = self.config
        assembly_time = solve_time = 0.0
        rebuilt_any = False
        x_tr, v_tr = x0, v0
        fixed = self._plan.fixed_dof if self._plan is not None else None
        side = None
        for it_newton in range(cfg.newton_iterations):
            ev[0].record()
            d_out = stage["d_out"] if host else None
            a, b, f_int, f_ext, rebuilt = self._assemble_device(
                x_tr, v_tr, fe_state, None if d_out is None else (d_out[3 * n:4 * n], d_out[4 * n:5 * n],
                                                                  d_out[5 * n:]))
            fixed = self._plan.fixed_dof
            ev[1].record()
            if host and it_newton == cfg.newton_iterations - 1:
                # b, f_int, f_ext are final: their D2H runs on a side stream under the solve
                side = self._d2h_stream()
                side.wait_event(ev[1])
                with t.cuda.stream(side):
                    ent[0][3 * n:].copy_(d_out[3 * n:], non_blocking=True)
            rebuilt_any = rebuilt_any or rebuilt
            accel, report = solve(a, b if dev_solve else b.cpu().numpy())
            ev[2].record()
            d_acc = self._flat_dev(accel)
            if host:  # results land in the staging buffer: [x1 | v1 | acc | b | f_int | f_ext]
                x1, v1, acc = (d_out[k * n:(k + 1) * n] for k in range(3))
                if d_acc.data_ptr() == acc.data_ptr():
                    d_acc = d_acc.clone()
            else:
                acc = t.empty(n, dtype=t.float64, device="cuda")
                v1 = t.empty(n, dtype=t.float64, device="cuda")
                x1 = t.empty(n, dtype=t.float64, device="cuda")
            P = _lib.ptr
            _lib.check(_lib.load().tsb_advance(n, P(d_acc), P(v0), P(x0), P(fixed), h, P(acc), P(v1),
                                               P(x1), P(self._plan.flags), _lib.stream_ptr()), "advance")
            if host and it_newton == cfg.newton_iterations - 1:  # x1, v1, acc with the same wait
                ent[0][:3 * n].copy_(d_out[:3 * n], non_blocking=True)
                t.cuda.current_stream().wait_stream(side)
            flags = self._plan.flags.cpu()  # one readback: model + accel flags (and the results' D2H)
            ev[2].synchronize()
            assembly_time += ev[0].elapsed_time(ev[1]) * 1e-3
            solve_time += ev[1].elapsed_time(ev[2]) * 1e-3
            self._raise_model_flags(flags)
            if not report.converged:
                raise StepError(
                    f"linear solve did not converge: residual {report.final_residual:g} "
                    f"after {report.iterations} iterations", report)
            if int(flags[1]):
                raise StepError("solver produced non-finite accelerations", report)
            x_tr, v_tr = x1, v1
        if host:
            o = ent[0].numpy()  # the six results are views of this pinned buffer, which is
            weakref.finalize(o, _release_buffer, ent)  # reused only once every view is gone
            part = lambda k: o[k * n:(k + 1) * n]  # noqa: E731
            pos, vel, acc_o = part(0).reshape(-1, 3), part(1).reshape(-1, 3), part(2).reshape(-1, 3)
            rhs, f_int_o, f_ext_o = part(3), part(4), part(5)
        else:
            pos, vel, acc_o = x_tr.view(-1, 3), v_tr.view(-1, 3), acc.view(-1, 3)
            f_int_o, f_ext_o, rhs = f_int, f_ext, b
        return StepResult(pos, vel, acc_o, f_int_o, f_ext_o, a, rhs, report, rebuilt_any,
                          assembly_time, solve_time)

    def capture(self, state: SimState, solve) -> "CapturedStep":
        """The device step (assembly + device PCG + kinematic update) of
        `state`'s shape captured once as a CUDA graph; see CapturedStep."""
        return CapturedStep(self, state, solve)

    def _host_stage(self, n):
        """Device staging of a host-state step (allocated once)."""
        st = getattr(self, "_stage", None)
        if st is None or st["n"] != n:
            t = _lib.torch()
            st = {"n": n,
                  "d_in": t.empty(3 * n, dtype=t.float64, device="cuda"),
                  "d_out": t.empty(6 * n, dtype=t.float64, device="cuda")}
            self._stage = st
            self._out_pool = []
        return st

    def _d2h_stream(self):
        st = getattr(self, "_side", None)
        if st is None:
            st = self._side = _lib.torch().cuda.Stream()
        return st

    def _out_buffer(self, n):
        """A pinned [6n] result buffer none of whose earlier results is still referenced."""
        for ent in self._out_pool:
            if ent[1]:
                ent[1] = False
                return ent
        t = _lib.torch()
        ent = [t.empty(6 * n, dtype=t.float64).pin_memory(), False]
        self._out_pool.append(ent)
        return ent

    def commit(self, state: SimState, result: StepResult):
        state.positions = result.positions
        state.velocities = result.velocities
        state.accelerations = result.accelerations
        state.f_int = result.f_int
        state.time += self.config.dt

    def step(self, state: SimState, solve) -> StepResult:
        result = self.compute_step(state, solve)
        self.commit(state, result)
        return result


def _release_buffer(ent):
    ent[1] = True


class CapturedStep:
    """compute_step as ONE CUDA graph: the fused assembly, the persistent PCG
    kernel (cooperative launch captured as a kernel node) and the kinematic
    update replay without any host work between them.

    `replay(state)` copies the state into the graph's static inputs, replays,
    reads the status words once and returns a StepResult whose tensors are the
    graph's static outputs -- valid until the next replay (clone to keep).
    The solver must be a device solver (`accepts_device`) whose preconditioner
    does not change between replays (same factor image / Jacobi of the step's
    own matrix).  Same kernels, same arithmetic as compute_step: results are
    bit-identical to it."""

    def __init__(self, integ: BackwardEulerIntegrator, state: SimState, solve):
        t = _lib.require_cuda()
        if not state.on_device:
            raise IntegratorError("CapturedStep needs a device-resident SimState")
        if not getattr(solve, "accepts_device", False):
            raise IntegratorError("CapturedStep needs a device solver (accepts_device)")
        self.integ, self.solve = integ, solve
        n = integ.mesh.ndof
        self.n = n
        self.x0, self.v0, self.fe = (t.empty(n, dtype=t.float64, device="cuda") for _ in range(3))
        self._load(state)
        integ.compute_step(state, solve)   # warm: plan, pattern, handles, launch grids
        from .krylov import _handle

        self._pcg = _handle(n)
        if self._pcg.pending is not None:
            self._pcg.pending._get()
            self._pcg.pending = None
        side = t.cuda.Stream()
        side.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(side):  # one eager pass on the capture stream (allocator warm-up)
            self._body()
            self._pcg.pending = None
        t.cuda.current_stream().wait_stream(side)
        t.cuda.synchronize()
        self.graph = t.cuda.CUDAGraph()
        l0 = _lib.launch_count()
        with t.cuda.graph(self.graph):
            self.outs = self._body()
        self.kernels = _lib.launch_count() - l0  # libtsb kernels in one replay
        self._pcg.pending = None

    def _load(self, state):
        self.x0.copy_(state.positions.reshape(-1))
        self.v0.copy_(state.velocities.reshape(-1))
        self.fe.copy_(state.f_ext.reshape(-1))

    def _body(self):
        integ, n = self.integ, self.n
        t = _lib.torch()
        a, b, f_int, f_ext, _ = integ._assemble_device(self.x0, self.v0, self.fe)
        accel, _ = self.solve(a, b)
        acc, v1, x1 = (t.empty(n, dtype=t.float64, device="cuda") for _ in range(3))
        P = _lib.ptr
        _lib.check(_lib.load().tsb_advance(n, P(accel), P(self.v0), P(self.x0), P(integ._plan.fixed_dof),
                                           integ.config.dt, P(acc), P(v1), P(x1), P(integ._plan.flags),
                                           _lib.stream_ptr()), "advance")
        return a, b, f_int, f_ext, acc, v1, x1

    def replay(self, state: SimState) -> StepResult:
        from .krylov import _DeviceReport

        t0 = time.perf_counter()
        self._load(state)
        self.graph.replay()
        a, b, f_int, f_ext, acc, v1, x1 = self.outs
        report = _DeviceReport(self._pcg, t0)
        flags = self.integ._plan.flags.cpu()
        self.integ._raise_model_flags(flags)
        if not report.converged:
            raise StepError(f"linear solve did not converge: residual {report.final_residual:g} "
                            f"after {report.iterations} iterations", report)
        if int(flags[1]):
            raise StepError("solver produced non-finite accelerations", report)
        # a fresh CsrMatrix per replay: a host snapshot cached by an earlier result's
        # `.values` must not be served for this replay's device values
        a = CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_ind, a.device_values())
        return StepResult(x1.view(-1, 3), v1.view(-1, 3), acc.view(-1, 3), f_int, f_ext, a, b, report, False,
                          0.0, time.perf_counter() - t0)
