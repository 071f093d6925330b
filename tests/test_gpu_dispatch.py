"""GPU parity of the reference caller's solver dispatch:
ScenarioRunner.solve (cli.py:334-343) with the _FactorPreconditioner adapter
(cli.py:290-298), restated here over the drop-in API exactly as the
reference writes it -- CG, PCG-LDL^T once the AsyncPreconditioner is READY,
and the PCG-Jacobi cold start before that.  Every solve must launch device
kernels and reproduce the oracle: same iteration count, x within 1e-10."""

import numpy as np
import pytest

from conftest import clamped_beam
from oracle import tetsim_oracle as O

pytestmark = pytest.mark.gpu

from paper_2306_05893_b200 import _lib, krylov, mesh as M, models, ndprecond as ND  # noqa: E402
from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState  # noqa: E402
from paper_2306_05893_b200.krylov import SolveMode, SolverConfig  # noqa: E402


class _FactorPreconditioner:
    """The reference's adapter (cli.py:290-298), verbatim in behaviour."""

    def __init__(self, factors, workers=1):
        self.factors = factors
        self.workers = workers

    def apply(self, r):
        return self.factors.apply(r, workers=self.workers)


class Runner:
    """ScenarioRunner's solve dispatch and step loop (cli.py:334-366)."""

    def __init__(self, dims, mode):
        self.mesh = clamped_beam(*dims)
        params = models.MaterialParams(1e5, 0.3, 1000.0)
        self.integrator = BackwardEulerIntegrator(self.mesh, models.make_model("corotational", self.mesh, params),
                                                  IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
        self.solver_config = SolverConfig(1e-9, 8000, mode)
        self.precond = None
        if mode is SolveMode.PCG_LDLT:
            plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(self.mesh), 16))
            self.precond = ND.AsyncPreconditioner(plan, refactor_every=1)
        self.state = SimState.rest(self.mesh)
        self.log = []
        self.step_index = 0

    def solve(self, a, b):
        scfg = self.solver_config
        launches = _lib.launch_count()
        if scfg.mode is SolveMode.CG:
            kind, out = "cg", krylov.cg(a, b, scfg)
        elif scfg.mode is SolveMode.PCG_LDLT and self.precond is not None \
                and self.precond.status is ND.PrecondStatus.READY:
            pre = _FactorPreconditioner(self.precond.factors)
            kind, out = ("ldlt", pre.factors), krylov.pcg(a, b, pre, scfg)
        else:
            kind, out = "jacobi", krylov.pcg(a, b, krylov.jacobi_precond(a), scfg)
        x, rep = out
        self.log.append((kind, a.row_ptr, a.col_ind, np.array(a.values), np.array(b), np.array(x),
                         rep.iterations, rep.final_residual, _lib.launch_count() - launches))
        return x, rep

    def run_step(self):
        self.step_index += 1
        if self.precond is not None:
            self.precond.poll()
        result = self.integrator.step(self.state, self.solve)
        if self.precond is not None:
            self.precond.update(result.matrix, self.step_index)
            self.precond.wait_ready()  # deterministic replay: publish before the next step
        return result


def _check(entry):
    kind, rp, ci, vals, b, x, it, res, launches = entry
    assert launches > 0, "solve ran without device kernels"
    if kind == "cg":
        pre = None
    elif kind == "jacobi":
        inv = O.jacobi_inv_diag(rp, ci, vals, len(b))
        pre = lambda r: r * inv  # noqa: E731
    else:
        f = kind[1]
        pre = lambda r: O.apply(f, r)  # noqa: E731
    ox, oit, ores, oconv = O.pcg(rp, ci, vals, b, pre, 1e-9, 8000)
    assert oconv and it == oit, (kind if isinstance(kind, str) else "ldlt", it, oit)
    assert np.abs(x - ox).max() <= 1e-10 * np.abs(ox).max()
    assert abs(res - ores) <= 1e-10


@pytest.mark.parametrize("mode", [SolveMode.CG, SolveMode.PCG_JACOBI, SolveMode.PCG_LDLT])
def test_scenario_runner_dispatch(mode):
    run = Runner((4, 4, 12), mode)
    for _ in range(4):
        run.run_step()
    kinds = [e[0] if isinstance(e[0], str) else "ldlt" for e in run.log]
    if mode is SolveMode.CG:
        assert kinds == ["cg"] * 4
    elif mode is SolveMode.PCG_JACOBI:
        assert kinds == ["jacobi"] * 4
    else:  # cold start on Jacobi, then the published factors of the previous step
        assert kinds == ["jacobi", "ldlt", "ldlt", "ldlt"]
        assert all(e[6] <= 5 for e in run.log[1:])  # fresh-ish factors: few iterations (test_acceptance.py:198-224)
    for e in run.log:
        _check(e)
    if run.precond is not None:
        run.precond.close()
