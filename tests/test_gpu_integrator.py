"""The reference's integrator behaviour tests (tests/test_integrator.py:95-200)
restated on the device path: closed-form free fall, exact pinned DOFs,
pattern reuse, damping to equilibrium, large stiff steps, Newton iterations
(incl. the pinned host staging), StepError on non-convergence, compute_step
leaves the state untouched."""

import numpy as np
import pytest

from conftest import clamped_beam

pytestmark = pytest.mark.gpu

import paper_2306_05893_b200 as P  # noqa: E402
from paper_2306_05893_b200 import krylov  # noqa: E402
from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState, StepError  # noqa: E402


@pytest.fixture
def cg_solve():
    cfg = krylov.SolverConfig(tolerance=1e-10, max_iterations=5000, mode=krylov.SolveMode.CG)
    return lambda a, b: krylov.cg(a, b, cfg)


@pytest.fixture
def small_beam():
    return clamped_beam(3, 3, 8)


def make(mesh, params, law="corotational", **cfg):
    return BackwardEulerIntegrator(mesh, P.make_model(law, mesh, params), IntegratorConfig(**cfg))


def test_no_forces_no_motion(small_beam, params, cg_solve):
    integ = make(small_beam, params, dt=0.01, gravity=(0.0, 0.0, 0.0))
    st = SimState.rest(small_beam)
    integ.step(st, cg_solve)
    assert np.abs(st.positions - small_beam.nodes).max() < 1e-14 * np.abs(small_beam.nodes).max()
    assert np.abs(st.velocities).max() < 1e-12


def test_free_fall_closed_form(params, cg_solve):
    mesh = P.generate_beam(2, 2, 3, 0.5)
    integ = make(mesh, params, dt=0.01, gravity=(0.0, 0.0, -9.81))
    st = SimState.rest(mesh)
    for _ in range(10):
        integ.step(st, cg_solve)
    assert np.allclose(st.velocities[:, 2], -0.981, atol=1e-7)
    assert np.allclose(st.velocities[:, :2], 0.0, atol=1e-9)


def test_fixed_dofs_exactly_constant(small_beam, params, cg_solve):
    integ = make(small_beam, params, dt=0.01)
    st = SimState.rest(small_beam)
    fixed = small_beam.fixed_nodes
    before = st.positions[fixed].copy()
    for _ in range(5):
        integ.step(st, cg_solve)
        assert np.array_equal(st.positions[fixed], before)
        assert np.all(st.velocities[fixed] == 0.0) and np.all(st.accelerations[fixed] == 0.0)


def test_pattern_reused_after_first_step(small_beam, params, cg_solve):
    integ = make(small_beam, params, dt=0.01)
    st = SimState.rest(small_beam)
    flags = [integ.step(st, cg_solve).pattern_rebuilt for _ in range(6)]
    assert flags == [True, False, False, False, False, False]
    assert integ.assembler.pattern_rebuilds == 1


def test_settles_toward_equilibrium(small_beam, params, cg_solve):
    integ = make(small_beam, params, dt=0.01, rayleigh_mass=0.5, rayleigh_stiffness=0.005)
    st = SimState.rest(small_beam)
    speeds, residuals = [], []
    for _ in range(200):
        res = integ.step(st, cg_solve)
        speeds.append(np.abs(st.velocities).max())
        residuals.append(np.linalg.norm(res.rhs))
    assert max(speeds) < 10.0
    assert np.median(speeds[-30:]) < 0.25 * max(speeds)
    assert np.median(residuals[-30:]) < 0.25 * max(residuals)


def test_stiff_large_step_stable(params, cg_solve):
    stiff = type(params)(young_modulus=1e6, poisson_ratio=0.3, density=1000.0)
    mesh = clamped_beam(2, 2, 5)
    integ = make(mesh, stiff, dt=0.04)
    st = SimState.rest(mesh)
    for _ in range(60):
        integ.step(st, cg_solve)
        assert np.abs(st.velocities).max() < 50.0


@pytest.mark.parametrize("device", [False, True])
def test_newton_iterations_config(small_beam, params, cg_solve, device):
    integ = make(small_beam, params, law="stvk", dt=0.01, newton_iterations=3)
    st = SimState.rest(small_beam, device=device)
    res = integ.step(st, cg_solve)
    pos = res.positions.cpu().numpy() if device else res.positions
    assert np.all(np.isfinite(pos))
    one = make(small_beam, params, law="stvk", dt=0.01, newton_iterations=1)
    r1 = one.step(SimState.rest(small_beam), cg_solve)
    assert np.abs(pos - r1.positions).max() < 1e-3  # a few Newton updates of the same step


def test_nonconvergence_raises_step_error(small_beam, params):
    integ = make(small_beam, params, dt=0.01)
    st = SimState.rest(small_beam)
    strict = krylov.SolverConfig(tolerance=1e-15, max_iterations=1, mode=krylov.SolveMode.CG)
    with pytest.raises(StepError) as err:
        integ.step(st, lambda a, b: krylov.cg(a, b, strict))
    assert err.value.report.iterations == 1


def test_compute_step_does_not_mutate_state(small_beam, params, cg_solve):
    integ = make(small_beam, params, dt=0.01)
    st = SimState.rest(small_beam)
    before = st.positions.copy()
    integ.compute_step(st, cg_solve)
    assert np.array_equal(st.positions, before) and st.time == 0.0


def test_host_results_survive_later_steps(small_beam, params, cg_solve):
    """Host results are views of pooled pinned buffers: a result kept by the
    caller is never overwritten by a later step."""
    integ = make(small_beam, params, dt=0.01)
    st = SimState.rest(small_beam)
    kept = integ.compute_step(st, cg_solve)
    snap = kept.positions.copy(), kept.velocities.copy(), kept.rhs.copy()
    for _ in range(4):
        integ.step(st, cg_solve)
    assert np.array_equal(kept.positions, snap[0]) and np.array_equal(kept.velocities, snap[1])
    assert np.array_equal(kept.rhs, snap[2])
