"""GPU parity: SpMV, merge, assembly, integrator step (device path vs oracle/golden)."""

import numpy as np
import pytest

from conftest import clamped_beam
from oracle import tetsim_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2306_05893_b200")
from paper_2306_05893_b200 import krylov, models  # noqa: E402
from paper_2306_05893_b200.assembly import CsrMatrix, TripletStream, build_pattern, compress  # noqa: E402
from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState  # noqa: E402


def rel(a, b):
    b = np.asarray(b)
    d = np.abs(np.asarray(a) - b).max() if b.size else 0.0
    s = np.abs(b).max() if b.size else 1.0
    return d / (s if s else 1.0)


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_spmv_bit_exact_vs_reference(golden, name):
    g = golden(name)
    a = CsrMatrix(len(g["row_ptr"]) - 1, len(g["row_ptr"]) - 1, g["row_ptr"], g["col_ind"], g["values"])
    y = krylov.spmv(a, g["spmv_x"])
    assert np.array_equal(y, g["spmv_y"])


def test_spmv_ragged_long_and_empty_rows(rng):
    # rows of length 0, 1, 7, 8, 9, 129, 300 (pairwise recursion) and a non-square shape
    lens = [0, 1, 7, 8, 9, 16, 17, 129, 130, 300, 0, 45]
    ncols = 400
    row_ptr = np.concatenate([[0], np.cumsum(lens)])
    col_ind = np.concatenate([np.sort(rng.choice(ncols, k, replace=False)) for k in lens])
    vals = rng.standard_normal(len(col_ind)) * 10.0 ** rng.integers(-8, 8, len(col_ind))
    x = rng.standard_normal(ncols)
    a = CsrMatrix(len(lens), ncols, row_ptr, col_ind, vals)
    assert np.array_equal(krylov.spmv(a, x), O.spmv(row_ptr, col_ind, vals, x))


def test_spmv_dimension_mismatch():
    a = CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 1.0]))
    with pytest.raises(krylov.SolverError):
        krylov.spmv(a, np.ones(3))


def test_compress_bit_exact(golden):
    g = golden("beam_small")
    s = TripletStream()
    s.begin_pass()
    s.add_block(g["trip_rows"], g["trip_cols"], g["trip_vals"])
    s.end_pass()
    fixed = (3 * g["fixed_nodes"][:, None] + np.arange(3)).ravel()
    _, mp = build_pattern(s, 3 * len(g["nodes"]), fixed)
    a = compress(s, mp, g["coeffs"])
    assert a.on_device
    assert np.array_equal(a.values, g["values"])
    b = compress(s, mp)
    ref = O.compress(g["trip_vals"], g["kept"], g["kept_slots"], len(g["col_ind"]), g["fixed_diag_slots"])
    assert np.array_equal(b.values, ref)


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_assemble_system_vs_reference(golden, params, name):
    g = golden(name)
    mesh = clamped_beam(*map(int, g["dims"]))
    model = models.make_model("corotational", mesh, params)
    integ = BackwardEulerIntegrator(mesh, model, IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    st = SimState(g["positions"], g["velocities"], np.zeros_like(g["positions"]), np.zeros(len(g["b"])),
                  g["f_ext_state"])
    a, b, info = integ.assemble_system(st)
    assert info["pattern_rebuilt"] and integ.assembler.pattern_rebuilds == 1
    assert np.array_equal(a.row_ptr, g["row_ptr"]) and np.array_equal(a.col_ind, g["col_ind"])
    assert rel(a.values, g["values"]) <= 1e-12          # north-star tolerance (fp64)
    assert rel(b, g["b"]) <= 1e-12
    assert rel(info["f_int"], g["f_int"]) <= 1e-12
    assert np.array_equal(info["f_ext"], g["f_ext"])    # pure elementwise: bit-exact
    # mass-only entries and pinned rows are exact
    fixed = g["fixed_diag_slots"]
    assert np.all(a.values[fixed] == 1.0)
    a2, _, info2 = integ.assemble_system(st)
    assert not info2["pattern_rebuilt"] and integ.assembler.pattern_rebuilds == 1


def test_model_accumulate_and_blocks(golden, params):
    g = golden("beam_small")
    mesh = clamped_beam(*map(int, g["dims"]))
    model = models.make_model("corotational", mesh, params)
    s = TripletStream()
    s.begin_pass()
    f, kv = model.accumulate(g["positions"], stream=s, velocities=g["velocities"].ravel())
    s.end_pass()
    assert rel(f, g["f_int"]) <= 1e-12 and rel(kv, g["kv"]) <= 1e-12
    stiff = g["trip_vals"][12 * mesh.element_count:]
    assert rel(s.vals(), stiff) <= 1e-12
    assert np.array_equal(s.rows(), g["trip_rows"][12 * mesh.element_count:])


def test_nonfinite_positions_raise(params):
    mesh = clamped_beam(3, 3, 8)
    model = models.make_model("corotational", mesh, params)
    integ = BackwardEulerIntegrator(mesh, model, IntegratorConfig(dt=0.01))
    st = SimState.rest(mesh)
    st.positions = st.positions.copy()
    st.positions[40, 1] = np.nan
    with pytest.raises(models.ModelError):
        integ.assemble_system(st)


def test_linear_law_is_r_identity(params):
    mesh = clamped_beam(3, 3, 8)
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    x = mesh.nodes + 0.01 * np.random.default_rng(3).standard_normal(mesh.nodes.shape)
    v = np.random.default_rng(4).standard_normal(mesh.nodes.shape)
    f_ref, kv_ref, _ = O.corotational(mesh.nodes, mesh.elements, rest, x, v, linear=True)
    model = models.make_model("linear", mesh, params)
    f, kv = model.accumulate(x, velocities=v.ravel())
    assert rel(f, f_ref) <= 1e-12 and rel(kv, kv_ref) <= 1e-12


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_integrator_step_vs_reference(golden, params, name):
    """One full step (assembly + Jacobi PCG + kinematics) through the drop-in API."""
    g = golden(name)
    mesh = clamped_beam(*map(int, g["dims"]))
    model = models.make_model("corotational", mesh, params)
    integ = BackwardEulerIntegrator(mesh, model, IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    cfg = krylov.SolverConfig(1e-9, 8000)
    st = SimState(g["positions"].copy(), g["velocities"].copy(), np.zeros_like(g["positions"]),
                  np.zeros(len(g["b"])), g["f_ext_state"])
    res = integ.step(st, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
    assert res.report.converged and res.report.iterations == int(g["next_iterations"])
    assert rel(res.accelerations, g["next_accel"]) <= 1e-10
    assert rel(res.velocities, g["next_velocities"]) <= 1e-10
    assert rel(res.positions - g["positions"], g["next_positions"] - g["positions"]) <= 1e-10
    fixed = mesh.fixed_nodes
    assert np.array_equal(res.positions[fixed], g["positions"][fixed])


def test_device_resident_state_matches_host_state(golden, params):
    g = golden("beam_cfg1")
    mesh = clamped_beam(*map(int, g["dims"]))
    model = models.make_model("corotational", mesh, params)
    integ = BackwardEulerIntegrator(mesh, model, IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    cfg = krylov.SolverConfig(1e-9, 8000)

    def solve(a, b):
        return krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)

    solve.accepts_device = True
    st_h = SimState.rest(mesh)
    st_d = SimState.rest(mesh, device=True)
    for _ in range(3):
        rh = integ.step(st_h, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
        rd = integ.step(st_d, solve)
        assert rh.report.iterations == rd.report.iterations
    assert np.array_equal(st_h.positions, st_d.positions.cpu().numpy())


def _stvk_setup(golden, params):
    g = golden("beam_stvk")
    mesh = clamped_beam(*map(int, g["dims"]))
    model = models.make_model("stvk", mesh, params)
    assert isinstance(model, models.StVenantKirchhoffModel)
    integ = BackwardEulerIntegrator(mesh, model, IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    st = SimState(g["positions"].copy(), g["velocities"].copy(), np.zeros_like(g["positions"]),
                  np.zeros(len(g["b"])), g["f_ext_state"])
    return g, mesh, model, integ, st


def test_stvk_assemble_system_vs_reference(golden, params):
    """St-Venant-Kirchhoff law (models.py:241-287) through the fused device assembly."""
    g, mesh, model, integ, st = _stvk_setup(golden, params)
    a, b, info = integ.assemble_system(st)
    assert np.array_equal(a.row_ptr, g["row_ptr"]) and np.array_equal(a.col_ind, g["col_ind"])
    assert rel(a.values, g["values"]) <= 1e-12
    assert rel(b, g["b"]) <= 1e-12
    assert rel(info["f_int"], g["f_int"]) <= 1e-12
    assert np.array_equal(info["f_ext"], g["f_ext"])


def test_stvk_accumulate_and_blocks(golden, params):
    g, mesh, model, integ, st = _stvk_setup(golden, params)
    s = TripletStream()
    s.begin_pass()
    f, kv = model.accumulate(g["positions"], stream=s, velocities=g["velocities"].ravel())
    s.end_pass()
    assert rel(f, g["f_int"]) <= 1e-12 and rel(kv, g["kv"]) <= 1e-12
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    _, _, kb = O.stvk(mesh.nodes, mesh.elements, rest, g["positions"], g["velocities"])
    assert rel(s.vals(), kb.reshape(-1)) <= 1e-12
    assert rel(models.stvk_forces_and_stiffness(model.precomp, g["positions"])[0], g["f_int"]) <= 1e-12


def test_stvk_integrator_step_vs_reference(golden, params):
    g, mesh, model, integ, st = _stvk_setup(golden, params)
    cfg = krylov.SolverConfig(1e-9, 8000)
    res = integ.step(st, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
    assert res.report.converged and res.report.iterations == int(g["next_iterations"])
    assert rel(res.accelerations, g["next_accel"]) <= 1e-10
    assert rel(res.velocities, g["next_velocities"]) <= 1e-10
    assert rel(res.positions - g["positions"], g["next_positions"] - g["positions"]) <= 1e-10


@pytest.mark.parametrize("precond", ["jacobi", "ldlt"])
def test_captured_step_equals_compute_step(params, precond):
    """CapturedStep (assembly + persistent PCG + kinematics as one CUDA graph)
    gives bit-identical results to the eager compute_step, replay after replay."""
    from paper_2306_05893_b200 import mesh as M, ndprecond as ND

    mesh = clamped_beam(6, 6, 28)
    integ = BackwardEulerIntegrator(mesh, models.make_model("corotational", mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    cfg = krylov.SolverConfig(1e-9, 8000)
    st = SimState.rest(mesh, device=True)

    def jac(a, b):
        return krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)

    jac.accepts_device = True
    for _ in range(3):
        integ.step(st, jac)
    solve = jac
    if precond == "ldlt":
        plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 64))
        f = ND.ldlt_factor(integ.assemble_system(st)[0], plan)

        def solve(a, b):
            return krylov.pcg(a, b, f, cfg)

        solve.accepts_device = True
    cap = integ.capture(st, solve)
    assert cap.kernels >= 3
    for _ in range(3):
        ref = integ.compute_step(st, solve)
        got = cap.replay(st)
        assert got.report.iterations == ref.report.iterations
        for name in ("positions", "velocities", "accelerations", "f_int", "rhs"):
            assert bool((getattr(got, name) == getattr(ref, name)).all()), name
        integ.commit(st, ref)
