"""GPU parity of the plane-contact stage (contact.py) against the reference's
drop scenario (contact_drop.npz) and the oracle; reference test cases of
tests/test_contact.py restated on the device path."""

import numpy as np
import pytest

from oracle import tetsim_oracle as O

pytestmark = pytest.mark.gpu

import paper_2306_05893_b200 as P  # noqa: E402
from paper_2306_05893_b200 import contact as CT, krylov, mesh as M, ndprecond as ND  # noqa: E402
from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState  # noqa: E402


def rel(a, b):
    b = np.asarray(b)
    s = np.abs(b).max()
    return np.abs(np.asarray(a) - b).max() / (s if s else 1.0)


def drop(params, dims, plane, dt=0.01, device=False):
    mesh = P.generate_beam(*dims, 0.1)
    integ = BackwardEulerIntegrator(mesh, P.make_model("corotational", mesh, params), IntegratorConfig(dt=dt))
    return mesh, integ, CT.PlaneContactPipeline(integ, plane), SimState.rest(mesh, device=device)


@pytest.mark.parametrize("factor", ["host", "device", "callable"])
def test_drop_scenario_matches_reference(golden, params, factor):
    """14 steps of the reference's drop (contacts from step 7) with LDL^T factors of the
    previous step's matrix: same contact counts, residuals ~0, positions within 1e-9."""
    g = golden("contact_drop")
    mesh, integ, pipe, st = drop(params, tuple(int(v) for v in g["c_dims"]), float(g["c_plane"]))
    cfg = krylov.SolverConfig(1e-10, 8000)
    solve = lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)  # noqa: E731
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 16))
    f = None
    for k in range(int(g["c_steps"])):
        if f is None:
            ai = None
        elif factor == "callable":
            ai = lambda rhs, f=f: f.apply(rhs)  # noqa: E731  (the reference's cli.py:359 form)
        else:
            ai = f
        info = pipe.step(st, solve, ai)
        assert info.ncontacts == int(g["c_ncontacts"][k])
        assert info.result.report.iterations == int(g["c_iterations"][k])
        if info.ncontacts:
            assert info.complementarity_residual <= 1e-8
        assert info.max_penetration <= 1e-5
        assert rel(st.positions - mesh.nodes, g[f"c_pos_{k}"] - mesh.nodes) <= 1e-9, k
        assert rel(st.velocities, g[f"c_vel_{k}"]) <= 1e-8, k
        f = (ND.ldlt_factor_device(info.result.matrix, plan) if factor == "device"
             else ND.ldlt_factor(info.result.matrix, plan))


def test_first_contact_multipliers_vs_reference(golden, params):
    g = golden("contact_drop")
    k = int(g["c_step"])
    mesh, integ, pipe, st = drop(params, tuple(int(v) for v in g["c_dims"]), float(g["c_plane"]))
    st.positions, st.velocities = g[f"c_pos_{k - 2}"].copy(), g[f"c_vel_{k - 2}"].copy()
    a_prev, _, _ = integ.assemble_system(st)
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 16))
    f = ND.ldlt_factor(a_prev, plan)
    st.positions, st.velocities = g["c_x"].copy(), g["c_v"].copy()
    cfg = krylov.SolverConfig(1e-10, 8000)
    info = pipe.step(st, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg), f)
    assert info.ncontacts == len(g["c_nodes"])
    assert rel(pipe.last["lam"].cpu().numpy(), g["c_lam"]) <= 1e-10
    assert rel(pipe.last_w.cpu().numpy() / 0.01 ** 2, g["c_w"]) <= 1e-12


def test_detection_and_pgs_kernels(rng):
    pos = rng.standard_normal((500, 3))
    cs = CT.detect_plane_contacts(pos, -0.3)
    nodes, cols, coefs, viol = O.detect_plane_contacts(pos, -0.3)
    assert np.array_equal(cs.col_ind, cols) and np.array_equal(cs.violation, viol)
    assert CT.detect_plane_contacts(pos, -100.0).nconstraints == 0
    # PGS vs the oracle: SPD W, unilateral + bilateral rows
    a = rng.standard_normal((40, 40))
    w = a @ a.T + 40 * np.eye(40)
    rhs = rng.standard_normal(40)
    types = [CT.UNILATERAL if i % 3 else CT.BILATERAL for i in range(40)]
    lam = CT.projected_gauss_seidel(w, rhs, types)
    ref = O.projected_gauss_seidel(w, rhs, np.array([t == CT.UNILATERAL for t in types]))
    assert rel(lam, ref) <= 1e-10
    assert np.all(lam[[i for i in range(40) if i % 3]] >= 0.0)
    # zero-diagonal row dropped (reference test_contact.py:69-73)
    w2 = np.diag([0.0, 2.0])
    assert np.array_equal(CT.projected_gauss_seidel(w2, np.array([1.0, 4.0]), [CT.UNILATERAL] * 2), [0.0, 2.0])
    assert CT.projected_gauss_seidel(np.zeros((0, 0)), np.zeros(0), []).size == 0


def test_build_compliance_matches_dense_inverse(rng):
    """reference test_contact.py:110-126: W = J A^-1 J^T against a dense inverse."""
    n = 30
    a = rng.standard_normal((n, n))
    a = a @ a.T + n * np.eye(n)
    cs = CT.ConstraintSet(ndof=n, indptr=np.array([0, 2, 3, 5]), col_ind=np.array([1, 4, 7, 2, 9]),
                          coeffs=np.array([1.0, -0.5, 2.0, 0.3, -1.0]), violation=np.array([0.1, 0.2, 0.3]),
                          types=[CT.BILATERAL] * 3)
    w, s = CT.build_compliance(cs, lambda rhs: np.linalg.solve(a, rhs))
    J = np.stack([cs.row_dense(i) for i in range(3)])
    ref = J @ np.linalg.solve(a, J.T)
    assert rel(w, 0.5 * (ref + ref.T)) <= 1e-13
    assert np.array_equal(w, w.T)


def test_no_contacts_equals_plain_step(params):
    mesh = P.generate_beam(2, 2, 3, 0.1)
    cfg = krylov.SolverConfig(1e-10, 5000)
    solve = lambda a, b: krylov.cg(a, b, cfg)  # noqa: E731
    ia = BackwardEulerIntegrator(mesh, P.make_model("corotational", mesh, params), IntegratorConfig(dt=0.01))
    ib = BackwardEulerIntegrator(mesh, P.make_model("corotational", mesh, params), IntegratorConfig(dt=0.01))
    pipe = CT.PlaneContactPipeline(ib, plane_z=-100.0)
    sa, sb = SimState.rest(mesh), SimState.rest(mesh)
    for _ in range(3):
        ia.step(sa, solve)
        assert pipe.step(sb, solve).ncontacts == 0
    assert np.array_equal(sa.positions, sb.positions) and np.array_equal(sa.velocities, sb.velocities)


def test_device_state_drop_with_async_device_factors(params):
    """Device-resident state, CG compliance on the first contact steps, then
    factors from AsyncPreconditioner(device=True): gaps closed every step."""
    mesh, integ, pipe, st = drop(params, (3, 3, 4), -0.012, dt=0.02, device=True)
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 16))
    pre = ND.AsyncPreconditioner(plan, device=True)
    cfg = krylov.SolverConfig(1e-10, 8000)
    solve = lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)  # noqa: E731
    landed = False
    for k in range(12):
        pre.poll()
        info = pipe.step(st, solve, pre if pre.status is ND.PrecondStatus.READY else None)
        gap = float(st.positions[:, 2].min()) - pipe.plane_z
        assert gap >= -1e-6
        if info.ncontacts:
            landed = True
            assert gap <= 1e-4
        pre.update(info.result.matrix, k)
    assert landed
    pre.close()


def test_factor_path_equals_column_path_for_general_rows(params, rng):
    """Multi-entry (bilateral) constraint rows: the lower-sweep compliance
    Y^T D^-1 Y and the one-upper-sweep correction equal the reference's
    column-by-column form with the same factors."""
    mesh = P.generate_beam(3, 3, 6, 0.1)
    integ = BackwardEulerIntegrator(mesh, P.make_model("corotational", mesh, params), IntegratorConfig(dt=0.01))
    cfg = krylov.SolverConfig(1e-10, 8000)
    st = SimState.rest(mesh)
    solve = lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)  # noqa: E731
    free = integ.compute_step(st, solve)
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 16))
    f = ND.ldlt_factor(free.matrix, plan)
    m = 7
    indptr = np.concatenate([[0], np.cumsum(rng.integers(1, 4, m))])
    cols = np.concatenate([rng.choice(mesh.ndof, indptr[i + 1] - indptr[i], replace=False) for i in range(m)])
    cs = CT.ConstraintSet(ndof=mesh.ndof, indptr=indptr, col_ind=cols, coeffs=rng.standard_normal(len(cols)),
                          violation=1e-4 * rng.standard_normal(m), types=[CT.BILATERAL] * m)
    pipe = CT.PlaneContactPipeline(integ, -100.0)
    lam_f, info_f, acc_f = pipe._resolve_with_factors(free, cs, f, 0.01)
    w_f = pipe.last_w.cpu().numpy()
    lam_c, info_c, acc_c = pipe._resolve_with_columns(free, cs, lambda r: f.apply(r), 0.01)
    J = np.stack([cs.row_dense(i) for i in range(m)])
    S = np.stack([O.apply(f, J[i]) for i in range(m)], axis=1)
    W = J @ S
    W = 0.5 * (W + W.T) * 0.01 ** 2
    assert rel(w_f, W) <= 1e-12
    lam = O.projected_gauss_seidel(W, cs.violation, np.zeros(m, dtype=bool))
    assert rel(lam_f.cpu().numpy(), lam) <= 1e-9 and rel(lam_c.cpu().numpy(), lam) <= 1e-9
    acc = free.accelerations.reshape(-1) - S @ lam
    assert rel(acc_f.cpu().numpy(), acc) <= 1e-9 and rel(acc_c.cpu().numpy(), acc) <= 1e-9


def test_zero_multiplier_correction_is_identity(params):
    """reference test_contact.py:183-196: lambda = 0 leaves the free motion unchanged (and m = 0 works)."""
    mesh = P.generate_beam(2, 2, 3, 0.1)
    integ = BackwardEulerIntegrator(mesh, P.make_model("corotational", mesh, params), IntegratorConfig(dt=0.01))
    st = SimState.rest(mesh)
    cfg = krylov.SolverConfig(1e-10, 5000)
    free = integ.compute_step(st, lambda a, b: krylov.cg(a, b, cfg))
    for plane in (-2.0, 100.0):
        cs = CT.detect_plane_contacts(free.positions - np.array([0, 0, 1.0]), plane_z=plane)
        lam = np.zeros(cs.nconstraints)
        s_cols = np.zeros((mesh.ndof, cs.nconstraints))
        corrected = CT.correct_motion(free, st, cs, lam, s_cols, 0.01, mesh.fixed_nodes)
        assert np.array_equal(corrected.positions, free.positions)
        assert np.array_equal(corrected.velocities, free.velocities)


def test_committed_penetration_bounded_and_pattern_constant(params):
    """reference test_contact.py:198-212: 40 steps of a drop onto z = -0.03 with CG
    compliance columns -- committed penetration <= 1e-5, complementarity residual
    <= 1e-8, and the CSR pattern is built once."""
    mesh, integ, pipe, st = drop(params, (3, 3, 4), -0.03)
    cfg = krylov.SolverConfig(1e-10, 5000)
    solve = lambda a, b: krylov.cg(a, b, cfg)  # noqa: E731
    contacts = 0
    for _ in range(40):
        info = pipe.step(st, solve)
        assert info.max_penetration <= 1e-5
        if info.ncontacts:
            contacts += 1
            assert info.complementarity_residual <= 1e-8
    assert contacts > 0
    assert integ.assembler.pattern_rebuilds == 1
