"""GPU parity: device PCG (identity / Jacobi / LDL^T) and the level-scheduled
LDL^T sweeps against the oracle and the reference's golden outputs."""

import numpy as np
import pytest

from conftest import GoldenFactors, clamped_beam
from oracle import tetsim_oracle as O

pytestmark = pytest.mark.gpu

from paper_2306_05893_b200 import krylov, mesh as M, ndprecond as ND  # noqa: E402
from paper_2306_05893_b200.assembly import CsrMatrix  # noqa: E402


def rel(a, b):
    b = np.asarray(b)
    s = np.abs(b).max()
    return np.abs(np.asarray(a) - b).max() / (s if s else 1.0)


def golden_matrix(g):
    n = len(g["row_ptr"]) - 1
    return CsrMatrix(n, n, g["row_ptr"], g["col_ind"], g["values"])


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_pcg_jacobi_and_cg_vs_reference(golden, name):
    g = golden(name)
    a = golden_matrix(g)
    cfg = krylov.SolverConfig(1e-9, 8000)
    x, rep = krylov.pcg(a, g["b"], krylov.jacobi_precond(a), cfg)
    assert rep.converged and rep.iterations == int(g["it_jacobi"])
    assert rel(x, g["x_jacobi"]) <= 1e-10
    x, rep = krylov.cg(a, g["b"], cfg)
    assert rep.converged and rep.iterations == int(g["it_cg"])
    assert rel(x, g["x_cg"]) <= 1e-10
    # relative residuals agree within 1e-10 (north-star tolerance)
    assert abs(rep.final_residual - float(g["res_cg"])) <= 1e-10


def test_pcg_device_jacobi_on_device_matrix_equals_host_diag(golden):
    g = golden("beam_cfg1")
    a = golden_matrix(g)
    import torch

    ad = CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_ind, torch.from_numpy(g["values"]).cuda())
    cfg = krylov.SolverConfig(1e-9, 8000)
    x1, r1 = krylov.pcg(a, g["b"], krylov.jacobi_precond(a), cfg)            # explicit host diagonal
    x2, r2 = krylov.pcg(ad, g["b"], krylov.jacobi_precond(ad), cfg)          # device-extracted diagonal
    assert r1.iterations == r2.iterations and np.array_equal(x1, x2)


def test_pcg_edge_cases(golden):
    g = golden("beam_small")
    a = golden_matrix(g)
    n = a.nrows
    cfg = krylov.SolverConfig(1e-9, 8000)
    x, rep = krylov.pcg(a, np.zeros(n), None, cfg)                         # krylov.py:133-134
    assert rep.iterations == 0 and rep.converged and rep.final_residual == 0.0 and not x.any()
    x0 = g["x_cg"]
    x, rep = krylov.cg(a, g["b"], cfg, x0=x0)                              # already converged
    assert rep.iterations == 0 and rep.converged and np.array_equal(x, x0)
    x, rep = krylov.cg(a, g["b"], krylov.SolverConfig(1e-9, 3))            # max_iterations hit
    ox, oit, ores, oconv = O.pcg(g["row_ptr"], g["col_ind"], g["values"], g["b"], None, 1e-9, 3)
    assert rep.iterations == 3 and not rep.converged and rel(x, ox) <= 1e-12
    x, rep = krylov.cg(a, g["b"], krylov.SolverConfig(1e-9, 0))
    assert rep.iterations == 0 and not rep.converged
    with pytest.raises(krylov.SolverError):
        krylov.SolverConfig(0.0)
    z = CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]))
    with pytest.raises(krylov.SolverError, match="zero diagonal entry at row 0"):
        krylov.jacobi_precond(z)


def test_pcg_warm_start_matches_oracle(golden):
    g = golden("beam_cfg1")
    a = golden_matrix(g)
    x0 = 0.5 * g["x_cg"]
    x, rep = krylov.cg(a, g["b"], krylov.SolverConfig(1e-9, 8000), x0=x0)
    ox, oit, ores, _ = O.pcg(g["row_ptr"], g["col_ind"], g["values"], g["b"], None, 1e-9, 8000, x0=x0)
    assert rep.iterations == oit and rel(x, ox) <= 1e-10


def test_pcg_custom_preconditioner_protocol(golden):
    g = golden("beam_small")
    a = golden_matrix(g)
    dense = a.to_dense()

    class Exact:
        def apply(self, r):
            return np.linalg.solve(dense, r)

    x, rep = krylov.pcg(a, g["b"], Exact(), krylov.SolverConfig(1e-9, 100))
    assert rep.converged and rep.iterations <= 2     # reference tests/test_krylov.py:140-152


def test_ldlt_sweeps_vs_reference_factors(golden):
    """Device sweeps on the REFERENCE's own factor values (golden) vs its outputs."""
    g = golden("ldlt_small")
    f = GoldenFactors(g)
    lf = ND.LdlFactors(f.d, f.plan, 0, [ND._BlockFactor(b.start, b.stop, b.level, b.anc, b.l11, b.l21,
                                                         b.tile, b.tile_inv) for b in f.blocks],
                       [[None]] * 0)
    lf.levels = [[lf.blocks[i] for i, b in enumerate(f.blocks) if b.level == lv] for lv in range(len(f.levels))]
    assert rel(ND.solve_lower(lf, g["r"]), g["lower"]) <= 1e-12
    assert rel(ND.solve_upper(lf, g["r"]), g["upper"]) <= 1e-12
    assert rel(ND.apply(lf, g["r"]), g["apply"]) <= 1e-12
    a = golden_matrix(g)
    x, rep = krylov.pcg(a, g["b"], lf, krylov.SolverConfig(1e-9, 8000))
    assert rep.converged and rep.iterations == int(g["it_ldlt"])
    assert rel(x, g["x_ldlt"]) <= 1e-10


@pytest.mark.parametrize("dims,leaf,tile", [((6, 6, 28), 64, 16), ((10, 10, 100), 64, 16),
                                            ((4, 4, 12), 16, 4), ((4, 4, 12), 16, 64)])
def test_ldlt_sweeps_vs_oracle(golden, params, dims, leaf, tile):
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState
    from paper_2306_05893_b200 import models

    mesh = clamped_beam(*dims)
    integ = BackwardEulerIntegrator(mesh, models.make_model("corotational", mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    a, b, _ = integ.assemble_system(SimState.rest(mesh))
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), leaf))
    f = ND.ldlt_factor(a, plan, tile=tile)
    r = np.random.default_rng(55).standard_normal(a.nrows)
    assert rel(ND.solve_lower(f, r), O.solve_lower(f, r)) <= 1e-12
    assert rel(ND.solve_upper(f, r), O.solve_upper(f, r)) <= 1e-12
    z = ND.apply(f, r)
    assert rel(z, O.apply(f, r)) <= 1e-12
    x = np.linalg.solve(a.to_dense(), r) if a.nrows <= 4000 else None
    if x is not None:
        assert rel(z, x) <= 1e-10


def test_stale_factor_pcg_vs_oracle(golden, params):
    """Factors of step 4 applied at step 7 (fixed staleness replay,
    reference tests/test_ndprecond.py:298-328): same iteration count as the oracle."""
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState
    from paper_2306_05893_b200 import models

    mesh = clamped_beam(10, 10, 100)
    integ = BackwardEulerIntegrator(mesh, models.make_model("corotational", mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    cfg = krylov.SolverConfig(1e-9, 8000)
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 64))
    st = SimState.rest(mesh)
    f = None
    for k in range(1, 7):
        res = integ.step(st, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
        if k == 4:
            f = ND.ldlt_factor(res.matrix, plan, source_step=k)
    a, b, _ = integ.assemble_system(st)
    x, rep = krylov.pcg(a, b, f, cfg)
    ox, oit, ores, oconv = O.pcg(a.row_ptr, a.col_ind, a.values, b, lambda r: O.apply(f, r), 1e-9, 8000)
    assert rep.converged and oconv and rep.iterations == oit and rep.iterations <= 8
    assert rel(x, ox) <= 1e-10


def test_async_preconditioner_lifecycle(params):
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState
    from paper_2306_05893_b200 import models

    mesh = clamped_beam(4, 4, 12)
    integ = BackwardEulerIntegrator(mesh, models.make_model("corotational", mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 16))
    pre = ND.AsyncPreconditioner(plan)
    assert pre.status is ND.PrecondStatus.EMPTY
    with pytest.raises(ND.LifecycleError):
        pre.apply(np.ones(mesh.ndof))
    cfg = krylov.SolverConfig(1e-9, 8000)
    st = SimState.rest(mesh)
    res = integ.step(st, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
    pre.update(res.matrix, 1)
    pre.wait_ready()
    assert pre.status is ND.PrecondStatus.READY and pre.staleness(3) == 2
    res = integ.step(st, lambda a, b: krylov.pcg(a, b, pre, cfg))
    assert res.report.converged and res.report.iterations <= 5
    pre.close()


@pytest.mark.parametrize("mode", [None, 1])
def test_ldlt_lower_input_modes_agree(params, mode):
    """Both ways of forming a block's input (items sum their contributions / the
    completing child item sums them once) give the oracle's sweeps; repeated
    applies are bitwise reproducible (fixed reduction order, counters reset)."""
    import torch
    from paper_2306_05893_b200._ldlt_pack import DevicePanels
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState
    from paper_2306_05893_b200 import models

    mesh = clamped_beam(10, 10, 60)
    integ = BackwardEulerIntegrator(mesh, models.make_model("corotational", mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    a, _, _ = integ.assemble_system(SimState.rest(mesh))
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 64))
    f = ND.ldlt_factor(a, plan)
    dev = DevicePanels(f, force_mode=mode)
    r = np.random.default_rng(5).standard_normal(a.nrows)
    dr = torch.from_numpy(r).cuda()
    outs = []
    for _ in range(3):
        z = torch.empty_like(dr)
        dev.run("apply", dr, z)
        outs.append(z.cpu().numpy())
    assert rel(outs[0], O.apply(f, r)) <= 1e-12
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    y = torch.empty_like(dr)
    dev.run("lower", dr, y)
    assert rel(y.cpu().numpy(), O.solve_lower(f, r)) <= 1e-12
