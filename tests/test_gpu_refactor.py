"""GPU parity of the device LDL^T refactorisation (csrc/refactor.cu) against
the reference's own factors (golden), the host multifrontal restatement and
the oracle's sweeps / PCG."""

import numpy as np
import pytest

from conftest import GoldenFactors, clamped_beam
from oracle import tetsim_oracle as O

pytestmark = pytest.mark.gpu

from paper_2306_05893_b200 import _ldlt_pack as K, krylov, mesh as M, models, ndprecond as ND  # noqa: E402
from paper_2306_05893_b200 import refactor as R  # noqa: E402
from paper_2306_05893_b200.assembly import CsrMatrix  # noqa: E402
from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState  # noqa: E402


def rel(a, b):
    b = np.asarray(b)
    s = np.abs(b).max()
    return np.abs(np.asarray(a) - b).max() / (s if s else 1.0)


def scenario(params, dims, steps=3):
    mesh = clamped_beam(*dims)
    integ = BackwardEulerIntegrator(mesh, models.make_model("corotational", mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    st = SimState.rest(mesh)
    cfg = krylov.SolverConfig(1e-9, 8000)
    for _ in range(steps):
        integ.step(st, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
    a, b, _ = integ.assemble_system(st)
    return mesh, a, b


def test_device_factor_matches_reference_factors(golden, params):
    """ldlt_factor on the device vs the reference's own factors (ldlt_small: the
    factors of step 4's matrix, applied in PCG at step 7)."""
    g = golden("ldlt_small")
    ref = GoldenFactors(g)
    mesh = clamped_beam(4, 4, 12)
    integ = BackwardEulerIntegrator(mesh, models.make_model("corotational", mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    cfg = krylov.SolverConfig(1e-9, 8000)
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 16))
    assert np.array_equal(plan.perm, ref.plan.perm)
    st = SimState.rest(mesh)
    for k in range(1, 5):
        res = integ.step(st, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
    f = ND.ldlt_factor_device(res.matrix, plan, tile=int(g["f_tile"]), source_step=4)
    h = f.to_host()
    assert rel(h.d, ref.d) <= 1e-11
    for hb, rb in zip(h.blocks, ref.blocks):
        assert hb.start == rb.start and np.array_equal(hb.anc, rb.anc)
        assert rel(hb.l11, rb.l11) <= 1e-11
        if len(rb.anc):
            assert rel(hb.l21, rb.l21) <= 1e-11
    assert rel(ND.apply(f, g["r"]), g["apply"]) <= 1e-11
    a = CsrMatrix(len(g["row_ptr"]) - 1, len(g["row_ptr"]) - 1, g["row_ptr"], g["col_ind"], g["values"])
    x, rep = krylov.pcg(a, g["b"], f, cfg)
    assert rep.converged and rep.iterations == int(g["it_ldlt"])
    assert rel(x, g["x_ldlt"]) <= 1e-10


@pytest.mark.parametrize("dims,leaf", [((6, 6, 28), 64), ((10, 10, 100), 64), ((4, 4, 12), 16)])
def test_device_factor_image_vs_host_pack(params, dims, leaf):
    mesh, a, b = scenario(params, dims)
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), leaf))
    hf = ND.ldlt_factor(a, plan)
    H = K.pack(hf)
    rf = R.DeviceRefactor(a, plan)
    df = rf.factor(a, source_step=3)
    img = df.device()
    assert rel(img.t["g"].cpu().numpy(), H["g"]) <= 1e-12
    assert rel(img.t["gt"].cpu().numpy(), H["gt"]) <= 1e-12
    assert rel(img.t["d"].cpu().numpy(), hf.d) <= 1e-12
    r = np.random.default_rng(55).standard_normal(a.nrows)
    assert rel(ND.apply(df, r), O.apply(hf, r)) <= 1e-12
    assert rel(ND.solve_lower(df, r), O.solve_lower(hf, r)) <= 1e-12
    # same PCG iterations as the host factor (oracle PCG)
    cfg = krylov.SolverConfig(1e-9, 8000)
    x, rep = krylov.pcg(a, b, df, cfg)
    ox, oit, ores, oconv = O.pcg(a.row_ptr, a.col_ind, a.values, b, lambda v: O.apply(hf, v), 1e-9, 8000)
    assert rep.converged and oconv and rep.iterations == oit
    assert rel(x, ox) <= 1e-10
    # run to run: bit-identical
    g1 = img.t["g"].clone()
    rf.factor(a)
    assert bool((img.t["g"] == g1).all())


def test_device_factor_reconstructs_matrix(params):
    mesh, a, b = scenario(params, (4, 4, 12), steps=2)
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 16))
    f = ND.ldlt_factor_device(a, plan)
    L = f.l_matrix.to_dense() + np.eye(a.nrows)
    Ap = a.to_dense()[np.ix_(plan.perm, plan.perm)]
    assert rel(L @ np.diag(f.to_host().d) @ L.T, Ap) <= 1e-10
    # same L as the host factorisation (the device's roundoff leaves tiny values
    # where the host produced exact zeros, so fill_in counts are not compared)
    Lh = ND.ldlt_factor(a, plan).l_matrix.to_dense() + np.eye(a.nrows)
    assert rel(L, Lh) <= 1e-12


def test_device_factor_indefinite_raises(params):
    mesh, a, b = scenario(params, (3, 3, 8), steps=1)
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 16))
    vals = a.values.copy()
    d = np.flatnonzero(a.col_ind == np.repeat(np.arange(a.nrows), np.diff(a.row_ptr)))
    vals[d[40]] = -1.0
    bad = CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_ind, vals)
    with pytest.raises(ND.IndefiniteMatrixError):
        ND.ldlt_factor_device(bad, plan)


def test_async_preconditioner_device_refactor(params):
    """AsyncPreconditioner(device=True): refactorisation on a side stream into
    the idle sweep image, published at step boundaries (ndprecond.py:714-831)."""
    mesh = clamped_beam(6, 6, 28)
    integ = BackwardEulerIntegrator(mesh, models.make_model("corotational", mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 64))
    pre = ND.AsyncPreconditioner(plan, device=True)
    assert pre.status is ND.PrecondStatus.EMPTY
    cfg = krylov.SolverConfig(1e-9, 8000)
    st = SimState.rest(mesh, device=True)
    seen = set()
    for k in range(1, 9):
        pre.poll()
        solve = (lambda a, b: krylov.pcg(a, b, pre, cfg)) if pre.status is ND.PrecondStatus.READY else \
            (lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
        res = integ.step(st, solve)
        assert res.report.converged
        if pre.status is ND.PrecondStatus.READY:
            assert res.report.iterations <= 8      # stale factors (reference acceptance: <= 15)
            seen.add(id(pre.factors.device()))
        pre.update(res.matrix, k)
        if k == 1:
            assert pre.status is ND.PrecondStatus.FACTORIZING
            pre.wait_ready()
            assert pre.staleness(2) == 1
    assert len(seen) == 2                      # both sweep images were used
    assert not pre.disabled
    pre.close()


@pytest.mark.parametrize("k", [1, 3, 8, 11])
def test_multi_rhs_lower_sweep_equals_single(params, k):
    """tsb_ldlt_lower_multi: k right-hand sides, bit-identical to k single sweeps
    (same per-RHS summation order), and equal to the oracle's lower solve."""
    import torch

    mesh, a, b = scenario(params, (10, 10, 60), steps=2)
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 64))
    f = ND.ldlt_factor(a, plan)
    dev = f.device()
    R = torch.randn(k, a.nrows, dtype=torch.float64, device="cuda")
    R[0].zero_()
    R[0, 17] = -1.0                      # a contact-like unit column
    Y = torch.empty_like(R)
    dev.lower_multi(R, Y)
    Y1 = torch.empty_like(R)
    for j in range(k):
        dev.run("lower", R[j], Y1[j])
    assert bool((Y == Y1).all())
    assert rel(Y[k - 1].cpu().numpy(), O.solve_lower(f, R[k - 1].cpu().numpy())) <= 1e-12


@pytest.mark.parametrize("k,leaf", [(30, 8), (45, 40)])
def test_device_factor_on_grid_laplacian(k, leaf):
    """Non-mesh pattern (2D 5-point Laplacian + random SPD perturbation,
    plan from graph_from_pattern as in the reference's random-SPD tests):
    ragged blocks, several pivot tiles per front, multi-child separators."""
    rng = np.random.default_rng(k)
    n = k * k
    rows, cols, vals = [], [], []
    for i in range(k):
        for j in range(k):
            p = i * k + j
            rows.append(p); cols.append(p); vals.append(4.5 + rng.random())
            for di, dj in ((0, 1), (1, 0)):
                if i + di < k and j + dj < k:
                    q = (i + di) * k + (j + dj)
                    w = -1.0 + 0.1 * rng.standard_normal()
                    rows += [p, q]; cols += [q, p]; vals += [w, w]
    rows, cols, vals = map(np.asarray, (rows, cols, vals))
    o = np.lexsort((cols, rows))
    rows, cols, vals = rows[o], cols[o], vals[o]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    a = CsrMatrix(n, n, row_ptr, cols.astype(np.int64), vals)
    plan = ND.nested_dissection(ND.graph_from_pattern(a), leaf)
    hf = ND.ldlt_factor(a, plan)
    df = ND.ldlt_factor_device(a, plan)
    r = rng.standard_normal(n)
    assert rel(ND.apply(df, r), O.apply(hf, r)) <= 1e-12
    assert rel(ND.apply(df, r), np.linalg.solve(a.to_dense(), r)) <= 1e-10
    assert rel(df.to_host().d, hf.d) <= 1e-12
