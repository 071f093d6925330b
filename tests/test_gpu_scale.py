"""GPU parity at the benchmark sizes: config 2 (10x10x100), config 3
(20x20x250, the north-star 100k-node beam) and one config-5 simulation
(20x20x125, 50k nodes) -- the device path through the public API against the
CPU oracle on the same scenario state.

Reference anchors: the large-scale solve / stale-factor PCG checks of
tests/test_ndprecond.py:298-328 and tests/test_acceptance.py:175-224
(criteria 5 and 6); assembly parity as tests/test_integrator.py:48-54 with
the north-star bar (CSR bit-exact, values 1e-12 relative in the inf-norm,
SURVEY.md App. A.9); PCG: identical iteration counts, x within 1e-10.
"""

import numpy as np
import pytest

from conftest import clamped_beam
from oracle import tetsim_oracle as O

pytestmark = pytest.mark.gpu

from paper_2306_05893_b200 import krylov, mesh as M, models, ndprecond as ND  # noqa: E402
from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState  # noqa: E402

CFG = krylov.SolverConfig(1e-9, 8000)
SCALES = {"cfg2": (10, 10, 100), "cfg3": (20, 20, 250), "cfg5": (20, 20, 125)}
STALE_FROM, AT = 4, 7


def rel(a, b):
    b = np.asarray(b)
    s = np.abs(b).max()
    return np.abs(np.asarray(a) - b).max() / (s if s else 1.0)


def jacobi(a, b):
    return krylov.pcg(a, b, krylov.jacobi_precond(a), CFG)


jacobi.accepts_device = True

_cache = {}


def scenario(name, with_factors):
    """Device scenario from rest to step AT (Jacobi steps), host factors of
    step STALE_FROM's matrix (fixed staleness 3), the oracle's rest data and
    cached mapping of the same mesh, and the oracle's system at step AT."""
    key = (name, with_factors)
    if key in _cache:
        return _cache[key]
    _cache.clear()  # one large scenario resident at a time
    params = models.MaterialParams(1e5, 0.3, 1000.0)
    mesh = clamped_beam(*SCALES[name])
    integ = BackwardEulerIntegrator(mesh, models.make_model("corotational", mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 64)) if with_factors else None
    st = SimState.rest(mesh, device=True)
    f = None
    for k in range(1, AT):
        res = integ.step(st, jacobi)
        assert res.report.converged
        if with_factors and k == STALE_FROM:
            f = ND.ldlt_factor(res.matrix, plan, source_step=k)
    host = st.to_host()
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    pattern = O.assembly_pattern(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest)
    ref = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, host.positions, host.velocities,
                            host.f_ext, 0.01, (0.0, -9.81, 0.0), pattern=pattern)
    out = dict(mesh=mesh, integ=integ, state=st, host=host, factors=f, ref=ref)
    _cache[key] = out
    return out


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_assembly_vs_oracle_at_scale(name):
    """Device fused assembly of the scenario state vs the oracle's: CSR indices
    bit-exact, A values within 1e-12 (inf-norm relative, north_star).

    b and f_int: f_e = R Ke (R^T x - x0) cancels |x| up to the beam length
    (10 / 25 m) against x0, so rounding-level differences of the polar factor
    R move them far more than A.  Their bar is the oracle's OWN sensitivity
    to R at rounding level: the oracle's b / f_int with every entry of R
    perturbed by a random relative 2^-52 (measured 1.3e-12 at cfg2, 4.5e-12
    at cfg3).  The device's R (per-element stop, cofactor inverse) must stay
    within 4x that floor -- and within 1e-10, the bar of the solve it feeds.
    """
    from oracle import tetsim_oracle as O2

    s = scenario(name, with_factors=(name == "cfg3"))
    a, b, info = s["integ"].assemble_system(s["state"])
    ref = s["ref"]
    assert np.array_equal(a.row_ptr, ref["row_ptr"]) and np.array_equal(a.col_ind, ref["col_ind"])
    assert rel(a.values, ref["values"]) <= 1e-12
    mesh, host = s["mesh"], s["host"]
    rest = O2.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    alt = O2.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, host.positions, host.velocities,
                             host.f_ext, 0.01, (0.0, -9.81, 0.0), extra_newton=np.random.default_rng(1))
    assert rel(alt["values"], ref["values"]) <= 1e-14  # A is insensitive to R at rounding level
    bh = b.cpu().numpy() if hasattr(b, "cpu") else b
    fi = info["f_int"]
    fi = fi.cpu().numpy() if hasattr(fi, "cpu") else fi
    for got, key in ((bh, "b"), (fi, "f_int")):
        floor = rel(alt[key], ref[key])
        err = rel(got, ref[key])
        assert err <= max(4.0 * floor, 1e-12) and err <= 1e-10, (key, err, floor)


def test_stale_ldlt_pcg_vs_oracle_cfg3():
    """Config 3, factors of step 4 at step 7: the device LDL^T-PCG takes the
    oracle's iteration count on the same factors; x within 1e-10; final
    relative residuals agree within 1e-10 (north_star)."""
    s = scenario("cfg3", with_factors=True)
    a, b, _ = s["integ"].assemble_system(s["state"])
    f = s["factors"]
    x, rep = krylov.pcg(a, b, f, CFG)
    ref = s["ref"]
    ox, oit, ores, oconv = O.pcg(ref["row_ptr"], ref["col_ind"], ref["values"], ref["b"],
                                 lambda r: O.apply(f, r), 1e-9, 8000)
    x = x.cpu().numpy() if hasattr(x, "cpu") else x
    assert rep.converged and oconv
    assert rep.iterations == oit and rep.iterations <= 15  # test_acceptance.py:198-224 (stale <= 15)
    assert rel(x, ox) <= 1e-10
    assert abs(rep.final_residual - ores) <= 1e-10


@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_jacobi_pcg_vs_oracle_at_scale(name):
    s = scenario(name, with_factors=(name == "cfg3"))
    a, b, _ = s["integ"].assemble_system(s["state"])
    x, rep = krylov.pcg(a, b, krylov.jacobi_precond(a), CFG)
    ref = s["ref"]
    inv = O.jacobi_inv_diag(ref["row_ptr"], ref["col_ind"], ref["values"], len(ref["b"]))
    ox, oit, ores, oconv = O.pcg(ref["row_ptr"], ref["col_ind"], ref["values"], ref["b"], lambda r: r * inv,
                                 1e-9, 8000)
    x = x.cpu().numpy() if hasattr(x, "cpu") else x
    assert rep.converged and oconv and rep.iterations == oit
    assert rel(x, ox) <= 1e-10
    assert abs(rep.final_residual - ores) <= 1e-10


def test_ldlt_apply_vs_oracle_cfg3():
    """Isolated device apply / lower / upper sweeps on the cfg3 factors vs the
    oracle's level-scheduled restatement (1e-12), seed 55 (test_acceptance.py:184-185)."""
    s = scenario("cfg3", with_factors=True)
    f = s["factors"]
    r = np.random.default_rng(55).standard_normal(f.plan.n)
    assert rel(ND.solve_lower(f, r), O.solve_lower(f, r)) <= 1e-12
    assert rel(ND.solve_upper(f, r), O.solve_upper(f, r)) <= 1e-12
    assert rel(ND.apply(f, r), O.apply(f, r)) <= 1e-12


def test_scenario_trajectory_vs_oracle_cfg2():
    """Six implicit steps from rest on the device vs six oracle steps (Jacobi-
    PCG): positions and velocities within 1e-10 at every step."""
    mesh = clamped_beam(10, 10, 100)
    params = models.MaterialParams(1e5, 0.3, 1000.0)
    integ = BackwardEulerIntegrator(mesh, models.make_model("corotational", mesh, params),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    st = SimState.rest(mesh, device=True)
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    pattern = O.assembly_pattern(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest)
    x, v, fe = mesh.nodes.copy(), np.zeros_like(mesh.nodes), np.zeros(mesh.ndof)
    for _ in range(6):
        res = integ.step(st, jacobi)
        out = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, x, v, fe, 0.01,
                                (0.0, -9.81, 0.0), pattern=pattern)
        inv = O.jacobi_inv_diag(out["row_ptr"], out["col_ind"], out["values"], len(out["b"]))
        acc, it, _, conv = O.pcg(out["row_ptr"], out["col_ind"], out["values"], out["b"], lambda r: r * inv,
                                 1e-9, 8000)
        assert conv and res.report.iterations == it
        x, v, _ = O.advance(acc, x, v, 0.01, mesh.fixed_nodes)
        h = st.to_host()
        assert rel(h.positions, x) <= 1e-10 and rel(h.velocities, v) <= 1e-10
