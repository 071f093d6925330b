"""Generate the golden fixtures by running the REFERENCE (tetsim) in the build container.

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden.py

/root/reference does not exist on the GPU box; the fixtures written here
(tests/golden/*.npz, committed) carry the reference's outputs there.  Every
array comes from the reference's own public API with workers=1 and one BLAS
thread (its parity configuration).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import tetsim  # noqa: E402
from tetsim import krylov, ndprecond  # noqa: E402
from tetsim.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState  # noqa: E402

OUT = Path(__file__).resolve().parent
PARAMS = tetsim.MaterialParams(young_modulus=1e5, poisson_ratio=0.3, density=1000.0)


def clamped(nx, ny, nz, spacing=0.1):
    mesh = tetsim.generate_beam(nx, ny, nz, spacing)
    return mesh.with_fixed_nodes(np.flatnonzero(mesh.nodes[:, 2] == 0.0))


def scenario_system(dims, steps, tol=1e-9, with_triplets=False, law="corotational"):
    """Run `steps` Jacobi-PCG steps from rest (gravity along -y), then record
    the next step's assembled system and its solves."""
    mesh = clamped(*dims)
    model = tetsim.make_model(law, mesh, PARAMS)
    integ = BackwardEulerIntegrator(mesh, model, IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    cfg = krylov.SolverConfig(tol, 8000)
    solve = lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)  # noqa: E731
    st = SimState.rest(mesh)
    for _ in range(steps):
        integ.step(st, solve)
    a, b, info = integ.assemble_system(st)
    _, kv = model.accumulate(st.positions, velocities=st.velocities.ravel())
    xj, rj = krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)
    xc, rc = krylov.cg(a, b, krylov.SolverConfig(tol, 8000))
    xr = np.random.default_rng(0).standard_normal(a.ncols)
    out = dict(
        dims=np.array(dims), positions=st.positions, velocities=st.velocities, f_ext_state=st.f_ext,
        fixed_nodes=mesh.fixed_nodes, elements=mesh.elements, nodes=mesh.nodes,
        row_ptr=a.row_ptr, col_ind=a.col_ind, values=a.values, b=b, f_int=info["f_int"],
        f_ext=info["f_ext"], kv=kv, fixed_diag_slots=integ.assembler.mapping.fixed_diag_slots,
        x_jacobi=xj, it_jacobi=rj.iterations, res_jacobi=rj.final_residual,
        x_cg=xc, it_cg=rc.iterations, res_cg=rc.final_residual,
        spmv_x=xr, spmv_y=krylov.spmv(a, xr),
        grads=model.precomp.grads, volume=model.precomp.volume, ke=model.precomp.ke,
        mass_diag=integ.mass_diag,
    )
    if with_triplets:
        s = integ.assembler.stream
        mp = integ.assembler.mapping
        out.update(trip_rows=s.rows().copy(), trip_cols=s.cols().copy(), trip_vals=s.vals().copy(),
                   coeffs=integ._coeffs.copy(), kept=mp.kept, kept_slots=mp.kept_slots,
                   slot_of_triplet=mp.slot_of_triplet)
    # one more committed step: next positions/velocities (integrator parity)
    res = integ.step(st, solve)
    out.update(next_positions=res.positions, next_velocities=res.velocities,
               next_accel=res.accelerations, next_iterations=res.report.iterations)
    return out


def pack_factors(f):
    blocks = f.blocks
    return dict(
        f_start=np.array([b.start for b in blocks]), f_stop=np.array([b.stop for b in blocks]),
        f_level=np.array([b.level for b in blocks]), f_tile=np.array(blocks[0].tile),
        f_anc_ptr=np.cumsum([0] + [len(b.anc) for b in blocks]),
        f_anc=np.concatenate([b.anc for b in blocks]),
        f_l11=np.concatenate([b.l11.ravel() for b in blocks]),
        f_l21=np.concatenate([b.l21.ravel() for b in blocks]),
        f_tinv=np.concatenate([np.concatenate([t.ravel() for t in b.tile_inv]) for b in blocks]),
        f_d=f.d, f_perm=f.plan.perm, f_iperm=f.plan.iperm, f_fill=np.array(f.fill_in),
    )


def ldlt_case(dims, leaf, stale_from, at, tile=16):
    """Factors of step `stale_from`'s matrix, used at step `at` (fixed staleness replay,
    as tests/test_ndprecond.py:298-328 of the reference)."""
    mesh = clamped(*dims)
    model = tetsim.make_model("corotational", mesh, PARAMS)
    integ = BackwardEulerIntegrator(mesh, model, IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    cfg = krylov.SolverConfig(1e-9, 8000)
    solve = lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)  # noqa: E731
    plan = ndprecond.expand_plan(ndprecond.nested_dissection(tetsim.vertex_adjacency(mesh), leaf))
    st = SimState.rest(mesh)
    factors = None
    for k in range(1, at):
        res = integ.step(st, solve)
        if k == stale_from:
            factors = ndprecond.ldlt_factor(res.matrix, plan, tile=tile, source_step=k)
    a, b, _ = integ.assemble_system(st)
    r = np.random.default_rng(55).standard_normal(a.nrows)
    x, rep = krylov.pcg(a, b, factors, cfg)
    fa = ndprecond.ldlt_factor(a, plan, tile=tile)
    out = dict(
        dims=np.array(dims), leaf=np.array(leaf), at=np.array(at), stale_from=np.array(stale_from),
        positions=st.positions, velocities=st.velocities, row_ptr=a.row_ptr, col_ind=a.col_ind,
        values=a.values, b=b, r=r,
        lower=ndprecond.solve_lower(factors, r), upper=ndprecond.solve_upper(factors, r),
        apply=ndprecond.apply(factors, r), x_ldlt=x, it_ldlt=rep.iterations, res_ldlt=rep.final_residual,
        fresh_d=fa.d,
    )
    out.update(pack_factors(factors))
    return out


def plan_arrays(prefix, plan):
    return {
        f"{prefix}_perm": plan.perm,
        f"{prefix}_blocks": np.array([[b.start, b.stop, b.tree_start, b.kind == "separator", b.level]
                                      for b in plan.blocks], dtype=np.int64).reshape(-1, 5),
        f"{prefix}_children": np.array([c for b in plan.blocks for c in b.children], dtype=np.int64),
        f"{prefix}_nchildren": np.array([len(b.children) for b in plan.blocks], dtype=np.int64),
    }


def nd_cases():
    out = {}
    path = tetsim.Graph(3, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]))
    out.update(plan_arrays("path3_leaf1", ndprecond.nested_dissection(path, 1)))
    k = 8
    edges = set()
    for i in range(k):
        for j in range(k):
            if i + 1 < k:
                edges |= {(i * k + j, (i + 1) * k + j), ((i + 1) * k + j, i * k + j)}
            if j + 1 < k:
                edges |= {(i * k + j, i * k + j + 1), (i * k + j + 1, i * k + j)}
    e = np.array(sorted(edges))
    indptr = np.zeros(k * k + 1, dtype=np.int64)
    np.cumsum(np.bincount(e[:, 0], minlength=k * k), out=indptr[1:])
    grid = tetsim.Graph(k * k, indptr, e[:, 1].astype(np.int64))
    out.update(plan_arrays("grid8_leaf4", ndprecond.nested_dissection(grid, 4)))
    # two disconnected components (component handling, ndprecond.py:187-196)
    two = tetsim.Graph(6, np.array([0, 1, 2, 3, 4, 5, 6]), np.array([1, 0, 3, 2, 5, 4]))
    out.update(plan_arrays("pairs_leaf1", ndprecond.nested_dissection(two, 1)))
    for dims, leaf in [((3, 3, 8), 16), ((6, 6, 28), 64), ((10, 10, 100), 64)]:
        g = tetsim.vertex_adjacency(tetsim.generate_beam(*dims, 0.1))
        name = "beam_%dx%dx%d_leaf%d" % (*dims, leaf)
        out.update(plan_arrays(name, ndprecond.nested_dissection(g, leaf)))
    return out


def main():
    meta = dict(numpy_version=np.array(np.__version__), reference=np.array("tetsim " + tetsim.__version__))
    stvk = dict(law=np.array("stvk"))
    if "--only-contact" not in sys.argv:
        np.savez_compressed(OUT / "beam_stvk.npz", **scenario_system((3, 3, 8), 6, law="stvk"), **stvk, **meta)
    if "--only-stvk" in sys.argv:
        return
    np.savez_compressed(OUT / "contact_drop.npz", **contact_case(), **meta)
    if "--only-contact" in sys.argv:
        return
    np.savez_compressed(OUT / "beam_small.npz", **scenario_system((3, 3, 8), 6, with_triplets=True), **meta)
    np.savez_compressed(OUT / "beam_cfg1.npz", **scenario_system((6, 6, 28), 6), **meta)
    np.savez_compressed(OUT / "ldlt_small.npz", **ldlt_case((4, 4, 12), 16, stale_from=4, at=7), **meta)
    np.savez_compressed(OUT / "nd_plans.npz", **nd_cases(), **meta)
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)



def contact_case(steps=14, plane_z=-0.03, dims=(3, 3, 4)):
    """Drop onto a plane through the reference's PlaneContactPipeline
    (contact.py:196-257): free beam, default gravity, LDL^T factors of the
    previous step's matrix as apply_inverse (deterministic staleness 1; CG
    compliance solves on the first step), Jacobi-PCG free motion."""
    from tetsim.contact import PlaneContactPipeline, build_compliance, detect_plane_contacts, projected_gauss_seidel

    mesh = tetsim.generate_beam(*dims, 0.1)
    model = tetsim.make_model("corotational", mesh, PARAMS)
    integ = BackwardEulerIntegrator(mesh, model, IntegratorConfig(dt=0.01))
    pipe = PlaneContactPipeline(integ, plane_z)
    cfg = krylov.SolverConfig(1e-10, 8000)
    solve = lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)  # noqa: E731
    plan = ndprecond.expand_plan(ndprecond.nested_dissection(tetsim.vertex_adjacency(mesh), 16))
    st = SimState.rest(mesh)
    out = dict(c_dims=np.array(dims), c_plane=np.array(plane_z), c_steps=np.array(steps))
    factors = None
    hist = {k: [] for k in ("ncontacts", "residual", "maxpen", "iterations")}
    first = None
    for k in range(steps):
        apply_inverse = (lambda rhs, f=factors: f.apply(rhs)) if factors is not None else None
        if first is None and factors is not None:
            free = integ.compute_step(st, solve)
            cs = detect_plane_contacts(free.positions, plane_z)
            if cs.nconstraints:
                w, s_cols = build_compliance(cs, apply_inverse)
                h = integ.config.dt
                lam = projected_gauss_seidel(h * h * w, cs.violation, cs.types)
                first = dict(c_step=np.array(k), c_x=st.positions.copy(), c_v=st.velocities.copy(),
                             c_nodes=(cs.col_ind - 2) // 3, c_violation=cs.violation, c_w=w, c_lam=lam,
                             c_free_pos=free.positions)
        info = pipe.step(st, solve, apply_inverse)
        hist["ncontacts"].append(info.ncontacts)
        hist["residual"].append(info.complementarity_residual)
        hist["maxpen"].append(info.max_penetration)
        hist["iterations"].append(info.result.report.iterations)
        factors = ndprecond.ldlt_factor(info.result.matrix, plan)
        out[f"c_pos_{k}"] = st.positions.copy()
        out[f"c_vel_{k}"] = st.velocities.copy()
    out.update({f"c_{k}": np.array(v) for k, v in hist.items()})
    out.update(first or {})
    return out


if __name__ == "__main__":
    main()
