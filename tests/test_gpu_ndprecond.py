"""The reference's LDL^T tests (tests/test_ndprecond.py:125-400) on the device
refactorisation + device sweeps: hand-eliminated KATs, a random-pattern
property sweep (leaf thresholds, tiles, disconnected graphs), exactness of
the apply, and the AsyncPreconditioner(device=True) lifecycle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import tetsim_oracle as O  # noqa: E402
from paper_2306_05893_b200 import krylov, ndprecond as ND  # noqa: E402
from paper_2306_05893_b200.assembly import CsrMatrix  # noqa: E402
from paper_2306_05893_b200.mesh import Graph  # noqa: E402


def csr_from_dense(d):
    d = np.asarray(d, dtype=np.float64)
    rows, cols = np.nonzero(d)
    row_ptr = np.zeros(d.shape[0] + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=d.shape[0]), out=row_ptr[1:])
    return CsrMatrix(d.shape[0], d.shape[1], row_ptr, cols.astype(np.int64), d[rows, cols])


def random_spd(rng, n, shift):
    m = rng.standard_normal((n, n))
    return m @ m.T + shift * np.eye(n)


def test_hand_elimination_2x2_and_diagonal():
    a = csr_from_dense([[4.0, 2.0], [2.0, 3.0]])
    plan = ND.nested_dissection(ND.graph_from_pattern(a), 4)
    f = ND.ldlt_factor_device(a, plan)
    h = f.to_host()
    assert h.d == pytest.approx([4.0, 2.0], rel=1e-15)
    assert f.l_matrix.to_dense()[1, 0] == pytest.approx(0.5, rel=1e-15)
    d = csr_from_dense(np.diag([4.0, 9.0]))
    fd = ND.ldlt_factor_device(d, ND.nested_dissection(ND.graph_from_pattern(d), 4))
    assert np.allclose(np.sort(fd.to_host().d), [4.0, 9.0])


def test_random_patterns_thresholds_tiles(rng):
    for _ in range(20):
        n = int(rng.integers(2, 60))
        dense = random_spd(rng, n, shift=float(n))
        mask = rng.random((n, n)) < 0.65
        mask = mask & mask.T
        np.fill_diagonal(mask, False)
        dense[mask] = 0.0
        a = csr_from_dense(dense)
        plan = ND.nested_dissection(ND.graph_from_pattern(a), int(rng.integers(1, 8)))
        assert ND.count_coupling_violations(a, plan) == 0
        tile = int(rng.integers(1, 20))
        f = ND.ldlt_factor_device(a, plan, tile=tile)
        r = rng.standard_normal(n)
        z = ND.apply(f, r)
        assert np.abs(krylov.spmv(a, z) - r).max() / np.abs(r).max() < 1e-9
        # the block-inverse device apply of the HOST factors vs the reference's
        # tile substitution (oracle) on the same factors, within the guard's bound
        fh = ND.ldlt_factor(a, plan, tile=tile)
        zo = O.apply(fh, r)
        cond = fh.device().cond_l11
        assert cond < 1e4
        assert np.abs(ND.apply(fh, r) - zo).max() <= 1e-14 * max(cond, 10.0) * np.abs(zo).max()


def test_disconnected_graph_expanded_and_factored(rng):
    edges = [(0, 1), (1, 2), (3, 4), (4, 5), (6, 7)]  # vertex 8 isolated
    pairs = sorted({(i, j) for a_, b_ in edges for i, j in ((a_, b_), (b_, a_))})
    src = np.array([p[0] for p in pairs], dtype=np.int64)
    indptr = np.zeros(10, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=9), out=indptr[1:])
    g = Graph(n=9, indptr=indptr, indices=np.array([p[1] for p in pairs], dtype=np.int64))
    plan = ND.expand_plan(ND.nested_dissection(g, 1), 3)
    dense = np.eye(27) * 5.0
    for i, j in edges:
        for k in range(3):
            dense[3 * i + k, 3 * j + k] = dense[3 * j + k, 3 * i + k] = -1.0
    a = csr_from_dense(dense)
    f = ND.ldlt_factor_device(a, plan)
    r = rng.standard_normal(27)
    assert np.abs(krylov.spmv(a, ND.apply(f, r)) - r).max() < 1e-12
    assert np.array_equal(ND.apply(f, np.zeros(27)), np.zeros(27))
    assert r @ ND.apply(f, r) > 0.0


def test_async_device_failure_disables():
    bad = csr_from_dense([[1.0, 2.0], [2.0, 1.0]])
    plan = ND.nested_dissection(ND.graph_from_pattern(bad), 4)
    pre = ND.AsyncPreconditioner(plan, device=True)
    pre.update(bad, step=1)
    with pytest.raises(ND.LifecycleError):
        pre.wait_ready()
    assert pre.disabled and pre.status is ND.PrecondStatus.EMPTY
    pre.close()


def test_async_device_every_k_policy_and_staleness(rng):
    dense = random_spd(rng, 40, shift=40.0)
    a = csr_from_dense(dense)
    plan = ND.nested_dissection(ND.graph_from_pattern(a), 6)
    pre = ND.AsyncPreconditioner(plan, policy="every-k", refactor_every=3, device=True)
    pre.update(a, step=1)
    pre.wait_ready()
    assert pre.staleness(1) == 0 and pre.staleness(4) == 3
    pre.update(a, step=2)  # too early, no resubmission
    assert pre.refresh_in_flight is False
    pre.update(a, step=4)  # fires
    assert pre.refresh_in_flight is True
    pre.wait_ready()
    assert pre.factors.source_step == 4
    x, rep = krylov.pcg(a, rng.standard_normal(40), pre, krylov.SolverConfig(1e-9, 50))
    assert rep.converged and rep.iterations <= 2
    pre.close()


@pytest.mark.parametrize("segs", [2, 8])
def test_whole_tile_items_apply_identical(monkeypatch, segs):
    """The sweeps with whole-tiles items (several one-chunk tiles per item,
    each emitted from the warp reduction) give the apply of the chunk-item
    packing bit for bit -- the per-tile sums are the same -- and match the
    oracle."""
    import torch

    from conftest import clamped_beam
    from paper_2306_05893_b200 import _ldlt_pack as K, mesh as M

    mesh = clamped_beam(10, 10, 60)
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    out = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, mesh.nodes,
                            np.zeros_like(mesh.nodes), np.zeros(mesh.ndof), 0.01, (0.0, -9.81, 0.0))
    a = CsrMatrix(mesh.ndof, mesh.ndof, out["row_ptr"], out["col_ind"], out["values"])
    f = ND.ldlt_factor(a, ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 64)))
    monkeypatch.setattr(K, "SEGS_PER_ITEM", segs)
    r = torch.from_numpy(np.random.default_rng(5).standard_normal(mesh.ndof)).cuda()
    zs = []
    for whole in (False, True):
        monkeypatch.setattr(K, "WHOLE_ITEMS", whole)
        dev = K.DevicePanels(f)
        z = torch.empty_like(r)
        dev.run("apply", r, z)
        zs.append(z.cpu().numpy())
        del dev
    assert np.array_equal(zs[0], zs[1])
    ref = O.apply(f, r.cpu().numpy())
    assert np.abs(zs[1] - ref).max() <= 1e-12 * np.abs(ref).max()
