"""The reference's element-law tests (tests/test_models.py:153-285) restated on
the device element pass: StVK at the identity, uniaxial stretch in closed
form, tangents against finite differences, symmetry, momentum conservation,
K v against the dense product of the emitted blocks, state-independent fill."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2306_05893_b200 as P  # noqa: E402
from paper_2306_05893_b200 import models as MD  # noqa: E402
from paper_2306_05893_b200.assembly import TripletStream  # noqa: E402
from paper_2306_05893_b200.mesh import Mesh  # noqa: E402

UNIT_TET = Mesh(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]), np.array([[0, 1, 2, 3]]))


def dense(fn, pre, x, ndof, **kw):
    s = TripletStream()
    s.begin_pass()
    out = fn(pre, x, stream=s, **kw)
    s.end_pass()
    k = np.zeros((ndof, ndof))
    np.add.at(k, (s.rows(), s.cols()), s.vals())
    return k, out


def fd_tangent(force, x, h):
    n = x.size
    k = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = h
        k[:, j] = (force((x.ravel() + e).reshape(x.shape)) - force((x.ravel() - e).reshape(x.shape))) / (2 * h)
    return k


def test_stvk_identity_gradient(params):
    mesh = P.generate_beam(3, 3, 8, 0.1)
    pre = MD.precompute(mesh, params)
    k, (f, _) = dense(MD.stvk_forces_and_stiffness, pre, mesh.nodes, mesh.ndof)
    assert np.abs(f).max() < 1e-9
    k_lin, _ = dense(MD.corotational_forces_and_stiffness, pre, mesh.nodes, mesh.ndof)
    assert np.allclose(k, k_lin, atol=1e-9 * np.abs(k_lin).max())


def test_stvk_uniaxial_stretch_closed_form(params):
    s_factor = 1.3
    lam, mu = params.lame_lambda, params.lame_mu
    pre = MD.precompute(UNIT_TET, params)
    x = UNIT_TET.nodes * np.array([s_factor, 1.0, 1.0])
    f, _ = MD.stvk_forces_and_stiffness(pre, x)
    s11 = lam * (s_factor ** 2 - 1) / 2 + mu * (s_factor ** 2 - 1)
    s22 = lam * (s_factor ** 2 - 1) / 2
    grads = np.linalg.inv(np.hstack([np.ones((4, 1)), UNIT_TET.nodes]))[1:, :].T
    expected = np.array([(1.0 / 6.0) * np.diag([s_factor, 1, 1]) @ np.diag([s11, s22, s22]) @ grads[a]
                         for a in range(4)])
    assert np.allclose(f.reshape(-1, 3), expected, rtol=1e-12)


@pytest.mark.parametrize("law", ["stvk", "corotational"])
def test_tangent_matches_fd(rng, params, law):
    """StVK: exact tangent at 5% strains; corotational: R Ke R^T is the tangent
    only near rest (the reference checks it at 1e-5 of the bounding box)."""
    mesh = P.generate_beam(2, 2, 3, 0.5)
    pre = MD.precompute(mesh, params)
    bbox = np.ptp(mesh.nodes)
    fn = MD.stvk_forces_and_stiffness if law == "stvk" else MD.corotational_forces_and_stiffness
    for _ in range(2):
        if law == "stvk":
            x = mesh.nodes * (1 + 0.05 * rng.standard_normal(mesh.nodes.shape))
        else:
            x = mesh.nodes + 1e-5 * bbox * rng.standard_normal(mesh.nodes.shape)
        k, _ = dense(fn, pre, x, mesh.ndof)
        k_fd = fd_tangent(lambda y: fn(pre, y)[0], x, 1e-6 * bbox)
        assert np.abs(k - k_fd).max() / np.abs(k).max() < 1e-4


def test_corotational_rest_and_rigid_rotation(params):
    mesh = P.generate_beam(3, 3, 8, 0.1)
    pre = MD.precompute(mesh, params)
    k, (f, _) = dense(MD.corotational_forces_and_stiffness, pre, mesh.nodes, mesh.ndof)
    assert np.abs(f).max() < 1e-8
    k_direct = np.zeros((mesh.ndof, mesh.ndof))
    rows, cols = pre.block_rows.reshape(pre.nelements, -1), pre.block_cols.reshape(pre.nelements, -1)
    for e in range(pre.nelements):
        np.add.at(k_direct, (rows[e], cols[e]), pre.ke[e].ravel())
    assert np.allclose(k, k_direct, atol=1e-9 * np.abs(k_direct).max())
    th = 0.9
    rot = np.array([[np.cos(th), 0, np.sin(th)], [0, 1.0, 0], [-np.sin(th), 0, np.cos(th)]])
    f, _ = MD.corotational_forces_and_stiffness(pre, mesh.nodes @ rot.T + np.array([0.3, -0.1, 0.2]))
    assert np.abs(f).max() < 1e-8 * np.abs(pre.ke).max() * np.ptp(mesh.nodes)


@pytest.mark.parametrize("law", ["corotational", "stvk"])
def test_assembled_symmetry_and_momentum(rng, params, law):
    mesh = P.generate_beam(2, 3, 3, 0.4)
    model = P.make_model(law, mesh, params)
    x = mesh.nodes + 0.01 * rng.standard_normal(mesh.nodes.shape)
    s = TripletStream()
    s.begin_pass()
    f, _ = model.accumulate(x, stream=s)
    s.end_pass()
    k = np.zeros((mesh.ndof, mesh.ndof))
    np.add.at(k, (s.rows(), s.cols()), s.vals())
    assert np.abs(k - k.T).max() < 1e-10 * np.abs(k).max()
    assert np.abs(f.reshape(-1, 3).sum(axis=0)).max() < 1e-10 * np.abs(f).sum()


@pytest.mark.parametrize("law", ["corotational", "stvk", "linear"])
def test_kv_matches_dense_product_and_fill_is_state_independent(rng, params, law):
    mesh = P.generate_beam(2, 2, 3, 0.5)
    model = P.make_model(law, mesh, params)
    x = mesh.nodes + 0.01 * rng.standard_normal(mesh.nodes.shape)
    v = rng.standard_normal(mesh.ndof)
    s = TripletStream()
    s.begin_pass()
    _, kv = model.accumulate(x, stream=s, velocities=v)
    s.end_pass()
    rows, cols = s.rows().copy(), s.cols().copy()
    k = np.zeros((mesh.ndof, mesh.ndof))
    np.add.at(k, (rows, cols), s.vals())
    assert np.allclose(kv, k @ v, rtol=1e-10, atol=1e-10 * np.abs(k @ v).max())
    s.begin_pass()
    model.accumulate(mesh.nodes + 0.1 * rng.standard_normal(mesh.nodes.shape), stream=s)
    s.end_pass()
    assert s.keep_struct is True and np.array_equal(rows, s.rows()) and np.array_equal(cols, s.cols())


def test_unknown_law_rejected(params):
    with pytest.raises(MD.ModelError, match="unknown material law"):
        P.make_model("neo-hookean", UNIT_TET, params)
