"""Element physics for linear tetrahedra (drop-in for tetsim.models, models.py:1-346).

The corotational, linear and St-Venant-Kirchhoff laws run on the B200 (libtsb elem/block/node kernels, see
csrc/assemble.cu): `accumulate` returns the internal forces and K v computed
on the device and, when a TripletStream is given, the rotated element blocks
in the reference's emission order (element-major, row-major 12x12,
models.py:196-197).  Rest-state precomputation is host setup and uses the
same LAPACK calls as the reference so the device receives identical inputs.

Sign convention (models.py:3-6): M a = f_ext - f(x, v), K = df/dx.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .mesh import Mesh

__all__ = [
    "MaterialParams",
    "ElementPrecomp",
    "ModelError",
    "precompute",
    "polar_rotations",
    "corotational_forces_and_stiffness",
    "lumped_mass",
    "CorotationalModel",
    "LinearElasticModel",
    "StVenantKirchhoffModel",
    "stvk_forces_and_stiffness",
    "make_model",
]


class ModelError(ValueError):
    pass


@dataclass(frozen=True)
class MaterialParams:
    young_modulus: float
    poisson_ratio: float
    density: float

    def __post_init__(self):
        if not self.young_modulus > 0:
            raise ModelError(f"young_modulus must be positive, got {self.young_modulus}")
        if not 0.0 <= self.poisson_ratio < 0.5:
            raise ModelError(f"poisson_ratio must be in [0, 0.5), got {self.poisson_ratio}")
        if not self.density > 0:
            raise ModelError(f"density must be positive, got {self.density}")

    @property
    def lame_lambda(self) -> float:
        e, nu = self.young_modulus, self.poisson_ratio
        return e * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))

    @property
    def lame_mu(self) -> float:
        return self.young_modulus / (2.0 * (1.0 + self.poisson_ratio))


@dataclass
class ElementPrecomp:
    """Rest-state data per element (reference models.py:67-92).

    Only grads (m,4,3) and volume (m,) reach the device (104 B per tet);
    `ke`, `block_rows`, `block_cols` are materialised lazily for API users.
    """

    elements: np.ndarray
    rest_positions: np.ndarray
    grads: np.ndarray
    volume: np.ndarray
    gdof: np.ndarray
    lame: tuple
    density: float
    _ke: np.ndarray | None = field(default=None, repr=False)
    _device: object = field(default=None, repr=False)

    @property
    def nelements(self) -> int:
        return len(self.elements)

    @property
    def ke(self) -> np.ndarray:
        """Rest stiffness V * B^T C B, assembled from the closed-form 3x3 blocks."""
        if self._ke is None:
            lam, mu = self.lame
            g = self.grads
            gg = np.einsum("eai,ebi->eab", g, g)
            k = lam * np.einsum("eai,ebj->eaibj", g, g) + mu * np.einsum("eaj,ebi->eaibj", g, g)
            k += mu * np.einsum("eab,ij->eaibj", gg, np.eye(3))
            k *= self.volume[:, None, None, None, None]
            k = k.reshape(self.nelements, 12, 12)
            self._ke = 0.5 * (k + np.transpose(k, (0, 2, 1)))
        return self._ke

    @property
    def block_rows(self) -> np.ndarray:
        return np.repeat(self.gdof, 12, axis=1).ravel()

    @property
    def block_cols(self) -> np.ndarray:
        return np.tile(self.gdof, (1, 12)).ravel()


def precompute(mesh: Mesh, params: MaterialParams) -> ElementPrecomp:
    """Rest gradients and volumes (host setup; models.py:126-166).

    Same NumPy/LAPACK expressions as the reference (det and inv of the edge
    matrix) so that the device consumes bit-identical rest data.
    """
    el = mesh.elements
    p = mesh.nodes[el]
    edges_t = np.transpose(p[:, 1:] - p[:, :1], (0, 2, 1))
    det = np.linalg.det(edges_t)
    if np.any(det <= 0.0):
        bad = int(np.flatnonzero(det <= 0.0)[0])
        raise ModelError(f"element {bad} is inverted or degenerate at rest (det={det[bad]:g})")
    inv = np.linalg.inv(edges_t)
    grads = np.empty((len(el), 4, 3))
    grads[:, 1:] = inv
    grads[:, 0] = -inv.sum(axis=1)
    gdof = (3 * el[:, :, None] + np.arange(3)).reshape(len(el), 12)
    return ElementPrecomp(
        elements=el, rest_positions=mesh.nodes, grads=grads, volume=det / 6.0, gdof=gdof,
        lame=(params.lame_lambda, params.lame_mu), density=params.density,
    )


def polar_rotations(f: np.ndarray, tol: float = 1e-12, max_iter: int = 50) -> np.ndarray:
    """Rotation factor of each 3x3 F by Newton R <- (R + R^-T)/2 (host utility,
    models.py:174-189).  The device path runs the same iteration per element
    inside the assembly kernel."""
    f = np.asarray(f, dtype=np.float64)
    if not np.all(np.isfinite(f)):
        raise ModelError("non-finite deformation gradient")
    r = f.copy()
    for _ in range(max_iter):
        nxt = 0.5 * (r + np.swapaxes(np.linalg.inv(r), 1, 2))
        done = np.abs(nxt - r).max() < tol
        r = nxt
        if done:
            break
    return r


def _device_plan(precomp: ElementPrecomp, mesh: Mesh | None = None):
    from ._plan import AssemblyPlan

    if precomp._device is None:
        precomp._device = AssemblyPlan.for_model(precomp)
    return precomp._device


def _element_pass(precomp, positions, velocities, stream, law):
    if not (_lib.is_tensor(positions) or np.all(np.isfinite(positions))):
        raise ModelError("non-finite positions")
    plan = _device_plan(precomp)
    f, kv, kblocks = plan.element_pass(positions, velocities, want_blocks=stream is not None,
                                       law=law)
    if stream is not None:
        stream.add_block(precomp.block_rows, precomp.block_cols, kblocks.reshape(-1))
    return f, kv


def corotational_forces_and_stiffness(precomp: ElementPrecomp, positions, stream=None, velocities=None):
    """Corotational f = R Ke (R^T x - x0) and K v on the device (models.py:200-238).

    Returns (f, kv) as NumPy arrays for NumPy input, CUDA tensors for tensor
    input; kv is None when velocities is None.
    """
    return _element_pass(precomp, positions, velocities, stream, "corotational")


def stvk_forces_and_stiffness(precomp: ElementPrecomp, positions, stream=None, velocities=None):
    """St-Venant-Kirchhoff forces V F S g_a and K v on the device (models.py:241-287).

    Same elem/block/node kernels as the corotational law with the law switch
    set (csrc/assemble.cu): the element pass stores h_a = F g_a, F F^T and S,
    the block pass forms V(lam h_a h_b^T + mu h_b h_a^T + mu (g_a.g_b) F F^T
    + (g_a^T S g_b) I) per contribution.
    """
    return _element_pass(precomp, positions, velocities, stream, "stvk")


def lumped_mass(mesh: Mesh, params: MaterialParams, stream=None) -> np.ndarray:
    """Lumped mass rho V / 4 per tet node (host setup; models.py:290-302)."""
    share = params.density * mesh.signed_volumes() / 4.0
    gdof = (3 * mesh.elements[:, :, None] + np.arange(3)).reshape(-1)
    vals = np.repeat(share, 12)
    if stream is not None:
        stream.add_block(gdof, gdof, vals)
    return np.bincount(gdof, weights=vals, minlength=mesh.ndof)


class CorotationalModel:
    law = "corotational"

    def __init__(self, mesh: Mesh, params: MaterialParams):
        self.mesh = mesh
        self.params = params
        self.precomp = precompute(mesh, params)

    def accumulate(self, positions, stream=None, velocities=None):
        return _element_pass(self.precomp, positions, velocities, stream, self.law)

    def internal_forces(self, positions):
        return self.accumulate(positions)[0]


class LinearElasticModel(CorotationalModel):
    """Small-strain linear elasticity: the corotational kernel with R := I
    (BASELINE config 1, 'linear elastic'); f = Ke (x - x0), K = Ke."""

    law = "linear"


class StVenantKirchhoffModel(CorotationalModel):
    """St-Venant-Kirchhoff hyperelasticity (models.py:320-331): exact tangent
    with material and geometric parts, assembled by the same device kernels."""

    law = "stvk"


_MODEL_CLASSES = {
    CorotationalModel.law: CorotationalModel,
    LinearElasticModel.law: LinearElasticModel,
    StVenantKirchhoffModel.law: StVenantKirchhoffModel,
}


def make_model(law: str, mesh: Mesh, params: MaterialParams):
    try:
        cls = _MODEL_CLASSES[law]
    except KeyError:
        raise ModelError(f"unknown material law {law!r}; expected one of {sorted(_MODEL_CLASSES)}") from None
    return cls(mesh, params)
