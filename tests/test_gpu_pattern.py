"""GPU pattern build (csrc/pattern.cu) == the host topology pattern == the
reference's triplet-built pattern (build_pattern, assembly.py:235-312)."""

import numpy as np
import pytest

from conftest import clamped_beam

pytestmark = pytest.mark.gpu

from paper_2306_05893_b200 import _plan  # noqa: E402
from paper_2306_05893_b200.mesh import Mesh  # noqa: E402


@pytest.mark.parametrize("dims", [(3, 3, 8), (6, 6, 28), (10, 10, 100)])
def test_device_pattern_equals_host_pattern(dims):
    mesh = clamped_beam(*dims)
    h = _plan.topology_pattern(mesh)
    d = _plan.device_topology_pattern(mesh)
    for k in ("row_ptr", "col_ind", "fixed_diag_slots", "blk", "blk_list", "node_ptr", "node_list"):
        assert np.array_equal(np.asarray(h[k]), np.asarray(d[k])), k


def test_device_pattern_matches_reference_golden(golden):
    g = golden("beam_small")
    mesh = clamped_beam(*map(int, g["dims"]))
    d = _plan.device_topology_pattern(mesh)
    assert np.array_equal(d["row_ptr"], g["row_ptr"]) and np.array_equal(d["col_ind"], g["col_ind"])
    assert np.array_equal(d["fixed_diag_slots"], g["fixed_diag_slots"])


def test_device_pattern_unpinned_and_shuffled_mesh():
    mesh = clamped_beam(4, 3, 6)
    rng = np.random.default_rng(7)
    perm = rng.permutation(mesh.node_count)
    inv = np.argsort(perm)
    el = inv[mesh.elements][rng.permutation(mesh.element_count)]
    m2 = Mesh(mesh.nodes[perm], el).with_fixed_nodes(inv[mesh.fixed_nodes[:3]])
    h = _plan.topology_pattern(m2)
    d = _plan.device_topology_pattern(m2)
    for k in ("row_ptr", "col_ind", "blk", "blk_list", "node_ptr", "node_list"):
        assert np.array_equal(np.asarray(h[k]), np.asarray(d[k])), k
