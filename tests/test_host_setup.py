"""Host-side setup of the product (mesh, pattern, ordering, factorisation)
against the reference's golden outputs and known-answer tests.  CPU only
(the ordering runs in libtsb's host code; no GPU call)."""

import numpy as np
import pytest

from conftest import GoldenFactors, clamped_beam
from oracle import tetsim_oracle as O
from paper_2306_05893_b200 import _plan, assembly, mesh as M, ndprecond as ND
from paper_2306_05893_b200.assembly import CsrMatrix, TripletStream, build_pattern


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_generate_beam_bit_identical(golden, name):
    g = golden(name)
    mesh = M.generate_beam(*map(int, g["dims"]), 0.1)
    assert np.array_equal(mesh.nodes, g["nodes"])
    assert np.array_equal(mesh.elements, g["elements"])


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_topology_pattern_is_reference_pattern(golden, name):
    g = golden(name)
    mesh = clamped_beam(*map(int, g["dims"]))
    p = _plan.topology_pattern(mesh)
    assert np.array_equal(p["row_ptr"], g["row_ptr"])
    assert np.array_equal(p["col_ind"], g["col_ind"])
    assert np.array_equal(p["fixed_diag_slots"], g["fixed_diag_slots"])


def test_block_lists_reproduce_reference_slots(golden):
    """Every stiffness triplet lands, through the block gather lists, in the
    slot the reference mapping assigns it (assembly.py:293-297)."""
    g = golden("beam_small")
    mesh = clamped_beam(*map(int, g["dims"]))
    p = _plan.topology_pattern(mesh)
    m = mesh.element_count
    sot = g["slot_of_triplet"][12 * m:].reshape(m, 4, 3, 4, 3)
    got = np.full((m, 4, 3, 4, 3), -1, dtype=np.int64)
    for s0, rl, lo, hi in p["blk"]:
        for c in p["blk_list"][lo:hi]:
            e, a, b = c >> 4, (c >> 2) & 3, c & 3
            for i in range(3):
                for j in range(3):
                    got[e, a, i, b, j] = s0 + i * rl + j
    assert np.array_equal(got, sot)
    # mass triplets: diagonal slots of the diagonal blocks
    ms = g["slot_of_triplet"][: 12 * m].reshape(m, 4, 3)
    for e in range(m):
        for a in range(4):
            for i in range(3):
                assert ms[e, a, i] == -1 or ms[e, a, i] == sot[e, a, i, a, i]


def test_build_pattern_matches_reference_mapping(golden):
    g = golden("beam_small")
    s = TripletStream()
    s.begin_pass()
    s.add_block(g["trip_rows"], g["trip_cols"], g["trip_vals"])
    s.end_pass()
    n = 3 * len(g["nodes"])
    fixed = (3 * g["fixed_nodes"][:, None] + np.arange(3)).ravel()
    _, mp = build_pattern(s, n, fixed)
    assert np.array_equal(mp.row_ptr, g["row_ptr"])
    assert np.array_equal(mp.col_ind, g["col_ind"])
    assert np.array_equal(mp.slot_of_triplet, g["slot_of_triplet"])
    assert np.array_equal(mp.kept, g["kept"])
    assert np.array_equal(mp.fixed_diag_slots, g["fixed_diag_slots"])


def test_build_pattern_known_answers():
    # duplicate merge -> slots [0, 1, 0] (reference tests/test_assembly.py:136-145)
    s = TripletStream()
    s.begin_pass()
    for r, c in [(0, 0), (0, 1), (0, 0)]:
        s.add(r, c, 1.0)
    s.end_pass()
    _, mp = build_pattern(s, 2)
    assert mp.slot_of_triplet.tolist() == [0, 1, 0]
    # pinned filter (test_assembly.py:147-158)
    s = TripletStream()
    s.begin_pass()
    for r, c in [(0, 0), (0, 1), (1, 1), (1, 0)]:
        s.add(r, c, 2.0)
    s.end_pass()
    _, mp = build_pattern(s, 2, fixed_dofs=[0])
    assert mp.slot_of_triplet.tolist() == [-1, -1, 1, -1]
    assert mp.fixed_diag_slots.tolist() == [0]
    # out-of-range triplet is named (test_assembly.py:160-167)
    s = TripletStream()
    s.begin_pass()
    s.add(0, 5, 1.0)
    s.end_pass()
    with pytest.raises(assembly.AssemblyError, match="triplet 0"):
        build_pattern(s, 3)


def test_random_stream_pattern_vs_sort_merge(rng):
    n = 40
    rows = rng.integers(0, n, 500)
    cols = rng.integers(0, n, 500)
    fixed = [3, 17]
    s = TripletStream()
    s.begin_pass()
    s.add_block(rows, cols, rng.standard_normal(500))
    s.end_pass()
    _, mp = build_pattern(s, n, fixed)
    rp, ci, slot, fs = O.sort_merge_pattern(rows, cols, n, fixed)
    assert np.array_equal(mp.row_ptr, rp) and np.array_equal(mp.col_ind, ci)
    assert np.array_equal(mp.slot_of_triplet, slot) and np.array_equal(mp.fixed_diag_slots, fs)


def test_triplet_stream_keep_struct():
    s = TripletStream()
    s.begin_pass()
    s.add_block(np.array([0, 1]), np.array([0, 1]), np.array([1.0, 2.0]))
    s.end_pass()
    assert not s.keep_struct
    s.begin_pass()
    s.add_block(np.array([0, 1]), np.array([0, 1]), np.array([3.0, 4.0]))
    s.end_pass()
    assert s.keep_struct and s.vals().tolist() == [3.0, 4.0]
    s.begin_pass()
    s.add(0, 0, 1.0)
    s.end_pass()
    assert not s.keep_struct


def _plan_from_golden(g, prefix):
    blocks = g[f"{prefix}_blocks"]
    nch = g[f"{prefix}_nchildren"]
    ch = g[f"{prefix}_children"]
    out, k = [], 0
    for row, c in zip(blocks, nch):
        out.append((int(row[0]), int(row[1]), int(row[2]), "separator" if row[3] else "leaf",
                    tuple(int(v) for v in ch[k:k + c]), int(row[4])))
        k += c
    return g[f"{prefix}_perm"], out


def _grid(k):
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
    return M.Graph(k * k, indptr, e[:, 1].astype(np.int64))


@pytest.mark.parametrize("prefix,graph,leaf", [
    ("path3_leaf1", lambda: M.Graph(3, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1])), 1),
    ("grid8_leaf4", lambda: _grid(8), 4),
    ("pairs_leaf1", lambda: M.Graph(6, np.arange(7), np.array([1, 0, 3, 2, 5, 4])), 1),
    ("beam_3x3x8_leaf16", lambda: M.vertex_adjacency(M.generate_beam(3, 3, 8, 0.1)), 16),
    ("beam_6x6x28_leaf64", lambda: M.vertex_adjacency(M.generate_beam(6, 6, 28, 0.1)), 64),
    ("beam_10x10x100_leaf64", lambda: M.vertex_adjacency(M.generate_beam(10, 10, 100, 0.1)), 64),
])
def test_nested_dissection_identical_to_reference(golden, prefix, graph, leaf):
    g = golden("nd_plans")
    perm, blocks = _plan_from_golden(g, prefix)
    plan = ND.nested_dissection(graph(), leaf)
    assert np.array_equal(plan.perm, perm)
    got = [(b.start, b.stop, b.tree_start, b.kind, b.children, b.level) for b in plan.blocks]
    assert got == blocks


def test_nested_dissection_known_answers():
    path = M.Graph(3, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]))
    plan = ND.nested_dissection(path, 1)
    assert plan.perm.tolist() == [0, 2, 1]  # reference tests/test_ndprecond.py:43-51
    ex = ND.expand_plan(plan)
    assert ex.perm.tolist() == [0, 1, 2, 6, 7, 8, 3, 4, 5]  # test_ndprecond.py:116-121
    with pytest.raises(ND.PrecondError):
        ND.nested_dissection(path, 0)


def test_ldlt_factor_matches_reference_factors(golden):
    g = golden("ldlt_small")
    ref = GoldenFactors(g)
    mesh = clamped_beam(*map(int, g["dims"]))
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), int(g["leaf"])))
    assert np.array_equal(plan.perm, g["f_perm"])
    # rebuild the stale matrix's factor input: refactor the golden system itself
    a = CsrMatrix(len(g["b"]), len(g["b"]), g["row_ptr"], g["col_ind"], g["values"])
    f = ND.ldlt_factor(a, plan, tile=16)
    assert np.abs(f.d - g["fresh_d"]).max() <= 1e-12 * np.abs(g["fresh_d"]).max()
    assert [(b.start, b.stop, b.level) for b in f.blocks] == [(b.start, b.stop, b.level) for b in ref.blocks]
    assert all(np.array_equal(x.anc, y.anc) for x, y in zip(f.blocks, ref.blocks))
    # apply of our host factor vs a dense solve
    r = g["r"]
    z = O.apply(f, r)
    dense = a.to_dense()
    x = np.linalg.solve(dense, r)
    assert np.abs(z - x).max() <= 1e-10 * np.abs(x).max()


def test_ldlt_two_by_two_known_answer():
    a = CsrMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([4.0, 2.0, 2.0, 3.0]))
    plan = ND.DissectionPlan(2, np.array([0, 1]), np.array([0, 1]),
                             (ND.Block(0, 2, 0, "leaf", (), 0),), ((0,),), 64)
    f = ND.ldlt_factor(a, plan)
    assert np.allclose(f.d, [4.0, 2.0])  # reference tests/test_ndprecond.py:132-138
    assert f.blocks[0].l11[1, 0] == pytest.approx(0.5)


def test_ldlt_indefinite_raises():
    a = CsrMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([1.0, 2.0, 2.0, 1.0]))
    plan = ND.DissectionPlan(2, np.array([0, 1]), np.array([0, 1]),
                             (ND.Block(0, 2, 0, "leaf", (), 0),), ((0,),), 64)
    with pytest.raises(ND.IndefiniteMatrixError):
        ND.ldlt_factor(a, plan)


def test_coupling_violations_zero_on_beam(golden):
    g = golden("beam_cfg1")
    mesh = clamped_beam(*map(int, g["dims"]))
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 64))
    a = CsrMatrix(len(g["b"]), len(g["b"]), g["row_ptr"], g["col_ind"], g["values"])
    assert ND.count_coupling_violations(a, plan) == 0


def test_fill_in_counts_without_materialising(golden):
    """LdlFactors.fill_in (counted per block) equals the nnz of l_matrix."""
    g = golden("ldlt_small")
    mesh = clamped_beam(*map(int, g["dims"]))
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), int(g["leaf"])))
    a = CsrMatrix(len(g["b"]), len(g["b"]), g["row_ptr"], g["col_ind"], g["values"])
    f = ND.ldlt_factor(a, plan, tile=16)
    n0 = f.fill_in
    assert n0 == f.l_matrix.nnz == int(g["f_fill"])
