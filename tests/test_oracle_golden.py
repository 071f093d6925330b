"""Pin the CPU oracle against the reference's own outputs (tests/golden, made by
tests/golden/make_golden.py from /root/reference).  CPU only."""

import numpy as np
import pytest

from conftest import GoldenFactors
from oracle import tetsim_oracle as O

G = 9.81


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_spmv_bit_exact(golden, name):
    g = golden(name)
    y = O.spmv(g["row_ptr"], g["col_ind"], g["values"], g["spmv_x"])
    assert np.array_equal(y, g["spmv_y"])


def test_compress_bit_exact(golden):
    g = golden("beam_small")
    vals = O.compress(g["trip_vals"], g["kept"], g["kept_slots"], len(g["col_ind"]),
                      g["fixed_diag_slots"], g["coeffs"])
    assert np.array_equal(vals, g["values"])


def test_sort_merge_pattern_matches_reference_mapping(golden):
    g = golden("beam_small")
    n = 3 * len(g["nodes"])
    fixed = (3 * g["fixed_nodes"][:, None] + np.arange(3)).ravel()
    rp, ci, slot, fs = O.sort_merge_pattern(g["trip_rows"], g["trip_cols"], n, fixed)
    assert np.array_equal(rp, g["row_ptr"])
    assert np.array_equal(ci, g["col_ind"])
    assert np.array_equal(slot, g["slot_of_triplet"])
    assert np.array_equal(fs, g["fixed_diag_slots"])


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_rest_data_matches_reference(golden, name):
    g = golden(name)
    rest = O.rest_data(g["nodes"], g["elements"], 1e5, 0.3, 1000.0)
    assert np.array_equal(rest["grads"], g["grads"])
    assert np.array_equal(rest["vol"], g["volume"])
    assert np.array_equal(rest["ke"], g["ke"])


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_assemble_system_matches_reference(golden, name):
    g = golden(name)
    rest = O.rest_data(g["nodes"], g["elements"], 1e5, 0.3, 1000.0)
    out = O.assemble_system(g["nodes"], g["elements"], g["fixed_nodes"], rest, g["positions"],
                            g["velocities"], g["f_ext_state"], 0.01, (0.0, -G, 0.0))
    assert np.array_equal(out["row_ptr"], g["row_ptr"])
    assert np.array_equal(out["col_ind"], g["col_ind"])
    # same NumPy/BLAS calls in the same order: bit-identical in this container
    assert np.array_equal(out["values"], g["values"])
    assert np.array_equal(out["b"], g["b"])
    assert np.array_equal(out["f_int"], g["f_int"])
    assert np.array_equal(out["f_ext"], g["f_ext"])


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_pcg_matches_reference(golden, name):
    g = golden(name)
    n = len(g["b"])
    inv = O.jacobi_inv_diag(g["row_ptr"], g["col_ind"], g["values"], n)
    x, it, res, conv = O.pcg(g["row_ptr"], g["col_ind"], g["values"], g["b"], lambda r: r * inv,
                             tol=1e-9, max_it=8000)
    assert conv and it == int(g["it_jacobi"])
    assert np.array_equal(x, g["x_jacobi"])
    x, it, res, conv = O.pcg(g["row_ptr"], g["col_ind"], g["values"], g["b"], None, tol=1e-9, max_it=8000)
    assert it == int(g["it_cg"]) and res == float(g["res_cg"])
    assert np.array_equal(x, g["x_cg"])


def test_ldlt_solves_match_reference(golden):
    g = golden("ldlt_small")
    f = GoldenFactors(g)
    assert np.array_equal(O.solve_lower(f, g["r"]), g["lower"])
    assert np.array_equal(O.solve_upper(f, g["r"]), g["upper"])
    assert np.array_equal(O.apply(f, g["r"]), g["apply"])
    x, it, res, conv = O.pcg(g["row_ptr"], g["col_ind"], g["values"], g["b"], lambda r: O.apply(f, r),
                             tol=1e-9, max_it=8000)
    assert conv and it == int(g["it_ldlt"])
    assert np.array_equal(x, g["x_ldlt"])


def test_textbook_substitution_agrees_with_level_solves(golden):
    g = golden("ldlt_small")
    f = GoldenFactors(g)
    n = len(g["r"])
    rows, cols, vals = [], [], []
    for b in f.blocks:
        m = b.stop - b.start
        ir, ic = np.tril_indices(m, -1)
        rows.append(b.start + ir), cols.append(b.start + ic), vals.append(b.l11[ir, ic])
        if len(b.anc):
            rows.append(np.repeat(b.anc, m)), cols.append(np.tile(np.arange(b.start, b.stop), len(b.anc)))
            vals.append(b.l21.ravel())
    rows, cols, vals = map(np.concatenate, (rows, cols, vals))
    o = np.lexsort((cols, rows))
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    y = O.forward_substitution(rp, cols[o], vals[o], g["r"])
    assert np.abs(y - g["lower"]).max() <= 1e-12 * np.abs(y).max()
    z = O.backward_substitution(rp, cols[o], vals[o], g["r"])
    assert np.abs(z - g["upper"]).max() <= 1e-12 * np.abs(z).max()


def test_corotational_kv_matches_reference(golden):
    g = golden("beam_cfg1")
    rest = O.rest_data(g["nodes"], g["elements"], 1e5, 0.3, 1000.0)
    f, kv, _ = O.corotational(g["nodes"], g["elements"], rest, g["positions"], g["velocities"])
    assert np.array_equal(kv, g["kv"])
    assert np.array_equal(f, g["f_int"])


def test_stvk_assembly_matches_reference(golden):
    """St-Venant-Kirchhoff law (models.py:241-287) through the fused assembly."""
    g = golden("beam_stvk")
    rest = O.rest_data(g["nodes"], g["elements"], 1e5, 0.3, 1000.0)
    out = O.assemble_system(g["nodes"], g["elements"], g["fixed_nodes"], rest, g["positions"], g["velocities"],
                            g["f_ext_state"], 0.01, (0.0, -G, 0.0), law="stvk")
    assert np.array_equal(out["row_ptr"], g["row_ptr"]) and np.array_equal(out["col_ind"], g["col_ind"])
    scale = np.abs(g["values"]).max()
    assert np.abs(out["values"] - g["values"]).max() <= 1e-12 * scale
    assert np.abs(out["b"] - g["b"]).max() <= 1e-12 * np.abs(g["b"]).max()
    assert np.abs(out["f_int"] - g["f_int"]).max() <= 1e-12 * np.abs(g["f_int"]).max()
    _, kv, _ = O.stvk(g["nodes"], g["elements"], rest, g["positions"], g["velocities"])
    assert np.abs(kv - g["kv"]).max() <= 1e-12 * np.abs(g["kv"]).max()


def test_contact_stage_matches_reference(golden):
    """First contact step of the reference's drop scenario (contact_drop.npz):
    free motion, detection, compliance with LDL^T factors of the previous
    step's matrix, PGS multipliers, corrected state (contact.py:89-257)."""
    from paper_2306_05893_b200 import mesh as M, ndprecond as ND
    from paper_2306_05893_b200.assembly import CsrMatrix

    g = golden("contact_drop")
    k = int(g["c_step"])
    dims = tuple(int(v) for v in g["c_dims"])
    plane = float(g["c_plane"])
    import paper_2306_05893_b200 as P

    mesh = P.generate_beam(*dims, 0.1)
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    nofix = np.zeros(0, dtype=np.int64)
    grav = (0.0, 0.0, -G)

    def system(x, v):
        return O.assemble_system(mesh.nodes, mesh.elements, nofix, rest, x, v, np.zeros(mesh.ndof), 0.01, grav)

    prev = system(g[f"c_pos_{k - 2}"], g[f"c_vel_{k - 2}"])
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), 16))
    f = ND.ldlt_factor(CsrMatrix(mesh.ndof, mesh.ndof, prev["row_ptr"], prev["col_ind"], prev["values"]), plan)
    x0, v0 = g["c_x"], g["c_v"]
    assert np.array_equal(x0, g[f"c_pos_{k - 1}"])
    cur = system(x0, v0)
    inv = O.jacobi_inv_diag(cur["row_ptr"], cur["col_ind"], cur["values"], mesh.ndof)
    acc, it, _, _ = O.pcg(cur["row_ptr"], cur["col_ind"], cur["values"], cur["b"], lambda r: r * inv, 1e-10, 8000)
    assert it == int(g["c_iterations"][k])
    pos, vel, acc = O.advance(acc, x0, v0, 0.01, nofix)
    assert np.abs(pos - g["c_free_pos"]).max() <= 1e-12
    nodes, cols, coefs, viol = O.detect_plane_contacts(pos, plane)
    assert np.array_equal(nodes, g["c_nodes"]) and np.abs(viol - g["c_violation"]).max() <= 1e-15
    w, s = O.build_compliance(cols, coefs, mesh.ndof, lambda e: O.apply(f, e))
    assert np.abs(w - g["c_w"]).max() <= 1e-12 * np.abs(g["c_w"]).max()
    lam = O.projected_gauss_seidel(0.01 ** 2 * w, viol, np.ones(len(viol), dtype=bool))
    assert np.abs(lam - g["c_lam"]).max() <= 1e-10 * np.abs(g["c_lam"]).max()
    pos2, vel2, _ = O.advance(acc.reshape(-1, 3) - (s @ lam).reshape(-1, 3), x0, v0, 0.01, nofix)
    assert np.abs(pos2 - g[f"c_pos_{k}"]).max() <= 1e-12
    assert np.abs(vel2 - g[f"c_vel_{k}"]).max() <= 1e-10 * np.abs(g[f"c_vel_{k}"]).max()


# ---------------------------------------------------------------------------
# oracle/tetsim_nd.py: mesh, dissection and factorisation restated for the
# reference arm of bench.py (which must not import the product package)
# ---------------------------------------------------------------------------

from oracle import tetsim_nd as OND  # noqa: E402


def _golden_plan(g, prefix):
    blocks, nch, ch = g[f"{prefix}_blocks"], g[f"{prefix}_nchildren"], g[f"{prefix}_children"]
    out, k = [], 0
    for row, c in zip(blocks, nch):
        out.append((int(row[0]), int(row[1]), int(row[2]), "separator" if row[3] else "leaf",
                    tuple(int(v) for v in ch[k:k + c]), int(row[4])))
        k += c
    return g[f"{prefix}_perm"], out


def _grid_graph(k):
    src, dst = [], []
    for i in range(k):
        for j in range(k):
            v = i * k + j
            for w in ([v - k] if i else []) + ([v - 1] if j else []) + ([v + 1] if j + 1 < k else []) \
                    + ([v + k] if i + 1 < k else []):
                src.append(v)
                dst.append(w)
    indptr = np.zeros(k * k + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=k * k), out=indptr[1:])
    return indptr, np.array(dst, dtype=np.int64)


def _beam_graph(dims):
    nodes, el = OND.generate_beam(*dims, 0.1)
    return OND.vertex_adjacency(len(nodes), el)


@pytest.mark.parametrize("prefix,graph,leaf", [
    ("path3_leaf1", lambda: (np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1])), 1),
    ("grid8_leaf4", lambda: _grid_graph(8), 4),
    ("pairs_leaf1", lambda: (np.arange(7), np.array([1, 0, 3, 2, 5, 4])), 1),
    ("beam_3x3x8_leaf16", lambda: _beam_graph((3, 3, 8)), 16),
    ("beam_6x6x28_leaf64", lambda: _beam_graph((6, 6, 28)), 64),
    ("beam_10x10x100_leaf64", lambda: _beam_graph((10, 10, 100)), 64),
])
def test_oracle_nested_dissection_identical_to_reference(golden, prefix, graph, leaf):
    perm, blocks = _golden_plan(golden("nd_plans"), prefix)
    plan = OND.nested_dissection(*graph(), leaf)
    assert np.array_equal(plan.perm, perm)
    assert [(b.start, b.stop, b.tree_start, b.kind, b.children, b.level) for b in plan.blocks] == blocks


@pytest.mark.parametrize("name", ["beam_small", "beam_cfg1"])
def test_oracle_beam_matches_reference(golden, name):
    g = golden(name)
    nodes, el = OND.generate_beam(*map(int, g["dims"]), 0.1)
    assert np.array_equal(nodes, g["nodes"]) and np.array_equal(el, g["elements"])
    assert np.array_equal(OND.clamped_nodes(nodes), g["fixed_nodes"])


def test_oracle_ldlt_factor_matches_reference(golden):
    """Factors of the golden system vs the reference's fresh d, and the stale
    factors' apply of the golden (reference) run: same blocks, same apply."""
    g = golden("ldlt_small")
    ref = GoldenFactors(g)
    nodes, el = OND.generate_beam(*map(int, g["dims"]), 0.1)
    plan = OND.expand_plan(OND.nested_dissection(*OND.vertex_adjacency(len(nodes), el), int(g["leaf"])))
    assert np.array_equal(plan.perm, g["f_perm"])
    f = OND.ldlt_factor(g["row_ptr"], g["col_ind"], g["values"], plan, tile=16)
    assert np.abs(f.d - g["fresh_d"]).max() <= 1e-13 * np.abs(g["fresh_d"]).max()
    assert [(b.start, b.stop, b.level) for b in f.blocks] == [(b.start, b.stop, b.level) for b in ref.blocks]
    assert all(np.array_equal(x.anc, y.anc) for x, y in zip(f.blocks, ref.blocks))
    z = O.apply(f, g["r"])
    x = np.linalg.solve(_dense(g), g["r"])
    assert np.abs(z - x).max() <= 1e-10 * np.abs(x).max()


def test_oracle_ldlt_factor_reproduces_reference_stale_factors(golden):
    """Re-run the reference's stale-factor case end to end with the oracle:
    scenario steps 1..at-1, factor at step stale_from, PCG at step at."""
    g = golden("ldlt_small")
    dims = tuple(map(int, g["dims"]))
    nodes, el = OND.generate_beam(*dims, 0.1)
    fixed = OND.clamped_nodes(nodes)
    plan = OND.expand_plan(OND.nested_dissection(*OND.vertex_adjacency(len(nodes), el), int(g["leaf"])))
    rest = O.rest_data(nodes, el, 1e5, 0.3, 1000.0)
    x, v, fe = nodes.copy(), np.zeros_like(nodes), np.zeros(3 * len(nodes))
    f = None
    for k in range(1, int(g["at"])):
        out = O.assemble_system(nodes, el, fixed, rest, x, v, fe, 0.01, (0.0, -G, 0.0))
        inv = O.jacobi_inv_diag(out["row_ptr"], out["col_ind"], out["values"], len(out["b"]))
        acc, _, _, conv = O.pcg(out["row_ptr"], out["col_ind"], out["values"], out["b"], lambda r: r * inv)
        assert conv
        if k == int(g["stale_from"]):
            f = OND.ldlt_factor(out["row_ptr"], out["col_ind"], out["values"], plan, tile=16)
        x, v, _ = O.advance(acc, x, v, 0.01, fixed)
    assert np.abs(x - g["positions"]).max() <= 1e-10 * np.abs(g["positions"]).max()
    for bf, rb in zip(f.blocks, GoldenFactors(g).blocks):
        assert np.abs(bf.l11 - rb.l11).max() <= 1e-11 and (not len(rb.anc) or np.abs(bf.l21 - rb.l21).max() <= 1e-11)
    out = O.assemble_system(nodes, el, fixed, rest, x, v, fe, 0.01, (0.0, -G, 0.0))
    sol, it, _, conv = O.pcg(out["row_ptr"], out["col_ind"], out["values"], out["b"], lambda r: O.apply(f, r))
    assert conv and it == int(g["it_ldlt"])
    assert np.abs(sol - g["x_ldlt"]).max() <= 1e-10 * np.abs(g["x_ldlt"]).max()


def _dense(g):
    n = len(g["b"])
    d = np.zeros((n, n))
    d[np.repeat(np.arange(n), np.diff(g["row_ptr"])), g["col_ind"]] = g["values"]
    return d
