"""CPU check of the device block-inverse layout and the DAG item lists
(csrc/ldlt.cu, ldlt_sweep.cuh): a serial NumPy emulator executes the work
items in dispatch order with the kernel's exact data flow (row chunks for the
lower sweep, column-slab x row tiles with last-tile reduction for the upper);
it must (a) only ever find its dependencies satisfied -- the order is
topological, hence deadlock-free on the persistent kernel -- and (b)
reproduce the oracle's level-scheduled sweeps (ndprecond.py:647-691)."""

import numpy as np
import pytest

from conftest import clamped_beam
from oracle import tetsim_oracle as O
from paper_2306_05893_b200 import _ldlt_pack as K, mesh as M, ndprecond as ND
from paper_2306_05893_b200.assembly import CsrMatrix


def _g(H, b):
    B = H["blocks"][b]
    m, na = int(B["m"]), int(B["na"])
    off = K.row_offsets(m, na)
    return H["g"][B["g_off"]: B["g_off"] + off[-1]], off, m, na


def emulate_lower(H, r):
    n, nb = H["n"], H["nb"]
    blocks = H["blocks"]
    y = np.zeros(n)
    xbuf = np.zeros(n)
    cbuf = np.zeros(max(H["ncbuf"], 1))
    cnt = np.zeros(nb, dtype=np.int64)
    ready = np.zeros(nb, dtype=bool)
    for b, r0, r1, _ in H["items_l"]:
        B = blocks[b]
        s, m = int(B["start"]), int(B["m"])
        g, off, _, _ = _g(H, b)
        if B["mode"] == K.MODE_FIN:
            assert ready[b], "lower item dispatched before its block input was final"
            xs = r[s:s + m] - xbuf[s:s + m]
        elif B["mode"] == K.MODE_GATHER:
            assert cnt[b] == B["target_l"], "lower item dispatched before its children finished"
            xs = np.array([r[s + i] - cbuf[H["cin_ptr"][s + i]: H["cin_ptr"][s + i + 1]].sum() for i in range(m)])
        else:
            assert B["target_l"] == 0
            xs = r[s:s + m].copy()
        for row in range(r0, r1):
            if row < m:
                y[s + row] = xs[row] + g[off[row]: off[row] + row] @ xs[:row]
            else:
                k = row - m
                cbuf[H["cslot"][B["anc_off"] + k]] = g[off[row]: off[row] + m] @ xs
        p = int(B["parent"])
        if p >= 0:
            cnt[p] += 1
            if cnt[p] == blocks[p]["target_l"] and blocks[p]["mode"] == K.MODE_FIN:
                P = blocks[p]  # this item finalises the parent's contribution sums
                for i in range(int(P["m"])):
                    row = int(P["start"]) + i
                    xbuf[row] = cbuf[H["cin_ptr"][row]: H["cin_ptr"][row + 1]].sum()
                ready[p] = True
    assert np.all(cnt == blocks["target_l"])
    return y


def test_both_lower_input_modes_are_exercised():
    _, f = _factors((6, 6, 28), 64)
    H = K.pack(f)
    modes = set(H["blocks"]["mode"].tolist())
    assert K.MODE_LEAF in modes and K.MODE_GATHER in modes
    # force the FIN path everywhere and re-check against the oracle
    H["blocks"]["mode"][H["blocks"]["mode"] == K.MODE_GATHER] = K.MODE_FIN
    r = np.random.default_rng(3).standard_normal(f.plan.n)
    ref = O.solve_lower(f, r)
    assert np.abs(emulate_lower(H, r) - ref).max() <= 1e-12 * np.abs(ref).max()


def emulate_upper(H, w):
    n, nb = H["n"], H["nb"]
    blocks = H["blocks"]
    z = np.zeros(n)
    done = np.zeros(nb, dtype=np.int64)
    for b, c0, c1, _ in H["items_u"]:
        B = blocks[b]
        s, m, na = int(B["start"]), int(B["m"]), int(B["na"])
        toff = K.gt_row_offsets(m, na)
        gt = H["gt"][B["gt_off"]: B["gt_off"] + toff[-1]]
        if na:
            p = int(B["parent"])
            assert done[p] == blocks[p]["n_u"], "upper item dispatched before the parent's z"
        v = np.concatenate([w[s:s + m], -z[H["anc"][B["anc_off"]: B["anc_off"] + na]]])
        for c in range(c0, c1):
            z[s + c] = v[c] + gt[toff[c]: toff[c] + (m + na - 1 - c)] @ v[c + 1:]
        done[b] += 1
    assert np.all(done == blocks["n_u"])
    return z


def _factors(dims, leaf):
    mesh = clamped_beam(*dims)
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    out = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, mesh.nodes,
                            np.zeros_like(mesh.nodes), np.zeros(mesh.ndof), 0.01, (0.0, -9.81, 0.0))
    a = CsrMatrix(mesh.ndof, mesh.ndof, out["row_ptr"], out["col_ind"], out["values"])
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), leaf))
    return mesh, ND.ldlt_factor(a, plan)


@pytest.mark.parametrize("dims,leaf", [((3, 3, 8), 16), ((4, 4, 12), 16), ((6, 6, 28), 64)])
def test_block_inverse_dag_emulation_matches_oracle(dims, leaf):
    mesh, f = _factors(dims, leaf)
    H = K.pack(f)
    r = np.random.default_rng(7).standard_normal(mesh.ndof)
    y = emulate_lower(H, r)
    ref = O.solve_lower(f, r)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    z = emulate_upper(H, r)
    ref = O.solve_upper(f, r)
    assert np.abs(z - ref).max() <= 1e-12 * np.abs(ref).max()


def test_block_layout_roundtrip_and_coverage():
    _, f = _factors((4, 4, 12), 16)
    H = K.pack(f)
    for b, bf in enumerate(f.blocks):
        g, off, m, na = _g(H, b)
        linv, mm = K.unpack_block(g, m, na)
        assert np.allclose(linv @ bf.l11, np.eye(m), atol=1e-12)
        assert np.allclose(mm, bf.l21 @ linv, atol=1e-12)
        assert np.all(off % 2 == 0)  # every row 16-byte aligned (TMA / cp.async)
    # lower items cover each block's G rows exactly once
    for b in range(H["nb"]):
        B = H["blocks"][b]
        rows = sorted((r0, r1) for bb, r0, r1, _ in H["items_l"] if bb == b)
        assert rows[0][0] == 0 and rows[-1][1] == B["m"] + B["na"]
        assert all(a[1] == c[0] for a, c in zip(rows, rows[1:]))
    # upper items cover each block's columns exactly once; G^T is G transposed
    for b, bf in enumerate(f.blocks):
        B = H["blocks"][b]
        m, na = int(B["m"]), int(B["na"])
        cols = sorted((c0, c1) for bb, c0, c1, _ in H["items_u"] if bb == b)
        assert cols[0][0] == 0 and cols[-1][1] == m and all(a[1] == c[0] for a, c in zip(cols, cols[1:]))
        toff = K.gt_row_offsets(m, na)
        gt = H["gt"][B["gt_off"]: B["gt_off"] + toff[-1]]
        linv, mm = K.block_matrix(bf)
        full = np.vstack([np.tril(linv, -1), mm])
        for c in range(m):
            assert np.array_equal(gt[toff[c]: toff[c] + m + na - 1 - c], full[c + 1:, c])
        assert np.all(toff % 2 == 0)
    assert H["g"].size == sum(len(_g(H, b)[0]) for b in range(H["nb"]))


def test_device_row_offset_formulas():
    """The closed forms in csrc (g_row_off, gt_row_off) equal the packer's offsets."""
    def g_row_off(r, m):
        return (r * r) >> 1 if r < m else ((m * m) >> 1) + (r - m) * (m + (m & 1))

    def gt_row_off(c, K):
        if c <= 0:
            return 0
        a = K - c + 1
        return ((K + a) * (K - a + 1)) // 2 + ((K + 1) >> 1) - (a >> 1)

    for m in (1, 2, 3, 7, 16, 33, 128):
        for na in (0, 1, 5, 64):
            off = K.row_offsets(m, na)
            assert [g_row_off(r, m) for r in range(m + na + 1)] == off.tolist()
            toff = K.gt_row_offsets(m, na)
            assert [gt_row_off(c, m + na - 1) for c in range(m + 1)] == toff.tolist()
