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
    part = np.zeros(max(H["npart"], 1))
    cnt_s = np.zeros(H["n_slabs"], dtype=np.int64)
    done = np.zeros(nb, dtype=np.int64)
    for b, slab, ra, rb, tile, has_dep, _, _ in H["items_u"]:
        B = blocks[b]
        s, m, sw = int(B["start"]), int(B["m"]), int(B["sw"])
        g, off, _, _ = _g(H, b)
        c0 = (slab - int(B["slab_base"])) * sw
        cw = min(sw, m - c0)
        if has_dep:
            p = int(B["parent"])
            assert done[p] == blocks[p]["nslabs"], "upper M tile dispatched before the parent's z"
        acc = np.zeros(cw)
        for row in range(ra, rb):
            if row < m:
                v = w[s + row]
                hi = min(c0 + cw, row)
                if hi > c0:
                    acc[: hi - c0] += g[off[row] + c0: off[row] + hi] * v
            else:
                v = -z[H["anc"][B["anc_off"] + row - m]]
                acc += g[off[row] + c0: off[row] + c0 + cw] * v
        part[H["slab_part"][slab] + tile * sw: H["slab_part"][slab] + tile * sw + cw] = acc
        cnt_s[slab] += 1
        if cnt_s[slab] == H["slab_ntiles"][slab]:
            nt = int(H["slab_ntiles"][slab])
            tot = sum(part[H["slab_part"][slab] + t * sw: H["slab_part"][slab] + t * sw + cw] for t in range(nt))
            z[s + c0: s + c0 + cw] = w[s + c0: s + c0 + cw] + tot
            done[b] += 1
    assert np.all(done == blocks["nslabs"])
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
    # every slab has at least one tile and the tile ids are 0..ntiles-1
    for sid in range(H["n_slabs"]):
        t = sorted(x[4] for x in H["items_u"] if x[1] == sid)
        assert t == list(range(H["slab_ntiles"][sid]))
    assert H["g"].size == sum(len(_g(H, b)[0]) for b in range(H["nb"]))
