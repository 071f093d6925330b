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


def _tile(H, up, t):
    """(block rows, dense tile rows over v-columns [tl, tl + 2 np), tl) of tile t."""
    T = H["tiles_u" if up else "tiles_l"][t]
    data = H["gt" if up else "g"]
    npair = int(T["np"])
    d = data[T["off"]: T["off"] + npair * K.TILE * 2].reshape(npair, K.TILE, 2).transpose(1, 0, 2)
    d = d.reshape(K.TILE, 2 * npair)[: T["nrows"]]
    return np.arange(T["row0"], T["row0"] + T["nrows"]), d, int(T["tl"])


def _padded(v, upto):
    out = np.zeros(max(upto, len(v)))
    out[: len(v)] = v
    return out


def emulate_lower(H, r):
    n, nb = H["n"], H["nb"]
    blocks = H["blocks"]
    y = np.zeros(n)
    xbuf = np.zeros(n)
    cbuf = np.zeros(max(H["ncbuf"], 1))
    cnt = np.zeros(nb, dtype=np.int64)
    ready = np.zeros(nb, dtype=np.int64)
    segs = np.zeros(len(H["tiles_l"]), dtype=np.int64)
    csum = lambda row: cbuf[H["cin_ptr"][row]: H["cin_ptr"][row + 1]].sum()  # noqa: E731
    for b, t0, t1, sg in H["items_l"]:
        B = blocks[b]
        s, m = int(B["start"]), int(B["m"])
        if sg < 0:  # finaliser item: x_b over rows [t0, t1) once the children are done
            assert B["mode"] == K.MODE_FIN and cnt[b] == B["target_l"], "finaliser before the children"
            for i in range(t0, t1):
                xbuf[s + i] = r[s + i] - csum(s + i)
            ready[b] += 1
            continue
        if B["mode"] == K.MODE_FIN:
            assert ready[b] == B["nfin"], "lower item dispatched before its block input was final"
            xs = xbuf[s:s + m].copy()
        elif B["mode"] == K.MODE_GATHER:
            assert cnt[b] == B["target_l"], "lower item dispatched before its children finished"
            xs = np.array([r[s + i] - csum(s + i) for i in range(m)])
        else:
            assert B["target_l"] == 0
            xs = r[s:s + m].copy()
        for t in ([t0] if 0 < sg < K.WHOLE else range(t0, t1)):
            if sg == K.WHOLE:  # whole-tiles item: each tile complete (one chunk)
                segs[t] += H["tiles_l"]["nseg"][t]
            elif sg:  # segment item: the tile's rows are emitted by its last segment
                segs[t] += 1
                if segs[t] < H["tiles_l"]["nseg"][t]:
                    continue
            rows, d, tl = _tile(H, False, t)
            vals = d @ _padded(xs, tl + d.shape[1])[tl: tl + d.shape[1]]
            for row, a in zip(rows, vals):
                if row < m:
                    y[s + row] = a  # unit diagonal stored: y_r = sum_{j <= r} Linv_rj x_j
                else:
                    cbuf[H["cslot"][B["anc_off"] + row - m]] = a
        p = int(B["parent"])
        if p >= 0:
            cnt[p] += 1
    assert np.all(cnt == blocks["target_l"])
    assert np.array_equal(segs, H["tiles_l"]["nseg"])
    emulate_lower.cbuf = cbuf
    return y


def test_all_lower_input_modes_are_exercised(monkeypatch):
    _, f = _factors((10, 10, 60), 64)
    for ratio in (1.0, 0.5, 0.25, 0.1):  # a gather/finaliser threshold that splits the inner blocks
        monkeypatch.setattr(K, "GATHER_RATIO", ratio)
        H = K.pack(f)
        if len(set(H["blocks"]["mode"].tolist())) == 3:
            break
    modes = set(H["blocks"]["mode"].tolist())
    assert modes == {K.MODE_LEAF, K.MODE_GATHER, K.MODE_FIN}
    assert (H["items_l"][:, 3] < 0).sum() == H["blocks"]["nfin"].sum() > 0
    r = np.random.default_rng(3).standard_normal(f.plan.n)
    ref = O.solve_lower(f, r)
    assert np.abs(emulate_lower(H, r) - ref).max() <= 1e-12 * np.abs(ref).max()


def emulate_upper(H, w, z=None):
    n, nb = H["n"], H["nb"]
    blocks = H["blocks"]
    z = np.zeros(n) if z is None else z
    done = np.zeros(nb, dtype=np.int64)
    segs = np.zeros(len(H["tiles_u"]), dtype=np.int64)
    for b, t0, t1, sg in H["items_u"]:
        B = blocks[b]
        s, m, na = int(B["start"]), int(B["m"]), int(B["na"])
        w0, w1 = K._window(H["tiles_u"], m + na, (t0, t1, sg))
        if na and B["parent"] >= 0 and w1 > m:  # the item reads -z_anc (as the kernel: window-based)
            p = int(B["parent"])
            assert done[p] == blocks[p]["n_u"], "upper item dispatched before the parent's z"
        v = np.concatenate([w[s:s + m], -z[H["anc"][B["anc_off"]: B["anc_off"] + na]]])
        for t in ([t0] if 0 < sg < K.WHOLE else range(t0, t1)):
            if sg == K.WHOLE:
                segs[t] += H["tiles_u"]["nseg"][t]
            elif sg:
                segs[t] += 1
                if segs[t] < H["tiles_u"]["nseg"][t]:
                    continue
            cols, d, tl = _tile(H, True, t)
            vals = d @ _padded(v, tl + d.shape[1])[tl: tl + d.shape[1]]
            z[s + cols] = vals  # unit diagonal stored
        done[b] += 1
    assert np.all(done == blocks["n_u"])
    assert np.array_equal(segs, H["tiles_u"]["nseg"])
    return z


def _factors(dims, leaf):
    mesh = clamped_beam(*dims)
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    out = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, mesh.nodes,
                            np.zeros_like(mesh.nodes), np.zeros(mesh.ndof), 0.01, (0.0, -9.81, 0.0))
    a = CsrMatrix(mesh.ndof, mesh.ndof, out["row_ptr"], out["col_ind"], out["values"])
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), leaf))
    f = ND.ldlt_factor(a, plan)
    f._a = a
    return mesh, f


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


def test_tile_layout_roundtrip_and_coverage():
    _, f = _factors((4, 4, 12), 16)
    H = K.pack(f)
    tl_ = H["tiles_l"]
    assert np.all(tl_["off"] % 64 == 0) and np.all(tl_["tl"] % 2 == 0)  # 512-B tiles, 16-B aligned v
    for up in (False, True):
        items = H["items_u" if up else "items_l"]
        for b, bf in enumerate(f.blocks):
            m, na = bf.stop - bf.start, len(bf.anc)
            linv, mm = K.block_matrix(bf)
            G = K.gfull(linv, mm)
            G = G.T if up else G
            rows_seen = []
            for bb, t0, t1, big in items:
                if bb != b or big > 1:
                    continue
                assert big >= 0 and (not big or t1 == t0 + 1)
                for t in range(t0, t1):
                    rows, d, tl = _tile(H, up, t)
                    rows_seen.extend(rows.tolist())
                    lo, hi = K.row_ranges(m, na, up)
                    for k, row in enumerate(rows):
                        full = np.zeros(d.shape[1])
                        a, e = lo[row] - tl, hi[row] - tl
                        full[a:e] = G[row, lo[row]:hi[row]]
                        assert np.array_equal(d[k], full)
            assert sorted(rows_seen) == list(range(m if up else m + na))
    assert H["g"].size == int(tl_["np"].sum()) * K.TILE * 2


def test_shard_subsets_compose_to_the_full_apply():
    """Two block subsets (a shard's subtrees S and the replicated top T) packed
    separately: lower(S) -> external sums -> lower(T, r - ext) -> upper(T) ->
    upper(S) equals the oracle's apply (the sharded preconditioner, shard.py)."""
    from paper_2306_05893_b200 import shard as SH

    mesh, f = _factors((4, 4, 16), 16)
    sp = SH.shard_blocks(f, 2)
    n = f.plan.n
    r = np.random.default_rng(11).standard_normal(n)
    rp = r[f.plan.perm]
    y = np.zeros(n)
    ext = np.zeros(n)
    for g in range(2):
        S = [i for i in range(len(f.blocks)) if sp.owner[i] == g]
        HS = K.pack(f, S)
        ys = emulate_lower(HS, rp)
        rows = sp.owned_rows(g)
        y[rows] = ys[rows]
        cb = emulate_lower.cbuf
        for e in HS["ext_rows"]:
            ext[e] += cb[HS["cin_ptr"][e]: HS["cin_ptr"][e + 1]].sum()
    T = [i for i in range(len(f.blocks)) if sp.owner[i] < 0]
    HT = K.pack(f, T)
    yt = emulate_lower(HT, rp - ext)
    y[sp.top_rows] = yt[sp.top_rows]
    w = y / f.d
    z = emulate_upper(HT, w)
    for g in range(2):
        S = [i for i in range(len(f.blocks)) if sp.owner[i] == g]
        z = emulate_upper(K.pack(f, S), w, z)
    out = np.empty(n)
    out[f.plan.perm] = z
    ref = O.apply(f, r)
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("max_rows", [150, 400, 100000])
def test_amalgamated_factors_apply_identically(max_rows):
    """Subtree amalgamation (one block per small elimination subtree) is the same
    L: the oracle's level-scheduled apply on the merged factors equals the
    original's, and the device layout of the merged factors emulates to it."""
    mesh, f = _factors((4, 4, 16), 16)
    g = K.amalgamate(f, max_rows)
    assert len(g.blocks) < len(f.blocks)
    r = np.random.default_rng(5).standard_normal(f.plan.n)
    ref = O.apply(f, r)
    assert np.abs(O.apply(g, r) - ref).max() <= 1e-12 * np.abs(ref).max()
    H = K.pack(g)
    rp = r[f.plan.perm]
    z = emulate_upper(H, emulate_lower(H, rp) / f.d)
    out = np.empty_like(z)
    out[f.plan.perm] = z
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()


def test_block_inverse_conditioning_guard(caplog):
    """pack() measures cond_1(L11) of every block (the explicit inverses' error
    grows like cond * eps): small on the beams (the reference's factors here:
    ~10), and a graded SPD system is flagged."""
    _, f = _factors((6, 6, 20), 64)
    H = K.pack(f)
    assert 1.0 <= H["cond_l11"] <= 20.0
    # ill-conditioned: a graded SPD chain
    n = 40
    s = np.logspace(0, 30, n)
    dense = np.diag(s * s)
    for i in range(n - 1):  # D T D with T = tridiag(0.49, 1, 0.49) (SPD), D graded: L11 entries grow ~3^k
        dense[i, i + 1] = dense[i + 1, i] = 0.49 * s[i] * s[i + 1]
    rows, cols = np.nonzero(dense)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    a = CsrMatrix(n, n, rp, cols.astype(np.int64), dense[rows, cols])
    plan = ND.nested_dissection(ND.graph_from_pattern(a), 64)
    fi = ND.ldlt_factor(a, plan)
    Hi = K.pack(fi)
    assert Hi["cond_l11"] > K.COND_WARN


@pytest.mark.parametrize("segs", [2, 8])
def test_whole_tile_items(monkeypatch, segs):
    """Whole-tiles items (seg == WHOLE): only large tiles of one chunk each,
    consecutive in one block, <= segs segments and <= MAIL_TILES tiles in all;
    every other large tile keeps its chunk items; the emulated sweeps still
    reproduce the oracle."""
    mesh, f = _factors((10, 10, 60), 64)
    monkeypatch.setattr(K, "SEGS_PER_ITEM", segs)
    H = K.pack(f)
    for up, key, tkey in ((False, "items_l", "tiles_l"), (True, "items_u", "tiles_u")):
        T = H[tkey]
        big = T["np"].astype(np.int64) * K.TILE * 16 > K.ITEM_BYTES
        nseg = (T["np"].astype(np.int64) + K.SEG_PAIRS - 1) // K.SEG_PAIRS
        seen = np.zeros(len(T), dtype=bool)
        for b, t0, t1, sg in H[key]:
            if sg == K.WHOLE:
                assert 0 < t1 - t0 <= K.MAIL_TILES and big[t0:t1].all() and (nseg[t0:t1] <= segs).all()
                assert nseg[t0:t1].sum() <= segs or t1 - t0 == 1
                assert not seen[t0:t1].any()
                seen[t0:t1] = True
            elif sg > 0:  # chunk item of a tile too wide for one chunk (or whole items off)
                assert big[t0]
        assert (seen == (big & (nseg <= segs))).all()  # every one-chunk large tile is in a whole item
    r = np.random.default_rng(11).standard_normal(mesh.ndof)
    assert np.abs(emulate_lower(H, r) - O.solve_lower(f, r)).max() <= 1e-12 * np.abs(O.solve_lower(f, r)).max()
    assert np.abs(emulate_upper(H, r) - O.solve_upper(f, r)).max() <= 1e-12 * np.abs(O.solve_upper(f, r)).max()
