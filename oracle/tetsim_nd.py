"""CPU oracle, part 2: mesh, nested dissection and LDL^T factorisation -- TEST
INFRASTRUCTURE ONLY (same rules as oracle/tetsim_oracle.py: only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import it).

A plain-NumPy restatement of the reference's host setup for the solve path,
so that bench.py's `--impl reference` arm builds its whole workload (mesh,
scenario state, dissection, stale factors) without touching the product
package:

  generate_beam / vertex_adjacency     mesh.py:139-181, 293-315
  nested_dissection / expand_plan      ndprecond.py:107-279
  ldlt_factor (+ symbolic, tile inv.)  ndprecond.py:355-587

Restated, not copied: BFS runs level-synchronously over the CSR graph with
array operations (distances are unique, so the result is the reference's),
and the greedy separator cover keeps per-vertex counts decrementally instead
of re-counting every cut edge per pick (same argmax, same lowest-index tie
break).  The factorisation follows the reference's right-looking block order
(dense Cholesky of the diagonal block, triangular solve of the coupling
panel, Schur update routed into the ancestor blocks).

Pinned: tests/test_oracle_golden.py checks the plans against the reference's
own `nd_plans.npz` (bit-identical perm/blocks/levels) and the factors
against `ldlt_small.npz` (the reference's l11/l21/d).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# mesh.py:139-181, 293-315
# ---------------------------------------------------------------------------


def generate_beam(nx, ny, nz, spacing):
    """(nodes, elements) of the reference beam: node id i + nx (j + ny k),
    cells k-major, 6 tets per cell along the main diagonal in
    itertools.permutations order, odd permutations swap ids 1 and 2."""
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    nodes = spacing * np.stack([i, j, k], axis=-1).reshape(-1, 3).astype(np.float64)
    ck, cj, ci = np.meshgrid(np.arange(nz - 1), np.arange(ny - 1), np.arange(nx - 1), indexing="ij")
    base = ci.ravel() + nx * (cj.ravel() + ny * ck.ravel())
    off = np.array([1, nx, nx * ny])
    tets = []
    for perm in itertools.permutations(range(3)):
        walk = np.cumsum(off[list(perm)])
        ids = [base] + [base + w for w in walk]
        odd = sum(a > b for a, b in itertools.combinations(perm, 2)) % 2
        if odd:
            ids[1], ids[2] = ids[2], ids[1]
        tets.append(np.stack(ids, axis=1))
    elements = np.stack(tets, axis=1).reshape(-1, 4).astype(np.int64)
    return nodes, elements


def clamped_nodes(nodes):
    """Nodes on the z = 0 face (test_acceptance.py:49-51)."""
    return np.flatnonzero(nodes[:, 2] == 0.0)


def vertex_adjacency(n, elements):
    """(indptr, indices): i ~ j iff they share an element, sorted, no loops."""
    el = np.asarray(elements, dtype=np.int64)
    a, b = np.nonzero(~np.eye(4, dtype=bool))
    codes = np.unique((el[:, a] * n + el[:, b]).ravel())
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(codes // n, minlength=n), out=indptr[1:])
    return indptr, codes % n


# ---------------------------------------------------------------------------
# ndprecond.py:69-279
# ---------------------------------------------------------------------------


@dataclass
class Block:
    start: int
    stop: int
    tree_start: int
    kind: str
    children: tuple
    level: int = 0

    @property
    def size(self):
        return self.stop - self.start


@dataclass
class Plan:
    n: int
    perm: np.ndarray
    iperm: np.ndarray
    blocks: list
    levels: list


def _neighbours(indptr, indices, frontier):
    lo, hi = indptr[frontier], indptr[frontier + 1]
    cnt = hi - lo
    if cnt.sum() == 0:
        return np.empty(0, dtype=np.int64)
    pos = np.repeat(lo - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt) + np.arange(cnt.sum())
    return indices[pos]


def _bfs(indptr, indices, source, in_sub):
    """Graph distances from source inside in_sub (-1 = unreached)
    (ndprecond.py:107-121)."""
    dist = np.full(len(in_sub), -1, dtype=np.int64)
    dist[source] = 0
    frontier = np.array([source], dtype=np.int64)
    d = 0
    while len(frontier):
        d += 1
        w = _neighbours(indptr, indices, frontier)
        w = np.unique(w[in_sub[w] & (dist[w] < 0)])
        dist[w] = d
        frontier = w
    return dist


def _pseudo_peripheral(indptr, indices, sub, in_sub):
    """ndprecond.py:124-138."""
    u = int(sub[0])
    dist = _bfs(indptr, indices, u, in_sub)
    ecc = int(dist[sub].max())
    for _ in range(10):
        v = int(sub[dist[sub] == ecc].min())
        dv = _bfs(indptr, indices, v, in_sub)
        ev = int(dv[sub].max())
        if ev <= ecc:
            break
        u, dist, ecc = v, dv, ev
    return u, dist


def _components(indptr, indices, sub):
    """Connected components of sub, in order of their first vertex in sub
    (ndprecond.py:141-154)."""
    in_sub = np.zeros(len(indptr) - 1, dtype=bool)
    in_sub[sub] = True
    comps = []
    left = np.ones(len(sub), dtype=bool)
    while left.any():
        s = int(sub[np.argmax(left)])
        dist = _bfs(indptr, indices, s, in_sub)
        hit = dist[sub] >= 0
        comp = sub[hit]
        comps.append(comp)
        in_sub[comp] = False
        left &= ~hit
    return comps


def _greedy_cover(ea, eb, n):
    """Greedy vertex cover of the cut edges, ties to the lowest index, capped
    by the smaller touched side (ndprecond.py:157-176)."""
    touched_a, touched_b = np.unique(ea), np.unique(eb)
    fallback = touched_a if len(touched_a) <= len(touched_b) else touched_b
    if len(ea) == 0:
        return np.empty(0, dtype=np.int64)
    verts, inv = np.unique(np.concatenate([ea, eb]), return_inverse=True)
    ia, ib = inv[: len(ea)], inv[len(ea):]
    cnt = np.bincount(ia, minlength=len(verts)) + np.bincount(ib, minlength=len(verts))
    ends = np.concatenate([ia, ib])
    edge = np.concatenate([np.arange(len(ea)), np.arange(len(ea))])
    order = np.argsort(ends, kind="stable")
    start = np.searchsorted(ends[order], np.arange(len(verts) + 1))
    alive = np.ones(len(ea), dtype=bool)
    cover = []
    left = len(ea)
    while left:
        v = int(np.argmax(cnt))  # first maximum = lowest vertex id (verts ascending)
        cover.append(verts[v])
        es = edge[order[start[v]:start[v + 1]]]
        es = es[alive[es]]
        alive[es] = False
        left -= len(es)
        np.subtract.at(cnt, ia[es], 1)
        np.subtract.at(cnt, ib[es], 1)
    cover = np.array(sorted(cover), dtype=np.int64)
    return fallback if len(cover) > len(fallback) else cover


def _dissect(g, sub, base, threshold, blocks, esrc, edst):
    """ndprecond.py:179-231 (halves first, separator last, leaves sorted)."""
    indptr, indices = g
    n = len(indptr) - 1

    def leaf():
        blocks.append(Block(base, base + len(sub), base, "leaf", ()))
        return np.sort(sub), [len(blocks) - 1]

    if len(sub) <= threshold:
        return leaf()
    comps = _components(indptr, indices, sub)
    if len(comps) > 1:
        orders, roots, off = [], [], base
        for comp in comps:
            o, r = _dissect(g, comp, off, threshold, blocks, esrc, edst)
            orders.append(o)
            roots += r
            off += len(comp)
        return np.concatenate(orders), roots
    in_sub = np.zeros(n, dtype=bool)
    in_sub[sub] = True
    _, dist = _pseudo_peripheral(indptr, indices, sub, in_sub)
    lv, counts = np.unique(dist[sub], return_counts=True)
    ell = lv[int(np.searchsorted(np.cumsum(counts), len(sub) / 2.0))]
    in_a = in_sub & (dist >= 0) & (dist <= ell)
    cut = in_a[esrc] & in_sub[edst] & ~in_a[edst]
    sep = _greedy_cover(esrc[cut], edst[cut], n)
    if len(sep) == 0 or len(sep) == len(sub):
        return leaf()
    in_sep = np.zeros(n, dtype=bool)
    in_sep[sep] = True
    orders, roots, off = [], [], base
    for half in (sub[in_a[sub] & ~in_sep[sub]], sub[~in_a[sub] & ~in_sep[sub]]):
        if len(half):
            o, r = _dissect(g, half, off, threshold, blocks, esrc, edst)
            orders.append(o)
            roots += r
            off += len(half)
    orders.append(np.sort(sep))
    blocks.append(Block(off, off + len(sep), base, "separator", tuple(roots)))
    return np.concatenate(orders), [len(blocks) - 1]


def nested_dissection(indptr, indices, leaf_threshold=64):
    """Vertex-space plan (ndprecond.py:234-267)."""
    import sys

    n = len(indptr) - 1
    sys.setrecursionlimit(max(sys.getrecursionlimit(), 10000))
    blocks = []
    esrc = np.repeat(np.arange(n), np.diff(indptr))
    order, _ = _dissect((np.asarray(indptr), np.asarray(indices)), np.arange(n, dtype=np.int64), 0,
                        leaf_threshold, blocks, esrc, np.asarray(indices))
    perm = np.asarray(order, dtype=np.int64)
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    for blk in blocks:  # children precede their parent in `blocks`
        blk.level = 0 if not blk.children else 1 + max(blocks[c].level for c in blk.children)
    nlev = 1 + max(b.level for b in blocks)
    levels = [sorted((i for i, b in enumerate(blocks) if b.level == lv), key=lambda i: blocks[i].start)
              for lv in range(nlev)]
    return Plan(n, perm, iperm, blocks, levels)


def expand_plan(plan, k=3):
    """Vertex plan -> DOF plan, k consecutive DOFs per vertex (ndprecond.py:270-279)."""
    perm = (k * plan.perm[:, None] + np.arange(k)).ravel()
    iperm = np.empty(len(perm), dtype=np.int64)
    iperm[perm] = np.arange(len(perm))
    blocks = [Block(k * b.start, k * b.stop, k * b.tree_start, b.kind, b.children, b.level) for b in plan.blocks]
    return Plan(k * plan.n, perm, iperm, blocks, plan.levels)


# ---------------------------------------------------------------------------
# ndprecond.py:355-587 -- numeric LDL^T
# ---------------------------------------------------------------------------


@dataclass
class BlockFactor:
    start: int
    stop: int
    level: int
    anc: np.ndarray
    l11: np.ndarray
    l21: np.ndarray
    tile: int
    tile_inv: list


@dataclass
class Factors:
    """Duck-type of the reference LdlFactors that tetsim_oracle.apply consumes."""

    d: np.ndarray
    plan: Plan
    blocks: list
    levels: list

    @property
    def fill_in(self):
        tot = 0
        for bf in self.blocks:
            tot += int(np.count_nonzero(np.tril(bf.l11, -1))) + int(np.count_nonzero(bf.l21))
        return tot


def tile_inverses(l11, tile):
    """Inverses of the unit-lower diagonal tiles (ndprecond.py:575-587)."""
    m = len(l11)
    out = [np.linalg.inv(l11[t:t + tile, t:t + tile]) for t in range(0, m - m % tile, tile)]
    if m % tile:
        t = m - m % tile
        out.append(np.linalg.inv(l11[t:, t:]))
    return out


def ldlt_factor(row_ptr, col_ind, values, plan, tile=16):
    """Right-looking block LDL^T in dissection order (ndprecond.py:355-572):
    per block in start order, dense Cholesky C of the diagonal block,
    d = diag(C)^2, L11 = C / diag(C), LS = C^-1 panel^T, L21 = LS / diag(C),
    and the Schur update LS LS^T subtracted from the ancestor blocks'
    diagonal blocks and coupling panels."""
    n = len(row_ptr) - 1
    row_ptr = np.asarray(row_ptr)
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    pi, pj = plan.iperm[rows], plan.iperm[np.asarray(col_ind)]
    vals = np.asarray(values, dtype=np.float64)
    owner = np.empty(n, dtype=np.int64)
    for bid, b in enumerate(plan.blocks):
        owner[b.start:b.stop] = bid
    order = sorted(range(len(plan.blocks)), key=lambda b: plan.blocks[b].start)
    # entries grouped by permuted row; coupling sets (fill propagates up
    # through the children's sets)
    couple = {}
    srt = np.lexsort((pj, pi))
    pi_s, pj_s, v_s = pi[srt], pj[srt], vals[srt]
    prp = np.searchsorted(pi_s, np.arange(n + 1))
    for bid in order:
        blk = plan.blocks[bid]
        lo, hi = prp[blk.start], prp[blk.stop]
        cols = pj_s[lo:hi]
        pieces = [cols[cols >= blk.stop]] + [couple[c][couple[c] >= blk.stop] for c in blk.children]
        couple[bid] = np.unique(np.concatenate(pieces))
    ds, panel = {}, {}
    for bid in order:
        blk = plan.blocks[bid]
        s, e, m = blk.start, blk.stop, blk.size
        lo, hi = prp[s], prp[e]
        r, c, v = pi_s[lo:hi] - s, pj_s[lo:hi], v_s[lo:hi]
        dsb = np.zeros((m, m))
        inb = (c >= s) & (c < e)
        dsb[r[inb], c[inb] - s] = v[inb]
        cb = couple[bid]
        pb = np.zeros((len(cb), m))
        rt = c >= e
        pb[np.searchsorted(cb, c[rt]), r[rt]] = v[rt]
        ds[bid], panel[bid] = dsb, pb
    d = np.empty(n)
    out = {}
    for bid in order:
        blk = plan.blocks[bid]
        s, e, m = blk.start, blk.stop, blk.size
        try:
            c = np.linalg.cholesky(ds[bid])
        except np.linalg.LinAlgError as exc:
            raise np.linalg.LinAlgError(f"non-positive pivot in block [{s}, {e}): {exc}") from None
        dv = np.diagonal(c).copy()
        d[s:e] = dv * dv
        l11 = c / dv[None, :]
        cb = couple[bid]
        if len(cb):
            ls = np.linalg.solve(c, panel[bid].T).T  # the reference's general solve (ndprecond.py:556)
            l21 = ls / dv[None, :]
            u = ls @ ls.T
            own = owner[cb]
            tgts = np.unique(own)
            for jj, gj in enumerate(tgts):
                sj = np.flatnonzero(own == gj)
                t0 = plan.blocks[gj].start
                ds[gj][np.ix_(cb[sj] - t0, cb[sj] - t0)] -= u[np.ix_(sj, sj)]
                for gi in tgts[jj + 1:]:
                    si = np.flatnonzero(own == gi)
                    pos = np.searchsorted(couple[gj], cb[si])
                    panel[gj][np.ix_(pos, cb[sj] - t0)] -= u[np.ix_(si, sj)]
        else:
            l21 = np.empty((0, m))
        out[bid] = BlockFactor(s, e, blk.level, cb, l11, l21, tile, tile_inverses(l11, tile))
        ds[bid] = panel[bid] = None
    blocks = [out[b] for b in order]
    levels = [[] for _ in range(1 + max(bf.level for bf in blocks))]
    for bf in blocks:
        levels[bf.level].append(bf)
    return Factors(d, plan, blocks, levels)
