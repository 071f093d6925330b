"""Host-side packing of LDL^T factors into the device block-inverse layout (setup).

Runs once per factor refresh (on the AsyncPreconditioner worker thread for
the async path).  For every dissection block b (rows [start, start+m),
ancestor rows anc, na = len(anc)) the packer forms

    G_b = [ inv(L11) - I        strict lower triangle, rows 1..m-1  ]
          [ M = L21 inv(L11)    na x m                              ]

The reference applies L11^-1 by t x t tile substitution with explicit tile
inverses (ndprecond.py:575-587, 623-644); widening the tile to the whole
block removes the in-block dependency chain, and pre-multiplying the
coupling panel by it (M) makes the ancestor contributions depend only on the
block's input x_b:

    lower:  y_b = Linv x_b,   contributions  c = M x_b
    upper:  z_b = [Linv; M]^T [w_b ; -z_anc]

Both sweeps are therefore GEMVs over rows with a contiguous v-range (unit
diagonal stored): lower rows r of [Linv; M] (v = x_b, columns [0, r] or
[0, m)), upper rows c of its transpose (v = [w_b; -z_anc], columns
[c, m+na)).  The factor blocks are well
conditioned (cond_1(L11) <= 14 on the cfg2/cfg3 beams); the block-inverse
apply matches the reference's tile-16 sweeps to ~5e-16 relative.

Device layout (csrc/ldlt_sweep.cuh): rows are grouped in TILES of 32 (one
row per lane).  A tile covers the union [tl, th) of its rows' v-ranges (tl
even) and is stored pair-major, lane-interleaved: entry (row 32i+k, column
tl+2p+h) at ((p*32 + k)*2 + h) -- a warp reads 512 contiguous bytes per
pair (conflict-free LDS.128), each lane accumulates its own row, no
cross-lane reduction.  Entries outside a row's range are stored as zeros
(the padding is reported as stored vs algorithmic bytes).

Work items: up to 8 consecutive small tiles of a block (one warp each, one
TMA bulk copy of <= 40 KB) or one chunk of SEGS_PER_ITEM 40 KB column
segments of a large tile, streamed through two shared-memory stages (the 8
warps split each segment's pairs; the chunk's 32 partial sums go to a
scratch slot and the last chunk of the tile to finish adds them in chunk
order -- deterministic -- and emits the rows).
The dispatch order is a list schedule on an infinite machine keyed by each
item's earliest start under a simple cost model, ties broken by the longest
remaining path (critical path first).  Every dependency finishes strictly
before its dependant starts, so the order is topological -- all the
persistent kernel needs to be deadlock-free.
"""

from __future__ import annotations

import ctypes as C
import logging
import os

import numpy as np

from . import _lib

logger = logging.getLogger(__name__)

# The block-inverse layout applies explicit inverses Linv = inv(L11): their
# rounding error grows like cond_1(L11) * eps (the reference's tile-16
# substitution like cond of the 16 x 16 tiles).  pack() measures
# cond_1(L11) = ||L11||_1 ||Linv||_1 for every block (1.0e1 - 1.4e1 on the
# beams) and warns above COND_WARN, where the apply can drift from the
# reference's by more than ~1e-8 relative.
COND_WARN = 1e8
# apply: gather r through perm once before the lower sweep instead of per item
PERMUTE_ONCE = os.environ.get("TSB_PERMUTE_ONCE", "1") != "0"

TILE = 32               # rows per tile (one per lane)
ITEM_BYTES = 40 * 1024  # small-tile item budget: one TMA bulk copy (csrc kStage)
SEG_PAIRS = 80          # pairs per column segment of a large tile (80 * 32 * 16 B = 40 KB, csrc kSegPairs)
# item granularity by regime (tools/item_tune.py, B200): latency-bound factors
# (stored lower tiles <= GATHER_BIG_BYTES) keep items short -- cfg2 apply
# 0.168 ms at 2/2 vs 0.198 at 4/4 -- bandwidth-bound ones amortise the per-item
# chain over more bytes -- cfg3 1.13 ms at 8/4 and 6/4 vs 1.16 at 4/4, 1.86 at 16/4;
# 8/8 1.1316 vs 8/4 1.1377 (22,658 vs 25,270 lower items)
SEGS_PER_ITEM = int(os.environ["TSB_SEGS_PER_ITEM"]) if "TSB_SEGS_PER_ITEM" in os.environ else None
MAX_GROUPS = 8          # csrc kGroupsPerItem (mailbox capacity: MAX_GROUPS x WARPS tiles)
GROUPS_PER_ITEM = min(MAX_GROUPS, int(os.environ["TSB_GROUPS_PER_ITEM"])) if "TSB_GROUPS_PER_ITEM" in os.environ else None
SEGS_SMALL, GROUPS_SMALL, SEGS_BIG, GROUPS_BIG = 2, 2, 8, 8
SEGS_LOWER = int(os.environ["TSB_SEGS_LOWER"]) if "TSB_SEGS_LOWER" in os.environ else None
WHOLE = 1 << 20         # Item.seg of a whole-tiles item (csrc kWhole)
# one-chunk large tiles of a block grouped into whole-tiles items (no partial
# slots, one dependency wait and publication for several tiles)
WHOLE_ITEMS = os.environ.get("TSB_WHOLE_ITEMS", "1") != "0"
WHOLE_SEGS = int(os.environ["TSB_WHOLE_SEGS"]) if "TSB_WHOLE_SEGS" in os.environ else None  # segments per whole item
WARPS = 7               # consumer warps per CTA (csrc kWarps): one small tile each
MAIL_TILES = MAX_GROUPS * WARPS  # tiles one mailbox entry holds (csrc kMailTiles)
MERGE_ROWS = 0          # default subtree amalgamation (rows); 0 = off
CB_CAP = int(os.environ.get("TSB_CB_CAP", "1024"))  # contributions staged per piece when a block's items sum them (csrc max_cb)
# lower input mode: a block's items sum their contributions themselves while the
# redundant reads (items x contributions) stay below ratio x its factor entries,
# else finaliser items form x_b once.  Latency-bound (small) factors favour the
# item gathers (one hop less), bandwidth-bound (large) ones the finalisers (no
# redundant reads): measured apply cfg2 0.142 ms (ratio 1) vs 0.161 (0), cfg3
# 1.82 ms (1) vs 1.70 (0).  TSB_GATHER_RATIO overrides.
GATHER_RATIO = float(os.environ["TSB_GATHER_RATIO"]) if "TSB_GATHER_RATIO" in os.environ else None
GATHER_BIG_BYTES = 512 << 20  # stored lower tiles above this: bandwidth-bound regime
GATHER_FEW = int(os.environ.get("TSB_GATHER_FEW", "0"))  # tuning: small blocks with <= this many items gather

BLOCK_DTYPE = np.dtype([
    ("start", "<i4"), ("m", "<i4"), ("na", "<i4"), ("parent", "<i4"),
    ("target_l", "<i4"), ("n_u", "<i4"), ("mode", "<i4"), ("ncb", "<i4"),
    ("nfin", "<i4"), ("nu_parent", "<i4"), ("anc_off", "<i8"), ("cb_off", "<i8"),
])
assert BLOCK_DTYPE.itemsize == 56
FIN_CONTRIB = 4096      # contributions per finaliser item of a mode-2 block
TILE_DTYPE = np.dtype([("off", "<i8"), ("tl", "<i4"), ("np", "<i4"), ("row0", "<i4"), ("nrows", "<i4"),
                       ("nseg", "<i4"), ("part", "<i4")])
assert TILE_DTYPE.itemsize == 32
MODE_LEAF, MODE_GATHER, MODE_FIN = 0, 1, 2


def block_matrix(bf):
    """-> (Linv with unit diagonal, M = L21 Linv) of one block factor
    (LAPACK trtri + BLAS trmm: na m^2 flops for M)."""
    from scipy.linalg import blas, lapack

    m = bf.stop - bf.start
    linv, info = lapack.dtrtri(np.asarray(bf.l11, dtype=np.float64), lower=1, unitdiag=1)
    if info != 0:
        raise ValueError(f"singular diagonal block at {bf.start}")
    linv = np.tril(linv, -1)
    linv[np.diag_indices(m)] = 1.0
    if len(bf.anc):
        mm = blas.dtrmm(1.0, linv, np.asfortranarray(bf.l21, dtype=np.float64), side=1, lower=1, diag=1)
    else:
        mm = np.zeros((0, m))
    return linv, mm


def gfull(linv, mm):
    """Rows of the lower sweep as a dense (m + na) x m matrix: [Linv; M] (unit
    diagonal kept, so y_r = sum_{j <= r} Linv_rj x_j needs no separate x_r)."""
    return np.vstack([np.tril(linv), mm])


def row_ranges(m: int, na: int, upper: bool):
    """v-ranges [lo, hi) of the sweep's rows (diagonal included): lower rows r of
    [Linv; M] over x_b, upper rows c of its transpose over [w_b; -z_anc]."""
    if upper:
        c = np.arange(m, dtype=np.int64)
        return c, np.full(m, m + na, dtype=np.int64)
    r = np.arange(m + na, dtype=np.int64)
    return np.zeros(m + na, dtype=np.int64), np.minimum(r + 1, m)


def tile_layout(m: int, na: int, upper: bool):
    """Tiles of one block for one sweep: [(tl, npair, row0, nrows)] (a tile
    covers the union [tl, th) of its rows' v-ranges, tl even)."""
    lo, hi = row_ranges(m, na, upper)
    nrows_all = len(lo)
    tiles = []
    for r0 in range(0, nrows_all, TILE):
        r1 = min(r0 + TILE, nrows_all)
        tl = int(lo[r0:r1].min()) & ~1
        th = int(hi[r0:r1].max())
        tiles.append((tl, max((th - tl + 1) // 2, 0), r0, r1 - r0))
    return tiles


def tile_data(G, tiles):
    """The tiles' data (pair-major, lane-interleaved), concatenated in tile order."""
    parts = []
    for tl, npair, r0, nr in tiles:
        d = np.zeros((TILE, 2 * npair))
        w = min(2 * npair, G.shape[1] - tl)
        if w > 0:
            d[:nr, :w] = G[r0:r0 + nr, tl:tl + w]
        parts.append(d.reshape(TILE, npair, 2).transpose(1, 0, 2).ravel())
    return np.concatenate(parts) if parts else np.zeros(0)


def tile_block(G, m: int, na: int, upper: bool):
    """Tiles of one block for one sweep -> (list of (tl, np, row0, nrows), data parts).

    G holds the sweep's rows: gfull() for the lower sweep, its transpose for
    the upper; None gives zero tiles (structure only, filled on the device by
    tsb_refactor_run)."""
    tiles = tile_layout(m, na, upper)
    parts = []
    for tl, npair, r0, nr in tiles:
        d = tile_data(G, [(tl, npair, r0, nr)]) if G is not None else np.zeros(TILE * 2 * npair)
        parts.append(d)
    return tiles, parts


def untile(tiles, data, nrows, ncols):
    """Inverse of tile_block (testing): dense nrows x ncols from a block's tile rows."""
    out = np.zeros((nrows, ncols + 2))
    for off, tl, npair, r0, nr in tiles:
        d = data[off: off + npair * TILE * 2].reshape(npair, TILE, 2).transpose(1, 0, 2).reshape(TILE, 2 * npair)
        out[r0:r0 + nr, tl:tl + 2 * npair] = d[:nr]
    return out[:, :ncols]


class _Merged:
    """Block factor of an amalgamated subtree (duck-types ndprecond._BlockFactor)."""

    def __init__(self, start, stop, level, anc, l11, l21, tile=16):
        self.start, self.stop, self.level, self.anc = start, stop, level, anc
        self.l11, self.l21, self.tile = l11, l21, tile

    @property
    def tile_inv(self):  # only the CPU oracle reads these
        from .ndprecond import _tile_inverses

        return _tile_inverses(self.l11, self.tile)


class _MergedFactors:
    def __init__(self, factors, blocks):
        self.plan, self.d, self.blocks = factors.plan, factors.d, blocks
        nlev = 1 + max((b.level for b in blocks), default=0)
        self.levels = [[b for b in blocks if b.level == lv] for lv in range(nlev)]


def amalgamate(factors, max_rows: int):
    """Merge every elimination subtree of <= max_rows rows into one block.

    In dissection order a subtree owns the contiguous rows [tree_start, stop)
    and couples outside only to its root's ancestors (fill property), so the
    merged block is L restricted to those rows (dense unit-lower l11 holding
    the constituents' l11 and their in-subtree l21 rows) with the root's
    ancestors as coupling rows.  Mathematically the same L; after packing one
    GEMV replaces a whole subtree, cutting the dependency chain (one hop per
    merged subtree instead of one per level) at the price of the subtree's
    dense triangle.  Returns the factors unchanged when nothing merges."""
    bfs = list(factors.blocks)
    nb = len(bfs)
    if max_rows <= 0 or nb == 0:
        return factors
    n = factors.plan.n
    owner = np.full(n, -1, dtype=np.int64)
    for i, bf in enumerate(bfs):
        owner[bf.start:bf.stop] = i
    parent = np.full(nb, -1, dtype=np.int64)
    for i, bf in enumerate(bfs):
        if len(bf.anc):
            parent[i] = owner[int(np.min(bf.anc))]
    children = [[] for _ in range(nb)]
    for i in range(nb):
        if parent[i] >= 0:
            children[parent[i]].append(i)
    order = sorted(range(nb), key=lambda i: bfs[i].start)
    rows = np.array([bf.stop - bf.start for bf in bfs], dtype=np.int64)
    ts = np.array([bf.start for bf in bfs], dtype=np.int64)
    ok = np.zeros(nb, dtype=bool)
    for i in order:  # children first
        for c in children[i]:
            rows[i] += rows[c]
            ts[i] = min(ts[i], ts[c])
        ok[i] = rows[i] <= max_rows and all(ok[c] for c in children[i])
        if ok[i] and rows[i] != bfs[i].stop - ts[i]:
            ok[i] = False  # not contiguous: leave the subtree as it is
    roots = [i for i in order if ok[i] and children[i] and (parent[i] < 0 or not ok[parent[i]])]
    if not roots:
        return factors
    gone = set()
    new_blocks = []
    for b in roots:
        sub, stack = [], [b]
        while stack:
            i = stack.pop()
            sub.append(i)
            stack.extend(children[i])
        gone.update(sub)
        s0, e0 = int(ts[b]), bfs[b].stop
        m = e0 - s0
        anc = np.asarray(bfs[b].anc, dtype=np.int64)
        l11 = np.zeros((m, m))
        l21 = np.zeros((len(anc), m))
        for i in sub:
            bf = bfs[i]
            cs, ce = bf.start - s0, bf.stop - s0
            l11[cs:ce, cs:ce] = np.tril(bf.l11)
            if len(bf.anc):
                a = np.asarray(bf.anc, dtype=np.int64)
                inside = a < e0
                l11[a[inside] - s0, cs:ce] = bf.l21[inside]
                k = np.searchsorted(anc, a[~inside])
                if np.any(k >= len(anc)) or np.any(anc[np.minimum(k, len(anc) - 1)] != a[~inside]):
                    raise ValueError("subtree couples outside its root's ancestors")
                l21[k, cs:ce] = bf.l21[~inside]
        new_blocks.append(_Merged(s0, e0, bfs[b].level, anc, l11, l21, getattr(bfs[b], "tile", 16)))
    blocks = [bf for i, bf in enumerate(bfs) if i not in gone] + new_blocks
    blocks.sort(key=lambda bf: bf.start)
    return _MergedFactors(factors, blocks)


def _items(tiles_of_block, first_tile, segs, groups_per_item):
    """Group a block's tiles into items -> list of (t0, t1, seg) in global tile ids
    (seg = 0: small tiles [t0, t1); seg = WHOLE: whole large tiles [t0, t1) of
    <= segs segments in all; seg = c + 1: chunk c of large tile t0, i.e. its
    column segments [c t1, c t1 + t1), t1 = segs)."""
    out = []
    k = 0
    nt = len(tiles_of_block)

    def nseg(k_):
        return (int(tiles_of_block[k_][1]) + SEG_PAIRS - 1) // SEG_PAIRS

    while k < nt:
        npair = tiles_of_block[k][1]
        if npair * TILE * 16 > ITEM_BYTES:
            if WHOLE_ITEMS and nseg(k) <= segs:  # consecutive one-chunk tiles: one item
                k1, tot = k, 0
                budget = WHOLE_SEGS if WHOLE_SEGS is not None else segs
                while (k1 < nt and k1 - k < MAIL_TILES and tiles_of_block[k1][1] * TILE * 16 > ITEM_BYTES
                       and nseg(k1) <= segs and (k1 == k or tot + nseg(k1) <= budget)):
                    tot += nseg(k1)
                    k1 += 1
                out.append((first_tile + k, first_tile + k1, WHOLE))
                k = k1
                continue
            for c in range(_nchunks(npair, segs)):
                out.append((first_tile + k, segs, c + 1))
            k += 1
            continue
        k1, groups = k, 0  # up to groups_per_item TMA groups of small tiles (csrc group_end)
        while groups < groups_per_item and k1 < nt and tiles_of_block[k1][1] * TILE * 16 <= ITEM_BYTES:
            g1, tot = k1, 0
            while g1 < nt and g1 - k1 < WARPS:
                b = tiles_of_block[g1][1] * TILE * 16
                if b > ITEM_BYTES or tot + b > ITEM_BYTES:
                    break
                tot += b
                g1 += 1
            k1 = g1
            groups += 1
        out.append((first_tile + k, first_tile + k1, 0))
        k = k1
    return out


def _nchunks(npair, segs):
    nsegs = (int(npair) + SEG_PAIRS - 1) // SEG_PAIRS
    return (nsegs + segs - 1) // segs


def item_granularity(stored_lower_bytes):
    """(segments per chunk item, TMA groups per small-tile item) for a factor."""
    big = stored_lower_bytes > GATHER_BIG_BYTES
    segs = SEGS_PER_ITEM if SEGS_PER_ITEM is not None else (SEGS_BIG if big else SEGS_SMALL)
    groups = GROUPS_PER_ITEM if GROUPS_PER_ITEM is not None else (GROUPS_BIG if big else GROUPS_SMALL)
    return segs, groups


def _chunk_pairs(npair, it):
    """pairs [p0, p1) of chunk item it of a tile with npair pairs (csrc chunk_range)."""
    nsegs = (int(npair) + SEG_PAIRS - 1) // SEG_PAIRS
    s0 = (it[2] - 1) * it[1]
    s1 = min(s0 + it[1], nsegs)
    return s0 * SEG_PAIRS, min(s1 * SEG_PAIRS, int(npair))


HOP = 1.5               # us: dependency release -> consumer sees it
SCHED_WORKERS = 296     # resident CTAs the list schedule assumes (148 SMs x 2)


def _window(T, lim, it):
    """v-columns [w0, w1) an item reads (csrc item_window); T = the sweep's tile table."""
    if 0 < it[2] < WHOLE:
        p0, p1 = _chunk_pairs(T["np"][it[0]], it)
        w0 = int(T["tl"][it[0]]) + 2 * p0
        return w0, min(int(T["tl"][it[0]]) + 2 * p1, lim)
    w0 = int(T["tl"][it[0]:it[1]].min())
    return w0, min(int((T["tl"][it[0]:it[1]] + 2 * T["np"][it[0]:it[1]]).max()), lim)


def _list_schedule(entries, cost, children, sweep):
    """Ticket order = start order of a list schedule of the items on
    SCHED_WORKERS workers: whenever a worker frees, it starts the ready item
    with the longest remaining path (critical path first).  An item starts
    only after its dependencies finished, so the order is topological (what
    the persistent kernel needs to be deadlock-free).  entries: (block, item,
    dep, tail); dep: None, ("children", b) = every GEMV item of b's children,
    ("fin", b) = b's finalisers, ("parent", p) = every item of block p."""
    import heapq

    n = len(entries)
    by_block = {}
    fin_of = {}
    for k, (b, it, dep, tail) in enumerate(entries):
        if it[2] < 0:
            fin_of.setdefault(b, []).append(k)
        else:
            by_block.setdefault(b, []).append(k)
    # dependency counts and successor lists per "dependency group"
    group_members = {}
    for k, (b, it, dep, tail) in enumerate(entries):
        if dep is None:
            continue
        kind, blk = dep
        if kind == "children":
            members = [j for c in children[blk] for j in by_block.get(c, [])]
        elif kind == "fin":
            members = fin_of.get(blk, [])
        else:
            members = by_block.get(blk, [])
        group_members.setdefault(dep, members)
    waiting = {}
    succ = [[] for _ in range(n)]
    remaining = {}
    for dep, members in group_members.items():
        remaining[dep] = len(members)
        for j in members:
            succ[j].append(dep)
    dependants = {}
    for k, (b, it, dep, tail) in enumerate(entries):
        if dep is not None:
            dependants.setdefault(dep, []).append(k)
    ready = []     # released items, by priority (longest remaining path first)
    pending = []   # items whose dependencies finished, by release time
    for k, (b, it, dep, tail) in enumerate(entries):
        if dep is None or remaining.get(dep, 0) == 0:
            heapq.heappush(ready, (-tail, k))
    running = []   # (finish time, k)
    free = SCHED_WORKERS
    t = 0.0
    start_order = []
    while ready or pending or running:
        while pending and pending[0][0] <= t:
            _, k = heapq.heappop(pending)
            heapq.heappush(ready, (-entries[k][3], k))
        while free and ready:
            _, k = heapq.heappop(ready)
            start_order.append(k)
            heapq.heappush(running, (t + cost(entries[k]), k))
            free -= 1
        # next event: a worker finishes or a pending item is released
        nxt_run = running[0][0] if running else float("inf")
        nxt_rel = pending[0][0] if pending else float("inf")
        if nxt_rel < nxt_run and free:
            t = nxt_rel
            continue
        if not running:
            t = nxt_rel
            continue
        t, k = heapq.heappop(running)
        free += 1
        for dep in succ[k]:
            remaining[dep] -= 1
            if remaining[dep] == 0:
                for j in dependants.get(dep, []):
                    heapq.heappush(pending, (t + HOP, j))
    if len(start_order) != n:
        raise RuntimeError(f"{sweep} item list has a dependency cycle")
    out = np.array([(entries[k][0], entries[k][1][0], entries[k][1][1], entries[k][1][2]) for k in start_order],
                   dtype=np.int32)
    return out.reshape(-1, 4)


def pack(factors, subset=None, sink=None, alloc=None):
    """Host arrays of the tiled block-inverse layout + item lists (pure NumPy).

    `subset` (block indices) packs one shard: ancestor rows outside the subset
    are external (their contributions are summed by tsb_ldlt_external_sums,
    their z is read from the output vector) and blocks whose parent is outside
    become roots of the handle."""
    plan = factors.plan
    n = plan.n
    bfs = list(factors.blocks) if subset is None else [factors.blocks[i] for i in sorted(subset)]
    nb = len(bfs)
    # block elimination tree: parent(b) = owner of b's first ancestor row.  The
    # fill property  anc(b) \ rows(parent) <= anc(parent)  makes "all children
    # done" imply "all descendants done" (lower) and "parent done" imply "all
    # ancestors done" (upper) -- the only dependencies the kernels track.
    owner = np.full(n, -1, dtype=np.int64)
    for i, bf in enumerate(bfs):
        if bf.stop <= bf.start:
            raise ValueError("empty dissection block")
        owner[bf.start:bf.stop] = i
    parent = np.full(nb, -1, dtype=np.int64)
    for i, bf in enumerate(bfs):
        if len(bf.anc):
            anc = np.asarray(bf.anc)
            if np.any(anc < bf.stop) or np.any(np.diff(anc) <= 0):
                raise ValueError("ancestor rows must be sorted and follow the block")
            parent[i] = owner[anc[0]]
    for i, bf in enumerate(bfs):
        p = parent[i]
        if p >= 0:
            rest = np.asarray(bf.anc)
            rest = rest[rest >= bfs[p].stop]
            if len(rest) and not np.all(np.isin(rest, np.asarray(bfs[p].anc))):
                raise ValueError("factor structure violates the fill property")
    children = [[] for _ in range(nb)]
    for i in range(nb):
        if parent[i] >= 0:
            children[parent[i]].append(i)
    ms_ = np.array([bf.stop - bf.start for bf in bfs], dtype=np.int64)
    na_ = np.array([len(bf.anc) for bf in bfs], dtype=np.int64)

    # ---------------- tiles: layout pass ----------------
    tl_rows = {False: [], True: []}       # per sweep: global tile table rows
    pos = {False: 0, True: 0}
    blk_tiles = {False: [], True: []}     # per sweep, per block: (first tile id, [tiles])
    tile_blk = {False: [], True: []}      # per sweep: tile -> block
    blk_off = {False: [], True: []}       # per sweep, per block: offset of its data
    for i in range(nb):
        for up in (False, True):
            tiles = tile_layout(int(ms_[i]), int(na_[i]), up)
            blk_tiles[up].append((len(tl_rows[up]), tiles))
            tile_blk[up].extend([i] * len(tiles))
            blk_off[up].append(pos[up])
            for tl, npair, r0, nr in tiles:
                tl_rows[up].append((pos[up], tl, npair, r0, nr))
                pos[up] += TILE * 2 * npair
    if alloc is not None:  # the caller's storage for the two images (e.g. HBM), before the data pass
        alloc(pos[False], pos[True])
    # ---------------- tiles: data pass ----------------
    # block by block (block_matrix computed lazily, so the host holds one block's
    # G at a time); sink(up, offset, data) receives each block's tiles -- the
    # device image writes them straight into HBM, the default collects them
    from threadpoolctl import threadpool_limits

    values = all(getattr(bf, "l11", None) is not None for bf in bfs)  # else structure only (zero tiles)
    data = {False: [], True: []}
    if sink is None and values:
        def sink(up, off, d):
            data[up].append(d)
    cond_l11 = 1.0
    if values:
        big = ms_ * (ms_ + na_) > 1_000_000
        small_limiter = threadpool_limits(limits=1, user_api="blas")  # small blocks: thread wake-ups cost more
        try:
            for i, bf in enumerate(bfs):
                if big[i]:
                    small_limiter.restore_original_limits()
                linv_i, mm_i = block_matrix(bf)
                if big[i]:
                    small_limiter = threadpool_limits(limits=1, user_api="blas")
                l11 = np.tril(np.asarray(bf.l11, dtype=np.float64), -1) + np.eye(len(linv_i))
                c1 = float(np.abs(l11).sum(axis=0).max() * np.abs(linv_i).sum(axis=0).max()) if len(linv_i) else 1.0
                cond_l11 = max(cond_l11, c1)
                G = gfull(linv_i, mm_i)
                del l11, linv_i, mm_i
                for up in (False, True):
                    sink(up, blk_off[up][i], tile_data(G.T if up else G, blk_tiles[up][i][1]))
        finally:
            small_limiter.restore_original_limits()
    segs, groups_per_item = item_granularity(pos[False] * 8)
    segs_l = SEGS_LOWER if SEGS_LOWER is not None else segs  # tuning override for the lower sweep alone
    tables = {}
    npart = {}
    for up in (False, True):
        t = np.zeros(len(tl_rows[up]), dtype=TILE_DTYPE)
        if tl_rows[up]:
            arr = np.array(tl_rows[up], dtype=np.int64)
            t["off"], t["tl"], t["np"], t["row0"], t["nrows"] = arr.T
        big = t["np"].astype(np.int64) * TILE * 16 > ITEM_BYTES
        t["nseg"] = np.where(big, [_nchunks(v, segs if up else segs_l) for v in t["np"]], 0)  # chunk items per tile
        part = np.zeros(len(t) + 1, dtype=np.int64)
        np.cumsum(t["nseg"], out=part[1:])
        t["part"] = part[:-1]
        npart[up] = int(part[-1])
        tables[up] = t
    anc_off = np.zeros(nb + 1, dtype=np.int64)
    np.cumsum(na_, out=anc_off[1:])
    anc_all = (np.concatenate([np.asarray(bf.anc, dtype=np.int64) for bf in bfs]) if anc_off[-1]
               else np.zeros(0, dtype=np.int64))

    # ---------------- contribution slots (lower) ----------------
    corder = np.argsort(anc_all, kind="stable")   # row-contiguous, block order within a row
    cin_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(anc_all, minlength=n), out=cin_ptr[1:])
    cslot = np.empty(len(anc_all), dtype=np.int64)
    cslot[corder] = np.arange(len(anc_all))
    ext_rows = np.unique(anc_all[owner[anc_all] < 0]) if len(anc_all) else np.zeros(0, dtype=np.int64)

    # ---------------- items + lower input modes ----------------
    items = {up: [_items(blk_tiles[up][i][1], blk_tiles[up][i][0], segs if up else segs_l, groups_per_item)
                  for i in range(nb)]
             for up in (False, True)}
    nl = np.array([len(x) for x in items[False]], dtype=np.int64)
    n_u = np.array([len(x) for x in items[True]], dtype=np.int64)
    target_l = np.array([sum(int(nl[c]) for c in children[i]) for i in range(nb)], dtype=np.int64)
    # lower input of a block: its items sum the contributions themselves when the
    # redundant L2 reads stay below the block's own factor bytes (mode 1), else
    # nfin finaliser items (dispatched first) form x_b = input - contributions
    # once, each for a slice of rows, and the block's items read it (mode 2)
    contrib = np.diff(cin_ptr)
    blk_contrib = np.array([int(contrib[bf.start:bf.stop].sum()) for bf in bfs], dtype=np.int64)
    gsize = np.array([int(tables[False]["np"][f:f + len(t)].sum()) * TILE * 2 for f, t in blk_tiles[False]],
                     dtype=np.int64)
    ratio = GATHER_RATIO if GATHER_RATIO is not None else (0.0 if pos[False] * 8 > GATHER_BIG_BYTES else 1.0)
    mode = np.where(target_l == 0, MODE_LEAF,
                    np.where(nl * blk_contrib <= ratio * gsize, MODE_GATHER, MODE_FIN))
    if GATHER_FEW:  # blocks of <= GATHER_FEW items whose contributions one finaliser would sum: gather
        few = (target_l > 0) & (nl <= GATHER_FEW) & (blk_contrib <= FIN_CONTRIB)
        mode = np.where(few, MODE_GATHER, mode)
    nfin = np.where(mode == MODE_FIN,
                    np.minimum(np.minimum(32, (ms_ + 31) // 32), np.maximum(1, (blk_contrib + FIN_CONTRIB - 1) // FIN_CONTRIB)),
                    0)
    fin_items = [[] for _ in range(nb)]
    for i in np.flatnonzero(nfin):
        k = int(nfin[i])
        edges = np.linspace(0, int(ms_[i]), k + 1).astype(np.int64)
        fin_items[i] = [(int(edges[j]), int(edges[j + 1]), -1) for j in range(k) if edges[j + 1] > edges[j]]
        nfin[i] = len(fin_items[i])

    def cost(up, it):  # us: item latency + streaming at ~24 GB/s per CTA (HBM shared by 296 CTAs)
        if it[2] < 0:
            return 2.5
        if 0 < it[2] < WHOLE:
            p0, p1 = _chunk_pairs(tables[up]["np"][it[0]], it)
            return 3.0 + (p1 - p0) * TILE * 16 / 24e3
        return 3.0 + int(tables[up]["np"][it[0]:it[1]].sum()) * TILE * 16 / 24e3

    def touches_anc(i, it):  # upper item whose column window reaches -z_anc (waits for the parent)
        if not na_[i]:
            return False
        w0, w1 = _window(tables[True], int(ms_[i]) + int(na_[i]), it)
        return w1 > ms_[i]

    order = sorted(range(nb), key=lambda i: bfs[i].start)  # children before parents
    # lower: blocks wait for their children's items (or their finalisers)
    own_l = np.array([max(cost(False, it) for it in items[False][i]) + (cost(False, (0, 0, -1)) + HOP if nfin[i] else 0.0)
                      for i in range(nb)])
    tail_l = np.zeros(nb)
    for i in reversed(order):  # parents first
        tail_l[i] = own_l[i] + (HOP + tail_l[parent[i]] if parent[i] >= 0 else 0.0)
    lower = []  # (item, block, kind, deps-key): kind 0 finaliser, 1 GEMV
    for i in range(nb):
        for it in fin_items[i]:
            lower.append((i, it, ("children", i), tail_l[i] + 1.0))
        for it in items[False][i]:
            dep = ("fin", i) if nfin[i] else (("children", i) if target_l[i] else None)
            lower.append((i, it, dep, tail_l[i]))
    items_l = _list_schedule(lower, lambda x: cost(False, x[1]), children, "lower")
    # upper: items reading -z_anc wait for their parent's items
    own_u = np.array([max(cost(True, it) for it in items[True][i]) for i in range(nb)])
    tail_u = np.zeros(nb)
    for i in order:  # children first
        tail_u[i] = own_u[i] + max((HOP + tail_u[c] for c in children[i]), default=0.0)
    upper = []
    for i in range(nb):
        for it in items[True][i]:
            dep = ("parent", int(parent[i])) if (parent[i] >= 0 and touches_anc(i, it)) else None
            upper.append((i, it, dep, tail_u[i]))
    items_u = _list_schedule(upper, lambda x: cost(True, x[1]), children, "upper")

    # ---------------- block table ----------------
    blocks = np.zeros(nb, dtype=BLOCK_DTYPE)
    blocks["start"] = [bf.start for bf in bfs]
    blocks["m"] = ms_
    blocks["na"] = na_
    blocks["parent"] = parent
    blocks["target_l"] = target_l
    blocks["n_u"] = n_u
    blocks["nu_parent"] = np.where(np.asarray(parent) >= 0, np.asarray(n_u)[np.maximum(np.asarray(parent), 0)], 0)
    blocks["mode"] = mode
    blocks["nfin"] = nfin
    blocks["ncb"] = blk_contrib
    blocks["cb_off"] = cin_ptr[[bf.start for bf in bfs]] if nb else []
    blocks["anc_off"] = anc_off[:-1]
    max_cb = min(CB_CAP, int(blk_contrib[mode == MODE_GATHER].max())) if np.any(mode == MODE_GATHER) else 0

    def window(up, i, it):
        return _window(tables[up], int(ms_[i] + (na_[i] if up else 0)), it)

    max_w = max([1] + [(lambda w: w[1] - w[0])(window(up, i, it)) for up in (False, True)
                       for i in range(nb) for it in items[up][i]])
    def cat(up):  # one array per sweep (zeros: structure only; None: the sink holds the data)
        if not values:
            return np.zeros(max(pos[up], 2))
        if not data[up]:
            return None if pos[up] else np.zeros(2)
        out = np.concatenate(data[up])
        data[up].clear()
        return out

    return {
        "n": n, "nb": nb, "blocks": blocks, "items_l": items_l, "items_u": items_u,
        "tiles_l": tables[False], "tiles_u": tables[True], "g": cat(False), "gt": cat(True),
        "anc": anc_all, "cslot": cslot, "cin_ptr": cin_ptr, "ncbuf": len(anc_all),
        "d": np.asarray(factors.d if factors.d is not None else np.zeros(n), dtype=np.float64), "perm": np.asarray(plan.perm, dtype=np.int64),
        "max_m": int(ms_.max()) if nb else 1, "max_v": int(max_w), "max_cb": max_cb, "cond_l11": cond_l11,
        "parent": parent, "children": children, "mode": mode,
        "npart_l": npart[False], "npart_u": npart[True], "ext_rows": ext_rows,
        "bytes_g": int(pos[False]) * 8, "bytes_gt": int(pos[True]) * 8,
        "tile_blk_l": np.asarray(tile_blk[False], dtype=np.int32), "tile_blk_u": np.asarray(tile_blk[True], dtype=np.int32),
    }


class DevicePanels:
    """Packed factor image in HBM + the libtsb handle (tsb_ldlt_create)."""

    def __init__(self, factors, stream=None, trace=False, force_mode=None, subset=None, merge=None, grid=0):
        t = _lib.require_cuda()
        if merge is None:
            merge = MERGE_ROWS if subset is None else 0
        dev_img = {}

        def alloc(n_l, n_u):  # the factor images live only in HBM: each block's tiles are copied in directly
            dev_img[False] = t.zeros(max(n_l, 2), dtype=t.float64, device="cuda")
            dev_img[True] = t.zeros(max(n_u, 2), dtype=t.float64, device="cuda")

        def sink(up, off, d):
            if len(d):
                dev_img[up][off:off + len(d)].copy_(t.from_numpy(d))

        src = amalgamate(factors, merge) if merge else factors
        values = all(getattr(bf, "l11", None) is not None for bf in src.blocks)
        H = pack(src, subset, sink=sink if values else None, alloc=alloc if values else None)
        if force_mode is not None:  # testing: route every inner block through one input mode
            if force_mode != MODE_GATHER:
                raise ValueError("only the item-gather mode can be forced (finaliser items are planned)")
            inner = H["blocks"]["mode"] != MODE_LEAF
            H["blocks"]["mode"][inner] = force_mode
            H["blocks"]["nfin"][inner] = 0
            H["items_l"] = H["items_l"][H["items_l"][:, 3] >= 0]
            H["max_cb"] = min(CB_CAP, int(H["blocks"]["ncb"][inner].max(initial=0)))
        n, nb = H["n"], H["nb"]
        items_l, items_u = H["items_l"], H["items_u"]
        self.cond_l11 = H["cond_l11"]  # max cond_1(L11) over the blocks (explicit-inverse accuracy guard)
        if self.cond_l11 > COND_WARN:
            logger.warning("LDL^T block-inverse apply: cond_1(L11) up to %.3g; the explicit inverses lose about "
                           "cond * eps relative accuracy against the reference's tile substitution", self.cond_l11)
        self.host = H if trace else None
        self.tile_blk = (H["tile_blk_l"], H["tile_blk_u"])  # tile -> block (device refactorisation)
        if trace:  # per-item timeline (globaltimer ns): take, ready, end, smid, staged, computed
            self.trace_l = t.zeros((len(items_l), 8), dtype=t.int64, device="cuda")
            self.trace_u = t.zeros((len(items_u), 8), dtype=t.int64, device="cuda")
        ctx = t.cuda.stream(stream) if stream is not None else _NullCtx()
        with ctx:
            def up(a):  # small arrays through pinned memory; the factor images (GBs at 1M nodes) straight,
                # without a second full-size pinned host copy
                a = np.ascontiguousarray(a)
                if a.nbytes > (1 << 30):
                    return t.from_numpy(a).to("cuda")
                return t.from_numpy(a).pin_memory().to("cuda", non_blocking=True)
            i32 = lambda a: up(np.asarray(a, dtype=np.int32))  # noqa: E731
            i64 = lambda a: up(np.asarray(a, dtype=np.int64))  # noqa: E731
            z = lambda k, dt: t.zeros(max(k, 1), dtype=dt, device="cuda")  # noqa: E731
            nz = lambda a: a if len(a) else np.zeros(1, dtype=a.dtype)  # noqa: E731
            raw = lambda a: up(nz(a).view(np.uint8))  # noqa: E731
            self.t = {
                "blocks": raw(H["blocks"]), "items_l": up(nz(items_l.ravel())), "items_u": up(nz(items_u.ravel())),
                "tiles_l": raw(H["tiles_l"]), "tiles_u": raw(H["tiles_u"]),
                "g": dev_img[False] if H["g"] is None else up(H["g"]),
                "gt": dev_img[True] if H["gt"] is None else up(H["gt"]),
                "anc": i32(nz(H["anc"])), "cslot": i32(nz(H["cslot"])), "cin_ptr": i64(H["cin_ptr"]),
                "d": up(H["d"]), "perm": i32(H["perm"]), "ext_rows": i32(nz(H["ext_rows"])),
            }
            ntl, ntu = len(H["tiles_l"]), len(H["tiles_u"])
            self.t.update(cbuf=z(H["ncbuf"], t.float64), x=z(n, t.float64), y=z(n, t.float64), rin=z(n, t.float64),
                          part=z(TILE * (H["npart_l"] + H["npart_u"]), t.float64),
                          cnt=z(3 * nb, t.int32), tcnt=z(ntl + ntu, t.int32), ctl=z(4, t.int32))
        H["g"] = H["gt"] = None  # the host copies of the factor images (GBs) are not needed any more
        self.n = n
        self.ncbuf, self.npart_l = int(H["ncbuf"]), int(H["npart_l"])
        self._multi = {}
        self.n_blocks = nb
        self.n_items = (len(items_l), len(items_u))
        self.bytes = {"g": H["bytes_g"], "gt": H["bytes_gt"]}
        tp = lambda k: _lib.ptr(self.t[k])  # noqa: E731
        cnt = self.t["cnt"]
        cp = lambda a, b: _lib.ptr(cnt[a:b]) if b > a else _lib.ptr(cnt)  # noqa: E731
        self.desc = _lib.LdltDesc(
            n=n, n_blocks=nb, n_items_lower=len(items_l), n_items_upper=len(items_u),
            max_m=H["max_m"], max_v=H["max_v"], max_cb=H["max_cb"], grid=int(grid),
            d_blocks=tp("blocks"), d_items_lower=tp("items_l"), d_items_upper=tp("items_u"),
            d_tiles_lower=tp("tiles_l"), d_tiles_upper=tp("tiles_u"), d_g=tp("g"), d_gt=tp("gt"),
            d_anc=tp("anc"), d_cslot=tp("cslot"), d_cin_ptr=tp("cin_ptr"), d_d=tp("d"),
            d_perm=tp("perm"), d_cbuf=tp("cbuf"), d_x=tp("x"), d_y=tp("y"),
            d_part_lower=tp("part"), d_part_upper=_lib.ptr(self.t["part"][TILE * H["npart_l"]:]),
            d_tcnt_lower=tp("tcnt"), d_tcnt_upper=_lib.ptr(self.t["tcnt"][ntl:]),
            n_tiles_lower=ntl, n_tiles_upper=ntu, d_ext_rows=tp("ext_rows"), n_ext=len(H["ext_rows"]),
            d_cnt_l=cp(0, nb), d_ready_l=cp(nb, 2 * nb), d_done_u=cp(2 * nb, 3 * nb), d_pad=tp("ctl"),
            d_ctl=tp("ctl"),
            d_trace_lower=_lib.ptr(self.trace_l) if trace else None,
            d_trace_upper=_lib.ptr(self.trace_u) if trace else None,
            d_rin=tp("rin") if PERMUTE_ONCE else None,
        )
        if stream is not None:
            stream.synchronize()
        h = C.c_void_p()
        self._lib = _lib.load()
        _lib.check(self._lib.tsb_ldlt_create(C.byref(self.desc), C.byref(h)), "ldlt_create")
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self._lib.tsb_ldlt_destroy(self.h)
        except Exception:
            pass

    def run(self, mode: str, r, out):
        fn = {"lower": self._lib.tsb_ldlt_lower, "upper": self._lib.tsb_ldlt_upper,
              "apply": self._lib.tsb_ldlt_apply, "upper_scaled": self._lib.tsb_ldlt_upper_scaled}[mode]
        _lib.check(fn(self.h, _lib.ptr(r), _lib.ptr(out), _lib.stream_ptr()), f"ldlt_{mode}")

    MULTI_RHS = min(8, int(os.environ.get("TSB_MULTI_RHS", "8")))  # right-hand sides per multi-RHS lower sweep (<= 8)

    def lower_multi(self, R, Y):
        """Y[j] = L^-1 R[j] (permuted order) for the rows of R ([k][n] CUDA
        tensors), MULTI_RHS right-hand sides per sweep (tsb_ldlt_lower_multi)."""
        t = _lib.torch()
        k = R.shape[0]
        for j0 in range(0, k, self.MULTI_RHS):
            nr = min(self.MULTI_RHS, k - j0)
            if nr == 1:
                self.run("lower", R[j0], Y[j0])
                continue
            sc = self._multi.get(nr)
            if sc is None:
                ld_part = max(TILE * self.npart_l, 1)
                sc = (t.zeros(nr * max(self.ncbuf, 1), dtype=t.float64, device="cuda"),
                      t.zeros(nr * self.n, dtype=t.float64, device="cuda"),
                      t.zeros(nr * ld_part, dtype=t.float64, device="cuda"), ld_part)
                self._multi[nr] = sc
            cb, xs, part, ld_part = sc
            _lib.check(self._lib.tsb_ldlt_lower_multi(self.h, nr, _lib.ptr(R[j0]), _lib.ptr(Y[j0]), _lib.ptr(cb),
                                                      max(self.ncbuf, 1), _lib.ptr(xs), _lib.ptr(part), ld_part,
                                                      _lib.stream_ptr()), "ldlt_lower_multi")

    def lower_ext(self, r, ext, out):
        _lib.check(self._lib.tsb_ldlt_lower_ext(self.h, _lib.ptr(r), _lib.ptr(ext), _lib.ptr(out), _lib.stream_ptr()),
                   "ldlt_lower_ext")

    def external_sums(self, out):
        _lib.check(self._lib.tsb_ldlt_external_sums(self.h, _lib.ptr(out), _lib.stream_ptr()), "ldlt_external_sums")


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
