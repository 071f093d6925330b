"""Host-side packing of LDL^T factors into the device block-inverse layout (setup).

Runs once per factor refresh (on the AsyncPreconditioner worker thread for
the async path).  For every dissection block b (rows [start, start+m),
ancestor rows anc, na = len(anc)) it stores one row-major matrix

    G_b = [ inv(L11) - I        strict lower triangle, rows 1..m-1  ]
          [ M = L21 inv(L11)    na x m                              ]

The reference applies L11^-1 by t x t tile substitution with explicit tile
inverses (ndprecond.py:575-587, 623-644); widening the tile to the whole
block removes the in-block dependency chain, and pre-multiplying the
coupling panel by it (M) makes the ancestor contributions depend only on the
block's input x_b:

    lower:  y_b = x_b + (Linv - I) x_b,   contributions  c = M x_b
    upper:  z_b = w_b + G_b^T [w_b ; -z_anc]

G_b has exactly the entries of [L11 ; L21] (same bytes per sweep), serves
both sweeps, and the only serial chain left is the depth of the dissection
tree.  The factor blocks are well conditioned (cond_1(L11) <= 12.5 on the
cfg2 beam); the block-inverse apply matches the reference's tile-16 sweeps
to ~4e-16 relative.

G_b is stored twice: row-major for the lower sweep and transposed for the
upper (row c of G_b^T = column c of G_b below the diagonal, i.e. the entries
multiplying v[c+1:]), so both sweeps are row-chunked GEMVs with one TMA bulk
copy per work item (~48 KB) and no cross-item reduction.  The
dispatch order is a list schedule on an infinite machine keyed by each
item's earliest start under a simple cost model, ties broken by the longest
remaining path (critical path first).  Every dependency finishes strictly
before its dependant starts, so the order is topological -- all the
persistent kernel needs to be deadlock-free.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

CHUNK = 6144          # doubles per lower item (48 KB, one TMA bulk copy)
CHUNK_ROWS = 512      # rows per lower item (csrc kMaxChunkRows)
CB_MAX = 4096         # contributions a block's items may sum themselves (csrc max_cb)

BLOCK_DTYPE = np.dtype([
    ("start", "<i4"), ("m", "<i4"), ("na", "<i4"), ("parent", "<i4"),
    ("target_l", "<i4"), ("n_u", "<i4"), ("mode", "<i4"), ("ncb", "<i4"),
    ("g_off", "<i8"), ("gt_off", "<i8"), ("anc_off", "<i8"), ("cb_off", "<i8"),
])
assert BLOCK_DTYPE.itemsize == 64
MODE_LEAF, MODE_GATHER, MODE_FIN = 0, 1, 2


def row_offsets(m: int, na: int) -> np.ndarray:
    """Offsets (doubles) of the m + na + 1 row boundaries of G_b (csrc g_row_off)."""
    r = np.arange(m + na + 1, dtype=np.int64)
    ms = m + (m & 1)
    return np.where(r < m, (r * r) // 2, (m * m) // 2 + (r - m) * ms)


def gt_row_offsets(m: int, na: int) -> np.ndarray:
    """Offsets (doubles) of the m + 1 row boundaries of G_b^T (csrc gt_row_off):
    row c holds v-entries [c+1, m+na), length K - c (K = m+na-1), padded to even."""
    K = m + na - 1
    lens = K - np.arange(m, dtype=np.int64)
    out = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens + (lens & 1), out=out[1:])
    return out


def block_matrix(bf):
    """-> (Linv with unit diagonal, M = L21 Linv) of one block factor."""
    from scipy.linalg import solve_triangular

    m = bf.stop - bf.start
    linv = solve_triangular(bf.l11, np.eye(m), lower=True, unit_diagonal=True, check_finite=False)
    mm = bf.l21 @ linv if len(bf.anc) else np.zeros((0, m))
    return linv, mm


def pack_block(bf) -> np.ndarray:
    """G_b in the device row layout (flat float64, even length)."""
    linv, mm = block_matrix(bf)
    return _pack_rows(bf, linv, mm)


def _pack_rows(bf, linv, mm):
    m, na = bf.stop - bf.start, len(bf.anc)
    off = row_offsets(m, na)
    g = np.zeros(int(off[-1]))
    ir, ic = np.tril_indices(m, -1)
    g[(ir * ir) // 2 + ic] = linv[ir, ic]
    if na:
        ms = m + (m & 1)
        g[off[m]:].reshape(na, ms)[:, :m] = mm
    return g


def pack_block_t(bf, linv=None, mm=None) -> np.ndarray:
    """G_b^T in the device row layout (flat float64, even length)."""
    m, na = bf.stop - bf.start, len(bf.anc)
    if linv is None:
        linv, mm = block_matrix(bf)
    full = np.vstack([np.tril(linv, -1), mm]) if na else np.tril(linv, -1)
    off = gt_row_offsets(m, na)
    g = np.zeros(int(off[-1]))
    for c in range(m):
        col = full[c + 1:, c]
        g[off[c]: off[c] + len(col)] = col
    return g


def unpack_block(g, m, na):
    """Inverse of pack_block -> (Linv with unit diagonal, M)."""
    off = row_offsets(m, na)
    linv = np.eye(m)
    ir, ic = np.tril_indices(m, -1)
    linv[ir, ic] = g[(ir * ir) // 2 + ic]
    ms = m + (m & 1)
    mm = g[off[m]:off[-1]].reshape(na, ms)[:, :m] if na else np.zeros((0, m))
    return linv, mm


def _lower_chunks(off, nrows):
    """Row ranges of G_b with <= CHUNK doubles each (at least one row)."""
    out, r0 = [], 0
    while r0 < nrows:
        r1 = int(np.searchsorted(off, off[r0] + CHUNK, side="right")) - 1
        r1 = min(max(r1, r0 + 1), nrows, r0 + CHUNK_ROWS)
        out.append((r0, r1))
        r0 = r1
    return out or [(0, 0)]


def pack(factors):
    """Host arrays of the block-inverse layout + item lists (pure NumPy)."""
    plan = factors.plan
    n = plan.n
    bfs = list(factors.blocks)
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
            pb = bfs[p]
            rest = np.asarray(bf.anc)
            rest = rest[rest >= pb.stop]
            if len(rest) and not np.all(np.isin(rest, np.asarray(pb.anc))):
                raise ValueError("factor structure violates the fill property")
    children = [[] for _ in range(nb)]
    for i in range(nb):
        if parent[i] >= 0:
            children[parent[i]].append(i)

    ms_ = np.array([bf.stop - bf.start for bf in bfs], dtype=np.int64)
    na_ = np.array([len(bf.anc) for bf in bfs], dtype=np.int64)
    # ---------------- G blobs ----------------
    g_parts, g_off = [], np.zeros(nb, dtype=np.int64)
    gt_parts, gt_off = [], np.zeros(nb, dtype=np.int64)
    pos = post = 0
    for i, bf in enumerate(bfs):
        linv, mm = block_matrix(bf)
        g = _pack_rows(bf, linv, mm)
        gt = pack_block_t(bf, linv, mm)
        g_off[i], gt_off[i] = pos, post
        g_parts.append(g)
        gt_parts.append(gt)
        pos += len(g)
        post += len(gt)
    anc_off = np.zeros(nb + 1, dtype=np.int64)
    np.cumsum(na_, out=anc_off[1:])
    anc_all = (np.concatenate([np.asarray(bf.anc, dtype=np.int64) for bf in bfs]) if anc_off[-1]
               else np.zeros(0, dtype=np.int64))
    # ---------------- lower items ----------------
    offs = [row_offsets(int(ms_[i]), int(na_[i])) for i in range(nb)]
    lchunks = [_lower_chunks(offs[i], int(ms_[i] + na_[i])) for i in range(nb)]
    nl = np.array([len(c) for c in lchunks], dtype=np.int64)
    target_l = np.array([sum(int(nl[c]) for c in children[i]) for i in range(nb)], dtype=np.int64)

    def cost(doubles):  # us: item overhead + streaming at ~40 GB/s per CTA
        return 1.0 + doubles * 8 / 40e3

    order = sorted(range(nb), key=lambda i: bfs[i].start)  # children before parents
    ready_l = np.zeros(nb)
    done_l = np.zeros(nb)
    for i in order:
        if children[i]:
            ready_l[i] = max(done_l[c] for c in children[i]) + 1.0 + 0.002 * ms_[i]
        worst = max(cost(offs[i][r1] - offs[i][r0]) for r0, r1 in lchunks[i])
        done_l[i] = ready_l[i] + worst
    tail_l = np.zeros(nb)
    for i in reversed(order):  # parents first
        tail_l[i] = (done_l[i] - ready_l[i]) + (tail_l[parent[i]] if parent[i] >= 0 else 0.0)
    lower = []
    for i in range(nb):
        for r0, r1 in lchunks[i]:
            lower.append((ready_l[i], -tail_l[i], bfs[i].start, r0, i, r1))
    lower.sort()
    items_l = np.array([(x[4], x[3], x[5], 0) for x in lower], dtype=np.int32).reshape(-1, 4)
    # ---------------- upper items ----------------
    toffs = [gt_row_offsets(int(ms_[i]), int(na_[i])) for i in range(nb)]
    uchunks = [_lower_chunks(toffs[i], int(ms_[i])) for i in range(nb)]
    n_u = np.array([len(c) for c in uchunks], dtype=np.int64)
    start_u = np.zeros(nb)
    done_u = np.zeros(nb)
    for i in reversed(order):  # parents first
        start_u[i] = done_u[parent[i]] if parent[i] >= 0 else 0.0
        done_u[i] = start_u[i] + max(cost(toffs[i][r1] - toffs[i][r0]) for r0, r1 in uchunks[i])
    tail_u = np.zeros(nb)
    for i in order:  # children first
        tail_u[i] = (done_u[i] - start_u[i]) + max((tail_u[c] for c in children[i]), default=0.0)
    upper = []
    for i in range(nb):
        for r0, r1 in uchunks[i]:
            upper.append((start_u[i], -tail_u[i], -bfs[i].start, r0, i, r1))
    upper.sort()
    items_u = np.array([(x[4], x[3], x[5], 0) for x in upper], dtype=np.int32).reshape(-1, 4)
    # ---------------- contribution slots (lower) ----------------
    corder = np.argsort(anc_all, kind="stable")   # row-contiguous, block order within a row
    cin_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(anc_all, minlength=n), out=cin_ptr[1:])
    cslot = np.empty(len(anc_all), dtype=np.int64)
    cslot[corder] = np.arange(len(anc_all))
    # ---------------- block table ----------------
    blocks = np.zeros(nb, dtype=BLOCK_DTYPE)
    blocks["start"] = [bf.start for bf in bfs]
    blocks["m"] = ms_
    blocks["na"] = na_
    blocks["parent"] = parent
    blocks["target_l"] = target_l
    blocks["n_u"] = n_u
    # lower input of a block: its items sum the contributions themselves when the
    # redundant L2 reads stay below the block's own factor bytes, else the child
    # item that completes the block sums them once (one extra hop)
    contrib = np.diff(cin_ptr)
    blk_contrib = np.array([int(contrib[bf.start:bf.stop].sum()) for bf in bfs], dtype=np.int64)
    gsize = np.array([len(g) for g in g_parts], dtype=np.int64)
    mode = np.where(target_l == 0, MODE_LEAF,
                    np.where((nl * blk_contrib <= gsize) & (blk_contrib <= CB_MAX), MODE_GATHER, MODE_FIN))
    blocks["mode"] = mode
    blocks["ncb"] = blk_contrib
    blocks["cb_off"] = cin_ptr[[bf.start for bf in bfs]] if nb else []
    blocks["gt_off"] = gt_off
    blocks["g_off"] = g_off
    blocks["anc_off"] = anc_off[:-1]
    max_lchunk = max(int(offs[i][r1] - offs[i][r0]) for i in range(nb) for r0, r1 in lchunks[i]) if nb else 2
    max_uchunk = max(int(toffs[i][r1] - toffs[i][r0]) for i in range(nb) for r0, r1 in uchunks[i]) if nb else 2
    stage = max(max_lchunk, max_uchunk, 2)
    stage += stage & 1
    max_cb = int(blk_contrib[mode == MODE_GATHER].max()) if np.any(mode == MODE_GATHER) else 0
    return {
        "n": n, "nb": nb, "blocks": blocks, "items_l": items_l, "items_u": items_u,
        "g": np.concatenate(g_parts) if g_parts else np.zeros(2),
        "gt": np.concatenate(gt_parts) if gt_parts else np.zeros(2),
        "anc": anc_all, "cslot": cslot, "cin_ptr": cin_ptr, "ncbuf": len(anc_all),
        "d": np.asarray(factors.d, dtype=np.float64), "perm": np.asarray(plan.perm, dtype=np.int64),
        "stage": int(stage), "max_m": int(ms_.max()) if nb else 1,
        "max_v": int((ms_ + na_).max()) if nb else 1, "max_cb": max_cb,
        "parent": parent, "children": children, "mode": mode,
        "bytes_g": int(pos) * 8, "bytes_gt": int(post) * 8,
    }


class DevicePanels:
    """Packed factor image in HBM + the libtsb handle (tsb_ldlt_create)."""

    def __init__(self, factors, stream=None, trace=False, force_mode=None):
        t = _lib.require_cuda()
        H = pack(factors)
        if force_mode is not None:  # testing: route every inner block through one input mode
            inner = H["blocks"]["mode"] != MODE_LEAF
            H["blocks"]["mode"][inner] = force_mode
            if force_mode == MODE_GATHER:
                H["max_cb"] = int(H["blocks"]["ncb"][inner].max(initial=0))
        n, nb = H["n"], H["nb"]
        items_l, items_u = H["items_l"], H["items_u"]
        self.host = H if trace else None
        if trace:  # per-item timeline (globaltimer ns): take, ready, end, smid, staged, computed
            self.trace_l = t.zeros((len(items_l), 8), dtype=t.int64, device="cuda")
            self.trace_u = t.zeros((len(items_u), 8), dtype=t.int64, device="cuda")
        ctx = t.cuda.stream(stream) if stream is not None else _NullCtx()
        with ctx:
            up = lambda a: t.from_numpy(np.ascontiguousarray(a)).pin_memory().to("cuda", non_blocking=True)  # noqa: E731
            i32 = lambda a: up(np.asarray(a, dtype=np.int32))  # noqa: E731
            i64 = lambda a: up(np.asarray(a, dtype=np.int64))  # noqa: E731
            z = lambda k, dt: t.zeros(max(k, 1), dtype=dt, device="cuda")  # noqa: E731
            nz = lambda a: a if len(a) else np.zeros(1, dtype=a.dtype)  # noqa: E731
            self.t = {
                "blocks": up(H["blocks"].view(np.uint8)), "items_l": up(nz(items_l.ravel())),
                "items_u": up(nz(items_u.ravel())), "g": up(H["g"]), "gt": up(H["gt"]),
                "anc": i32(nz(H["anc"])), "cslot": i32(nz(H["cslot"])), "cin_ptr": i64(H["cin_ptr"]),
                "d": up(H["d"]), "perm": i32(H["perm"]),
            }
            self.t.update(cbuf=z(H["ncbuf"], t.float64), x=z(n, t.float64), y=z(n, t.float64),
                          cnt=z(3 * nb, t.int32), ctl=z(4, t.int32))
        self.n = n
        self.n_blocks = nb
        self.n_items = (len(items_l), len(items_u))
        self.bytes = {"g": H["bytes_g"], "gt": H["bytes_gt"]}
        tp = lambda k: _lib.ptr(self.t[k])  # noqa: E731
        cnt = self.t["cnt"]
        cp = lambda a, b: _lib.ptr(cnt[a:b]) if b > a else _lib.ptr(cnt)  # noqa: E731
        self.desc = _lib.LdltDesc(
            n=n, n_blocks=nb, n_items_lower=len(items_l), n_items_upper=len(items_u),
            stage_doubles=H["stage"], max_m=H["max_m"], max_v=H["max_v"], max_cb=H["max_cb"], grid=0, pad_=0,
            d_blocks=tp("blocks"), d_items_lower=tp("items_l"), d_items_upper=tp("items_u"), d_g=tp("g"),
            d_gt=tp("gt"), d_anc=tp("anc"), d_cslot=tp("cslot"), d_cin_ptr=tp("cin_ptr"), d_d=tp("d"),
            d_perm=tp("perm"), d_cbuf=tp("cbuf"), d_x=tp("x"), d_y=tp("y"),
            d_cnt_l=cp(0, nb), d_ready_l=cp(nb, 2 * nb), d_done_u=cp(2 * nb, 3 * nb), d_pad=tp("ctl"),
            d_ctl=tp("ctl"),
            d_trace_lower=_lib.ptr(self.trace_l) if trace else None,
            d_trace_upper=_lib.ptr(self.trace_u) if trace else None,
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
              "apply": self._lib.tsb_ldlt_apply}[mode]
        _lib.check(fn(self.h, _lib.ptr(r), _lib.ptr(out), _lib.stream_ptr()), f"ldlt_{mode}")


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
