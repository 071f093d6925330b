"""Host-side packing of LDL^T factors into the device panel layout (setup).

Runs once per factor refresh (on the AsyncPreconditioner worker thread for
the async path).  Cuts every dissection block of `LdlFactors` into column
panels of <= PANEL_W columns, lays out the diagonal-triangle inverses and
the below panels contiguously for streaming, builds the work-item lists of
the two sweeps (csrc/ldlt.cu) and orders them critical-path first.

Item dispatch order = list schedule on an infinite machine: each item is
keyed by its earliest start time under a simple cost model (tile-chain
latency for diagonal items, bytes / per-CTA bandwidth for panel chunks).
Because every dependency finishes before its dependant starts, the order is
topological, which is all the persistent kernel needs to be deadlock-free.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

PANEL_W = 128          # panel width (columns), multiple of the 16-wide tile
TILE = 16
CHUNK_ELEMS = 6144     # ~48 KB of factor per off-diagonal item
CRIT_ROWS = 32         # chunk rows for the next panel of the same block (critical path)

IT_DIAG, IT_OFF, IT_OFFT, IT_DIAGT = 0, 1, 2, 3


def packed_inverse(l):
    """Strict lower part of inv(l) for a unit-lower l -> (column-packed, row-packed).

    Column-packed: column j holds rows j+1..w-1 at j(2w-j-1)/2 (lower sweep:
    thread per row reads consecutive words); row-packed: row i holds columns
    0..i-1 at i(i-1)/2 (upper sweep).  Padded to an even length (16-byte TMA).
    """
    from scipy.linalg import solve_triangular

    w = len(l)
    inv = solve_triangular(l, np.eye(w), lower=True, unit_diagonal=True, check_finite=False)
    rows = inv[np.tril_indices(w, -1)]
    cols = inv.T[np.triu_indices(w, 1)]
    if len(rows) == 0:
        return np.zeros(2), np.zeros(2)
    if len(rows) % 2:
        rows, cols = np.append(rows, 0.0), np.append(cols, 0.0)
    return cols, rows


def _inverse(order):
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order))
    return inv


def _chunks(nb, n_crit, w):
    """Row ranges of a panel's below list: critical rows first, in small chunks."""
    out = []
    r = 0
    while r < n_crit:
        out.append((r, min(r + CRIT_ROWS, n_crit)))
        r = out[-1][1]
    step = max(32, CHUNK_ELEMS // max(w + (w & 1), 1))
    while r < nb:
        out.append((r, min(r + step, nb)))
        r = out[-1][1]
    return out


def pack(factors):
    """Host arrays of the panel layout + item lists (pure NumPy; see DevicePanels)."""
    if True:
        n = factors.plan.n
        order = [bf for lvl in factors.levels for bf in lvl]
        # -------- panels --------
        p_start, p_w, p_blk = [], [], []
        tri_parts, tri_u_parts, pan_parts, below_parts = [], [], [], []
        p_tri, p_tri_len, p_pan, p_below, p_cb = [], [], [], [], []
        ct = cp = cb = cbuf = 0
        panel_of_row = np.empty(n, dtype=np.int64)
        crit = []
        for bi, bf in enumerate(order):
            s, m = bf.start, bf.stop - bf.start
            anc = np.asarray(bf.anc, dtype=np.int64)
            for c0 in range(0, m, PANEL_W):
                w = min(PANEL_W, m - c0)
                pid = len(p_start)
                panel_of_row[s + c0:s + c0 + w] = pid
                below = np.concatenate([np.arange(s + c0 + w, s + m, dtype=np.int64), anc])
                # rows padded to an even stride so every chunk is a 16-byte-aligned TMA copy
                ws = w + (w & 1)
                pan = np.zeros((len(below), ws))
                pan[: m - c0 - w, :w] = bf.l11[c0 + w:, c0:c0 + w]
                pan[m - c0 - w:, :w] = bf.l21[:, c0:c0 + w]
                pan = pan.ravel()
                blob, blob_u = packed_inverse(bf.l11[c0:c0 + w, c0:c0 + w])
                p_start.append(s + c0)
                p_w.append(w)
                p_blk.append(bi)
                p_tri.append(ct)
                p_tri_len.append(len(blob))
                p_pan.append(cp)
                p_below.append(cb)
                p_cb.append(cbuf)
                tri_parts.append(blob)
                tri_u_parts.append(blob_u)
                pan_parts.append(pan)
                below_parts.append(below)
                ct += len(blob)
                cp += len(pan)
                cb += len(below)
                cbuf += len(below)
                crit.append(min(PANEL_W, max(0, m - c0 - w)))
        P = len(p_start)
        p_w = np.asarray(p_w, dtype=np.int64)
        # -------- items --------
        chunks = [_chunks(len(below_parts[p]), crit[p], int(p_w[p])) for p in range(P)]
        deps, dep_off, dep_cnt = [], [], []
        E = np.zeros(P, dtype=np.int64)
        owner_lists = []
        for p in range(P):
            lst = []
            for r0, r1 in chunks[p]:
                tg = np.unique(panel_of_row[below_parts[p][r0:r1]])
                lst.append((len(deps), len(tg)))
                deps.extend(tg.tolist())
                E[tg] += 1
            owner_lists.append(lst)
        part_off = np.zeros(P + 1, dtype=np.int64)
        np.cumsum([len(chunks[p]) * int(p_w[p]) for p in range(P)], out=part_off[1:])
        tri_len = np.asarray(p_tri_len, dtype=np.int64)

        def cost_diag(p):
            return 1.5 + tri_len[p] * 8 / 100e3

        def cost_chunk(p, r0, r1):
            return 0.8 + (r1 - r0) * p_w[p] * 8 / 40e3

        # lower schedule (panels are in a topological order already)
        ready = np.zeros(P)
        lower = []
        for p in range(P):
            st = ready[p]
            fin = st + cost_diag(p)
            lower.append((st, 0, p, IT_DIAG, p, 0, 0, 0, int(E[p]), 0))
            for q, (r0, r1) in enumerate(chunks[p]):
                off, cnt = owner_lists[p][q]
                cf = fin + cost_chunk(p, r0, r1)
                lower.append((fin, 1, p, IT_OFF, p, r0, r1, off, cnt, 0))
                tg = deps[off:off + cnt]
                ready[tg] = np.maximum(ready[tg], cf)
        # upper schedule: reverse topological order of panels
        done = np.zeros(P)
        upper = []
        for p in range(P - 1, -1, -1):
            st_d = 0.0
            for q, (r0, r1) in enumerate(chunks[p]):
                off, cnt = owner_lists[p][q]
                tg = deps[off:off + cnt]
                st = float(done[tg].max()) if cnt else 0.0
                upper.append((st, 0, -p, IT_OFFT, p, r0, r1, off, cnt, int(part_off[p] + q * p_w[p])))
                st_d = max(st_d, st + cost_chunk(p, r0, r1))
            upper.append((st_d, 1, -p, IT_DIAGT, p, 0, 0, 0, len(chunks[p]), int(part_off[p])))
            done[p] = st_d + cost_diag(p)
        lower.sort(key=lambda x: (x[0], x[1], x[2]))
        upper.sort(key=lambda x: (x[0], x[1], x[2]))
        to_items = lambda L: np.array([x[3:] for x in L], dtype=np.int32).reshape(-1, 7)  # noqa: E731
        items_l = np.concatenate([to_items(lower), np.zeros((len(lower), 1), dtype=np.int32)], axis=1)
        items_u = np.concatenate([to_items(upper), np.zeros((len(upper), 1), dtype=np.int32)], axis=1)
        # -------- contribution gather lists (lower) --------
        rows_all = np.concatenate(below_parts) if cb else np.zeros(0, dtype=np.int64)
        corder = np.argsort(rows_all, kind="stable")
        cin_ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows_all, minlength=n), out=cin_ptr[1:])
        max_chunk = max((r1 - r0 for ch in chunks for r0, r1 in ch), default=1)
        # staging buffer: the largest tri blob or factor chunk (rows x padded width)
        stage = max([int(tri_len.max()) if P else 0] +
                    [(r1 - r0) * (int(p_w[p]) + int(p_w[p]) % 2) for p in range(P) for r0, r1 in chunks[p]])

        cat = lambda parts, dt: (np.concatenate(parts).astype(dt, copy=False) if parts  # noqa: E731
                                 else np.zeros(1, dtype=dt))
    return {
        "n": n, "P": P, "items_l": items_l, "items_u": items_u, "p_start": np.asarray(p_start, dtype=np.int64),
        "p_w": p_w, "p_tri": np.asarray(p_tri, dtype=np.int64), "p_tri_len": tri_len,
        "p_pan": np.asarray(p_pan, dtype=np.int64), "p_cb": np.asarray(p_cb, dtype=np.int64),
        "p_below": np.asarray(p_below, dtype=np.int64), "tri": cat(tri_parts, np.float64),
        "tri_u": cat(tri_u_parts, np.float64),
        "pan": cat(pan_parts, np.float64), "below": cat(below_parts, np.int64),
        "deps": np.asarray(deps if deps else [0], dtype=np.int64), "cin_ptr": cin_ptr,
        # contributions land row-contiguous: entry i of the concatenated below lists
        # (panel order) goes to slot cslot[i]; row r reads cbuf[cin_ptr[r]:cin_ptr[r+1]]
        "cslot": _inverse(corder) if len(corder) else np.zeros(1, dtype=np.int64),
        "d": np.asarray(factors.d, dtype=np.float64), "perm": np.asarray(factors.plan.perm, dtype=np.int64),
        "ncbuf": cbuf, "npart": int(part_off[-1]), "max_chunk": int(max_chunk), "stage": int(stage),
        "bytes_tri": ct * 8,
        "bytes_pan": cp * 8,
    }


class DevicePanels:
    """Packed factor image in HBM + the libtsb handle (tsb_ldlt_create)."""

    def __init__(self, factors, stream=None, trace=False):
        t = _lib.require_cuda()
        H = pack(factors)
        n, P = H["n"], H["P"]
        items_l, items_u, tri_len = H["items_l"], H["items_u"], H["p_tri_len"]
        self.host = H if trace else None
        if trace:  # per-item timeline (globaltimer ns): take, ready, end, smid
            self.trace_l = t.zeros((len(items_l), 8), dtype=t.int64, device="cuda")
            self.trace_u = t.zeros((len(items_u), 8), dtype=t.int64, device="cuda")
        ctx = t.cuda.stream(stream) if stream is not None else _NullCtx()
        with ctx:
            up = lambda a: t.from_numpy(np.ascontiguousarray(a)).pin_memory().to("cuda", non_blocking=True)  # noqa: E731
            i32 = lambda a: up(np.asarray(a, dtype=np.int32))  # noqa: E731
            i64 = lambda a: up(np.asarray(a, dtype=np.int64))  # noqa: E731
            self.t = {
                "items_l": up(items_l), "items_u": up(items_u), "p_start": i32(H["p_start"]),
                "p_w": i32(H["p_w"]), "p_tri": i64(H["p_tri"]), "p_tri_len": i64(tri_len),
                "p_pan": i64(H["p_pan"]), "p_cb": i64(H["p_cb"]), "p_below": i64(H["p_below"]),
                "tri": up(H["tri"]), "tri_u": up(H["tri_u"]), "pan": up(H["pan"]), "below": i32(H["below"]), "deps": i32(H["deps"]),
                "cin_ptr": i64(H["cin_ptr"]), "cslot": i32(H["cslot"]), "d": up(H["d"]),
                "perm": i32(H["perm"]),
            }
            z = lambda k, dt: t.zeros(max(k, 1), dtype=dt, device="cuda")  # noqa: E731
            self.t.update(cbuf=z(H["ncbuf"], t.float64), part=z(H["npart"], t.float64), y=z(n, t.float64),
                          cnt=z(4 * P, t.int32), ctl=z(4, t.int32))
        self.n = n
        self.n_panels = P
        self.n_items = (len(items_l), len(items_u))
        self.bytes = {"tri": H["bytes_tri"], "pan": H["bytes_pan"]}
        max_chunk = H["max_chunk"]
        tp = lambda k: _lib.ptr(self.t[k])  # noqa: E731
        cnt = self.t["cnt"]
        self.desc = _lib.LdltDesc(
            n=n, n_panels=P, n_items_lower=len(items_l), n_items_upper=len(items_u), tile=TILE,
            panel_width=PANEL_W, stage_doubles=H["stage"], max_chunk_rows=int(max_chunk),
            grid=0, pad_=0,
            d_items_lower=tp("items_l"), d_items_upper=tp("items_u"), d_p_start=tp("p_start"), d_p_w=tp("p_w"),
            d_p_tri=tp("p_tri"), d_p_tri_len=tp("p_tri_len"), d_p_pan=tp("p_pan"), d_p_cb=tp("p_cb"),
            d_p_below=tp("p_below"), d_tri=tp("tri"), d_tri_u=tp("tri_u"), d_pan=tp("pan"), d_below=tp("below"), d_deps=tp("deps"),
            d_cin_ptr=tp("cin_ptr"), d_cslot=tp("cslot"), d_d=tp("d"), d_perm=tp("perm"),
            d_cbuf=tp("cbuf"), d_part=tp("part"), d_y=tp("y"),
            d_cnt0=_lib.ptr(cnt[0:P]) if P else tp("cnt"), d_cnt1=_lib.ptr(cnt[P:2 * P]) if P else tp("cnt"),
            d_cnt2=_lib.ptr(cnt[2 * P:3 * P]) if P else tp("cnt"), d_cnt3=_lib.ptr(cnt[3 * P:]) if P else tp("cnt"),
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
