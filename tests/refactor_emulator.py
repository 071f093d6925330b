"""NumPy emulator of the device refactorisation program (csrc/refactor.cu).

Test infrastructure: executes the host program planned by
paper_2306_05893_b200.refactor.plan_refactor op by op with the kernels'
tile semantics (64 x 64 tiles, task lists decoded the way the kernels decode
them), so the planner and the index math are checked on CPU against the host
factorisation before any GPU run.
"""

import numpy as np

from paper_2306_05893_b200 import refactor as R

NB = R.NB


def _tile(f, t):
    P, m, nf = int(f["P"]), int(f["m"]), int(f["nf"])
    s = t * NB if t < P else m + (t - P) * NB
    w = min(NB, m - t * NB) if t < P else min(NB, nf - s)
    return s, w


def _find(lists, lo, n, field, task):
    col = lists[lo:lo + n, field]
    e = int(np.searchsorted(col, task, side="right")) - 1
    return lo + e, task - int(col[e])


def _view(buf, off, ld, rows, cols):
    """Column-major (rows x cols) window at buf[off] with leading dimension ld (a copy)."""
    idx = off + np.arange(cols)[None, :] * ld + np.arange(rows)[:, None]
    return buf[idx]


def _put(buf, off, ld, val, mode="set", lower=False):
    rows, cols = val.shape
    r, c = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    msk = np.ones_like(r, dtype=bool) if not lower else r >= c
    idx = off + c * ld + r
    if mode == "set":
        buf[idx[msk]] = val[msk]
    else:
        buf[idx[msk]] -= val[msk]


def run(rp: R.RefactorPlan, values, tiles_l, tiles_u, tblk_l, tblk_u, n):
    ws = np.zeros(rp.ws_size)
    wb = np.zeros(rp.wb_size)
    inv = np.zeros(max(rp.inv_size, 1))
    F = rp.fronts
    L = rp.lists
    g = np.zeros(int((tiles_l["off"] + tiles_l["np"].astype(np.int64) * 64).max(initial=0)))
    gt = np.zeros(int((tiles_u["off"] + tiles_u["np"].astype(np.int64) * 64).max(initial=0)))
    d = np.zeros(n)
    bad = -1
    for op in rp.prog:
        kind, a, b, c, dd = (int(x) for x in op[:5])
        if kind in (R.OP_RECORD, R.OP_WAIT):  # stream ordering: the emulator runs ops in program order
            continue
        if kind == R.OP_SCATTER:
            ws[:] = 0.0
            ws[rp.sc_dst] = values[rp.sc_src]
        elif kind == R.OP_IDENT:
            wb[:] = 0.0
            for f in F:
                m = int(f["m"])
                wb[int(f["woff"]) + np.arange(m) * (m + 1)] = 1.0
        elif kind == R.OP_EXTEND:
            for pr in rp.pairs[a:b]:
                cf, pf = F[pr["child"]], F[pr["parent"]]
                tp = rp.tp[pr["tp_off"]: pr["tp_off"] + cf["na"]].astype(np.int64)
                mc, nc = int(cf["m"]), int(cf["nf"])
                U = _view(ws, int(cf["off"]) + mc * nc + mc, nc, int(cf["na"]), int(cf["na"]))
                i, j = np.tril_indices(int(cf["na"]))
                np.add.at(ws, int(pf["off"]) + tp[j] * int(pf["nf"]) + tp[i], U[i, j])
        elif kind == R.OP_DIAG:
            for e in range(b, b + c):
                fi = int(L[e, 0])
                f = F[fi]
                nf, k = int(f["nf"]), a
                w = min(NB, int(f["m"]) - k * NB)
                base = int(f["off"]) + k * NB * nf + k * NB
                S = np.tril(_view(ws, base, nf, w, w))
                try:
                    Cc = np.linalg.cholesky(S)
                except np.linalg.LinAlgError:
                    bad = fi if bad < 0 else bad
                    Cc = np.eye(w)
                W = np.linalg.inv(Cc)
                ws[base + np.arange(w) * (nf + 1)] = np.diagonal(Cc)  # the kernel stores diag(C_kk) only
                Wf = np.zeros((NB, NB))
                Wf[:w, :w] = np.tril(W)
                inv[int(f["ioff"]) + k * NB * NB + np.arange(NB * NB)] = Wf.T.ravel()  # column-major
        elif kind in (R.OP_PANEL, R.OP_UPDATE):
            k = a
            for task in range(dd):
                e, local = _find(L, b, c, 1 if kind == R.OP_PANEL else 2, task)
                f = F[int(L[e, 0])]
                nf, c0 = int(f["nf"]), k * NB
                w = min(NB, int(f["m"]) - c0)
                if kind == R.OP_PANEL:
                    r0, h = _tile(f, k + 1 + local)
                    src = int(f["off"]) + c0 * nf + r0
                    A = _view(ws, src, nf, h, w)
                    Wm = inv[int(f["ioff"]) + k * NB * NB + np.arange(NB * NB)].reshape(NB, NB).T[:w, :w]
                    _put(ws, src, nf, A @ Wm.T)
                else:
                    rr = int((np.sqrt(8 * local + 1) - 1) // 2)
                    while (rr + 1) * (rr + 2) // 2 <= local:
                        rr += 1
                    while rr * (rr + 1) // 2 > local:
                        rr -= 1
                    ss = local - rr * (rr + 1) // 2
                    i, j = k + 1 + rr, k + 1 + ss
                    ri, hi = _tile(f, i)
                    rj, hj = _tile(f, j)
                    Ai = _view(ws, int(f["off"]) + c0 * nf + ri, nf, hi, w)
                    Aj = _view(ws, int(f["off"]) + c0 * nf + rj, nf, hj, w)
                    _put(ws, int(f["off"]) + rj * nf + ri, nf, Ai @ Aj.T, mode="sub", lower=(i == j))
        elif kind in (R.OP_TSCALE, R.OP_TUPDATE):
            k = a
            for task in range(dd):
                e, local = _find(L, b, c, 1 if kind == R.OP_TSCALE else 2, task)
                f = F[int(L[e, 0])]
                m, nf, P = int(f["m"]), int(f["nf"]), int(f["P"])
                idx = local if kind == R.OP_TSCALE else local // k
                if idx < P - k:
                    i = k + idx
                    buf, base, ld, rows = wb, int(f["woff"]) + i * NB, m, min(NB, m - i * NB)
                else:
                    bb = idx - (P - k)
                    buf, base, ld, rows = ws, int(f["off"]) + m + bb * NB, nf, min(NB, int(f["na"]) - bb * NB)
                w = min(NB, m - k * NB)
                X = _view(buf, base + k * NB * ld, ld, rows, w)
                if kind == R.OP_TSCALE:
                    Wm = inv[int(f["ioff"]) + k * NB * NB + np.arange(NB * NB)].reshape(NB, NB).T[:w, :w]
                    _put(buf, base + k * NB * ld, ld, X @ Wm)
                else:
                    j = local % k
                    Ckj = _view(ws, int(f["off"]) + j * NB * nf + k * NB, nf, w, NB)
                    _put(buf, base + j * NB * ld, ld, X @ Ckj, mode="sub")
        elif kind == R.OP_PACK:
            def gvals(f, r, col):  # vectorised gval of the kernel
                m, nf = int(f["m"]), int(f["nf"])
                top = r < m
                rt = np.where(top, r, 0)
                lin = ws[int(f["off"]) + rt * nf + rt] * wb[int(f["woff"]) + np.where(top, col, 0) * m + rt]
                lin = np.where(r == col, 1.0, np.where(r < col, 0.0, lin))
                mm = ws[int(f["off"]) + np.where(top, 0, col) * nf + np.where(top, m, r)]
                return np.where(top, lin, mm)

            for up, T, tb, out in ((False, tiles_l, tblk_l, g), (True, tiles_u, tblk_u, gt)):
                for t, tb_i in zip(T, tb):
                    f = F[tb_i]
                    idx = np.arange(int(t["np"]) * 64)
                    p, rem = np.divmod(idx, 64)
                    kk, hh = np.divmod(rem, 2)
                    row, col = int(t["row0"]) + kk, int(t["tl"]) + 2 * p + hh
                    live = kk < int(t["nrows"])
                    if not up:
                        live &= col < np.minimum(row + 1, int(f["m"]))
                        rr, cc = row, col
                    else:
                        live &= (col >= row) & (col < int(f["nf"]))
                        rr, cc = col, row
                    v = np.zeros(len(idx))
                    if live.any():
                        v[live] = gvals(f, rr[live], cc[live])
                    out[int(t["off"]) + idx] = v
            for f in F:
                m, nf = int(f["m"]), int(f["nf"])
                cdiag = ws[int(f["off"]) + np.arange(m) * (nf + 1)]
                d[int(f["start"]) + np.arange(m)] = cdiag * cdiag
        else:
            raise AssertionError(f"unknown op {kind}")
    return g, gt, d, bad
