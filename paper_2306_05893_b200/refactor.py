"""Device LDL^T refactorisation (numeric phase of ldlt_factor, ndprecond.py:501-572).

The reference refactors on a host thread (AsyncPreconditioner, ndprecond.py:
714-831) and the factor is several steps stale when it lands; here the
numeric factorisation runs on the B200 straight from the device matrix into
the sweep layout the apply reads (csrc/refactor.cu):

    plan_refactor(symbolic, plan)   once per pattern (host): fronts, task
                                    lists, A-entry scatter map, extend-add
                                    pairs and the launch program
    DeviceRefactor(a, plan)         device workspaces + a structure-only
                                    sweep image (same tiles/items as the
                                    host-packed factor of the same pattern)
    .factor(a, source_step)         one tsb_refactor_run -> LdlFactors whose
                                    device image holds the new values

Front layout (column-major, nf = m + na): rows [0, m) the block, rows
[m, nf) its coupling rows `couple` (= the factor's anc); pivot tiles of 64
end at m, coupling tiles start at m.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

NB = 64

FRONT_DTYPE = np.dtype([("off", "<i8"), ("woff", "<i8"), ("ioff", "<i8"), ("m", "<i4"), ("na", "<i4"),
                        ("nf", "<i4"), ("P", "<i4"), ("NT", "<i4"), ("start", "<i4")])
assert FRONT_DTYPE.itemsize == 48
PAIR_DTYPE = np.dtype([("child", "<i4"), ("parent", "<i4"), ("tp_off", "<i8")])
assert PAIR_DTYPE.itemsize == 16
OP_SCATTER, OP_EXTEND, OP_DIAG, OP_PANEL, OP_UPDATE, OP_TSCALE, OP_TUPDATE, OP_PACK, OP_IDENT, OP_RECORD, OP_WAIT = \
    range(1, 12)
SIDE = 1  # op[5]: the handle's side stream


class _StructBlock:
    """Block of a factor whose values live on the device (duck-types _BlockFactor)."""

    l11 = None
    l21 = None

    def __init__(self, start, stop, level, anc, tile):
        self.start, self.stop, self.level, self.anc, self.tile = start, stop, level, anc, tile


class _StructFactors:
    def __init__(self, plan, blocks):
        self.plan, self.d, self.blocks = plan, None, blocks


@dataclass
class RefactorPlan:
    fronts: np.ndarray        # FRONT_DTYPE per front (= handle block, start order)
    lists: np.ndarray         # int32 [.][4]
    sc_src: np.ndarray        # int32
    sc_dst: np.ndarray        # int64
    pairs: np.ndarray         # PAIR_DTYPE
    tp: np.ndarray            # int32
    prog: np.ndarray          # int64 [.][8]
    ws_size: int
    wb_size: int
    inv_size: int
    blocks: list              # _StructBlock per front
    heights: np.ndarray
    flops: float              # dense fp64 flops of one refactorisation (FMA = 2)


def plan_refactor(symbolic, plan) -> RefactorPlan:
    """Host plan of the device refactorisation of one pattern (see module doc)."""
    order = list(symbolic.order)
    nb = len(order)
    pos = {b: i for i, b in enumerate(order)}
    m = np.array([plan.blocks[b].size for b in order], dtype=np.int64)
    na = np.array([len(symbolic.couple[b]) for b in order], dtype=np.int64)
    nf = m + na
    P = (m + NB - 1) // NB
    NT = P + (na + NB - 1) // NB

    def excl(x):
        o = np.zeros(len(x) + 1, dtype=np.int64)
        np.cumsum(x, out=o[1:])
        return o

    off, woff, ioff = excl(nf * nf), excl(m * m), excl(P * NB * NB)
    fronts = np.zeros(nb, dtype=FRONT_DTYPE)
    fronts["off"], fronts["woff"], fronts["ioff"] = off[:-1], woff[:-1], ioff[:-1]
    fronts["m"], fronts["na"], fronts["nf"], fronts["P"], fronts["NT"] = m, na, nf, P, NT
    fronts["start"] = [plan.blocks[b].start for b in order]

    parent = np.array([pos[symbolic.parent[b]] if b in symbolic.parent else -1 for b in order], dtype=np.int64)
    children = [[] for _ in range(nb)]
    for i in range(nb):
        if parent[i] >= 0 and na[i] > 0:
            children[parent[i]].append(i)
    height = np.zeros(nb, dtype=np.int64)
    for i in range(nb):  # start order: children first
        if children[i]:
            height[i] = 1 + max(height[c] for c in children[i])
            if any(c >= i for c in children[i]):
                raise ValueError("dissection blocks are not in start order")

    # A entries -> fronts (lower triangle of the diagonal block + the coupling panel)
    src, dst = [], []
    for i, b in enumerate(order):
        mi, fi = int(m[i]), int(nf[i])
        lr, lc = np.divmod(symbolic.ds_dst[b], mi)
        keep = lr >= lc
        src.append(symbolic.ds_src[b][keep])
        dst.append(off[i] + lc[keep] * fi + lr[keep])
        if len(symbolic.pn_dst[b]):
            k, lr = np.divmod(symbolic.pn_dst[b], mi)
            src.append(symbolic.pn_src[b])
            dst.append(off[i] + lr * fi + mi + k)
    sc_src = np.concatenate(src).astype(np.int32) if src else np.zeros(0, np.int32)
    sc_dst = np.concatenate(dst).astype(np.int64) if dst else np.zeros(0, np.int64)

    prog, lists, pairs, tps = [], [], [], []
    tp_pos = 0

    def op(*a, stream=0):
        row = list(a) + [0] * (8 - len(a))
        row[5] = stream
        prog.append(row)

    def add_list(entries):
        o = len(lists)
        lists.extend(entries)
        return o

    op(OP_SCATTER, len(sc_src))
    op(OP_IDENT)
    flops = 0.0
    H = int(height.max()) + 1 if nb else 0
    for h in range(H):
        at = np.flatnonzero(height == h)
        if h > 0:
            nq = max(len(children[p]) for p in at)
            for q in range(nq):
                p0 = len(pairs)
                mx = 0
                for p in at:
                    if q < len(children[p]):
                        c = children[p][q]
                        tp = np.asarray(symbolic.to_parent[order[c]], dtype=np.int64)
                        pairs.append((c, p, tp_pos))
                        tps.append(tp)
                        tp_pos += len(tp)
                        mx = max(mx, int(na[c]))
                op(OP_EXTEND, p0, len(pairs), mx)
        kmax = int(P[at].max()) if len(at) else 0
        for k in range(kmax):
            act = [int(i) for i in at if P[i] > k]
            ent, pp, uu = [], 0, 0
            for i in act:
                R = int(NT[i]) - k - 1
                ent.append((i, pp, uu, 0))
                pp += R
                uu += R * (R + 1) // 2
            lo = add_list(ent)
            op(OP_DIAG, k, lo, len(act))
            op(OP_PANEL, k, lo, len(act), pp)
            op(OP_UPDATE, k, lo, len(act), uu)
        # right solve of this height on the side stream (it only touches the
        # fronts' L21 / C^-1 parts, never the update matrices the parents read)
        if len(at):
            op(OP_RECORD, h)
            op(OP_WAIT, h, stream=SIDE)
            for k in range(kmax - 1, -1, -1):
                act = [int(i) for i in at if P[i] > k]
                ent, ss, uu = [], 0, 0
                for i in act:
                    rows = int(P[i]) - k + (int(na[i]) + NB - 1) // NB
                    ent.append((i, ss, uu, 0))
                    ss += rows
                    uu += rows * k
                lo = add_list(ent)
                op(OP_TSCALE, k, lo, len(act), ss, stream=SIDE)
                op(OP_TUPDATE, k, lo, len(act), uu, stream=SIDE)
    for i in range(nb):  # partial Cholesky + U + right solve (FMA = 2 flops)
        mi, ai = float(m[i]), float(na[i])
        flops += mi ** 3 / 3 + mi * mi * ai + mi * ai * ai + mi ** 3 / 3 + ai * mi * mi
    op(OP_RECORD, H, stream=SIDE)
    op(OP_WAIT, H)
    op(OP_PACK)

    pair_arr = np.zeros(len(pairs), dtype=PAIR_DTYPE)
    if pairs:
        arr = np.array(pairs, dtype=np.int64)
        pair_arr["child"], pair_arr["parent"], pair_arr["tp_off"] = arr.T
    blocks = [_StructBlock(plan.blocks[b].start, plan.blocks[b].stop, plan.blocks[b].level,
                           np.asarray(symbolic.couple[b], dtype=np.int64), symbolic.tile) for b in order]
    return RefactorPlan(
        fronts=fronts, lists=np.asarray(lists, dtype=np.int32).reshape(-1, 4),
        sc_src=sc_src, sc_dst=sc_dst, pairs=pair_arr,
        tp=np.concatenate(tps).astype(np.int32) if tps else np.zeros(0, np.int32),
        prog=np.asarray(prog, dtype=np.int64).reshape(-1, 8),
        ws_size=int(off[-1]), wb_size=int(woff[-1]), inv_size=int(ioff[-1]),
        blocks=blocks, heights=height, flops=flops,
    )


class DeviceRefactor:
    """Device refactorisation of one matrix pattern + dissection plan.

    `buffers` sweep images are kept and filled round-robin, so a factor
    handed out earlier stays valid while the next one is computed (the
    AsyncPreconditioner swaps them at step boundaries)."""

    def __init__(self, a, plan, tile: int = 16, symbolic=None, buffers: int = 1):
        from ._ldlt_pack import DevicePanels
        from .ndprecond import _build_symbolic, _pattern_key

        t = _lib.require_cuda()
        if symbolic is None or symbolic.pattern_key != _pattern_key(a) or symbolic.tile != tile:
            symbolic = _build_symbolic(a, plan, tile)
        self.symbolic, self.plan, self.tile = symbolic, plan, tile
        R = plan_refactor(symbolic, plan)
        self.rplan = R
        self.struct = _StructFactors(plan, R.blocks)
        nlev = 1 + max((bf.level for bf in R.blocks), default=0)
        self.levels = [[bf for bf in R.blocks if bf.level == lv] for lv in range(nlev)]
        self.images = [DevicePanels(self.struct, merge=0) for _ in range(max(1, buffers))]
        self._next = 0
        img = self.images[0]
        if len(img.tile_blk[0]) != img.t["tiles_l"].numel() // 32 or len(R.fronts) != img.n_blocks:
            raise ValueError("sweep image does not match the refactor plan")
        up = lambda a_: t.from_numpy(np.ascontiguousarray(a_)).to("cuda")  # noqa: E731
        nz = lambda a_: a_ if len(a_) else np.zeros(1, dtype=a_.dtype)  # noqa: E731
        self.d = {
            "fronts": up(nz(R.fronts).view(np.uint8)), "lists": up(nz(R.lists.ravel())),
            "sc_src": up(nz(R.sc_src)), "sc_dst": up(nz(R.sc_dst)), "pairs": up(nz(R.pairs).view(np.uint8)),
            "tp": up(nz(R.tp)), "tbl": up(nz(img.tile_blk[0])), "tbu": up(nz(img.tile_blk[1])),
            "ws": t.empty(max(R.ws_size, 1), dtype=t.float64, device="cuda"),
            "wb": t.empty(max(R.wb_size, 1), dtype=t.float64, device="cuda"),
            "inv": t.empty(max(R.inv_size, 1), dtype=t.float64, device="cuda"),
            "ctl": t.zeros(4, dtype=t.int32, device="cuda"),
        }
        self._prog = np.ascontiguousarray(R.prog)
        P = lambda k: _lib.ptr(self.d[k])  # noqa: E731
        self.desc = _lib.RefactorDesc(
            n_fronts=len(R.fronts), n_prog=len(R.prog), h_prog=self._prog.ctypes.data,
            d_fronts=P("fronts"), d_lists=P("lists"), d_sc_src=P("sc_src"), d_sc_dst=P("sc_dst"),
            d_pairs=P("pairs"), d_tp=P("tp"), d_tiles_lower=_lib.ptr(img.t["tiles_l"]),
            d_tiles_upper=_lib.ptr(img.t["tiles_u"]), d_tile_blk_lower=P("tbl"), d_tile_blk_upper=P("tbu"),
            n_tiles_lower=len(img.tile_blk[0]), n_tiles_upper=len(img.tile_blk[1]),
            d_ws=P("ws"), d_wb=P("wb"), d_inv=P("inv"), ws_size=R.ws_size, wb_size=R.wb_size, d_ctl=P("ctl"),
        )
        self._lib = _lib.load()
        h = C.c_void_p()
        _lib.check(self._lib.tsb_refactor_create(C.byref(self.desc), C.byref(h)), "refactor_create")
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self._lib.tsb_refactor_destroy(self.h)
        except Exception:
            pass

    @property
    def workspace_bytes(self) -> int:
        return 8 * (self.rplan.ws_size + self.rplan.wb_size + self.rplan.inv_size)

    def enqueue(self, a, image=None):
        """Enqueue the refactorisation of `a`'s values into a sweep image (current stream)."""
        img = image if image is not None else self.images[0]
        vals = a.device_values()
        if vals.numel() != len(a.col_ind):
            raise ValueError("matrix values do not match the pattern")
        _lib.check(self._lib.tsb_refactor_run(self.h, _lib.ptr(vals), _lib.ptr(img.t["g"]), _lib.ptr(img.t["gt"]),
                                              _lib.ptr(img.t["d"]), _lib.stream_ptr()), "refactor_run")
        return img

    def failed_block(self) -> int:
        """-1, or the dissection block whose pivot was not positive (synchronises)."""
        v = int(self.d["ctl"][0].item())
        return -1 if v == 0 else v - 1

    def factor(self, a, source_step: int = 0, check: bool = True):
        """Refactor `a` on the device -> LdlFactors backed by the next sweep image."""
        from .ndprecond import IndefiniteMatrixError, _pattern_key

        if _pattern_key(a) != self.symbolic.pattern_key:
            raise ValueError("matrix pattern differs from the planned one")
        img = self.images[self._next]
        self._next = (self._next + 1) % len(self.images)
        self.enqueue(a, img)
        if check:
            bad = self.failed_block()
            if bad >= 0:
                bf = self.rplan.blocks[bad]
                raise IndefiniteMatrixError(f"non-positive pivot while factoring block [{bf.start}, {bf.stop})")
        return make_factors(self, img, source_step)


def make_factors(rf: DeviceRefactor, img, source_step: int):
    from .ndprecond import DeviceLdlFactors

    return DeviceLdlFactors(d=None, plan=rf.plan, source_step=source_step, blocks=rf.rplan.blocks,
                            levels=rf.levels, symbolic=rf.symbolic, _device=img)


def ldlt_factor_device(a, plan, tile: int = 16, symbolic=None, source_step: int = 0):
    """ldlt_factor (ndprecond.py:501-572) computed on the device; the returned
    factors live in HBM (their host view is downloaded on demand)."""
    from .ndprecond import PrecondError

    if a.nrows != a.ncols or a.nrows != plan.n:
        raise PrecondError(f"matrix is {a.nrows}x{a.ncols} but the plan covers {plan.n} indices")
    if tile < 1:
        raise PrecondError(f"tile must be >= 1, got {tile}")
    return DeviceRefactor(a, plan, tile, symbolic).factor(a, source_step)
