"""Nested-dissection LDL^T preconditioner (drop-in for tetsim.ndprecond, ndprecond.py:1-831).

Split exactly as the paper splits it:
  host setup   nested_dissection (native C++, same algorithm/tie-breaks as the
               reference so plans are identical), ldlt_factor (dense per-front
               Cholesky on the host BLAS, multifrontal extend-add), packing of
               the factor into the device layout, AsyncPreconditioner's
               background refactorisation;
  device       solve_lower / solve_upper / apply: level-scheduled sweeps over
               the dissection tree in libtsb (csrc/ldlt.cu), uploaded once per
               factor refresh on a side stream and swapped at step boundaries.
"""

from __future__ import annotations

import ctypes as C
import enum
import logging
from concurrent.futures import Future, ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .assembly import CsrMatrix
from .mesh import Graph

__all__ = [
    "PrecondError",
    "IndefiniteMatrixError",
    "LifecycleError",
    "Block",
    "DissectionPlan",
    "LdlFactors",
    "PrecondStatus",
    "AsyncPreconditioner",
    "nested_dissection",
    "expand_plan",
    "graph_from_pattern",
    "count_coupling_violations",
    "ldlt_factor",
    "ldlt_factor_device",
    "DeviceLdlFactors",
    "solve_lower",
    "solve_upper",
    "apply",
]

logger = logging.getLogger(__name__)


class PrecondError(ValueError):
    pass


class IndefiniteMatrixError(PrecondError):
    """Zero or negative pivot: the assembled system is not positive definite."""


class LifecycleError(PrecondError):
    """Preconditioner applied before factors are ready."""


@dataclass(frozen=True)
class Block:
    """Dissection-tree node owning permuted range [start, stop); [tree_start, stop) spans its subtree."""

    start: int
    stop: int
    tree_start: int
    kind: str
    children: tuple
    level: int = 0

    @property
    def size(self) -> int:
        return self.stop - self.start


@dataclass(frozen=True)
class DissectionPlan:
    n: int
    perm: np.ndarray
    iperm: np.ndarray
    blocks: tuple
    levels: tuple
    leaf_threshold: int

    def block_of_index(self) -> np.ndarray:
        owner = np.empty(self.n, dtype=np.int64)
        for bid, blk in enumerate(self.blocks):
            owner[blk.start: blk.stop] = bid
        return owner


# ---------------------------------------------------------------------------
# ordering (host setup, native)
# ---------------------------------------------------------------------------

def nested_dissection(graph: Graph, leaf_threshold: int = 64) -> DissectionPlan:
    """Recursive bisection -> permutation, block tree, level schedule (ndprecond.py:234-267)."""
    if leaf_threshold < 1:
        raise PrecondError(f"leaf_threshold must be >= 1, got {leaf_threshold}")
    n = graph.n
    if n == 0:
        return DissectionPlan(0, np.empty(0, dtype=np.int64), np.empty(0, dtype=np.int64), (), (), leaf_threshold)
    lib = _lib.load()
    indptr = np.ascontiguousarray(graph.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(graph.indices, dtype=np.int64)
    perm = np.empty(n, dtype=np.int64)
    nb = C.c_int64(0)
    start = np.empty(n, dtype=np.int64)
    stop = np.empty(n, dtype=np.int64)
    tstart = np.empty(n, dtype=np.int64)
    is_sep = np.empty(n, dtype=np.int32)
    cptr = np.empty(n + 1, dtype=np.int64)
    child = np.empty(max(n, 1), dtype=np.int64)
    p = lambda a: a.ctypes.data  # noqa: E731
    st = lib.tsb_nested_dissection(n, p(indptr), p(indices), int(leaf_threshold), p(perm), C.byref(nb),
                                   p(start), p(stop), p(tstart), p(is_sep), p(cptr), p(child))
    if st != 0:
        raise PrecondError("nested dissection failed")
    nb = nb.value
    level = np.zeros(nb, dtype=np.int64)
    raw = []
    for b in range(nb):
        ch = tuple(int(c) for c in child[cptr[b]:cptr[b + 1]])
        level[b] = 0 if not ch else 1 + max(level[c] for c in ch)
        raw.append(Block(int(start[b]), int(stop[b]), int(tstart[b]),
                         "separator" if is_sep[b] else "leaf", ch, int(level[b])))
    nlev = int(level.max()) + 1
    groups = [[] for _ in range(nlev)]
    for b, blk in enumerate(raw):
        groups[blk.level].append(b)
    levels = tuple(tuple(sorted(g, key=lambda b: raw[b].start)) for g in groups)
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    return DissectionPlan(n, perm, iperm, tuple(raw), levels, leaf_threshold)


def expand_plan(plan: DissectionPlan, dofs_per_vertex: int = 3) -> DissectionPlan:
    k = dofs_per_vertex
    perm = (k * plan.perm[:, None] + np.arange(k)).ravel()
    iperm = np.empty(k * plan.n, dtype=np.int64)
    iperm[perm] = np.arange(k * plan.n)
    blocks = tuple(Block(k * b.start, k * b.stop, k * b.tree_start, b.kind, b.children, b.level)
                   for b in plan.blocks)
    return DissectionPlan(k * plan.n, perm, iperm, blocks, plan.levels, plan.leaf_threshold)


def graph_from_pattern(a: CsrMatrix) -> Graph:
    """Vertex graph of a CSR pattern (ndprecond.py:282-292): i ~ j when
    A_ij or A_ji is stored, i != j; neighbour lists sorted, no self loops.
    Restated: one symmetric boolean structure through scipy.sparse."""
    import scipy.sparse as sp

    n = a.nrows
    pat = sp.csr_matrix((np.ones(a.nnz, dtype=np.int8), np.asarray(a.col_ind), np.asarray(a.row_ptr)), shape=(n, n))
    sym = ((pat + pat.T) != 0).tocsr()
    sym.setdiag(0)
    sym.eliminate_zeros()
    sym.sort_indices()
    return Graph(n=n, indptr=sym.indptr.astype(np.int64), indices=sym.indices.astype(np.int64))


def count_coupling_violations(a: CsrMatrix, plan: DissectionPlan) -> int:
    """Stored entries (i, j) whose permuted positions lie in blocks that are
    not on one root path (ndprecond.py:295-309): an entry is legal iff one
    position falls inside the other block's subtree range [tree_start, stop)."""
    owner = plan.block_of_index()
    lo = np.fromiter((b.tree_start for b in plan.blocks), dtype=np.int64, count=len(plan.blocks))
    hi = np.fromiter((b.stop for b in plan.blocks), dtype=np.int64, count=len(plan.blocks))
    p_row = plan.iperm[np.repeat(np.arange(a.nrows), np.diff(a.row_ptr))]
    p_col = plan.iperm[np.asarray(a.col_ind)]
    in_row_tree = (lo[owner[p_row]] <= p_col) & (p_col < hi[owner[p_row]])
    in_col_tree = (lo[owner[p_col]] <= p_row) & (p_row < hi[owner[p_col]])
    return int(np.sum(~(in_row_tree | in_col_tree)))


# ---------------------------------------------------------------------------
# factorisation (host setup; multifrontal restatement of ndprecond.py:312-587)
# ---------------------------------------------------------------------------

def _pattern_key(a: CsrMatrix) -> tuple:
    return (id(a.row_ptr), id(a.col_ind), a.nnz)


@dataclass
class LdlSymbolic:
    """Pattern-dependent data: per block the CSR entries of its diagonal block
    and coupling panel, its ancestor set, and where it lands in its parent front."""

    n: int
    tile: int
    order: list
    couple: dict
    ds_src: dict
    ds_dst: dict
    pn_src: dict
    pn_dst: dict
    parent: dict
    to_parent: dict
    pattern_key: tuple


def _build_symbolic(a: CsrMatrix, plan: DissectionPlan, tile: int) -> LdlSymbolic:
    n = a.nrows
    row_of = np.repeat(np.arange(n), np.diff(a.row_ptr))
    pi = plan.iperm[row_of]
    pj = plan.iperm[a.col_ind]
    by_row = np.argsort(pi, kind="stable")
    rptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(pi, minlength=n), out=rptr[1:])
    order = sorted(range(len(plan.blocks)), key=lambda b: plan.blocks[b].start)
    parent = {}
    for b, blk in enumerate(plan.blocks):
        for c in blk.children:
            parent[c] = b
    couple, ds_src, ds_dst, pn_src, pn_dst, to_parent = {}, {}, {}, {}, {}, {}
    for b in order:
        blk = plan.blocks[b]
        s, e, m = blk.start, blk.stop, blk.size
        ent = by_row[rptr[s]:rptr[e]]
        lr, cols = pi[ent] - s, pj[ent]
        inb = (cols >= s) & (cols < e)
        right = cols >= e
        ds_src[b] = ent[inb]
        ds_dst[b] = lr[inb] * m + (cols[inb] - s)
        parts = [cols[right]] + [couple[c][couple[c] >= e] for c in blk.children]
        cb = np.unique(np.concatenate(parts)) if parts else np.empty(0, dtype=np.int64)
        couple[b] = cb
        pn_src[b] = ent[right]
        pn_dst[b] = np.searchsorted(cb, cols[right]) * m + lr[right]
    for b in order:
        cb = couple[b]
        if not len(cb):
            to_parent[b] = np.empty(0, dtype=np.int64)
            continue
        p = parent.get(b)
        if p is None:
            raise PrecondError("symbolic coupling sets are inconsistent (root block with ancestors)")
        pb = plan.blocks[p]
        in_rows = (cb >= pb.start) & (cb < pb.stop)
        pos = np.empty(len(cb), dtype=np.int64)
        pos[in_rows] = cb[in_rows] - pb.start
        pc = couple[p]
        k = np.searchsorted(pc, cb[~in_rows])
        if np.any(k >= len(pc)) or np.any(pc[np.minimum(k, len(pc) - 1)] != cb[~in_rows]):
            raise PrecondError("symbolic coupling sets are inconsistent")
        pos[~in_rows] = pb.size + k
        to_parent[b] = pos
    return LdlSymbolic(n, tile, order, couple, ds_src, ds_dst, pn_src, pn_dst, parent, to_parent,
                       _pattern_key(a))


@dataclass
class _BlockFactor:
    start: int
    stop: int
    level: int
    anc: np.ndarray
    l11: np.ndarray
    l21: np.ndarray
    tile: int
    tile_inv: list


def _tile_inverses(l11: np.ndarray, tile: int) -> list:
    m = len(l11)
    out = []
    full = m // tile
    if full:
        idx = np.arange(full) * tile
        stacked = np.stack([l11[i:i + tile, i:i + tile] for i in idx])
        out.extend(np.linalg.inv(stacked))
    if m % tile:
        out.append(np.linalg.inv(l11[full * tile:, full * tile:]))
    return out


@dataclass
class LdlFactors:
    """LDL^T factors in dissection order (reference ndprecond.py:470-498) plus
    their device image (`device()`, built once per factor object)."""

    d: np.ndarray
    plan: DissectionPlan
    source_step: int
    blocks: list
    levels: list
    symbolic: LdlSymbolic = field(repr=False, default=None)
    _l_matrix: CsrMatrix | None = field(repr=False, default=None)
    _device: object = field(repr=False, default=None)

    @property
    def l_matrix(self) -> CsrMatrix:
        if self._l_matrix is None:
            self._l_matrix = _blocks_to_csr(self.plan.n, self.blocks)
        return self._l_matrix

    @property
    def fill_in(self) -> int:
        """nnz of the strict lower triangle of L, exact zeros dropped
        (ndprecond.py:493-495) -- counted block by block, without
        materialising l_matrix (~100 GB of COO at 1M nodes)."""
        if self._l_matrix is not None:
            return self._l_matrix.nnz
        return int(sum(np.count_nonzero(np.tril(np.asarray(bf.l11), -1)) + np.count_nonzero(bf.l21)
                       for bf in self.blocks))

    def device(self) -> "DeviceFactors":
        if self._device is None:
            self._device = DeviceFactors(self)
        return self._device

    def apply(self, r, workers: int = 1):
        return apply(self, r, workers=workers)


@dataclass
class DeviceLdlFactors(LdlFactors):
    """LdlFactors computed on the device (refactor.DeviceRefactor): the values
    exist only in the sweep image (`device()`); `to_host()` downloads them as
    a plain LdlFactors (L11 = inv(Linv), L21 = M L11) for host-side use."""

    _host: LdlFactors | None = field(repr=False, default=None)

    def to_host(self) -> LdlFactors:
        if self._host is None:
            from scipy.linalg import lapack

            from ._ldlt_pack import TILE_DTYPE, untile

            img = self._device
            tiles = img.t["tiles_l"].cpu().numpy().view(TILE_DTYPE)
            g = img.t["g"].cpu().numpy()
            tblk = img.tile_blk[0]
            blocks = []
            for i, bf in enumerate(self.blocks):
                m, na = bf.stop - bf.start, len(bf.anc)
                sel = np.flatnonzero(tblk == i)
                tl = [(int(x["off"]), int(x["tl"]), int(x["np"]), int(x["row0"]), int(x["nrows"])) for x in tiles[sel]]
                G = untile(tl, g, m + na, m)
                l11, info = lapack.dtrtri(np.ascontiguousarray(G[:m]), lower=1, unitdiag=1)
                if info != 0:
                    raise PrecondError(f"singular device factor block at {bf.start}")
                l11 = np.tril(l11, -1) + np.eye(m)
                l21 = G[m:] @ l11 if na else np.empty((0, m))
                blocks.append(_BlockFactor(bf.start, bf.stop, bf.level, bf.anc, l11, l21, bf.tile,
                                           _tile_inverses(l11, bf.tile)))
            d = img.t["d"].cpu().numpy().copy()
            nlev = len(self.levels)
            levels = [[b for b in blocks if b.level == lv] for lv in range(nlev)]
            self._host = LdlFactors(d, self.plan, self.source_step, blocks, levels, self.symbolic)
        return self._host

    @property
    def l_matrix(self) -> CsrMatrix:
        return self.to_host().l_matrix

    @property
    def fill_in(self) -> int:
        return self.to_host().fill_in


def ldlt_factor(a: CsrMatrix, plan: DissectionPlan, tile: int = 16, symbolic: LdlSymbolic | None = None,
                source_step: int = 0) -> LdlFactors:
    """Sparse LDL^T of an SPD matrix, front by front in start order (host BLAS).

    Front of block b = [A_bb, A_b,anc; A_anc,b, 0] plus the extend-added
    update matrices of its children; dense Cholesky C of the leading block
    gives d = diag(C)^2, L11 = C / diag(C); the coupling panel
    L21 = F21 C^-T / diag(C); U = F22 - (F21 C^-T)(F21 C^-T)^T goes to the parent.
    """
    if a.nrows != a.ncols or a.nrows != plan.n:
        raise PrecondError(f"matrix is {a.nrows}x{a.ncols} but the plan covers {plan.n} indices")
    if tile < 1:
        raise PrecondError(f"tile must be >= 1, got {tile}")
    if symbolic is None or symbolic.pattern_key != _pattern_key(a) or symbolic.tile != tile:
        symbolic = _build_symbolic(a, plan, tile)
    from scipy.linalg import solve_triangular
    from threadpoolctl import threadpool_limits

    vals = np.asarray(a.values, dtype=np.float64)
    limiter = threadpool_limits(limits=1, user_api="blas")  # small fronts: threads only thrash
    try:
        n = a.nrows
        d_out = np.empty(n)
        pending: dict[int, list] = {}
        factors = {}
        for b in symbolic.order:
            blk = plan.blocks[b]
            s, e, m = blk.start, blk.stop, blk.size
            cb = symbolic.couple[b]
            na = len(cb)
            F = np.zeros((m + na, m + na))
            F.reshape(-1)[_front_index(symbolic.ds_dst[b], m, m + na)] = vals[symbolic.ds_src[b]]
            if na:
                r_, c_ = np.divmod(symbolic.pn_dst[b], m)
                F[m + r_, c_] = vals[symbolic.pn_src[b]]
            for pos, U in pending.pop(b, []):
                F[np.ix_(pos, pos)] += U
            big = m + na >= _BIG_FRONT
            if big:
                limiter.restore_original_limits()
            try:
                c = np.linalg.cholesky(F[:m, :m])
            except np.linalg.LinAlgError as exc:
                raise IndefiniteMatrixError(f"non-positive pivot while factoring block [{s}, {e}): {exc}") from None
            dv = np.diagonal(c).copy()
            d_out[s:e] = dv * dv
            l11 = c / dv[None, :]
            if na:
                ls = solve_triangular(c, F[m:, :m].T, lower=True, check_finite=False).T
                l21 = ls / dv[None, :]
                U = F[m:, m:] - ls @ ls.T
                pending.setdefault(symbolic.parent[b], []).append((symbolic.to_parent[b], U))
            else:
                l21 = np.empty((0, m))
            if big:
                limiter = threadpool_limits(limits=1, user_api="blas")
            factors[b] = _BlockFactor(s, e, blk.level, cb, l11, l21, tile, _tile_inverses(l11, tile))
    finally:
        limiter.restore_original_limits()  # also on IndefiniteMatrixError
    blocks = [factors[b] for b in symbolic.order]
    nlev = 1 + max((bf.level for bf in blocks), default=0)
    levels = [[] for _ in range(nlev)]
    for bf in blocks:
        levels[bf.level].append(bf)
    return LdlFactors(d_out, plan, source_step, blocks, levels, symbolic)


_BIG_FRONT = 1536  # fronts at least this wide use the multithreaded host BLAS


def _front_index(ds_dst, m, width):
    r, c = np.divmod(ds_dst, m)
    return r * width + c


def _blocks_to_csr(n, blocks) -> CsrMatrix:
    """Strict lower triangle of L (l11 strict lower + l21 panels) in CSR with
    exact zeros dropped (the reference's l_matrix, ndprecond.py:479-495).
    Restated: every block's strict-lower triangle and panel become COO
    entries of one scipy.sparse matrix, converted once."""
    import scipy.sparse as sp

    r_parts, c_parts, v_parts = [], [], []
    for bf in blocks:
        m = bf.stop - bf.start
        cols = np.arange(bf.start, bf.stop)
        tri = np.tril(np.asarray(bf.l11), -1)
        rr, cc = np.nonzero(tri)
        r_parts.append(bf.start + rr)
        c_parts.append(bf.start + cc)
        v_parts.append(tri[rr, cc])
        if len(bf.anc):
            rr, cc = np.nonzero(np.asarray(bf.l21))
            r_parts.append(np.asarray(bf.anc)[rr])
            c_parts.append(cols[cc])
            v_parts.append(np.asarray(bf.l21)[rr, cc])
    cat = lambda parts, dt: np.concatenate(parts) if parts else np.empty(0, dtype=dt)  # noqa: E731
    coo = sp.coo_matrix((cat(v_parts, np.float64), (cat(r_parts, np.int64), cat(c_parts, np.int64))), shape=(n, n))
    csr = coo.tocsr()
    csr.sort_indices()
    return CsrMatrix(n, n, csr.indptr.astype(np.int64), csr.indices.astype(np.int64), csr.data)


# ---------------------------------------------------------------------------
# device image of the factors + level-scheduled solves
# ---------------------------------------------------------------------------

from ._ldlt_pack import DevicePanels as DeviceFactors  # noqa: E402  (device image of the factors)


def as_factors(obj):
    """LdlFactors behind a preconditioner-like object, or None."""
    if isinstance(obj, LdlFactors):
        return obj
    f = getattr(obj, "factors", None)
    if isinstance(f, LdlFactors):
        return f
    if isinstance(obj, AsyncPreconditioner):
        raise LifecycleError(f"preconditioner is {obj.status.value}, not ready")
    return None


def _run(factors: LdlFactors, mode: str, r):
    t = _lib.require_cuda()
    n = factors.plan.n
    host = not _lib.is_tensor(r)
    dr = (t.from_numpy(np.ascontiguousarray(np.asarray(r, dtype=np.float64))).cuda() if host
          else r.to(dtype=t.float64).contiguous())
    if dr.numel() != n:
        raise PrecondError(f"vector has {dr.numel()} entries, factors cover {n}")
    out = t.empty(n, dtype=t.float64, device="cuda")
    if n:
        factors.device().run(mode, dr, out)
    return out.cpu().numpy() if host else out


def solve_lower(factors: LdlFactors, r, workers: int = 1):
    """L y = r in permuted order (ndprecond.py:647-671), level-scheduled on the device."""
    return _run(factors, "lower", r)


def solve_upper(factors: LdlFactors, w, workers: int = 1):
    """L^T z = w in permuted order (ndprecond.py:674-691), levels reversed on the device."""
    return _run(factors, "upper", w)


def apply(factors: LdlFactors, r, workers: int = 1):
    """z = (L D L^T)^-1 r in original order (ndprecond.py:694-700)."""
    return _run(factors, "apply", r)


def ldlt_factor_device(a: CsrMatrix, plan: DissectionPlan, tile: int = 16, symbolic: LdlSymbolic | None = None,
                       source_step: int = 0) -> DeviceLdlFactors:
    """ldlt_factor computed on the B200 (refactor.py / csrc/refactor.cu)."""
    from .refactor import ldlt_factor_device as _f

    return _f(a, plan, tile, symbolic, source_step)


# ---------------------------------------------------------------------------
# asynchronous lifecycle (host thread; device upload on a side stream)
# ---------------------------------------------------------------------------

class PrecondStatus(enum.Enum):
    EMPTY = "empty"
    FACTORIZING = "factorizing"
    READY = "ready"


def _factor_job(snapshot: CsrMatrix, plan, tile, symbolic, step, upload: bool, ready=None):
    """Worker thread: host factorisation of the value snapshot, then the
    device upload on a side stream; returns (factors, event)."""
    if ready is not None:
        ready.synchronize()
    factors = ldlt_factor(snapshot, plan, tile, symbolic, step)
    event = None
    if upload:
        t = _lib.torch()
        side = t.cuda.Stream()
        factors._device = DeviceFactors(factors, stream=side)
        event = t.cuda.Event()
        event.record(side)
    return factors, event


class AsyncPreconditioner:
    """Background-factored LDL^T preconditioner (ndprecond.py:714-831).

    `update(a, step)` submits a value snapshot (a D2D clone for device
    matrices) to the worker thread when the policy fires; `poll()` publishes
    finished factors at step boundaries and orders the current stream after
    their upload -- the simulation thread never blocks.
    """

    def __init__(self, plan: DissectionPlan, policy: str = "on-completion",
                 refactor_every: int = 4, tile: int = 16, device: bool = False):
        if policy not in ("on-completion", "every-k"):
            raise PrecondError(f"unknown refactor policy {policy!r}")
        self.plan = plan
        self.policy = policy
        self.refactor_every = refactor_every
        self.tile = tile
        # device=True: the refactorisation runs on the GPU (refactor.py) on a
        # side stream into a second sweep image; no host thread, no download
        self.device = device
        self._rf = None
        self._dev_job = None
        self.factors: LdlFactors | None = None
        self.disabled = False
        self._pool: ThreadPoolExecutor | None = None
        self._future: Future | None = None
        self._symbolic = None
        self._last_submitted = None
        self._pattern_key = None

    @property
    def status(self) -> PrecondStatus:
        if self.factors is not None:
            return PrecondStatus.READY
        return PrecondStatus.FACTORIZING if self.refresh_in_flight else PrecondStatus.EMPTY

    @property
    def refresh_in_flight(self) -> bool:
        return self._future is not None or self._dev_job is not None

    def staleness(self, step: int) -> int:
        return -1 if self.factors is None else step - self.factors.source_step

    def _policy_fires(self, step: int) -> bool:
        if self._last_submitted is None or self.policy == "on-completion":
            return True
        return step - self._last_submitted >= self.refactor_every

    def _publish_device(self, wait: bool = False):
        job = self._dev_job
        if job is None:
            return
        factors, event, flag, _ = job
        if not wait and not event.query():
            return
        event.synchronize()
        self._dev_job = None
        if int(flag[0]) != 0:
            bf = self._rf.rplan.blocks[int(flag[0]) - 1]
            logger.warning("device factorization failed (non-positive pivot in block [%d, %d)); "
                           "preconditioner disabled", bf.start, bf.stop)
            self.disabled = True
            return
        _lib.torch().cuda.current_stream().wait_event(event)
        self.factors = factors

    def prepare(self, a: CsrMatrix):
        """device=True: plan the device refactorisation of `a`'s pattern now
        (host setup: symbolic structure, front maps, launch program, the two
        sweep images -- seconds at 100k nodes) instead of inside the first
        update(), which then only enqueues device work."""
        if not self.device:
            return
        from .refactor import DeviceRefactor

        if self._rf is None or self._rf.symbolic.pattern_key != _pattern_key(a):
            t = _lib.torch()
            self._rf = DeviceRefactor(a, self.plan, self.tile, buffers=2)
            self._side = t.cuda.Stream()
            self._flag = t.zeros(4, dtype=t.int32).pin_memory()

    def _submit_device(self, a: CsrMatrix, step: int):
        """Refactor `a` on a side stream into the sweep image not in use."""
        from .refactor import make_factors

        t = _lib.torch()
        self.prepare(a)
        rf = self._rf
        img = rf.images[rf._next]
        rf._next = (rf._next + 1) % len(rf.images)
        snapshot = a.copy_values()          # the caller may overwrite a's values next step
        self._side.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(self._side):
            rf.enqueue(snapshot, img)
            self._flag.copy_(rf.d["ctl"], non_blocking=True)
            event = t.cuda.Event()
            event.record(self._side)
        self._dev_job = (make_factors(rf, img, step), event, self._flag, snapshot)  # snapshot lives until publish

    def _publish_if_done(self):
        if self.device:
            self._publish_device()
            return
        if self._future is not None and self._future.done():
            try:
                factors, event = self._future.result()
                if event is not None:
                    _lib.torch().cuda.current_stream().wait_event(event)
                self.factors = factors
                self._symbolic = factors.symbolic
            except Exception:
                logger.warning("background factorization failed; preconditioner disabled", exc_info=True)
                self.disabled = True
            self._future = None

    def poll(self):
        self._publish_if_done()

    def update(self, a: CsrMatrix, step: int):
        self._publish_if_done()
        if self.disabled or self.refresh_in_flight:
            return
        key = _pattern_key(a)
        if self._pattern_key is not None and key != self._pattern_key:
            self._symbolic = None
            self.factors = None
        self._pattern_key = key
        if not self._policy_fires(step):
            return
        if self.device:
            self._last_submitted = step
            self._submit_device(a, step)
            return
        snapshot = a.copy_values()
        ready = None
        if snapshot.on_device:  # D2D clone now; the worker waits for it, then downloads
            ready = _lib.torch().cuda.Event()
            ready.record()
        self._last_submitted = step
        if self._pool is None:
            self._pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="ldlt-worker")
        upload = _lib.is_cuda_ready()
        self._future = self._pool.submit(_factor_job, snapshot, self.plan, self.tile, self._symbolic,
                                         step, upload, ready)

    def wait_ready(self, timeout: float = 60.0):
        if not self.refresh_in_flight and self.factors is None:
            raise LifecycleError("no factorization in flight")
        if self.device:
            self._publish_device(wait=True)
            if self.disabled:
                raise LifecycleError("factorization failed; preconditioner disabled")
            return
        if self._future is not None:
            self._future.exception(timeout=timeout)
            self._publish_if_done()
        if self.disabled:
            raise LifecycleError("factorization failed; preconditioner disabled")

    def apply(self, r, workers: int = 1):
        if self.factors is None:
            raise LifecycleError(f"preconditioner is {self.status.value}, not ready")
        return self.factors.apply(r, workers=workers)

    def close(self):
        if self._pool is not None:
            self._pool.shutdown(wait=True)
            self._pool = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False
