"""Nested-dissection sharding of the solve across GPUs.

The reference has no distributed path; its domain decomposition is a solver
structure only (`_dissect`, ndprecond.py:180-231): subtrees of the
dissection are independent and couple only through their ancestor
separators (`count_coupling_violations`, ndprecond.py:295-309).  That makes
top-level subtrees the natural unit of distribution:

  * rank g owns the rows (permuted order) of its subtrees -- their diagonal
    blocks, their rows of A and their L panels;
  * the separators above the cut ("top" blocks) are replicated on every rank.

Per PCG iteration the only exchanges are sums over the top rows:
  1. SpMV: a top row's entries span several subtrees; every rank adds the
     products of its own columns (rank 0 also the top columns), then one
     all-reduce over the top rows;
  2. forward sweep: every rank solves its subtrees and pre-accumulates their
     contributions into the top rows (the column-major pre-accumulation of
     the paper); one all-reduce of those sums, then every rank solves the
     replicated top blocks redundantly; the backward sweep needs no exchange
     (top values are replicated and identical);
  3. dots: owned rows on every rank, top rows on rank 0 only (weights), one
     all-reduce of the packed scalars.

Everything here is host setup or a CPU emulation of the device loop for the
world_size > 1 tests (gloo); the device loop is `DistributedPcg`.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

logger = logging.getLogger(__name__)


def block_etree(factors):
    """Block elimination tree of LdlFactors: parent(b) = owner of b's first
    ancestor row (-1 = root), plus children lists (same rule as _ldlt_pack)."""
    bfs = list(factors.blocks)
    n = factors.plan.n
    owner = np.full(n, -1, dtype=np.int64)
    for i, bf in enumerate(bfs):
        owner[bf.start:bf.stop] = i
    parent = np.full(len(bfs), -1, dtype=np.int64)
    for i, bf in enumerate(bfs):
        if len(bf.anc):
            parent[i] = owner[int(np.min(bf.anc))]
    children = [[] for _ in bfs]
    for i, p in enumerate(parent):
        if p >= 0:
            children[p].append(i)
    return parent, children


def block_weights(factors):
    """Work per block: factor entries of its diagonal triangle and coupling panel."""
    return np.array([(bf.stop - bf.start) * ((bf.stop - bf.start) + 1) / 2 + (bf.stop - bf.start) * len(bf.anc)
                     for bf in factors.blocks])


@dataclass
class ShardPlan:
    """Block -> rank map (-1 = replicated top block) and the row sets it induces."""

    nranks: int
    owner: np.ndarray          # [n_blocks] rank or -1
    row_owner: np.ndarray      # [n] (permuted rows) rank or -1 (top)
    top_rows: np.ndarray       # sorted permuted rows of the top blocks
    load: np.ndarray           # [nranks] block weight per rank

    def owned_rows(self, rank: int) -> np.ndarray:
        return np.flatnonzero(self.row_owner == rank)

    def weights(self, rank: int) -> np.ndarray:
        """Dot-product weights in permuted order: owned rows 1, top rows 1 on rank 0 only."""
        w = (self.row_owner == rank).astype(np.float64)
        if rank == 0:
            w[self.row_owner < 0] = 1.0
        return w


def shard_blocks(factors, nranks: int) -> ShardPlan:
    """Cut the block elimination tree into >= nranks subtrees and assign them.

    Repeatedly split the heaviest subtree (its root joins the replicated top)
    until there are at least `nranks` subtrees, then assign subtrees to ranks
    longest-processing-time first.  A separator can have more than two
    children (disconnected halves, ndprecond.py:187-196), so the cut balances
    by weight instead of assuming a binary tree."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    parent, children = block_etree(factors)
    w = block_weights(factors)
    nb = len(w)
    sub = w.copy()
    for i in sorted(range(nb), key=lambda i: factors.blocks[i].start):  # children first
        if parent[i] >= 0:
            sub[parent[i]] += sub[i]
    roots = [i for i in range(nb) if parent[i] < 0]
    top = set()
    front = list(roots)
    while len(front) < nranks:
        splittable = [r for r in front if children[r]]
        if not splittable:
            break
        r = max(splittable, key=lambda r: sub[r])
        front.remove(r)
        top.add(r)
        front.extend(children[r])
    load = np.zeros(nranks)
    root_rank = {}
    for r in sorted(front, key=lambda r: -sub[r]):
        g = int(np.argmin(load))
        root_rank[r] = g
        load[g] += sub[r]
    owner = np.full(nb, -1, dtype=np.int64)
    for i in sorted(range(nb), key=lambda i: -factors.blocks[i].start):  # parents first
        if i in top:
            owner[i] = -1
        elif i in root_rank:
            owner[i] = root_rank[i]
        else:
            owner[i] = owner[parent[i]]
    n = factors.plan.n
    row_owner = np.full(n, -1, dtype=np.int64)
    for i, bf in enumerate(factors.blocks):
        row_owner[bf.start:bf.stop] = owner[i]
    return ShardPlan(nranks, owner, row_owner, np.flatnonzero(row_owner < 0), load)


def permuted_matrix(a, perm):
    """(row_ptr, col_ind, values) of P A P^T in CSR (columns sorted per row)."""
    n = a.nrows
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    rows = np.repeat(np.arange(n), np.diff(a.row_ptr))
    pr, pc = iperm[rows], iperm[np.asarray(a.col_ind)]
    order = np.lexsort((pc, pr))
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(pr, minlength=n), out=row_ptr[1:])
    return row_ptr, pc[order], np.asarray(a.values)[order]


def local_matrix(row_ptr, col_ind, values, plan: ShardPlan, rank: int):
    """Rank-local CSR (permuted, full-size index space): owned rows complete,
    top rows restricted to the rank's columns (rank 0 also the top columns),
    every other row empty.  Raises if an owned row couples to another rank."""
    n = len(row_ptr) - 1
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    ro = plan.row_owner
    own_row = ro[rows] == rank
    bad = own_row & (ro[col_ind] >= 0) & (ro[col_ind] != rank)
    if np.any(bad):
        raise ValueError("owned rows couple to another rank's subtree: not a dissection cut")
    top_row = ro[rows] < 0
    col_ok = (ro[col_ind] == rank) | ((ro[col_ind] < 0) & (rank == 0))
    keep = own_row | (top_row & col_ok)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=n), out=rp[1:])
    return rp, col_ind[keep], values[keep]


# ---------------------------------------------------------------------------
# sharded assembly (SURVEY.md 8e "Assembly"): each rank assembles only its
# elements; owned rows come out complete, top-separator rows as partial sums
# that the SpMV's top-row all-reduce adds up.
# ---------------------------------------------------------------------------

def node_ranks(plan: ShardPlan, perm) -> np.ndarray:
    """Rank owning each mesh node (-1: a replicated top-separator node); the
    dissection orders whole nodes (expand_plan), so a node's dofs agree."""
    perm = np.asarray(perm)
    ro = np.empty(len(perm), dtype=np.int64)
    ro[perm] = plan.row_owner  # original dof -> owner
    ro = ro.reshape(-1, 3)
    if np.any(ro != ro[:, :1]):
        raise ValueError("a node's dofs are split across ranks")
    return ro[:, 0].copy()


def element_ranks(elements, node_rank: np.ndarray) -> np.ndarray:
    """Rank assembling each element: the rank of its non-separator nodes (all
    the same: a tet spanning two subtrees would be an uncut edge), rank 0 for
    elements entirely inside the top separators."""
    nr = node_rank[np.asarray(elements)]
    hi, lo = nr.max(axis=1), np.where(nr >= 0, nr, np.iinfo(np.int64).max).min(axis=1)
    if np.any((hi >= 0) & (lo != hi)):
        raise ValueError("an element spans two ranks' subtrees: not a dissection cut")
    return np.where(hi >= 0, hi, 0)


def rank_mesh(mesh, plan: ShardPlan, perm, rank: int):
    """(mesh of rank `rank`'s elements over all nodes, node ranks): what the
    rank's integrator assembles; its owned rows are the full assembly's."""
    from .mesh import Mesh

    nr = node_ranks(plan, perm)
    er = element_ranks(mesh.elements, nr)
    return Mesh(mesh.nodes, np.asarray(mesh.elements)[er == rank], mesh.element_kind, mesh.fixed_nodes), nr


def rank_f_ext(f_ext, node_rank: np.ndarray, rank: int) -> np.ndarray:
    """The state's external forces as rank `rank` passes them to its partial
    assembly: its owned nodes, plus the top nodes on rank 0 (counted once)."""
    keep = (node_rank == rank) | ((node_rank < 0) & (rank == 0))
    return np.where(np.repeat(keep, 3), np.asarray(f_ext, dtype=np.float64).reshape(-1), 0.0)


def local_system(row_ptr, col_ind, values, b, plan: ShardPlan, perm, rank: int, fixed_dofs):
    """Rank-local permuted CSR and rhs from the rank's partial assembly (its
    elements only, original dof order): owned rows kept as assembled
    (complete), top rows kept as partial sums, pinned top rows (identity) kept
    on rank 0 only, every other row dropped.  The sum over ranks of the local
    matrices is P A P^T; owned rows are bit-identical to the full assembly's."""
    from .assembly import CsrMatrix

    perm = np.asarray(perm)
    n = len(perm)
    rp, ci, va = permuted_matrix(CsrMatrix(n, n, row_ptr, col_ind, values), perm)
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    pinned = np.zeros(n, dtype=bool)
    pinned[iperm[np.asarray(fixed_dofs, dtype=np.int64)]] = True
    ro = plan.row_owner
    rows = np.repeat(np.arange(n), np.diff(rp))
    keep = (ro[rows] == rank) | ((ro[rows] < 0) & (~pinned[rows] | (rank == 0)))
    lrp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=n), out=lrp[1:])
    bp = np.asarray(b, dtype=np.float64)[perm]
    lb = np.where((ro == rank) | (ro < 0), bp, 0.0)
    return lrp, ci[keep], va[keep], lb


class LocalSystem:
    """Per-step extraction of a rank's local system ON THE DEVICE.

    local_system() is planned once per (pattern, shard plan, rank) on index
    arrays -- the entry values are their own positions -- which yields the
    source slot of every local entry; each step is then one gather of the
    rank's assembled values (still in HBM) and one masked gather of its rhs,
    instead of a host NumPy lexsort of every new matrix."""

    def __init__(self, row_ptr, col_ind, plan: ShardPlan, perm, rank: int, fixed_dofs):
        from . import _lib

        t = _lib.require_cuda()
        nnz, n = len(col_ind), len(perm)
        idx = np.arange(nnz, dtype=np.float64)  # exact below 2^53
        lrp, lci, src, _ = local_system(row_ptr, col_ind, idx, np.zeros(n), plan, perm, rank, fixed_dofs)
        self.row_ptr, self.col_ind = lrp, lci
        self.src = t.from_numpy(src.astype(np.int64)).cuda()
        ro = plan.row_owner
        self.mask = t.from_numpy(((ro == rank) | (ro < 0)).astype(np.float64)).cuda()
        self.perm = t.from_numpy(np.asarray(perm, dtype=np.int64)).cuda()

    def values(self, values):
        """Local entry values from the rank's assembled values (device tensor)."""
        return values.index_select(0, self.src)

    def rhs(self, b):
        """Permuted local rhs: owned and top rows of the rank's partial b."""
        return b.index_select(0, self.perm) * self.mask

    def system(self, values, b):
        """(row_ptr, col_ind, values, b) -- the DistributedPcg `local=` tuple."""
        return self.row_ptr, self.col_ind, self.values(values), self.rhs(b)


# ---------------------------------------------------------------------------
# CPU emulation of the distributed loop (world_size > 1 tests over gloo)
# ---------------------------------------------------------------------------

def _sharded_rhs(lb, plan: ShardPlan, perm, allreduce):
    """Original-order rhs as a rank's solve consumes it: owned rows as
    assembled, top rows summed over ranks (other rows are never read)."""
    top = plan.top_rows
    seg = np.array(lb[top], dtype=np.float64)
    allreduce(seg)
    bp = np.array(lb, dtype=np.float64)
    bp[top] = seg
    out = np.empty_like(bp)
    out[np.asarray(perm)] = bp
    return out


def _lower_blocks(factors, idx, r, ext=None):
    """Forward sweep over the blocks `idx` (start order): y = L^{-1} r on their
    rows; contributions to rows outside them returned in `ext` (summed)."""
    y = np.array(r, dtype=np.float64)
    if ext is not None:
        y = y - ext
    out = np.zeros_like(y)
    mine = np.zeros(len(y), dtype=bool)
    for i in idx:
        mine[factors.blocks[i].start:factors.blocks[i].stop] = True
    for i in sorted(idx, key=lambda i: factors.blocks[i].start):
        bf = factors.blocks[i]
        s, e = bf.start, bf.stop
        from scipy.linalg import solve_triangular

        seg = solve_triangular(bf.l11, y[s:e], lower=True, unit_diagonal=True)
        y[s:e] = seg
        if len(bf.anc):
            c = bf.l21 @ seg
            inside = mine[bf.anc]
            y[bf.anc[inside]] -= c[inside]
            out[bf.anc[~inside]] += c[~inside]
    return y, out


def _upper_blocks(factors, idx, w, z):
    """Backward sweep over the blocks `idx` (reverse start order) into z."""
    from scipy.linalg import solve_triangular

    for i in sorted(idx, key=lambda i: -factors.blocks[i].start):
        bf = factors.blocks[i]
        s, e = bf.start, bf.stop
        seg = w[s:e].copy()
        if len(bf.anc):
            seg -= bf.l21.T @ z[bf.anc]
        z[s:e] = solve_triangular(bf.l11, seg, lower=True, unit_diagonal=True, trans="T")
    return z


def emulate_pcg(a, b, factors, plan: ShardPlan, rank: int, allreduce, tol=1e-9, max_it=1000, local=None):
    """One rank of the distributed PCG, NumPy kernels; `allreduce(np.ndarray)`
    sums over ranks in place.  Works in permuted order like the device loop;
    returns (x in original order, iterations, final residual, converged).
    local=(row_ptr, col_ind, values, b) from local_system (sharded assembly)
    replaces a and b: the top rows of b are all-reduced first."""
    perm = np.asarray(factors.plan.perm)
    n = len(perm)
    if local is not None:
        lrp, lci, lva, lb = local
        b = _sharded_rhs(lb, plan, perm, allreduce)
    else:
        rp, ci, va = permuted_matrix(a, perm)
        lrp, lci, lva = local_matrix(rp, ci, va, plan, rank)
    wgt = plan.weights(rank)
    top = plan.top_rows
    mine = [i for i in range(len(factors.blocks)) if plan.owner[i] == rank]
    tops = [i for i in range(len(factors.blocks)) if plan.owner[i] < 0]
    valid = (plan.row_owner == rank) | (plan.row_owner < 0)

    def spmv(p):
        y = np.zeros(n)
        nz = np.flatnonzero(np.diff(lrp))
        y[nz] = np.add.reduceat(lva * p[lci], lrp[:-1][nz]) if len(lci) else 0.0
        seg = y[top].copy()
        allreduce(seg)
        y[top] = seg
        return y

    def dot(u, v):
        s = np.array([np.sum(wgt * u * v)])
        allreduce(s)
        return float(s[0])

    def precond(r):
        y, ext = _lower_blocks(factors, mine, np.where(valid, r, 0.0))
        ext_top = ext[top].copy()
        allreduce(ext_top)
        e = np.zeros(n)
        e[top] = ext_top
        y2, _ = _lower_blocks(factors, tops, np.where(plan.row_owner < 0, r, 0.0), ext=e)
        y = np.where(plan.row_owner < 0, y2, y)
        wv = y / factors.d
        z = np.zeros(n)
        _upper_blocks(factors, tops, wv, z)
        _upper_blocks(factors, mine, wv, z)
        return np.where(valid, z, 0.0)

    bp = np.asarray(b, dtype=np.float64)[perm]
    x = np.zeros(n)
    bnorm = np.sqrt(dot(bp, bp))
    if bnorm == 0.0:
        return np.zeros(n), 0, 0.0, True
    r = np.where(valid, bp, 0.0)
    res = np.sqrt(dot(r, r)) / bnorm
    if res <= tol:
        return np.zeros(n), 0, res, True
    z = precond(r)
    p = z.copy()
    rz = dot(r, z)
    it, conv = 0, False
    while it < max_it:
        ap = spmv(p)
        alpha = rz / dot(p, ap)
        x = x + alpha * p
        r = r - alpha * ap
        it += 1
        res = np.sqrt(dot(r, r)) / bnorm
        if res <= tol:
            conv = True
            break
        z = precond(r)
        rz_new = dot(r, z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    xg = wgt * x  # every rank contributes its owned rows (rank 0 the top rows)
    allreduce(xg)
    xo = np.zeros(n)
    xo[perm] = xg
    return xo, it, res, conv


# ---------------------------------------------------------------------------
# device loop (one process per GPU; torch.distributed for the all-reduces)
# ---------------------------------------------------------------------------

class PeerAllreduce:
    """All-reduce of small device vectors over peer memory (csrc/peer.cu).

    Every rank allocates a double-buffered exchange buffer and an epoch word;
    they are shared with the other ranks once through CUDA IPC (the handles
    travel over the process group with all_gather_object), after which an
    exchange is ONE kernel: gather the rows into the rank's buffer, publish
    the epoch (release, system scope), wait for every peer's epoch (acquire),
    sum the ranks' rows in rank order and scatter them back -- no NCCL call,
    no host synchronisation.  Between GPUs the peers' buffers are read over
    NVLink / NVSwitch."""

    def __init__(self, world: int, rank: int, capacity: int, group=None):
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor

        from . import _lib

        t = _lib.require_cuda()
        self.world, self.rank, self.half = world, rank, int(max(capacity, 1))
        self.buf = t.zeros(2 * self.half, dtype=t.float64, device="cuda")
        self.flag = t.zeros(1, dtype=t.int64, device="cuda")
        t.cuda.synchronize()
        mine = (reduce_tensor(self.buf), reduce_tensor(self.flag))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self._peers = []  # keep the mapped peer tensors alive
        bufs, flags = [], []
        for r, (hb, hf) in enumerate(allh):
            if r == rank:
                b, f = self.buf, self.flag
            else:
                b, f = hb[0](*hb[1]), hf[0](*hf[1])
                self._peers.append((b, f))
            bufs.append(b.data_ptr())
            flags.append(f.data_ptr())
        self.d_bufs = t.tensor(bufs, dtype=t.int64, device="cuda")
        self.d_flags = t.tensor(flags, dtype=t.int64, device="cuda")
        self.epoch = 0
        self._lib, self._L = _lib.load(), _lib
        dist.barrier(group=group)

    def spmv(self, nrows, rp, ci, va, x, y, idx):
        """y = A x on this rank's rows, then y[idx] all-reduced -- one fused kernel (tsb_spmv_peer)."""
        L = self._L
        if not hasattr(self, "_ticket"):
            self._ticket = L.torch().zeros(1, dtype=L.torch().int32, device="cuda")
        m = int(idx.numel())
        self.epoch += 1
        L.check(self._lib.tsb_spmv_peer(nrows, L.ptr(rp), L.ptr(ci), L.ptr(va), L.ptr(x), L.ptr(y), m, self.world,
                                        self.rank, L.ptr(self.d_bufs), L.ptr(self.d_flags), L.ptr(idx), self.epoch,
                                        self.half, L.ptr(self._ticket), L.stream_ptr()), "spmv_peer")

    def external_sums(self, panels, out, idx):
        """panels' external contribution sums into out, then out[idx] all-reduced (one kernel)."""
        L = self._L
        if not hasattr(self, "_ticket2"):
            self._ticket2 = L.torch().zeros(1, dtype=L.torch().int32, device="cuda")
        self.epoch += 1
        L.check(self._lib.tsb_ldlt_external_sums_peer(panels.h, L.ptr(out), int(idx.numel()), self.world, self.rank,
                                                      L.ptr(self.d_bufs), L.ptr(self.d_flags), L.ptr(idx), self.epoch,
                                                      self.half, L.ptr(self._ticket2), L.stream_ptr()),
                "external_sums_peer")

    def __call__(self, x, idx=None, m=None):
        """x[idx] (or x[:m]) := the sum over ranks, in place, on the current stream."""
        L = self._L
        m = int(idx.numel() if idx is not None else (x.numel() if m is None else m))
        if m > self.half:
            raise ValueError(f"exchange of {m} rows exceeds the buffer ({self.half})")
        self.epoch += 1
        L.check(self._lib.tsb_peer_allreduce(m, self.world, self.rank, L.ptr(self.d_bufs), L.ptr(self.d_flags),
                                             L.ptr(idx), L.ptr(x), self.epoch, self.half, L.stream_ptr()),
                "peer_allreduce")


class DistributedPcg:
    """Sharded PCG with the nested-dissection LDL^T preconditioner.

    Every rank runs the libtsb kernels on its shard (permuted order, full-length
    vectors, only owned + top rows live): rank-local SpMV (tsb_spmv), the
    subtree sweeps and the replicated top sweeps (tsb_ldlt_lower_ext /
    tsb_ldlt_upper_scaled over block subsets), weighted dots and the fused
    vector updates (tsb_pcg_update / tsb_pcg_direction, alpha and beta on the
    device).  Exchanges: one all-reduce of the top rows after the SpMV and one
    after the subtree forward sweep, plus the packed scalars; the host reads
    the residual norm once per iteration for the stop test.  `allreduce`
    defaults to torch.distributed.all_reduce (NCCL over NVLink between GPUs).
    """

    def __init__(self, a, factors, rank=None, world=None, allreduce=None, grid=0, exchange="nccl", local=None):
        from . import _lib
        from ._ldlt_pack import DevicePanels

        t = _lib.require_cuda()
        if rank is None or world is None:
            import torch.distributed as dist

            rank = dist.get_rank() if dist.is_initialized() else 0
            world = dist.get_world_size() if dist.is_initialized() else 1
        if allreduce is None:
            import torch.distributed as dist

            allreduce = (lambda x: dist.all_reduce(x)) if world > 1 else (lambda x: None)
        self.rank, self.world, self.allreduce = rank, world, allreduce
        self.factors = factors
        self.plan = shard_blocks(factors, world)
        perm = np.asarray(factors.plan.perm)
        self.n = n = len(perm)
        # local=(row_ptr, col_ind, values, b) from local_system: this rank's share of a
        # sharded assembly (owned rows complete, top rows partial); a is not needed
        self._lb = None
        if local is not None:
            lrp, lci, lva, self._lb = local
        else:
            rp, ci, va = permuted_matrix(a, perm)
            lrp, lci, lva = local_matrix(rp, ci, va, self.plan, rank)
        dev = lambda x, dt: t.from_numpy(np.ascontiguousarray(x, dtype=dt)).cuda()  # noqa: E731
        self.rp, self.ci = dev(lrp, np.int32), dev(lci, np.int32)
        self.va = lva.to(dtype=t.float64).clone() if _lib.is_tensor(lva) else dev(lva, np.float64)
        self.w = dev(self.plan.weights(rank), np.float64)
        self.top = dev(self.plan.top_rows, np.int32)
        self.perm = dev(perm, np.int32)
        iperm = np.empty(n, dtype=np.int64)
        iperm[perm] = np.arange(n)
        self.iperm = dev(iperm, np.int32)
        mine = [i for i in range(len(factors.blocks)) if self.plan.owner[i] == rank]
        tops = [i for i in range(len(factors.blocks)) if self.plan.owner[i] < 0]
        self.S = DevicePanels(factors, subset=mine, grid=grid) if mine else None
        self.T = DevicePanels(factors, subset=tops, grid=grid) if tops else None
        z = lambda k: t.zeros(max(k, 1), dtype=t.float64, device="cuda")  # noqa: E731
        self.v = {k: z(n) for k in ("x", "r", "z", "p", "ap", "y", "ext", "b")}
        self.topbuf = z(len(self.plan.top_rows))
        self.part = z(2 * 148)
        self.sc = z(8)  # [rz, pAp] / [rz_new, rz_old] / scratch
        self.done = t.zeros(1, dtype=t.int32, device="cuda")   # device stop flag
        self.it = t.zeros(1, dtype=t.int64, device="cuda")     # iteration count
        self.res = z(1)                                          # final relative residual
        self.done_host = t.zeros(1, dtype=t.int32).pin_memory()
        self._lib = _lib.load()
        self._L = _lib
        # exchange="peer": the top-row exchanges and the scalars go through
        # PeerAllreduce (one kernel each over IPC-mapped peer memory) instead
        # of the process group's all-reduce
        self.peer = None
        if exchange == "peer" and world > 1:
            self.peer = PeerAllreduce(world, rank, max(len(self.plan.top_rows), n))
            self.allreduce = lambda x: self.peer(x)

    def set_values(self, values, b=None):
        """New values (same local pattern) and, for a sharded assembly, the
        rank's new local rhs -- e.g. LocalSystem.values / .rhs of the next step;
        the factor panels (the preconditioner) are kept."""
        self.va.copy_(values)
        if b is not None:
            self._lb = b

    # -- pieces ------------------------------------------------------------
    def _exchange_top(self, vec):
        m = len(self.plan.top_rows)
        if self.world == 1 or m == 0:
            return
        if self.peer is not None:  # gather + exchange + scatter in one kernel
            self.peer(vec, idx=self.top)
            return
        L, s = self._L, self._L.stream_ptr()
        L.check(self._lib.tsb_gather_rows(m, L.ptr(self.top), L.ptr(vec), L.ptr(self.topbuf), s), "gather")
        self.allreduce(self.topbuf[:m])
        L.check(self._lib.tsb_scatter_rows(m, L.ptr(self.top), L.ptr(self.topbuf), L.ptr(vec), s), "scatter")

    def _dot(self, a, b, slot):
        L = self._L
        L.check(self._lib.tsb_wdot(self.n, L.ptr(self.w), L.ptr(a), L.ptr(b), L.ptr(self.part),
                                   L.ptr(self.sc[slot:slot + 1]), L.stream_ptr()), "wdot")
        self.allreduce(self.sc[slot:slot + 1])

    def _spmv(self, p, out):
        L = self._L
        if self.peer is not None and len(self.plan.top_rows):  # product + exchange in one kernel
            self.peer.spmv(self.n, self.rp, self.ci, self.va, p, out, self.top)
            return
        L.check(self._lib.tsb_spmv(self.n, L.ptr(self.rp), L.ptr(self.ci), L.ptr(self.va), L.ptr(p), L.ptr(out),
                                   L.stream_ptr()), "spmv")
        self._exchange_top(out)

    def _precond(self, r, out):
        v = self.v
        v["ext"].zero_()
        if self.S is not None:
            self.S.lower_ext(r, None, v["y"])
            if self.peer is not None and len(self.plan.top_rows):  # sums + exchange in one kernel
                self.peer.external_sums(self.S, v["ext"], self.top)
            else:
                self.S.external_sums(v["ext"])
                self._exchange_top(v["ext"])
        else:
            self._exchange_top(v["ext"])
        if self.T is not None:
            self.T.lower_ext(r, v["ext"], v["y"])
            self.T.run("upper_scaled", v["y"], out)
        if self.S is not None:
            self.S.run("upper_scaled", v["y"], out)

    # -- solve -----------------------------------------------------------------
    def _iteration(self, bnorm, tol, max_it):
        """One PCG iteration, entirely on the device: alpha, beta, the stop test
        and the iteration count never leave it (tsb_pcg_check sets the stop
        flag; the updates are no-ops once it is set)."""
        L, v, n = self._L, self.v, self.n
        s = L.stream_ptr()
        self._spmv(v["p"], v["ap"])
        self._dot(v["p"], v["ap"], 1)  # sc[1] = pAp; alpha = sc[0] / sc[1]
        L.check(self._lib.tsb_pcg_update(n, L.ptr(self.w), L.ptr(v["x"]), L.ptr(v["p"]), L.ptr(v["r"]),
                                         L.ptr(v["ap"]), L.ptr(self.sc), L.ptr(self.part), L.ptr(self.sc[5:6]),
                                         L.ptr(self.done), s), "pcg_update")
        self.allreduce(self.sc[5:6])
        L.check(self._lib.tsb_pcg_check(L.ptr(self.sc[5:6]), bnorm, tol, max_it, L.ptr(self.done),
                                        L.ptr(self.it), L.ptr(self.res), s), "pcg_check")
        self._precond(v["r"], v["z"])
        self.sc[1:2].copy_(self.sc[0:1])  # rz_old
        self._dot(v["r"], v["z"], 0)       # rz_new; beta = sc[0] / sc[1]
        L.check(self._lib.tsb_pcg_direction(n, L.ptr(v["p"]), L.ptr(v["z"]), L.ptr(self.sc), L.ptr(self.done), s),
                "pcg_direction")

    def _graph_ok(self):
        """CUDA-graph replay needs capturable exchanges: our peer kernels, NCCL,
        or none (one rank); a gloo process group runs the iterations eagerly."""
        if getattr(self, "_graph_failed", False):
            return False
        if self.world == 1 or self.peer is not None:
            return True
        import torch.distributed as dist

        return dist.is_initialized() and dist.get_backend() == "nccl"

    GRAPH_ITERS = 4  # iterations per graph replay: one host read of the stop flag per replay

    def solve(self, b=None, tol=1e-9, max_it=1000, graph=None):
        """-> (x in original order as a CUDA tensor, iterations, residual, converged).
        b=None with a sharded assembly: the rank's partial rhs, top rows all-reduced.

        The iterations run device-resident: alpha, beta, the residual test and
        the count stay on the device, and (graph=True, the default where the
        exchanges allow it) GRAPH_ITERS iterations are replayed as one CUDA
        graph, the stop flag read once per replay -- no host round trip per
        iteration."""
        L, t = self._L, self._L.torch()
        v, n = self.v, self.n
        s = L.stream_ptr()
        if b is None:
            if self._lb is None:
                raise ValueError("solve() needs b unless built from a sharded assembly (local=)")
            if L.is_tensor(self._lb):
                v["b"].copy_(self._lb)
            else:
                v["b"].copy_(t.from_numpy(np.ascontiguousarray(self._lb, dtype=np.float64)))
            self._exchange_top(v["b"])
        else:
            bd = b if L.is_tensor(b) else t.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).cuda()
            L.check(self._lib.tsb_gather_rows(n, L.ptr(self.perm), L.ptr(bd), L.ptr(v["b"]), s), "gather")
        l0, replays, captured = L.launch_count(), 0, 0
        v["r"].copy_(v["b"])
        v["x"].zero_()
        self._dot(v["b"], v["b"], 4)
        bnorm = float(self.sc[4].item()) ** 0.5  # one read per solve (the reference's ||b||)
        x_out = t.zeros(n, dtype=t.float64, device="cuda")
        if bnorm == 0.0:
            return x_out, 0, 0.0, True
        # x0 = 0: r = b, the initial relative residual is 1 > tol
        self.done.zero_()
        self.it.zero_()
        self.res.fill_(1.0)
        if max_it > 0 and tol < 1.0:
            self._precond(v["r"], v["z"])
            v["p"].copy_(v["z"])
            self._dot(v["r"], v["z"], 0)  # sc[0] = rz
            use_graph = self._graph_ok() if graph is None else graph
            if use_graph:
                key = (bnorm, tol, max_it)
                if getattr(self, "_graph_key", None) != key:
                    c0 = L.launch_count()
                    try:
                        self._capture(bnorm, tol, max_it)
                    except RuntimeError as e:  # an exchange that cannot be captured: iterate eagerly
                        logger.warning("sharded PCG: CUDA-graph capture failed (%s); eager iterations", e)
                        self._graph_failed = True
                        use_graph = False
                    else:
                        captured = L.launch_count() - c0 - self._graph_kernels
                        self._graph_key = key
            if use_graph:
                while True:
                    self._graph.replay()
                    replays += 1
                    self.done_host.copy_(self.done, non_blocking=True)
                    t.cuda.current_stream().synchronize()
                    if int(self.done_host[0]):
                        break
            else:
                while True:
                    self._iteration(bnorm, tol, max_it)
                    if int(self.done.item()):
                        break
        it = int(self.it.item())
        res = float(self.res.item())
        conv = res <= tol
        # x: owned rows from every rank, top rows from rank 0
        xw = v["y"]
        self._weighted_copy(v["x"], xw)
        self.allreduce(xw)
        L.check(self._lib.tsb_gather_rows(n, L.ptr(self.iperm), L.ptr(xw), L.ptr(x_out), s), "gather")
        # libtsb kernels this solve ran: eager launches + the kernels of each graph replay
        self.last_replayed = replays * getattr(self, "_graph_kernels", 0)
        self.last_launches = L.launch_count() - l0 - captured + self.last_replayed
        return x_out, it, res, conv

    def _capture(self, bnorm, tol, max_it):
        t = self._L.torch()
        side = t.cuda.Stream()
        side.wait_stream(t.cuda.current_stream())
        saved = (self.done.clone(), self.it.clone(), self.res.clone(), self.sc.clone(),
                 *(self.v[k].clone() for k in ("x", "r", "z", "p")))
        with t.cuda.stream(side):  # one eager pass on the capture stream warms every handle
            self._iteration(bnorm, tol, max_it)
        t.cuda.current_stream().wait_stream(side)
        t.cuda.synchronize()
        self._graph = t.cuda.CUDAGraph()
        k0 = self._L.launch_count()
        try:
            with t.cuda.graph(self._graph):
                for _ in range(self.GRAPH_ITERS):
                    self._iteration(bnorm, tol, max_it)
            self._graph_kernels = self._L.launch_count() - k0  # libtsb kernels per replay
        finally:
            t.cuda.synchronize()
            # capture does not execute: restore the state the warm-up pass advanced
            for dst, src in zip((self.done, self.it, self.res, self.sc,
                                 *(self.v[k] for k in ("x", "r", "z", "p"))), saved):
                dst.copy_(src)

    def _weighted_copy(self, x, out):
        """out = x on the rows this rank contributes (owned, top on rank 0), else 0."""
        L = self._L
        out.zero_()
        rows = np.flatnonzero(self.plan.weights(self.rank) > 0).astype(np.int32)
        if not hasattr(self, "_live"):
            t = L.torch()
            self._live = t.from_numpy(rows).cuda()
            self._livebuf = t.zeros(max(len(rows), 1), dtype=t.float64, device="cuda")
        m = len(rows)
        s = L.stream_ptr()
        L.check(self._lib.tsb_gather_rows(m, L.ptr(self._live), L.ptr(x), L.ptr(self._livebuf), s), "gather")
        L.check(self._lib.tsb_scatter_rows(m, L.ptr(self._live), L.ptr(self._livebuf), L.ptr(out), s), "scatter")
