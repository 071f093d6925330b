"""Device-side assembly plan: HBM layout of the mesh, the fixed CSR pattern and
the deterministic gather lists (host setup, built once per mesh/BC).

Pattern contract (bit-exact with the reference's build_pattern,
assembly.py:235-312): with whole pinned nodes the pattern is an exact 3x3
block pattern over free nodes -- row 3I+c holds columns 3J+d for every free
node J sharing an element with free node I (J ascending, d inner); pinned
DOFs keep one diagonal slot.  It is derived here straight from the element
topology (no 156 m-entry triplet sort), and `tests/` check it equals the
reference's triplet-built pattern.

HBM layout (all int32 indices):
  conn      [4][m]      element node ids (SoA -> coalesced per node slot)
  grads     [m][12]     rest gradients, 96 B per tet (6 x 16 B loads)
  vol, share [m]        rest volume, rho V / 4
  blk       [nb][4]     slot0, row length, list begin, list end per 3x3 block
  blk_list  [16 m']     e*16 + a*4 + b, grouped by block, ascending e
  node_ptr/node_list    e*4 + a per node, ascending e
  work      [m][36]     rotated gradients, f_e, (K v)_e (element pass output)
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib


def topology_pattern(mesh):
    """-> dict with row_ptr, col_ind, fixed_diag_slots, block arrays, node lists."""
    N = mesh.node_count
    el = mesh.elements
    m = len(el)
    pinned = np.zeros(N, dtype=bool)
    pinned[mesh.fixed_nodes] = True

    a_idx = np.repeat(np.arange(4), 4)
    b_idx = np.tile(np.arange(4), 4)
    I = el[:, a_idx].ravel()
    J = el[:, b_idx].ravel()
    code = (np.arange(m, dtype=np.int64)[:, None] * 16 + a_idx * 4 + b_idx).ravel()
    keep = ~(pinned[I] | pinned[J])
    I, J, code = I[keep], J[keep], code[keep]
    key = I * N + J
    order = np.argsort(key, kind="stable")
    key = key[order]
    code = code[order]
    first = np.ones(len(key), dtype=bool)
    first[1:] = key[1:] != key[:-1]
    starts = np.flatnonzero(first)
    ends = np.append(starts[1:], len(key))
    bkey = key[starts]
    bI, bJ = bkey // N, bkey % N
    nb_row = np.bincount(bI, minlength=N)
    nblk = len(bkey)

    rowlen = np.where(pinned, 1, 3 * nb_row)           # per node, each of its 3 rows
    row_len_dof = np.repeat(rowlen, 3)
    row_ptr = np.zeros(3 * N + 1, dtype=np.int64)
    np.cumsum(row_len_dof, out=row_ptr[1:])
    nnz = int(row_ptr[-1])

    first_blk_of_row = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(nb_row, out=first_blk_of_row[1:])
    k_in_row = np.arange(nblk) - first_blk_of_row[bI]
    slot0 = row_ptr[3 * bI] + 3 * k_in_row
    brow = 3 * nb_row[bI]

    col_ind = np.empty(nnz, dtype=np.int64)
    for c in range(3):
        for d in range(3):
            col_ind[slot0 + c * brow + d] = 3 * bJ + d
    fixed_dofs = mesh.fixed_dofs()
    fixed_slots = row_ptr[fixed_dofs]
    col_ind[fixed_slots] = fixed_dofs

    node_flat = el.ravel()
    norder = np.argsort(node_flat, kind="stable")
    node_ptr = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(np.bincount(node_flat, minlength=N), out=node_ptr[1:])

    for a in (row_ptr, col_ind, fixed_slots):
        a.setflags(write=False)
    return {
        "row_ptr": row_ptr, "col_ind": col_ind, "fixed_diag_slots": fixed_slots,
        "blk": np.stack([slot0, brow, starts, ends], axis=1),
        "blk_list": code, "node_ptr": node_ptr, "node_list": norder,
    }


def device_topology_pattern(mesh, keep_device=False):
    """topology_pattern built on the device (csrc/pattern.cu, tsb_pattern_count/fill):
    the same arrays, downloaded for the host-side CsrMatrix; with keep_device
    the int32 device copies the assembly plan uses are returned under "dev"."""
    import ctypes as C

    t = _lib.require_cuda()
    N, el = mesh.node_count, mesh.elements
    m = len(el)
    dev = "cuda"
    conn = t.from_numpy(_i32(el.T)).to(dev)
    pinned = np.zeros(N, dtype=np.uint8)
    pinned[mesh.fixed_nodes] = 1
    pin = t.from_numpy(pinned).to(dev)
    i64 = lambda k: t.empty(max(k, 1), dtype=t.int64, device=dev)  # noqa: E731
    i32 = lambda k: t.empty(max(k, 1), dtype=t.int32, device=dev)  # noqa: E731
    buf = {"tmp": i64(N), "sums": i64(N // 1024 + 2), "node_ptr": i64(N + 1), "node_list": i32(4 * m),
           "cand": i32(16 * m), "nbr": i64(N), "blk_ptr": i64(N + 1), "row_base": i64(N + 1)}
    P = _lib.ptr
    d = _lib.PatternDesc(n_nodes=N, n_elems=m, d_conn=P(conn), d_pinned=P(pin), d_tmp=P(buf["tmp"]),
                         d_sums=P(buf["sums"]), d_node_ptr=P(buf["node_ptr"]), d_node_list=P(buf["node_list"]),
                         d_cand=P(buf["cand"]), d_nbr=P(buf["nbr"]), d_blk_ptr=P(buf["blk_ptr"]),
                         d_row_base=P(buf["row_base"]), n_blocks=-1, nnz=-1, n_contrib=-1)
    lib = _lib.load()
    _lib.check(lib.tsb_pattern_count(C.byref(d), _lib.stream_ptr()), "pattern_count")
    nb, nnz = int(d.n_blocks), int(d.nnz)
    if nnz >= 2**31:
        raise OverflowError("pattern exceeds int32 range of the device layout")
    buf.update(sums2=i64(nb // 1024 + 2), ccount=i64(nb), cptr=i64(nb + 1), row_ptr=i32(3 * N + 1),
               col_ind=i32(nnz), blk=i32(4 * nb), blk_list=i32(16 * m))
    d.d_sums = P(buf["sums2"])
    d.d_ccount, d.d_cptr, d.d_row_ptr = P(buf["ccount"]), P(buf["cptr"]), P(buf["row_ptr"])
    d.d_col_ind, d.d_blk, d.d_blk_list = P(buf["col_ind"]), P(buf["blk"]), P(buf["blk_list"])
    _lib.check(lib.tsb_pattern_fill(C.byref(d), _lib.stream_ptr()), "pattern_fill")
    nc = int(d.n_contrib)
    row_ptr = buf["row_ptr"][:3 * N + 1].cpu().numpy().astype(np.int64)
    col_ind = buf["col_ind"][:nnz].cpu().numpy().astype(np.int64)
    fixed_dofs = mesh.fixed_dofs()
    out = {
        "row_ptr": row_ptr, "col_ind": col_ind, "fixed_diag_slots": row_ptr[fixed_dofs],
        "blk": buf["blk"][:4 * nb].cpu().numpy().astype(np.int64).reshape(nb, 4),
        "blk_list": buf["blk_list"][:nc].cpu().numpy().astype(np.int64),
        "node_ptr": buf["node_ptr"][:N + 1].cpu().numpy(),
        "node_list": buf["node_list"][:4 * m].cpu().numpy().astype(np.int64),
    }
    for a in (out["row_ptr"], out["col_ind"], out["fixed_diag_slots"]):
        a.setflags(write=False)
    if keep_device:
        out["dev"] = {k: buf[k] for k in ("row_ptr", "col_ind", "blk", "blk_list", "node_list")}
    return out


def _i32(a):
    a = np.asarray(a)
    if a.size and (a.max() >= 2**31 or a.min() < -(2**31)):
        raise OverflowError("index exceeds int32 range of the device layout")
    return np.ascontiguousarray(a, dtype=np.int32)


BLK_WINDOW = int(os.environ.get("TSB_BLK_WINDOW", "2048"))


MIRROR_BLOCKS = os.environ.get("TSB_MIRROR_BLOCKS", "1") != "0"


def _mirror_work(pattern, n_nodes):
    """Block gather work list using K_ba = K_ab^T: only blocks (I, J) with
    I <= J are summed; each off-diagonal one also writes block (J, I) (same
    contributing elements, same ascending order).  -> (work [nw][4], mirror
    [nw][2] = slot0, row length of (J, I), or -1 for a diagonal block)."""
    blk = np.asarray(pattern["blk"], dtype=np.int64)
    row_ptr = np.asarray(pattern["row_ptr"], dtype=np.int64)
    col_ind = np.asarray(pattern["col_ind"], dtype=np.int64)
    bI = (np.searchsorted(row_ptr, blk[:, 0], side="right") - 1) // 3
    bJ = col_ind[blk[:, 0]] // 3
    key = bI * n_nodes + bJ  # CSR order: ascending
    up = bI <= bJ
    mk = np.searchsorted(key, bJ[up] * n_nodes + bI[up])
    mirror = np.where((bI[up] < bJ[up])[:, None], blk[mk][:, :2], -1)
    return blk[up], mirror


def _warp_uniform_order(blk):
    """Block gather work order (a permutation of the work list): within
    windows of BLK_WINDOW consecutive CSR blocks (about the same node rows, so
    the element scratch they read is still shared through L2), blocks sorted
    by contribution count, heaviest first -- a warp's 32 threads then loop over
    about the same number of contributions instead of every warp waiting for
    its one diagonal block (~4x the contributions of an off-diagonal one).
    Each entry carries its own CSR slot, so the order changes nothing in the
    sums."""
    blk = np.asarray(blk)
    if BLK_WINDOW <= 0 or len(blk) == 0:
        return np.arange(len(blk))
    cnt = blk[:, 3] - blk[:, 2]
    return np.concatenate([w0 + np.argsort(-cnt[w0:w0 + BLK_WINDOW], kind="stable")
                           for w0 in range(0, len(blk), BLK_WINDOW)])


LAWS = {"corotational": 0, "linear": 1, "stvk": 2}  # tsb.h TSB_LAW_*


def law_code(law) -> int:
    try:
        return LAWS[law]
    except KeyError:
        raise ValueError(f"no device kernel for material law {law!r}") from None


class AssemblyPlan:
    """Device buffers + the C struct handed to tsb_assemble_corot."""

    def __init__(self, precomp, pattern=None, mass_share=None, mass_diag=None, gravity=None,
                 fixed_dof=None, n_nodes=None):
        t = _lib.require_cuda()
        dev = "cuda"
        el = precomp.elements
        m = len(el)
        N = len(precomp.rest_positions) if n_nodes is None else n_nodes
        self.m, self.N = m, N

        def up(a, dtype):
            return t.from_numpy(np.array(a, dtype=dtype, copy=True)).to(dev)

        self.conn = t.from_numpy(_i32(el.T)).to(dev)
        self.grads = up(precomp.grads.reshape(m, 12), np.float64)
        self.vol = up(precomp.volume, np.float64)
        self.rest = up(precomp.rest_positions.reshape(-1), np.float64)
        self.share = up(mass_share if mass_share is not None else np.zeros(m), np.float64)
        self.mass_diag = up(mass_diag if mass_diag is not None else np.zeros(3 * N), np.float64)
        self.gravity = up(gravity if gravity is not None else np.zeros(3 * N), np.float64)
        fd = np.zeros(3 * N, dtype=np.uint8)
        if fixed_dof is not None:
            fd[fixed_dof] = 1
        self.fixed_dof = up(fd, np.uint8)
        self.work = t.empty(max(m, 1) * 48, dtype=t.float64, device=dev)
        self.gab = t.empty(max(m, 1) * 10, dtype=t.float64, device=dev)  # g_a . g_b per tet (tsb_assembly_setup)
        self.flags = t.zeros(4, dtype=t.int32, device=dev)
        self.pattern = pattern
        self.blk_mirror = None
        if pattern is not None:
            work, mirror = _mirror_work(pattern, N) if MIRROR_BLOCKS else (np.asarray(pattern["blk"]), None)
            order = _warp_uniform_order(work)
            self.blk = t.from_numpy(_i32(work[order])).to(dev)
            if mirror is not None:
                self.blk_mirror = t.from_numpy(_i32(mirror[order])).to(dev)
            self.blk_list = t.from_numpy(_i32(pattern["blk_list"])).to(dev)
            self.fixed_slots = t.from_numpy(_i32(pattern["fixed_diag_slots"])).to(dev)
            node_ptr, node_list = pattern["node_ptr"], pattern["node_list"]
            nb, nnz, nfix = len(self.blk), len(pattern["col_ind"]), len(pattern["fixed_diag_slots"])
        else:
            self.blk = self.blk_list = self.fixed_slots = None
            flat = el.ravel()
            node_list = np.argsort(flat, kind="stable")
            node_ptr = np.zeros(N + 1, dtype=np.int64)
            np.cumsum(np.bincount(flat, minlength=N), out=node_ptr[1:])
            nb = nnz = nfix = 0
        self.node_ptr = t.from_numpy(_i32(node_ptr)).to(dev)
        self.node_list = t.from_numpy(_i32(node_list)).to(dev)
        P = _lib.ptr
        self.c = _lib.AsmPlan(
            n_nodes=N, n_elems=m, n_blocks=nb, nnz=nnz, n_fixed_slots=nfix,
            d_conn=P(self.conn), d_grads=P(self.grads), d_vol=P(self.vol), d_mass_share=P(self.share),
            d_rest=P(self.rest), d_mass_diag=P(self.mass_diag), d_gravity=P(self.gravity),
            d_fixed_dof=P(self.fixed_dof), d_blk=P(self.blk), d_blk_list=P(self.blk_list),
            d_node_ptr=P(self.node_ptr), d_node_list=P(self.node_list),
            d_fixed_slots=P(self.fixed_slots), d_work=P(self.work), d_flags=P(self.flags),
            d_gab=P(self.gab), d_blk_mirror=P(self.blk_mirror),
        )
        import ctypes as C

        _lib.check(_lib.load().tsb_assembly_setup(C.byref(self.c), _lib.stream_ptr()), "assembly_setup")
        self.lame = precomp.lame

    @classmethod
    def for_model(cls, precomp):
        return cls(precomp)

    def coeffs(self, h=0.0, beta=0.0, alpha=0.0, cm=1.0, ck=1.0, law="corotational", want_matrix=True):
        lam, mu = self.lame
        return _lib.AsmCoeffs(lam=lam, mu=mu, h=h, rayleigh_stiffness=beta, rayleigh_mass=alpha,
                              cm=cm, ck=ck, law=law_code(law), want_matrix=int(want_matrix))

    def run(self, coeffs, x, v, f_ext_state, values, b, f_int, kv, f_ext):
        import ctypes as C

        P = _lib.ptr
        _lib.check(_lib.load().tsb_assemble_corot(
            C.byref(self.c), C.byref(coeffs), P(x), P(v), P(f_ext_state), P(values), P(b),
            P(f_int), P(kv), P(f_ext), _lib.stream_ptr()), "assemble")

    def element_pass(self, positions, velocities, want_blocks=False, law="corotational"):
        """Model-level pass (no matrix): (f, kv, kblocks|None) in the caller's array kind."""
        import ctypes as C

        t = _lib.torch()
        host = not _lib.is_tensor(positions)
        x = _lib.to_device(np.asarray(positions, dtype=np.float64).reshape(-1) if host
                           else positions.reshape(-1), t.float64)
        v = None
        if velocities is not None:
            v = _lib.to_device(np.asarray(velocities, dtype=np.float64).reshape(-1)
                               if not _lib.is_tensor(velocities) else velocities.reshape(-1), t.float64)
        n = 3 * self.N
        f = t.empty(n, dtype=t.float64, device="cuda")
        kv = t.empty(n, dtype=t.float64, device="cuda")
        co = self.coeffs(law=law, want_matrix=False)
        vz = v if v is not None else t.zeros(n, dtype=t.float64, device="cuda")
        self.run(co, x, vz, None, None, None, f, kv, None)
        kb = None
        if want_blocks:
            kb = t.empty(self.m * 144, dtype=t.float64, device="cuda")
            _lib.check(_lib.load().tsb_element_blocks(C.byref(self.c), C.byref(co), _lib.ptr(x),
                                                      _lib.ptr(kb), _lib.stream_ptr()), "element_blocks")
        if int(self.flags[0].item()):
            from .models import ModelError

            raise ModelError("non-finite positions")
        if host:
            return (f.cpu().numpy(), kv.cpu().numpy() if v is not None else None,
                    kb.cpu().numpy().reshape(self.m, 12, 12) if kb is not None else None)
        return f, (kv if v is not None else None), (kb.view(self.m, 12, 12) if kb is not None else None)
