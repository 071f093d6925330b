"""CPU oracle for the implicit-FEM hot path -- TEST INFRASTRUCTURE ONLY.

A plain-NumPy restatement of the reference algorithm (tetsim,
/root/reference/pkg/src/tetsim) for the functions on the north-star path.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import it, and only as the checker or the timed
CPU baseline -- never as the product path.

Pinned against the reference: tests/golden/make_golden.py ran the reference
in the build container and stored its outputs in tests/golden/*.npz;
tests/test_oracle_golden.py checks every function here against those
fixtures (bit-exact where the reference is deterministic integer/merge work,
1e-13..1e-12 relative where BLAS summation order is involved).

Every function cites the reference file:line it restates.  Arrays only (no
dependence on the product package), so the oracle can check any
implementation that hands it NumPy arrays.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# SpMV -- krylov.py:63-96
# ---------------------------------------------------------------------------


def spmv(row_ptr, col_ind, values, x):
    """y_i = reduceat of a_ij * x_j over row i (krylov.py:63-70, 73-96).

    np.add.reduceat seeds each row with its first product and adds NumPy's
    pairwise sum of the rest; that summation order is the reference's.
    """
    row_ptr = np.asarray(row_ptr)
    nrows = len(row_ptr) - 1
    y = np.zeros(nrows)
    if len(col_ind) == 0:
        return y
    prod = np.asarray(values) * np.asarray(x)[np.asarray(col_ind)]
    starts = row_ptr[:-1]
    nonempty = np.flatnonzero(row_ptr[1:] > starts)
    if nonempty.size:
        y[nonempty] = np.add.reduceat(prod, starts[nonempty])
    return y


# ---------------------------------------------------------------------------
# Triplet merge -- assembly.py:322-343
# ---------------------------------------------------------------------------


def compress(vals, kept, kept_slots, nnz, fixed_diag_slots, coeffs=None):
    """values[s] = sum over kept triplets of coeff*val in ascending triplet order
    (np.bincount accumulates sequentially from 0.0, assembly.py:341); pinned
    diagonal slots forced to 1.0 (assembly.py:342)."""
    w = np.asarray(vals)[kept]
    if coeffs is not None:
        w = w * np.asarray(coeffs)[kept]
    out = np.bincount(kept_slots, weights=w, minlength=nnz)
    out[np.asarray(fixed_diag_slots, dtype=np.int64)] = 1.0
    return out


def sort_merge_pattern(rows, cols, n, fixed_dofs):
    """CSR pattern + slot of every triplet by a plain sort-merge (the pattern
    contract of build_pattern, assembly.py:235-312): pinned rows/cols dropped,
    one diagonal per pinned DOF, slots in (row, col) order."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    fixed = np.unique(np.asarray(fixed_dofs, dtype=np.int64))
    pinned = np.zeros(n, dtype=bool)
    pinned[fixed] = True
    kept = np.flatnonzero(~(pinned[rows] | pinned[cols]))
    pairs = set(zip(rows[kept].tolist(), cols[kept].tolist())) | {(int(f), int(f)) for f in fixed}
    keys = sorted(pairs)
    index = {k: i for i, k in enumerate(keys)}
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    for r, _ in keys:
        row_ptr[r + 1] += 1
    row_ptr = np.cumsum(row_ptr)
    col_ind = np.array([c for _, c in keys], dtype=np.int64)
    slot = np.full(len(rows), -1, dtype=np.int64)
    slot[kept] = [index[(int(r), int(c))] for r, c in zip(rows[kept], cols[kept])]
    fixed_slots = np.array([index[(int(f), int(f))] for f in fixed], dtype=np.int64)
    return row_ptr, col_ind, slot, fixed_slots


# ---------------------------------------------------------------------------
# Element physics -- models.py:95-238, 290-302
# ---------------------------------------------------------------------------


def rest_data(nodes, elements, young, poisson, density):
    """Rest gradients, volumes, Ke = V B^T C B (symmetrised), lumped-mass share
    (models.py:95-166, 290-302; integrator.py:127-132)."""
    el = np.asarray(elements)
    p = np.asarray(nodes)[el]
    dm = np.transpose(p[:, 1:] - p[:, :1], (0, 2, 1))
    vol = np.linalg.det(dm) / 6.0
    inv = np.linalg.inv(dm)
    g = np.empty((len(el), 4, 3))
    g[:, 1:] = inv
    g[:, 0] = -inv.sum(axis=1)
    lam = young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson))
    mu = young / (2.0 * (1.0 + poisson))
    m = len(el)
    B = np.zeros((m, 6, 12))
    for a in range(4):
        gx, gy, gz = g[:, a, 0], g[:, a, 1], g[:, a, 2]
        c = 3 * a
        B[:, 0, c], B[:, 1, c + 1], B[:, 2, c + 2] = gx, gy, gz
        B[:, 3, c], B[:, 3, c + 1] = gy, gx
        B[:, 4, c + 1], B[:, 4, c + 2] = gz, gy
        B[:, 5, c], B[:, 5, c + 2] = gz, gx
    Cm = np.zeros((6, 6))
    Cm[:3, :3] = lam
    Cm[np.arange(3), np.arange(3)] += 2.0 * mu
    Cm[np.arange(3, 6), np.arange(3, 6)] = mu
    ke = np.einsum("eji,jk,ekl->eil", B, Cm, B) * vol[:, None, None]
    ke = 0.5 * (ke + np.transpose(ke, (0, 2, 1)))
    edges = p[:, 1:] - p[:, :1]
    share = density * (np.linalg.det(edges) / 6.0) / 4.0
    gdof = (3 * el[:, :, None] + np.arange(3)).reshape(m, 12)
    return {"grads": g, "vol": vol, "ke": ke, "share": share, "gdof": gdof, "lam": lam, "mu": mu}


def polar(F, tol=1e-12, max_iter=50, extra=0):
    """Newton R <- (R + R^-T)/2, global stop on max |dR| (models.py:174-189).
    `extra` > 0 runs that many more iterations after the stop; a Generator
    perturbs every entry of the result by a random relative 2^-52 (test
    knobs: the rounding-level sensitivity of the forces to R)."""
    r = F.copy()
    for _ in range(max_iter):
        nxt = 0.5 * (r + np.transpose(np.linalg.inv(r), (0, 2, 1)))
        d = np.abs(nxt - r).max()
        r = nxt
        if d < tol:
            break
    if isinstance(extra, np.random.Generator):
        return r * (1.0 + 2.0 ** -52 * extra.uniform(-1.0, 1.0, r.shape))
    for _ in range(extra):
        r = 0.5 * (r + np.transpose(np.linalg.inv(r), (0, 2, 1)))
    return r


def corotational(nodes, elements, rest, positions, velocities, linear=False, extra_newton=0):
    """(f, kv, krot) of the corotational law (models.py:200-238); linear=True
    uses R = I (BASELINE config 1)."""
    el = np.asarray(elements)
    m = len(el)
    ndof = 3 * len(positions)
    xe = np.asarray(positions)[el]
    F = np.einsum("eai,eaj->eij", xe, rest["grads"])
    R = np.broadcast_to(np.eye(3), (m, 3, 3)).copy() if linear else polar(F, extra=extra_newton)
    rb = np.zeros((m, 12, 12))
    for a in range(4):
        rb[:, 3 * a:3 * a + 3, 3 * a:3 * a + 3] = R
    xf = xe.reshape(m, 12)
    x0 = np.asarray(nodes)[el].reshape(m, 12)
    u = np.einsum("eqp,eq->ep", rb, xf) - x0
    fe = np.einsum("epq,eq->ep", rb, np.einsum("epq,eq->ep", rest["ke"], u))
    f = np.bincount(rest["gdof"].ravel(), weights=fe.ravel(), minlength=ndof)
    krot = rb @ rest["ke"] @ np.transpose(rb, (0, 2, 1))
    ve = np.asarray(velocities).reshape(-1, 3)[el].reshape(m, 12)
    kv = np.bincount(rest["gdof"].ravel(), weights=np.einsum("epq,eq->ep", krot, ve).ravel(), minlength=ndof)
    return f, kv, krot


def stvk(nodes, elements, rest, positions, velocities):
    """(f, kv, kblocks) of the St-Venant-Kirchhoff law (models.py:241-287):
    F = sum_a x_a g_a^T, G = (F^T F - I)/2, S = lam tr(G) I + 2 mu G,
    f_a = V F S g_a, K_ab = V(lam h_a h_b^T + mu h_b h_a^T + mu (g_a.g_b) F F^T
    + (g_a^T S g_b) I) with h_a = F g_a (material + geometric tangent)."""
    el = np.asarray(elements)
    m = len(el)
    ndof = 3 * len(positions)
    g, vol, lam, mu = rest["grads"], rest["vol"], rest["lam"], rest["mu"]
    xe = np.asarray(positions)[el]
    f = np.einsum("eai,eaj->eij", xe, g)
    green = 0.5 * (np.einsum("eki,ekj->eij", f, f) - np.eye(3))
    s = lam * np.trace(green, axis1=1, axis2=2)[:, None, None] * np.eye(3) + 2.0 * mu * green
    fe = vol[:, None, None] * np.einsum("eij,eaj->eai", f @ s, g)
    force = np.bincount(rest["gdof"].ravel(), weights=fe.reshape(m, 12).ravel(), minlength=ndof)
    fg = np.einsum("eij,eaj->eai", f, g)
    fft = f @ np.transpose(f, (0, 2, 1))
    gg = np.einsum("eai,ebi->eab", g, g)
    gsg = np.einsum("eai,eij,ebj->eab", g, s, g)
    k = lam * np.einsum("eai,ebk->eaibk", fg, fg)
    k += mu * np.einsum("eak,ebi->eaibk", fg, fg)
    k += mu * np.einsum("eab,eik->eaibk", gg, fft)
    k += np.einsum("eab,ik->eaibk", gsg, np.eye(3))
    k *= vol[:, None, None, None, None]
    kblocks = k.reshape(m, 12, 12)
    ve = np.asarray(velocities).reshape(-1, 3)[el].reshape(m, 12)
    kv = np.bincount(rest["gdof"].ravel(), weights=np.einsum("epq,eq->ep", kblocks, ve).ravel(), minlength=ndof)
    return force, kv, kblocks


def assembly_pattern(nodes, elements, fixed_nodes, rest):
    """Triplet -> CSR slot mapping of the fused pass (the reference's full
    assembly, assembly.py:235-312; reused while the fill order and the pinned
    DOFs do not change, assembly.py:399-405): mass triplets first, then 144
    stiffness triplets per element."""
    ndof = 3 * len(nodes)
    gdof = rest["gdof"]
    mass_rows = gdof.reshape(-1)
    rows = np.concatenate([mass_rows, np.repeat(gdof, 12, axis=1).ravel()])
    cols = np.concatenate([mass_rows, np.tile(gdof, (1, 12)).ravel()])
    fixed = (3 * np.asarray(fixed_nodes, dtype=np.int64)[:, None] + np.arange(3)).ravel()
    row_ptr, col_ind, slot, fixed_slots = _fast_pattern(rows, cols, ndof, fixed)
    kept = np.flatnonzero(slot >= 0)
    return {"row_ptr": row_ptr, "col_ind": col_ind, "kept": kept, "kept_slots": slot[kept],
            "fixed_slots": fixed_slots, "fixed": fixed}


def assemble_system(nodes, elements, fixed_nodes, rest, positions, velocities, f_ext_state,
                    dt, gravity, rayleigh_mass=0.0, rayleigh_stiffness=0.0, linear=False, law=None,
                    pattern=None, extra_newton=0):
    """A values (CSR order), b, f_int, f_ext, row_ptr, col_ind of one fused pass
    (integrator.py:145-169): mass triplets first, then 144 stiffness triplets
    per element, per-triplet coefficients, bincount merge, pinned rows identity.
    `pattern` (assembly_pattern) is the cached mapping of the reference's fast
    path; without it the mapping is rebuilt (full assembly)."""
    el = np.asarray(elements)
    m = len(el)
    ndof = 3 * len(nodes)
    gdof = rest["gdof"]
    mass_rows = gdof.reshape(-1)
    mass_vals = np.repeat(rest["share"], 12)
    if law == "stvk":
        f_int, kv, krot = stvk(nodes, elements, rest, positions, velocities)
    else:
        f_int, kv, krot = corotational(nodes, elements, rest, positions, velocities, linear or law == "linear",
                                       extra_newton)
    vals = np.concatenate([mass_vals, krot.reshape(-1)])
    h = dt
    coeffs = np.empty(len(vals))
    coeffs[: 12 * m] = 1.0 + h * rayleigh_mass
    coeffs[12 * m:] = h * (h + rayleigh_stiffness)
    if pattern is None:
        pattern = assembly_pattern(nodes, elements, fixed_nodes, rest)
    row_ptr, col_ind, fixed = pattern["row_ptr"], pattern["col_ind"], pattern["fixed"]
    fixed_slots = pattern["fixed_slots"]
    values = compress(vals, pattern["kept"], pattern["kept_slots"], len(col_ind), fixed_slots, coeffs)
    mass_diag = np.bincount(mass_rows, weights=mass_vals, minlength=ndof)
    f_ext = np.asarray(f_ext_state) + (mass_diag.reshape(-1, 3) * np.asarray(gravity)).ravel()
    b = f_ext - f_int - (h + rayleigh_stiffness) * kv
    if rayleigh_mass:
        b -= rayleigh_mass * (mass_diag * np.asarray(velocities).ravel())
    b[fixed] = 0.0
    return {"values": values, "row_ptr": row_ptr, "col_ind": col_ind, "b": b, "f_int": f_int,
            "f_ext": f_ext, "kv": kv, "fixed_slots": fixed_slots}


def _fast_pattern(rows, cols, n, fixed):
    """Vectorised sort-merge (same contract as sort_merge_pattern)."""
    pinned = np.zeros(n, dtype=bool)
    pinned[fixed] = True
    kept = np.flatnonzero(~(pinned[rows] | pinned[cols]))
    keys = np.concatenate([rows[kept] * n + cols[kept], fixed * n + fixed])
    order = np.argsort(keys, kind="stable")
    sk = keys[order]
    first = np.ones(len(sk), dtype=bool)
    first[1:] = sk[1:] != sk[:-1]
    ids = np.cumsum(first) - 1
    uniq = sk[first]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(uniq // n, minlength=n), out=row_ptr[1:])
    work_slot = np.empty(len(keys), dtype=np.int64)
    work_slot[order] = ids
    slot = np.full(len(rows), -1, dtype=np.int64)
    slot[kept] = work_slot[: len(kept)]
    return row_ptr, uniq % n, slot, work_slot[len(kept):]


# ---------------------------------------------------------------------------
# PCG -- krylov.py:104-158
# ---------------------------------------------------------------------------


def jacobi_inv_diag(row_ptr, col_ind, values, n):
    """1 / diag(A) (krylov.py:112-117, assembly.py:154-159)."""
    row_of = np.repeat(np.arange(n), np.diff(row_ptr))
    d = np.zeros(n)
    on = row_of == np.asarray(col_ind)
    d[np.asarray(col_ind)[on]] = np.asarray(values)[on]
    if np.any(d == 0.0):
        raise ZeroDivisionError(f"zero diagonal entry at row {int(np.flatnonzero(d == 0.0)[0])}")
    return 1.0 / d


def pcg(row_ptr, col_ind, values, b, precond=None, tol=1e-9, max_it=1000, x0=None):
    """Textbook PCG with the reference's exits and ordering (krylov.py:120-158).

    precond: callable r -> z (None = identity).  Returns (x, iterations,
    final_residual, converged)."""
    n = len(row_ptr) - 1
    apply = (lambda r: r) if precond is None else precond
    x = np.zeros(n) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    b = np.asarray(b, dtype=np.float64)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return np.zeros(n), 0, 0.0, True
    r = b - spmv(row_ptr, col_ind, values, x) if x0 is not None else b.copy()
    res = float(np.linalg.norm(r)) / bnorm
    if res <= tol:
        return x, 0, res, True
    z = apply(r)
    p = z.copy()
    rz = float(r @ z)
    it = 0
    conv = False
    while it < max_it:
        ap = spmv(row_ptr, col_ind, values, p)
        alpha = rz / float(p @ ap)
        x += alpha * p
        r -= alpha * ap
        it += 1
        res = float(np.linalg.norm(r)) / bnorm
        if res <= tol:
            conv = True
            break
        z = apply(r)
        rzn = float(r @ z)
        p = z + (rzn / rz) * p
        rz = rzn
    return x, it, res, conv


# ---------------------------------------------------------------------------
# Level-scheduled LDL^T solves -- ndprecond.py:623-700
# Factors are duck-typed: .blocks/.levels (objects with start, stop, anc,
# l11, l21, tile, tile_inv), .d, .plan.perm, .plan.iperm.
# ---------------------------------------------------------------------------


def _forward(bf, seg):
    m = len(seg)
    for it, t0 in enumerate(range(0, m, bf.tile)):
        t1 = min(t0 + bf.tile, m)
        seg[t0:t1] = bf.tile_inv[it] @ seg[t0:t1]
        if t1 < m:
            seg[t1:] -= bf.l11[t1:, t0:t1] @ seg[t0:t1]


def _backward(bf, seg):
    m = len(seg)
    nt = (m + bf.tile - 1) // bf.tile
    for it in range(nt - 1, -1, -1):
        t0 = it * bf.tile
        t1 = min(t0 + bf.tile, m)
        if t1 < m:
            seg[t0:t1] -= bf.l11[t1:, t0:t1].T @ seg[t1:]
        seg[t0:t1] = bf.tile_inv[it].T @ seg[t0:t1]


def solve_lower(factors, r):
    """L y = r, column-major with ancestor pre-accumulation applied in block
    order at each level barrier (ndprecond.py:623-631, 647-671)."""
    y = np.array(r, dtype=np.float64, copy=True)
    for level in factors.levels:
        contribs = []
        for bf in level:
            seg = y[bf.start:bf.stop]
            _forward(bf, seg)
            contribs.append(bf.l21 @ seg if len(bf.anc) else None)
        for bf, c in zip(level, contribs):
            if c is not None:
                y[bf.anc] -= c
    return y


def solve_upper(factors, w):
    """L^T z = w, levels reversed, row-major gathers (ndprecond.py:634-644, 674-691)."""
    z = np.array(w, dtype=np.float64, copy=True)
    for level in reversed(factors.levels):
        for bf in level:
            seg = z[bf.start:bf.stop]
            if len(bf.anc):
                seg -= bf.l21.T @ z[bf.anc]
            _backward(bf, seg)
    return z


def apply(factors, r):
    """z = P^T L^-T D^-1 L^-1 P r (ndprecond.py:694-700)."""
    y = solve_lower(factors, np.asarray(r, dtype=np.float64)[factors.plan.perm])
    y /= factors.d
    return solve_upper(factors, y)[factors.plan.iperm]


def forward_substitution(row_ptr, col_ind, values, r):
    """Textbook (I + L) y = r for strict-lower CSR L (tests/helpers.py:115-123 of the reference)."""
    y = np.asarray(r, dtype=np.float64).copy()
    for i in range(len(row_ptr) - 1):
        lo, hi = row_ptr[i], row_ptr[i + 1]
        if hi > lo:
            y[i] -= values[lo:hi] @ y[col_ind[lo:hi]]
    return y


def backward_substitution(row_ptr, col_ind, values, w):
    """Textbook (I + L)^T z = w (tests/helpers.py:126-132 of the reference)."""
    z = np.asarray(w, dtype=np.float64).copy()
    for j in range(len(row_ptr) - 2, -1, -1):
        lo, hi = row_ptr[j], row_ptr[j + 1]
        if hi > lo:
            z[col_ind[lo:hi]] -= values[lo:hi] * z[j]
    return z


# ---------------------------------------------------------------------------
# Plane contact stage -- contact.py:89-257
# ---------------------------------------------------------------------------


def detect_plane_contacts(positions, plane_z):
    """Unilateral rows for nodes below z = plane_z (contact.py:89-106):
    -> (nodes, dof columns 3i+2, coefficients -1, violation plane_z - z)."""
    pen = plane_z - np.asarray(positions)[:, 2]
    nodes = np.flatnonzero(pen > 0.0)
    return nodes, 3 * nodes + 2, np.full(len(nodes), -1.0), pen[nodes]


def build_compliance(cols, coefs, ndof, solve_fn):
    """W = J A^-1 J^T column by column for one-entry rows (contact.py:109-125),
    symmetrised by averaging; -> (W, S)."""
    m = len(cols)
    s = np.empty((ndof, m))
    for i in range(m):
        e = np.zeros(ndof)
        e[cols[i]] = coefs[i]
        s[:, i] = solve_fn(e)
    w = np.empty((m, m))
    for i in range(m):
        w[i] = coefs * s[cols, i]
    return 0.5 * (w + w.T), s


def projected_gauss_seidel(w, rhs, unilateral, tol=1e-12, max_sweeps=500):
    """Projected Gauss-Seidel in constraint order (contact.py:128-166)."""
    m = len(rhs)
    lam = np.zeros(m)
    if m == 0:
        return lam
    diag = np.diagonal(w).copy()
    usable = diag != 0.0
    for _ in range(max_sweeps):
        dmax = 0.0
        for i in range(m):
            if not usable[i]:
                lam[i] = 0.0
                continue
            new = lam[i] + (rhs[i] - w[i] @ lam) / diag[i]
            if unilateral[i] and new < 0.0:
                new = 0.0
            dmax = max(dmax, abs(new - lam[i]))
            lam[i] = new
        scale = np.abs(lam).max()
        if dmax <= tol * scale or scale == 0.0:
            break
    return lam


def advance(acc, x, v, dt, fixed_nodes):
    """Kinematic update of an implicit step (integrator.py:192-208 /
    contact.py:169-195): a[pinned] = 0, v' = v + h a, x' = x + h v', pinned keep."""
    acc = np.asarray(acc, dtype=np.float64).reshape(-1, 3).copy()
    acc[fixed_nodes] = 0.0
    vel = v + dt * acc
    pos = x + dt * vel
    vel[fixed_nodes] = v[fixed_nodes]
    pos[fixed_nodes] = x[fixed_nodes]
    return pos, vel, acc
