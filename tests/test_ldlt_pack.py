"""CPU check of the device panel layout and the DAG item lists (csrc/ldlt.cu):
a serial NumPy emulator executes the work items in dispatch order with the
kernel's exact data flow; it must (a) only ever find its dependencies
satisfied (the order is topological, hence deadlock-free on the persistent
kernel) and (b) reproduce the oracle's level-scheduled sweeps."""

import numpy as np
import pytest

from conftest import clamped_beam
from oracle import tetsim_oracle as O
from paper_2306_05893_b200 import _ldlt_pack as K, mesh as M, ndprecond as ND
from paper_2306_05893_b200.assembly import CsrMatrix


def _panel_inverse(H, p, which):
    """Unpack the panel's explicit diagonal-triangle inverse (unit lower) from the
    lower sweep's column-packed copy or the upper sweep's row-packed copy."""
    w = int(H["p_w"][p])
    blob = H[which][H["p_tri"][p]: H["p_tri"][p] + H["p_tri_len"][p]]
    Li = np.eye(w)
    if which == "tri":
        cj, ri = np.triu_indices(w, 1)
        Li[ri, cj] = blob[: len(ri)]
    else:
        ri, cj = np.tril_indices(w, -1)
        Li[ri, cj] = blob[: len(ri)]
    return Li


def emulate_lower(H, r):
    n, P = H["n"], H["P"]
    y = np.zeros(n)
    cbuf = np.zeros(max(H["ncbuf"], 1))
    contrib = np.zeros(P, dtype=np.int64)
    flag = np.zeros(P, dtype=bool)
    for typ, p, r0, r1, doff, dcnt, _, _ in H["items_l"]:
        s, w = int(H["p_start"][p]), int(H["p_w"][p])
        if typ == K.IT_DIAG:
            assert contrib[p] == dcnt, "DIAG dispatched before its contributions"
            seg = np.empty(w)
            for k in range(w):
                row = s + k
                v = r[row]
                for q in range(H["cin_ptr"][row], H["cin_ptr"][row + 1]):
                    v -= cbuf[q]
                seg[k] = v
            y[s:s + w] = _panel_inverse(H, p, "tri") @ seg
            flag[p] = True
        else:
            assert typ == K.IT_OFF and flag[p]
            nb = H["p_below"][p + 1] - H["p_below"][p] if p + 1 < P else len(H["below"]) - H["p_below"][p]
            ws = w + (w & 1)  # rows padded to an even stride (16-byte TMA chunks)
            pan = H["pan"][H["p_pan"][p]: H["p_pan"][p] + nb * ws].reshape(nb, ws)[:, :w]
            cbuf[H["cslot"][H["p_cb"][p] + r0: H["p_cb"][p] + r1]] = pan[r0:r1] @ y[s:s + w]
            contrib[H["deps"][doff: doff + dcnt]] += 1
    return y


def emulate_upper(H, w_in):
    n, P = H["n"], H["P"]
    z = np.zeros(n)
    part = np.zeros(max(H["npart"], 1))
    ready = np.zeros(P, dtype=np.int64)
    flag = np.zeros(P, dtype=bool)
    for typ, p, r0, r1, doff, dcnt, ooff, _ in H["items_u"]:
        s, w = int(H["p_start"][p]), int(H["p_w"][p])
        if typ == K.IT_OFFT:
            assert all(flag[H["deps"][doff: doff + dcnt]]), "OFFT dispatched before its owners"
            nb = H["p_below"][p + 1] - H["p_below"][p] if p + 1 < P else len(H["below"]) - H["p_below"][p]
            ws = w + (w & 1)  # rows padded to an even stride (16-byte TMA chunks)
            pan = H["pan"][H["p_pan"][p]: H["p_pan"][p] + nb * ws].reshape(nb, ws)[:, :w]
            below = H["below"][H["p_below"][p]: H["p_below"][p] + nb]
            part[ooff: ooff + w] = pan[r0:r1].T @ z[below[r0:r1]]
            ready[p] += 1
        else:
            assert typ == K.IT_DIAGT and ready[p] == dcnt
            seg = w_in[s:s + w] - sum(part[ooff + q * w: ooff + (q + 1) * w] for q in range(dcnt))
            z[s:s + w] = _panel_inverse(H, p, "tri_u").T @ seg
            flag[p] = True
    return z


@pytest.mark.parametrize("dims,leaf", [((3, 3, 8), 16), ((4, 4, 12), 16), ((6, 6, 28), 64)])
def test_panel_dag_emulation_matches_oracle(params, dims, leaf):
    mesh = clamped_beam(*dims)
    from oracle import tetsim_oracle as O2  # noqa: F401

    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    out = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, mesh.nodes,
                            np.zeros_like(mesh.nodes), np.zeros(mesh.ndof), 0.01, (0.0, -9.81, 0.0))
    a = CsrMatrix(mesh.ndof, mesh.ndof, out["row_ptr"], out["col_ind"], out["values"])
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), leaf))
    f = ND.ldlt_factor(a, plan)
    H = K.pack(f)
    r = np.random.default_rng(7).standard_normal(mesh.ndof)
    y = emulate_lower(H, r)
    ref = O.solve_lower(f, r)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    z = emulate_upper(H, r)
    ref = O.solve_upper(f, r)
    assert np.abs(z - ref).max() <= 1e-12 * np.abs(ref).max()
    # item lists cover every panel exactly once per sweep
    assert sorted(H["items_l"][H["items_l"][:, 0] == K.IT_DIAG, 1]) == list(range(H["P"]))
    assert sorted(H["items_u"][H["items_u"][:, 0] == K.IT_DIAGT, 1]) == list(range(H["P"]))
