"""Device refactorisation planner (refactor.py) checked on CPU: the NumPy
emulator of the launch program (tests/refactor_emulator.py) must reproduce
the host multifrontal factorisation (ndprecond.ldlt_factor, the restatement
of ndprecond.py:501-572) packed into the sweep layout."""

import numpy as np
import pytest

import refactor_emulator as EM
from oracle import tetsim_oracle as O
from paper_2306_05893_b200 import _ldlt_pack as K, ndprecond as ND, refactor as R
from test_ldlt_pack import _factors


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("dims,leaf", [((3, 3, 8), 16), ((4, 4, 12), 16), ((6, 6, 28), 64)])
def test_program_emulation_matches_host_factor(dims, leaf):
    mesh, f = _factors(dims, leaf)
    a = f._a
    rp = R.plan_refactor(f.symbolic, f.plan)
    H = K.pack(f)
    Hs = K.pack(R._StructFactors(f.plan, rp.blocks))
    # the structure-only image has the same tiles as the host-packed factor
    assert np.array_equal(H["tiles_l"], Hs["tiles_l"]) and np.array_equal(H["tiles_u"], Hs["tiles_u"])
    assert np.array_equal(H["items_l"], Hs["items_l"]) and not Hs["g"].any()
    assert len(rp.fronts) == H["nb"] and rp.heights.max() >= 2
    g, gt, d, bad = EM.run(rp, a.values, H["tiles_l"], H["tiles_u"], H["tile_blk_l"], H["tile_blk_u"], f.plan.n)
    assert bad == -1
    assert rel(d, f.d) <= 1e-12
    assert rel(g, H["g"]) <= 1e-12 and rel(gt, H["gt"]) <= 1e-12
    # exact zeros of the layout stay zero
    assert np.array_equal(g == 0.0, H["g"] == 0.0) or np.abs(g[H["g"] == 0.0]).max() <= 1e-13


def test_program_flags_indefinite_front():
    mesh, f = _factors((3, 3, 8), 16)
    a = f._a
    rp = R.plan_refactor(f.symbolic, f.plan)
    H = K.pack(f)
    vals = a.values.copy()
    vals[a.row_ptr[5]:a.row_ptr[6]] *= -1.0  # a negative diagonal entry
    _, _, _, bad = EM.run(rp, vals, H["tiles_l"], H["tiles_u"], H["tile_blk_l"], H["tile_blk_u"], f.plan.n)
    assert bad >= 0
