import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtsb.so")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            with np.load(GOLDEN / f"{name}.npz") as z:
                cache[name] = {k: z[k] for k in z.files}
        return cache[name]

    return load


@pytest.fixture
def params():
    from paper_2306_05893_b200 import MaterialParams

    return MaterialParams(young_modulus=1e5, poisson_ratio=0.3, density=1000.0)


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def clamped_beam(nx, ny, nz, spacing=0.1):
    from paper_2306_05893_b200 import generate_beam

    mesh = generate_beam(nx, ny, nz, spacing)
    return mesh.with_fixed_nodes(np.flatnonzero(mesh.nodes[:, 2] == 0.0))


class GoldenFactors:
    """Duck-typed LdlFactors rebuilt from a golden fixture (reference factors)."""

    class _B:
        def __init__(self, **kw):
            self.__dict__.update(kw)

    def __init__(self, g):
        start, stop, level = g["f_start"], g["f_stop"], g["f_level"]
        tile = int(g["f_tile"])
        aptr = g["f_anc_ptr"]
        o11 = o21 = otv = 0
        self.blocks = []
        for i in range(len(start)):
            m = int(stop[i] - start[i])
            anc = g["f_anc"][aptr[i]:aptr[i + 1]]
            l11 = g["f_l11"][o11:o11 + m * m].reshape(m, m)
            o11 += m * m
            # the reference's l21 is a transposed solve result (Fortran order), which
            # selects a different BLAS gemv path; keep that layout for bitwise replay
            l21 = np.asfortranarray(g["f_l21"][o21:o21 + len(anc) * m].reshape(len(anc), m))
            o21 += len(anc) * m
            inv = []
            for t0 in range(0, m, tile):
                w = min(tile, m - t0)
                inv.append(g["f_tinv"][otv:otv + w * w].reshape(w, w))
                otv += w * w
            self.blocks.append(self._B(start=int(start[i]), stop=int(stop[i]), level=int(level[i]),
                                       anc=anc, l11=l11, l21=l21, tile=tile, tile_inv=inv))
        nlev = int(level.max()) + 1
        self.levels = [[b for b in self.blocks if b.level == lv] for lv in range(nlev)]
        self.d = g["f_d"]
        self.plan = self._B(perm=g["f_perm"], iperm=g["f_iperm"], n=len(g["f_perm"]))
