"""Multi-GPU sharding of the solve, host logic on CPU.

The dissection cut, the rank-local matrices and the exchange pattern are
checked directly; the distributed PCG loop is run in 2 (and 4) processes over
gloo with NumPy kernels (shard.emulate_pcg mirrors the device loop step by
step) and must reproduce the single-process oracle PCG on the same factors
(ndprecond.py:694-700, krylov.py:120-158): same iteration count, x within
1e-10."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import clamped_beam
from oracle import tetsim_oracle as O
from paper_2306_05893_b200 import mesh as M, ndprecond as ND, shard as S
from paper_2306_05893_b200.assembly import CsrMatrix


def _system(dims=(4, 4, 16), leaf=16):
    mesh = clamped_beam(*dims)
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    n = mesh.ndof
    out0 = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, mesh.nodes, np.zeros_like(mesh.nodes),
                             np.zeros(n), 0.01, (0.0, -9.81, 0.0))
    a0 = CsrMatrix(n, n, out0["row_ptr"], out0["col_ind"], out0["values"])
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), leaf))
    f = ND.ldlt_factor(a0, plan)
    rng = np.random.default_rng(3)
    x = mesh.nodes + 2e-3 * rng.standard_normal(mesh.nodes.shape)
    x[mesh.fixed_nodes] = mesh.nodes[mesh.fixed_nodes]
    v = 1e-2 * rng.standard_normal(mesh.nodes.shape)
    v[mesh.fixed_nodes] = 0.0
    out = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, x, v, np.zeros(n), 0.01,
                            (0.0, -9.81, 0.0))
    a = CsrMatrix(n, n, out["row_ptr"], out["col_ind"], out["values"])
    return a, out["b"], f


def test_cut_is_a_dissection_cut():
    a, _, f = _system()
    for nr in (1, 2, 4):
        sp = S.shard_blocks(f, nr)
        assert set(np.unique(sp.owner[sp.owner >= 0])) == set(range(nr))
        rp, ci, va = S.permuted_matrix(a, f.plan.perm)
        for g in range(nr):
            S.local_matrix(rp, ci, va, sp, g)  # raises if an owned row couples to another rank
        # top blocks are exactly the ancestors of the cut: every block's ancestors of
        # a top block are top blocks
        parent, _ = S.block_etree(f)
        for i in range(len(sp.owner)):
            if sp.owner[i] < 0 and parent[i] >= 0:
                assert sp.owner[parent[i]] < 0
        # the rank-local matrices add up to the permuted matrix
        n = a.nrows
        dense = np.zeros((n, n))
        for g in range(nr):
            lrp, lci, lva = S.local_matrix(rp, ci, va, sp, g)
            rows = np.repeat(np.arange(n), np.diff(lrp))
            np.add.at(dense, (rows, lci), lva)
        ref = np.zeros((n, n))
        ref[np.repeat(np.arange(n), np.diff(rp)), ci] = va
        assert np.array_equal(dense, ref)


def test_load_balance_on_the_beam():
    _, _, f = _system((6, 6, 40), 32)
    sp = S.shard_blocks(f, 4)
    assert sp.load.max() / sp.load.min() < 2.0
    assert len(sp.top_rows) < 0.25 * f.plan.n


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b, f = _system()
        sp = S.shard_blocks(f, world)

        def allreduce(arr):
            t = torch.from_numpy(arr)
            dist.all_reduce(t)

        x, it, res, conv = S.emulate_pcg(a, b, f, sp, rank, allreduce, tol=1e-9, max_it=200)
        q.put((rank, x, it, res, conv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_pcg_matches_single_process(world):
    a, b, f = _system()
    ox, oit, ores, oconv = O.pcg(a.row_ptr, a.col_ind, a.values, b, lambda r: O.apply(f, r), 1e-9, 200)
    assert oconv and oit >= 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, x, it, res, conv in outs:
        assert conv and it == oit, (rank, it, oit)
        assert np.abs(x - ox).max() <= 1e-10 * np.abs(ox).max()
        assert abs(res - ores) <= 1e-6 * ores
