"""Sharded assembly (SURVEY.md 8e "Assembly"), host logic on CPU.

Each rank assembles only the elements of its subtree (rank 0 also the
elements inside the top separators) with its share of the external forces.
Owned rows come out complete and bit-identical to the full assembly; top rows
are partial sums that add up to the full rows (within 1e-12: a different
summation split); the distributed PCG over the local systems (2 and 4 gloo
processes) converges in the same iterations as the single-process oracle PCG
on the full system (krylov.py:120-158), x within 1e-10."""

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

DT, G = 0.01, (0.0, -9.81, 0.0)


def _case(dims=(4, 4, 16), leaf=16):
    mesh = clamped_beam(*dims)
    n = mesh.ndof
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    out0 = O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, mesh.nodes,
                             np.zeros_like(mesh.nodes), np.zeros(n), DT, G)
    a0 = CsrMatrix(n, n, out0["row_ptr"], out0["col_ind"], out0["values"])
    plan = ND.expand_plan(ND.nested_dissection(M.vertex_adjacency(mesh), leaf))
    f = ND.ldlt_factor(a0, plan)
    rng = np.random.default_rng(11)
    x = mesh.nodes + 2e-3 * rng.standard_normal(mesh.nodes.shape)
    x[mesh.fixed_nodes] = mesh.nodes[mesh.fixed_nodes]
    v = 1e-2 * rng.standard_normal(mesh.nodes.shape)
    v[mesh.fixed_nodes] = 0.0
    fe = 0.5 * rng.standard_normal(n)
    return mesh, f, x, v, fe


def _full(mesh, x, v, fe):
    rest = O.rest_data(mesh.nodes, mesh.elements, 1e5, 0.3, 1000.0)
    return O.assemble_system(mesh.nodes, mesh.elements, mesh.fixed_nodes, rest, x, v, fe, DT, G)


def _rank_local(mesh, f, x, v, fe, sp, rank):
    nr = S.node_ranks(sp, f.plan.perm)
    er = S.element_ranks(mesh.elements, nr)
    sub = np.asarray(mesh.elements)[er == rank]
    rest = O.rest_data(mesh.nodes, sub, 1e5, 0.3, 1000.0)
    out = O.assemble_system(mesh.nodes, sub, mesh.fixed_nodes, rest, x, v, S.rank_f_ext(fe, nr, rank), DT, G)
    fixed = (3 * np.asarray(mesh.fixed_nodes)[:, None] + np.arange(3)).ravel()
    return S.local_system(out["row_ptr"], out["col_ind"], out["values"], out["b"], sp, f.plan.perm, rank, fixed)


def _dense(rp, ci, va, n):
    d = np.zeros((n, n))
    np.add.at(d, (np.repeat(np.arange(n), np.diff(rp)), ci), va)
    return d


@pytest.mark.parametrize("world", [1, 2, 4])
def test_local_systems_add_up_to_the_full_system(world):
    mesh, f, x, v, fe = _case()
    n = mesh.ndof
    sp = S.shard_blocks(f, world)
    er = S.element_ranks(mesh.elements, S.node_ranks(sp, f.plan.perm))
    assert set(np.unique(er)) <= set(range(world))
    full = _full(mesh, x, v, fe)
    perm = np.asarray(f.plan.perm)
    rp, ci, va = S.permuted_matrix(CsrMatrix(n, n, full["row_ptr"], full["col_ind"], full["values"]), perm)
    ref, bref = _dense(rp, ci, va, n), full["b"][perm]
    tot, btot = np.zeros((n, n)), np.zeros(n)
    for g in range(world):
        lrp, lci, lva, lb = _rank_local(mesh, f, x, v, fe, sp, g)
        d = _dense(lrp, lci, lva, n)
        own = sp.row_owner == g
        # owned rows: complete and bit-identical (same elements, same ascending order)
        assert np.array_equal(d[own], ref[own])
        assert np.array_equal(lb[own], bref[own])
        tot += d
        btot += np.where(sp.row_owner < 0, lb, 0.0) + np.where(own, lb, 0.0)
    scale = np.abs(ref).max()
    assert np.abs(tot - ref).max() <= 1e-12 * scale
    assert np.abs(btot - bref).max() <= 1e-12 * np.abs(bref).max()
    top = sp.row_owner < 0
    if world > 1:
        assert top.any()


def test_element_spanning_two_subtrees_is_rejected():
    mesh, f, *_ = _case()
    sp = S.shard_blocks(f, 2)
    nr = S.node_ranks(sp, f.plan.perm)
    a0 = np.flatnonzero(nr == 0)[0]
    a1 = np.flatnonzero(nr == 1)[0]
    bad = np.array([[a0, a1, a0, a1]])
    with pytest.raises(ValueError):
        S.element_ranks(bad, nr)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh, f, x, v, fe = _case()
        sp = S.shard_blocks(f, world)
        local = _rank_local(mesh, f, x, v, fe, sp, rank)

        def allreduce(arr):
            t = torch.from_numpy(arr)
            dist.all_reduce(t)
            arr[...] = t.numpy()

        xs, it, res, conv = S.emulate_pcg(None, None, f, sp, rank, allreduce, tol=1e-9, max_it=200, local=local)
        q.put((rank, xs, it, res, conv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_pcg_over_sharded_assembly(world):
    mesh, f, x, v, fe = _case()
    full = _full(mesh, x, v, fe)
    ox, oit, ores, oconv = O.pcg(full["row_ptr"], full["col_ind"], full["values"], full["b"],
                                 lambda r: O.apply(f, r), 1e-9, 200)
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
    for rank, xs, it, res, conv in outs:
        assert conv and it == oit, (rank, it, oit)
        assert np.abs(xs - ox).max() <= 1e-10 * np.abs(ox).max()


@pytest.mark.parametrize("world", [2, 4])
def test_rank_meshes_partition_the_elements(world):
    mesh, f, _, _, fe = _case()
    sp = S.shard_blocks(f, world)
    parts = [S.rank_mesh(mesh, sp, f.plan.perm, g) for g in range(world)]
    rows = np.concatenate([p.elements for p, _ in parts])
    assert len(rows) == len(mesh.elements)
    assert len(np.unique(rows, axis=0)) == len(np.unique(np.asarray(mesh.elements), axis=0))
    # every rank keeps the full node set and the pinned nodes
    for p, _ in parts:
        assert p.node_count == mesh.node_count
        assert np.array_equal(p.fixed_nodes, mesh.fixed_nodes)
    # the external forces are handed out exactly once
    nr = parts[0][1]
    tot = sum(S.rank_f_ext(fe, nr, g) for g in range(world))
    assert np.array_equal(tot, fe)


def test_local_system_index_map_equals_value_extraction():
    """shard.LocalSystem plans local_system once on index arrays and gathers
    values per step: the gathered values equal local_system on the values."""
    mesh, f, x, v, fe = _case()
    full = _full(mesh, x, v, fe)
    sp = S.shard_blocks(f, 2)
    perm = f.plan.perm
    fixed = (3 * np.asarray(mesh.fixed_nodes)[:, None] + np.arange(3)).ravel()
    rp, ci, va, b = full["row_ptr"], full["col_ind"], full["values"], full["b"]
    for rank in range(2):
        lrp, lci, lva, lb = S.local_system(rp, ci, va, b, sp, perm, rank, fixed)
        irp, ici, src, _ = S.local_system(rp, ci, np.arange(len(ci), dtype=np.float64), b, sp, perm, rank, fixed)
        assert np.array_equal(lrp, irp) and np.array_equal(lci, ici)
        assert np.array_equal(va[src.astype(np.int64)], lva)
        ro = sp.row_owner
        assert np.array_equal(np.where((ro == rank) | (ro < 0), np.asarray(b)[perm], 0.0), lb)
