"""Sharded (multi-GPU) PCG through the device kernels (shard.DistributedPcg).

Only one GPU is available to the test suite, so the 2-rank run places both
ranks on cuda:0 with the gloo backend over CUDA tensors: the kernels, the
block-subset sweeps and the exchange pattern are exactly the NCCL path's;
only the transport differs.  Results must match the single-GPU PCG and the
CPU oracle on the same factors (same iterations, x within 1e-10)."""

import os
import socket

import numpy as np
import pytest

from test_shard import _system

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("graph", [True, False])
def test_single_rank_equals_device_pcg(graph):
    """One rank, device-resident loop replayed as CUDA graphs (device stop
    flag, no host read per iteration) or eagerly: same as the single-GPU PCG."""
    from oracle import tetsim_oracle as O
    from paper_2306_05893_b200 import krylov, shard as S

    a, b, f = _system()
    dp = S.DistributedPcg(a, f, rank=0, world=1)
    x, it, res, conv = dp.solve(b, 1e-9, 200, graph=graph)
    x2, it2, res2, _ = dp.solve(b, 1e-9, 200, graph=graph)  # replays the captured graph
    assert it2 == it and np.array_equal(x.cpu().numpy(), x2.cpu().numpy())
    ox, oit, ores, oconv = O.pcg(a.row_ptr, a.col_ind, a.values, b, lambda r: O.apply(f, r), 1e-9, 200)
    assert conv and it == oit
    assert np.abs(x.cpu().numpy() - ox).max() <= 1e-10 * np.abs(ox).max()
    xd, rep = krylov.pcg(a, b, f, krylov.SolverConfig(1e-9, 200))
    assert rep.iterations == it


def _worker(rank, world, port, q, exchange="nccl"):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), TSB_SHARED_DEVICE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_05893_b200 import shard as S

        a, b, f = _system()
        # both ranks share the one GPU: small persistent grids so the two processes'
        # cooperative sweep launches fit on the device side by side
        x, it, res, conv = S.DistributedPcg(a, f, rank=rank, world=world, grid=32,
                                            exchange=exchange).solve(b, 1e-9, 200)
        q.put((rank, x.cpu().numpy(), it, res, conv))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e), -1, 0.0, False))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["nccl", "peer"])
def test_two_ranks_match_the_oracle(exchange):
    """exchange="nccl": the process group's all-reduce (gloo here); "peer": the
    IPC-mapped peer-memory all-reduce kernel (csrc/peer.cu)."""
    import torch.multiprocessing as mp
    from oracle import tetsim_oracle as O

    a, b, f = _system()
    ox, oit, _, _ = O.pcg(a.row_ptr, a.col_ind, a.values, b, lambda r: O.apply(f, r), 1e-9, 200)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, exchange)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, x, it, res, conv in outs:
        assert conv and it == oit, (rank, x if isinstance(x, str) else it, oit)
        assert np.abs(x - ox).max() <= 1e-10 * np.abs(ox).max()


def _worker_sharded(rank, world, port, q, exchange):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), TSB_SHARED_DEVICE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2306_05893_b200 as P
        from paper_2306_05893_b200 import shard as S
        from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState
        from test_shard_assembly import DT, G, _case

        mesh, f, x, v, fe = _case()
        sp = S.shard_blocks(f, world)
        perm = f.plan.perm
        sub, nr = S.rank_mesh(mesh, sp, perm, rank)
        integ = BackwardEulerIntegrator(sub, P.make_model("corotational", sub, P.MaterialParams(1e5, 0.3, 1000.0)),
                                        IntegratorConfig(dt=DT, gravity=G))
        n = mesh.ndof
        st = SimState(x.copy(), v.copy(), np.zeros_like(x), np.zeros(n), S.rank_f_ext(fe, nr, rank))
        a, b, _ = integ.assemble_system(st)
        host = lambda z: z.cpu().numpy() if hasattr(z, "cpu") else np.asarray(z)  # noqa: E731
        fixed = (3 * np.asarray(mesh.fixed_nodes)[:, None] + np.arange(3)).ravel()
        if exchange == "peer":  # device-side extraction (planned once, two gathers per step)
            ls = S.LocalSystem(host(a.row_ptr), host(a.col_ind), sp, perm, rank, fixed)
            bd = b if hasattr(b, "cuda") else torch.from_numpy(np.asarray(b)).cuda()
            local = ls.system(a.device_values(), bd)
        else:
            local = S.local_system(host(a.row_ptr), host(a.col_ind), host(a.values), host(b), sp, perm, rank, fixed)
        xs, it, res, conv = S.DistributedPcg(None, f, rank=rank, world=world, grid=32, exchange=exchange,
                                             local=local).solve(None, 1e-9, 200)
        q.put((rank, xs.cpu().numpy(), it, res, conv))
    except Exception as e:  # surface the failure in the parent
        import traceback

        q.put((rank, repr(e) + traceback.format_exc(), -1, 0.0, False))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["nccl", "peer"])
def test_two_ranks_sharded_device_assembly(exchange):
    """Each rank assembles only its subtree's elements on the device
    (shard.rank_mesh / local_system; with the peer exchange the local system
    is extracted on the device by LocalSystem and the iterations replay as
    CUDA graphs with the device stop flag); the distributed PCG over the
    partial systems matches the oracle PCG on the full assembly."""
    import torch.multiprocessing as mp
    from oracle import tetsim_oracle as O
    from test_shard_assembly import _case, _full

    mesh, f, x, v, fe = _case()
    full = _full(mesh, x, v, fe)
    ox, oit, _, _ = O.pcg(full["row_ptr"], full["col_ind"], full["values"], full["b"],
                          lambda r: O.apply(f, r), 1e-9, 200)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sharded, args=(r, 2, port, q, exchange)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, xs, it, res, conv in outs:
        assert conv and it == oit, (rank, xs if isinstance(xs, str) else it, oit)
        assert np.abs(xs - ox).max() <= 1e-10 * np.abs(ox).max()
