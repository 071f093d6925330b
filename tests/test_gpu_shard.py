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


def test_single_rank_equals_device_pcg():
    from oracle import tetsim_oracle as O
    from paper_2306_05893_b200 import krylov, shard as S

    a, b, f = _system()
    x, it, res, conv = S.DistributedPcg(a, f, rank=0, world=1).solve(b, 1e-9, 200)
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
