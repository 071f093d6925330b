import os, sys, socket
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import torch, torch.distributed as dist, torch.multiprocessing as mp

def worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), TSB_SHARED_DEVICE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from test_shard import _system
    from paper_2306_05893_b200 import shard as S
    a, b, f = _system()
    ds = S.DistributedPcg(a, f, rank=rank, world=world, grid=32)
    for nm in ("S", "T"):
        h = getattr(ds, nm)
        if h is not None:
            d = h.desc
            print(rank, nm, "grid", d.grid, "blocks", d.n_blocks, "items", d.n_items_lower, d.n_items_upper, "max_v", d.max_v, "max_cb", d.max_cb, flush=True)
    try:
        x, it, res, conv = ds.solve(b, 1e-9, 200)
        print(rank, "ok", it, conv, flush=True)
    except Exception as e:
        print(rank, "ERR", e, flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.spawn(worker, args=(2, port), nprocs=2)
