"""Sharded index with real torch.distributed ranks: two processes, one shard
each, a gloo process group with host staging of the records (both ranks share the one GPU of
this box; across GPUs the same TorchExchange moves device buffers over NCCL).  Exercises the
protocol driver, the C-ABI shard contexts and the exchange end to end; results and the union of
both shards' indexes must equal the sequential oracle's."""
import os
import socket

import numpy as np
import pytest

from oracle import Oracle
from workloads import c1_tiny, c2_shared_prompt

pytestmark = pytest.mark.gpu
SEED = 0x5011D000


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, outdir, nc=1):
    import torch
    import torch.distributed as dist
    import paper_2603_10726_b200 as P
    from paper_2603_10726_b200.dist import ShardedIndex, TorchExchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    s = c1_tiny() if name == "c1" else c2_shared_prompt(users=30, reqs_per_user=10)
    n = s.n_requests
    lo, hi = n * rank // world, n * (rank + 1) // world
    part = s.slice(lo, hi)
    shard = ShardedIndex(world, rank, "solidarity", capacity_blocks=max(4 * s.n_blocks(), 4096),
                         max_batch_tokens=s.n_tokens + 64, max_batch_requests=n, seed=SEED,
                         hash_components=nc)
    ex = TorchExchange(shard, staging=True)
    d = P.to_device(part)
    res, rounds = ex.admit(d["tokens"], d["offsets"], d["users"], d["enforce"], seq_base=lo)
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, f"res{rank}.npy"), P.as_numpy(res))
    np.save(os.path.join(outdir, f"dump{rank}.npy"), shard.index.dump())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,nc", [("c1", 1), ("c2_small", 1), ("c2_small", 2)])
def test_two_ranks_gloo_staging(name, nc, tmp_path):
    """nc = 2: H-def v3 two-component keys across real ranks."""
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path), nc), nprocs=world,
             join=True)
    s = c1_tiny() if name == "c1" else c2_shared_prompt(users=30, reqs_per_user=10)
    o = Oracle(16, SEED, 2, components=nc)
    exp = o.process(s)
    got = np.concatenate([np.load(tmp_path / f"res{r}.npy") for r in range(world)])
    assert np.array_equal(got, exp)
    dumps = np.concatenate([np.load(tmp_path / f"dump{r}.npy") for r in range(world)])
    dumps = dumps[np.argsort(dumps["key"])]
    ed = o.dump()
    assert all(np.array_equal(dumps[f], ed[f]) for f in ["key", "owner", "sharer"])
