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


def _p2p_worker(rank, world, port, name, outdir, nc, dc=False):
    import torch
    import torch.distributed as dist
    import paper_2603_10726_b200 as P
    from paper_2603_10726_b200.dist import PeerExchange, ShardedIndex
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    s = c1_tiny() if name == "c1" else c2_shared_prompt(users=30, reqs_per_user=10)
    n = s.n_requests
    shard = ShardedIndex(world, rank, "solidarity", capacity_blocks=max(4 * s.n_blocks(), 4096),
                         max_batch_tokens=s.n_tokens + 64, max_batch_requests=n, seed=SEED,
                         hash_components=nc)
    ex = PeerExchange(shard, device_counts=dc)
    # two batches: the second finds the first's entries on their owners
    for k, (a, b) in enumerate([(0, n // 2), (n // 2, n)]):
        lo = a + (b - a) * rank // world
        hi = a + (b - a) * (rank + 1) // world
        d = P.to_device(s.slice(lo, hi))
        res, rounds = ex.admit(d["tokens"], d["offsets"], d["users"], d["enforce"], seq_base=lo)
        torch.cuda.synchronize()
        np.save(os.path.join(outdir, f"res{k}_{rank}.npy"), P.as_numpy(res))
    np.save(os.path.join(outdir, f"dump{rank}.npy"), shard.index.dump())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,nc,world,dc", [("c1", 1, 2, False), ("c2_small", 1, 2, False),
                                              ("c2_small", 2, 3, False), ("c1", 1, 2, True),
                                              ("c2_small", 1, 3, True)])
def test_ranks_peer_memory_exchange(name, nc, world, dc, tmp_path):
    """The library's own exchange over CUDA IPC peer memory (solid_dist_p2p_*):
    2-3 processes (sharing this box's GPU: IPC-mapped buffers of one device), two batches;
    dc: device-resident counts (one host wait per round)."""
    import torch.multiprocessing as mp
    mp.spawn(_p2p_worker, args=(world, _free_port(), name, str(tmp_path), nc, dc), nprocs=world,
             join=True)
    s = c1_tiny() if name == "c1" else c2_shared_prompt(users=30, reqs_per_user=10)
    n = s.n_requests
    o = Oracle(16, SEED, 2, components=nc)
    for k, (a, b) in enumerate([(0, n // 2), (n // 2, n)]):
        exp = o.process(s.slice(a, b))
        got = np.concatenate([np.load(tmp_path / f"res{k}_{r}.npy") for r in range(world)])
        assert np.array_equal(got, exp), k
    dumps = np.concatenate([np.load(tmp_path / f"dump{r}.npy") for r in range(world)])
    dumps = dumps[np.argsort(dumps["key"])]
    ed = o.dump()
    assert all(np.array_equal(dumps[f], ed[f]) for f in ["key", "owner", "sharer"])


def _fuzz_cases(world):
    from workloads import random_small
    rng = np.random.default_rng(4242 + world)
    cases = []
    for case in range(8):
        policy = ["apc", "user_isolation", "solidarity"][int(rng.integers(3))]
        s = random_small(int(rng.integers(20, 160)), users=int(rng.integers(1, 6)),
                         alphabet_blocks=int(rng.integers(2, 6)), max_blocks=int(rng.integers(1, 9)),
                         seed=2000 + case, enforce_prob=float(rng.choice([1.0, 0.6])))
        k = int(rng.integers(1, 4))
        cuts = sorted(set([0, s.n_requests] + [int(x) for x in rng.integers(0, s.n_requests, k - 1)]))
        cases.append((policy, s, [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a],
                      bool(rng.integers(2))))
    return cases


def _fuzz_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    import paper_2603_10726_b200 as P
    from paper_2603_10726_b200.dist import PeerExchange, ShardedIndex
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    for c, (policy, s, batches, dc) in enumerate(_fuzz_cases(world)):
        shard = ShardedIndex(world, rank, policy, capacity_blocks=4096,
                             max_batch_tokens=s.n_tokens + 64, max_batch_requests=s.n_requests,
                             seed=SEED)
        ex = PeerExchange(shard, device_counts=dc)
        for k, (a, b) in enumerate(batches):
            lo, hi = a + (b - a) * rank // world, a + (b - a) * (rank + 1) // world
            d = P.to_device(s.slice(lo, hi))
            res, _ = ex.admit(d["tokens"], d["offsets"], d["users"], d["enforce"], seq_base=lo)
            torch.cuda.synchronize()
            np.save(os.path.join(outdir, f"f{c}_b{k}_res{rank}.npy"), P.as_numpy(res))
        np.save(os.path.join(outdir, f"f{c}_dump{rank}.npy"), shard.index.dump())
        dist.barrier()
        shard.index.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fuzz_peer_memory_exchange(world, tmp_path):
    """Seeded random cases through the peer-memory exchange in real processes (host- and
    device-counts modes, random policy, 1-3 global batches): every result and the union of the
    shards bit-exact against the oracle."""
    import torch.multiprocessing as mp
    mp.spawn(_fuzz_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for c, (policy, s, batches, dc) in enumerate(_fuzz_cases(world)):
        o = Oracle(16, SEED, ["apc", "user_isolation", "solidarity"].index(policy))
        for k, (a, b) in enumerate(batches):
            exp = o.process(s.slice(a, b))
            got = np.concatenate([np.load(tmp_path / f"f{c}_b{k}_res{r}.npy")
                                  for r in range(world)])
            assert got.dtype == exp.dtype and len(got) == len(exp)
            assert np.array_equal(got, exp), (c, policy, dc, k)
        dumps = np.concatenate([np.load(tmp_path / f"f{c}_dump{r}.npy") for r in range(world)])
        dumps = dumps[np.argsort(dumps["key"])]
        ed = o.dump()
        assert len(dumps) == len(ed), (c, policy, dc)
        assert all(np.array_equal(dumps[f], ed[f]) for f in ["key", "owner", "sharer"]), (c, dc)
