"""The sharded admission as ONE C-ABI call (solid_dist_admit, include/solid.h; SURVEY §8(b),
§8(e)): real processes (sharing this box's GPU through CUDA IPC peer memory), each calling the
library once per batch with its slice.  The library runs the agreement on the slices, the
resolver rounds, the commit and the overflow vote itself; Python only all-gathers the 64-byte
IPC handles once.  Results and the union of the shards must equal the sequential oracle's; the
collective failure paths (non-contiguous slices, an invalid slice on one rank, one shard over
capacity) must fail on every rank alike without hanging and leave every shard as it was."""
import os
import socket

import numpy as np
import pytest

from oracle import Oracle
from workloads import c1_tiny, c2_shared_prompt

pytestmark = pytest.mark.gpu
SEED = 0x5011D000
POLICIES = ["apc", "user_isolation", "solidarity"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stream(name):
    if name == "c1":
        return c1_tiny()
    if name == "c2_small":
        return c2_shared_prompt(users=30, reqs_per_user=10)
    from workloads import random_small
    return random_small(150, users=4, alphabet_blocks=4, max_blocks=8, seed=77, enforce_prob=0.7)


def _setup(rank, world, port):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)


def _parity_worker(rank, world, port, name, policy, outdir):
    import torch
    import torch.distributed as dist
    import paper_2603_10726_b200 as P
    from paper_2603_10726_b200.dist import PeerExchange, ShardedIndex
    _setup(rank, world, port)
    s = _stream(name)
    n = s.n_requests
    shard = ShardedIndex(world, rank, policy, capacity_blocks=max(4 * s.n_blocks(), 4096),
                         max_batch_tokens=s.n_tokens + 64, max_batch_requests=n, seed=SEED)
    ex = PeerExchange(shard)
    cuts = [0, n // 3, n]
    for k, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
        lo, hi = a + (b - a) * rank // world, a + (b - a) * (rank + 1) // world
        d = P.to_device(s.slice(lo, hi))
        res, tm = ex.admit_native(d["tokens"], d["offsets"], d["users"], d["enforce"], seq_base=lo)
        torch.cuda.synchronize()
        np.save(os.path.join(outdir, f"res{k}_{rank}.npy"), P.as_numpy(res))
        np.save(os.path.join(outdir, f"tm{k}_{rank}.npy"),
                np.array([tm.rounds, tm.exchanges, tm.record_bytes, tm.recv_records_remote,
                          tm.recv_records_local], dtype=np.int64))
    np.save(os.path.join(outdir, f"dump{rank}.npy"), shard.index.dump())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,policy,world", [("c1", "solidarity", 2),
                                               ("c2_small", "solidarity", 3),
                                               ("c2_small", "solidarity", 4),
                                               ("random", "solidarity", 2),
                                               ("random", "apc", 3),
                                               ("random", "user_isolation", 2)])
def test_native_admit_parity(name, policy, world, tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_parity_worker, args=(world, _free_port(), name, policy, str(tmp_path)),
             nprocs=world, join=True)
    s = _stream(name)
    n = s.n_requests
    o = Oracle(16, SEED, POLICIES.index(policy))
    cuts = [0, n // 3, n]
    for k, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
        exp = o.process(s.slice(a, b))
        got = np.concatenate([np.load(tmp_path / f"res{k}_{r}.npy") for r in range(world)])
        assert np.array_equal(got, exp), k
        tms = [np.load(tmp_path / f"tm{k}_{r}.npy") for r in range(world)]
        assert len({int(t[0]) for t in tms}) == 1          # every rank ran the same rounds
        rounds, exchanges, rb = int(tms[0][0]), int(tms[0][1]), int(tms[0][2])
        assert rb == 24
        # REG + PULL + per round (INT + PULL) - the last PULL
        assert exchanges == 2 + 2 * rounds - 1
        if policy != "solidarity":
            assert rounds == 1
        assert sum(int(t[3]) for t in tms) > 0              # records crossed ranks
    dumps = np.concatenate([np.load(tmp_path / f"dump{r}.npy") for r in range(world)])
    dumps = dumps[np.argsort(dumps["key"])]
    ed = o.dump()
    assert all(np.array_equal(dumps[f], ed[f]) for f in ["key", "owner", "sharer"])


def _failure_worker(rank, world, port, case, outdir):
    import torch
    import torch.distributed as dist
    import paper_2603_10726_b200 as P
    from paper_2603_10726_b200.dist import PeerExchange, ShardedIndex
    _setup(rank, world, port)
    s = c2_shared_prompt(users=30, reqs_per_user=10)
    n = s.n_requests
    cap = max(4 * s.n_blocks(), 4096)
    if case == "capacity":
        # each shard holds about half the keys: the first batch's whole key count fits every
        # shard, the remaining 260 requests overflow at least one
        o = Oracle(16, SEED, 2)
        o.process(s.slice(0, 40))
        cap = len(o.dump())
    shard = ShardedIndex(world, rank, "solidarity", capacity_blocks=cap,
                         max_batch_tokens=s.n_tokens + 64, max_batch_requests=n, seed=SEED)
    ex = PeerExchange(shard)
    statuses = []

    def run(a, b, seq_shift=0, poison=False):
        lo, hi = a + (b - a) * rank // world, a + (b - a) * (rank + 1) // world
        part = s.slice(lo, hi)
        if poison:
            part.tokens = part.tokens.copy()
            part.tokens[:16] = 1 << 20                       # invalid token id on this rank only
        d = P.to_device(part)
        try:
            res, tm = ex.admit_native(d["tokens"], d["offsets"], d["users"], d["enforce"],
                                      seq_base=lo + seq_shift)
            torch.cuda.synchronize()
            statuses.append(0)
            return P.as_numpy(res)
        except P.SolidError as e:
            statuses.append(e.status)
            return None

    half = n // 2
    first = run(0, 40)                                        # a committed batch
    dump0 = shard.index.dump()
    if case == "contiguity":
        run(40, half, seq_shift=1 if rank == world - 1 else 0)
    elif case == "invalid":
        run(40, half, poison=(rank == 1))
    else:
        run(40, n)                                            # too many new entries
    dump1 = shard.index.dump()
    unchanged = len(dump0) == len(dump1) and all(
        np.array_equal(dump0[f], dump1[f]) for f in ["key", "owner", "sharer"])
    again = run(40, half)                                     # a valid batch afterwards works
    np.save(os.path.join(outdir, f"st{rank}.npy"), np.array(statuses + [int(unchanged)]))
    np.save(os.path.join(outdir, f"first{rank}.npy"), first)
    if again is not None:
        np.save(os.path.join(outdir, f"again{rank}.npy"), again)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["contiguity", "invalid", "capacity"])
def test_native_admit_collective_failures(case, tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_failure_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world,
             join=True)
    st = [np.load(tmp_path / f"st{r}.npy") for r in range(world)]
    for r in range(world):
        assert st[r][0] == 0, "first batch"
        assert st[r][1] != 0, ("the bad batch must fail on every rank", r)
        assert st[r][3] == 1, ("index unchanged by the failed batch", r)
    codes = sorted(int(x[1]) for x in st)
    if case == "contiguity":
        assert codes == [1, 1]                                # INVALID on every rank
    elif case == "invalid":
        assert codes == [1, 3]                                # INVALID here, STATE on the peer
    else:
        assert codes == [2, 2]                                # CAPACITY on every rank
    s = c2_shared_prompt(users=30, reqs_per_user=10)
    o = Oracle(16, SEED, 2)
    exp_first = o.process(s.slice(0, 40))
    got_first = np.concatenate([np.load(tmp_path / f"first{r}.npy") for r in range(world)])
    assert np.array_equal(got_first, exp_first)
    if all(x[2] == 0 for x in st):
        exp_again = o.process(s.slice(40, s.n_requests // 2))
        got = np.concatenate([np.load(tmp_path / f"again{r}.npy") for r in range(world)])
        assert np.array_equal(got, exp_again)
    else:
        assert case == "capacity"       # the retry may overflow too; it must fail alike
        assert len({int(x[2]) for x in st}) == 1
