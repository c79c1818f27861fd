"""Differential fuzzing of the CUDA path against the oracle (seeded, so reproducible): random
small streams (users, alphabet, lengths, tails, enforce bits), random policy, random batch
partitions, with or without LRU eviction at a random capacity, one- or two-component keys.
Every case must be bit-exact on every result field and on the final index."""
import os

import numpy as np
import pytest

from oracle import Oracle
from workloads import random_small

pytestmark = pytest.mark.gpu
SEED = 0x5011D000
POLS = ["apc", "user_isolation", "solidarity"]


def _case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 260))
    s = random_small(n, users=int(rng.integers(1, 7)), alphabet_blocks=int(rng.integers(2, 7)),
                     max_blocks=int(rng.integers(0, 9)), seed=int(seed) + 1000,
                     tail_prob=float(rng.random()), enforce_prob=float(rng.choice([1.0, 0.7, 0.3])))
    policy = POLS[int(rng.integers(3))]
    evict = bool(rng.random() < 0.5)
    cap = int(rng.integers(8, 60)) if evict else 1 << 14
    nc = int(rng.choice([1, 2]))
    cuts = [0]
    while cuts[-1] < n:
        cuts.append(min(n, cuts[-1] + int(rng.choice([1, 3, 17, 64, 1000]))))
    return s, policy, evict, cap, nc, cuts


def _admit(P, idx, b, evict):
    try:
        return P.as_numpy(idx.admit(**P.to_device(b)))
    except P.SolidError as e:                 # evict: a batch that must be split (R1)
        if not evict or e.status != P.SOLID_ERR_CAPACITY or b.n_requests < 2:
            raise
        h = b.n_requests // 2
        return np.concatenate([_admit(P, idx, b.slice(0, h), evict),
                               _admit(P, idx, b.slice(h, b.n_requests), evict)])


# FUZZ_CHUNKS=N widens the campaign (40 cases per chunk; the suite runs 4)
@pytest.mark.parametrize("chunk", range(int(os.environ.get("FUZZ_CHUNKS", "4"))))
def test_fuzz(chunk):
    import torch
    import paper_2603_10726_b200 as P
    for seed in range(chunk * 40, chunk * 40 + 40):
        s, policy, evict, cap, nc, cuts = _case(seed)
        idx = P.Index(policy, capacity_blocks=cap, max_batch_tokens=max(s.n_tokens, 64) + 64,
                      max_batch_requests=max(s.n_requests, 1), max_blocks=8, seed=SEED,
                      evict=evict, hash_components=nc)
        got = np.concatenate([_admit(P, idx, s.slice(a, b), evict)
                              for a, b in zip(cuts[:-1], cuts[1:])])
        torch.cuda.synchronize()
        o = Oracle(16, SEED, POLS.index(policy), capacity=cap if evict else 0, components=nc)
        exp = o.process(s)
        ctx = (seed, policy, evict, cap, nc)
        assert np.array_equal(got, exp), ctx
        gd = idx.dump_ex() if evict else idx.dump()
        ed = o.dump_ex() if evict else o.dump()
        assert len(gd) == len(ed), ctx
        for f in ed.dtype.names:
            assert np.array_equal(gd[f], ed[f]), (ctx, f)
        idx.close()


def _admit_bt(P, idx, o, b, evict, ctx):
    """Admit with splitting; the oracle takes the same sub-batches; every accepted sub-batch's
    block table (covered positions) must equal the oracle's."""
    import torch
    try:
        got = P.as_numpy(idx.admit(**P.to_device(b)))
        torch.cuda.synchronize()
    except P.SolidError as e:
        if not evict or e.status != P.SOLID_ERR_CAPACITY or b.n_requests < 2:
            raise
        h = b.n_requests // 2
        _admit_bt(P, idx, o, b.slice(0, h), evict, ctx)
        _admit_bt(P, idx, o, b.slice(h, b.n_requests), evict, ctx)
        return
    assert np.array_equal(got, o.process(b)), ctx
    if b.n_requests:
        bt = idx.block_table(b.n_tokens).cpu().numpy().view(np.uint32)
        ob, offs = o.block_table(), b.offsets.astype(np.int64)
        for j in range(b.n_requests):
            a, n = offs[j] // 16, (offs[j + 1] - offs[j]) // 16
            assert np.array_equal(bt[a:a + n], ob[a:a + n]), (ctx, j)


@pytest.mark.parametrize("chunk", range(int(os.environ.get("FUZZ_CHUNKS", "4")) // 2 or 1))
def test_fuzz_block_tables(chunk):
    """The same random cases with physical block ids on: every block table and every live
    entry's block equal the oracle's FIFO pool (R26-R28)."""
    import paper_2603_10726_b200 as P
    for seed in range(10_000 + chunk * 40, 10_000 + chunk * 40 + 40):
        s, policy, evict, cap, nc, cuts = _case(seed)
        idx = P.Index(policy, capacity_blocks=cap, max_batch_tokens=max(s.n_tokens, 64) + 64,
                      max_batch_requests=max(s.n_requests, 1), max_blocks=8, seed=SEED,
                      evict=evict, hash_components=nc, block_table=True)
        o = Oracle(16, SEED, POLS.index(policy), capacity=cap if evict else 0, components=nc,
                   pool=cap)
        ctx = (seed, policy, evict, cap, nc)
        for a, b in zip(cuts[:-1], cuts[1:]):
            _admit_bt(P, idx, o, s.slice(a, b), evict, ctx)
        gk, gp = idx.dump_phys()
        ek, ep = o.dump_phys()
        assert np.array_equal(gk, ek) and np.array_equal(gp, ep), ctx
        idx.close()
