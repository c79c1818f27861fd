"""Pins for the oracle's physical block pool and block tables ("mapping entries
to paged KV block ids"; readings R26-R28).  CPU only, seconds.

What fixes the allocator from outside the oracle:
  * closed forms: without eviction the k-th entry ever inserted holds block k (first-insertion
    order); one-block prompts cycled through an LRU cache one block too small take blocks
    0, 1, ..., C-1, 0, 1, ... (each request re-uses the block its own eviction just freed);
  * an independent brute force (tests/trie_ref.py: content-keyed trie, free blocks chosen by a
    minimum scan over "freed at" stamps instead of a FIFO) on random multi-user streams, all
    policies, with and without eviction: every block table and every live entry's block;
  * invariants: live entries hold distinct blocks < pool; a live entry's block never changes;
    free + live = pool; a block-table row names the live entries the request used.
"""
import numpy as np
import pytest

from oracle import Oracle, POLICY_APC, POLICY_SOLIDARITY, POLICY_USER_ISOLATION
from oracle_helpers import Blocks, NONE, prompts_of
from trie_ref import TrieRef
from workloads.gen import random_small

SEED = 0x5011D000


def _rows(o, s):
    """Per request, its block-table row (the last process call covered all of s)."""
    bt = o.block_table()
    offs = s.offsets.astype(np.int64)
    return [bt[offs[j] // 16: offs[j] // 16 + (offs[j + 1] - offs[j]) // 16]
            for j in range(s.n_requests)]


def test_first_insertion_order_without_eviction():
    """No eviction: block ids are handed out 0, 1, 2, ... in insertion order (request order,
    block order within a request)."""
    B = Blocks(seed=3)
    o = Oracle(16, SEED, POLICY_APC, pool=64)
    prompts = [B.prompt(["a", "b"]), B.prompt(["a", "c", "d"]), B.prompt(["e"]),
               B.prompt(["a", "b", "f"])]
    o.process_prompts(prompts, [1, 2, 3, 4])
    bt = o.block_table()
    # a b | a c d | e | a b f  ->  new entries in order: a b c d e f = 0..5
    assert list(bt[0:2]) == [0, 1]
    assert list(bt[2:5]) == [0, 2, 3]
    assert list(bt[5:6]) == [4]
    assert list(bt[6:9]) == [0, 1, 5]
    keys, phys = o.dump_phys()
    assert sorted(phys) == list(range(6))


def test_cyclic_thrash_block_ids():
    """m one-block prompts cycled with C = m-1: request i takes block i mod (m-1)."""
    B = Blocks(seed=5)
    m = 7
    prompts = [B.prompt([f"c{i % m}"]) for i in range(5 * m)]
    o = Oracle(16, SEED, POLICY_APC, capacity=m - 1, pool=m - 1)
    o.process_prompts(prompts, [1] * len(prompts))
    bt = o.block_table()
    assert list(bt) == [i % (m - 1) for i in range(5 * m)]


def test_pool_exhaustion_is_reported():
    B = Blocks(seed=7)
    o = Oracle(16, SEED, POLICY_APC, pool=2)
    with pytest.raises(ValueError, match="pool exhausted"):
        o.process_prompts([B.prompt(["a", "b", "c"])], [1])


def _keyfn(o):
    def f(name):
        if name[0] == "S":
            toks = np.concatenate([np.array(b, np.uint32) for b in name[1]])
            return int(o.chain(toks)[1][-1])
        _, root, u, path = name
        toks = np.concatenate([np.array(b, np.uint32) for b in root + path])
        return int(o.chain(toks, u, len(root))[1][-1])
    return f


def _streams():
    for seed in range(1, 7):
        yield random_small(140, users=int(1 + seed % 4), alphabet_blocks=3, max_blocks=5,
                           seed=seed, enforce_prob=0.8 if seed % 2 else 1.0)


@pytest.mark.parametrize("policy", [POLICY_APC, POLICY_USER_ISOLATION, POLICY_SOLIDARITY])
@pytest.mark.parametrize("capacity", [0, 5, 9])
def test_trie_pool_reference_agrees(policy, capacity):
    """The brute-force allocator over the content-keyed trie gives the same block table row for
    every request and the same block for every live entry."""
    for s in _streams():
        pool = capacity if capacity else 4096
        o = Oracle(16, SEED, policy, capacity=capacity, pool=pool)
        o.process(s)
        rows = _rows(o, s)
        t = TrieRef(16, policy, capacity=capacity, keyfn=_keyfn(o), pool=pool)
        en = s.enforce if s.enforce is not None else np.ones(s.n_requests, np.uint8)
        for j, p in enumerate(prompts_of(s)):
            t.admit(p, int(s.users[j]), bool(en[j]))
            assert list(rows[j]) == t.table_row, (s.name, j)
        keys, phys = o.dump_phys()
        kf = _keyfn(o)
        exp = {kf(name): t.phys[name] for name, _, _ in t.entries()}
        assert dict(zip(keys.tolist(), phys.tolist())) == exp


@pytest.mark.parametrize("policy", [POLICY_APC, POLICY_SOLIDARITY])
def test_pool_invariants(policy):
    """Request by request: live blocks distinct and < pool, a live entry keeps its block, every
    non-NONE block-table entry is the block of a live entry; NONE only where the request's own
    eviction removed an entry it referenced without touching it."""
    for s in list(_streams())[:3]:
        cap = 6
        o = Oracle(16, SEED, policy, capacity=cap, pool=cap)
        prev = {}
        for p, u, e in zip(prompts_of(s), s.users, s.enforce if s.enforce is not None
                           else np.ones(s.n_requests, np.uint8)):
            o.process_prompts([p], [int(u)], np.array([e], np.uint8))
            keys, phys = o.dump_phys()
            cur = dict(zip(keys.tolist(), phys.tolist()))
            assert len(set(cur.values())) == len(cur) and all(b < cap for b in cur.values())
            for k, b in cur.items():
                if k in prev:
                    assert prev[k] == b
            row = o.block_table()
            live_blocks = set(cur.values())
            assert all(b == NONE or b in live_blocks for b in row)
            prev = cur
