"""Pins for in-flight pinning (SURVEY §8 row f4 "mapping entries to paged KV block ids with
pinning/refcount"; the paper's artifact extends vLLM's KVCacheBlock, whose reference count keeps
a running request's blocks from being reclaimed; reading R38).  CPU only.

Semantics: with pin on, every admitted request holds one pin on each entry of its block-table
row (the entries holding its KV) until the caller releases that row; the LRU victim is the
smallest (last_used, key) among UNPINNED entries; a request whose eviction step would need more
victims than there are unpinned entries it does not use itself is refused, nothing of it applied.

What fixes it from outside the oracle:
  * a brute-force reference (tests/trie_ref.py with pin=True: content-keyed trie, victim by a
    linear minimum scan over the unpinned entries, pins counted per entry name) on random
    streams with random releases — results, rows, pin counts and refusals identical;
  * the invariant the feature exists for: a block named by an unreleased row keeps holding the
    same entry until released (never reclaimed);
  * closed forms: C one-block prompts pin the whole cache, the next new prompt is refused;
    releasing one row lets exactly that entry be evicted and its block reused.
"""
import numpy as np
import pytest

from oracle import Oracle, PinRefused, POLICY_APC, POLICY_SOLIDARITY, POLICY_USER_ISOLATION
from oracle_helpers import Blocks, NONE, prompts_of
from test_oracle_pool import _keyfn
from trie_ref import TrieRef
from workloads.gen import random_small

SEED = 0x5011D000


def _one(o, p, u, e=1):
    """Admit one prompt; returns (result, row) or (None, None) if refused."""
    try:
        res = o.process_prompts([p], [int(u)], np.array([e], np.uint8))[0]
    except PinRefused as r:
        assert r.admitted == 0
        return None, None
    return res, o.block_table()[:len(p) // 16]


def test_closed_form_full_pin_refuses_then_release_frees_one():
    B = Blocks(seed=11)
    C = 5
    o = Oracle(16, SEED, POLICY_APC, capacity=C, pool=C, pin=True)
    rows = []
    for i in range(C):
        res, row = _one(o, B.prompt([f"x{i}"]), 1)
        rows.append(row)
        assert list(row) == [i]
    # every entry is pinned: a new prompt needs a victim and none is evictable
    res, _ = _one(o, B.prompt(["y"]), 1)
    assert res is None and o.size() == C
    # a hit needs no victim: still admitted (and pins x2 a second time)
    res, row = _one(o, B.prompt(["x2"]), 1)
    assert res["reused"] == 1 and list(row) == [2]
    # release x3's row: now exactly x3 is evictable; y takes its block 3
    o.release(rows[3])
    res, row = _one(o, B.prompt(["y"]), 1)
    assert res is not None and list(row) == [3]
    keys, pins = o.dump_pins()
    assert sorted(pins.tolist()) == [1, 1, 1, 1, 2]
    # releasing a block whose entry holds no pin is an error
    o.release(rows[0])
    with pytest.raises(ValueError):
        o.release(rows[0])


def test_pinned_blocks_are_never_reclaimed():
    """Random traffic with a small cache; every outstanding (unreleased) row's blocks keep
    holding the same keys until the row is released."""
    rng = np.random.default_rng(5)
    for seed in range(1, 5):
        s = random_small(300, users=3, alphabet_blocks=6, max_blocks=4, seed=seed)
        cap = 12
        o = Oracle(16, SEED, POLICY_SOLIDARITY, capacity=cap, pool=cap, pin=True)
        outstanding = []                        # (row, {block: key})
        refused = 0
        for j, p in enumerate(prompts_of(s)):
            res, row = _one(o, p, s.users[j])
            if res is None:
                refused += 1
            else:
                keys, phys = o.dump_phys()
                held = dict(zip(phys.tolist(), keys.tolist()))
                outstanding.append((row.copy(), {b: held[b] for b in row if b != NONE}))
            keys, phys = o.dump_phys()
            now = dict(zip(phys.tolist(), keys.tolist()))
            for _, m in outstanding:
                for b, k in m.items():
                    assert now.get(b) == k, "a pinned block was reclaimed"
            # random completions
            while outstanding and rng.random() < 0.45:
                row, _ = outstanding.pop(int(rng.integers(len(outstanding))))
                o.release(row)
        assert refused > 0                      # the cache was really under pin pressure


@pytest.mark.parametrize("policy", [POLICY_APC, POLICY_USER_ISOLATION, POLICY_SOLIDARITY])
@pytest.mark.parametrize("capacity", [6, 10])
def test_trie_pin_reference_agrees(policy, capacity):
    """Oracle == brute force with pins: per request the result (or the refusal), the row, and
    after every step the live entries' blocks and pin counts."""
    rng = np.random.default_rng(capacity + policy)
    for seed in range(1, 5):
        s = random_small(160, users=int(1 + seed % 3), alphabet_blocks=4, max_blocks=4,
                         seed=seed, enforce_prob=0.8)
        o = Oracle(16, SEED, policy, capacity=capacity, pool=capacity, pin=True)
        t = TrieRef(16, policy, capacity=capacity, keyfn=_keyfn(o), pool=capacity, pin=True)
        kf = _keyfn(o)
        en = s.enforce if s.enforce is not None else np.ones(s.n_requests, np.uint8)
        outstanding = []
        for j, p in enumerate(prompts_of(s)):
            res, row = _one(o, p, s.users[j], en[j])
            try:
                exp = t.admit(p, int(s.users[j]), bool(en[j]))
            except TrieRef.Refused:
                exp = None
            assert (res is None) == (exp is None), (s.name, j)
            if res is not None:
                assert tuple(int(res[f]) for f in ("n_blocks", "shared_hits", "reused",
                                                    "divert_at", "flag_depth", "bits")) == exp
                assert list(row) == t.table_row
                outstanding.append(row.copy())
            if outstanding and rng.random() < 0.4:
                row = outstanding.pop(int(rng.integers(len(outstanding))))
                o.release(row)
                t.release(row)
            keys, pins = o.dump_pins()
            exp_pins = {kf(nm): t.pins.get(nm, 0) for nm, _, _ in t.entries()}
            assert dict(zip(keys.tolist(), pins.tolist())) == exp_pins
            keys, phys = o.dump_phys()
            assert dict(zip(keys.tolist(), phys.tolist())) == \
                {kf(nm): t.phys[nm] for nm, _, _ in t.entries()}
