"""Pins for the oracle's LRU eviction (SPEC evict_lru S:117-125, insert_blocks
S:108-116; readings R22-R25).  CPU only, seconds.

What fixes the eviction arithmetic from outside the oracle:
  * the SPEC's own examples, replayed as request streams;
  * Mattson's stack-distance theorem: with one-block prompts under Prefix Caching, a reference
    hits under LRU with capacity C iff fewer than C distinct other blocks were referenced since
    its previous reference (brute force over the reference string, no cache simulated);
  * the cyclic-thrash closed form (m blocks cycled: C = m-1 never hits, C = m hits all but m);
  * an independent brute-force implementation (tests/trie_ref.py: content-keyed trie, victim by a
    linear min scan) on random multi-user streams for all three policies, entry by entry incl.
    last_used;
  * capacity / lifetime invariants of SPEC "Invariants & Properties".
"""
import numpy as np
import pytest

from oracle import Oracle, POLICY_APC, POLICY_SOLIDARITY, POLICY_USER_ISOLATION
from oracle_helpers import Blocks, NONE, prompts_of
from trie_ref import TrieRef
from workloads.gen import random_small

SEED = 0x5011D000


def _ex(o):
    return {int(e["key"]): (int(e["owner"]), int(e["sharer"]), int(e["last_used"]))
            for e in o.dump_ex()}


def _key(o, blocks, names, user=0, divert_at=-1):
    _, K = o.chain(blocks.prompt(names), user, divert_at)
    return int(K[-1])


def test_spec_insert_examples():
    """2 blocks into an empty cache of capacity 4 -> 2 entries, unflagged, owner set;
    3 blocks into a full cache of capacity 3 -> the 3 least-recently-used prior entries go."""
    B = Blocks()
    o = Oracle(16, SEED, POLICY_SOLIDARITY, capacity=4)
    o.process_prompts([B.prompt(["A", "B"])], [7])
    t = _ex(o)
    assert len(t) == 2 and all(v[0] == 7 and v[1] == NONE for v in t.values())
    o = Oracle(16, SEED, POLICY_SOLIDARITY, capacity=3)
    o.process_prompts([B.prompt(["A"]), B.prompt(["B"]), B.prompt(["C"])], [1, 1, 1])
    assert o.size() == 3
    o.process_prompts([B.prompt(["D", "E", "F"])], [1])
    keys = set(_ex(o))
    assert keys == {_key(o, B, ["D"]), _key(o, B, ["D", "E"]), _key(o, B, ["D", "E", "F"])}
    assert o.evictions() == 3


def test_spec_evict_examples():
    """last_used {1,5,3}, one eviction -> the entry with last_used 1 goes; equal
    last_used -> the smaller hash goes first; an evicted flagged entry re-inserted is unflagged
    with the new owner."""
    B = Blocks()
    o = Oracle(16, SEED, POLICY_APC, capacity=3)
    short = B.prompt([], tail=5)                      # 0 full blocks: advances the clock only
    o.process_prompts([short, B.prompt(["A"]), B.prompt(["B"]), B.prompt(["C"]), short,
                       B.prompt(["B"])], [1] * 6)
    t = _ex(o)
    kA, kB, kC = (_key(o, B, [x]) for x in "ABC")
    assert {k: v[2] for k, v in t.items()} == {kA: 1, kB: 5, kC: 3}
    o.process_prompts([B.prompt(["D"])], [1])
    assert set(_ex(o)) == {kB, kC, _key(o, B, ["D"])}

    o = Oracle(16, SEED, POLICY_APC, capacity=2)
    o.process_prompts([B.prompt(["P", "Q"])], [1])   # both entries carry last_used 0
    kP, kPQ = _key(o, B, ["P"]), _key(o, B, ["P", "Q"])
    o.process_prompts([B.prompt(["R"])], [1])
    assert set(_ex(o)) == {max(kP, kPQ), _key(o, B, ["R"])}

    o = Oracle(16, SEED, POLICY_SOLIDARITY, capacity=2)
    o.process_prompts([B.prompt(["A"]), B.prompt(["A"])], [1, 2])   # u2 flags A (D2)
    kA = _key(o, B, ["A"])
    assert _ex(o)[kA][:2] == (1, 2)
    o.process_prompts([B.prompt(["X"]), B.prompt(["Y"])], [5, 5])   # A is the LRU victim
    assert kA not in _ex(o)
    o.process_prompts([B.prompt(["A"])], [3])
    assert _ex(o)[kA][:2] == (3, NONE)


def _stack_distance_hits(refs, C):
    """Mattson et al.: LRU(C) hits reference i iff the number of distinct other items referenced
    since the previous reference of refs[i] is < C (cold misses otherwise)."""
    hits = []
    for i, x in enumerate(refs):
        prev = max((p for p in range(i) if refs[p] == x), default=None)
        hits.append(prev is not None and len(set(refs[prev + 1:i]) - {x}) < C)
    return np.array(hits)


@pytest.mark.parametrize("policy", [POLICY_APC, POLICY_SOLIDARITY])
def test_mattson_stack_distance(policy):
    """One-block prompts, one user: the oracle's hits equal the stack-distance brute force for
    every capacity (no chains, so no tie-break is involved)."""
    B = Blocks(seed=99)
    rng = np.random.default_rng(3)
    w = 1.0 / np.arange(1, 41) ** 0.9
    refs = list(rng.choice(40, size=700, p=w / w.sum()))
    prompts = [B.prompt([f"b{x}"]) for x in refs]
    for C in (1, 2, 5, 17, 39, 40):
        o = Oracle(16, SEED, policy, capacity=C)
        res = o.process_prompts(prompts, [4] * len(prompts))
        assert np.array_equal(res["reused"] == 1, _stack_distance_hits(refs, C)), C
        assert o.size() == min(C, len(set(refs)))


def test_cyclic_thrash_closed_form():
    """m one-block prompts cycled 5 times: LRU with C = m-1 misses every time (each block is the
    victim just before it comes back); C = m misses only the first cycle."""
    B = Blocks(seed=5)
    m = 8
    prompts = [B.prompt([f"c{i % m}"]) for i in range(5 * m)]
    o = Oracle(16, SEED, POLICY_APC, capacity=m - 1)
    assert int(o.process_prompts(prompts, [1] * len(prompts))["reused"].sum()) == 0
    o = Oracle(16, SEED, POLICY_APC, capacity=m)
    assert int(o.process_prompts(prompts, [1] * len(prompts))["reused"].sum()) == 4 * m


def _streams():
    for seed in range(1, 9):
        yield random_small(140, users=int(1 + seed % 4), alphabet_blocks=3, max_blocks=5,
                           seed=seed, enforce_prob=0.8 if seed % 2 else 1.0)


def _keyfn(o):
    def f(name):
        if name[0] == "S":
            toks = np.concatenate([np.array(b, np.uint32) for b in name[1]])
            return int(o.chain(toks)[1][-1])
        _, root, u, path = name
        toks = np.concatenate([np.array(b, np.uint32) for b in root + path])
        return int(o.chain(toks, u, len(root))[1][-1])
    return f


@pytest.mark.parametrize("policy", [POLICY_APC, POLICY_USER_ISOLATION, POLICY_SOLIDARITY])
@pytest.mark.parametrize("capacity", [4, 7, 12])
def test_trie_lru_reference_agrees(policy, capacity):
    """Brute-force LRU over the content-keyed trie equals the oracle request by request and
    entry by entry (owner, sharer, last_used), with evictions in every stream."""
    for s in _streams():
        o = Oracle(16, SEED, policy, capacity=capacity)
        res = o.process(s)
        t = TrieRef(16, policy, capacity=capacity, keyfn=_keyfn(o))
        en = s.enforce if s.enforce is not None else np.ones(s.n_requests, np.uint8)
        for j, p in enumerate(prompts_of(s)):
            exp = t.admit(p, int(s.users[j]), bool(en[j]))
            got = tuple(int(res[j][f]) for f in
                        ["n_blocks", "shared_hits", "reused", "divert_at", "flag_depth", "bits"])
            assert got == exp, (s.name, j, got, exp)
        tab = _ex(o)
        kf = _keyfn(o)
        assert len(tab) == len(t.table) <= capacity
        for name, owner, sharer in t.entries():
            assert tab[kf(name)] == (owner, sharer, t.last_used[name])
        assert o.evictions() == t.evictions > 0


@pytest.mark.parametrize("policy", [POLICY_APC, POLICY_USER_ISOLATION, POLICY_SOLIDARITY])
def test_lifetime_invariants(policy):
    """capacity never exceeded after any request; a live entry's owner never changes;
    its flag only goes unset -> set; last_used never decreases while it lives."""
    for s in list(_streams())[:4]:
        o = Oracle(16, SEED, policy, capacity=6)
        prev = {}
        for p, u, e in zip(prompts_of(s), s.users, s.enforce if s.enforce is not None
                           else np.ones(s.n_requests, np.uint8)):
            o.process_prompts([p], [int(u)], np.array([e], np.uint8))
            cur = _ex(o)
            assert len(cur) <= 6
            for k, (ow, sh, lu) in cur.items():
                if k in prev:
                    pow_, psh, plu = prev[k]
                    assert ow == pow_ and lu >= plu
                    assert psh == NONE or sh == psh
            prev = cur


@pytest.mark.parametrize("policy", [POLICY_APC, POLICY_USER_ISOLATION, POLICY_SOLIDARITY])
def test_unbounded_capacity_is_no_eviction(policy):
    """Capacity above the number of distinct keys: no eviction, identical results and table to
    the unbounded oracle (R9 behaviour)."""
    for s in list(_streams())[:4]:
        a, b = Oracle(16, SEED, policy), Oracle(16, SEED, policy, capacity=10_000)
        ra, rb = a.process(s), b.process(s)
        assert np.array_equal(ra, rb) and b.evictions() == 0
        assert np.array_equal(a.dump_ex(), b.dump_ex())
