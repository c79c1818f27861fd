"""Pins for the two-component key derivation (H-def v3, SURVEY §8 row f4 hardening, DESIGN.md
§11): a second, independent polynomial chain (base B2, salts sigma2) and keys that depend on both
61-bit chain values.  Checked against the closed-form big-integer polynomials, an exhaustive
no-collision enumeration, and the method's decisions, which must not depend on the key function
(absent collisions)."""
import itertools

import numpy as np
import pytest

from oracle import Oracle, POLICY_APC, POLICY_SOLIDARITY, POLICY_USER_ISOLATION
from oracle_helpers import prompts_of
from workloads.gen import random_small

P = (1 << 61) - 1
MASK = (1 << 64) - 1


@pytest.mark.parametrize("seed", [0, 7, 0x5011D000, MASK])
def test_second_base_derivation(seed):
    o = Oracle(16, seed, POLICY_APC, components=2)
    B2, M2 = o.params2()
    assert B2 == (1 << 32) + Oracle.splitmix64(seed ^ 0xA0761D6478BD642F) % (P - (1 << 33))
    assert M2 == pow(B2, 16, P)
    assert B2 != o.params()[0]


@pytest.mark.parametrize("bs,seed", [(16, 3), (4, 0x5011D000), (1, 9)])
def test_both_chains_equal_closed_form(bs, seed):
    """S and S2 are each the closed-form polynomial of their own base; the key combines both."""
    o = Oracle(bs, seed, POLICY_APC, components=2)
    o1 = Oracle(bs, seed, POLICY_APC)
    B, M = o.params()
    B2, M2 = o.params2()
    rng = np.random.default_rng(seed & 0xFFFF)
    for _ in range(8):
        n = int(rng.integers(0, 24))
        toks = rng.integers(0, 1 << 20, size=n * bs, dtype=np.uint32)
        u = int(rng.integers(0, 0xFFFFFFFF))
        f = int(rng.integers(-1, n + 1))
        S, S2, K = o.chain2(toks, u, f)
        S1, _ = o1.chain(toks, u, f)
        assert np.array_equal(S, S1)          # component 1 is H-def v2's chain
        sg2 = 1 + Oracle.splitmix64(seed ^ 0xE7037ED1A0B428DB ^ u) % (P - 1)
        for b in range(1, n + 1):
            poly2 = sum((int(toks[q]) + 1) * pow(B2, q, P) for q in range(bs * b)) % P
            if f >= 0:
                poly2 = (poly2 + sum(sg2 * pow(M2, t - 1, P) for t in range(f + 1, b + 1))) % P
            assert int(S2[b - 1]) == poly2
            x = (int(S[b - 1]) ^ ((poly2 * 0x9E3779B97F4A7C15) & MASK))
            k = Oracle.fmix64((x + 0x9E3779B97F4A7C15) & MASK)
            assert int(K[b - 1]) == (k if k else 1)


def test_exhaustive_small_vocab_no_collisions_two_components():
    o = Oracle(2, 99, POLICY_APC, components=2)
    seen = {}
    for toks in itertools.product(range(3), repeat=6):
        arr = np.array(toks, dtype=np.uint32)
        for f, u in [(-1, 0), (0, 5), (1, 5), (2, 6)]:
            _, _, K = o.chain2(arr, u, f)
            for b in range(1, 4):
                name = ("S", toks[:2 * b]) if (f < 0 or b <= f) else ((f, u), toks[:2 * f], toks[:2 * b])
                k = int(K[b - 1])
                assert seen.setdefault(k, name) == name
    assert len(seen) > 3 ** 6


@pytest.mark.parametrize("policy", [POLICY_APC, POLICY_USER_ISOLATION, POLICY_SOLIDARITY])
def test_decisions_do_not_depend_on_the_key_function(policy):
    for seed in range(1, 6):
        s = random_small(200, users=1 + seed % 4, alphabet_blocks=3, max_blocks=6, seed=seed,
                         enforce_prob=0.8 if seed % 2 else 1.0)
        a, b = Oracle(16, 1, policy), Oracle(16, 1, policy, components=2)
        assert np.array_equal(a.process(s), b.process(s))
        da, db = a.dump(), b.dump()
        assert len(da) == len(db)
        assert sorted(zip(da["owner"], da["sharer"])) == sorted(zip(db["owner"], db["sharer"]))
        assert not np.array_equal(np.sort(da["key"]), np.sort(db["key"]))


def test_unsplitmix_inverts_splitmix():
    from hash_collide import splitmix64, unsplitmix64
    rng = np.random.default_rng(11)
    for x in rng.integers(0, 1 << 63, size=500, dtype=np.uint64).tolist() + [0, 1, MASK]:
        assert unsplitmix64(splitmix64(x)) == x
        assert splitmix64(x) == Oracle.splitmix64(x)


def _prompt_stream(prompts, users):
    from workloads.gen import _pack
    return _pack("collide", list(prompts), list(users))


def test_constructed_chain_collision_separated_by_second_component():
    """key2_of pinned by construction (not by retyping it): two prompts whose FIRST chain values
    are equal at depth 2 (a collision built from the secret base, tests/hash_collide.py) must get
    equal H-def v2 keys — a false prefix hit, user 2 reusing user 1's block 2 under APC — and
    different H-def v3 keys, so the second component (S2) must enter the key: a key2_of that
    dropped S2, or mixed it so that it cancels, fails here."""
    from hash_collide import colliding_seed_and_prompts
    blk1 = np.arange(16, dtype=np.uint32) * 101 + 3
    seed, pa, pb = colliding_seed_and_prompts(blk1, tail_len=5)
    o1 = Oracle(16, seed, POLICY_APC)
    o2 = Oracle(16, seed, POLICY_APC, components=2)
    Sa, Ka = o1.chain(pa)
    Sb, Kb = o1.chain(pb)
    assert Sa[0] == Sb[0] and Sa[1] == Sb[1] and Ka[1] == Kb[1]       # the built collision
    S1a, S2a, K2a = o2.chain2(pa)
    S1b, S2b, K2b = o2.chain2(pb)
    assert S1a[1] == S1b[1] and S2a[1] != S2b[1]                       # only S2 tells them apart
    assert K2a[0] == K2b[0] and K2a[1] != K2b[1]
    # consequence for the method (P:102-104 longest cached prefix): one-component keys serve
    # user 2 user 1's block 2 (content it never sent); two-component keys do not
    s = _prompt_stream([pa, pb], [1, 2])
    assert o1.process(s)["reused"].tolist() == [0, 2]
    assert o2.process(s)["reused"].tolist() == [0, 1]


def test_key2_recovers_second_chain_by_inversion():
    """The key is an invertible function of (S, S2): undoing fmix64 (its independently derived
    inverse, test_oracle_hash._unfmix), the offset, the XOR with S and the odd multiplier gives
    back S2 — the closed-form second polynomial — for every depth."""
    from test_oracle_hash import _unfmix
    o = Oracle(16, 0x5011D000, POLICY_APC, components=2)
    rng = np.random.default_rng(4)
    inv_mix = pow(0x9E3779B97F4A7C15, -1, 1 << 64)
    for _ in range(6):
        toks = rng.integers(0, 1 << 20, size=16 * int(rng.integers(1, 9)), dtype=np.uint32)
        S, S2, K = o.chain2(toks, int(rng.integers(0, 1 << 31)), -1)
        for b in range(len(K)):
            x = (_unfmix(int(K[b])) - 0x9E3779B97F4A7C15) & MASK
            assert ((x ^ int(S[b])) * inv_mix) & MASK == int(S2[b])
