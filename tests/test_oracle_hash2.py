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
