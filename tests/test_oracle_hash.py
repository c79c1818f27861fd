"""Pins for the oracle's chunking and key derivation (DESIGN.md §2.1 H-def v2).

The paper fixes no hash (P:937 is the only 'hash' in PAPER.md); these tests pin the oracle's
arithmetic against things other than itself: a published splitmix64 vector, the closed-form
big-integer polynomial that the chain must equal, exhaustive no-collision checks, and chunking.
"""
import numpy as np
import pytest

from oracle import Oracle, POLICY_APC
from workloads.gen import run

P = (1 << 61) - 1
MASK = (1 << 64) - 1


def test_splitmix64_published_vector():
    # Vigna's splitmix64.c reference output for seed 1234567 (state advances by the golden gamma
    # before each output): 6457827717110365317, 3203168211198807973, 9817491932198370423, ...
    expected = [6457827717110365317, 3203168211198807973, 9817491932198370423,
                4593380528125082431, 16408922859458223821]
    got = [Oracle.splitmix64((1234567 + i * 0x9E3779B97F4A7C15) & MASK) for i in range(5)]
    assert got == expected


def _unfmix(k):
    # inverse of the MurmurHash3 finaliser, derived independently (modular inverses of the odd
    # multipliers; x ^= x >> 33 is an involution because 33 >= 32)
    inv1 = pow(0xff51afd7ed558ccd, -1, 1 << 64)
    inv2 = pow(0xc4ceb9fe1a85ec53, -1, 1 << 64)
    k ^= k >> 33
    k = (k * inv2) & MASK
    k ^= k >> 33
    k = (k * inv1) & MASK
    k ^= k >> 33
    return k


def test_fmix64_is_a_bijection():
    rng = np.random.default_rng(3)
    for x in rng.integers(0, 1 << 63, size=2000, dtype=np.uint64).tolist() + [0, 1, MASK]:
        assert _unfmix(Oracle.fmix64(x)) == x
    assert Oracle.fmix64(0) == 0   # the only preimage of 0: keys (S + offset != 0) are never 0


@pytest.mark.parametrize("seed", [0, 1, 0xDEADBEEF, (1 << 64) - 1])
def test_B_and_M_derivation(seed):
    o = Oracle(16, seed, POLICY_APC)
    B, M = o.params()
    assert B == (1 << 32) + Oracle.splitmix64(seed) % (P - (1 << 33))
    assert (1 << 32) <= B < P
    assert M == pow(B, 16, P)


@pytest.mark.parametrize("bs,seed", [(16, 7), (16, 0x5011D000), (4, 11), (1, 5)])
def test_chain_equals_closed_form_polynomial(bs, seed):
    """S[b] must equal sum_{P < bs*b} (tok_P + 1) * B^P  +  sum_{t=f+1..b} sigma_u * M^(t-1)
    (mod p): the composable form the GPU scan relies on, evaluated here with Python big ints."""
    o = Oracle(bs, seed, POLICY_APC)
    B, M = o.params()
    rng = np.random.default_rng(seed)
    for trial in range(12):
        n = int(rng.integers(0, 40))
        toks = rng.integers(0, 1 << 20, size=n * bs, dtype=np.uint32)
        user = int(rng.integers(0, 0xFFFFFFFF))
        f = int(rng.integers(-1, n + 1))
        S, K = o.chain(toks, user, f)
        sigma = 1 + Oracle.splitmix64(seed ^ 0xD1B54A32D192ED03 ^ user) % (P - 1)
        assert o.sigma(user) == sigma and 1 <= sigma < P
        acc = 0
        for b in range(1, n + 1):
            poly = sum((int(toks[q]) + 1) * pow(B, q, P) for q in range(bs * b)) % P
            if f >= 0:
                poly = (poly + sum(sigma * pow(M, t - 1, P) for t in range(f + 1, b + 1))) % P
            assert int(S[b - 1]) == poly, (trial, b)
            key = Oracle.fmix64((poly + 0x9E3779B97F4A7C15) & MASK)
            assert int(K[b - 1]) == (key if key else 1) and key != 0
            acc += 1


def test_chain_is_prefix_faithful():
    """Two prompts share the first b keys iff their first b*bs tokens are equal."""
    o = Oracle(16, 1, POLICY_APC)
    a = run(1, 1, 0, 16 * 6)
    b = a.copy()
    b[16 * 3 + 5] ^= 1
    _, Ka = o.chain(a)
    _, Kb = o.chain(b)
    assert (Ka[:3] == Kb[:3]).all() and (Ka[3:] != Kb[3:]).all()


@pytest.mark.parametrize("bs,nblk", [(2, 2), (3, 3), (1, 6)])
def test_exhaustive_small_vocab_no_collisions(bs, nblk):
    """S:56 'exhaustive check over a 3-token vocabulary ... zero collisions', scaled so every
    prompt of nblk blocks is enumerable: every distinct (namespace, prefix) gets a distinct key."""
    import itertools
    o = Oracle(bs, 99, POLICY_APC)
    seen = {}
    for toks in itertools.product(range(3), repeat=bs * nblk):
        arr = np.array(toks, dtype=np.uint32)
        for ns in [(-1, 0), (0, 5), (1, 5), (1, 6)]:
            f, u = ns
            if f > nblk:
                continue
            _, K = o.chain(arr, u, f)
            for b in range(1, nblk + 1):
                if f < 0 or b <= f:
                    name = ("S", toks[:bs * b])
                else:
                    name = (ns, toks[:bs * f] if f > 0 else (), toks[:bs * b])
                k = int(K[b - 1])
                if k in seen:
                    assert seen[k] == name, (seen[k], name)
                else:
                    seen[k] = name
    assert len(seen) > 3 ** (bs * nblk)


@pytest.mark.parametrize("length,blocks", [(35, 2), (16, 1), (7, 0), (0, 0), (32, 2), (47, 2)])
def test_chunking(length, blocks):
    """35 tokens -> 2 blocks + tail 3; 16 -> 1 + 0; 7 -> 0 + 7.  The tail is never
    hashed or cached."""
    o = Oracle(16, 3, POLICY_APC)
    res = o.process_prompts([run(3, 9, length, length)], [0])
    assert int(res["n_blocks"][0]) == blocks
    assert o.size() == blocks


def test_invalid_batches_are_rejected_without_side_effects():
    o = Oracle(16, 3, POLICY_APC)
    good = run(3, 9, 0, 40)
    bad = good.copy()
    bad[5] = 1 << 20
    with pytest.raises(ValueError):
        o.process_prompts([good, bad], [0, 1])
    assert o.size() == 0
    with pytest.raises(ValueError):
        o.process_prompts([good], [0xFFFFFFFF])
    with pytest.raises(ValueError):
        o.process_arrays(good, np.array([0, 30, 20], np.uint64), np.array([0, 1], np.uint32))
    assert o.size() == 0
