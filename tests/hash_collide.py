"""A constructed H-def v2 chain collision (test helper; no method arithmetic of the product path).

H-def v2 keys one 61-bit polynomial in the secret base B: h(block) =
sum_i (tok_i + 1) B^i mod p.  Two blocks that differ by d0 at position 0 and by c at position 1
have equal hashes iff d0 + c B == 0 (mod p), i.e. B == -d0 / c.  B is derived from the seed as
2^32 + (splitmix64(seed) mod (p - 2^33)), and splitmix64 is a bijection, so a seed that yields
that B can be written down: seed = splitmix64^-1(B - 2^32).  With it, two prompts that share
block 1 and differ in block 2 get the SAME depth-2 chain value — a false prefix hit under a
one-component key; H-def v3's second, independent chain (base B2 from another salt) must
separate them.
"""
P = (1 << 61) - 1
MASK = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
M1, M2 = 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def splitmix64(x: int) -> int:
    """Vigna's splitmix64 output function (pinned by its published vector in test_oracle_hash)."""
    z = (x + GAMMA) & MASK
    z = ((z ^ (z >> 30)) * M1) & MASK
    z = ((z ^ (z >> 27)) * M2) & MASK
    return z ^ (z >> 31)


def _unxorshift(y: int, s: int) -> int:
    x = y
    for _ in range(64 // s + 1):
        x = y ^ (x >> s)
    return x & MASK


def unsplitmix64(z: int) -> int:
    z = _unxorshift(z, 31)
    z = (z * pow(M2, -1, 1 << 64)) & MASK
    z = _unxorshift(z, 27)
    z = (z * pow(M1, -1, 1 << 64)) & MASK
    z = _unxorshift(z, 30)
    return (z - GAMMA) & MASK


def base_of(seed: int) -> int:
    return (1 << 32) + splitmix64(seed) % (P - (1 << 33))


def colliding_seed_and_prompts(block1, tail_len: int = 0):
    """(seed, prompt_a, prompt_b): equal block 1, block 2 differing at positions 0 and 1 so that
    their H-def v2 block hashes collide under the returned seed."""
    import numpy as np
    for d0 in range(1, 5000):
        for c in (1, 2, 3, 5, 7):
            b_star = (-d0 * pow(c, -1, P)) % P
            if (1 << 32) <= b_star < P - (1 << 32):
                seed = unsplitmix64(b_star - (1 << 32))
                assert base_of(seed) == b_star
                blk = np.arange(16, dtype=np.uint32) * 37 + 11
                a, b = blk.copy(), blk.copy()
                a[0], b[0] = 20000 + d0, 20000          # a0 - b0 = d0
                a[1], b[1] = 10000 + c, 10000           # a1 - b1 = c
                tail = np.arange(tail_len, dtype=np.uint32) + 5
                pa = np.concatenate([np.asarray(block1, np.uint32), a, tail])
                pb = np.concatenate([np.asarray(block1, np.uint32), b, tail])
                return seed, pa, pb
    raise AssertionError("no in-range base found")
