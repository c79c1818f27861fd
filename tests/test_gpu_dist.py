"""Sharded index on one GPU: G logical shards in one process with a
loopback exchange.  Every shard runs the same kernels as a multi-GPU rank; only the record
transport differs (NCCL there).  Bar: results and the union of the shard indexes bit-exact
against the sequential oracle; every entry lives on its owner shard."""
import numpy as np
import pytest

from oracle import Oracle
from workloads import c1_tiny, c2_shared_prompt, c4_attackers, random_small

pytestmark = pytest.mark.gpu
SEED = 0x5011D000
POL = {"apc": 0, "user_isolation": 1, "solidarity": 2}


def _shards(G, policy, streams, nc=1):
    from paper_2603_10726_b200.dist import ShardedIndex
    tok = max(max(s.n_tokens for s in streams), 64)
    req = max(max(s.n_requests for s in streams), 1)
    blocks = sum(s.n_blocks() for s in streams)
    return [ShardedIndex(G, r, policy, capacity_blocks=max(4 * blocks, 4096),
                         max_batch_tokens=tok + 64, max_batch_requests=req, seed=SEED,
                         hash_components=nc)
            for r in range(G)]


def _split(s, G):
    n = s.n_requests
    cuts = [n * r // G for r in range(G + 1)]
    return [s.slice(cuts[r], cuts[r + 1]) for r in range(G)], cuts[:-1]


def sharded_run(streams, G, policy, nc=1):
    import torch
    import paper_2603_10726_b200 as P
    from paper_2603_10726_b200.dist import loopback_admit
    shards = _shards(G, policy, streams, nc)
    out, rounds = [], []
    seq = 0
    for s in streams:
        parts, starts = _split(s, G)
        res, t = loopback_admit(shards, [P.to_device(p) for p in parts], [seq + c for c in starts])
        torch.cuda.synchronize()
        out.append(np.concatenate([P.as_numpy(r) for r in res]))
        rounds.append(t)
        seq += s.n_requests
    dumps = [sh.index.dump() for sh in shards]
    for r, d in enumerate(dumps):
        own = (((d["key"] >> np.uint64(32)) * np.uint64(G)) >> np.uint64(32)).astype(np.int64)
        assert (own == r).all(), "entry stored on a non-owner shard"
    merged = np.concatenate(dumps)
    merged = merged[np.argsort(merged["key"], kind="stable")]
    return np.concatenate(out), merged, rounds


def oracle_run(streams, policy):
    o = Oracle(16, SEED, POL[policy])
    res = [o.process(s) for s in streams]
    return np.concatenate(res), o.dump()


def assert_same(got, exp, gd, ed, what):
    for f in exp.dtype.names:
        bad = np.nonzero(got[f].astype(np.int64) != exp[f].astype(np.int64))[0]
        assert bad.size == 0, (what, f, int(bad[0]), got[bad[0]], exp[bad[0]])
    assert len(gd) == len(ed), (what, len(gd), len(ed))
    for f in ["key", "owner", "sharer"]:
        bad = np.nonzero(gd[f] != ed[f])[0]
        assert bad.size == 0, (what, "dump", f, int(bad[0]))


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("policy", list(POL))
def test_random_streams_sharded(G, policy):
    s = random_small(300, users=4, alphabet_blocks=3, max_blocks=20, seed=G * 7 + 1,
                     enforce_prob=0.8)
    exp, ed = oracle_run([s], policy)
    got, gd, _ = sharded_run([s], G, policy)
    assert_same(got, exp, gd, ed, f"random G={G} {policy}")


@pytest.mark.parametrize("G", [2, 4])
def test_c1_sharded_multi_batch(G):
    s = c1_tiny()
    parts = [s.slice(0, 20), s.slice(20, 41), s.slice(41, 64)]
    exp, ed = oracle_run(parts, "solidarity")
    got, gd, rounds = sharded_run(parts, G, "solidarity")
    assert_same(got, exp, gd, ed, f"c1 G={G}")
    assert all(t >= 2 for t in rounds)


@pytest.mark.parametrize("G", [2, 4])
def test_c2_small_sharded(G):
    s = c2_shared_prompt(users=40, reqs_per_user=25)
    exp, ed = oracle_run([s], "solidarity")
    got, gd, _ = sharded_run([s], G, "solidarity")
    assert_same(got, exp, gd, ed, f"c2 G={G}")


def test_c4_small_sharded():
    s = c4_attackers(benign_users=300, benign_requests=6000, victims=6, templates=3,
                     candidates=30)
    exp, ed = oracle_run([s.slice(0, 4000), s.slice(4000, s.n_requests)], "solidarity")
    got, gd, _ = sharded_run([s.slice(0, 4000), s.slice(4000, s.n_requests)], 3, "solidarity")
    assert_same(got, exp, gd, ed, "c4 G=3")


def test_c2_full_size_sharded_two_shards():
    """BASELINE configs[1] at full size through the sharded protocol (2 shards, loopback):
    exactly the sequential answer, like the single-GPU path."""
    s = c2_shared_prompt()
    exp, ed = oracle_run([s], "solidarity")
    got, gd, rounds = sharded_run([s], 2, "solidarity")
    assert_same(got, exp, gd, ed, "c2full G=2")


def test_fuzz_sharded():
    """Seeded random cases for the sharded protocol (loopback): G in 2..5 shards, random
    policy, streams cut into several global batches — results and the union of the shards bit
    exact against the oracle."""
    rng = np.random.default_rng(77)
    for case in range(24):
        G = int(rng.integers(2, 6))
        policy = list(POL)[int(rng.integers(3))]
        s = random_small(int(rng.integers(20, 200)), users=int(rng.integers(1, 6)),
                         alphabet_blocks=int(rng.integers(2, 6)), max_blocks=int(rng.integers(1, 9)),
                         seed=1000 + case, enforce_prob=float(rng.choice([1.0, 0.6])))
        k = int(rng.integers(1, 4))
        cuts = sorted(set([0, s.n_requests] + list(rng.integers(0, s.n_requests, k - 1))))
        streams = [s.slice(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
        got, gd, _ = sharded_run(streams, G, policy)
        exp, ed = oracle_run(streams, policy)
        assert_same(got, exp, gd, ed, f"fuzz{case}-G{G}-{policy}")


@pytest.mark.parametrize("policy", list(POL))
def test_two_component_keys_sharded(policy):
    """H-def v3 keys with the sharded index (G = 3): results and the shard union (keys
    included) equal the oracle with components=2."""
    s = random_small(300, users=4, alphabet_blocks=3, max_blocks=10, seed=31, enforce_prob=0.8)
    got, gd, _ = sharded_run([s.slice(0, 150), s.slice(150, 300)], 3, policy, nc=2)
    o = Oracle(16, SEED, POL[policy], components=2)
    exp = np.concatenate([o.process(s.slice(0, 150)), o.process(s.slice(150, 300))])
    assert_same(got, exp, gd, o.dump(), f"v3-sharded-{policy}")
