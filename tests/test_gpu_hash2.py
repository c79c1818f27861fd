"""GPU parity of the two-component keys (H-def v3): the CUDA
path with hash_components=2 against the oracle with components=2 — every result field and the
final index (keys included) bit-exact, all policies, several batch partitions; with LRU eviction
too."""
import numpy as np
import pytest

from oracle import Oracle
from workloads import c1_tiny, c2_shared_prompt, c4_attackers, random_small

pytestmark = pytest.mark.gpu
SEED = 0x5011D000
POL = {"apc": 0, "user_isolation": 1, "solidarity": 2}


def _run(policy, s, batch, **kw):
    import torch
    import paper_2603_10726_b200 as P
    idx = P.Index(policy, capacity_blocks=kw.pop("capacity", max(4 * s.n_blocks(), 1024)),
                  max_batch_tokens=s.n_tokens + 64, max_batch_requests=max(s.n_requests, 1),
                  seed=SEED, hash_components=2, **kw)
    out = []
    for i in range(0, s.n_requests, batch):
        out.append(P.as_numpy(idx.admit(**P.to_device(s.slice(i, min(i + batch, s.n_requests))))))
    torch.cuda.synchronize()
    return np.concatenate(out), idx


@pytest.mark.parametrize("policy", ["apc", "user_isolation", "solidarity"])
@pytest.mark.parametrize("batch", [1, 37, 100000])
def test_random_streams(policy, batch):
    for seed in (1, 2):
        s = random_small(250, users=2 + seed, alphabet_blocks=3, max_blocks=6, seed=seed,
                         enforce_prob=0.8)
        got, idx = _run(policy, s, batch)
        o = Oracle(16, SEED, POL[policy], components=2)
        assert np.array_equal(got, o.process(s))
        gd, ed = idx.dump(), o.dump()
        assert all(np.array_equal(gd[f], ed[f]) for f in ["key", "owner", "sharer"])


@pytest.mark.parametrize("policy", ["apc", "solidarity"])
def test_c1_c2_c4_small(policy):
    for s in (c1_tiny(), c2_shared_prompt(users=60, reqs_per_user=20),
              c4_attackers(benign_users=100, benign_requests=2000, victims=4, templates=2,
                           victim_repeats=3, colluders_per_victim=2, candidates=20)):
        got, idx = _run(policy, s, 5000)
        o = Oracle(16, SEED, POL[policy], components=2)
        assert np.array_equal(got, o.process(s)), s.name
        gd, ed = idx.dump(), o.dump()
        assert all(np.array_equal(gd[f], ed[f]) for f in ["key", "owner", "sharer"])


def test_two_components_with_eviction():
    s = random_small(400, users=3, alphabet_blocks=4, max_blocks=6, seed=5)
    got, idx = _run("solidarity", s, 1, capacity=16, max_blocks=8, evict=True)
    o = Oracle(16, SEED, 2, capacity=16, components=2)
    assert np.array_equal(got, o.process(s))
    gd, ed = idx.dump_ex(), o.dump_ex()
    assert all(np.array_equal(gd[f], ed[f]) for f in ["key", "owner", "sharer", "last_used"])


@pytest.mark.parametrize("components,reuse", [(1, 2), (2, 1)])
def test_constructed_collision(components, reuse):
    """The CUDA path on the constructed H-def v2 collision (tests/hash_collide.py): one-component
    keys give user 2 a false hit on user 1's block 2, two-component keys do not — equal to the
    oracle, results and index."""
    import torch
    import paper_2603_10726_b200 as P
    from hash_collide import colliding_seed_and_prompts
    from workloads.gen import _pack
    blk1 = np.arange(16, dtype=np.uint32) * 101 + 3
    seed, pa, pb = colliding_seed_and_prompts(blk1, tail_len=5)
    s = _pack("collide", [pa, pb, pb, pa], [1, 2, 3, 3])
    for policy in ("apc", "solidarity"):
        idx = P.Index(policy, capacity_blocks=1024, max_batch_tokens=s.n_tokens + 64,
                      max_batch_requests=8, seed=seed, hash_components=components)
        got = P.as_numpy(idx.admit(**P.to_device(s)))
        torch.cuda.synchronize()
        o = Oracle(16, seed, POL[policy], components=components)
        exp = o.process(s)
        assert np.array_equal(got, exp)
        assert int(got["reused"][1]) == reuse
        gd, ed = idx.dump(), o.dump()
        assert all(np.array_equal(gd[f], ed[f]) for f in ["key", "owner", "sharer"])
