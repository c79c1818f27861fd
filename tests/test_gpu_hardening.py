"""GPU tests of the boundary's failure behaviour and of the resolver's worst cases (round 2):

* capacity overflow decided BEFORE any claim — including a batch with more new entries than the
  index has slots (k_commit's linear probe would never meet an EMPTY slot otherwise);
* host admission of a batch large enough to be copied in pieces is still all-or-nothing;
* the block table is unavailable after a failed batch;
* deep Jacobi streams (tests/golden/deep_jacobi_streams.json) and a resolver round limit low
  enough to force non-convergence: the batch is committed in parts, results and index still
  equal to the oracle (R1).
"""
import json
import os

import numpy as np
import pytest

from oracle import Oracle
from workloads import c2_shared_prompt, random_small
from workloads.gen import _pack

pytestmark = pytest.mark.gpu
SEED = 0x5011D000
POL = {"apc": 0, "user_isolation": 1, "solidarity": 2}
HERE = os.path.dirname(os.path.abspath(__file__))


def _same(got, exp, gd, ed, what=""):
    for f in exp.dtype.names:
        bad = np.nonzero(got[f].astype(np.int64) != exp[f].astype(np.int64))[0]
        assert bad.size == 0, (what, f, int(bad[0]), got[bad[0]], exp[bad[0]])
    assert len(gd) == len(ed), (what, len(gd), len(ed))
    for f in ["key", "owner", "sharer"]:
        assert np.array_equal(gd[f], ed[f]), (what, f)


def _symbol_stream(name, prompts, users, enforce):
    """Symbol s -> one 16-token block of token s + 1 (block contents distinct per symbol)."""
    toks = [np.repeat(np.asarray(p, np.uint32) + 1, 16) for p in prompts]
    return _pack(name, toks, users, enforce)


def _deep_streams():
    with open(os.path.join(HERE, "golden", "deep_jacobi_streams.json")) as f:
        d = json.load(f)
    return [_symbol_stream(f"deep{i}", s["prompts"], s["users"], s["enforce"])
            for i, s in enumerate(d["streams"])]


@pytest.mark.parametrize("asynchronous", [False, True])
def test_batch_larger_than_the_table_fails_cleanly(asynchronous):
    """capacity 100 -> 1024 index slots; a batch with ~3000 new entries must fail with
    SOLID_ERR_CAPACITY without touching the index (and without spinning in the commit)."""
    import torch
    import paper_2603_10726_b200 as P
    s = random_small(400, users=4, alphabet_blocks=400, max_blocks=12, seed=21)
    assert s.n_blocks() > 2048
    idx = P.Index("solidarity", capacity_blocks=100, max_batch_tokens=s.n_tokens + 64,
                  max_batch_requests=s.n_requests, seed=SEED)
    small = s.slice(0, 4)
    o = Oracle(16, SEED, POL["solidarity"])
    e0 = o.process(small)
    g0 = P.as_numpy(idx.admit(**P.to_device(small)))
    torch.cuda.synchronize()
    before = idx.dump()
    with pytest.raises(P.SolidError) as ei:
        if asynchronous:
            idx.admit_async(**P.to_device(s))
            idx.status()
        else:
            idx.admit(**P.to_device(s))
    assert ei.value.status == P.SOLID_ERR_CAPACITY
    after = idx.dump()
    assert all(np.array_equal(before[f], after[f]) for f in ["key", "owner", "sharer"])
    assert idx.stats()["live_entries"] == len(before)
    # the context stays usable: the next small batch matches the oracle that skipped the big one
    nxt = s.slice(4, 8)
    e1 = o.process(nxt)
    g1 = P.as_numpy(idx.admit(**P.to_device(nxt)))
    torch.cuda.synchronize()
    _same(np.concatenate([g0, g1]), np.concatenate([e0, e1]), idx.dump(), o.dump(), "after")


def test_block_table_unavailable_after_failed_batch():
    import torch
    import paper_2603_10726_b200 as P
    s = random_small(300, users=3, alphabet_blocks=300, max_blocks=10, seed=23)
    idx = P.Index("solidarity", capacity_blocks=200, max_batch_tokens=s.n_tokens + 64,
                  max_batch_requests=s.n_requests, seed=SEED, block_table=True)
    small = s.slice(0, 3)
    idx.admit(**P.to_device(small))
    torch.cuda.synchronize()
    idx.block_table(small.n_tokens)           # available after a committed batch
    with pytest.raises(P.SolidError) as ei:
        idx.admit(**P.to_device(s))
    assert ei.value.status == P.SOLID_ERR_CAPACITY
    with pytest.raises(P.SolidError) as ei:
        idx.block_table(s.n_tokens)
    assert ei.value.status == P.SOLID_ERR_STATE


@pytest.mark.parametrize("fault", ["token", "capacity"])
def test_host_admission_in_pieces_is_all_or_nothing(fault):
    """A host batch of >= 64 MiB of token ids is copied and hashed in 4 pieces; a fault in the
    LAST piece (a token >= 2^20, or the index capacity) must leave the index untouched."""
    import paper_2603_10726_b200 as P
    s = c2_shared_prompt(users=200, reqs_per_user=45)            # 9000 x 2000 tokens = 72 MB
    assert s.n_tokens * 4 >= 64 << 20
    cap = s.n_blocks() if fault == "token" else 1000
    idx = P.Index("solidarity", capacity_blocks=cap, max_batch_tokens=s.n_tokens + 64,
                  max_batch_requests=s.n_requests, seed=SEED)
    warm = s.slice(0, 10)
    idx.admit_host(warm.tokens, warm.offsets, warm.users, None,
                   out=np.zeros(10, dtype=P.RESULT_DTYPE))
    before = idx.dump()
    toks = s.tokens.copy()
    if fault == "token":
        toks[-40] = 1 << 20
    out = np.zeros(s.n_requests, dtype=P.RESULT_DTYPE)
    with pytest.raises(P.SolidError) as ei:
        idx.admit_host(toks, s.offsets, s.users, None, out=out)
    assert ei.value.status == (P.SOLID_ERR_INVALID if fault == "token" else P.SOLID_ERR_CAPACITY)
    after = idx.dump()
    assert len(after) == len(before)
    assert all(np.array_equal(before[f], after[f]) for f in ["key", "owner", "sharer"])
    # non-monotone offsets are rejected on the host before anything starts
    bad = s.offsets.copy()
    bad[5] = bad[7]
    with pytest.raises(P.SolidError) as ei:
        idx.admit_host(s.tokens, bad, s.users, None, out=out)
    assert ei.value.status == P.SOLID_ERR_INVALID


def test_host_admission_in_pieces_matches_oracle():
    import paper_2603_10726_b200 as P
    s = c2_shared_prompt(users=200, reqs_per_user=45)
    idx = P.Index("solidarity", capacity_blocks=s.n_blocks(), max_batch_tokens=s.n_tokens + 64,
                  max_batch_requests=s.n_requests, seed=SEED)
    out = np.zeros(s.n_requests, dtype=P.RESULT_DTYPE)
    idx.admit_host_u16(s.tokens.astype(np.uint16), s.offsets, s.users, None, out=out)
    o = Oracle(16, SEED, POL["solidarity"])
    o.reserve(s.n_blocks())
    _same(out, o.process(s), idx.dump(), o.dump(), "host pieces")
    assert idx.stats()["batches"] == 1


@pytest.mark.parametrize("policy", ["solidarity", "apc"])
@pytest.mark.parametrize("batch", [1, 7, 1000])
def test_deep_jacobi_streams(policy, batch):
    import torch
    import paper_2603_10726_b200 as P
    for s in _deep_streams():
        o = Oracle(16, SEED, POL[policy])
        exp = o.process(s)
        idx = P.Index(policy, capacity_blocks=1024, max_batch_tokens=s.n_tokens + 64,
                      max_batch_requests=s.n_requests, seed=SEED)
        got = np.concatenate([P.as_numpy(idx.admit(**P.to_device(s.slice(i, min(i + batch,
                                                                                s.n_requests)))))
                              for i in range(0, s.n_requests, batch)])
        torch.cuda.synchronize()
        _same(got, exp, idx.dump(), o.dump(), s.name)


@pytest.mark.parametrize("limit", [2, 3, 5])
def test_round_limit_splits_the_batch(limit):
    """With the resolver limited to `limit` rounds the deep streams and a C2-shaped stream (4
    rounds) cannot converge in one piece: the synchronous admission commits them in parts, and
    the results and index still equal the oracle's."""
    import torch
    import paper_2603_10726_b200 as P
    streams = _deep_streams() + [c2_shared_prompt(users=30, reqs_per_user=20)]
    for s in streams:
        o = Oracle(16, SEED, POL["solidarity"])
        exp = o.process(s)
        idx = P.Index("solidarity", capacity_blocks=max(4 * s.n_blocks(), 1024),
                      max_batch_tokens=s.n_tokens + 64, max_batch_requests=s.n_requests,
                      seed=SEED)
        idx.debug_set_max_rounds(limit)
        got = P.as_numpy(idx.admit(**P.to_device(s)))
        torch.cuda.synchronize()
        _same(got, exp, idx.dump(), o.dump(), f"{s.name} limit {limit}")
        # through host buffers too (admit_host splits the same way)
        idx.reset()
        out = np.zeros(s.n_requests, dtype=P.RESULT_DTYPE)
        idx.admit_host(s.tokens, s.offsets, s.users, s.enforce, out=out)
        _same(out, exp, idx.dump(), o.dump(), f"{s.name} host limit {limit}")
        # the asynchronous path cannot split: a batch that does not converge fails whole with
        # SOLID_ERR_STATE and commits nothing; one that converges matches the oracle
        idx.reset()
        o2 = idx.admit_async(**P.to_device(s))
        try:
            idx.status()
        except P.SolidError as e:
            assert e.status == P.SOLID_ERR_STATE
            assert len(idx.dump()) == 0
        else:
            _same(P.as_numpy(o2), exp, idx.dump(), o.dump(), f"{s.name} async limit {limit}")
