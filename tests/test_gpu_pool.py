"""GPU parity of physical block ids and block tables (R26-R28):
the CUDA path through the C ABI against the oracle's FIFO pool, bit-exact on every block-table
entry of every batch and on every live entry's physical block, with and without LRU eviction,
for all policies and batch partitions."""
import numpy as np
import pytest

from oracle import Oracle
from workloads import c1_tiny, c3_multiturn, random_small

pytestmark = pytest.mark.gpu
SEED = 0x5011D000
POL = {"apc": 0, "user_isolation": 1, "solidarity": 2}
NONE = 0xFFFFFFFF


def _index(policy, streams, capacity, max_blocks, evict):
    import paper_2603_10726_b200 as P
    tok = max(max(s.n_tokens for s in streams), 64)
    req = max(max(s.n_requests for s in streams), 1)
    return P.Index(policy, capacity_blocks=capacity, max_batch_tokens=tok + 64,
                   max_batch_requests=req, max_blocks=max_blocks, seed=SEED, evict=evict,
                   block_table=True)


def _rows_equal(got, exp, s, what):
    """Covered positions (each request's full blocks) must match; others are not written.
    Returns the number of NONE entries in the covered rows."""
    offs = s.offsets.astype(np.int64)
    nones = 0
    for j in range(s.n_requests):
        a, n = offs[j] // 16, (offs[j + 1] - offs[j]) // 16
        if n and not np.array_equal(got[a:a + n], exp[a:a + n]):
            raise AssertionError((what, j, got[a:a + n], exp[a:a + n]))
        nones += int((exp[a:a + n] == NONE).sum())
    return nones


def admit_compare(idx, o, s, what, splits=None):
    """Admit s on the GPU (split on SOLID_ERR_CAPACITY in evict mode), the same sub-batches on
    the oracle; compare results and block tables.  Returns the NONE entries seen."""
    import torch
    import paper_2603_10726_b200 as P
    try:
        got = P.as_numpy(idx.admit(**P.to_device(s)))
        torch.cuda.synchronize()
    except P.SolidError as e:
        if e.status != P.SOLID_ERR_CAPACITY or s.n_requests < 2 or splits is None:
            raise
        splits.append(s.n_requests)
        h = s.n_requests // 2
        return (admit_compare(idx, o, s.slice(0, h), what, splits) +
                admit_compare(idx, o, s.slice(h, s.n_requests), what, splits))
    exp = o.process(s)
    assert np.array_equal(got, exp), what
    if s.n_requests == 0:
        return 0
    bt = idx.block_table(s.n_tokens).cpu().numpy().view(np.uint32)
    return _rows_equal(bt, o.block_table(), s, what)


def final_compare(idx, o):
    gk, gp = idx.dump_phys()
    ek, ep = o.dump_phys()
    assert np.array_equal(gk, ek) and np.array_equal(gp, ep)
    assert len(set(gp.tolist())) == len(gp)


@pytest.mark.parametrize("policy", list(POL))
@pytest.mark.parametrize("batch", [1, 9, 64, 1000])
def test_no_eviction(policy, batch):
    for seed in (1, 2):
        s = random_small(300, users=1 + seed, alphabet_blocks=3, max_blocks=6, seed=seed,
                         enforce_prob=0.8)
        parts = [s.slice(i, min(i + batch, 300)) for i in range(0, 300, batch)]
        cap = 4096
        idx = _index(policy, parts, cap, 8, False)
        o = Oracle(16, SEED, POL[policy], pool=cap)
        for k, b in enumerate(parts):
            admit_compare(idx, o, b, f"{policy}/{batch}/{k}")
        final_compare(idx, o)


@pytest.mark.parametrize("policy", list(POL))
@pytest.mark.parametrize("capacity", [8, 13, 40])
@pytest.mark.parametrize("batch", [1, 7, 64, 1000])
def test_lru_eviction(policy, capacity, batch):
    for seed in (1, 2, 3):
        s = random_small(300, users=1 + seed, alphabet_blocks=3, max_blocks=6, seed=seed,
                         enforce_prob=0.8 if seed % 2 else 1.0)
        parts = [s.slice(i, min(i + batch, 300)) for i in range(0, 300, batch)]
        idx = _index(policy, parts, capacity, 8, True)
        o = Oracle(16, SEED, POL[policy], capacity=capacity, pool=capacity)
        for k, b in enumerate(parts):
            admit_compare(idx, o, b, f"{policy}/{capacity}/{batch}/{k}", [])
        final_compare(idx, o)
        assert o.evictions() > 0


@pytest.mark.parametrize("policy", ["apc", "solidarity"])
def test_multiturn_under_pressure(policy):
    """Window keys (revisited entries the batch evicts) in the block tables."""
    warm, timed = c3_multiturn(users=60, warm_blocks=3000, timed_rounds=6, seed=11)
    cap = 1500
    parts = [warm.slice(i, min(i + 60, warm.n_requests)) for i in range(0, warm.n_requests, 60)]
    parts += [timed.slice(i, min(i + 60, timed.n_requests)) for i in range(0, timed.n_requests, 60)]
    idx = _index(policy, parts, cap, 512, True)
    o = Oracle(16, SEED, POL[policy], capacity=cap, pool=cap)
    for k, b in enumerate(parts):
        admit_compare(idx, o, b, f"{policy}/{k}", [])
    final_compare(idx, o)
    assert idx.stats()["window_evicted"] > 0


def test_rebuild_keeps_blocks():
    """Many batches through a small cache: table rebuilds move the physical ids with the slots."""
    s = random_small(60000, users=6, alphabet_blocks=400, max_blocks=6, seed=9)
    cap = 600
    parts = [s.slice(i, min(i + 600, s.n_requests)) for i in range(0, s.n_requests, 600)]
    idx = _index("solidarity", parts, cap, 8, True)
    o = Oracle(16, SEED, 2, capacity=cap, pool=cap)
    for k, b in enumerate(parts):
        admit_compare(idx, o, b, f"rebuild/{k}", [])
    final_compare(idx, o)
    assert idx.stats()["rebuilds"] >= 1


def test_host_admission_and_checkpoint():
    """admit_host (one chunk when the pool is on), checkpoint / restore and reset."""
    import torch
    import paper_2603_10726_b200 as P
    s = c1_tiny()
    a, b = s.slice(0, 32), s.slice(32, s.n_requests)
    idx = _index("solidarity", [s], 4096, 64, False)
    o = Oracle(16, SEED, 2, pool=4096)
    got = idx.admit_host(a.tokens, a.offsets, a.users, a.enforce)
    assert np.array_equal(got, o.process(a))
    d = P.to_device(a)       # block table of the host batch: positions from its own offsets
    bt = idx.block_table(a.n_tokens).cpu().numpy().view(np.uint32)
    _rows_equal(bt, o.block_table(), a, "host")
    idx.checkpoint()
    r1 = P.as_numpy(idx.admit(**P.to_device(b)))
    t1 = idx.block_table(b.n_tokens).cpu().numpy().view(np.uint32)
    idx.restore()
    r2 = P.as_numpy(idx.admit(**P.to_device(b)))
    t2 = idx.block_table(b.n_tokens).cpu().numpy().view(np.uint32)
    torch.cuda.synchronize()
    assert np.array_equal(r1, r2)
    _rows_equal(t2, t1, b, "restore")
    assert np.array_equal(r1, o.process(b))
    _rows_equal(t1, o.block_table(), b, "after checkpoint")
    final_compare(idx, o)
    idx.reset()
    o2 = Oracle(16, SEED, 2, pool=4096)
    admit_compare(idx, o2, s, "after reset")
    del d


def test_pool_refusals():
    import paper_2603_10726_b200 as P
    with pytest.raises(P.SolidError):
        P.Index("apc", capacity_blocks=64, world=2, rank=0, block_table=True)
    idx = P.Index("apc", capacity_blocks=64, max_batch_tokens=1 << 12, max_batch_requests=64,
                  max_blocks=8, block_table=True)
    with pytest.raises(P.SolidError):
        idx.block_table(16)                          # nothing committed yet
    s = random_small(10, users=2, alphabet_blocks=3, max_blocks=4, seed=1)
    # solid_admit_batch on a block-table context: admitted at submission, collected in order
    r1 = P.as_numpy(idx.admit_async(**P.to_device(s))).copy()
    idx.status()
    t1 = idx.block_table(s.n_tokens).cpu().numpy()
    idx.reset()
    r2 = P.as_numpy(idx.admit(**P.to_device(s)))
    assert np.array_equal(r1, r2)
    assert np.array_equal(t1, idx.block_table(s.n_tokens).cpu().numpy())
    plain = P.Index("apc", capacity_blocks=64, max_batch_tokens=1 << 12, max_batch_requests=64,
                    max_blocks=8)
    plain.admit(**P.to_device(s))
    with pytest.raises(P.SolidError):
        plain.block_table(s.n_tokens)


def test_none_rows_are_exercised():
    """Batches whose own evictions remove entries their requests referenced without being served
    them: those rows hold NONE on both sides (and match)."""
    nones = 0
    for seed in (1, 2, 3):
        s = random_small(300, users=1 + seed, alphabet_blocks=3, max_blocks=6, seed=seed,
                         enforce_prob=0.8)
        for cap in (8, 13):
            idx = _index("solidarity", [s], cap, 8, True)
            o = Oracle(16, SEED, 2, capacity=cap, pool=cap)
            nones += admit_compare(idx, o, s, "none-rows", [])
            final_compare(idx, o)
    assert nones > 0
