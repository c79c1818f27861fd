"""GPU parity: the CUDA path (through the C ABI) against the sequential oracle, element by element,
on identical seeded streams.  Bar: bit-exact on every result field and on the final index
(key, owner, sharer), for every policy, any batch partition (R1), any token alignment."""
import numpy as np
import pytest

from oracle import Oracle
from oracle_helpers import NONE
from workloads import (c1_tiny, c2_shared_prompt, c3_multiturn, c4_attackers, random_small,
                       concat_streams)

pytestmark = pytest.mark.gpu
SEED = 0x5011D000
POL = {"apc": 0, "user_isolation": 1, "solidarity": 2}


def _index(policy, stream_list, capacity=None, **kw):
    import paper_2603_10726_b200 as P
    tok = max(max(s.n_tokens for s in stream_list), 64)
    req = max(max(s.n_requests for s in stream_list), 1)
    blocks = sum(s.n_blocks() for s in stream_list)
    return P.Index(policy, capacity_blocks=capacity or max(4 * blocks, 1024),
                   max_batch_tokens=tok + 64, max_batch_requests=req, seed=SEED, **kw)


def _admit(idx, s, shift=0):
    import torch
    import paper_2603_10726_b200 as P
    d = P.to_device(s)
    if shift:
        t = torch.zeros(d["tokens"].numel() + 4, dtype=torch.int32, device="cuda")
        t[shift:shift + d["tokens"].numel()] = d["tokens"]
        d["tokens"] = t[shift:]
    out = idx.admit(**d)
    torch.cuda.synchronize()
    return P.as_numpy(out)


def gpu_run(streams, policy, shift=0, idx=None):
    if not isinstance(streams, list):
        streams = [streams]
    idx = idx or _index(policy, streams)
    res = [_admit(idx, s, shift) for s in streams]
    return np.concatenate(res) if res else np.zeros(0), idx.dump(), idx


def oracle_run(streams, policy):
    if not isinstance(streams, list):
        streams = [streams]
    o = Oracle(16, SEED, POL[policy])
    o.reserve(sum(s.n_blocks() for s in streams) + 16)
    res = [o.process(s) for s in streams]
    return np.concatenate(res), o.dump()


def assert_same(got, exp, gdump, edump, what=""):
    assert got.shape == exp.shape, what
    for f in exp.dtype.names:
        g = got[f].astype(np.int64)
        e = exp[f].astype(np.int64)
        bad = np.nonzero(g != e)[0]
        assert bad.size == 0, (what, f, int(bad[0]), int(g[bad[0]]), int(e[bad[0]]),
                               got[bad[0]], exp[bad[0]])
    assert len(gdump) == len(edump), (what, len(gdump), len(edump))
    for f in ["key", "owner", "sharer"]:
        bad = np.nonzero(gdump[f] != edump[f])[0]
        assert bad.size == 0, (what, "dump", f, int(bad[0]), gdump[bad[0]], edump[bad[0]])


def _batches(s, size):
    return [s.slice(i, min(i + size, s.n_requests)) for i in range(0, s.n_requests, size)]


@pytest.mark.parametrize("policy", list(POL))
def test_c1_tiny(policy):
    s = c1_tiny()
    exp, ed = oracle_run(s, policy)
    got, gd, _ = gpu_run(s, policy)
    assert_same(got, exp, gd, ed, "c1")


@pytest.mark.parametrize("policy", list(POL))
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_random_streams(policy, seed):
    s = random_small(400, users=int(1 + seed % 5), alphabet_blocks=3, max_blocks=40, seed=seed,
                     enforce_prob=0.7 if seed % 2 else 1.0)
    exp, ed = oracle_run(s, policy)
    got, gd, _ = gpu_run(s, policy)
    assert_same(got, exp, gd, ed, f"random{seed}")


@pytest.mark.parametrize("size", [1, 7, 64, 1000])
def test_batch_partition_invariance(size):
    """R1: cutting the stream into batches of any size gives the same results and index."""
    s = random_small(300, users=4, alphabet_blocks=3, max_blocks=12, seed=11)
    exp, ed = oracle_run(s, "solidarity")
    got, gd, _ = gpu_run(_batches(s, size), "solidarity")
    assert_same(got, exp, gd, ed, f"batch{size}")


@pytest.mark.parametrize("shift", [1, 2, 3])
def test_unaligned_token_buffers(shift):
    s = c1_tiny()
    exp, ed = oracle_run(s, "solidarity")
    got, gd, _ = gpu_run(s, "solidarity", shift=shift)
    assert_same(got, exp, gd, ed, f"shift{shift}")


def test_empty_and_degenerate_requests():
    prompts = [np.zeros(0, np.uint32), np.arange(15, dtype=np.uint32),
               np.arange(16, dtype=np.uint32), np.arange(16, dtype=np.uint32),
               np.arange(33, dtype=np.uint32), np.zeros(0, np.uint32),
               np.full(16 * 40 + 3, (1 << 20) - 1, np.uint32), np.zeros(16 * 40, np.uint32)]
    from workloads.gen import _pack
    s = _pack("degenerate", prompts, [0, 1, 2, 3, 0, 1, 2, 3])
    for policy in POL:
        exp, ed = oracle_run(s, policy)
        got, gd, _ = gpu_run(s, policy)
        assert_same(got, exp, gd, ed, f"degenerate-{policy}")


def test_max_blocks_boundary():
    """A request of exactly max_blocks full blocks (plus a tail) is admitted and matches the
    oracle; one block more is SOLID_ERR_INVALID with the index untouched."""
    import paper_2603_10726_b200 as P
    from workloads.gen import _pack, run
    mb = 64
    ok = [run(1, 5, i, 16 * mb + 7) for i in range(3)] + [run(1, 5, 0, 16 * mb)]
    s = _pack("maxb", ok, [0, 1, 2, 1])
    idx = P.Index("solidarity", capacity_blocks=1 << 12, max_batch_tokens=1 << 16,
                  max_batch_requests=16, max_blocks=mb, seed=SEED)
    got = _admit(idx, s)
    exp, ed = oracle_run(s, "solidarity")
    assert_same(got, exp, idx.dump(), ed, "max_blocks")
    before = idx.dump()
    bad = _pack("over", [run(1, 6, 0, 16 * (mb + 1))], [3])
    with pytest.raises(P.SolidError) as ei:
        _admit(idx, bad)
    assert ei.value.status == P.SOLID_ERR_INVALID
    assert (idx.dump() == before).all()


def test_empty_batch():
    import torch
    import paper_2603_10726_b200 as P
    idx = P.Index("solidarity", capacity_blocks=1024, max_batch_tokens=1024,
                  max_batch_requests=16)
    z = torch.zeros(4, dtype=torch.int32, device="cuda")
    out = idx.admit(z, torch.zeros(1, dtype=torch.int64, device="cuda"),
                    torch.zeros(0, dtype=torch.int32, device="cuda"))
    assert out.shape[0] == 0 and len(idx.dump()) == 0


def test_invalid_batches_leave_the_index_untouched():
    import torch
    import paper_2603_10726_b200 as P
    s = random_small(50, users=3, alphabet_blocks=3, max_blocks=8, seed=3)
    idx = _index("solidarity", [s])
    _admit(idx, s)
    before = idx.dump()
    bad = s.slice(0, 10)
    bad.tokens = bad.tokens.copy()
    bad.tokens[5] = 1 << 20
    with pytest.raises(P.SolidError) as ei:
        _admit(idx, bad)
    assert ei.value.status == P.SOLID_ERR_INVALID
    bad2 = s.slice(0, 10)
    bad2.users = bad2.users.copy()
    bad2.users[3] = NONE
    with pytest.raises(P.SolidError):
        _admit(idx, bad2)
    after = idx.dump()
    assert (before == after).all()
    # the index still works and matches the oracle afterwards
    exp, ed = oracle_run([s, s.slice(0, 20)], "solidarity")
    got = _admit(idx, s.slice(0, 20))
    assert (got["reused"] == exp[len(s.users):]["reused"]).all()
    d = P.to_device(s.slice(0, 5))
    idx.lookup(**d)
    with pytest.raises(P.SolidError) as ei:
        idx.lookup(**d)
    assert ei.value.status == P.SOLID_ERR_STATE
    idx.insert()


def test_capacity_overflow_is_all_or_nothing():
    import paper_2603_10726_b200 as P
    s = random_small(60, users=3, alphabet_blocks=50, max_blocks=10, seed=9)
    idx = _index("apc", [s], capacity=s.n_blocks() // 3)
    with pytest.raises(P.SolidError) as ei:
        _admit(idx, s)
    assert ei.value.status == P.SOLID_ERR_CAPACITY
    assert len(idx.dump()) == 0
    small = s.slice(0, 3)
    exp, ed = oracle_run(small, "apc")
    got = _admit(idx, small)
    assert (got["reused"] == exp["reused"]).all() and len(idx.dump()) == len(ed)


def test_async_admission_matches_and_rolls_back_on_device():
    """solid_admit_batch: up to MAX_INFLIGHT batches queued with no host sync in between, collected
    oldest first; results and index match the oracle.  An over-capacity batch is rolled back on
    the device, reported by its own solid_batch_status, and the batches queued behind it see the
    index without it."""
    import torch
    import paper_2603_10726_b200 as P
    s = c2_shared_prompt(users=40, reqs_per_user=25)
    parts = _batches(s, 120)
    exp, ed = oracle_run(parts, "solidarity")
    idx = _index("solidarity", parts)
    dev = [P.to_device(p) for p in parts]
    outs, inflight = [], 0
    for d in dev:
        if inflight == P.MAX_INFLIGHT:
            with pytest.raises(P.SolidError) as ei:
                idx.admit_async(**d)
            assert ei.value.status == P.SOLID_ERR_STATE
            idx.status()
            inflight -= 1
        outs.append(idx.admit_async(**d))
        inflight += 1
    with pytest.raises(P.SolidError):
        idx.dump()                         # outstanding batches must be collected first
    for _ in range(inflight):
        idx.status()
    idx.status()                           # none outstanding: no-op
    got = np.concatenate([P.as_numpy(o) for o in outs])
    assert_same(got, exp, idx.dump(), ed, "async")
    st = idx.stats()
    assert st["batches"] == len(parts) and st["live_entries"] == len(ed)

    # [small, too-big, small2] queued together: the middle one rolls back on the device
    r = random_small(60, users=3, alphabet_blocks=50, max_blocks=10, seed=9)
    small, small2 = r.slice(0, 3), r.slice(3, 6)
    e1, ed1 = oracle_run([small, small2], "apc")
    idx2 = _index("apc", [r], capacity=r.n_blocks() // 3)
    o1 = idx2.admit_async(**P.to_device(small))
    idx2.admit_async(**P.to_device(r))
    o3 = idx2.admit_async(**P.to_device(small2))
    idx2.status()
    with pytest.raises(P.SolidError) as ei:
        idx2.status()
    assert ei.value.status == P.SOLID_ERR_CAPACITY
    idx2.status()
    got = np.concatenate([P.as_numpy(o1), P.as_numpy(o3)])
    assert_same(got, e1, idx2.dump(), ed1, "async rollback in the middle")
    assert idx2.stats()["live_entries"] == len(ed1)


def test_reset_with_batches_in_flight():
    """solid_reset behind outstanding batches is stream-ordered: the next batch sees an empty
    index; the older batches still report their status."""
    import paper_2603_10726_b200 as P
    s = c1_tiny()
    exp, ed = oracle_run(s, "solidarity")
    idx = _index("solidarity", [s])
    d = P.to_device(s)
    idx.admit_async(**d)
    idx.reset()
    out = idx.admit_async(**d)
    idx.status()
    idx.status()
    assert_same(P.as_numpy(out), exp, idx.dump(), ed, "reset in flight")
    st = idx.stats()
    assert st["batches"] == 1 and st["live_entries"] == len(ed)


def test_host_buffer_admission_matches():
    s = c1_tiny()
    exp, ed = oracle_run(s, "solidarity")
    idx = _index("solidarity", [s])
    got = idx.admit_host(s.tokens, s.offsets, s.users, s.enforce)
    assert_same(got, exp, idx.dump(), ed, "admit_host")


@pytest.mark.parametrize("name", ["c1", "c2_small", "random"])
def test_host_buffer_admission_u16_matches(name):
    """solid_admit_host_u16: 16-bit token ids widened on the device give the oracle's results
    (ragged token counts, so the widening tail is exercised)."""
    s = {"c1": c1_tiny, "c2_small": lambda: c2_shared_prompt(users=40, reqs_per_user=10),
         "random": lambda: random_small(301, users=3, alphabet_blocks=4, max_blocks=6, seed=3)}[name]()
    assert int(s.tokens.max()) < 65536
    exp, ed = oracle_run(s, "solidarity")
    idx = _index("solidarity", [s])
    got = idx.admit_host_u16(s.tokens.astype(np.uint16), s.offsets, s.users, s.enforce)
    assert_same(got, exp, idx.dump(), ed, "admit_host_u16")


@pytest.mark.parametrize("u16", [False, True])
def test_host_buffer_admission_chunked_pipeline(u16):
    """Batches with >= 64 MB of token ids are copied in 4 pieces whose hashing starts as each
    piece arrives; the batch is still ONE admission (all or nothing): same results and index
    as the oracle."""
    s = c2_shared_prompt(users=170, reqs_per_user=100)
    assert s.n_tokens * (2 if u16 else 4) >= 64 << 20
    exp, ed = oracle_run(s, "solidarity")
    idx = _index("solidarity", [s])
    if u16:
        got = idx.admit_host_u16(s.tokens.astype(np.uint16), s.offsets, s.users, s.enforce)
    else:
        got = idx.admit_host(s.tokens, s.offsets, s.users, s.enforce)
    assert_same(got, exp, idx.dump(), ed, "chunked admit_host")
    assert idx.stats()["batches"] == 1


@pytest.mark.parametrize("policy", ["apc", "user_isolation", "solidarity"])
def test_block_keys_table(policy):
    """solid_block_keys: per block, the key of the entry that holds its KV — the oracle's chain
    keys with the request's own divert depth (Shared, isolated from f, or U under isolation)."""
    import torch
    s = concat_streams("bk", [c1_tiny(), random_small(200, users=3, alphabet_blocks=4,
                                                       max_blocks=6, seed=2)])
    idx = _index(policy, [s])
    res = _admit(idx, s)
    keys = idx.block_keys(s.n_tokens).cpu().numpy().view(np.uint64)
    torch.cuda.synchronize()
    o = Oracle(16, SEED, POL[policy])
    exp = o.process(s)
    assert np.array_equal(res, exp)
    for j in range(s.n_requests):
        o0, o1 = int(s.offsets[j]), int(s.offsets[j + 1])
        f = int(exp["divert_at"][j])
        _, K = o.chain(s.tokens[o0:o1], int(s.users[j]), f)
        n = int(exp["n_blocks"][j])
        assert np.array_equal(keys[o0 // 16:o0 // 16 + n], K[:n]), j


@pytest.mark.parametrize("evict", [False, True])
def test_scratch_epoch_restart(evict):
    """The batch-scratch tag space restarts after ~2^20 batches (a long-running server crosses
    it): batches admitted across the restart still match the oracle, with and without LRU."""
    import torch
    import paper_2603_10726_b200 as P
    s = random_small(300, users=3, alphabet_blocks=4, max_blocks=6, seed=6)
    cap = 40 if evict else 1 << 12
    idx = P.Index("solidarity", capacity_blocks=cap, max_batch_tokens=1 << 16,
                  max_batch_requests=64, max_blocks=8, seed=SEED, evict=evict)
    kmax = 0xFFFFFFFF // 4096 - 1
    idx.debug_set_epoch(kmax - 3)
    got = []
    for lo in range(0, 300, 30):
        b = s.slice(lo, lo + 30)
        try:
            got.append(P.as_numpy(idx.admit(**P.to_device(b))))
        except P.SolidError as e:             # evict: a batch that must split
            assert evict and e.status == P.SOLID_ERR_CAPACITY
            got += [P.as_numpy(idx.admit(**P.to_device(b.slice(q, q + 1)))) for q in range(30)]
    torch.cuda.synchronize()
    o = Oracle(16, SEED, 2, capacity=cap if evict else 0)
    assert np.array_equal(np.concatenate(got), o.process(s))
    gd = idx.dump_ex() if evict else idx.dump()
    ed = o.dump_ex() if evict else o.dump()
    assert all(np.array_equal(gd[f], ed[f]) for f in ed.dtype.names)


def test_stats_are_consistent():
    s = c1_tiny()
    got, gd, idx = gpu_run(s, "solidarity")
    st = idx.stats()
    assert st["inserted"] == len(gd) == st["live_entries"]
    assert st["blocks"] == int(got["n_blocks"].sum())
    assert st["reused_blocks"] == int(got["reused"].sum())
    assert st["last_rounds"] >= 2
    assert st["flagged"] == int(((got["bits"] & 16) > 0).sum())


@pytest.mark.parametrize("policy", list(POL))
def test_c2_small(policy):
    s = c2_shared_prompt(users=40, reqs_per_user=25)
    exp, ed = oracle_run(s, policy)
    got, gd, _ = gpu_run(s, policy)
    assert_same(got, exp, gd, ed, "c2small")


def test_c3_small_warm_then_timed():
    warm, timed = c3_multiturn(users=300, warm_blocks=30000, timed_rounds=3)
    exp, ed = oracle_run([warm, timed], "solidarity")
    got, gd, _ = gpu_run([warm] + _batches(timed, 300), "solidarity")
    assert_same(got, exp, gd, ed, "c3small")


def test_c4_small():
    s = c4_attackers(benign_users=300, benign_requests=6000, victims=6, templates=3,
                     candidates=30)
    exp, ed = oracle_run(s, "solidarity")
    got, gd, _ = gpu_run(_batches(s, 2500), "solidarity")
    assert_same(got, exp, gd, ed, "c4small")


def test_c2_full_size_bench_configuration():
    """BASELINE configs[1] at full size (100 000 requests, 12.5 M blocks), one batch, exactly as
    bench.py launches it: every result and every index entry against the oracle."""
    s = c2_shared_prompt()
    exp, ed = oracle_run(s, "solidarity")
    got, gd, idx = gpu_run(s, "solidarity")
    assert_same(got, exp, gd, ed, "c2full")


def test_c3_full_size_warm_then_timed():
    """BASELINE configs[2] at full size: 10 000 users, conversations to 8 k tokens, warm phase
    (~3 M cached blocks) then the timed rounds as one 80 000-request batch."""
    warm, timed = c3_multiturn()
    exp, ed = oracle_run([warm, timed], "solidarity")
    got, gd, _ = gpu_run([warm, timed], "solidarity")
    assert_same(got, exp, gd, ed, "c3full")


def test_c4_full_size():
    """BASELINE configs[3] at full size: 500 k benign requests + 100 victims x 10 + 1 000
    colluding attackers x 500 probes, isolation-heavy, one batch."""
    s = c4_attackers()
    exp, ed = oracle_run(s, "solidarity")
    got, gd, _ = gpu_run(s, "solidarity")
    assert_same(got, exp, gd, ed, "c4full")
