"""C5 — the large index (BASELINE.json configs[4]; workloads/c5.py).

* reduced scale (0.1: 20 000 users, ~1.1e7 warm entries, a 400 000-request timed batch): the
  CUDA path against the oracle, every result field and the whole index;
* full scale on ONE GPU (200 000 users, ~1.02e8 warm entries, ONE 4 000 000-request batch of
  4.2e9 tokens): the per-request values C5's structure fixes (tests/c5_props.py: continuing
  conversations reuse their cached prefix, new sessions divert at the flagged system prompt,
  no probe is ever served beyond the system prompt — the §5 guarantee) for every request, and
  R1 at full size: the same batch admitted as 4 consecutive parts gives identical results
  and an identical index;
* the sharded protocol (loopback, G = 8 shards on one GPU) at reduced scale against the oracle.
A full-size oracle comparison runs with SOLID_C5_ORACLE=1 (host RAM ~40 GB, ~3 min).
"""
import os

import numpy as np
import pytest

from c5_props import c5_check
from oracle import Oracle
from workloads.c5 import c5_large

pytestmark = pytest.mark.gpu
SEED = 0x5011D000


def _same(got, exp, gd, ed, what=""):
    for f in exp.dtype.names:
        bad = np.nonzero(got[f].astype(np.int64) != exp[f].astype(np.int64))[0]
        assert bad.size == 0, (what, f, int(bad[0]), got[bad[0]], exp[bad[0]])
    assert len(gd) == len(ed), (what, len(gd), len(ed))
    for f in ["key", "owner", "sharer"]:
        bad = np.nonzero(gd[f] != ed[f])[0]
        assert bad.size == 0, (what, "dump", f, int(bad[0]))


def _index(warm, timed, **kw):
    import paper_2603_10726_b200 as P
    cap = warm.n_blocks() + timed.n_blocks() // 4 + (1 << 16)
    return P.Index("solidarity", capacity_blocks=cap,
                   max_batch_tokens=max(warm.n_tokens, timed.n_tokens) + 64,
                   max_batch_requests=max(warm.n_requests, timed.n_requests), seed=SEED,
                   max_blocks=1024, **kw)


def _admit_dev(idx, seg, asynchronous=False):
    import torch
    import paper_2603_10726_b200 as P
    t, o, u = seg.materialize_torch("cuda")
    out = torch.empty((seg.n_requests, 6), dtype=torch.int32, device="cuda")
    if asynchronous:
        idx.admit_async(t, o, u, None, out=out)
        idx.status()
    else:
        idx.admit(t, o, u, None, out=out)
    torch.cuda.synchronize()
    del t, o, u
    return P.as_numpy(out)


def _oracle(warm, timed):
    o = Oracle(16, SEED, 2)
    o.reserve(int((warm.n_blocks() + timed.n_blocks()) * 0.7))
    o.process(warm.materialize())
    return o.process(timed.materialize()), o.dump()


def test_c5_reduced_scale_oracle_parity():
    warm, timed = c5_large(scale=0.1)
    idx = _index(warm, timed)
    _admit_dev(idx, warm)
    st = idx.stats()
    assert st["live_entries"] >= 10_000_000
    got = _admit_dev(idx, timed, asynchronous=True)
    exp, ed = _oracle(warm, timed)
    _same(got, exp, idx.dump(), ed, "c5 x0.1")
    assert c5_check(timed, got)["status"] == "exact"


def test_c5_full_size_single_gpu():
    """One B200 holds C5: the warm index of ~1.06e8 entries and the 4e6-request
    batch; exact per-request properties and R1 (4 consecutive parts) at full size."""
    import torch
    warm, timed = c5_large(scale=1.0)
    idx = _index(warm, timed)
    _admit_dev(idx, warm)
    live0 = idx.stats()["live_entries"]
    assert live0 >= 100_000_000, live0
    idx.checkpoint()
    got = _admit_dev(idx, timed, asynchronous=True)
    st = idx.stats()
    chk = c5_check(timed, got)
    assert chk["status"] == "exact", chk
    assert chk["counts"] == (2_000_000, 1_600_000, 400_000)
    d_one = idx.dump()
    assert len(d_one) == live0 + st["last_inserted"]
    # R1: the same batch as 4 consecutive parts
    idx.restore()
    t, o, u = timed.materialize_torch("cuda")
    out = torch.empty((timed.n_requests, 6), dtype=torch.int32, device="cuda")
    n = timed.n_requests
    cuts = [n * k // 4 for k in range(5)]
    import paper_2603_10726_b200 as P
    for a, b in zip(cuts[:-1], cuts[1:]):
        oo = o[a:b + 1] - o[a]
        tt = t[int(o[a]):int(o[b])]
        idx.admit(tt, oo, u[a:b], None, out=out[a:b])
    torch.cuda.synchronize()
    parts = P.as_numpy(out)
    assert all(np.array_equal(parts[f], got[f]) for f in got.dtype.names)
    d_parts = idx.dump()
    assert all(np.array_equal(d_parts[f], d_one[f]) for f in ["key", "owner", "sharer"])


@pytest.mark.skipif(os.environ.get("SOLID_C5_ORACLE") != "1",
                    reason="full-size C5 oracle comparison: set SOLID_C5_ORACLE=1 (~40 GB host RAM)")
def test_c5_full_size_oracle_parity():
    warm, timed = c5_large(scale=1.0)
    idx = _index(warm, timed)
    _admit_dev(idx, warm)
    got = _admit_dev(idx, timed, asynchronous=True)
    gd = idx.dump()
    del idx
    exp, ed = _oracle(warm, timed)
    _same(got, exp, gd, ed, "c5 full")


def test_c5_sharded_loopback_eight_shards():
    """The sharded protocol with G = 8 shards (loopback transport, one GPU) on C5 at scale 0.02:
    warm batch then timed batch, results and the union of the shards equal the oracle."""
    import torch
    import paper_2603_10726_b200 as P
    from paper_2603_10726_b200.dist import ShardedIndex, loopback_admit
    warm, timed = c5_large(scale=0.02)
    G = 8
    ws, ts = warm.materialize(), timed.materialize()
    cap = (warm.n_blocks() + timed.n_blocks()) // 4 + 4096
    shards = [ShardedIndex(G, r, "solidarity", capacity_blocks=cap,
                           max_batch_tokens=max(ws.n_tokens, ts.n_tokens) // 4 + 65536,
                           max_batch_requests=ts.n_requests // 4 + 1024, seed=SEED,
                           max_blocks=1024)
              for r in range(G)]
    out, seq = [], 0
    for s in (ws, ts):
        n = s.n_requests
        cuts = [n * r // G for r in range(G + 1)]
        parts = [s.slice(cuts[r], cuts[r + 1]) for r in range(G)]
        res, _t = loopback_admit(shards, [P.to_device(p) for p in parts],
                                 [seq + c for c in cuts[:-1]])
        torch.cuda.synchronize()
        out.append(np.concatenate([P.as_numpy(r) for r in res]))
        seq += n
    merged = np.concatenate([sh.index.dump() for sh in shards])
    merged = merged[np.argsort(merged["key"], kind="stable")]
    o = Oracle(16, SEED, 2)
    exp = np.concatenate([o.process(ws), o.process(ts)])
    _same(np.concatenate(out), exp, merged, o.dump(), "c5 x0.02 G=8")
