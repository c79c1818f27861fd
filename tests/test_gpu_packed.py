"""The packed K_A (csrc/solid_pack.inc: lanes packed across request boundaries, segmented chain
scan) against the warp-per-request K_A and the oracle: identical results, identical final index,
for every policy, one- and two-component keys, aligned and misaligned token buffers, empty and
sub-block requests, zero-block requests inside a warp's span, and batches large enough that
several warps and CTAs share the packed block space."""
import os

import numpy as np
import pytest

from oracle import Oracle
from workloads import c4_attackers, random_small
from workloads.gen import _pack, run

pytestmark = pytest.mark.gpu
SEED = 0x5011D000
POL = {"apc": 0, "user_isolation": 1, "solidarity": 2}


def _run(s, policy, pack, shift=0, nc=1):
    import torch
    import paper_2603_10726_b200 as P
    old = os.environ.get("SOLID_PACK")
    os.environ["SOLID_PACK"] = "1" if pack else "0"
    try:
        idx = P.Index(policy, capacity_blocks=max(4 * s.n_blocks(), 4096),
                      max_batch_tokens=s.n_tokens + 128, max_batch_requests=max(s.n_requests, 1),
                      seed=SEED, hash_components=nc)
    finally:
        if old is None:
            os.environ.pop("SOLID_PACK")
        else:
            os.environ["SOLID_PACK"] = old
    d = P.to_device(s)
    if shift:
        t = torch.zeros(d["tokens"].numel() + 4, dtype=torch.int32, device="cuda")
        t[shift:shift + d["tokens"].numel()] = d["tokens"]
        d["tokens"] = t[shift:]
    out = P.as_numpy(idx.admit(**d))
    torch.cuda.synchronize()
    return out, idx.dump()


def _same(a, b, what):
    ra, da = a
    rb, db = b
    for f in ra.dtype.names:
        assert np.array_equal(ra[f], rb[f]), (what, f)
    assert len(da) == len(db), what
    for f in ["key", "owner", "sharer"]:
        assert np.array_equal(da[f], db[f]), (what, f)


def _ragged(seed, n=3000):
    """Short requests of every shape: empty, under one block, exact blocks, tails, a few long
    ones, runs of zero-block requests (so a 32-lane group can cover more than 32 request
    starts), shared stems across users."""
    rng = np.random.default_rng(seed)
    stems = [run(seed, 3, k, 16 * int(rng.integers(1, 12))) for k in range(12)]
    prompts, users = [], []
    for j in range(n):
        r = rng.random()
        if r < 0.05:
            p = np.zeros(0, np.uint32)
        elif r < 0.10:
            p = run(seed, 4, j, int(rng.integers(1, 16)))
        elif 600 <= j < 680:                        # a run of zero-block requests
            p = run(seed, 4, j, int(rng.integers(0, 16)))
        else:
            p = np.concatenate([stems[int(rng.integers(12))],
                                run(seed, 5, j, int(rng.integers(0, 16 * 40)))])
            if rng.random() < 0.02:
                p = np.concatenate([p, run(seed, 6, j, 16 * 150)])   # a long one
        prompts.append(p.astype(np.uint32))
        users.append(int(rng.integers(0, 9)))
    return _pack(f"ragged{seed}", prompts, users)


@pytest.mark.parametrize("policy", list(POL))
@pytest.mark.parametrize("shift", [0, 1, 3])
def test_packed_equals_warp_per_request_and_oracle(policy, shift):
    s = _ragged(11 + shift)
    assert s.n_blocks() < 96 * s.n_requests       # the packed kernel takes this batch
    got = _run(s, policy, True, shift)
    ref = _run(s, policy, False, shift)
    _same(got, ref, f"{policy}/shift{shift}")
    o = Oracle(16, SEED, POL[policy])
    o.reserve(s.n_blocks() + 16)
    exp = o.process(s)
    _same(got, (exp, o.dump()), f"{policy}/shift{shift}/oracle")


def test_packed_two_component_keys():
    s = _ragged(23)
    _same(_run(s, "solidarity", True, nc=2), _run(s, "solidarity", False, nc=2), "nc2")


def test_packed_c4_shape():
    """The C4 attacker shape at reduced size (short, 16-byte aligned requests): both K_A forms
    and the oracle agree."""
    s = c4_attackers(benign_users=400, benign_requests=20_000, victims=10, templates=5,
                     colluders_per_victim=4, candidates=40)
    got = _run(s, "solidarity", True)
    _same(got, _run(s, "solidarity", False), "c4")
    o = Oracle(16, SEED, 2)
    o.reserve(s.n_blocks() + 16)
    _same(got, (o.process(s), o.dump()), "c4/oracle")
