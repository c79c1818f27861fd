"""GPU parity of in-flight pinning (pin = 1; R38) against the oracle
(tests/test_oracle_pins.py pins the oracle itself against a brute force).

Harness: the GPU admits batches (split in halves on SOLID_ERR_CAPACITY down to single requests;
a single request that fails is refused, as the oracle refuses it); between batches random
earlier rows are released on both sides.  Per request: result (or refusal) and block-table row;
after every batch: the index, every live entry's block and every block's pin count."""
import numpy as np
import pytest

from oracle import Oracle, PinRefused
from oracle_helpers import NONE
from workloads import c3_multiturn, random_small

pytestmark = pytest.mark.gpu
SEED = 0x5011D000
POL = {"apc": 0, "user_isolation": 1, "solidarity": 2}


class Pair:
    def __init__(self, policy, cap, s, evict=True, nc=1, max_blocks=8):
        import paper_2603_10726_b200 as P
        self.P = P
        self.cap = cap
        self.idx = P.Index(policy, capacity_blocks=cap, max_batch_tokens=s.n_tokens + 64,
                           max_batch_requests=max(s.n_requests, 1), max_blocks=max_blocks, seed=SEED,
                           evict=evict, block_table=True, pin=True, hash_components=nc)
        self.o = Oracle(16, SEED, POL[policy], capacity=cap if evict else 0, pool=cap, pin=True,
                        components=nc)
        self.rows = []           # (gpu row tensor, oracle row) of admitted, unreleased requests

    def _gpu(self, b):
        """Admit b on the GPU; returns per request (result or None if refused, row)."""
        import torch
        P = self.P
        d = P.to_device(b)           # the block table reads the batch's offsets: keep them alive
        try:
            res = P.as_numpy(self.idx.admit(**d))
        except P.SolidError as e:
            assert e.status == P.SOLID_ERR_CAPACITY, e
            if b.n_requests == 1:
                return [(None, None)]
            h = b.n_requests // 2
            return self._gpu(b.slice(0, h)) + self._gpu(b.slice(h, b.n_requests))
        torch.cuda.synchronize()
        bt = self.idx.block_table(b.n_tokens)
        offs = b.offsets.astype(np.int64)
        out = []
        for j in range(b.n_requests):
            a, nb = offs[j] // 16, (offs[j + 1] - offs[j]) // 16
            out.append((res[j], bt[a:a + nb].clone()))
        return out

    def batch(self, b):
        got = self._gpu(b)
        for j in range(b.n_requests):
            try:
                exp = self.o.process(b.slice(j, j + 1))[0]
                erow = self.o.block_table()[:(int(b.offsets[j + 1]) - int(b.offsets[j])) // 16]
            except PinRefused:
                exp, erow = None, None
            g, grow = got[j]
            assert (g is None) == (exp is None), (b.name, j)
            if g is None:
                continue
            assert all(int(g[f]) == int(exp[f]) for f in exp.dtype.names), (j, g, exp)
            assert np.array_equal(grow.cpu().numpy().view(np.uint32), erow), j
            self.rows.append((grow, erow))
        return sum(g is None for g, _ in got)

    def release_some(self, rng, frac):
        keep = []
        for grow, erow in self.rows:
            if rng.random() < frac:
                self.idx.release(grow)
                self.o.release(erow)
            else:
                keep.append((grow, erow))
        self.rows = keep

    def check_state(self):
        gd, ed = self.idx.dump(), self.o.dump()
        assert len(gd) == len(ed)
        assert all(np.array_equal(gd[f], ed[f]) for f in ["key", "owner", "sharer"])
        gk, gp = self.idx.dump_phys()
        ek, ep = self.o.dump_phys()
        assert np.array_equal(gk, ek) and np.array_equal(gp, ep)
        pins = self.idx.pins(self.cap)
        ok, opins = self.o.dump_pins()
        exp = np.zeros(self.cap, np.uint32)
        exp[ep] = opins
        assert np.array_equal(pins, exp)


@pytest.mark.parametrize("policy", ["apc", "solidarity", "user_isolation"])
@pytest.mark.parametrize("batch", [1, 8, 64])
@pytest.mark.parametrize("cap", [12, 40])
def test_random_streams_with_releases(policy, batch, cap):
    rng = np.random.default_rng(cap * 7 + batch)
    for seed in (1, 2):
        s = random_small(300, users=3, alphabet_blocks=6, max_blocks=5, seed=seed,
                         enforce_prob=0.8)
        pr = Pair(policy, cap, s)
        refused = 0
        for lo in range(0, s.n_requests, batch):
            refused += pr.batch(s.slice(lo, min(lo + batch, s.n_requests)))
            pr.check_state()
            pr.release_some(rng, 0.5)
            pr.check_state()
        if cap == 12:
            assert refused > 0


def test_pins_without_eviction():
    """evict = 0: pins are counted (nothing is ever reclaimed); release brings them to 0."""
    rng = np.random.default_rng(3)
    s = random_small(200, users=3, alphabet_blocks=5, max_blocks=5, seed=9)
    pr = Pair("solidarity", 4096, s, evict=False)
    for lo in range(0, s.n_requests, 25):
        pr.batch(s.slice(lo, lo + 25))
        pr.check_state()
        pr.release_some(rng, 0.3)
    pr.release_some(rng, 1.1)
    pr.check_state()
    assert not pr.idx.pins(4096).any()


def test_multiturn_under_pin_pressure_two_component_keys():
    """C3-shaped conversations through a small pinned cache, H-def v3 keys."""
    rng = np.random.default_rng(11)
    warm, timed = c3_multiturn(users=30, warm_blocks=600, timed_rounds=2, seed=SEED + 3,
                               max_ctx=700)
    pr = Pair("solidarity", 400, warm, nc=2, max_blocks=64)
    for s in (warm, timed):
        for lo in range(0, s.n_requests, 20):
            pr.batch(s.slice(lo, min(lo + 20, s.n_requests)))
            pr.release_some(rng, 0.7)
        pr.check_state()


def test_release_errors_and_refusal():
    import torch
    import paper_2603_10726_b200 as P
    s = random_small(10, users=1, alphabet_blocks=50, max_blocks=3, seed=4)
    idx = P.Index("apc", capacity_blocks=64, max_batch_tokens=s.n_tokens + 64,
                  max_batch_requests=16, max_blocks=64, evict=True, block_table=True, pin=True)
    idx.admit(**P.to_device(s))
    torch.cuda.synchronize()
    bad = torch.tensor([63], dtype=torch.int32, device="cuda")      # a block with no pin
    with pytest.raises(P.SolidError) as ei:
        idx.release(bad)
    assert ei.value.status == P.SOLID_ERR_INVALID
    with pytest.raises(P.SolidError):
        P.Index("apc", capacity_blocks=64, pin=True)                  # pin needs block_table
