"""GPU: policy evaluation with the CUDA library as the cache.  Every W1-W5
workload (single- and two-level templates) under every policy gives, request by request, the
oracle's results; the θ sweep runs the closed loop on the GPU (CUDA Activator -> enforce bits ->
CUDA admission -> synthetic TTFT samples) and matches the oracle loop fed the same bits, with
the enforce bits themselves equal to the oracle Activator's away from the threshold."""
import numpy as np
import pytest

from oracle import Oracle
from oracle.activator import ActivatorConfig, enforce_stream
from workloads.policy_eval import PRESETS, closed_loop, hit_rate, preset, two_level

pytestmark = pytest.mark.gpu
SEED = 0x5011D000
POL = {"apc": 0, "user_isolation": 1, "solidarity": 2}


def _gpu_admit(policy, s):
    import torch
    import paper_2603_10726_b200 as P
    idx = P.Index(policy, capacity_blocks=1 << 16, max_batch_tokens=s.n_tokens + 64,
                  max_batch_requests=max(s.n_requests, 1), seed=SEED)

    def admit(b):
        out = P.as_numpy(idx.admit(**P.to_device(b)))
        torch.cuda.synchronize()
        return out
    return admit, idx


@pytest.mark.parametrize("gen", [preset, two_level])
@pytest.mark.parametrize("w", list(PRESETS))
@pytest.mark.parametrize("policy", ["apc", "user_isolation", "solidarity"])
def test_workload_parity(gen, w, policy):
    s = gen(w)
    admit, idx = _gpu_admit(policy, s)
    got = np.concatenate([admit(s.slice(i, min(i + 100, s.n_requests)))
                          for i in range(0, s.n_requests, 100)])
    o = Oracle(16, SEED, POL[policy])
    exp = o.process(s)
    assert np.array_equal(got, exp)
    gd, ed = idx.dump(), o.dump()
    assert all(np.array_equal(gd[f], ed[f]) for f in ["key", "owner", "sharer"])


@pytest.mark.parametrize("theta", [0.0, 0.3, 0.45, 0.5, 0.6, 1.0])
def test_theta_sweep_closed_loop(theta):
    import torch
    import paper_2603_10726_b200 as P
    s = two_level("W4")
    admit, _ = _gpu_admit("solidarity", s)
    act = P.Activator(theta=theta, window_len=256, min_samples=16, grid=512,
                      max_samples=s.n_requests + 1, max_queries=64)
    dev = lambda a, t: torch.from_numpy(np.ascontiguousarray(a)).to(dtype=t, device="cuda")
    overl = []

    def gpu_act(tt, pt, fr, cuts):
        ov, en = act.run(dev(tt, torch.float64), dev(pt.astype(np.int32), torch.int32),
                         dev(fr, torch.float64), dev(cuts, torch.int64))
        overl.append(ov.cpu().numpy())
        return en.cpu().numpy()
    res, en, (tt, pt, fr) = closed_loop(s, admit, gpu_act, batch=50)
    # the oracle loop fed the GPU's enforce bits gives the same results and samples
    o = Oracle(16, SEED, 2)
    res_o, _, (tt_o, _, fr_o) = closed_loop(s, lambda b: o.process(b), None, batch=50,
                                            enforce_override=en)
    assert np.array_equal(res, res_o) and np.array_equal(tt, tt_o) and np.array_equal(fr, fr_o)
    # the GPU Activator's bits equal the oracle Activator's on those samples (threshold margin)
    cfg = ActivatorConfig(theta=theta)
    cuts = np.repeat(np.arange(50, s.n_requests, 50), 50)[:s.n_requests - 50]
    en_o, ov_o = enforce_stream(tt, pt, fr, cuts, cfg)
    ov_g = np.concatenate(overl)
    en = en[50:]                              # the first batch: fail-safe, no Activator call
    near = np.abs(np.nan_to_num(ov_o, nan=-9) - theta) <= 1e-9
    assert np.array_equal(en[~near], en_o[~near])
    ok = ~np.isnan(ov_o)
    assert np.array_equal(np.isnan(ov_g), np.isnan(ov_o))
    assert np.abs(ov_g[ok] - ov_o[ok]).max() <= 1e-9
    assert 0.0 <= hit_rate(res) <= 1.0


@pytest.mark.parametrize("w", ["W3", "W5"])
@pytest.mark.parametrize("policy", ["apc", "user_isolation", "solidarity"])
def test_workload_parity_under_lru_pressure(w, policy):
    """The policy evaluation under a 1000-entry LRU cap (evict mode) matches the LRU oracle."""
    import torch
    import paper_2603_10726_b200 as P
    s = two_level(w)
    idx = P.Index(policy, capacity_blocks=1000, max_batch_tokens=s.n_tokens + 64,
                  max_batch_requests=25, max_blocks=64, seed=SEED, evict=True)

    def one(b):
        try:
            return P.as_numpy(idx.admit(**P.to_device(b)))
        except P.SolidError as e:
            assert e.status == P.SOLID_ERR_CAPACITY and b.n_requests > 1
            h = b.n_requests // 2
            return np.concatenate([one(b.slice(0, h)), one(b.slice(h, b.n_requests))])
    got = np.concatenate([one(s.slice(i, min(i + 25, s.n_requests)))
                          for i in range(0, s.n_requests, 25)])
    torch.cuda.synchronize()
    o = Oracle(16, SEED, POL[policy], capacity=1000)
    assert np.array_equal(got, o.process(s))
    gd, ed = idx.dump_ex(), o.dump_ex()
    assert all(np.array_equal(gd[f], ed[f]) for f in ["key", "owner", "sharer", "last_used"])
