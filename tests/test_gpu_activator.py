"""GPU parity of the Activator (solid_activator_run, through the C ABI) against the fp64 oracle
on identical seeded TTFT streams.  Bar: overlap within 1e-9 absolute (both sides
fp64; only summation order differs), identical fail-safe (NaN) positions, identical enforce bits
wherever |overlap − θ| > 1e-9."""
import numpy as np
import pytest

from oracle.activator import ActivatorConfig, enforce_stream
from workloads import query_cuts, ttft_stream

pytestmark = pytest.mark.gpu


def _run(s, cuts, cfg, **kw):
    import torch
    import paper_2603_10726_b200 as P
    act = P.Activator(theta=cfg.theta, window_len=cfg.window_len, min_samples=cfg.min_samples,
                      hit_hi=cfg.hit_hi, hit_lo=cfg.hit_lo, grid=cfg.grid,
                      max_samples=max(s.n, 1), max_queries=max(len(cuts), 1), **kw)
    d = lambda a, t: torch.from_numpy(np.ascontiguousarray(a)).to(dtype=t, device="cuda")
    ov, en = act.run(d(s.ttft_ms, torch.float64), d(s.prompt_tokens.astype(np.int32), torch.int32),
                     d(s.reuse_fraction, torch.float64), d(cuts, torch.int64))
    torch.cuda.synchronize()
    return ov.cpu().numpy(), en.cpu().numpy()


def _check(s, cuts, cfg):
    got_ov, got_en = _run(s, cuts, cfg)
    exp_en, exp_ov = enforce_stream(s.ttft_ms, s.prompt_tokens, s.reuse_fraction, cuts, cfg)
    assert np.array_equal(np.isnan(got_ov), np.isnan(exp_ov))
    ok = ~np.isnan(exp_ov)
    if ok.any():
        err = np.abs(got_ov[ok] - exp_ov[ok])
        assert err.max() <= 1e-9, (err.max(), int(np.argmax(err)))
    decided = np.isnan(exp_ov) | (np.abs(exp_ov - cfg.theta) > 1e-9)
    assert np.array_equal(got_en[decided], exp_en[decided])
    return got_ov, got_en


@pytest.mark.parametrize("window,grid", [(256, 512), (64, 512), (1000, 300), (2, 2)])
def test_parity_window_and_grid_shapes(window, grid):
    s = ttft_stream(12000, seed=window * 31 + grid, phase_len=2500)
    cuts = query_cuts(700, s.n, stride=7)
    _, en = _check(s, cuts, ActivatorConfig(window_len=window, grid=grid))
    if window >= 64:
        assert en.min() == 0 and en.max() == 1      # both regimes on this stream


def test_every_query_its_own_window_and_ragged_tiles():
    s = ttft_stream(3001, seed=5, phase_len=700)     # 3001: ragged last 1024-sample tile
    cuts = np.arange(0, 3001, 3, dtype=np.int64)     # a new window at every query
    _check(s, cuts, ActivatorConfig(window_len=128, min_samples=5))


@pytest.mark.parametrize("theta", [0.0, 1.0, 0.37])
def test_thresholds(theta):
    s = ttft_stream(5000, seed=9)
    cuts = query_cuts(200, s.n, stride=1)
    _, en = _check(s, cuts, ActivatorConfig(theta=theta))
    if theta == 0.0:
        assert en[cuts >= 2000].max() == 0           # populated windows never active at θ = 0


def test_degenerate_streams():
    from workloads.ttft import TtftStream
    # all excluded samples: every query fail-safe; zero spread windows; empty query list
    n = 500
    s = TtftStream(np.full(n, 5.0), np.full(n, 10, np.uint32), np.full(n, 0.5))
    ov, en = _check(s, np.arange(0, n, 5, dtype=np.int64), ActivatorConfig())
    assert np.isnan(ov).all() and en.all()
    s = TtftStream(np.full(n, 5.0), np.full(n, 10, np.uint32),
                   np.where(np.arange(n) % 2 == 0, 1.0, 0.0))
    _check(s, np.arange(0, n, 5, dtype=np.int64), ActivatorConfig())
    ov, en = _run(s, np.zeros(0, dtype=np.int64), ActivatorConfig())
    assert ov.size == 0 and en.size == 0


def test_invalid_inputs_are_rejected():
    import paper_2603_10726_b200 as P
    from workloads.ttft import TtftStream
    s = ttft_stream(1000, seed=2)
    with pytest.raises(P.SolidError) as ei:
        _run(s, np.array([10, 5], dtype=np.int64), ActivatorConfig())   # decreasing cuts
    assert ei.value.status == P.SOLID_ERR_INVALID
    with pytest.raises(P.SolidError):
        _run(s, np.array([5, 2000], dtype=np.int64), ActivatorConfig())  # beyond the stream
    bad = TtftStream(s.ttft_ms.copy(), s.prompt_tokens.copy(), s.reuse_fraction)
    bad.prompt_tokens[17] = 0
    with pytest.raises(P.SolidError):
        _run(bad, np.array([5], dtype=np.int64), ActivatorConfig())
    with pytest.raises(P.SolidError):
        P.Activator(window_len=5000)


def test_enforce_bits_drive_the_admission_path():
    """The activator's output is the batch's enforce[] (R11: enforce 0 = no diversion, flags still
    recorded): admission with those bits equals the oracle fed the same bits."""
    import torch
    import paper_2603_10726_b200 as P
    from oracle import Oracle
    from workloads import c2_shared_prompt
    st = c2_shared_prompt(users=30, reqs_per_user=20)
    s = ttft_stream(4000, seed=3, phase_len=1000)
    cuts = query_cuts(st.n_requests, s.n, stride=25)
    _, en = _run(s, cuts, ActivatorConfig(window_len=128))
    assert 0 < en.sum() < en.size
    st.enforce = en.astype(np.uint8)
    o = Oracle(16, 0x5011D000, 2)
    exp = o.process(st)
    idx = P.Index("solidarity", capacity_blocks=4 * st.n_blocks() + 1024,
                  max_batch_tokens=st.n_tokens + 64, max_batch_requests=st.n_requests,
                  seed=0x5011D000)
    got = P.as_numpy(idx.admit(**P.to_device(st)))
    torch.cuda.synchronize()
    for f in exp.dtype.names:
        assert np.array_equal(got[f].astype(np.int64), exp[f].astype(np.int64)), f
