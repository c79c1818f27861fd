"""Pins of the Activator oracle (oracle/activator.py) against the paper / SPEC and against an
independent density + integrator (scipy), closed forms and hand-derived values — never against
itself.  SURVEY §8 row f2; DESIGN.md §8."""
import json
import math
import os

import numpy as np
import pytest
from scipy import integrate, stats

from oracle.activator import (EXCLUDED, HIT, MISS, ActivatorConfig, classify, enforce_stream,
                              isolation_active, kde, kde_overlap, silverman, windows)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "activator.json")))


@pytest.mark.parametrize("case", GOLD["silverman"])
def test_silverman_hand_derived(case):
    assert silverman(np.array(case["x"])) == pytest.approx(case["h"], rel=1e-12, abs=1e-15)


def test_classification_examples():
    """SPEC S:249-252 examples (defaults hi = 0.8, lo = 0.2)."""
    cfg = ActivatorConfig()
    assert classify(1.0, cfg) == HIT
    assert classify(0.0, cfg) == MISS
    assert classify(0.5, cfg) == EXCLUDED
    assert classify(0.8, cfg) == HIT and classify(0.2, cfg) == MISS   # cutoffs inclusive


def test_windows_are_per_token_fifo():
    """Per-token values (ttft / prompt tokens), oldest-first eviction per class."""
    cfg = ActivatorConfig(window_len=3)
    ttft = np.array([10.0, 20.0, 30.0, 40.0, 50.0, 60.0, 70.0])
    ptok = np.array([10, 10, 10, 10, 10, 10, 10], dtype=np.uint32)
    reuse = np.array([1.0, 0.0, 1.0, 1.0, 0.5, 1.0, 0.1])
    h, m = windows(ttft, ptok, reuse, 7, cfg)
    assert h.tolist() == [3.0, 4.0, 6.0]          # 1.0 evicted (oldest of four hits)
    assert m.tolist() == [2.0, 7.0]               # 5.0 excluded (reuse 0.5)
    h, m = windows(ttft, ptok, reuse, 2, cfg)
    assert h.tolist() == [1.0] and m.tolist() == [2.0]


def test_identical_samples_overlap_at_least_099():
    a = np.array([1.0, 1.1, 0.9, 1.05])
    assert kde_overlap(a, a.copy()) >= 0.99


def test_disjoint_samples_overlap_at_most_001():
    rng = np.random.default_rng(7)
    a = 1.0 + 0.01 * rng.standard_normal(100)
    b = 50.0 + 0.01 * rng.standard_normal(100)
    assert kde_overlap(a, b) <= 0.01


def _independent_overlap(a, b, points=65536):
    """scipy's gaussian_kde (its own kernel sum; bandwidth factor h/sd so the kernel sd equals the
    Silverman h) on a 65 536-point grid, and scipy.integrate.quad of min(f, g)."""
    ha, hb = silverman(a), silverman(b)
    fa = stats.gaussian_kde(a, bw_method=ha / np.std(a, ddof=1))
    fb = stats.gaussian_kde(b, bw_method=hb / np.std(b, ddof=1))
    hm = max(ha, hb)
    lo, hi = min(a.min(), b.min()) - 3 * hm, max(a.max(), b.max()) + 3 * hm
    x = np.linspace(lo, hi, points)
    grid = float(np.sum(np.diff(x) * (np.minimum(fa(x), fb(x))[1:] + np.minimum(fa(x), fb(x))[:-1]) / 2))
    quad, _ = integrate.quad(lambda t: min(fa(t)[0], fb(t)[0]), lo, hi, limit=400)
    return grid, quad


@pytest.mark.parametrize("seed", range(10))
def test_matches_independent_fine_grid_within_003(seed):
    """SPEC S:262 / S:545: 200 draws N(0,1) vs 200 draws N(1,1), ten seeds: within ±0.03 of a
    65 536-point numerical integral of an independent KDE implementation."""
    rng = np.random.default_rng(1000 + seed)
    a, b = rng.normal(0, 1, 200), rng.normal(1, 1, 200)
    grid, quad = _independent_overlap(a, b)
    ov = kde_overlap(a, b)
    assert abs(ov - grid) <= 0.03 and abs(ov - quad) <= 0.03
    assert abs(grid - quad) < 1e-3      # the two independent integrals agree


def test_density_matches_scipy_pointwise():
    rng = np.random.default_rng(3)
    a = rng.lognormal(0, 0.5, 300)
    h = silverman(a)
    ref = stats.gaussian_kde(a, bw_method=h / np.std(a, ddof=1))
    x = np.linspace(a.min() - 1, a.max() + 1, 101)
    np.testing.assert_allclose(kde(a, h, x), ref(x), rtol=1e-10, atol=1e-14)


def test_large_sample_overlap_approaches_gaussian_closed_form():
    """Two large normal samples N(0,1), N(1,1): the KDEs tend to N(μ, 1 + h²), whose overlap is
    2Φ(−|Δμ| / (2·sqrt(1 + h²))) (equal-variance normals)."""
    rng = np.random.default_rng(11)
    a, b = rng.normal(0, 1, 4000), rng.normal(1, 1, 4000)
    h = 0.5 * (silverman(a) + silverman(b))
    closed = 2 * stats.norm.cdf(-1.0 / (2 * math.sqrt(1 + h * h)))
    assert abs(kde_overlap(a, b, grid=2048) - closed) < 0.02


@pytest.mark.parametrize("seed", range(5))
def test_symmetry_and_bounds(seed):
    rng = np.random.default_rng(seed)
    a = rng.gamma(2.0, 1.0, 50 + seed)
    b = rng.gamma(2.5, 1.2, 80)
    ab, ba = kde_overlap(a, b), kde_overlap(b, a)
    assert abs(ab - ba) <= 1e-12
    assert 0.0 <= ab <= 1.0


def test_isolation_active_rules():
    """fail-safe with too few samples; θ = 0 never active; θ = 1 active unless
    the overlap is 1."""
    rng = np.random.default_rng(5)
    a, b = rng.normal(0, 1, 100), rng.normal(0.3, 1, 100)
    assert isolation_active(np.array([]), np.array([]), ActivatorConfig())[0]
    assert isolation_active(a[:1], b, ActivatorConfig())[0]
    assert isolation_active(a[:4], b, ActivatorConfig(min_samples=5))[0]
    # SPEC S:282 default min_samples = 16: 15 samples in a class keep the fail-safe on, 16 do not
    assert ActivatorConfig().min_samples == 16
    assert isolation_active(a[:15], b, ActivatorConfig(theta=0.0))[0]
    assert not isolation_active(a[:16], b, ActivatorConfig(theta=0.0))[0]
    assert not isolation_active(a, b, ActivatorConfig(theta=0.0))[0]
    en, ov = isolation_active(a, b, ActivatorConfig(theta=1.0))
    assert ov < 1.0 and en
    en, ov = isolation_active(a, b, ActivatorConfig(theta=0.5))
    assert en == (ov < 0.5)


def test_enforce_stream_uses_the_window_before_each_query():
    from workloads import query_cuts, ttft_stream
    s = ttft_stream(9000, phase_len=3000)
    cfg = ActivatorConfig(window_len=128)
    cuts = query_cuts(300, s.n, stride=10)
    en, ov = enforce_stream(s.ttft_ms, s.prompt_tokens, s.reuse_fraction, cuts, cfg)
    for j in [0, 57, 123, 299]:
        h, m = windows(s.ttft_ms, s.prompt_tokens, s.reuse_fraction, int(cuts[j]), cfg)
        e2, o2 = isolation_active(h, m, cfg)
        assert en[j] == e2 and (np.isnan(ov[j]) and np.isnan(o2) or ov[j] == o2)
    # the load phases move the decision: both regimes appear
    assert en.min() == 0 and en.max() == 1
