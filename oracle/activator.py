"""Activator oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 numpy restatement of the paper's Activator: per request, isolation is enforced
iff the hit and miss TTFT distributions of the most recent sliding window are distinguishable,
i.e. their KDE overlap is below the administrator's threshold θ.

  P:521-531 (§4.3 "Activator Optimization"): "continuously monitors the latency gap between hits
    and misses over a sliding time window and computes the Kernel Density Estimation (KDE)
    overlap between their distributions ... When the overlap exceeds a threshold θ, CacheSolidarity
    deactivates selective isolation ... when the overlap falls below θ ... activates its detection
    and prefix isolation mechanism.  This decision is evaluated at every request using the most
    recent sliding window of TTFT samples."
  P:(§2.2) overlap = "the integral of the minimum of their density functions".
  SPEC S:245-268 fixes what the paper leaves open (readings R17-R21): per-token TTFT,
    the hit/miss classification cutoffs, per-class FIFO windows, Gaussian kernels with Silverman
    bandwidth h = 0.9·min(σ, IQR/1.34)·n^(-1/5) floored at 1e-9, a 512-point trapezoid over
    [min(all) − 3·h_max, max(all) + 3·h_max], clamp to [0, 1], fail-safe "active" with fewer than
    min_samples in either class.

Pinned by tests/test_oracle_activator.py against scipy.stats.gaussian_kde + scipy.integrate (an
independent density and integrator), hand-computed bandwidths (tests/golden/activator.json), the
SPEC's examples and the closed-form overlap of two normals.  Nothing here is imported by the
product path (paper_2603_10726_b200/).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

HIT, MISS, EXCLUDED = 0, 1, 2


@dataclass
class ActivatorConfig:
    theta: float = 0.5          # P:523 threshold θ in [0, 1]
    window_len: int = 256       # samples kept per class
    min_samples: int = 16       # fewer in either class -> fail-safe active (default)
    hit_hi: float = 0.8         # reuse fraction >= hit_hi -> Hit
    hit_lo: float = 0.2         # reuse fraction <= hit_lo -> Miss
    grid: int = 512             # trapezoid points


def classify(reuse_fraction: float, cfg: ActivatorConfig) -> int:
    """Hit if reuse_fraction >= hi, Miss if <= lo, else Excluded."""
    if reuse_fraction >= cfg.hit_hi:
        return HIT
    if reuse_fraction <= cfg.hit_lo:
        return MISS
    return EXCLUDED


def windows(ttft_ms, prompt_tokens, reuse_fraction, cut: int, cfg: ActivatorConfig):
    """The two FIFO windows after recording samples 0..cut-1 in order: each
    sample's per-token TTFT (ttft / prompt tokens) joins its class; each class keeps its
    window_len most recent values."""
    hit, miss = [], []
    for i in range(cut):
        c = classify(float(reuse_fraction[i]), cfg)
        v = float(ttft_ms[i]) / float(prompt_tokens[i])
        if c == HIT:
            hit.append(v)
            if len(hit) > cfg.window_len:
                hit.pop(0)                       # oldest-first eviction
        elif c == MISS:
            miss.append(v)
            if len(miss) > cfg.window_len:
                miss.pop(0)
    return np.array(hit, dtype=np.float64), np.array(miss, dtype=np.float64)


def silverman(x: np.ndarray) -> float:
    """h = 0.9 · min(σ, IQR/1.34) · n^(-1/5), floored at 1e-9.  σ is the sample
    standard deviation (ddof = 1) and the quartiles are linear-interpolation percentiles
    (readings R19, R20)."""
    n = x.size
    sigma = float(np.std(x, ddof=1))
    q75, q25 = np.percentile(x, [75.0, 25.0])
    iqr = float(q75 - q25)
    h = 0.9 * min(sigma, iqr / 1.34) * n ** (-0.2)
    return max(h, 1e-9)


def kde(x: np.ndarray, h: float, pts: np.ndarray) -> np.ndarray:
    """Gaussian-kernel density estimate at pts: (1/(n·h·√(2π))) Σ_i exp(−(pts − x_i)² / (2h²))."""
    d = (pts[:, None] - x[None, :]) / h
    return np.exp(-0.5 * d * d).sum(axis=1) / (x.size * h * math.sqrt(2.0 * math.pi))


def kde_overlap(a: np.ndarray, b: np.ndarray, grid: int = 512) -> float:
    """∫ min(f̂_a, f̂_b) by the trapezoid rule on `grid` uniform points spanning
    [min(a ∪ b) − 3·h_max, max(a ∪ b) + 3·h_max], clamped to [0, 1]."""
    ha, hb = silverman(a), silverman(b)
    hmax = max(ha, hb)
    lo = min(a.min(), b.min()) - 3.0 * hmax
    hi = max(a.max(), b.max()) + 3.0 * hmax
    pts = np.linspace(lo, hi, grid)
    m = np.minimum(kde(a, ha, pts), kde(b, hb, pts))
    ov = float(np.trapezoid(m, pts))
    return min(max(ov, 0.0), 1.0)


def isolation_active(hit: np.ndarray, miss: np.ndarray, cfg: ActivatorConfig):
    """active (enforce) if either class has fewer than min_samples (fail-safe),
    else iff overlap < θ.  Returns (enforce, overlap or NaN)."""
    if hit.size < max(cfg.min_samples, 2) or miss.size < max(cfg.min_samples, 2):
        return True, float("nan")
    ov = kde_overlap(hit, miss, cfg.grid)
    return ov < cfg.theta, ov


def enforce_stream(ttft_ms, prompt_tokens, reuse_fraction, cuts, cfg: ActivatorConfig):
    """Per query j: the decision on the window after samples 0..cuts[j]-1 ("evaluated at
    every request using the most recent sliding window")."""
    en = np.zeros(len(cuts), dtype=np.uint8)
    ov = np.full(len(cuts), np.nan)
    memo = {}
    for j, c in enumerate(cuts):
        c = int(c)
        if c not in memo:
            memo[c] = isolation_active(*windows(ttft_ms, prompt_tokens, reuse_fraction, c, cfg), cfg)
        en[j], ov[j] = memo[c]
    return en, ov
