"""Seeded synthetic TTFT sample streams for the Activator.

No arithmetic of the method here (no classification, no KDE): only the inputs a serving system
would report for completed requests — TTFT (ms), prompt length (tokens) and reuse fraction —
shaped after the paper's characterisation (P:§2.2 Observations 1-2): cache hits have a lower
per-token TTFT than misses, and the gap is masked as load grows.  The load follows phases, so
the windows move between distinguishable and indistinguishable regimes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class TtftStream:
    ttft_ms: np.ndarray          # float64 [M]
    prompt_tokens: np.ndarray    # uint32 [M]
    reuse_fraction: np.ndarray   # float64 [M]

    @property
    def n(self) -> int:
        return int(self.ttft_ms.size)


def ttft_stream(n: int, seed: int = 0x5011D0F2, phase_len: int = 4096,
                hit_share: float = 0.4, miss_share: float = 0.4) -> TtftStream:
    """n completed requests.  Reuse fraction: hit_share near 1, miss_share near 0, the rest in
    between.  Per-token TTFT (ms/token) is log-normal; the miss/hit gap shrinks in high-load
    phases (gap alternates 1.0 / 0.05 in log space every phase_len samples)."""
    rng = np.random.default_rng(seed)
    u = rng.random(n)
    reuse = np.where(u < hit_share, rng.uniform(0.85, 1.0, n),
                     np.where(u < hit_share + miss_share, rng.uniform(0.0, 0.15, n),
                              rng.uniform(0.3, 0.7, n)))
    prompt = rng.integers(256, 4097, n).astype(np.uint32)
    phase = (np.arange(n) // phase_len) % 2
    gap = np.where(phase == 0, 1.0, 0.05)
    log_pt = -3.0 + rng.normal(0.0, 0.35, n) + gap * (1.0 - reuse)
    ttft = np.exp(log_pt) * prompt
    return TtftStream(ttft.astype(np.float64), prompt, reuse.astype(np.float64))


def query_cuts(n_queries: int, n_samples: int, stride: int = 1) -> np.ndarray:
    """Per query (request in sequence order) the number of samples completed before it: the
    window advances every `stride` queries, evenly over the stream (non-decreasing)."""
    j = (np.arange(n_queries, dtype=np.int64) // stride) * stride
    return (j * n_samples // max(n_queries, 1)).astype(np.int64)
