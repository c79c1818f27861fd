"""Policy-evaluation workloads and harness: the five multi-user reuse
workloads of the paper's §6.2.1 (fig:eval_workloads) and the KDE-threshold sweep of
§6.3 (fig:kde_threshold_results), with the library as the cache.

No arithmetic of the method here: the generators only emit token ids, users and enforce bits,
and the closed loop only moves data between an admission function (the CUDA library, or the
oracle in tests) and an Activator function (likewise).  The latency stand-in that turns a
request's recomputed tokens into a TTFT sample is NOT the paper's (which measures an A100 running
LLMs, OUT of scope): it only makes hits faster than misses per token, as P:§2.2 Observation 1
states, so the Activator has windows to compare.

Readings: reuse levels Zero/Low/Moderate/High = 0 / 0.2 / 0.5 / 0.9 (
the paper gives levels only); presets W1 = (High intra, Zero inter), W2 = (High,
Moderate), W3 = (Moderate, Moderate), W4 = (High, High), W5 = (Zero, High) (W1, W2,
W5 from the §6.2.1 prose); per request: with p_intra repeat one of the user's own earlier stems,
else with p_inter adopt a shared template the user has not used yet, else a fresh stem;
the per-user secret slot sits late in the stem (block 6 of 8; S:366 secret_position); arrival
order is a seeded merge of per-user Poisson processes (order only).
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np

from .gen import VOCAB, Stream, _pack, run

LEVELS = {"zero": 0.0, "low": 0.2, "moderate": 0.5, "high": 0.9}
PRESETS = {"W1": ("high", "zero"), "W2": ("high", "moderate"), "W3": ("moderate", "moderate"),
           "W4": ("high", "high"), "W5": ("zero", "high")}
K_TEMPLATE, K_SECRET, K_FRESH, K_QTAIL = 41, 42, 43, 44


def reuse_workload(intra: str, inter: str, users: int = 10, requests_per_user: int = 100,
                   stem_blocks: int = 8, secret_at: int = 6, templates: int = 64,
                   family_size: int = 1, family_blocks: int = 3,
                   seed: int = 0x5011D0F3, block_size: int = 16, vocab: int = VOCAB) -> Stream:
    """One §6.2.1 workload: each prompt = stem (stem_blocks blocks, block `secret_at` replaced
    by the user's secret block) + a fresh query (1-3 blocks plus a partial tail).  Shared
    templates may come in families of `family_size` whose first `family_blocks` blocks coincide
    (a task preamble shared by several templates: two-level inter-user sharing, where selective
    isolation costs reuse); the W1-W5 presets use single templates (family_size 1), the θ sweep
    the two-level variant."""
    rng = np.random.default_rng(seed)
    p_intra, p_inter = LEVELS[intra], LEVELS[inter]
    bs = block_size
    secret = [run(seed, K_SECRET, u, bs, vocab) for u in range(users)]
    own = [[] for _ in range(users)]          # stems (template keys) each user has used
    used_tpl = [set() for _ in range(users)]
    fresh_ctr = 0
    per_user = []
    for u in range(users):
        reqs = []
        for i in range(requests_per_user):
            if own[u] and rng.random() < p_intra:
                stem = own[u][int(rng.integers(len(own[u])))]
            elif rng.random() < p_inter and len(used_tpl[u]) < templates:
                free = [t for t in range(templates) if t not in used_tpl[u]]
                t = free[int(rng.integers(len(free)))]
                used_tpl[u].add(t)
                stem = ("T", t)
                own[u].append(stem)
            else:
                fresh_ctr += 1
                stem = ("F", fresh_ctr)
                own[u].append(stem)
            blocks = []
            for b in range(stem_blocks):
                if b == secret_at:
                    blocks.append(secret[u])
                elif stem[0] == "T":
                    tid = (stem[1] // family_size) * 4096 if b < family_blocks else stem[1]
                    blocks.append(run(seed, K_TEMPLATE, tid * 1024 + b, bs, vocab))
                else:
                    blocks.append(run(seed, K_FRESH, stem[1] * 1024 + b, bs, vocab))
            qn = int(rng.integers(bs, 3 * bs + 1)) + int(rng.integers(1, bs))
            blocks.append(run(seed, K_QTAIL, (u * requests_per_user + i), qn, vocab))
            reqs.append(np.concatenate(blocks))
        per_user.append(reqs)
    # arrival order: merge of per-user Poisson processes (equal rates) = seeded interleave
    t = [np.cumsum(rng.exponential(1.0, requests_per_user)) for _ in range(users)]
    order = sorted(((t[u][i], u, i) for u in range(users) for i in range(requests_per_user)))
    prompts = [per_user[u][i] for _, u, i in order]
    us = [u for _, u, _ in order]
    return _pack(f"reuse_{intra}_{inter}", prompts, us,
                 meta=dict(intra=intra, inter=inter, users=users))


def preset(name: str, **kw) -> Stream:
    intra, inter = PRESETS[name]
    return reuse_workload(intra, inter, **kw)


def hit_rate(results, exclude_users=None, users=None) -> float:
    """Block-weighted hit rate sum(r) / sum(n) (R20), optionally excluding users."""
    r = results["reused"].astype(np.int64)
    n = results["n_blocks"].astype(np.int64)
    if exclude_users is not None and users is not None:
        keep = ~np.isin(users, list(exclude_users))
        r, n = r[keep], n[keep]
    return float(r.sum() / max(n.sum(), 1))


def synthetic_ttft_ms(prompt_tokens: np.ndarray, reused_blocks: np.ndarray, rng,
                      base_ms: float = 20.0, per_token_ms: float = 0.05,
                      noise: float = 0.15, block_size: int = 16) -> np.ndarray:
    """Stand-in latency: base + per-token cost of the recomputed tokens, log-normal noise."""
    recompute = np.maximum(prompt_tokens.astype(np.float64) - block_size * reused_blocks, 1.0)
    return (base_ms + per_token_ms * recompute) * np.exp(rng.normal(0.0, noise, recompute.size))


def closed_loop(stream: Stream, admit: Callable, activator: Optional[Callable], batch: int = 50,
                seed: int = 0x5011D0F4, enforce_override: Optional[np.ndarray] = None):
    """Admission with the Activator in the loop: the requests of each batch get their enforce
    bits from the samples of every request completed before the batch (completion lag = one
    batch); after admission their TTFT samples join the stream.

    admit(batch_stream_with_enforce) -> results;  activator(ttft, prompt_tokens, reuse_fraction,
    cuts) -> enforce bits.  activator None = isolation always active (enforce = all 1).
    enforce_override replays given bits (parity runs).  Returns (results, enforce, samples)."""
    rng = np.random.default_rng(seed)
    n = stream.n_requests
    ttft = np.zeros(n, np.float64)
    ptok = np.diff(stream.offsets.astype(np.int64)).astype(np.uint32)
    frac = np.zeros(n, np.float64)
    enforce = np.ones(n, np.uint8)
    out = []
    for lo in range(0, n, batch):
        hi = min(lo + batch, n)
        b = stream.slice(lo, hi)
        if enforce_override is not None:
            enforce[lo:hi] = enforce_override[lo:hi]
        elif activator is not None and lo > 0:   # no samples yet: fail-safe enforce (R21)
            cuts = np.full(hi - lo, lo, np.int64)
            enforce[lo:hi] = activator(ttft[:lo], ptok[:lo], frac[:lo], cuts)
        b.enforce = np.ascontiguousarray(enforce[lo:hi])
        res = admit(b)
        out.append(res)
        nb = res["n_blocks"].astype(np.float64)
        frac[lo:hi] = np.where(nb > 0, res["reused"] / np.maximum(nb, 1), 0.0)
        ttft[lo:hi] = synthetic_ttft_ms(ptok[lo:hi], res["reused"].astype(np.float64), rng)
    return np.concatenate(out), enforce, (ttft, ptok, frac)


def two_level(name: str, **kw) -> Stream:
    """A preset with two-level templates (families of 8 sharing a 3-block preamble)."""
    kw.setdefault("family_size", 8)
    kw.setdefault("family_blocks", 3)
    return preset(name, **kw)
