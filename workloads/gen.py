"""Seeded synthetic workloads shaped like the paper's.

Token ids come from a counter-based generator: token = splitmix64(stream_key + idx) mod V, where the
stream key names a *segment* (a system prompt, a user profile, one query, ...).  Equal segment keys
give equal token runs, which is how shared prefixes are built.  Structural choices (orders, lengths,
candidate positions) use numpy's PCG64 seeded per config.

Nothing here hashes blocks, probes a cache or applies a detector rule; the oracle (``oracle/``) and
the CUDA path (``paper_2603_10726_b200``) both consume these streams unchanged.

Paper anchors for the shapes:
  * block size 16, Llama-2 vocabulary (tab:models P:661-680)            -> VOCAB = 32000
  * shared system prompts / templates with private fields
  * multi-turn chats ("Multiturn Chat")
  * attacker probing a victim prefix candidate by candidate
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

VOCAB = 32000
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _splitmix(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 (Vigna) used as a counter-based RNG; x is uint64."""
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _key(seed: int, *parts: int) -> np.uint64:
    """Mix a segment name (seed, kind, id, ...) into one 64-bit stream key."""
    k = np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    for p in parts:
        k = _splitmix(k ^ np.uint64(p & 0xFFFFFFFFFFFFFFFF))
    return k[0]


def run(seed: int, kind: int, ident: int, n: int, vocab: int = VOCAB) -> np.ndarray:
    """n tokens of segment (kind, ident): uint32 in [0, vocab)."""
    base = _key(seed, kind, ident)
    with np.errstate(over="ignore"):
        idx = np.arange(n, dtype=np.uint64) * _GOLD + base
    return (_splitmix(idx) % np.uint64(vocab)).astype(np.uint32)


@dataclass
class Stream:
    """A request stream in global sequence order (CSR tokens)."""
    name: str
    tokens: np.ndarray            # uint32[T]
    offsets: np.ndarray           # uint64[N+1], offsets[0] == 0, monotone
    users: np.ndarray             # uint32[N]
    enforce: Optional[np.ndarray] = None   # uint8[N] or None (= all 1)
    meta: dict = field(default_factory=dict)

    @property
    def n_requests(self) -> int:
        return int(self.users.shape[0])

    @property
    def n_tokens(self) -> int:
        return int(self.offsets[-1])

    def n_blocks(self, block_size: int = 16) -> int:
        lens = np.diff(self.offsets.astype(np.int64))
        return int((lens // block_size).sum())

    def slice(self, lo: int, hi: int, name: Optional[str] = None) -> "Stream":
        """Requests [lo, hi) as a standalone stream (offsets rebased to 0)."""
        t0, t1 = int(self.offsets[lo]), int(self.offsets[hi])
        return Stream(name or f"{self.name}[{lo}:{hi}]",
                      np.ascontiguousarray(self.tokens[t0:t1]),
                      (self.offsets[lo:hi + 1] - np.uint64(t0)).astype(np.uint64),
                      np.ascontiguousarray(self.users[lo:hi]),
                      None if self.enforce is None else np.ascontiguousarray(self.enforce[lo:hi]),
                      dict(self.meta))


def _pack(name: str, prompts: list, users: list, enforce=None, meta=None) -> Stream:
    lens = np.array([len(p) for p in prompts], dtype=np.uint64)
    offsets = np.zeros(len(prompts) + 1, dtype=np.uint64)
    np.cumsum(lens, out=offsets[1:])
    tokens = (np.concatenate(prompts).astype(np.uint32) if prompts and int(offsets[-1]) > 0
              else np.zeros(0, dtype=np.uint32))
    en = None if enforce is None else np.asarray(enforce, dtype=np.uint8)
    return Stream(name, tokens, offsets, np.asarray(users, dtype=np.uint32), en, meta or {})


def concat_streams(name: str, streams: list) -> Stream:
    prompts, users, enf = [], [], []
    any_en = any(s.enforce is not None for s in streams)
    for s in streams:
        for j in range(s.n_requests):
            prompts.append(s.tokens[int(s.offsets[j]):int(s.offsets[j + 1])])
        users.extend(s.users.tolist())
        enf.extend((s.enforce if s.enforce is not None else np.ones(s.n_requests, np.uint8)).tolist())
    return _pack(name, prompts, users, enf if any_en else None)


# --------------------------------------------------------------------------------------------
# C1 tiny: 4 users, 64 requests <= 512 tokens, scripted prompt-stealing attacker (BASELINE cfg 0)
# --------------------------------------------------------------------------------------------
K_SYS, K_TPL, K_KNOWN, K_FILL, K_TAIL, K_STEM, K_QUERY, K_PROFILE, K_MSG, K_REPLY, K_SUFFIX, \
    K_CAND = range(1, 13)


def c1_tiny(seed: int = 0x5011D001) -> Stream:
    """BASELINE.json configs[0].

    u0 = victim, u1/u2 = benign, u3 = attacker.  Victim prompt (240 tokens = 15 blocks):
    system(96) + template(64) + secret block #1 (15 known + 1 secret token) + filler(16)
    + secret block #2 (15 known + 1 secret) + tail(32).  The attacker probes block #1
    with 4 candidates (the correct one 3rd), then block #2 with the true block #1 (worst case) and
    4 candidates (correct one 2nd).  The schedule is fixed (non-adaptive), so the stream does not
    depend on any cache decision.  Benign users share the 96-token system prompt; half of their
    requests repeat an own earlier stem; lengths leave partial tails.
    """
    rng = np.random.default_rng(seed)
    sys_ = run(seed, K_SYS, 0, 96)
    tpl = run(seed, K_TPL, 0, 64)
    known1 = run(seed, K_KNOWN, 1, 15)
    known2 = run(seed, K_KNOWN, 2, 15)
    filler = run(seed, K_FILL, 0, 16)
    tail = run(seed, K_TAIL, 0, 32)
    cand = run(seed, K_CAND, 0, 8)          # 8 distinct-ish candidate tokens
    s1, s2 = int(cand[2]), int(cand[5])     # the secrets
    c1 = [int(cand[0]), int(cand[1]), s1, int(cand[3])]        # correct at index 3 (1-based)
    c2 = [int(cand[4]), s2, int(cand[6]), int(cand[7])]        # correct at index 2 (1-based)
    victim = np.concatenate([sys_, tpl, known1, [s1], filler, known2, [s2], tail]).astype(np.uint32)

    probes = []
    for c in c1:
        probes.append(np.concatenate([sys_, tpl, known1, [c], filler[:8]]).astype(np.uint32))
    for c in c2:
        probes.append(np.concatenate([sys_, tpl, known1, [s1], filler, known2, [c], tail[:5]])
                      .astype(np.uint32))

    stems = {1: [], 2: []}
    benign = []
    for i in range(54):
        u = 1 + (i % 2)
        if stems[u] and rng.random() < 0.5:
            stem = stems[u][int(rng.integers(len(stems[u])))]
        else:
            stem = run(seed, K_STEM, 1000 * u + len(stems[u]), int(rng.integers(16, 200)))
            stems[u].append(stem)
        q = run(seed, K_QUERY, i, int(rng.integers(1, 200)))
        p = np.concatenate([sys_, stem, q]).astype(np.uint32)[:512]
        benign.append((u, p))

    # schedule: victim first, victim repeat at 20; probes interleaved from request 4 on.
    prompts, users = [], []
    bi = pi = 0
    for t in range(64):
        if t == 0 or t == 20:
            prompts.append(victim); users.append(0)
        elif t >= 4 and t % 6 == 4 and pi < len(probes):
            prompts.append(probes[pi]); users.append(3); pi += 1
        elif bi < len(benign):
            u, p = benign[bi]; bi += 1
            prompts.append(p); users.append(u)
        else:
            prompts.append(probes[pi]); users.append(3); pi += 1
    assert pi == len(probes), (pi, len(probes))
    return _pack("c1_tiny", prompts, users,
                 meta=dict(victim_user=0, attacker_user=3, secret_tokens=[s1, s2],
                           cand_block1=c1, cand_block2=c2))


# --------------------------------------------------------------------------------------------
# C2 shared system prompt: 1k users x 100 requests, 2000-token prompts, 80% common prefix
# --------------------------------------------------------------------------------------------
def c2_shared_prompt(users: int = 1000, reqs_per_user: int = 100, sys_tokens: int = 1600,
                     profile_tokens: int = 256, query_tokens: int = 144,
                     seed: int = 0x5011D002, lo: int = 0, hi: int = -1) -> Stream:
    """BASELINE.json configs[1]: every request = common system prompt (1600 tokens = 100 blocks,
    80% of the prompt) + fixed per-user profile (256) + fresh query (144) = 2000 tokens = 125
    blocks.  Request order is a seeded shuffle of users x reqs_per_user.  [lo, hi) selects a
    contiguous slice of that global stream (a rank's share in the sharded benchmark) without
    materialising the rest."""
    n_all = users * reqs_per_user
    rng = np.random.default_rng(seed)
    order = np.repeat(np.arange(users, dtype=np.uint32), reqs_per_user)
    rng.shuffle(order)
    hi = n_all if hi < 0 else hi
    order = order[lo:hi]
    n = hi - lo
    L = sys_tokens + profile_tokens + query_tokens
    tok = np.empty((n, L), dtype=np.uint32)
    tok[:, :sys_tokens] = run(seed, K_SYS, 0, sys_tokens)
    if profile_tokens:
        uu = np.unique(order)
        prof = np.zeros((users, profile_tokens), dtype=np.uint32)
        for u in uu:
            prof[int(u)] = run(seed, K_PROFILE, int(u), profile_tokens)
        tok[:, sys_tokens:sys_tokens + profile_tokens] = prof[order]
    if query_tokens:
        base = _key(seed, K_QUERY, 0)
        with np.errstate(over="ignore"):
            idx = (np.arange(lo * query_tokens, hi * query_tokens, dtype=np.uint64) * _GOLD + base)
        tok[:, sys_tokens + profile_tokens:] = (_splitmix(idx) % np.uint64(VOCAB)).astype(
            np.uint32).reshape(n, query_tokens)
    offsets = np.arange(n + 1, dtype=np.uint64) * np.uint64(L)
    return Stream("c2_shared_prompt", tok.reshape(-1), offsets, order, None,
                  dict(users=users, reqs_per_user=reqs_per_user, prompt_tokens=L, lo=lo, hi=hi))


# --------------------------------------------------------------------------------------------
# C3 multi-turn chat: 10k users, conversations growing to 8k tokens, warm to ~1M cached blocks
# --------------------------------------------------------------------------------------------
def c3_multiturn(users: int = 10000, warm_blocks: int = 1_000_000, timed_rounds: int = 8,
                 sys_tokens: int = 256, max_ctx: int = 8192, seed: int = 0x5011D003):
    """BASELINE.json configs[2].  Returns (warm, timed) streams.

    Conversation = shared chat system prompt + turns (user msg U[32,256], assistant reply
    U[64,512]).  The request at turn t is the whole history through msg_t, so reply_{t-1} is
    cached only once it reappears in the next prompt.  A conversation longer than max_ctx
    restarts.  Each round issues one request per user in a shuffled order.  Warm rounds run until
    the cumulative number of distinct full blocks of the histories reaches warm_blocks (a token
    count, not a cache query); the next `timed_rounds` rounds form the timed stream."""
    rng = np.random.default_rng(seed)
    sys_ = run(seed, K_SYS, 0, sys_tokens)
    hist = [[sys_] for _ in range(users)]
    hist_len = np.full(users, sys_tokens, dtype=np.int64)
    conv = np.zeros(users, dtype=np.int64)
    turn = np.zeros(users, dtype=np.int64)
    pending_reply = [None] * users

    def one_round(r):
        order = rng.permutation(users)
        prompts, us = [], []
        new_blocks = 0
        for u in order:
            u = int(u)
            if pending_reply[u] is not None:
                hist[u].append(pending_reply[u]); hist_len[u] += len(pending_reply[u])
                pending_reply[u] = None
            mlen = int(rng.integers(32, 257))
            if hist_len[u] + mlen > max_ctx:
                conv[u] += 1; turn[u] = 0
                hist[u] = [sys_]; hist_len[u] = sys_tokens
            ident = (u * 4096 + int(conv[u])) * 4096 + int(turn[u])
            msg = run(seed, K_MSG, ident, mlen)
            before = hist_len[u] // 16
            hist[u].append(msg); hist_len[u] += mlen
            new_blocks += hist_len[u] // 16 - before
            prompts.append(np.concatenate(hist[u]))
            us.append(u)
            pending_reply[u] = run(seed, K_REPLY, ident, int(rng.integers(64, 513)))
            turn[u] += 1
        return prompts, us, new_blocks

    warm_p, warm_u, total = [], [], 0
    r = 0
    while total < warm_blocks:
        p, u, nb = one_round(r); r += 1
        warm_p += p; warm_u += u; total += nb
        if users * r > 50 * max(1, warm_blocks):   # safety for tiny configs
            break
    timed_p, timed_u = [], []
    for _ in range(timed_rounds):
        p, u, _nb = one_round(r); r += 1
        timed_p += p; timed_u += u
    meta = dict(users=users, warm_rounds=r - timed_rounds, timed_rounds=timed_rounds)
    return (_pack("c3_warm", warm_p, warm_u, meta=meta),
            _pack("c3_timed", timed_p, timed_u, meta=meta))


# --------------------------------------------------------------------------------------------
# C4 mixed benign + many attackers probing victim prefixes token by token, isolation-heavy
# --------------------------------------------------------------------------------------------
def c4_attackers(benign_users: int = 10000, benign_requests: int = 500_000, victims: int = 100,
                 templates: int = 10, victim_repeats: int = 10, colluders_per_victim: int = 10,
                 secret_blocks: int = 4, candidates: int = 125, sys_prompts: int = 8,
                 seed: int = 0x5011D004) -> Stream:
    """BASELINE.json configs[3] (defaults = 1M requests).

    Benign: sys_prompts x 512-token system prompts, a 128-token per-user part and 64 fresh tokens
    (704 tokens).  Victims: `templates` 512-token templates shared by victims/templates victims
    each; a victim prompt = template + secret_blocks x (15 known + 1 secret token) + 64 suffix,
    issued `victim_repeats` times.  Attackers: colluders_per_victim users per victim; together
    they probe every secret block s with `candidates` candidate tokens (true token at a seeded
    index >= 2), each probe carrying the TRUE blocks < s (worst case for the defense) and a 16-token
    suffix.  Requests are merged in a seeded random interleave, except that each victim's first
    request precedes all probes of that victim."""
    rng = np.random.default_rng(seed)
    sysp = [run(seed, K_SYS, i, 512) for i in range(sys_prompts)]
    tpl = [run(seed, K_TPL, i, 512) for i in range(templates)]
    sfx16 = run(seed, K_SUFFIX, 999, 16)
    items = []          # (priority key, user, prompt)
    # benign
    bu = rng.integers(0, benign_users, size=benign_requests)
    bprio = rng.random(benign_requests)
    qbase = _key(seed, K_QUERY, 0)
    with np.errstate(over="ignore"):
        qidx = np.arange(benign_requests * 64, dtype=np.uint64) * _GOLD + qbase
    queries = (_splitmix(qidx) % np.uint64(VOCAB)).astype(np.uint32).reshape(benign_requests, 64)
    sys_arr = np.stack(sysp)
    uniq = np.unique(bu)
    upart = np.zeros((benign_users, 128), dtype=np.uint32)
    for u in uniq:
        upart[int(u)] = run(seed, K_PROFILE, int(u), 128)
    btok = np.concatenate([sys_arr[bu % sys_prompts], upart[bu], queries], axis=1)
    for i in range(benign_requests):
        items.append((float(bprio[i]), 1 + int(bu[i]), btok[i]))
    # victims + probes
    vbase = 1 + benign_users
    abase = vbase + victims
    probes_per_victim = secret_blocks * candidates
    for v in range(victims):
        t = tpl[v % templates]
        known = [run(seed, K_KNOWN, v * 64 + s, 15) for s in range(secret_blocks)]
        secrets = run(seed, K_CAND, v, secret_blocks)
        true_blocks = [np.concatenate([known[s], secrets[s:s + 1]]) for s in range(secret_blocks)]
        vprompt = np.concatenate([t] + true_blocks + [run(seed, K_SUFFIX, v, 64)])
        first = float(rng.random()) * 0.5
        items.append((first, vbase + v, vprompt))
        for r in range(1, victim_repeats):
            items.append((first + float(rng.random()) * (1 - first), vbase + v, vprompt))
        k = 0
        for s in range(secret_blocks):
            true_idx = int(rng.integers(2, candidates))
            cands = run(seed, K_CAND, 1_000_000 + v * 64 + s, candidates)
            cands[true_idx] = secrets[s]
            # make the wrong candidates differ from the secret
            wrong = np.nonzero(cands == secrets[s])[0]
            for w in wrong:
                if w != true_idx:
                    cands[w] = (cands[w] + 1) % VOCAB
            for ci in range(candidates):
                p = np.concatenate([t] + true_blocks[:s] + [known[s], cands[ci:ci + 1], sfx16])
                # every colluder runs the whole probe sequence (500 probes each),
                # the colluders interleaved with jitter
                for c in range(colluders_per_victim):
                    a = abase + v * colluders_per_victim + c
                    items.append((first + (1 - first) * (k + float(rng.random())) /
                                  probes_per_victim, a, p))
                k += 1
    items.sort(key=lambda x: x[0])
    prompts = [it[2].astype(np.uint32) for it in items]
    users = [it[1] for it in items]
    return _pack("c4_attackers", prompts, users,
                 meta=dict(benign_users=benign_users, victims=victims,
                           attacker_base=abase, victim_base=vbase))


# --------------------------------------------------------------------------------------------
# random small streams for property / brute-force tests
# --------------------------------------------------------------------------------------------
def random_small(n_requests: int, users: int, alphabet_blocks: int, max_blocks: int,
                 block_size: int = 16, seed: int = 1, tail_prob: float = 0.5,
                 enforce_prob: float = 1.0, vocab: int = VOCAB) -> Stream:
    """Prompts built from a small alphabet of whole blocks (so prefixes collide often), with
    optional partial tails and random enforce bits."""
    rng = np.random.default_rng(seed)
    alpha = [run(seed, K_STEM, a, block_size, vocab) for a in range(alphabet_blocks)]
    prompts, us, en = [], [], []
    for i in range(n_requests):
        nb = int(rng.integers(0, max_blocks + 1))
        parts = [alpha[int(rng.integers(alphabet_blocks))] for _ in range(nb)]
        if rng.random() < tail_prob:
            parts.append(run(seed, K_QUERY, i, int(rng.integers(1, block_size)), vocab))
        prompts.append(np.concatenate(parts) if parts else np.zeros(0, np.uint32))
        us.append(int(rng.integers(users)))
        en.append(1 if rng.random() < enforce_prob else 0)
    return _pack(f"random_small_{seed}", prompts, us, en)
