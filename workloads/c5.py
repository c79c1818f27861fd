"""C5 — the large index (BASELINE.json configs[4], SURVEY §8(d) "C5 large sharded index").

A warm phase that fills the index to ~1.0e8 entries, then ONE timed batch of 4e6 requests:
50 % continuing conversations (a prefix of the user's cached conversation + a new message,
~1.2 k tokens on average), 40 % new sessions (one of 16 system prompts x 512 tokens + 256 fresh
tokens) and 10 % C4-style probes (colluding attackers trying 125 candidates for the last token
of a victim's profile).  T ~ 4.1e9 tokens in the timed batch.

Recipe (every count scales with `scale`; scale = 1 is the configuration BASELINE names):
  * users U = 200 000 x scale; user u's conversation = system prompt S[u mod 16] (512 tokens)
    + profile_u (256) + turns (message U[32, 256], reply U[64, 512]) until its length reaches a
    per-user target U[6 700, 10 700] tokens (last segment cut) — ~512 distinct blocks per user
    beyond the shared system prompt, so the warm phase (one request per user = the whole
    conversation, seeded order) leaves ~1.0e8 entries at scale 1;
  * continuing request: the user's conversation cut after m segments (m uniform in
    [2, m_max(u)], m_max = the last segment boundary within 1 800 tokens) + a fresh message
    U[32, 256];
  * new session: S[k] (k uniform) + 256 fresh tokens, user uniform;
  * probes: 320 x scale victims (users 0..), 10 colluding attackers each (user ids U + ...),
    every attacker sends the whole candidate sequence: S[v mod 16] + profile_v[0:255] +
    candidate token + 16 fresh tokens; candidate index 0..124, the true token (profile_v[255])
    at a seeded index >= 2;
  * the timed batch is a seeded shuffle of all of them.

Tokens are counter-based exactly as workloads/gen.py: a segment (kind, ident) has token i =
splitmix64(key(seed, kind, ident) + i * GOLD) mod 32 000.  A prompt is a list of (key, start,
length) segments, so the stream is held as a segment table and materialised either with numpy
(host, for the oracle) or with torch on a device (the GPU path; 16 GB of tokens need not go
through host memory).  Both evaluate the same function (tests/test_workloads_c5.py checks they
agree).  Nothing here hashes blocks or applies a rule of the method.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .gen import (VOCAB, K_CAND, K_MSG, K_PROFILE, K_QUERY, K_REPLY, K_SUFFIX, K_SYS, Stream,
                  _GOLD, _splitmix)

K_NEWMSG = 21
SEED = 0x5011D005
MASK = (1 << 64) - 1


def _keys(seed: int, kind: int, ident: np.ndarray) -> np.ndarray:
    """Vectorised gen._key(seed, kind, ident): splitmix(splitmix(seed ^ kind) ^ ident)."""
    k0 = _splitmix(np.array([seed & MASK], dtype=np.uint64) ^ np.uint64(kind))
    return _splitmix(k0 ^ np.asarray(ident, dtype=np.uint64))


@dataclass
class SegStream:
    """Requests as segment lists: request j = segments [ptr[j], ptr[j+1]) in order; segment s =
    tokens start[s] .. start[s] + length[s] - 1 of the counter stream `key[s]`."""
    name: str
    key: np.ndarray        # uint64[S]
    start: np.ndarray      # int64[S]
    length: np.ndarray     # int64[S]
    ptr: np.ndarray        # int64[N+1]
    users: np.ndarray      # uint32[N]
    meta: dict

    @property
    def n_requests(self) -> int:
        return int(self.users.shape[0])

    def offsets(self) -> np.ndarray:
        tok = np.concatenate([[0], np.cumsum(self.length)])
        return tok[self.ptr].astype(np.uint64)

    @property
    def n_tokens(self) -> int:
        return int(self.length.sum())

    def n_blocks(self) -> int:
        return int((np.diff(self.offsets().astype(np.int64)) // 16).sum())

    def materialize(self, chunk_tokens: int = 1 << 19, threads: int = 4) -> Stream:
        """numpy (host) tokens, in cache-sized chunks of segments over a thread pool (numpy
        releases the GIL in its ufuncs)."""
        import os
        from concurrent.futures import ThreadPoolExecutor
        T = self.n_tokens
        out = np.empty(T, dtype=np.uint32)
        seg_off = np.concatenate([[0], np.cumsum(self.length)])
        S = self.key.shape[0]
        cuts = [0]
        while cuts[-1] < S:
            s = cuts[-1]
            e = int(np.searchsorted(seg_off, seg_off[s] + chunk_tokens, side="right")) - 1
            cuts.append(min(max(e, s + 1), S))

        def work(i):
            s, e = cuts[i], cuts[i + 1]
            lens = self.length[s:e]
            n = int(lens.sum())
            rel = np.arange(n, dtype=np.int64) - np.repeat(seg_off[s:e] - seg_off[s], lens)
            idx = (rel + np.repeat(self.start[s:e], lens)).astype(np.uint64)
            with np.errstate(over="ignore"):
                x = idx * _GOLD + np.repeat(self.key[s:e], lens)
            out[seg_off[s]:seg_off[s] + n] = (_splitmix(x) % np.uint64(VOCAB)).astype(np.uint32)

        with ThreadPoolExecutor(threads or min(16, os.cpu_count() or 1)) as ex:
            list(ex.map(work, range(len(cuts) - 1)))
        return Stream(self.name, out, self.offsets(), self.users.copy(), None, dict(self.meta))

    def materialize_torch(self, device, chunk_tokens: int = 1 << 27):
        """The same tokens generated by torch on `device` (int32, CUDA or CPU); returns
        (tokens, offsets, users) tensors laid out like paper_2603_10726_b200.to_device."""
        import torch
        T = self.n_tokens
        out = torch.empty(max(T, 1), dtype=torch.int32, device=device)
        seg_off = np.concatenate([[0], np.cumsum(self.length)])
        S = self.key.shape[0]
        m2 = {s: torch.tensor(np.int64(np.uint64(v).view(np.int64)), device=device)
              for s, v in (("g", 0x9E3779B97F4A7C15), ("m1", 0xBF58476D1CE4E5B9),
                           ("m2", 0x94D049BB133111EB))}
        two64_mod_v = (1 << 64) % VOCAB

        def lsr(x, k):
            return (x >> k) & ((1 << (64 - k)) - 1)

        s = 0
        while s < S:
            e = int(np.searchsorted(seg_off, seg_off[s] + chunk_tokens, side="right")) - 1
            e = min(max(e, s + 1), S)
            lens = torch.from_numpy(self.length[s:e]).to(device)
            n = int(self.length[s:e].sum())
            base = torch.from_numpy(seg_off[s:e] - seg_off[s]).to(device)
            rel = torch.arange(n, dtype=torch.int64, device=device) - \
                torch.repeat_interleave(base, lens)
            idx = rel + torch.repeat_interleave(torch.from_numpy(self.start[s:e]).to(device), lens)
            key = torch.repeat_interleave(
                torch.from_numpy(self.key[s:e].view(np.int64)).to(device), lens)
            z = idx * m2["g"] + key + m2["g"]            # splitmix64(x), x = idx * GOLD + key
            z = (z ^ lsr(z, 30)) * m2["m1"]
            z = (z ^ lsr(z, 27)) * m2["m2"]
            z = z ^ lsr(z, 31)
            r = torch.remainder(z, VOCAB)                # unsigned z mod V from the signed value
            r = torch.where(z < 0, torch.remainder(r + two64_mod_v, VOCAB), r)
            out[seg_off[s]:seg_off[s] + n] = r.to(torch.int32)
            s = e
        offs = torch.from_numpy(self.offsets().view(np.int64)).to(device)
        users = torch.from_numpy(self.users.view(np.int32)).to(device)
        return out, offs, users


def c5_large(scale: float = 1.0, seed: int = SEED):
    """Returns (warm, timed) SegStreams (module docstring)."""
    rng = np.random.default_rng(seed)
    U = max(16, int(round(200_000 * scale)))
    sys_keys = _keys(seed, K_SYS, np.arange(16))
    # ---- conversations: per user sys + profile + up to MT (msg, reply) pairs, cut at target
    MT = 64
    target = rng.integers(6700, 10701, size=U)
    msg = rng.integers(32, 257, size=(U, MT))
    rep = rng.integers(64, 513, size=(U, MT))
    seg_len = np.empty((U, 2 + 2 * MT), dtype=np.int64)
    seg_len[:, 0] = 512
    seg_len[:, 1] = 256
    seg_len[:, 2::2] = msg
    seg_len[:, 3::2] = rep
    cum = np.cumsum(seg_len, axis=1)
    nseg = (cum < target[:, None]).sum(axis=1) + 1           # segments until target reached
    last = nseg - 1
    seg_len[np.arange(U), last] -= cum[np.arange(U), last] - target   # cut the last segment
    uid = np.arange(U, dtype=np.uint64)
    turn_ident = (uid[:, None] * np.uint64(4096) + np.arange(MT, dtype=np.uint64)[None, :])
    seg_key = np.empty((U, 2 + 2 * MT), dtype=np.uint64)
    seg_key[:, 0] = sys_keys[np.arange(U) % 16]
    seg_key[:, 1] = _keys(seed, K_PROFILE, uid)
    seg_key[:, 2::2] = _keys(seed, K_MSG, turn_ident.reshape(-1)).reshape(U, MT)
    seg_key[:, 3::2] = _keys(seed, K_REPLY, turn_ident.reshape(-1)).reshape(U, MT)
    valid = np.arange(2 + 2 * MT)[None, :] < nseg[:, None]

    # ---- warm: one request per user (the whole conversation), seeded order
    worder = rng.permutation(U)
    wv = valid[worder]
    w_key = seg_key[worder][wv]
    w_len = seg_len[worder][wv]
    w_ptr = np.concatenate([[0], np.cumsum(nseg[worder])]).astype(np.int64)
    warm = SegStream("c5_warm", w_key, np.zeros_like(w_len), w_len, w_ptr,
                     worder.astype(np.uint32), dict(users=U, scale=scale))

    # ---- timed batch
    N = int(round(4_000_000 * scale))
    V = max(1, int(round(320 * scale)))
    C, CAND = 10, 125
    n_probe = V * C * CAND
    n_cont = N // 2
    n_new = max(N - n_cont - n_probe, 0)
    kinds = np.concatenate([np.zeros(n_cont, np.int8), np.ones(n_new, np.int8),
                            np.full(n_probe, 2, np.int8)])
    kinds = kinds[rng.permutation(kinds.size)]
    rid = np.arange(kinds.size, dtype=np.uint64)               # request ident for fresh parts
    segs_per = np.where(kinds == 1, 2, 5).astype(np.int64)
    # continuing: m history segments + 1 new message
    ci = np.nonzero(kinds == 0)[0]
    cu = rng.integers(0, U, size=ci.size)
    m_max = np.maximum((cum[cu] <= 1800).sum(axis=1), 2)
    m_max = np.minimum(m_max, nseg[cu])
    m = rng.integers(2, m_max + 1)
    segs_per[ci] = m + 1
    ptr = np.concatenate([[0], np.cumsum(segs_per)]).astype(np.int64)
    S = int(ptr[-1])
    key = np.zeros(S, np.uint64)
    start = np.zeros(S, np.int64)
    length = np.zeros(S, np.int64)
    users = np.zeros(kinds.size, np.uint32)
    # continuing: history prefix (vectorised over the segment index)
    users[ci] = cu
    pos = ptr[ci]
    for q in range(int(m.max()) if m.size else 0):
        sel = q < m
        key[pos[sel] + q] = seg_key[cu[sel], q]
        length[pos[sel] + q] = seg_len[cu[sel], q]
    nm = pos + m
    key[nm] = _keys(seed, K_NEWMSG, rid[ci])
    length[nm] = rng.integers(32, 257, size=ci.size)
    # new sessions
    ni = np.nonzero(kinds == 1)[0]
    users[ni] = rng.integers(0, U, size=ni.size)
    p0 = ptr[ni]
    key[p0] = sys_keys[rng.integers(0, 16, size=ni.size)]
    length[p0] = 512
    key[p0 + 1] = _keys(seed, K_QUERY, rid[ni])
    length[p0 + 1] = 256
    # probes (victim v, colluder c, candidate q): attacker (v, c) sends its candidates in order,
    # the attackers interleaved — probe times (q + jitter) / CAND, sorted onto the probe slots
    pi = np.nonzero(kinds == 2)[0]
    vv = np.repeat(np.arange(V), C * CAND)
    cc = np.tile(np.repeat(np.arange(C), CAND), V)
    qq = np.tile(np.arange(CAND), V * C)
    t = (qq + rng.random(n_probe)) / CAND
    assign = np.empty(n_probe, np.int64)
    assign[np.argsort(t, kind="stable")] = pi
    grp = vv * C + cc
    p0 = ptr[assign]
    users[assign] = (U + grp).astype(np.uint32)
    true_idx = rng.integers(2, CAND, size=V)
    prof_keys = _keys(seed, K_PROFILE, np.arange(V, dtype=np.uint64))
    key[p0] = sys_keys[vv % 16]
    length[p0] = 512
    key[p0 + 1] = prof_keys[vv]
    length[p0 + 1] = 255
    is_true = qq == true_idx[vv]
    key[p0 + 2] = np.where(is_true, prof_keys[vv], _keys(seed, K_CAND, vv.astype(np.uint64)))
    start[p0 + 2] = np.where(is_true, 255, qq)
    length[p0 + 2] = 1
    key[p0 + 3] = _keys(seed, K_SUFFIX, rid[assign])
    length[p0 + 3] = 16
    # a zero-length pad keeps 5 segments per probe (no tokens)
    key[p0 + 4] = key[p0 + 3]
    length[p0 + 4] = 0
    timed = SegStream("c5_timed", key, start, length, ptr, users,
                      dict(users=U, scale=scale, continuing=int(ci.size), new_sessions=int(ni.size),
                           probes=int(pi.size), victims=V, attacker_base=U))
    return warm, timed
