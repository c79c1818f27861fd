"""Per-request values that C5's structure fixes (workloads/c5.py), usable at full size without
the oracle (a check of the method's outcome, so it lives with the tests; bench.py uses it on its
timed batch).  For every request of the timed batch:

* continuing conversation (cached history prefix p + a new message): r = floor(p / 16), or one
  more when the block straddling the end of the prefix happens to be cached too (its few new-
  message tokens equal the conversation's next tokens, or an earlier request of the same user
  with the same cut sent the same ones: p mod 16 != 0 and ~1/32 000 per pair);
* new session (system prompt + 256 fresh tokens): r = 32 and diverted at 32 — the end of every
  system prompt is flagged since the warm phase (R7);
* probe (system prompt + victim profile[0:255] + candidate + suffix): diverted at 32 — no probe
  is ever served the victim's entries beyond the system prompt (the §5 guarantee);
  r = 32 for an attacker's first probe, then 47 (its own isolated copy of profile[0:240]), 48
  only when the same attacker already sent the same candidate token.
"""
import numpy as np

from workloads.gen import VOCAB, _GOLD, _splitmix


def c5_check(timed, got):
    U = timed.meta["users"]
    segs = np.diff(timed.ptr)
    attacker = timed.users >= U
    new = (segs == 2) & ~attacker
    cont = ~new & ~attacker
    seg_end = np.concatenate([[0], np.cumsum(timed.length)])
    prefix = seg_end[timed.ptr[1:] - 1] - seg_end[timed.ptr[:-1]]
    r = got["reused"].astype(np.int64)
    f = got["divert_at"].astype(np.int64)
    base = prefix // 16
    extra = r - base
    cont_bad = cont & ~((extra == 0) | ((extra == 1) & (prefix % 16 != 0)))
    ai = np.nonzero(attacker)[0]
    cs = timed.ptr[ai] + 2                               # the candidate's 1-token segment
    with np.errstate(over="ignore"):
        tok = (_splitmix(timed.start[cs].astype(np.uint64) * _GOLD + timed.key[cs])
               % np.uint64(VOCAB)).astype(np.int64)
    att = timed.users[ai].astype(np.int64)
    pair = att * VOCAB + tok
    seen_att = np.zeros(ai.size, bool)
    seen_att[np.unique(att, return_index=True)[1]] = True          # first probe of the attacker
    rep_tok = np.ones(ai.size, bool)
    rep_tok[np.unique(pair, return_index=True)[1]] = False         # token sent before by it
    exp_probe = np.where(seen_att, 32, np.where(rep_tok, 48, 47))
    bad = {"continuing": int(cont_bad.sum()),
           "new_session": int(((r[new] != 32) | (f[new] != 32)).sum()),
           "probe_not_diverted_at_32": int((f[ai] != 32).sum()),
           "probe_reuse": int((r[ai] != exp_probe).sum())}
    return {"status": "exact" if not any(bad.values()) else "MISMATCH", "violations": bad,
            "continuing_straddle_hits": int((cont & (extra == 1)).sum()),
            "probe_repeated_tokens": int(rep_tok.sum()),
            "requests_checked": int(cont.sum() + new.sum() + ai.size),
            "counts": (int(cont.sum()), int(new.sum()), int(ai.size))}
