"""Debug helper: first evict-mode mismatch against the oracle, with context."""
import sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from oracle import Oracle
from workloads import random_small
import paper_2603_10726_b200 as P
import torch

SEED = 0x5011D000
POL = {"apc": 0, "user_isolation": 1, "solidarity": 2}
policy, cap, batch, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
s = random_small(300, users=1 + seed, alphabet_blocks=3, max_blocks=6, seed=seed,
                 enforce_prob=0.8 if seed % 2 else 1.0)
o = Oracle(16, SEED, POL[policy], capacity=cap)
idx = P.Index(policy, capacity_blocks=cap, max_batch_tokens=s.n_tokens + 64,
              max_batch_requests=s.n_requests, max_blocks=8, seed=SEED, evict=True)

def show(b, lo, got, exp, before):
    st = idx.stats()
    print("MISMATCH in batch starting at", lo, "size", b.n_requests, "stats", {k: st[k] for k in ["last_evict_iters", "last_window_keys", "last_evicted", "last_rounds"]})
    print("table before (key, owner, sharer, lu):")
    for e in before:
        print("   ", hex(int(e["key"])), int(e["owner"]), hex(int(e["sharer"])), int(e["last_used"]))
    for j in range(b.n_requests):
        _, K = o.chain(b.tokens[int(b.offsets[j]):int(b.offsets[j+1])])
        print(j + lo, "user", int(b.users[j]), "en", None if b.enforce is None else int(b.enforce[j]),
              "got", tuple(got[j]), "exp", tuple(exp[j]), "*" if tuple(got[j]) != tuple(exp[j]) else "",
              [hex(int(k)) for k in K])
    print("gpu after:", [(hex(int(e["key"])), int(e["owner"]), hex(int(e["sharer"])), int(e["last_used"])) for e in idx.dump_ex()])
    print("orc after:", [(hex(int(e["key"])), int(e["owner"]), hex(int(e["sharer"])), int(e["last_used"])) for e in o.dump_ex()])
    sys.exit(0)


def admit(b, lo):
    try:
        before = o.dump_ex()
        got = P.as_numpy(idx.admit(**P.to_device(b)))
        torch.cuda.synchronize()
    except P.SolidError as e:
        h = b.n_requests // 2
        admit(b.slice(0, h), lo)
        admit(b.slice(h, b.n_requests), lo + h)
        return
    exp = o.process(b)
    if not np.array_equal(got, exp) or not np.array_equal(idx.dump_ex(), o.dump_ex()):
        show(b, lo, got, exp, before)


for lo in range(0, s.n_requests, batch):
    admit(s.slice(lo, min(lo + batch, s.n_requests)), lo)
print("all equal")
