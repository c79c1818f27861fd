"""Per-round resolver path counters on the bench workload (profiling build; perturbs timing).

  python -m paper_2603_10726_b200.build --counters
  SOLID_LIB=paper_2603_10726_b200/lib/libsolid_counters.so python scripts/counters.py
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_10726_b200 as P  # noqa: E402
from workloads import c2_shared_prompt, c3_multiturn, c4_attackers  # noqa: E402

NAMES = ["evaluated", "changed", "new_divert", "same_divert", "flag_atomic", "insert_atomics",
         "walk_k", "iso_blocks", "stamp_fired", "stamp_checks", "defer_pass_ns", "deferred"]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    pre = []
    if cfg == "c2":
        s = c2_shared_prompt()
    elif cfg == "c3":
        w, s = c3_multiturn()
        pre = [w]
    else:
        s = c4_attackers()
    mt = max([s.n_tokens] + [w.n_tokens for w in pre]) + 64
    mr = max([s.n_requests] + [w.n_requests for w in pre])
    blocks = s.n_blocks() + sum(w.n_blocks() for w in pre)
    idx = P.Index("solidarity", capacity_blocks=max(blocks, 1 << 20),
                  max_batch_tokens=mt, max_batch_requests=mr)
    for w in pre:
        idx.admit(**P.to_device(w))
    d = P.to_device(s)
    idx.admit(**d)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 192)()
    rc = idx.lib.solid_debug_counters(idx.h, buf)
    assert rc == 0, "not the counters build (set SOLID_LIB)"
    c = np.array(buf, dtype=np.uint64).reshape(16, 12)
    st = idx.stats()
    print("rounds", st["last_rounds"], "round_us", [round(x, 1) for x in st["round_us"]])
    print("K_A2 registration: stab_probes", int(c[0][0]), "cas", int(c[0][1]), "cas_failed",
          int(c[0][2]), "guess_atomics", int(c[0][3]))
    print("t  " + " ".join(f"{n:>14s}" for n in NAMES))
    for t in range(1, st["last_rounds"] + 1):
        print(f"{t:<3d}" + " ".join(f"{int(v):14d}" for v in c[t]))


if __name__ == "__main__":
    main()
