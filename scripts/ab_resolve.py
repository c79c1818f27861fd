"""A/B of resolver variants chosen by environment variables read at solid_init (one process).

  python scripts/ab_resolve.py 'SOLID_STAMP=1' 'SOLID_STAMP=0' ...   [--configs c2,c4] [--reps 5]

Per variant and config: median batch time (CUDA events around admit_async, index restored to the
same pre-batch state before each batch), resolver rounds and per-round times (device timer).
Every variant's results are compared with the first variant's (exactness check across variants).
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_10726_b200 as P  # noqa: E402
from workloads import c2_shared_prompt, c3_multiturn, c4_attackers  # noqa: E402

SEED = 0x5011D002


def load(cfg):
    if cfg == "c2":
        return c2_shared_prompt(), []
    if cfg == "c3":
        w, s = c3_multiturn()
        return s, [w]
    return c4_attackers(), []


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--configs", default="c2,c3,c4")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    for cfg in a.configs.split(","):
        s, pre = load(cfg)
        d = P.to_device(s, "cuda:0")
        pre_d = [P.to_device(w, "cuda:0") for w in pre]
        mt = max([s.n_tokens] + [w.n_tokens for w in pre]) + 64
        mr = max([s.n_requests] + [w.n_requests for w in pre])
        blocks = s.n_blocks() + sum(w.n_blocks() for w in pre)
        ref = None
        for v in a.variants:
            env = dict(kv.split("=", 1) for kv in v.split(",") if kv and not kv.startswith("lib="))
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            idx = P.Index("solidarity", capacity_blocks=max(blocks, 1 << 20), max_batch_tokens=mt,
                          max_batch_requests=mr, seed=SEED, device=0)
            for k, val in old.items():
                if val is None:
                    os.environ.pop(k)
                else:
                    os.environ[k] = val
            for w in pre_d:
                idx.admit(**w)
            idx.checkpoint()
            o = torch.empty((s.n_requests, 6), dtype=torch.int32, device="cuda:0")
            ms, rounds, rus = [], [], []
            for k in range(2 + a.reps):
                idx.restore()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                idx.admit_async(d["tokens"], d["offsets"], d["users"], d["enforce"], out=o)
                e1.record()
                idx.status()
                if k >= 2:
                    ms.append(e0.elapsed_time(e1))
                    st = idx.stats()
                    rounds.append(st["last_rounds"])
                    rus.append([round(x, 1) for x in st["round_us"] if x > 0])
            st = idx.stats()
            r = P.as_numpy(o)
            same = ""
            if ref is None:
                ref = r.copy()
            else:
                same = "same" if all(np.array_equal(r[f], ref[f]) for f in r.dtype.names) else "DIFFERENT"
            print(f"{cfg} [{v}] ms {statistics.median(ms):.4f} hash {st['ms_hash']:.3f} "
                  f"resolve {st['ms_resolve']:.3f} commit {st['ms_commit']:.3f} rounds {rounds[-1]} "
                  f"round_us {rus[-1]} ids {st['last_distinct_keys']} {same}", flush=True)
            del idx, o
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
