"""e2e (host-buffer admission, 16-bit ids) of C2 under environment-variable variants, beside a
plain pinned copy of the same bytes.   python scripts/e2e_ab.py 'SOLID_HOST_CHUNKS=4' ..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_10726_b200 as P  # noqa: E402
from workloads import c2_shared_prompt  # noqa: E402

SEED = 0x5011D002
s = c2_shared_prompt(seed=SEED + 2)
N, nblk = s.n_requests, s.n_blocks()
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
h16, ho, hu = pin(s.tokens.astype(np.uint16)), pin(s.offsets), pin(s.users)
hout = torch.zeros(N * P.RESULT_DTYPE.itemsize, dtype=torch.uint8).pin_memory().numpy().view(P.RESULT_DTYPE)
src = torch.from_numpy(h16.view(np.uint8)).pin_memory()
dst = torch.empty(src.numel(), dtype=torch.uint8, device="cuda:0")
for v in sys.argv[1:] * 2:
    env = dict(kv.split("=", 1) for kv in v.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    idx = P.Index("solidarity", capacity_blocks=max(nblk // 6, 1 << 20),
                  max_batch_tokens=s.n_tokens + 64, max_batch_requests=N, seed=SEED, device=0)
    for k, val in old.items():
        os.environ.pop(k) if val is None else os.environ.__setitem__(k, val)
    ts = []
    for step in range(6):
        idx.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        idx.admit_host_u16(h16, ho, hu, None, out=hout)
        if step:
            ts.append(time.perf_counter() - t0)
    cps = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        cps.append(time.perf_counter() - t0)
    med = sorted(ts)[len(ts) // 2]
    print(f"[{v}] e2e {med * 1e3:.3f} ms = {N / med / 1e6:.2f} M req/s (min {min(ts) * 1e3:.3f}); "
          f"plain copy of the tokens {min(cps) * 1e3:.3f} ms; reused {int(hout['reused'].sum())}",
          flush=True)
    del idx
    torch.cuda.empty_cache()
