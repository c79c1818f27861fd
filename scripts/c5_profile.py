"""One C5 batch (BASELINE configs[4], one GPU) for ncu: warm index admitted untimed, then the
4e6-request batch between cudaProfilerStart/Stop (run ncu with --profile-from-start off)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_10726_b200 as P  # noqa: E402
from workloads.c5 import c5_large  # noqa: E402

SEED = 0x5011D002
dev = torch.device("cuda", 0)
warm, timed = c5_large(scale=1.0)
cap = warm.n_blocks() + timed.n_blocks() // 4 + (1 << 16)
idx = P.Index("solidarity", capacity_blocks=cap,
              max_batch_tokens=max(warm.n_tokens, timed.n_tokens) + 64,
              max_batch_requests=max(warm.n_requests, timed.n_requests), seed=SEED, device=0,
              max_blocks=1024)
wt, wo, wu = warm.materialize_torch(dev)
idx.admit(wt, wo, wu, None)
torch.cuda.synchronize()
del wt, wo, wu
torch.cuda.empty_cache()
tt, to, tu = timed.materialize_torch(dev)
out = torch.empty((timed.n_requests, 6), dtype=torch.int32, device=dev)
torch.cuda.synchronize()
torch.cuda.profiler.start()
idx.admit_async(tt, to, tu, None, out=out)
idx.status()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
st = idx.stats()
print({k: st[k] for k in ("ms_hash", "ms_resolve", "ms_commit", "last_rounds", "last_inserted")})
