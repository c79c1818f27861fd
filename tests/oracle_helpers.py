"""Shared helpers for the oracle pin tests (test infrastructure)."""
import numpy as np

from oracle import Oracle
from workloads.gen import run

NONE = 0xFFFFFFFF


class Blocks:
    """Symbolic 16-token blocks: Blocks()['T1'] is a fixed random block per name."""

    def __init__(self, seed=12345, bs=16):
        self.seed, self.bs, self.ids = seed, bs, {}

    def __getitem__(self, name):
        if name not in self.ids:
            self.ids[name] = len(self.ids)
        return run(self.seed, 77, self.ids[name], self.bs)

    def prompt(self, names, tail=0):
        parts = [self[n] for n in names]
        if tail:
            parts.append(run(self.seed, 78, len(names) * 1000 + tail, tail))
        return np.concatenate(parts) if parts else np.zeros(0, np.uint32)


def table_as_dict(o: Oracle):
    d = o.dump()
    return {int(e["key"]): (int(e["owner"]), int(e["sharer"])) for e in d}


def lcp_blocks(a, b, bs=16):
    n = min(len(a) // bs, len(b) // bs)
    k = 0
    while k < n and np.array_equal(a[k * bs:(k + 1) * bs], b[k * bs:(k + 1) * bs]):
        k += 1
    return k


def prompts_of(stream):
    return [stream.tokens[int(stream.offsets[j]):int(stream.offsets[j + 1])]
            for j in range(stream.n_requests)]
