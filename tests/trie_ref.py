"""Content-keyed trie reference of the DESIGN.md §2 rules (TEST INFRASTRUCTURE, pin I10).

No hashing at all: an entry is named by the block CONTENTS of its path and by its namespace:
    ("S", (blk_1, ..., blk_b))                        Shared namespace
    ("I", (blk_1, ..., blk_f), u, (blk_f+1, ..., blk_b))   Iso(u) rooted at the Shared depth f
USER_ISOLATION uses ("I", (), u, path).  This is a different data structure from the hash-keyed
dict in oracle/solid_oracle.cpp (keys, namespace salts and the Iso closed form play no role here),
so agreement pins the oracle's key derivation and namespace handling.  Rules: P:454-459 with the
DESIGN.md readings R1-R11.
"""
from __future__ import annotations

NONE = 0xFFFFFFFF


class TrieRef:
    """capacity > 0 adds LRU eviction (SPEC evict_lru S:117-125, R22-R25), brute force:
    every entry carries last_used = the clock of the last request served it or that inserted it;
    after a request's inserts, while more than `capacity` entries are live, the one with the
    smallest (last_used, key) is removed by a linear scan.  `keyfn(name)` gives the entry's hash
    value, needed only for the tie-break ("ties broken by smaller hash value")."""

    def __init__(self, block_size: int = 16, policy: int = 2, capacity: int = 0, keyfn=None,
                 pool: int = 0, pin: bool = False):
        self.bs = block_size
        self.policy = policy
        self.table = {}     # name -> [owner, sharer]
        self.capacity = capacity
        self.keyfn = keyfn
        self.last_used = {}  # name -> clock
        self.clock = 0
        self.evictions = 0
        # physical blocks (R26-R28), brute force: every block carries the event stamp at which it
        # was last freed (never-used block i: stamp i - pool, before any event); a request's new
        # entries each take the free block with the smallest stamp, in block order, after the
        # request's evictions freed theirs
        self.pool = pool
        self.freed_at = {i: i - pool for i in range(pool)}   # free block -> stamp
        self.phys = {}                                       # name -> block
        self.events = 0
        self.fresh = []
        # in-flight pinning (R38), brute force: every admitted request adds one pin to each entry
        # of its row until released; eviction takes the min (last_used, key) over unpinned
        # entries only; a request that would need more victims than there are unpinned entries
        # it does not use itself is refused before anything changes
        self.pin = pin
        self.pins = {}                                       # name -> pin count

    class Refused(Exception):
        pass

    def _check(self, served, inserts):
        if not (self.pin and self.capacity):
            return
        new = [nm for nm in inserts if nm not in self.table]
        need = len(self.table) + len(new) - self.capacity
        own = set(served)
        avail = sum(1 for nm in self.table if self.pins.get(nm, 0) == 0 and nm not in own)
        if need > avail:
            raise TrieRef.Refused()

    def release(self, row):
        """Drop one pin per physical block of a row (NONE skipped)."""
        by_block = {b: nm for nm, b in self.phys.items() if nm in self.table}
        for b in row:
            if b == NONE:
                continue
            nm = by_block[b]
            assert self.pins.get(nm, 0) > 0
            self.pins[nm] -= 1

    def _served(self, names):
        for nm in names:
            self.last_used[nm] = self.clock

    def _insert(self, t, name, u):
        if name not in t:
            t[name] = [u, NONE]
            self.last_used[name] = self.clock
            self.fresh.append(name)

    def _evict(self):
        while self.capacity and len(self.table) > self.capacity:
            victim = min((nm for nm in self.table if self.pins.get(nm, 0) == 0),
                         key=lambda nm: (self.last_used[nm], self.keyfn(nm)))
            del self.table[victim]
            del self.last_used[victim]
            self.pins.pop(victim, None)
            self.evictions += 1
            if self.pool:
                self.freed_at[self.phys.pop(victim)] = self.events
                self.events += 1

    def _blocks(self, toks):
        n = len(toks) // self.bs
        return [tuple(int(t) for t in toks[i * self.bs:(i + 1) * self.bs]) for i in range(n)]

    def admit(self, toks, u: int, e: bool = True):
        blk = self._blocks(toks)
        n = len(blk)
        t = self.table
        k = r = flagd = 0
        f = -1
        self.fresh = []
        if self.policy == 1:
            names = [("I", (), u, tuple(blk[:b])) for b in range(1, n + 1)]
            while r < n and names[r] in t:
                r += 1
            self._check(names[:r], names[r:])
            self._served(names[:r])
            for b in range(r, n):
                self._insert(t, names[b], u)
            f = 0
            used = names
        else:
            shared = [("S", tuple(blk[:b])) for b in range(1, n + 1)]
            while k < n and shared[k] in t:
                k += 1
            if self.policy == 0:
                r = k
                self._check(shared[:k], shared[k:])
                self._served(shared[:k])
                for b in range(k, n):
                    self._insert(t, shared[b], u)
                used = shared
            else:
                if e:
                    for b in range(1, k + 1):
                        ent = t[shared[b - 1]]
                        nxt_own = t[shared[b]][0] if b < k else None
                        if ent[1] != NONE and not (b < k and nxt_own == u):
                            f = b
                            break
                if f < 0:
                    r = k
                    self._check(shared[:k], shared[k:])
                    if k >= 1:
                        ent = t[shared[k - 1]]
                        if ent[0] != u and ent[1] == NONE:
                            ent[1] = u
                            flagd = k
                    self._served(shared[:k])
                    for b in range(k, n):
                        self._insert(t, shared[b], u)
                    used = shared
                else:
                    root = tuple(blk[:f])
                    iso = [("I", root, u, tuple(blk[f:b])) for b in range(f + 1, n + 1)]
                    m = 0
                    while m < len(iso) and iso[m] in t:
                        m += 1
                    r = f + m
                    self._check(shared[:f] + iso[:m], iso[m:])
                    self._served(shared[:f] + iso[:m])
                    for name in iso[m:]:
                        self._insert(t, name, u)
                    used = shared[:f] + iso
        self._evict()
        if self.pool:
            for name in self.fresh:
                if not self.freed_at:
                    raise RuntimeError("pool exhausted")
                blk_id = min(self.freed_at, key=lambda i: self.freed_at[i])
                del self.freed_at[blk_id]
                self.phys[name] = blk_id
            self.table_row = [self.phys.get(nm, NONE) if nm in t else NONE for nm in used]
            if self.pin:
                for nm in used:
                    if nm in t:
                        self.pins[nm] = self.pins.get(nm, 0) + 1
        self.clock += 1
        bits = ((1 if r > 0 else 0) | (2 if (n > 0 and r == n) else 0) | (4 if f >= 0 else 0)
                | (8 if (f >= 0 and f < k) else 0) | (16 if flagd > 0 else 0))
        return (n, 0 if self.policy == 1 else k, r, f, flagd, bits)

    def entries(self):
        """[(name, owner, sharer)]"""
        return [(name, v[0], v[1]) for name, v in self.table.items()]
