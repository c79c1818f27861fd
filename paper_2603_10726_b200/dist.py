"""Sharded index driver: plumbing only.

Every step runs in the C ABI (`solid_dist_*` kernels); this module only moves the exchange
records between shards and runs the protocol of include/solid.h:

    begin -> [REG] -> owner_ingest(0) -> [PULL] -> { round(t) -> [INT] -> owner_ingest(t)
          -> allreduce(changed) -> [PULL] } -> commit (-> rollback on any overflow)

Two transports:
  * `TorchExchange` — one shard per process/GPU; counts by `all_to_all_single`, records by
    `all_to_all` over the process group (NCCL across GPUs; gloo works for host tensors).
  * `loopback_admit` — G shards in one process (tests, one GPU): records copied region to region.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

import numpy as np

from . import Index, RECORD_BYTES, SOLID_ERR_CAPACITY, SOLID_OK, SolidError, as_numpy


class _CudaBuf:
    """Zero-copy torch view of a device buffer owned by the library."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}


class ShardedIndex:
    """One shard of the key-hash-partitioned index (one C-ABI context with world > 1)."""

    def __init__(self, world: int, rank: int, policy: str = "solidarity", **kw):
        import torch
        self.world, self.rank, self.policy = world, rank, policy
        self.index = Index(policy, world=world, rank=rank, **kw)
        lib, h = self.index.lib, self.index.h
        send, recv, cap = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
        self.index._check(lib.solid_dist_buffers(h, ctypes.byref(send), ctypes.byref(recv),
                                                 ctypes.byref(cap)))
        self.cap = int(cap.value)
        nbytes = world * self.cap * RECORD_BYTES
        dev = torch.device("cuda", self.index.device)
        self.send = torch.as_tensor(_CudaBuf(send.value, nbytes), device=dev)
        self.recv = torch.as_tensor(_CudaBuf(recv.value, nbytes), device=dev)
        self.out = None

    # ---- regions (byte views) ------------------------------------------------------------
    def send_region(self, peer: int, records: int):
        o = peer * self.cap * RECORD_BYTES
        return self.send[o:o + records * RECORD_BYTES]

    def recv_region(self, peer: int, records: int):
        o = peer * self.cap * RECORD_BYTES
        return self.recv[o:o + records * RECORD_BYTES]

    def counts(self) -> np.ndarray:
        c = (ctypes.c_uint64 * self.world)()
        self.index._check(self.index.lib.solid_dist_counts(self.index.h, c))
        return np.array(list(c), dtype=np.int64)

    @staticmethod
    def _u64arr(v):
        return (ctypes.c_uint64 * len(v))(*[int(x) for x in v])

    # ---- protocol steps ------------------------------------------------------------------
    def begin(self, tokens, offsets, users, enforce=None, seq_base: int = 0, stream=None):
        import torch
        from . import _Batch
        n = int(users.numel())
        self.out = torch.empty((max(n, 1), 6), dtype=torch.int32, device=offsets.device)
        b = _Batch(n, tokens.data_ptr(), offsets.data_ptr(), users.data_ptr(),
                   enforce.data_ptr() if enforce is not None else None)
        self.n = n
        self.index._check(self.index.lib.solid_dist_begin(
            self.index.h, ctypes.byref(b), ctypes.c_void_p(self.out.data_ptr()), seq_base,
            Index._stream(stream)))
        return self.counts()

    def owner_ingest(self, phase: int, recv_counts, stream=None):
        """recv_counts None: device-resident counts (peer-memory exchange, device-counts mode)."""
        rc = None if recv_counts is None else self._u64arr(recv_counts)
        self.index._check(self.index.lib.solid_dist_owner_ingest(
            self.index.h, phase, rc, Index._stream(stream)))
        return None if recv_counts is None else self.counts()

    def round(self, t: int, recv_counts, stream=None):
        ch = ctypes.c_uint32()
        rc = None if recv_counts is None else self._u64arr(recv_counts)
        self.index._check(self.index.lib.solid_dist_round(
            self.index.h, t, rc, ctypes.byref(ch), Index._stream(stream)))
        return (None if recv_counts is None else self.counts()), int(ch.value)

    def commit(self, mode: int, stream=None):
        add = ctypes.c_uint64()
        rc = self.index.lib.solid_dist_commit(self.index.h, mode, ctypes.byref(add),
                                              Index._stream(stream))
        if rc not in (SOLID_OK, SOLID_ERR_CAPACITY):
            self.index._check(rc)
        return rc, int(add.value)

    def results(self):
        return self.out[:self.n]


# ------------------------------------------------------------------------------------------
# the protocol, shared by both transports
# ------------------------------------------------------------------------------------------
def run_protocol(shards_local: Sequence[ShardedIndex], begin_args, exchange, allreduce_max):
    """Drive the sharded admission for the shards owned by this process.

    exchange(send_counts_per_shard, flags=None) -> recv_counts_per_shard (moves the records);
    with flags (one int per local shard) it returns (recv_counts_per_shard, global max flag) —
    the round's "some decision changed" rides on the INT exchange's counts, so no separate
    all-reduce per round.  allreduce_max(list of ints) -> global max (the commit's overflow
    vote).  Returns the per-shard result tensors."""
    policy = shards_local[0].policy
    counts = [s.begin(*a) for s, a in zip(shards_local, begin_args)]
    recv = exchange(counts)                                       # REG
    counts = [s.owner_ingest(0, rc) for s, rc in zip(shards_local, recv)]
    recv = exchange(counts)                                       # PULL
    t = 1
    while True:
        outs = [s.round(t, rc) for s, rc in zip(shards_local, recv)]
        counts = [o[0] for o in outs]
        recv, changed = exchange(counts, flags=[o[1] for o in outs])   # INT (+ changed)
        counts = [s.owner_ingest(t, rc) for s, rc in zip(shards_local, recv)]
        if policy != "solidarity" or (t >= 2 and not changed):
            break
        recv = exchange(counts)                                   # PULL
        t += 1
        if t > 4093:
            raise SolidError(3, "sharded resolver did not converge")
    rcs = [s.commit(1)[0] for s in shards_local]
    if allreduce_max([int(rc == SOLID_ERR_CAPACITY) for rc in rcs]):
        for s in shards_local:
            s.commit(2)
        raise SolidError(SOLID_ERR_CAPACITY, "index shard capacity exceeded; batch rolled back")
    return [s.results() for s in shards_local], t


def loopback_admit(shards: List[ShardedIndex], local_batches, seq_bases):
    """All shards in this process: REG/PULL/INT records are copied region to region."""
    import torch
    G = len(shards)

    def exchange(send_counts, flags=None):
        recv_counts = [[int(send_counts[s][r]) for s in range(G)] for r in range(G)]
        for r in range(G):
            for s in range(G):
                k = recv_counts[r][s]
                if k:
                    shards[r].recv_region(s, k).copy_(shards[s].send_region(r, k))
        torch.cuda.synchronize()
        return recv_counts if flags is None else (recv_counts, max(flags))

    args = [(b["tokens"], b["offsets"], b["users"], b.get("enforce"), sb)
            for b, sb in zip(local_batches, seq_bases)]
    return run_protocol(shards, args, exchange, lambda xs: max(xs))


class DistTiming(ctypes.Structure):
    """solid_dist_timing (include/solid.h): rounds and exchange figures of one admission."""
    _fields_ = [("rounds", ctypes.c_uint32), ("exchanges", ctypes.c_uint32),
                ("exchange_ms", ctypes.c_float), ("record_bytes", ctypes.c_uint32),
                ("recv_records_remote", ctypes.c_uint64), ("recv_records_local", ctypes.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class PeerUnavailable(RuntimeError):
    """Some rank could not map its peers' regions (no CUDA IPC / peer access): raised on every
    rank alike, so callers can fall back to another transport together."""


class PeerExchange:
    """One shard per process on one node, records moved by the library itself over peer memory
    (solid_dist_p2p_*: CUDA IPC-mapped receive buffers, NVLink / NVSwitch stores, mailbox flags;
    DESIGN.md §7.4).  torch.distributed (any backend) only all-gathers the 64-byte handles once
    and takes the per-batch overflow vote."""

    def __init__(self, shard: ShardedIndex, group=None, device_counts: bool = False):
        """device_counts=True: counts stay on the device and only the INT exchange of each
        round synchronises the host (for the stop decision) — see admit()."""
        import torch.distributed as dist
        self.shard, self.group, self.device_counts = shard, group, device_counts
        lib, h = shard.index.lib, shard.index.h
        lib.solid_dist_p2p_export.restype = ctypes.c_int
        lib.solid_dist_p2p_export.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.solid_dist_p2p_connect.restype = ctypes.c_int
        lib.solid_dist_p2p_connect.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.solid_dist_p2p_exchange.restype = ctypes.c_int
        lib.solid_dist_p2p_exchange.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_void_p]
        mine = ctypes.create_string_buffer(64)
        ok = lib.solid_dist_p2p_export(h, mine) == SOLID_OK
        allh = [None] * shard.world
        dist.all_gather_object(allh, bytes(mine.raw) if ok else b"", group=self.group)
        ok = all(len(x) == 64 for x in allh)
        # every pair of GPUs must have peer access (NVLink / NVSwitch, or PCIe P2P); ranks on the
        # same device map each other's buffers directly
        import torch
        devs = [None] * shard.world
        dist.all_gather_object(devs, int(shard.index.device), group=self.group)
        me = int(shard.index.device)
        ok = ok and all(d == me or torch.cuda.can_device_access_peer(me, d) for d in devs)
        if ok:
            table = ctypes.create_string_buffer(b"".join(allh), 64 * shard.world)
            ok = lib.solid_dist_p2p_connect(h, table) == SOLID_OK
        votes = [None] * shard.world
        dist.all_gather_object(votes, ok, group=self.group)
        if not all(votes):
            raise PeerUnavailable("peer-memory exchange unavailable on some rank: "
                                  + shard.index.last_error())
        lib.solid_dist_p2p_device_counts.restype = ctypes.c_int
        lib.solid_dist_p2p_device_counts.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
        lib.solid_dist_p2p_exchange_dev.restype = ctypes.c_int
        lib.solid_dist_p2p_exchange_dev.argtypes = [ctypes.c_void_p, ctypes.c_uint32,
                                                    ctypes.c_void_p, ctypes.c_void_p]
        shard.index._check(lib.solid_dist_p2p_device_counts(h, 1 if device_counts else 0))
        dist.barrier(group=self.group)

    def exchange(self, send_counts_list, flags=None):
        sh = self.shard
        rc = (ctypes.c_uint64 * sh.world)()
        g = ctypes.c_uint32()
        sh.index._check(sh.index.lib.solid_dist_p2p_exchange(
            sh.index.h, 1 if flags and flags[0] else 0, rc, ctypes.byref(g), Index._stream(None)))
        recv = np.array(list(rc), dtype=np.int64)
        return [recv] if flags is None else ([recv], int(g.value))

    def allreduce_max(self, xs):
        import torch
        import torch.distributed as dist
        v = torch.tensor([max(xs)], dtype=torch.int64)
        if dist.get_backend(self.group) == "nccl":
            v = v.to(self.shard.send.device)
        dist.all_reduce(v, op=dist.ReduceOp.MAX, group=self.group)
        return int(v.item())

    def exchange_dev(self, sync: bool) -> int:
        sh = self.shard
        g = ctypes.c_uint32()
        sh.index._check(sh.index.lib.solid_dist_p2p_exchange_dev(
            sh.index.h, 1 if sync else 0, ctypes.byref(g), Index._stream(None)))
        return int(g.value)

    def admit_native(self, tokens, offsets, users, enforce=None, seq_base: int = 0):
        """The whole sharded admission as ONE C-ABI call (solid_dist_admit): agreement on the
        slices, rounds, commit and overflow vote run inside the library over peer memory.
        Returns (results tensor, DistTiming)."""
        import torch
        from . import _Batch
        sh = self.shard
        lib, h = sh.index.lib, sh.index.h
        if not getattr(lib, "_dist_admit_typed", False):
            lib.solid_dist_admit.restype = ctypes.c_int
            lib.solid_dist_admit.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
            lib._dist_admit_typed = True
        n = int(users.numel())
        sh.out = torch.empty((max(n, 1), 6), dtype=torch.int32, device=offsets.device)
        sh.n = n
        b = _Batch(n, tokens.data_ptr(), offsets.data_ptr(), users.data_ptr(),
                   enforce.data_ptr() if enforce is not None else None)
        tm = DistTiming()
        sh.index._check(lib.solid_dist_admit(h, ctypes.byref(b), ctypes.c_void_p(sh.out.data_ptr()),
                                             seq_base, ctypes.byref(tm), Index._stream(None)))
        return sh.results(), tm

    def admit(self, tokens, offsets, users, enforce=None, seq_base: int = 0):
        if not self.device_counts:
            res, rounds = run_protocol([self.shard], [(tokens, offsets, users, enforce, seq_base)],
                                       self.exchange, self.allreduce_max)
            return res[0], rounds
        return run_protocol_device(self.shard, (tokens, offsets, users, enforce, seq_base),
                                   self.exchange_dev, self.allreduce_max)


def run_protocol_device(shard: ShardedIndex, begin_args, exchange_dev, allreduce_max):
    """The protocol of run_protocol with device-resident counts (peer-memory exchange): the
    host only waits at each round's INT exchange (stop decision) and at the commit."""
    shard.begin(*begin_args)
    exchange_dev(False)                                           # REG
    shard.owner_ingest(0, None)
    exchange_dev(False)                                           # PULL
    t = 1
    while True:
        shard.round(t, None)
        changed = exchange_dev(True)                              # INT (+ changed)
        shard.owner_ingest(t, None)
        if shard.policy != "solidarity" or (t >= 2 and not changed):
            break
        exchange_dev(False)                                       # PULL
        t += 1
        if t > 4093:
            raise SolidError(3, "sharded resolver did not converge")
    rc = shard.commit(1)[0]
    if allreduce_max([int(rc == SOLID_ERR_CAPACITY)]):
        shard.commit(2)
        raise SolidError(SOLID_ERR_CAPACITY, "index shard capacity exceeded; batch rolled back")
    return shard.results(), t


class TorchExchange:
    """One shard per rank of a torch.distributed process group (NCCL for CUDA buffers).

    staging=True moves the records through host tensors (for a gloo group, whose point-to-point
    ops take CPU tensors: several ranks sharing one GPU in tests)."""

    def __init__(self, shard: ShardedIndex, group=None, staging: bool = False):
        self.shard, self.group, self.staging = shard, group, staging

    def exchange(self, send_counts_list, flags=None):
        """Counts by all_to_all_single, records by batched point-to-point (NCCL groups them;
        gloo supports it too, which the CPU tests use).  flags: this rank's flag is sent to every
        peer in bit 62 of the counts; returns (recv_counts, max flag over all ranks)."""
        import torch
        import torch.distributed as dist
        sh = self.shard
        rank = dist.get_rank(self.group)
        send_counts = np.asarray(send_counts_list[0], dtype=np.int64)
        wire = send_counts | (np.int64(1) << np.int64(62)) if flags and flags[0] else send_counts
        sc = torch.tensor(wire, device="cpu" if self.staging else sh.send.device)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=self.group)
        got = rc.cpu().numpy()
        recv_counts = got & ((np.int64(1) << np.int64(62)) - 1)
        gflag = int((got >> np.int64(62)).max()) if flags is not None else None
        if self.staging and sh.send.is_cuda:
            torch.cuda.synchronize()
        ops, landing = [], []
        for p in range(sh.world):
            ns, nr = int(send_counts[p]), int(recv_counts[p])
            if p == rank:
                if ns:
                    sh.recv_region(p, ns).copy_(sh.send_region(p, ns))
                continue
            if ns:
                src = sh.send_region(p, ns)
                ops.append(dist.P2POp(dist.isend, src.cpu() if self.staging else src, p,
                                      self.group))
            if nr:
                dst = sh.recv_region(p, nr)
                buf = torch.empty(dst.numel(), dtype=dst.dtype) if self.staging else dst
                ops.append(dist.P2POp(dist.irecv, buf, p, self.group))
                if self.staging:
                    landing.append((dst, buf))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for dst, buf in landing:
            dst.copy_(buf)
        if sh.send.is_cuda:
            torch.cuda.synchronize()
        return [recv_counts] if flags is None else ([recv_counts], gflag)

    def allreduce_max(self, xs):
        import torch
        import torch.distributed as dist
        v = torch.tensor([max(xs)], dtype=torch.int64,
                         device="cpu" if self.staging else self.shard.send.device)
        dist.all_reduce(v, op=dist.ReduceOp.MAX, group=self.group)
        return int(v.item())

    def admit(self, tokens, offsets, users, enforce=None, seq_base: int = 0):
        res, rounds = run_protocol([self.shard], [(tokens, offsets, users, enforce, seq_base)],
                                   self.exchange, self.allreduce_max)
        return res[0], rounds
