"""Host logic of the sharded index on CPU (gloo, world_size 2): the record exchange (counts by
all_to_all_single, records by batched point-to-point) and the protocol driver's round /
convergence / rollback coordination, with fake shards standing in for the CUDA contexts."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_10726_b200 import RECORD_BYTES, SOLID_ERR_CAPACITY, SOLID_OK, SolidError
from paper_2603_10726_b200.dist import TorchExchange, run_protocol


class FakeShard:
    """Host-tensor stand-in with the ShardedIndex interface used by the driver."""

    def __init__(self, world, rank, cap=8, policy="solidarity", converge_at=3, overflow=False):
        self.world, self.rank, self.cap, self.policy = world, rank, cap, policy
        self.send = torch.zeros(world * cap * RECORD_BYTES, dtype=torch.uint8)
        self.recv = torch.zeros_like(self.send)
        self.log = []
        self.converge_at, self.overflow = converge_at, overflow

    def send_region(self, peer, records):
        o = peer * self.cap * RECORD_BYTES
        return self.send[o:o + records * RECORD_BYTES]

    def recv_region(self, peer, records):
        o = peer * self.cap * RECORD_BYTES
        return self.recv[o:o + records * RECORD_BYTES]

    def _pack(self, tag):
        # peer p gets (rank + p + 1) records stamped with (tag, rank, p)
        counts = np.array([self.rank + p + 1 for p in range(self.world)], dtype=np.int64)
        for p in range(self.world):
            self.send_region(p, int(counts[p])).fill_((tag * 16 + self.rank * 4 + p) % 256)
        return counts

    def _check_recv(self, tag, recv_counts):
        for s in range(self.world):
            assert recv_counts[s] == s + self.rank + 1
            reg = self.recv_region(s, int(recv_counts[s]))
            assert (reg == (tag * 16 + s * 4 + self.rank) % 256).all()

    def begin(self, *a):
        self.log.append("begin")
        return self._pack(1)

    def owner_ingest(self, phase, rc):
        self.log.append(f"ingest{phase}")
        self._check_recv(1 if phase == 0 else 3, rc)
        return self._pack(2)

    def round(self, t, rc):
        self.log.append(f"round{t}")
        self._check_recv(2, rc)
        # rank 1 changes its decisions until converge_at - 1, rank 0 never after round 1
        changed = int(t == 1 or (self.rank == 1 and t < self.converge_at))
        return self._pack(3), changed

    def commit(self, mode):
        self.log.append(f"commit{mode}")
        if mode == 1 and self.overflow:
            return SOLID_ERR_CAPACITY, 0
        return SOLID_OK, 0

    def results(self):
        return self.log


def _worker(rank, world, port, overflow_rank, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = FakeShard(world, rank, overflow=(rank == overflow_rank))
        ex = TorchExchange(sh)
        try:
            res, t = run_protocol([sh], [()], ex.exchange, ex.allreduce_max)
            q.put((rank, "ok", t, sh.log))
        except SolidError as e:
            q.put((rank, "err", e.status, sh.log))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(overflow_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, overflow_rank, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def test_exchange_and_protocol_world2_gloo():
    out = _spawn(overflow_rank=-1)
    for rank, status, t, log in out:
        assert status == "ok"
        # rank 1 keeps changing until round 2 -> converged (no change) at round 3 on both ranks
        assert t == 3
        assert log == ["begin", "ingest0", "round1", "ingest1", "round2", "ingest2", "round3",
                       "ingest3", "commit1"]


def test_overflow_on_one_shard_rolls_back_everywhere():
    out = _spawn(overflow_rank=1)
    for rank, status, code, log in out:
        assert status == "err" and code == SOLID_ERR_CAPACITY
        assert log[-2:] == ["commit1", "commit2"]


class FakeDevShard(FakeShard):
    """Device-counts mode stand-in: the protocol passes no counts; the round's changed flag
    travels with the next synchronised exchange (run_protocol_device)."""

    def owner_ingest(self, phase, rc):
        assert rc is None
        self.log.append(f"ingest{phase}")

    def round(self, t, rc):
        assert rc is None
        self.log.append(f"round{t}")
        self.changed = int(t == 1 or (self.rank == 1 and t < self.converge_at))
        return None, 0

    def begin(self, *a):
        self.log.append("begin")


def _dev_worker(rank, world, port, overflow_rank, q):
    from paper_2603_10726_b200.dist import run_protocol_device
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = FakeDevShard(world, rank, overflow=(rank == overflow_rank))

        def exchange_dev(sync):
            sh.log.append("x!" if sync else "x")
            if not sync:
                return 0
            v = torch.tensor([sh.changed], dtype=torch.int64)     # the mailbox flags' max
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            return int(v.item())

        def allreduce_max(xs):
            v = torch.tensor([max(xs)], dtype=torch.int64)
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            return int(v.item())

        try:
            res, t = run_protocol_device(sh, (), exchange_dev, allreduce_max)
            q.put((rank, "ok", t, sh.log))
        except SolidError as e:
            q.put((rank, "err", e.status, sh.log))
    finally:
        dist.destroy_process_group()


def _spawn_dev(overflow_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dev_worker, args=(r, 2, port, overflow_rank, q))
             for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def test_device_counts_protocol_world2_gloo():
    """run_protocol_device: REG and PULL exchanges asynchronous, one synchronised INT exchange
    per round carrying the changed flag, same stop round as the host-counts protocol."""
    for rank, status, t, log in _spawn_dev(overflow_rank=-1):
        assert status == "ok" and t == 3
        assert log == ["begin", "x", "ingest0", "x", "round1", "x!", "ingest1", "x", "round2",
                       "x!", "ingest2", "x", "round3", "x!", "ingest3", "commit1"]


def test_device_counts_overflow_rolls_back_everywhere():
    for rank, status, code, log in _spawn_dev(overflow_rank=0):
        assert status == "err" and code == SOLID_ERR_CAPACITY
        assert log[-2:] == ["commit1", "commit2"]
