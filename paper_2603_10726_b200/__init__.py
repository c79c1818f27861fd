"""Python binding of the B200-native CacheSolidarity hot path (include/solid.h).

Argument marshalling only: every step of the path runs in the CUDA kernels of lib/libsolid.so.
PyTorch provides device memory and streams.  There is NO CPU fallback — importing this package
on a machine without the built library raises, and Index() needs a CUDA device.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SOLID_LIB") or os.path.join(_PKG, "lib", "libsolid.so")

SOLID_OK, SOLID_ERR_INVALID, SOLID_ERR_CAPACITY, SOLID_ERR_STATE, SOLID_ERR_CUDA, \
    SOLID_ERR_NCCL, SOLID_ERR_OOM = range(7)
POLICY = {"apc": 0, "user_isolation": 1, "solidarity": 2}
HIT, FULL, DIVERTED, TRUNCATED, FLAGGED = 1, 2, 4, 8, 16
USER_NONE = 0xFFFFFFFF

RESULT_DTYPE = np.dtype([("n_blocks", "<u4"), ("shared_hits", "<u4"), ("reused", "<u4"),
                         ("divert_at", "<i4"), ("flag_depth", "<u4"), ("bits", "<u4")])
ENTRY_DTYPE = np.dtype([("key", "<u8"), ("owner", "<u4"), ("sharer", "<u4")])
ENTRY_EX_DTYPE = np.dtype([("key", "<u8"), ("owner", "<u4"), ("sharer", "<u4"),
                           ("last_used", "<u8")])

# C ABI entry points declared in include/solid.h (checked by tests/test_abi.py)
ABI_SYMBOLS = ["solid_abi_version", "solid_init", "solid_destroy", "solid_lookup_batch",
               "solid_insert_batch", "solid_admit_host", "solid_admit_host_u16", "solid_stats", "solid_dump", "solid_dump_ex",
               "solid_admit_batch", "solid_batch_status", "solid_block_keys", "solid_debug_set_epoch", "solid_debug_set_max_rounds",
               "solid_block_table", "solid_dump_phys", "solid_release", "solid_pins",
               "solid_reset", "solid_checkpoint", "solid_restore", "solid_last_error",
               "solid_dist_buffers", "solid_dist_counts", "solid_dist_begin",
               "solid_dist_owner_ingest", "solid_dist_round", "solid_dist_commit",
               "solid_dist_p2p_export", "solid_dist_p2p_connect", "solid_dist_p2p_exchange",
               "solid_dist_p2p_device_counts", "solid_dist_p2p_exchange_dev", "solid_dist_admit",
               "solid_activator_init", "solid_activator_destroy", "solid_activator_run",
               "solid_activator_last_error"]
RECORD_BYTES = 24   # sharded-mode exchange record
MAX_INFLIGHT = 4    # SOLID_MAX_INFLIGHT


class SolidError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"solid status {status}: {msg}")
        self.status = status


class _Config(ctypes.Structure):
    _fields_ = [("block_size", ctypes.c_uint32), ("max_blocks", ctypes.c_uint32),
                ("capacity_blocks", ctypes.c_uint64), ("max_batch_tokens", ctypes.c_uint64),
                ("max_batch_requests", ctypes.c_uint64), ("hash_seed", ctypes.c_uint64),
                ("policy", ctypes.c_int32), ("device", ctypes.c_int32),
                ("world", ctypes.c_uint32), ("rank", ctypes.c_uint32),
                ("evict", ctypes.c_uint32), ("hash_components", ctypes.c_uint32),
                ("block_table", ctypes.c_uint32), ("pin", ctypes.c_uint32)]


class _Batch(ctypes.Structure):
    _fields_ = [("n_requests", ctypes.c_uint64), ("tokens", ctypes.c_void_p),
                ("offsets", ctypes.c_void_p), ("users", ctypes.c_void_p),
                ("enforce", ctypes.c_void_p)]


class _Stats(ctypes.Structure):
    _fields_ = [("batches", ctypes.c_uint64), ("requests", ctypes.c_uint64),
                ("blocks", ctypes.c_uint64), ("reused_blocks", ctypes.c_uint64),
                ("inserted", ctypes.c_uint64), ("flagged", ctypes.c_uint64),
                ("diverted", ctypes.c_uint64), ("truncated", ctypes.c_uint64),
                ("live_entries", ctypes.c_uint64), ("last_rounds", ctypes.c_uint32),
                ("last_distinct_keys", ctypes.c_uint32), ("last_requests", ctypes.c_uint64),
                ("last_blocks", ctypes.c_uint64), ("last_inserted", ctypes.c_uint64),
                ("last_flagged", ctypes.c_uint64), ("ms_hash", ctypes.c_float),
                ("ms_resolve", ctypes.c_float), ("ms_commit", ctypes.c_float),
                ("algorithmic_bytes", ctypes.c_uint64),
                ("last_kernel_launches", ctypes.c_uint64), ("ms_hash_kernel", ctypes.c_float),
                ("ms_round_first", ctypes.c_float), ("round_us", ctypes.c_float * 8),
                ("evicted", ctypes.c_uint64), ("last_evicted", ctypes.c_uint64),
                ("last_evict_iters", ctypes.c_uint32), ("last_window_keys", ctypes.c_uint32),
                ("window_evicted", ctypes.c_uint64), ("max_evict_iters", ctypes.c_uint32),
                ("rebuilds", ctypes.c_uint32), ("compactions", ctypes.c_uint32),
                ("last_shared_keys", ctypes.c_uint32)]


class _ActConfig(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_double), ("hit_hi", ctypes.c_double),
                ("hit_lo", ctypes.c_double), ("window_len", ctypes.c_uint32),
                ("min_samples", ctypes.c_uint32), ("grid", ctypes.c_uint32),
                ("device", ctypes.c_int32), ("max_samples", ctypes.c_uint64),
                ("max_queries", ctypes.c_uint64)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libsolid.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -m paper_2603_10726_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, st = ctypes.c_void_p, ctypes.c_int
    lib.solid_abi_version.restype = ctypes.c_uint32
    lib.solid_init.restype = st
    lib.solid_init.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(vp)]
    lib.solid_destroy.restype = st
    lib.solid_destroy.argtypes = [vp]
    lib.solid_lookup_batch.restype = st
    lib.solid_lookup_batch.argtypes = [vp, ctypes.POINTER(_Batch), vp, vp]
    lib.solid_insert_batch.restype = st
    lib.solid_insert_batch.argtypes = [vp, vp]
    lib.solid_admit_batch.restype = st
    lib.solid_admit_batch.argtypes = [vp, ctypes.POINTER(_Batch), vp, vp]
    lib.solid_batch_status.restype = st
    lib.solid_batch_status.argtypes = [vp]
    lib.solid_admit_host.restype = st
    lib.solid_admit_host.argtypes = [vp, ctypes.POINTER(_Batch), vp, vp]
    lib.solid_admit_host_u16.restype = st
    lib.solid_admit_host_u16.argtypes = [vp, ctypes.POINTER(_Batch), vp, vp]   # same layout
    lib.solid_stats.restype = st
    lib.solid_stats.argtypes = [vp, ctypes.POINTER(_Stats)]
    lib.solid_dump.restype = st
    lib.solid_dump.argtypes = [vp, vp, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
    lib.solid_debug_set_epoch.restype = st
    lib.solid_debug_set_epoch.argtypes = [vp, ctypes.c_uint32]
    lib.solid_debug_set_max_rounds.restype = st
    lib.solid_debug_set_max_rounds.argtypes = [vp, ctypes.c_uint32]
    lib.solid_block_keys.restype = st
    lib.solid_block_keys.argtypes = [vp, vp, vp]
    lib.solid_dump_ex.restype = st
    lib.solid_block_table.restype = st
    lib.solid_block_table.argtypes = [vp, vp, vp]
    lib.solid_dump_phys.restype = st
    lib.solid_dump_phys.argtypes = [vp, vp, vp, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
    lib.solid_dump_ex.argtypes = [vp, vp, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
    lib.solid_release.restype = st
    lib.solid_release.argtypes = [vp, vp, ctypes.c_uint64, vp]
    lib.solid_pins.restype = st
    lib.solid_pins.argtypes = [vp, vp]
    for name in ["solid_reset", "solid_checkpoint", "solid_restore"]:
        getattr(lib, name).restype = st
        getattr(lib, name).argtypes = [vp]
    lib.solid_last_error.restype = ctypes.c_char_p
    lib.solid_last_error.argtypes = [vp]
    u64p = ctypes.POINTER(ctypes.c_uint64)
    lib.solid_dist_buffers.restype = st
    lib.solid_dist_buffers.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), u64p]
    lib.solid_dist_counts.restype = st
    lib.solid_dist_counts.argtypes = [vp, u64p]
    lib.solid_dist_begin.restype = st
    lib.solid_dist_begin.argtypes = [vp, ctypes.POINTER(_Batch), vp, ctypes.c_uint64, vp]
    lib.solid_dist_owner_ingest.restype = st
    lib.solid_dist_owner_ingest.argtypes = [vp, ctypes.c_uint32, u64p, vp]
    lib.solid_dist_round.restype = st
    lib.solid_dist_round.argtypes = [vp, ctypes.c_uint32, u64p, ctypes.POINTER(ctypes.c_uint32), vp]
    lib.solid_dist_commit.restype = st
    lib.solid_dist_commit.argtypes = [vp, ctypes.c_int, u64p, vp]
    lib.solid_activator_init.restype = st
    lib.solid_activator_init.argtypes = [ctypes.POINTER(_ActConfig), ctypes.POINTER(vp)]
    lib.solid_activator_destroy.restype = st
    lib.solid_activator_destroy.argtypes = [vp]
    lib.solid_activator_run.restype = st
    lib.solid_activator_run.argtypes = [vp, vp, vp, vp, ctypes.c_uint64, vp, ctypes.c_uint64, vp,
                                        vp, vp]
    lib.solid_activator_last_error.restype = ctypes.c_char_p
    lib.solid_activator_last_error.argtypes = [vp]
    _lib = lib
    return lib


def _np_ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


class Index:
    """One GPU-resident prefix index (C ABI context).

    lookup(...) + insert() admit one batch; results are a torch int32 tensor [N, 6] on the device
    (fields of RESULT_DTYPE).  `as_numpy(results)` converts a host copy to the structured dtype.
    """

    def __init__(self, policy: str = "solidarity", capacity_blocks: int = 1 << 20,
                 max_batch_tokens: int = 1 << 24, max_batch_requests: int = 1 << 16,
                 max_blocks: int = 8192, seed: int = 0x5011D000, device: int = 0,
                 world: int = 1, rank: int = 0, evict: bool = False, hash_components: int = 1,
                 block_table: bool = False, pin: bool = False):
        """evict=True: LRU eviction at capacity_blocks instead of
        SOLID_ERR_CAPACITY; lookup() then synchronises its stream.  hash_components=2: H-def v3
        two-component keys.  block_table=True: physical KV block ids and
        per-request block tables (admission synchronous).  pin=True (with
        block_table): in-flight pinning — each admitted request pins its row's entries until
        release() (R38)."""
        self.lib = load_library()
        cfg = _Config(16, max_blocks, capacity_blocks, max_batch_tokens, max_batch_requests,
                      seed & 0xFFFFFFFFFFFFFFFF, POLICY[policy], device, world, rank,
                      1 if evict else 0, hash_components, 1 if block_table else 0,
                      1 if pin else 0)
        self.world, self.rank = world, rank
        h = ctypes.c_void_p()
        rc = self.lib.solid_init(ctypes.byref(cfg), ctypes.byref(h))
        if rc != SOLID_OK:
            raise SolidError(rc, "solid_init failed (needs a CUDA device and valid sizes)")
        self.h = h
        self.device = device
        self.policy = policy
        self.seed = seed
        self.evict = evict

    def close(self):
        if getattr(self, "h", None):
            self.lib.solid_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != SOLID_OK:
            raise SolidError(rc, self.last_error())

    def last_error(self) -> str:
        msg = self.lib.solid_last_error(self.h)
        return msg.decode() if msg else ""

    @staticmethod
    def _stream(stream):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream()
        return ctypes.c_void_p(stream.cuda_stream)

    # ---- device-buffer admission ---------------------------------------------------------
    def lookup(self, tokens, offsets, users, enforce=None, out=None, stream=None):
        """tokens int32/uint32 [T], offsets int64 [N+1], users int32/uint32 [N], enforce uint8
        [N] or None — all CUDA tensors.  Returns the result tensor (int32 [N, 6])."""
        import torch
        n = int(users.numel())
        if out is None:
            out = torch.empty((max(n, 1), 6), dtype=torch.int32, device=offsets.device)
        for t in (tokens, offsets, users, out) + ((enforce,) if enforce is not None else ()):
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError("batch tensors must be contiguous CUDA tensors")
        b = _Batch(n, tokens.data_ptr(), offsets.data_ptr(), users.data_ptr(),
                   enforce.data_ptr() if enforce is not None else None)
        self._check(self.lib.solid_lookup_batch(self.h, ctypes.byref(b),
                                                ctypes.c_void_p(out.data_ptr()),
                                                self._stream(stream)))
        return out[:n]

    def insert(self, stream=None):
        self._check(self.lib.solid_insert_batch(self.h, self._stream(stream)))

    def admit(self, tokens, offsets, users, enforce=None, out=None, stream=None):
        out = self.lookup(tokens, offsets, users, enforce, out, stream)
        self.insert(stream)
        return out

    def admit_split(self, tokens, offsets, users, enforce=None, stream=None):
        """Evict mode: admit, and if the batch would have to evict entries it touched itself
        (SOLID_ERR_CAPACITY, nothing mutated) admit its two halves in order instead — the same
        results as one request at a time (reading R1).  Returns the result tensor [N, 6]."""
        import torch
        try:
            return self.admit(tokens, offsets, users, enforce, None, stream)
        except SolidError as e:
            n = int(users.numel())
            if not self.evict or e.status != SOLID_ERR_CAPACITY or n < 2:
                raise
        h = n // 2
        off = offsets.to(torch.int64)
        parts = []
        for lo, hi in ((0, h), (h, n)):
            t0, t1 = int(off[lo]), int(off[hi])
            parts.append(self.admit_split(tokens[t0:t1] if t1 > t0 else tokens[:4],
                                          (off[lo:hi + 1] - t0).contiguous(),
                                          users[lo:hi].contiguous(),
                                          None if enforce is None else enforce[lo:hi].contiguous(),
                                          stream).clone())
        return torch.cat(parts)

    def admit_async(self, tokens, offsets, users, enforce=None, out=None, stream=None):
        """Lookup + insert without a host synchronisation (solid_admit_batch): the capacity
        check and exact rollback run on the device.  Up to MAX_INFLIGHT batches may be
        outstanding; `status()` collects the oldest (and raises its error, if any)."""
        import torch
        n = int(users.numel())
        if out is None:
            out = torch.empty((max(n, 1), 6), dtype=torch.int32, device=offsets.device)
        for t in (tokens, offsets, users, out) + ((enforce,) if enforce is not None else ()):
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError("batch tensors must be contiguous CUDA tensors")
        b = _Batch(n, tokens.data_ptr(), offsets.data_ptr(), users.data_ptr(),
                   enforce.data_ptr() if enforce is not None else None)
        self._check(self.lib.solid_admit_batch(self.h, ctypes.byref(b),
                                               ctypes.c_void_p(out.data_ptr()),
                                               self._stream(stream)))
        return out[:n]

    def status(self):
        """Wait for the oldest outstanding asynchronous batch and raise its error, if any."""
        self._check(self.lib.solid_batch_status(self.h))

    # ---- host-buffer admission (copies inside the C ABI call) -----------------------------
    def admit_host(self, tokens: np.ndarray, offsets: np.ndarray, users: np.ndarray,
                   enforce: Optional[np.ndarray] = None, out: Optional[np.ndarray] = None,
                   stream=None) -> np.ndarray:
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        users = np.ascontiguousarray(users, dtype=np.uint32)
        en = None if enforce is None else np.ascontiguousarray(enforce, dtype=np.uint8)
        n = users.shape[0]
        if out is None:
            out = np.zeros(max(n, 1), dtype=RESULT_DTYPE)
        if tokens.size == 0:
            tokens = np.zeros(4, np.uint32)
        b = _Batch(n, _np_ptr(tokens), _np_ptr(offsets), _np_ptr(users), _np_ptr(en))
        self._check(self.lib.solid_admit_host(self.h, ctypes.byref(b),
                                              ctypes.c_void_p(out.ctypes.data),
                                              self._stream(stream)))
        return out[:n]

    def admit_host_u16(self, tokens: np.ndarray, offsets: np.ndarray, users: np.ndarray,
                       enforce: Optional[np.ndarray] = None, out: Optional[np.ndarray] = None,
                       stream=None) -> np.ndarray:
        """admit_host with 16-bit token ids (solid_admit_host_u16): tokens must be uint16."""
        if tokens.dtype != np.uint16 or not tokens.flags.c_contiguous:
            raise ValueError("tokens must be a contiguous uint16 array")
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        users = np.ascontiguousarray(users, dtype=np.uint32)
        en = None if enforce is None else np.ascontiguousarray(enforce, dtype=np.uint8)
        n = users.shape[0]
        if out is None:
            out = np.zeros(max(n, 1), dtype=RESULT_DTYPE)
        if tokens.size == 0:
            tokens = np.zeros(8, np.uint16)
        b = _Batch(n, _np_ptr(tokens), _np_ptr(offsets), _np_ptr(users), _np_ptr(en))
        self._check(self.lib.solid_admit_host_u16(self.h, ctypes.byref(b),
                                                  ctypes.c_void_p(out.ctypes.data),
                                                  self._stream(stream)))
        return out[:n]

    # ---- inspection / state --------------------------------------------------------------
    def stats(self) -> dict:
        s = _Stats()
        self._check(self.lib.solid_stats(self.h, ctypes.byref(s)))
        d = {name: getattr(s, name) for name, _ in _Stats._fields_}
        d["round_us"] = list(d["round_us"])
        return d

    def dump(self) -> np.ndarray:
        n = ctypes.c_uint64()
        self._check(self.lib.solid_dump(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros(max(int(n.value), 1), dtype=ENTRY_DTYPE)
        self._check(self.lib.solid_dump(self.h, ctypes.c_void_p(out.ctypes.data), n.value,
                                        ctypes.byref(n)))
        return out[:int(n.value)]

    def block_keys(self, n_tokens: int, stream=None):
        """Block table of the last batch (solid_block_keys): uint64 tensor [ceil(T/16)], the key
        of the entry holding each block's KV (index offsets[j] // 16 + b)."""
        import torch
        out = torch.zeros(max((n_tokens + 15) // 16, 1), dtype=torch.int64,
                          device=torch.device("cuda", self.device))
        self._check(self.lib.solid_block_keys(self.h, ctypes.c_void_p(out.data_ptr()),
                                              self._stream(stream)))
        return out

    def dump_ex(self) -> np.ndarray:
        """Evict mode: live entries with their LRU clock (ENTRY_EX_DTYPE), sorted by key."""
        n = ctypes.c_uint64()
        self._check(self.lib.solid_dump_ex(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros(max(int(n.value), 1), dtype=ENTRY_EX_DTYPE)
        self._check(self.lib.solid_dump_ex(self.h, ctypes.c_void_p(out.ctypes.data), n.value,
                                           ctypes.byref(n)))
        return out[:int(n.value)]

    def block_table(self, n_tokens: int, stream=None):
        """Block table of the last committed batch (solid_block_table, R27): int32 tensor
        [ceil(T/16)] (uint32 values; -1 = NONE), the physical block of request j's block b at
        index offsets[j] // 16 + b.  Positions no full block covers keep -2."""
        import torch
        out = torch.full((max((n_tokens + 15) // 16, 1),), -2, dtype=torch.int32,
                         device=torch.device("cuda", self.device))
        self._check(self.lib.solid_block_table(self.h, ctypes.c_void_p(out.data_ptr()),
                                               self._stream(stream)))
        return out

    def dump_phys(self):
        """(keys uint64, physical blocks uint32) of the live entries, sorted by key."""
        n = ctypes.c_uint64()
        self._check(self.lib.solid_dump_phys(self.h, None, None, 0, ctypes.byref(n)))
        m = int(n.value)
        k = np.zeros(max(m, 1), dtype=np.uint64)
        p = np.zeros(max(m, 1), dtype=np.uint32)
        self._check(self.lib.solid_dump_phys(self.h, ctypes.c_void_p(k.ctypes.data),
                                             ctypes.c_void_p(p.ctypes.data), m, ctypes.byref(n)))
        return k[:m], p[:m]

    def release(self, phys, stream=None):
        """solid_release: one pin less on the entry holding each physical block of `phys` (a
        CUDA int32/uint32 tensor, e.g. a finished request's block-table row; -1 = NONE)."""
        self._check(self.lib.solid_release(self.h, ctypes.c_void_p(phys.data_ptr()),
                                           int(phys.numel()), self._stream(stream)))

    def pins(self, n_blocks: int) -> np.ndarray:
        """solid_pins: pin count per physical block (uint32 [capacity_blocks])."""
        out = np.zeros(max(n_blocks, 1), dtype=np.uint32)
        self._check(self.lib.solid_pins(self.h, ctypes.c_void_p(out.ctypes.data)))
        return out[:n_blocks]

    def reset(self):
        self._check(self.lib.solid_reset(self.h))

    def debug_set_epoch(self, epoch: int):
        """Test hook (solid_debug_set_epoch): jump the scratch epoch towards its restart."""
        self._check(self.lib.solid_debug_set_epoch(self.h, epoch))

    def debug_set_max_rounds(self, rounds: int):
        """Test hook (solid_debug_set_max_rounds): the resolver's round limit; a synchronous
        admission that does not converge within it is committed in parts."""
        self._check(self.lib.solid_debug_set_max_rounds(self.h, rounds))

    def checkpoint(self):
        self._check(self.lib.solid_checkpoint(self.h))

    def restore(self):
        self._check(self.lib.solid_restore(self.h))


def as_numpy(results) -> np.ndarray:
    """int32 [N, 6] result tensor/array -> structured RESULT_DTYPE array (host)."""
    if hasattr(results, "cpu"):
        results = results.cpu().numpy()
    return np.ascontiguousarray(results).view(RESULT_DTYPE).reshape(-1)


def to_device(stream_obj, device="cuda"):
    """workloads.Stream -> dict of CUDA tensors for Index.lookup (marshalling helper)."""
    import torch
    tok = torch.from_numpy(stream_obj.tokens.view(np.int32)).to(device)
    if tok.numel() == 0:
        tok = torch.zeros(4, dtype=torch.int32, device=device)
    d = dict(tokens=tok,
             offsets=torch.from_numpy(stream_obj.offsets.view(np.int64)).to(device),
             users=torch.from_numpy(stream_obj.users.view(np.int32)).to(device),
             enforce=None if stream_obj.enforce is None else
             torch.from_numpy(stream_obj.enforce).to(device))
    return d


class Activator:
    """The Activator (solid_activator_*): per-request enforce bits from the KDE overlap of the
    hit / miss per-token-TTFT windows (estimator SPEC S:245-268)."""

    def __init__(self, theta: float = 0.5, window_len: int = 256, min_samples: int = 16,
                 hit_hi: float = 0.8, hit_lo: float = 0.2, grid: int = 512,
                 max_samples: int = 1 << 20, max_queries: int = 1 << 20, device: int = 0):
        self.lib = load_library()
        cfg = _ActConfig(theta, hit_hi, hit_lo, window_len, min_samples, grid, device,
                         max_samples, max_queries)
        h = ctypes.c_void_p()
        rc = self.lib.solid_activator_init(ctypes.byref(cfg), ctypes.byref(h))
        if rc != SOLID_OK:
            raise SolidError(rc, "solid_activator_init failed (needs a CUDA device and valid sizes)")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.solid_activator_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, ttft_ms, prompt_tokens, reuse_fraction, cuts, overlap=None, enforce=None,
            stream=None):
        """CUDA tensors: ttft_ms float64 [M], prompt_tokens int32/uint32 [M], reuse_fraction
        float64 [M], cuts int64 [N] (non-decreasing, <= M).  Returns (overlap float64 [N],
        enforce uint8 [N]); enforce can be passed as a batch's `enforce`."""
        import torch
        n, m = int(cuts.numel()), int(ttft_ms.numel())
        dev = cuts.device
        if overlap is None:
            overlap = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        if enforce is None:
            enforce = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        for t in (ttft_ms, prompt_tokens, reuse_fraction, cuts, overlap, enforce):
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError("activator tensors must be contiguous CUDA tensors")
        st = Index._stream(stream)
        rc = self.lib.solid_activator_run(self.h, ttft_ms.data_ptr(), prompt_tokens.data_ptr(),
                                          reuse_fraction.data_ptr(), m, cuts.data_ptr(), n,
                                          overlap.data_ptr(), enforce.data_ptr(), st)
        if rc != SOLID_OK:
            msg = self.lib.solid_activator_last_error(self.h)
            raise SolidError(rc, msg.decode() if msg else "")
        return overlap[:n], enforce[:n]
