"""ctypes wrapper around oracle/solid_oracle.cpp (TEST INFRASTRUCTURE ONLY; see solid_oracle.cpp).

The oracle processes requests strictly one at a time; this wrapper only marshals
numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "solid_oracle.cpp")
LIB_PATH = os.path.join(HERE, "liboracle.so")

POLICY_APC, POLICY_USER_ISOLATION, POLICY_SOLIDARITY = 0, 1, 2

RESULT_DTYPE = np.dtype([("n_blocks", "<u4"), ("shared_hits", "<u4"), ("reused", "<u4"),
                         ("divert_at", "<i4"), ("flag_depth", "<u4"), ("bits", "<u4")])
ENTRY_DTYPE = np.dtype([("key", "<u8"), ("owner", "<u4"), ("sharer", "<u4")])
ENTRY_EX_DTYPE = np.dtype([("key", "<u8"), ("owner", "<u4"), ("sharer", "<u4"),
                           ("last_used", "<u8")])


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with g++ (plain -O2; the oracle is never tuned)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC):
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-o", tmp, SRC])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(LIB_PATH)
        vp, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32
        lib.oracle_create.restype = vp
        lib.oracle_create.argtypes = [u32, u64, ctypes.c_int]
        lib.oracle_destroy.argtypes = [vp]
        lib.oracle_size.restype = u64
        lib.oracle_size.argtypes = [vp]
        lib.oracle_params.argtypes = [vp, ctypes.POINTER(u64), ctypes.POINTER(u64)]
        lib.oracle_sigma.restype = u64
        lib.oracle_sigma.argtypes = [vp, u32]
        lib.oracle_splitmix64.restype = u64
        lib.oracle_splitmix64.argtypes = [u64]
        lib.oracle_fmix64.restype = u64
        lib.oracle_fmix64.argtypes = [u64]
        lib.oracle_chain.argtypes = [vp, vp, u32, u32, i32, vp, vp]
        lib.oracle_process.restype = ctypes.c_int
        lib.oracle_process.argtypes = [vp, u64, vp, vp, vp, vp, vp]
        lib.oracle_dump.restype = u64
        lib.oracle_dump.argtypes = [vp, vp, u64]
        lib.oracle_copy_table.argtypes = [vp, vp]
        lib.oracle_reserve.argtypes = [vp, u64]
        lib.oracle_set_capacity.restype = ctypes.c_int
        lib.oracle_set_capacity.argtypes = [vp, u64]
        lib.oracle_evictions.restype = u64
        lib.oracle_evictions.argtypes = [vp]
        lib.oracle_next_seq.restype = u64
        lib.oracle_next_seq.argtypes = [vp]
        lib.oracle_set_components.restype = ctypes.c_int
        lib.oracle_set_components.argtypes = [vp, ctypes.c_int]
        lib.oracle_params2.argtypes = [vp, ctypes.POINTER(u64), ctypes.POINTER(u64)]
        lib.oracle_chain2.argtypes = [vp, vp, u32, u32, i32, vp, vp, vp]
        lib.oracle_dump_ex.restype = u64
        lib.oracle_dump_ex.argtypes = [vp, vp, u64]
        lib.oracle_set_pool.restype = ctypes.c_int
        lib.oracle_set_pool.argtypes = [vp, u64]
        lib.oracle_block_table.restype = u64
        lib.oracle_block_table.argtypes = [vp, vp, u64]
        lib.oracle_dump_phys.restype = u64
        lib.oracle_dump_phys.argtypes = [vp, vp, vp, u64]
        lib.oracle_set_pin.restype = ctypes.c_int
        lib.oracle_set_pin.argtypes = [vp, ctypes.c_int]
        lib.oracle_release.restype = ctypes.c_int
        lib.oracle_release.argtypes = [vp, vp, u64]
        lib.oracle_admitted.restype = u64
        lib.oracle_admitted.argtypes = [vp]
        lib.oracle_dump_pins.restype = u64
        lib.oracle_dump_pins.argtypes = [vp, vp, vp, u64]
        _lib = lib
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class PinRefused(ValueError):
    """A request's eviction step would need a pinned entry (R38): it was refused, nothing of it
    applied; `admitted` requests of the call before it were admitted."""

    def __init__(self, admitted: int):
        super().__init__(f"request {admitted} of the call refused: too few unpinned entries")
        self.admitted = admitted


class Oracle:
    """Sequential reference: Oracle(block_size, seed, policy).process(stream) -> results."""

    def __init__(self, block_size: int = 16, seed: int = 0, policy: int = POLICY_SOLIDARITY,
                 capacity: int = 0, components: int = 1, pool: int = 0, pin: bool = False):
        self.lib = _load()
        self.block_size, self.seed, self.policy = block_size, seed, policy
        self.h = self.lib.oracle_create(block_size, seed & 0xFFFFFFFFFFFFFFFF, policy)
        if not self.h:
            raise ValueError("oracle_create: bad arguments")
        self.capacity = capacity
        self.components = components
        if components != 1 and self.lib.oracle_set_components(self.h, components):
            raise ValueError("components must be 1 or 2")
        if capacity:
            self.lib.oracle_set_capacity(self.h, capacity)   # LRU eviction (R22-R25)
        self.pool = pool
        if pool and self.lib.oracle_set_pool(self.h, pool):  # physical blocks (R26-R28)
            raise ValueError("bad pool size")
        if pin and self.lib.oracle_set_pin(self.h, 1):        # in-flight pinning (R38)
            raise ValueError("pin needs a pool")

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.oracle_destroy(h)
            self.h = None

    # -- admission -------------------------------------------------------------------------
    def process_arrays(self, tokens, offsets, users, enforce=None) -> np.ndarray:
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        users = np.ascontiguousarray(users, dtype=np.uint32)
        en = None if enforce is None else np.ascontiguousarray(enforce, dtype=np.uint8)
        n = users.shape[0]
        out = np.zeros(n, dtype=RESULT_DTYPE)
        if tokens.size == 0:
            tokens = np.zeros(1, dtype=np.uint32)
        err = self.lib.oracle_process(self.h, n, _ptr(tokens), _ptr(offsets), _ptr(users),
                                      _ptr(en), _ptr(out))
        if err == 4:
            raise ValueError("oracle_process: physical block pool exhausted")
        if err == 5:
            raise PinRefused(int(self.lib.oracle_admitted(self.h)))
        if err:
            raise ValueError(f"oracle_process: invalid batch (code {err})")
        return out

    def process(self, stream) -> np.ndarray:
        return self.process_arrays(stream.tokens, stream.offsets, stream.users, stream.enforce)

    def process_prompts(self, prompts, users, enforce=None) -> np.ndarray:
        lens = np.array([len(p) for p in prompts], dtype=np.uint64)
        offs = np.zeros(len(prompts) + 1, dtype=np.uint64)
        np.cumsum(lens, out=offs[1:])
        toks = (np.concatenate([np.asarray(p, dtype=np.uint32) for p in prompts])
                if int(offs[-1]) else np.zeros(0, np.uint32))
        return self.process_arrays(toks, offs, users, enforce)

    # -- inspection ------------------------------------------------------------------------
    def size(self) -> int:
        return int(self.lib.oracle_size(self.h))

    def dump(self) -> np.ndarray:
        n = self.size()
        out = np.zeros(max(n, 1), dtype=ENTRY_DTYPE)
        self.lib.oracle_dump(self.h, _ptr(out), n)
        return out[:n]

    def dump_ex(self) -> np.ndarray:
        """Live entries with their LRU clock (last_used), sorted by key."""
        n = self.size()
        out = np.zeros(max(n, 1), dtype=ENTRY_EX_DTYPE)
        self.lib.oracle_dump_ex(self.h, _ptr(out), n)
        return out[:n]

    def block_table(self) -> np.ndarray:
        """Block table of the last process call (R27): index offsets[j] // 16 + b."""
        n = int(self.lib.oracle_block_table(self.h, None, 0))
        out = np.zeros(max(n, 1), dtype=np.uint32)
        self.lib.oracle_block_table(self.h, _ptr(out), n)
        return out[:n]

    def dump_phys(self):
        """(keys, physical blocks) of the live entries, sorted by key."""
        n = self.size()
        k = np.zeros(max(n, 1), dtype=np.uint64)
        p = np.zeros(max(n, 1), dtype=np.uint32)
        self.lib.oracle_dump_phys(self.h, _ptr(k), _ptr(p), n)
        return k[:n], p[:n]

    def release(self, phys) -> None:
        """Drop one pin on the entry holding each physical block (NONE entries skipped)."""
        phys = np.ascontiguousarray(phys, dtype=np.uint32)
        if self.lib.oracle_release(self.h, _ptr(phys if phys.size else np.zeros(1, np.uint32)),
                                   phys.size):
            raise ValueError("oracle_release: a block holds no pinned live entry")

    def dump_pins(self):
        """(keys, pin counts) of the live entries, sorted by key."""
        n = self.size()
        k = np.zeros(max(n, 1), dtype=np.uint64)
        p = np.zeros(max(n, 1), dtype=np.uint32)
        self.lib.oracle_dump_pins(self.h, _ptr(k), _ptr(p), n)
        return k[:n], p[:n]

    def evictions(self) -> int:
        return int(self.lib.oracle_evictions(self.h))

    def next_seq(self) -> int:
        return int(self.lib.oracle_next_seq(self.h))

    def params(self):
        B, M = ctypes.c_uint64(), ctypes.c_uint64()
        self.lib.oracle_params(self.h, ctypes.byref(B), ctypes.byref(M))
        return int(B.value), int(M.value)

    def sigma(self, user: int) -> int:
        return int(self.lib.oracle_sigma(self.h, user))

    def params2(self):
        B2, M2 = ctypes.c_uint64(), ctypes.c_uint64()
        self.lib.oracle_params2(self.h, ctypes.byref(B2), ctypes.byref(M2))
        return int(B2.value), int(M2.value)

    def chain2(self, tokens, user: int = 0, divert_at: int = -1):
        """(S, S2, keys) of both H-def components (keys per the context's component count)."""
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        n = tokens.size // self.block_size
        S = np.zeros(max(n, 1), dtype=np.uint64)
        S2 = np.zeros(max(n, 1), dtype=np.uint64)
        K = np.zeros(max(n, 1), dtype=np.uint64)
        self.lib.oracle_chain2(self.h, _ptr(tokens if tokens.size else np.zeros(1, np.uint32)),
                               n, user, divert_at, _ptr(S), _ptr(S2), _ptr(K))
        return S[:n], S2[:n], K[:n]

    def chain(self, tokens, user: int = 0, divert_at: int = -1):
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        n = tokens.size // self.block_size
        S = np.zeros(max(n, 1), dtype=np.uint64)
        K = np.zeros(max(n, 1), dtype=np.uint64)
        self.lib.oracle_chain(self.h, _ptr(tokens if tokens.size else np.zeros(1, np.uint32)),
                              n, user, divert_at, _ptr(S), _ptr(K))
        return S[:n], K[:n]

    def copy_table_from(self, other: "Oracle"):
        self.lib.oracle_copy_table(self.h, other.h)

    def reserve(self, n: int):
        self.lib.oracle_reserve(self.h, n)

    @staticmethod
    def splitmix64(x: int) -> int:
        return int(_load().oracle_splitmix64(x & 0xFFFFFFFFFFFFFFFF))

    @staticmethod
    def fmix64(x: int) -> int:
        return int(_load().oracle_fmix64(x & 0xFFFFFFFFFFFFFFFF))
