"""Seeded synthetic request streams shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no hashing, no cache rules): it only emits token
ids, request boundaries, user ids and enforce bits.  See ``workloads.gen``.
"""
from .gen import (Stream, c1_tiny, c2_shared_prompt, c3_multiturn, c4_attackers, random_small,
                  concat_streams, VOCAB)
from .ttft import TtftStream, query_cuts, ttft_stream

__all__ = ["Stream", "c1_tiny", "c2_shared_prompt", "c3_multiturn", "c4_attackers",
           "random_small", "concat_streams", "VOCAB", "TtftStream", "ttft_stream", "query_cuts"]
