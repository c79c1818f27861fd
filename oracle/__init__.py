"""CacheSolidarity oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this package.  The product path (paper_2603_10726_b200) never imports it.
"""
from .oracle import Oracle, PinRefused, build_oracle, LIB_PATH, POLICY_APC, \
    POLICY_USER_ISOLATION, POLICY_SOLIDARITY, RESULT_DTYPE, ENTRY_DTYPE, ENTRY_EX_DTYPE

__all__ = ["Oracle", "PinRefused", "build_oracle", "LIB_PATH", "POLICY_APC", "POLICY_USER_ISOLATION",
           "POLICY_SOLIDARITY", "RESULT_DTYPE", "ENTRY_DTYPE", "ENTRY_EX_DTYPE"]
