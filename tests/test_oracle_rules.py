"""Pins for the oracle's detector / isolation rules against the paper.

golden/p1_example.json   worked example t1-t4 + owner extension
golden/p2_attack.json    attacker-perceived experiment
plus SPEC detector examples, the Q5/D2 counterexample to SPEC S:179's literal rule,
and owner immutability / flag monotonicity.
"""
import json
import os

import numpy as np
import pytest

from oracle import Oracle, POLICY_APC, POLICY_SOLIDARITY, POLICY_USER_ISOLATION
from oracle_helpers import Blocks, NONE, table_as_dict

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SEED = 0x5011D000


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_p1_worked_example():
    g = _load("p1_example.json")
    B = Blocks()
    users = g["users"]
    o = Oracle(16, SEED, POLICY_SOLIDARITY)
    for req in g["requests"]:
        u = users[req["user"]]
        res = o.process_prompts([B.prompt(req["blocks"])], [u])[0]
        assert int(res["shared_hits"]) == req["k"], req
        assert int(res["divert_at"]) == req["f"], req
        assert int(res["reused"]) == req["r"], req
        flag_depth = req["blocks"].index(req["flag"]) + 1 if req["flag"] else 0
        assert int(res["flag_depth"]) == flag_depth, req
        n = len(req["blocks"])
        bits = ((req["r"] > 0) | ((req["r"] == n) << 1) | ((req["f"] >= 0) << 2)
                | ((0 <= req["f"] < req["k"]) << 3) | ((flag_depth > 0) << 4))
        assert int(res["bits"]) == bits, req
    # final table: map each expected (namespace, path) to its key through the chain
    tab = table_as_dict(o)
    assert len(tab) == len(g["final_table"]) == 12
    for ent in g["final_table"]:
        toks = B.prompt(ent["path"])
        if ent["ns"] == "S":
            _, K = o.chain(toks)
        else:
            _, K = o.chain(toks, users[ent["user"]], ent["divert_at"])
        key = int(K[-1])
        owner = users[ent["owner"]]
        sharer = users[ent["sharer"]] if ent["sharer"] else NONE
        assert tab[key] == (owner, sharer), ent
    # baselines on the same stream
    for policy, field in [(POLICY_APC, "apc_r"), (POLICY_USER_ISOLATION, "user_isolation_r")]:
        ob = Oracle(16, SEED, policy)
        r = [int(ob.process_prompts([B.prompt(q["blocks"])], [users[q["user"]]])[0]["reused"])
             for q in g["requests"]]
        assert r == g[field], (field, r)


def _p2_stream(g, B):
    prompts = [B.prompt(g["victim_blocks"])]
    users = [g["victim_user"]]
    for i in range(1, g["n_probes"] + 1):
        cand = "S" if i == g["correct_probe"] else f"C{i}"
        prompts.append(B.prompt([cand if b == "C_i" else b for b in g["probe_blocks"]]))
        users.append(g["attacker_user"])
    return prompts, users


def test_p2_attacker_experiment():
    g = _load("p2_attack.json")
    B = Blocks(seed=4242)
    prompts, users = _p2_stream(g, B)
    apc = Oracle(16, SEED, POLICY_APC).process_prompts(prompts, users)
    assert apc["reused"][1:].tolist() == g["apc_probe_r"]
    # the spike: the correct probe is a full hit (P:816 'hit rate reaches 100%')
    c = g["correct_probe"]
    assert apc["reused"][c] == apc["n_blocks"][c]
    cs = Oracle(16, SEED, POLICY_SOLIDARITY).process_prompts(prompts, users)
    assert cs["reused"][1:].tolist() == g["solidarity_probe_r"]
    p1 = cs[1]
    assert (int(p1["shared_hits"]), int(p1["divert_at"]), int(p1["flag_depth"])) == (4, -1, 4)
    for i in range(2, g["n_probes"] + 1):
        assert int(cs[i]["divert_at"]) == 4
        if i != c:
            assert int(cs[i]["shared_hits"]) == 4
    cp = cs[c]
    assert (int(cp["shared_hits"]), int(cp["divert_at"]), int(cp["reused"])) == (7, 4, 4)
    assert int(cp["bits"]) & 8  # TRUNCATED
    # uniformity: no probe's reuse exceeds another's
    assert len(set(cs["reused"][1:].tolist())) == 1


def test_q5_flag_rule_counterexample():
    """D2 vs SPEC S:179 literal.  u1 [T1 T2 X3]; u2 [T1 T2 Y3] (flags T2); u2 [T1 T2 Y3 Y4];
    u2 [T1 T2 Y3 Y4 Y5] must reuse 4 blocks (P:513-514 'User 2 would be allowed to further
    extend their own path'); S:179's literal rule would flag T1 at request 3 and give r = 1."""
    B = Blocks(seed=5)
    o = Oracle(16, SEED, POLICY_SOLIDARITY)
    res = o.process_prompts([B.prompt(["T1", "T2", "X3"]), B.prompt(["T1", "T2", "Y3"]),
                             B.prompt(["T1", "T2", "Y3", "Y4"]),
                             B.prompt(["T1", "T2", "Y3", "Y4", "Y5"])], [1, 2, 2, 2])
    assert res["reused"].tolist() == [0, 2, 3, 4]
    assert res["flag_depth"].tolist() == [0, 2, 0, 0]
    _, K = o.chain(B.prompt(["T1", "T2"]))
    tab = table_as_dict(o)
    assert tab[int(K[0])] == (1, NONE) and tab[int(K[1])] == (1, 2)


def test_spec_detector_examples():
    """S:182-185 (with R7 for the flagged-last-hit case)."""
    B = Blocks(seed=6)
    o = Oracle(16, SEED, POLICY_SOLIDARITY)
    # t2: chain [e1(u1), e2(u1)], requester u2 -> reused 2, flags e2, Shared
    r = o.process_prompts([B.prompt(["E1", "E2", "E3"]), B.prompt(["E1", "E2", "N1"])], [1, 2])
    assert (int(r[1]["reused"]), int(r[1]["flag_depth"]), int(r[1]["divert_at"])) == (2, 2, -1)
    # t3: chain [e1(u1), e2(u1, flagged), e3(u1)], requester u1 -> reused 3, no flags
    r = o.process_prompts([B.prompt(["E1", "E2", "E3", "N2"])], [1])
    assert (int(r[0]["reused"]), int(r[0]["flag_depth"]), int(r[0]["divert_at"])) == (3, 0, -1)
    # chain [e1, e2(flagged), e3(u1)], requester u3 -> f=2, reused 2, truncated
    r = o.process_prompts([B.prompt(["E1", "E2", "E3", "N3"])], [3])
    assert (int(r[0]["reused"]), int(r[0]["divert_at"]), int(r[0]["shared_hits"])) == (2, 2, 3)
    assert int(r[0]["bits"]) & 8
    # t4-like: flagged entry is the last hit -> divert (R7), not truncated
    r = o.process_prompts([B.prompt(["E1", "E2", "Z9"])], [4])
    assert (int(r[0]["reused"]), int(r[0]["divert_at"]), int(r[0]["shared_hits"])) == (2, 2, 2)
    assert not int(r[0]["bits"]) & 8


def test_flagged_last_hit_diverts_even_for_its_owner():
    """R7 (SPEC S:177/S:184 literal, P:458 'if not, reuse stops at the flagged prefix'): with
    no next cached entry, even the flagged entry's owner continues in its own Iso namespace,
    and still reuses what it cached there."""
    B = Blocks(seed=8)
    o = Oracle(16, SEED, POLICY_SOLIDARITY)
    r = o.process_prompts([B.prompt(["A", "B"]), B.prompt(["A", "B", "C"]),
                           B.prompt(["A", "B", "W"]), B.prompt(["A", "B", "W", "V"])],
                          [1, 2, 1, 1])
    assert r["flag_depth"].tolist() == [0, 2, 0, 0]
    assert r["divert_at"].tolist() == [-1, -1, 2, 2]
    assert r["reused"].tolist() == [0, 2, 2, 3]


def test_metadata_updated_when_isolation_deactivated():
    """enforce=0 still flags (R11) and never diverts."""
    B = Blocks(seed=7)
    o = Oracle(16, SEED, POLICY_SOLIDARITY)
    r = o.process_prompts([B.prompt(["A", "B", "C"]), B.prompt(["A", "B", "D"]),
                           B.prompt(["A", "B", "C", "E"])], [1, 2, 3], enforce=[1, 0, 0])
    assert r["flag_depth"].tolist() == [0, 2, 3]   # u3 reuses u1's C -> flags it
    assert r["divert_at"].tolist() == [-1, -1, -1]
    assert r["reused"].tolist() == [0, 2, 3]     # would be f=2 / r=2 with enforce on


def test_owner_immutable_and_flag_monotone():
    """I1/I2 (P:441 'set exactly once ... immutable'; S:88-89 flag monotone): replay a random
    stream request by request and check every transition of the dump."""
    from workloads.gen import random_small
    s = random_small(300, users=4, alphabet_blocks=3, max_blocks=5, seed=21)
    o = Oracle(16, SEED, POLICY_SOLIDARITY)
    prev = {}
    for j in range(s.n_requests):
        sj = s.slice(j, j + 1)
        o.process(sj)
        cur = table_as_dict(o)
        for k, (own, sh) in prev.items():
            assert k in cur                       # no eviction on this path (R9/D6)
            assert cur[k][0] == own               # owner immutable
            if sh != NONE:
                assert cur[k][1] == sh            # flag monotone, sharer written once
        for k, (own, sh) in cur.items():
            if k not in prev:
                assert own == int(s.users[j])     # new entries carry the requester
        prev = cur
