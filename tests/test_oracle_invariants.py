"""Invariant, brute-force and independent-reference pins for the oracle (SURVEY §8(c) I4-I10, P3,
P4).  All streams are small; everything runs on CPU in seconds."""
import itertools

import numpy as np
import pytest

from oracle import Oracle, POLICY_APC, POLICY_SOLIDARITY, POLICY_USER_ISOLATION
from oracle_helpers import Blocks, NONE, lcp_blocks, prompts_of, table_as_dict
from trie_ref import TrieRef
from workloads.gen import random_small

SEED = 0x5011D000


def _streams():
    for seed in range(1, 9):
        yield random_small(160, users=int(1 + seed % 4), alphabet_blocks=3, max_blocks=6,
                           seed=seed, enforce_prob=0.8 if seed % 2 else 1.0)


@pytest.mark.parametrize("policy", [POLICY_APC, POLICY_USER_ISOLATION, POLICY_SOLIDARITY])
def test_trie_reference_agrees(policy):
    """I10: an independent content-keyed trie (no hashing) gives the same per-request results
    and the same table, entry by entry (keys mapped through oracle.chain)."""
    for s in _streams():
        o = Oracle(16, SEED, policy)
        res = o.process(s)
        t = TrieRef(16, policy)
        en = s.enforce if s.enforce is not None else np.ones(s.n_requests, np.uint8)
        for j, p in enumerate(prompts_of(s)):
            exp = t.admit(p, int(s.users[j]), bool(en[j]))
            got = tuple(int(res[j][f]) for f in
                        ["n_blocks", "shared_hits", "reused", "divert_at", "flag_depth", "bits"])
            assert got == exp, (s.name, j, got, exp)
        tab = table_as_dict(o)
        assert len(tab) == len(t.table)
        for name, owner, sharer in t.entries():
            if name[0] == "S":
                toks = np.concatenate([np.array(b, np.uint32) for b in name[1]])
                _, K = o.chain(toks)
            else:
                _, root, u, path = name
                toks = np.concatenate([np.array(b, np.uint32) for b in root + path])
                _, K = o.chain(toks, u, len(root))
            assert tab[int(K[-1])] == (owner, sharer)


def test_apc_equals_bruteforce_lcp():
    """I9: under Prefix Caching (no eviction) r_j = max_{i<j} full-block LCP(prompt_i, prompt_j)."""
    for s in _streams():
        r = Oracle(16, SEED, POLICY_APC).process(s)["reused"]
        ps = prompts_of(s)
        for j in range(len(ps)):
            exp = max([lcp_blocks(ps[i], ps[j]) for i in range(j)], default=0)
            assert int(r[j]) == exp


def test_user_isolation_equals_per_user_lcp():
    """I6: full isolation = per-user caches: r_j = max over earlier SAME-user requests."""
    for s in _streams():
        res = Oracle(16, SEED, POLICY_USER_ISOLATION).process(s)
        ps = prompts_of(s)
        for j in range(len(ps)):
            exp = max([lcp_blocks(ps[i], ps[j]) for i in range(j) if s.users[i] == s.users[j]],
                      default=0)
            assert int(res["reused"][j]) == exp
            assert int(res["shared_hits"][j]) == 0 and int(res["divert_at"][j]) == 0


def test_no_isolation_equals_apc():
    """I5: enforce=0 everywhere => same r as APC per request and
    the same key set with the same owners; only `sharer` metadata differs."""
    for s in _streams():
        s.enforce = np.zeros(s.n_requests, np.uint8)
        o1, o2 = Oracle(16, SEED, POLICY_APC), Oracle(16, SEED, POLICY_SOLIDARITY)
        r1, r2 = o1.process(s), o2.process(s)
        assert (r1["reused"] == r2["reused"]).all()
        assert (r2["divert_at"] == -1).all()
        t1, t2 = table_as_dict(o1), table_as_dict(o2)
        assert t1.keys() == t2.keys()
        assert all(t1[k][0] == t2[k][0] for k in t1)
        assert all(v[1] == NONE for v in t1.values())


def test_single_user_and_disjoint_users():
    """I7 owner totality: a single-user stream behaves as APC with no flags.
    I8 (W1): users with no shared first block -> all three policies give equal r."""
    s = random_small(200, users=1, alphabet_blocks=3, max_blocks=6, seed=31)
    ra = Oracle(16, SEED, POLICY_APC).process(s)
    rc = Oracle(16, SEED, POLICY_SOLIDARITY).process(s)
    assert (ra["reused"] == rc["reused"]).all() and (rc["flag_depth"] == 0).all()
    B = Blocks(seed=32)
    rng = np.random.default_rng(32)
    prompts, users = [], []
    for i in range(150):
        u = int(rng.integers(4))
        names = [f"F{u}"] + [f"x{int(rng.integers(3))}" for _ in range(int(rng.integers(0, 5)))]
        prompts.append(B.prompt(names)); users.append(u)
    outs = [Oracle(16, SEED, p).process_prompts(prompts, users)["reused"] for p in range(3)]
    assert (outs[0] == outs[1]).all() and (outs[0] == outs[2]).all()


def test_solidarity_never_exceeds_apc():
    """I4: with no eviction, CacheSolidarity reuses at most what Prefix Caching reuses."""
    for s in _streams():
        ra = Oracle(16, SEED, POLICY_APC).process(s)["reused"]
        rc = Oracle(16, SEED, POLICY_SOLIDARITY).process(s)["reused"]
        assert (rc <= ra).all()


def test_isolated_entries_hit_only_for_their_owner():
    """I3 (north star): every Iso-namespace entry is owned by its namespace user and is only
    ever reused by that user (checked through the trie's explicit namespaces)."""
    for s in _streams():
        t = TrieRef(16, POLICY_SOLIDARITY)
        en = s.enforce if s.enforce is not None else np.ones(s.n_requests, np.uint8)
        for j, p in enumerate(prompts_of(s)):
            before = set(t.table)
            n, k, r, f, _, _ = t.admit(p, int(s.users[j]), bool(en[j]))
            if f > 0 and r > f:       # reused isolated entries: all pre-existing and u's own
                blk = t._blocks(p)
                for b in range(f + 1, r + 1):
                    name = ("I", tuple(blk[:f]), int(s.users[j]), tuple(blk[f:b]))
                    assert name in before
        for name, owner, _ in t.entries():
            if name[0] == "I":
                assert owner == name[2]


# ----------------------------------------------------------------------------------------------
# P3: the §5 security guarantee by brute force
# ----------------------------------------------------------------------------------------------
def victim_of(history):
    return history[-1][0] if history else 1


def _guarantee_run(history, pre, secret, cands, attackers, benign, order, capacity=0,
                   victim_between=None):
    """Replay `history` (list of (user, names)), then the probing sequence pre.v_i issued by
    attackers (round robin), interleaved with disjoint benign requests (order = list of 'p'/'b').
    Returns (precondition_holds, literal_precondition, leaked).  A leak is a probe pre.secret whose
    reuse passes pre through the SHARED chain, i.e. serves the victim's pre.secret entry; reuse of
    the attacker's own isolated copies (divert at f <= |pre|) reveals nothing about the victim.
    The premise "c contains pre.secret owned by u" is part of precondition_holds."""
    B = Blocks(seed=77)
    o = Oracle(16, SEED, POLICY_SOLIDARITY, capacity=capacity)
    for u, names in history:
        o.process_prompts([B.prompt(names)], [u])
    tab = table_as_dict(o)
    pre_flagged = False
    if pre:
        _, Kpre = o.chain(B.prompt(pre))
        pre_key = int(Kpre[-1])
        pre_flagged = pre_key in tab and tab[pre_key][1] != NONE
    _, Kv1 = o.chain(B.prompt(pre + [cands[0]]))
    child_v1_present = int(Kv1[-1]) in tab
    _, Ksec = o.chain(B.prompt(pre + [secret]))
    premise = tab.get(int(Ksec[-1]), (None,))[0] == victim_of(history)
    refined = premise and len(pre) >= 1 and (pre_flagged or not child_v1_present)
    literal = premise and len(pre) >= 1 and (pre_flagged or cands[0] != secret)
    sec_key = int(Ksec[-1])
    victim = victim_of(history)
    leaked = False
    pi = bi = 0
    for kind in order:
        if kind == "p" and pi < len(cands):
            v = cands[pi]
            # with eviction the victim's entry may be gone (nothing left to leak) or re-inserted
            # by someone else: only a probe that serves the VICTIM's pre.secret entry leaks
            victims_entry = table_as_dict(o).get(sec_key, (None,))[0] == victim
            res = o.process_prompts([B.prompt(pre + [v])], [attackers[pi % len(attackers)]])[0]
            f = int(res["divert_at"])
            if (v == secret and victims_entry and int(res["reused"]) > len(pre)
                    and (f < 0 or f > len(pre))):
                leaked = True
            pi += 1
        elif kind == "b" and bi < len(benign):
            u, names = benign[bi]
            o.process_prompts([B.prompt(names)], [u])
            bi += 1
        elif kind == "v" and victim_between is not None:
            o.process_prompts([B.prompt(victim_between)], [victim])
    return refined, literal, leaked


def _histories(victim, others, alphabet, max_len, max_hist):
    prompts = [list(p) for L in range(1, max_len + 1) for p in itertools.product(alphabet, repeat=L)]
    rng = np.random.default_rng(2024)
    users = [victim] + others
    for _ in range(4000):
        h = []
        for _ in range(int(rng.integers(0, max_hist + 1))):
            h.append((users[int(rng.integers(len(users)))], prompts[int(rng.integers(len(prompts)))]))
        yield h


def test_p3_security_guarantee_bruteforce():
    """Under the refined precondition (R12: pre's final entry flagged, or no Shared
    child of pre equal to v1), no probe from a user != victim ever reuses the victim's secret
    entry, for random reachable histories (victim, 2 colluders, 1 benign; alphabet of 3 block
    contents; prompts <= 3 blocks; histories <= 6 requests) and every interleaving pattern."""
    victim, a1, a2, ben = 1, 2, 3, 4
    alphabet = ["a", "b", "c"]
    checked = leaks_refined = 0
    rng = np.random.default_rng(7)
    for hist in _histories(victim, [a1, a2, ben], alphabet, 3, 6):
        pre = [alphabet[int(rng.integers(3))] for _ in range(int(rng.integers(1, 3)))]
        secret = alphabet[int(rng.integers(3))]
        hist = hist + [(victim, pre + [secret])]
        cands = [c for c in alphabet if c != secret]
        rng.shuffle(cands)
        cands = cands + [secret]          # the correct guess is never first
        benign = [(ben, ["d", "e"]), (ben, ["e"])]
        order = list(rng.permutation(["p"] * len(cands) + ["b"] * len(benign)))
        refined, _, leaked = _guarantee_run(hist, pre, secret, cands, [a1, a2], benign, order)
        if refined:
            checked += 1
            leaks_refined += leaked
    assert checked > 1000
    assert leaks_refined == 0


def test_p3_documented_exclusions_leak():
    """The two exclusions of P:577-597 are real (witnesses), and the Q18 sibling case shows why
    the literal precondition (2) needs the refinement R12."""
    # |pre| = 0: the first entry is unprotected
    _, _, leaked = _guarantee_run([(1, ["s"])], [], "s", ["x", "s"], [2], [], ["p", "p"])
    assert leaked
    # first attempt correct on an unflagged prefix
    _, _, leaked = _guarantee_run([(1, ["p", "s"])], ["p"], "s", ["s", "x"], [2], [], ["p", "p"])
    assert leaked
    # Q18: victim cached [P V1] and [P S]; literal (2) holds (v1 != secret) but the probe of V1
    # flags V1 (the deepest reused entry, R2), not P, so the probe of S then hits.
    refined, literal, leaked = _guarantee_run([(1, ["P", "V1"]), (1, ["P", "S"])], ["P"], "S",
                                              ["V1", "S"], [2], [], ["p", "p"])
    assert literal and not refined and leaked


@pytest.mark.parametrize("capacity", [3, 4, 6])
def test_p3_security_guarantee_under_lru_eviction(capacity):
    """§5 with eviction ("eviction is benign for security"; S:117-125 LRU, flags die with
    their entry S:120/S:124): the same brute force with a capacity of 3-6 entries and the probes
    interleaved with disjoint benign requests (which evict), under the premise of P:566-572
    (probes by non-victims; the victim sends nothing during the probing): no probe ever serves
    the victim's pre.secret entry while the refined precondition held at the start."""
    victim, a1, a2, ben = 1, 2, 3, 4
    alphabet = ["a", "b", "c"]
    checked = leaks = 0
    rng = np.random.default_rng(100 + capacity)
    for hist in _histories(victim, [a1, a2, ben], alphabet, 3, 6):
        pre = [alphabet[int(rng.integers(3))] for _ in range(int(rng.integers(1, 3)))]
        secret = alphabet[int(rng.integers(3))]
        hist = hist + [(victim, pre + [secret])]
        cands = [c for c in alphabet if c != secret]
        rng.shuffle(cands)
        cands = cands + [secret]
        benign = [(ben, ["d", "e"]), (ben, ["e"]), (ben, ["f", "d"]), (ben, ["g"])]
        order = list(rng.permutation(["p"] * len(cands) + ["b"] * len(benign)))
        refined, _, leaked = _guarantee_run(hist, pre, secret, cands, [a1, a2], benign, order,
                                            capacity=capacity)
        if refined:
            checked += 1
            leaks += leaked
    assert checked > 800
    assert leaks == 0


def test_p3_eviction_reincarnation_exclusion():
    """Documented exclusion (3) (R31): outside P:566-572's premise — the VICTIM
    re-sends pre.secret after eviction removed pre and its flag — every re-cached incarnation of
    pre is unflagged again, so the attacker gets a fresh first attempt per incarnation (the
    first-attempt exclusion of P:588-595, repeated).  Witness: capacity 2; the attacker's wrong
    guess flags P; benign traffic evicts P and S (the flag dies with P); the victim
    re-sends [P S]; the attacker's next guess, the right one, is served the victim's S."""
    refined, _, leaked = _guarantee_run(
        [(1, ["P", "S"])], ["P"], "S", ["X", "S"], [2], [(4, ["d", "e"])], ["p", "b", "v", "p"],
        capacity=2, victim_between=["P", "S"])
    assert refined and leaked
    # the same sequence without the victim's re-request: no leak (the entry is gone)
    refined, _, leaked = _guarantee_run(
        [(1, ["P", "S"])], ["P"], "S", ["X", "S"], [2], [(4, ["d", "e"])], ["p", "b", "p"],
        capacity=2)
    assert refined and not leaked


# ----------------------------------------------------------------------------------------------
# P4: incremental prompt reconstruction, adaptive attacker
# ----------------------------------------------------------------------------------------------
def _reconstruct(policy, first_guess_correct=False):
    """The attacker knows the template and, for each of 2 secret blocks, 4 candidates.  It issues
    pre.cand probes and picks the candidate whose probe reused the most blocks (the timing signal);
    on success it extends pre with the recovered block and attacks the next one."""
    B = Blocks(seed=99)
    o = Oracle(16, SEED, policy)
    secret = ["S1", "S2"]
    o.process_prompts([B.prompt(["T1", "T2", "S1", "S2", "Q"])], [1])
    pre = ["T1", "T2"]
    recovered, signals = [], []
    for blk in range(2):
        cands = [f"W{blk}{i}" for i in range(3)]
        cands.insert(0 if first_guess_correct else 2, secret[blk])
        rs = []
        for c in cands:
            rs.append(int(o.process_prompts([B.prompt(pre + [c, "Q"])], [2])[0]["reused"]))
        signals.append(rs)
        best = cands[int(np.argmax(rs))] if max(rs) > min(rs) else None
        recovered.append(best)
        pre = pre + [secret[blk]]     # worst case: assume the attacker learned it anyway
    return recovered, signals


def test_p4_isolation_kicks_in():
    rec, sig = _reconstruct(POLICY_APC)
    assert rec == ["S1", "S2"]                       # Prefix Caching leaks both blocks
    rec, sig = _reconstruct(POLICY_SOLIDARITY)
    assert rec == [None, None]                       # every probe after the first is uniform
    for rs in sig:
        assert len(set(rs[1:])) == 1
    rec, _ = _reconstruct(POLICY_SOLIDARITY, first_guess_correct=True)
    assert rec[0] == "S1"                            # documented exclusion
