#!/usr/bin/env python
"""Benchmark: prefix lookups/s of the CacheSolidarity hot path on B200 (BASELINE.json metric).

A step = one batch admission (solid_admit_batch = lookup + insert: hash, scan, probe, Detector
resolution, commit) of the C2 workload (BASELINE configs[1]: 1000 users x 100 requests x 2000
tokens, 80% common system prompt), inputs resident in HBM, on an index restored to the same
(empty) pre-batch state before every step (restore is outside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

N > 1 (torchrun, one process per GPU): one key-hash-sharded index across the ranks (DESIGN.md
§7): the global batch is the C2 shape scaled by N, rank r admits its contiguous slice, records
move over NCCL once per resolver round (timed separately); weak scaling; the time is the max over
ranks.  `--impl reference` times the sequential CPU oracle on the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefix lookups/sec (requests & blocks) at 1/2/4/8 B200; % HBM roofline"
SEED = 0x5011D000


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _workload(name: str, rank: int):
    from workloads import c2_shared_prompt
    if name == "c2":
        s = c2_shared_prompt(seed=SEED + 2 + 1000 * rank)
        desc = ("c2_shared_prompt: 1000 users x 100 requests, 2000-token prompts (1600-token common "
                "system prompt = 80%, 256-token per-user profile, 144 fresh), one 100k-request batch")
        return s, desc
    if name == "c2_small":
        s = c2_shared_prompt(users=100, reqs_per_user=100, seed=SEED + 2 + 1000 * rank)
        return s, "c2_shared_prompt scaled to 100 users x 100 requests (quick check)"
    raise SystemExit(f"unknown config {name}")


def config_n1(desc: str, n_req: int, n_blk: int, n_tok: int) -> dict:
    """The N = 1 line's `config` (shared by both arms, so the driver compares like with like)."""
    return {"workload": desc, "policy": "solidarity", "batch_requests": n_req,
            "blocks_per_batch": n_blk, "tokens_per_batch": n_tok,
            "parallelism": "1 independent tenant partitions (weak)",
            "l2": "inputs (800 MB tokens) larger than L2 (126 MB); no flush",
            "restore": "index reset to empty before every step, outside the events "
                       "(stream-ordered between consecutive steps)",
            "submission": "solid_admit_batch pipelined: step k+1 enqueued before "
                          "step k's status is collected"}


def sharded_shape(config: str, world: int):
    """Requests per GPU and users of the N > 1 (weak-scaling) workload."""
    per = 100_000 if config == "c2" else 10_000
    users = (1000 if config == "c2" else 100) * world
    return per, users


def config_sharded(world: int, users: int, per: int) -> dict:
    """The N > 1 line's `config` (shared by both arms; the transport is reported beside it)."""
    return {"workload": f"c2_shared_prompt x{world}: {users} users x 100 requests, "
                        f"2000-token prompts, {per} requests per GPU",
            "policy": "solidarity", "parallelism": f"key-hash-sharded index over "
            f"{world} GPUs, record exchange per resolver round",
            "l2": "inputs larger than L2", "restore": "index reset before each step"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.path = gpu, None, None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm.append(float(parts[0])); mx.append(float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[2:]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            os.unlink(self.path)
        except Exception:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(stream, sample_requests: int):
    """The oracle as it stands (sequential, one thread) on the first `sample_requests` requests.
    Returns (baseline object, oracle results, oracle index dump) — the last two let the caller
    check the timed GPU step against the oracle on the same stream (parity of what is timed)."""
    from oracle import Oracle
    s = stream.slice(0, min(sample_requests, stream.n_requests))
    o = Oracle(16, SEED, 2)
    o.reserve(s.n_blocks() // 8 + 1024)
    t0 = time.perf_counter()
    res = o.process(s)
    dt = time.perf_counter() - t0
    info = {"value": s.n_requests / dt, "unit": "requests/s", "cores": 1, "kind": "oracle",
            "blocks_per_s": s.n_blocks() / dt, "seconds": dt, "host_cores": os.cpu_count(),
            "cpu_model": _cpu_model(),
            "sample": f"first {s.n_requests} requests ({s.n_blocks()} blocks) of the same stream, "
                      f"sequential C++ oracle, 1 thread (host has {os.cpu_count()} cores)"}
    return info, res, o.dump()


def parity_of_timed_step(res, dump, exp, exp_dump):
    """Element-by-element comparison of the last timed step's results and the index it left with
    the oracle's on the same stream (every result field; key, owner, sharer of every entry)."""
    fields = list(exp.dtype.names)
    bad = {f: int((res[f].astype(np.int64) != exp[f].astype(np.int64)).sum()) for f in fields}
    same_len = len(dump) == len(exp_dump)
    bad_idx = {f: (int((dump[f] != exp_dump[f]).sum()) if same_len else None)
               for f in ("key", "owner", "sharer")}
    ok = same_len and not any(bad.values()) and not any(bad_idx.values())
    return {"status": "exact" if ok else "MISMATCH", "requests": int(len(exp)),
            "entries": int(len(exp_dump)), "result_fields": fields, "mismatches": bad,
            "index_mismatches": bad_idx, "index_entries_gpu": int(len(dump)),
            "what": "last timed step's solid_result[] and the index it committed vs the oracle "
                    "on the same 100 000-request stream"}


def measure_activator(dev, args):
    """the Activator over a C2-sized query list — 100 000 queries against a
    stream of 2^20 completed-request TTFT samples, the window advancing every 100 queries (1 000
    distinct windows of up to 256 + 256 samples, 512-point grid), inputs resident in HBM."""
    import torch
    import paper_2603_10726_b200 as P
    from workloads import query_cuts, ttft_stream
    M, N, stride, W, G = 1 << 20, 100_000, 100, 256, 512
    s = ttft_stream(M, seed=SEED + 0xF2)
    cuts_np = query_cuts(N, M, stride=stride)
    d = lambda a, t: torch.from_numpy(np.ascontiguousarray(a)).to(dtype=t, device=dev)
    tt, pt = d(s.ttft_ms, torch.float64), d(s.prompt_tokens.astype(np.int32), torch.int32)
    rf, cuts = d(s.reuse_fraction, torch.float64), d(cuts_np, torch.int64)
    act = P.Activator(theta=0.5, window_len=W, grid=G, max_samples=M, max_queries=N,
                      device=dev.index or 0)
    cs = torch.cuda.current_stream(dev)
    ov, en = act.run(tt, pt, rf, cuts)
    reps, ms = 5, []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        act.run(tt, pt, rf, cuts, overlap=ov, enforce=en)
        e1.record(cs)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    med = statistics.median(ms)
    # work accounting: distinct windows and Gaussian-kernel evaluations (grid x window sizes)
    hit = np.concatenate([[0], np.cumsum(s.reuse_fraction >= 0.8)])
    miss = np.concatenate([[0], np.cumsum(s.reuse_fraction <= 0.2)])
    heads = np.unique(cuts_np)
    wh, wm = np.minimum(hit[heads], W), np.minimum(miss[heads], W)
    full = (wh >= 2) & (wm >= 2)
    evals = int((G * (wh + wm))[full].sum())
    en_np = en.cpu().numpy()
    out = {"workload": f"{N} queries, {M} TTFT samples (ttft_stream seed {SEED + 0xF2:#x}), "
                       f"window every {stride} queries, window_len {W}, grid {G}, theta 0.5",
           "ms_per_call": med, "ms_all": ms, "queries_per_s": N / (med / 1e3),
           "windows": int(heads.size), "windows_per_s": heads.size / (med / 1e3),
           "kernel_evals_per_s": evals / (med / 1e3), "enforced_fraction": float(en_np.mean()),
           "dtype": "f64", "launches_per_call": 5}
    # ALU roofline of the window kernel (fp64-bound): fp64 instructions per call from the ncu
    # capture of this same workload (profiles/latest_ncu.json) over the measured call time,
    # against the measured DFMA rate (scripts/micro/fp64.cu): instructions, not flops.
    try:
        with open(os.path.join(ROOT, "profiles", "latest_ncu.json")) as f:
            pa = json.load(f)["activator"]
        inst = pa["k_act_window"]["fp64_warp_instructions"] * 32
        peak = pa["fp64_peak"]["fma_tflops"] / 2 * 1e12          # DFMA instructions / s
        out["roofline"] = {"bound": "alu", "kernel": "k_act_window (fp64 KDE)",
                           "achieved": inst / (med / 1e3) / 1e12, "peak": peak / 1e12,
                           "unit": "T fp64 instr/s", "frac": inst / (med / 1e3) / peak,
                           "fp64_pipe_active_pct_ncu": pa["k_act_window"]["fp64_pipe_active_pct"],
                           "source": "profiles/latest_ncu.json"}
    except Exception:
        pass
    if not args.no_cpu:
        from oracle.activator import ActivatorConfig, isolation_active, windows
        cfg = ActivatorConfig(theta=0.5, window_len=W, grid=G)
        sample = [int(c) for c in np.linspace(2000, 40000, 8).astype(np.int64)]
        t0 = time.perf_counter()
        for c in sample:
            isolation_active(*windows(s.ttft_ms, s.prompt_tokens, s.reuse_fraction, c, cfg), cfg)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": len(sample) / dt, "unit": "windows/s", "cores": 1,
                               "kind": "oracle", "sample": f"{len(sample)} windows, cuts 2000-40000"}
    return out


def measure_evict(dev, args):
    """LRU eviction (evict mode) on the C3 multi-turn shape
    (BASELINE configs[2]: 10k users, conversations growing to 8k tokens) with the index capped
    at 1M entries: warmed (untimed, on the GPU) until the cache is full and evicting, then one
    step = one batch of 2 000 requests (a fifth of a round) admitted with lookup + insert,
    index restored to the same warm state before every step (outside the events)."""
    import torch
    import paper_2603_10726_b200 as P
    from workloads import c3_multiturn
    cap, users, bsz = 1_000_000, 10_000, 2_000
    warm, timed = c3_multiturn(users=users, warm_blocks=cap, timed_rounds=1, seed=SEED + 3)
    batch = timed.slice(0, bsz)
    wb = [warm.slice(i, min(i + bsz, warm.n_requests)) for i in range(0, warm.n_requests, bsz)]
    max_tok = max(max(b.n_tokens for b in wb), batch.n_tokens) + 64
    idx = P.Index("solidarity", capacity_blocks=cap, max_batch_tokens=max_tok,
                  max_batch_requests=bsz, seed=SEED, device=dev.index or 0, evict=True)

    def admit_split(b):
        try:
            idx.admit(**P.to_device(b, dev))
        except P.SolidError as e:
            if e.status != P.SOLID_ERR_CAPACITY or b.n_requests < 2:
                raise
            h = b.n_requests // 2
            admit_split(b.slice(0, h)); admit_split(b.slice(h, b.n_requests))
    t0 = time.perf_counter()
    for b in wb:
        admit_split(b)
    warm_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    idx.checkpoint()
    d = P.to_device(batch, dev)
    out = torch.empty((bsz, 6), dtype=torch.int32, device=dev)
    cs = torch.cuda.current_stream(dev)
    ms, st = [], None
    prof = os.environ.get("SOLID_PROFILE_EVICT")   # ncu --profile-from-start off: last step only
    nsteps = args.warmup + max(args.steps, 3)
    for k in range(nsteps):
        idx.restore()
        torch.cuda.synchronize()
        if prof and k == nsteps - 1:
            torch.cuda.profiler.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        idx.lookup(d["tokens"], d["offsets"], d["users"], None, out=out)
        idx.insert()
        e1.record(cs)
        torch.cuda.synchronize()
        if prof and k == nsteps - 1:
            torch.cuda.profiler.stop()
        if k >= args.warmup:
            ms.append(e0.elapsed_time(e1))
            st = idx.stats()
    med = statistics.median(ms)
    nblk = batch.n_blocks()
    res = P.as_numpy(out)
    r = {"workload": f"c3_multiturn {users} users, index capped at {cap} entries (LRU), warmed "
                     f"with {warm.n_requests} requests ({warm.n_blocks()} blocks) until full; "
                     f"one batch = {bsz} requests ({nblk} blocks, {batch.n_tokens} tokens)",
         "ms_per_batch": med, "ms_all": ms, "requests_per_s": bsz / (med / 1e3),
         "blocks_per_s": nblk / (med / 1e3), "evicted_per_batch": st["last_evicted"],
         "inserted_per_batch": st["last_inserted"], "reused_blocks": int(res["reused"].sum()),
         "window_keys": st["last_window_keys"], "evict_iterations": st["last_evict_iters"],
         "resolver_rounds": st["last_rounds"], "launches_per_batch": st["last_kernel_launches"],
         "phases_ms": {"hash": st["ms_hash"], "resolve_and_window": st["ms_resolve"],
                       "commit_evict_lru": st["ms_commit"]},
         "live_entries": st["live_entries"], "warm_wall_s": warm_s,
         "how": "lookup (synchronises: host-driven eviction-time iteration) + insert, CUDA "
                "events on the stream around both, median"}
    if not args.no_cpu:
        from oracle import Oracle
        sample = warm.slice(0, 6000)
        o = Oracle(16, SEED, 2, capacity=20_000)
        t0 = time.perf_counter()
        o.process(sample)
        dt = time.perf_counter() - t0
        r["cpu_baseline"] = {"value": sample.n_requests / dt, "unit": "requests/s", "cores": 1,
                             "kind": "oracle", "blocks_per_s": sample.n_blocks() / dt,
                             "sample": f"first {sample.n_requests} warm requests "
                                       f"({sample.n_blocks()} blocks) with capacity 20 000 "
                                       f"(evicting: {o.evictions()} evictions), 1 thread"}
    return r


def measure_policy_eval(dev, args):
    """hit rates of the three policies on W1-W5 (P:744-772, 10 users x 100
    requests, single- and two-level templates) and the θ sweep on two-level W4, the
    CUDA library as the cache and the CUDA Activator in the loop (workloads/policy_eval.py)."""
    import torch
    import paper_2603_10726_b200 as P
    from workloads.policy_eval import PRESETS, closed_loop, hit_rate, preset, two_level

    def admit_fn(policy, s):
        idx = P.Index(policy, capacity_blocks=1 << 16, max_batch_tokens=s.n_tokens + 64,
                      max_batch_requests=s.n_requests, seed=SEED, device=dev.index or 0)
        return lambda b: P.as_numpy(idx.admit(**P.to_device(b, dev)))
    t0 = time.perf_counter()
    table = {}
    for gname, gen in (("single", preset), ("two_level", two_level)):
        for w in PRESETS:
            s = gen(w)
            row = {}
            for pol in ("apc", "user_isolation", "solidarity"):
                a = admit_fn(pol, s)
                res = np.concatenate([a(s.slice(i, min(i + 100, s.n_requests)))
                                      for i in range(0, s.n_requests, 100)])
                row[pol] = round(hit_rate(res), 4)
            table[f"{gname}:{w}"] = row
    # the same workloads under cache pressure: LRU eviction (evict mode) at 1000 entries, about a
    # third of the smallest working set (cf. the paper's LLaMA-13B remark)
    def admit_lru(policy, s, cap=1000, batch=25):
        idx = P.Index(policy, capacity_blocks=cap, max_batch_tokens=s.n_tokens + 64,
                      max_batch_requests=batch, max_blocks=64, seed=SEED, device=dev.index or 0,
                      evict=True)

        def one(b):
            try:
                return P.as_numpy(idx.admit(**P.to_device(b, dev)))
            except P.SolidError as e:
                if e.status != P.SOLID_ERR_CAPACITY or b.n_requests < 2:
                    raise
                h = b.n_requests // 2
                return np.concatenate([one(b.slice(0, h)), one(b.slice(h, b.n_requests))])
        return np.concatenate([one(s.slice(i, min(i + batch, s.n_requests)))
                               for i in range(0, s.n_requests, batch)])
    table_lru = {}
    for gname, gen in (("single", preset), ("two_level", two_level)):
        for w in PRESETS:
            s = gen(w)
            table_lru[f"{gname}:{w}"] = {pol: round(hit_rate(admit_lru(pol, s)), 4)
                                         for pol in ("apc", "user_isolation", "solidarity")}
    s = two_level("W4")
    d = lambda a, t: torch.from_numpy(np.ascontiguousarray(a)).to(dtype=t, device=dev)
    sweep = {}
    for th in np.linspace(0.0, 1.0, 11):
        act = P.Activator(theta=float(th), max_samples=s.n_requests + 1, max_queries=64,
                          device=dev.index or 0)
        fn = lambda tt, pt, fr, c: act.run(d(tt, torch.float64), d(pt.astype(np.int32), torch.int32),
                                           d(fr, torch.float64), d(c, torch.int64))[1].cpu().numpy()
        res, en, _ = closed_loop(s, admit_fn("solidarity", s), fn, batch=50)
        sweep[f"{th:.1f}"] = {"hit_rate": round(hit_rate(res), 4),
                              "enforced": round(float(en.mean()), 3)}
    return {"workloads": "W1-W5 presets (10 users x 100 requests, seed 0x5011D0F3); two_level = "
                         "templates in families of 8 sharing a 3-block preamble",
            "hit_rates": table, "hit_rates_lru_1000_entries": table_lru,
            "theta_sweep_two_level_W4": sweep,
            "wall_s": time.perf_counter() - t0,
            "how": "library admission in batches of 100 (sweep: 50, Activator windows of the "
                   "samples completed before each batch; synthetic TTFT stand-in)"}


def measure_hash2(dev, args, d, stream_np):
    """the same C2 step with H-def v3 two-component keys (hash_components=2,
    DESIGN.md §11) — the ALU price of the hardening on the fused hash kernel."""
    import torch
    import paper_2603_10726_b200 as P
    N, nblk = stream_np.n_requests, stream_np.n_blocks()
    idx = P.Index("solidarity", capacity_blocks=max(nblk // 6, 1 << 20),
                  max_batch_tokens=stream_np.n_tokens + 64, max_batch_requests=N, seed=SEED,
                  device=dev.index or 0, hash_components=2)
    out = torch.empty((N, 6), dtype=torch.int32, device=dev)
    cs = torch.cuda.current_stream(dev)
    ms, hk = [], []
    for k in range(args.warmup + max(args.steps, 3)):
        idx.reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        idx.admit_async(d["tokens"], d["offsets"], d["users"], d["enforce"], out=out)
        e1.record(cs)
        idx.status()
        if k >= args.warmup:
            ms.append(e0.elapsed_time(e1))
            hk.append(idx.stats()["ms_hash_kernel"])
    med = statistics.median(ms)
    return {"ms_per_step": med, "requests_per_s": N / (med / 1e3),
            "hash_kernel_ms": statistics.median(hk),
            "workload": "C2 bench batch (same inputs), hash_components=2"}


def measure_block_table(dev, args, d, stream_np):
    """the C2 step with physical block ids and the block table
    (block_table=True) against the same synchronous step without — the price of
    the allocator (pre-pass, count, scan, assign, table, copy-out)."""
    import torch
    import paper_2603_10726_b200 as P
    N, nblk = stream_np.n_requests, stream_np.n_blocks()
    cs = torch.cuda.current_stream(dev)
    res = {}
    for bt in (False, True):
        idx = P.Index("solidarity", capacity_blocks=max(nblk // 6, 1 << 20),
                      max_batch_tokens=stream_np.n_tokens + 64, max_batch_requests=N, seed=SEED,
                      device=dev.index or 0, block_table=bt)
        out = torch.empty((N, 6), dtype=torch.int32, device=dev)
        table = torch.empty(((stream_np.n_tokens + 15) // 16,), dtype=torch.int32, device=dev)
        ms = []
        for k in range(args.warmup + max(args.steps // 5, 3)):
            idx.reset()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            idx.admit(d["tokens"], d["offsets"], d["users"], d["enforce"], out=out)
            if bt:
                idx._check(idx.lib.solid_block_table(idx.h, ctypes.c_void_p(table.data_ptr()),
                                                      idx._stream(None)))
            e1.record(cs)
            torch.cuda.synchronize(dev)
            if k >= args.warmup:
                ms.append(e0.elapsed_time(e1))
        res["with_block_table" if bt else "without"] = statistics.median(ms)
        idx.close()
    res["overhead_ms"] = res["with_block_table"] - res["without"]
    res["workload"] = ("C2 bench batch, synchronous admit (lookup + insert) "
                       "± physical block ids + block table copy-out")
    res["table_entries"] = nblk
    return res


def measure_configs(dev, args):
    """The other BASELINE configs as timed single-GPU batches (their full-size parity tests are
    test_c3_full_size_warm_then_timed / test_c4_full_size):
      configs[2] C3: 10 000 users, conversations to 8 k tokens, warm phase admitted untimed
                 (index checkpointed), then the 8 timed rounds as one 80 000-request batch;
      configs[3] C4: 1 M requests (500 k benign + victims + 500 k colluding probes), one batch.
    Per step the index is restored to the pre-batch state outside the CUDA events."""
    import torch
    import paper_2603_10726_b200 as P
    from workloads import c3_multiturn, c4_attackers
    out = {}
    cs = torch.cuda.current_stream(dev)
    for name in ("c3", "c4"):
        if name == "c3":
            warm, s = c3_multiturn()
            pre = [warm]
            desc = ("c3_multiturn: 10 000 users, warm phase untimed, timed = 8 rounds as one "
                    f"{s.n_requests}-request batch")
        else:
            s, pre = c4_attackers(), []
            desc = f"c4_attackers: {s.n_requests} requests (50 % colluding probes), one batch"
        mt = max([s.n_tokens] + [w.n_tokens for w in pre]) + 64
        mr = max([s.n_requests] + [w.n_requests for w in pre])
        blocks = s.n_blocks() + sum(w.n_blocks() for w in pre)
        idx = P.Index("solidarity", capacity_blocks=max(blocks, 1 << 20), max_batch_tokens=mt,
                      max_batch_requests=mr, seed=SEED, device=dev.index or 0)
        for w in pre:
            idx.admit(**P.to_device(w, dev))
        idx.checkpoint()
        d = P.to_device(s, dev)
        o = torch.empty((s.n_requests, 6), dtype=torch.int32, device=dev)
        ms, rounds = [], []
        for k in range(args.warmup + max(args.steps // 5, 3)):
            idx.restore()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            idx.admit_async(d["tokens"], d["offsets"], d["users"], d["enforce"], out=o)
            e1.record(cs)
            idx.status()
            if k >= args.warmup:
                ms.append(e0.elapsed_time(e1))
                rounds.append(idx.stats()["last_rounds"])
        med = statistics.median(ms)
        st = idx.stats()
        r = P.as_numpy(o)
        out[name] = {"workload": desc, "ms_per_batch": med, "requests_per_s": s.n_requests / (med / 1e3),
                     "blocks_per_s": s.n_blocks() / (med / 1e3), "resolver_rounds": rounds[-1],
                     "resolver_round_us": [round(x, 1) for x in st["round_us"]],
                     "phases_ms": {"hash": st["ms_hash"], "resolve": st["ms_resolve"],
                                   "commit": st["ms_commit"]},
                     "algorithmic_bytes": st["algorithmic_bytes"],
                     "whole_step_hbm_frac": st["algorithmic_bytes"] / (med / 1e3) / 1e9 / _peaks()[0],
                     "diverted": int(((r["bits"] & 4) > 0).sum()),
                     "hit_rate": float(r["reused"].sum() / max(r["n_blocks"].sum(), 1))}
        del idx, d, o
        torch.cuda.empty_cache()
    return out


def measure_c5(dev, args):
    """BASELINE configs[4] C5 on ONE GPU (one B200 holds it): warm phase (200 000
    users' conversations, ~1.06e8 entries) admitted untimed, index checkpointed; one step = the
    4 000 000-request batch (4.2e9 tokens, 16.9 GB of token ids) admitted with
    solid_admit_batch; the index restored to the warm state before every step (outside the
    events).  Tokens are generated on the device (workloads/c5.py materialize_torch)."""
    import torch
    import paper_2603_10726_b200 as P
    from workloads.c5 import c5_large
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from c5_props import c5_check        # the per-request values C5's structure fixes
    t0 = time.perf_counter()
    warm, timed = c5_large(scale=1.0)
    cap = warm.n_blocks() + timed.n_blocks() // 4 + (1 << 16)
    idx = P.Index("solidarity", capacity_blocks=cap,
                  max_batch_tokens=max(warm.n_tokens, timed.n_tokens) + 64,
                  max_batch_requests=max(warm.n_requests, timed.n_requests), seed=SEED,
                  device=dev.index or 0, max_blocks=1024)
    wt, wo, wu = warm.materialize_torch(dev)
    idx.admit(wt, wo, wu, None)
    torch.cuda.synchronize()
    live0 = idx.stats()["live_entries"]
    del wt, wo, wu
    torch.cuda.empty_cache()
    idx.checkpoint()
    tt, to, tu = timed.materialize_torch(dev)
    out = torch.empty((timed.n_requests, 6), dtype=torch.int32, device=dev)
    setup_s = time.perf_counter() - t0
    cs = torch.cuda.current_stream(dev)
    ms, st = [], None
    for k in range(1 + max(args.steps // 10, 3)):
        idx.restore()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        idx.admit_async(tt, to, tu, None, out=out)
        e1.record(cs)
        idx.status()
        if k >= 1:
            ms.append(e0.elapsed_time(e1))
            st = idx.stats()
    med = statistics.median(ms)
    got = P.as_numpy(out)
    nblk = timed.n_blocks()
    r = {"workload": f"c5_large: warm {warm.n_requests} conversations -> {live0} entries "
                     f"(untimed); timed = ONE batch of {timed.n_requests} requests "
                     f"({timed.n_tokens} tokens, {nblk} blocks): "
                     f"{timed.meta['continuing']} continuing, {timed.meta['new_sessions']} new "
                     f"sessions, {timed.meta['probes']} probes",
         "n_gpus": 1, "ms_per_batch": med, "ms_all": ms,
         "requests_per_s": timed.n_requests / (med / 1e3), "blocks_per_s": nblk / (med / 1e3),
         "resolver_rounds": st["last_rounds"],
         "phases_ms": {"hash": st["ms_hash"], "resolve": st["ms_resolve"],
                       "commit": st["ms_commit"]},
         "round_us": st["round_us"], "algorithmic_bytes": st["algorithmic_bytes"],
         "whole_step_hbm_frac": st["algorithmic_bytes"] / (med / 1e3) / 1e9 / _peaks()[0],
         "hash_kernel_hbm_frac": (64 * nblk + 12 * timed.n_requests + 16 * st["last_shared_keys"])
                                 / (st["ms_hash_kernel"] / 1e3) / 1e9 / _peaks()[0],
         "live_entries_before": live0, "inserted": st["last_inserted"],
         "index_slots": int(1 << (2 * cap - 1).bit_length()),
         "parity": c5_check(timed, got), "setup_s": setup_s,
         "hit_rate": float(got["reused"].sum() / max(got["n_blocks"].sum(), 1))}
    del idx, tt, to, tu, out
    torch.cuda.empty_cache()
    return r


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    stream, desc = _workload(args.config, 0)
    from oracle import Oracle
    n_sample = min(stream.n_requests, args.ref_sample)
    s = stream.slice(0, n_sample)
    if args.gpus > 1:       # the arm it stands beside: the sharded C2 x N workload
        per, users = sharded_shape(args.config, args.gpus)
        cfg = config_sharded(args.gpus, users, per)
    else:
        cfg = config_n1(desc, stream.n_requests, stream.n_blocks(), stream.n_tokens)
    times = []
    for step in range(args.warmup + args.steps):
        o = Oracle(16, SEED, 2)
        o.reserve(s.n_blocks() // 8 + 1024)
        t0 = time.perf_counter()
        o.process(s)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    tot = sum(times)
    v = n_sample * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "requests/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "blocks_per_s": s.n_blocks() * args.steps / tot,
            "config": cfg,
            "cpu_baseline": {"value": v, "unit": "requests/s", "cores": 1, "kind": "oracle",
                             "sample": f"first {n_sample} requests ({s.n_blocks()} blocks) of the "
                                       f"workload per step, sequential oracle, 1 thread"},
            "e2e": {"value": v, "unit": "requests/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_sharded(args, world, rank, local):
    """N > 1: one key-hash-sharded index over all ranks.  The global batch is the
    C2 shape scaled by N (N x 1000 users sharing the system prompt, N x 100 000 requests, one
    seeded shuffle); rank r admits its contiguous slice; keys live on their owner shard; the
    REG / PULL / INT records move each resolver round (peer memory, or NCCL).  Weak scaling: fixed requests
    per GPU.  Collectives are timed separately (host clock around the exchange calls, after a
    stream sync; the step itself by CUDA events, max over ranks)."""
    import torch
    import torch.distributed as dist
    import paper_2603_10726_b200 as P
    from paper_2603_10726_b200.dist import (PeerExchange, PeerUnavailable, ShardedIndex,
                                            TorchExchange, run_protocol, run_protocol_device)
    from workloads import c2_shared_prompt

    per, users = sharded_shape(args.config, world)
    lo, hi = rank * per, (rank + 1) * per
    s = c2_shared_prompt(users=users, reqs_per_user=100, lo=lo, hi=hi, seed=SEED + 2)
    nblk = s.n_blocks()
    dev = torch.device("cuda", local)
    d = P.to_device(s, dev)
    shard = ShardedIndex(world, rank, "solidarity", capacity_blocks=max(nblk // 6, 1 << 20),
                         max_batch_tokens=s.n_tokens + 64, max_batch_requests=per, seed=SEED,
                         device=local)
    # Transport (SOLID_DIST_EXCHANGE): "native" (default) = the whole sharded admission as ONE
    # C-ABI call, solid_dist_admit (agreement, rounds, commit and overflow vote
    # inside the library over CUDA-IPC peer memory); "p2p-dev" / "p2p" = the same exchange
    # driven from Python (device- / host-resident counts); "torch" = torch.distributed (NCCL, or
    # gloo with host staging).  If some rank cannot map its peers, every rank falls back to torch.
    xport = os.environ.get("SOLID_DIST_EXCHANGE", "native")
    ex = None

    def make_shard():
        return ShardedIndex(world, rank, "solidarity", capacity_blocks=max(nblk // 6, 1 << 20),
                            max_batch_tokens=s.n_tokens + 64, max_batch_requests=per, seed=SEED,
                            device=local)

    if xport in ("native", "p2p", "p2p-dev"):
        try:
            ex = PeerExchange(shard, device_counts=xport == "p2p-dev")
            xname = {"native": "solid_dist_admit (one C-ABI call; CUDA IPC peer stores + mailbox "
                               "flags, device-resident counts)",
                     "p2p-dev": "p2p (CUDA IPC peer stores + mailbox flags), device-resident counts",
                     "p2p": "p2p (CUDA IPC peer stores + mailbox flags)"}[xport]
        except PeerUnavailable as e:
            print(f"[bench] {e}; falling back to torch.distributed", file=sys.stderr)
            shard = make_shard()
            xport = "torch"
    if ex is None:
        staging = os.environ.get("SOLID_DIST_BACKEND", "nccl") != "nccl"
        ex = TorchExchange(shard, staging=staging)
        xname = "gloo, host-staged" if staging else "nccl all_to_all + batched p2p"
    coll = {"s": 0.0, "bytes": 0, "exchanges": 0}

    def timed_exchange(counts, flags=None):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ex.exchange(counts, flags=flags)
        coll["s"] += time.perf_counter() - t0
        return r

    def timed_exchange_dev(sync):
        t0 = time.perf_counter()
        r = ex.exchange_dev(sync)
        coll["s"] += time.perf_counter() - t0     # host time of the enqueue (+ wait if sync)
        return r

    def step():
        if xport == "native":
            res, tm = ex.admit_native(d["tokens"], d["offsets"], d["users"], None, lo)
            coll["s"] += tm.exchange_ms / 1e3      # device time in the exchange waits
            coll["bytes"] += tm.recv_records_remote * tm.record_bytes
            coll["exchanges"] += tm.exchanges
            return res, tm.rounds
        if xport == "p2p-dev":
            return run_protocol_device(shard, (d["tokens"], d["offsets"], d["users"], None, lo),
                                       timed_exchange_dev, ex.allreduce_max)
        res, t = run_protocol([shard], [(d["tokens"], d["offsets"], d["users"], None, lo)],
                              timed_exchange, ex.allreduce_max)
        return res[0], t

    for _ in range(max(args.warmup, 1)):
        shard.index.reset()
        step()
    torch.cuda.synchronize()
    cs = torch.cuda.current_stream(dev)
    ms, rounds, colls, cbytes = [], [], [], []
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            shard.index.reset()
            dist.barrier()
            coll["s"], coll["bytes"], coll["exchanges"] = 0.0, 0, 0
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cs)
            res, t = step()
            b.record(cs)
            b.synchronize()
            ms.append(a.elapsed_time(b))
            rounds.append(t)
            colls.append(coll["s"] * 1e3)
            cbytes.append(coll["bytes"])
        torch.cuda.synchronize()
        dist.barrier()
    clocks = clk.summary()
    tot = torch.tensor([sum(ms), sum(colls), sum(cbytes)], dtype=torch.float64, device=dev)
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    tot_ms, coll_ms = float(tot[0]), float(tot[1])
    xbytes = torch.tensor([sum(cbytes)], dtype=torch.float64, device=dev)
    dist.all_reduce(xbytes, op=dist.ReduceOp.SUM)
    value = per * world * args.steps / (tot_ms / 1e3)
    peak, peak_src = _peaks()
    alg = (64 * nblk + 37 * per) * world
    # parity of the timed configuration: rank 0's slice is the first `per` requests of the global
    # sequence, so its results depend on nothing else (R1) — the sequential oracle on that slice
    # alone must give them exactly; every rank's results must also equal a second transport's
    # (NCCL all-to-all-v through a second shard set) on the same batch
    parity = {"rank0_vs_oracle": None, "transport": None}
    mism = 0
    if rank == 0 and not args.no_cpu:
        from oracle import Oracle
        o = Oracle(16, SEED, 2)
        o.reserve(nblk // 8 + 1024)
        exp = o.process(s)
        got = P.as_numpy(res)
        mism = sum(int((got[f] != exp[f]).sum()) for f in exp.dtype.names)
        parity["rank0_vs_oracle"] = {"requests": per, "mismatches": mism}
    if xport != "torch" and os.environ.get("SOLID_DIST_BACKEND", "nccl") == "nccl" and \
            os.environ.get("SOLID_DIST_CHECK", "1") == "1":
        first = P.as_numpy(res).copy()
        shard2 = make_shard()
        ex2 = TorchExchange(shard2)
        r2, _ = ex2.admit(d["tokens"], d["offsets"], d["users"], None, lo)
        torch.cuda.synchronize()
        bad = torch.tensor([sum(int((P.as_numpy(r2)[f] != first[f]).sum())
                                for f in first.dtype.names)], dtype=torch.int64, device=dev)
        dist.all_reduce(bad, op=dist.ReduceOp.SUM)
        parity["transport"] = {"other": "nccl all_to_all + batched p2p (TorchExchange)",
                               "mismatches": int(bad.item())}
        del shard2, ex2
    parity["status"] = "exact" if (mism == 0 and (parity["transport"] is None or
                                                  parity["transport"]["mismatches"] == 0)) \
        else "MISMATCH"
    res_np = P.as_numpy(res)
    # e2e: the same sharded admission from pinned host buffers (H2D + admit + D2H per step)
    e2e = None
    if args.e2e_steps > 0:
        pin = lambda a: torch.from_numpy(a).pin_memory()
        ht, ho, hu = pin(s.tokens.view(np.int32)), pin(s.offsets.view(np.int64)), pin(s.users.view(np.int32))
        et = 0.0
        for _ in range(args.e2e_steps):
            shard.index.reset()
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dt, do, du = ht.to(dev, non_blocking=True), ho.to(dev, non_blocking=True), hu.to(dev, non_blocking=True)
            r = [ex.admit_native(dt, do, du, None, lo)[0] if xport == "native"
                 else ex.admit(dt, do, du, None, lo)[0]]
            r[0].cpu()
            et += time.perf_counter() - t0
        tt = torch.tensor([et], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": per * world * args.e2e_steps / float(tt.item()), "unit": "requests/s",
               "h2d_bytes_per_step": int(ht.numel() * 4 + ho.numel() * 8 + hu.numel() * 4),
               "d2h_bytes_per_step": int(res_np.nbytes)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "requests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic",
            "blocks_per_s": nblk * world * args.steps / (tot_ms / 1e3),
            "config": config_sharded(world, users, per),
            "exchange": xname,
            "roofline": {"bound": "hbm", "kernel": "whole sharded step (per GPU)",
                         "achieved": alg / world / (tot_ms / args.steps / 1e3) / 1e9,
                         "peak": peak, "unit": "GB/s",
                         "frac": alg / world / (tot_ms / args.steps / 1e3) / 1e9 / peak,
                         "traffic": None, "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": e2e,
            # begin 3 + REG 2 + ingest0 4 + PULL 2 + 15 per round (round 5, INT 2, ingest 6, PULL
            # 2; no PULL after the last) + commit 2 + three value exchanges (native) 6
            "gpu_launches": int(sum((17 if xport == "native" else 11) + 15 * r if xport != "torch"
                                    else 9 + 11 * r for r in rounds)),
            "collectives_ms_per_step": coll_ms / args.steps,
            "collectives": {"ms_per_step_max_rank": coll_ms / args.steps,
                            "what": ("device time inside the exchange waits (post -> every peer "
                                     "posted), from solid_dist_timing" if xport == "native" else
                                     "host time around the exchange calls"),
                            "remote_bytes_per_step_all_ranks": float(xbytes.item()) / args.steps,
                            "exchanges_per_step": coll["exchanges"]},
            "parity": parity,
            "resolver_rounds": rounds[-1],
            "clocks": clocks,
            "step_ms": ms,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=100_000)
    ap.add_argument("--ref-sample", type=int, default=20_000)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-activator", action="store_true")
    ap.add_argument("--no-evict", action="store_true")
    ap.add_argument("--no-policy-eval", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/cpu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2603_10726_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SOLID_DIST_BACKEND=gloo: ranks may share GPUs (records staged through host memory) — a
    # functional check of the N > 1 path on a one-GPU box; the measured runs use NCCL
    backend = os.environ.get("SOLID_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        return run_sharded(args, world, rank, local)

    stream_np, desc = _workload(args.config, rank)
    N = stream_np.n_requests
    nblk = stream_np.n_blocks()
    dev = torch.device("cuda", local)
    d = P.to_device(stream_np, dev)
    idx = P.Index("solidarity", capacity_blocks=max(nblk // 6, 1 << 20),   # C2: ~0.92 M new entries
                  max_batch_tokens=stream_np.n_tokens + 64, max_batch_requests=N,
                  seed=SEED, device=local)
    out = torch.empty((N, 6), dtype=torch.int32, device=dev)
    cs = torch.cuda.current_stream(dev)

    def step():
        # solid_admit_batch: lookup + commit + device-side capacity check, no host sync inside
        idx.admit_async(d["tokens"], d["offsets"], d["users"], d["enforce"], out=out)

    # warm-up
    for _ in range(args.warmup):
        idx.reset()
        step()
        idx.status()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    phase = {"hash": [], "resolve": [], "commit": [], "hash_kernel": [], "round1": [],
             "shared_keys": []}
    rounds, launches = [], []
    stats = None
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        def collect():
            idx.status()                # the oldest batch's status (raises on error)
            st = idx.stats()
            for key, f in [("hash", "ms_hash"), ("resolve", "ms_resolve"),
                           ("commit", "ms_commit"), ("hash_kernel", "ms_hash_kernel"),
                           ("round1", "ms_round_first"), ("shared_keys", "last_shared_keys")]:
                phase[key].append(st[f])
            rounds.append(st["last_rounds"])
            launches.append(st["last_kernel_launches"])
            return st

        # pipelined like a server: step k+1 is enqueued before step k's status is collected,
        # so the host never stalls the device; the restore of the empty pre-batch index is
        # stream-ordered between the events of consecutive steps (outside the timed regions)
        for k in range(args.steps):
            idx.reset()
            ev[k][0].record(cs)
            step()
            ev[k][1].record(cs)
            if k:
                stats = collect()
        stats = collect()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    clocks = clk.summary()
    ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(ms)
    t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms = float(t.item())
    reqs_all = N * world
    value = reqs_all * args.steps / (tot_ms / 1000.0)

    # the last timed step's results and index, checked against the oracle below (cpu_baseline
    # runs the oracle on the same stream)
    res = P.as_numpy(out)
    timed_dump = idx.dump()

    # roofline.  The kernel that moves the algorithmic bytes is k_hash_register (every token is
    # read there); the resolver rounds (k_eval) take the larger share of the step but carry no
    # algorithmic bytes of their own, so both are reported.
    peak, peak_src = _peaks()
    alg_bytes = stats["algorithmic_bytes"]
    hash_ms = statistics.median(phase["hash_kernel"])
    # SURVEY §8(d) bytes of K_A per launch: the tokens of every full block (64 B), offsets + user
    # per request (12 B), and one 16-byte index slot per distinct key it probes (the snapshot of
    # every Shared key of the batch); the 4 B/block id scratch is implementation, not counted
    probes = statistics.median(phase["shared_keys"])
    hash_bytes = 64 * nblk + 12 * N + 16 * probes
    step_ms = tot_ms / args.steps
    roof_step = alg_bytes / (step_ms / 1e3) / 1e9
    traffic, l2hit, res_inst = None, None, None
    try:
        with open(os.path.join(ROOT, "profiles", "latest_ncu.json")) as f:
            prof = json.load(f)
        traffic = prof["kernels"]["k_hash_register"][-1]["traffic"]
        l2hit = prof["kernels"]["k_hash_register"][-1].get("l2_hit_pct")
        res_inst = prof["kernels"]["k_resolve"][-1].get("warp_instructions")
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": "k_hash_register (hash + scan + probe/register)",
                "whole_step_frac": roof_step / peak,
                "achieved": hash_bytes / (hash_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": hash_bytes / (hash_ms / 1e3) / 1e9 / peak, "traffic": traffic,
                "traffic_source": "profiles/latest_ncu.json (ncu dram__bytes_read+write, same cmd)",
                "l2_hit_pct": l2hit,
                "algorithmic_bytes_per_launch": hash_bytes, "launch_ms": hash_ms,
                "bytes_formula": "64 B x full blocks + 12 B x requests + 16 B x distinct keys "
                                 "probed in the index (SURVEY 8(d))",
                "snapshot_probes": probes,
                "share_of_step": hash_ms / step_ms, "peak_source": peak_src,
                "whole_step": {"achieved": roof_step, "frac": roof_step / peak,
                               "algorithmic_bytes": alg_bytes,
                               "resolver_share": statistics.median(phase["resolve"]) / step_ms}}

    # the resolver (the largest share of the step, no algorithmic bytes) is bound by instruction
    # issue: its warp instructions per launch (ncu, same batch) over its measured time, against
    # 148 SMs x 4 schedulers x one warp instruction per clock at the sampled SM clock
    resolver_roofline = None
    if res_inst:
        res_ms = statistics.median(phase["resolve"])
        clk = (clocks or {}).get("sm_mhz") or 1965.0
        peak_issue = 148 * 4 * clk * 1e6
        resolver_roofline = {"bound": "issue", "kernel": "k_resolve (all rounds, one launch)",
                             "achieved": res_inst / (res_ms / 1e3) / 1e12, "peak": peak_issue / 1e12,
                             "unit": "T warp instr/s", "frac": res_inst / (res_ms / 1e3) / peak_issue,
                             "warp_instructions_per_launch": res_inst,
                             "source": "profiles/latest_ncu.json (smsp__inst_executed.sum)"}

    # e2e: same metric through the C ABI with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not args.profile and args.e2e_steps > 0:
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
        ht, ho, hu = pin(stream_np.tokens), pin(stream_np.offsets), pin(stream_np.users)
        hout = (torch.zeros(N * P.RESULT_DTYPE.itemsize, dtype=torch.uint8).pin_memory().numpy()
                .view(P.RESULT_DTYPE))                   # pinned: the result copy is a DMA
        idx.reset()
        idx.admit_host(ht, ho, hu, None, out=hout)
        e2e_t = 0.0
        for _ in range(args.e2e_steps):
            idx.reset()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            idx.admit_host(ht, ho, hu, None, out=hout)
            e2e_t += time.perf_counter() - t0
        tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": reqs_all * args.e2e_steps / float(tt.item()), "unit": "requests/s",
               "h2d_bytes_per_step": int(ht.nbytes + ho.nbytes + hu.nbytes),
               "d2h_bytes_per_step": int(hout.nbytes),
               "how": "solid_admit_host: pinned host buffers -> H2D -> lookup -> insert -> D2H, "
                      "host wall clock (perf_counter) around the call"}
        assert (hout["reused"] == res["reused"]).all()
        # the same with 16-bit token ids (vocabulary 32 000 < 2^16): half the H2D bytes, widened
        # on the device (solid_admit_host_u16); this is the headline e2e, the u32 one is kept
        if int(stream_np.tokens.max()) < 65536:
            h16 = pin(stream_np.tokens.astype(np.uint16))
            idx.reset()
            idx.admit_host_u16(h16, ho, hu, None, out=hout)
            e16 = 0.0
            for _ in range(args.e2e_steps):
                idx.reset()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                idx.admit_host_u16(h16, ho, hu, None, out=hout)
                e16 += time.perf_counter() - t0
            tt = torch.tensor([e16], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            assert (hout["reused"] == res["reused"]).all()
            e2e_u32 = e2e
            # the bound: the same bytes as one plain pinned host->device copy (PCIe)
            hb = int(h16.nbytes + ho.nbytes + hu.nbytes)
            src = torch.from_numpy(h16.view(np.uint8)).pin_memory()
            dst = torch.empty(src.numel(), dtype=torch.uint8, device=dev)
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            cps = []
            for _ in range(3):
                t0 = time.perf_counter()
                dst.copy_(src, non_blocking=True)
                torch.cuda.synchronize()
                cps.append(time.perf_counter() - t0)
            copy_gbps = src.numel() / min(cps) / 1e9
            del src, dst
            e2e_s = float(tt.item()) / args.e2e_steps
            e2e = {"value": reqs_all * args.e2e_steps / float(tt.item()), "unit": "requests/s",
                   "h2d_bytes_per_step": hb,
                   "d2h_bytes_per_step": int(hout.nbytes), "token_bits": 16,
                   "how": "solid_admit_host_u16: pinned host buffers (16-bit token ids) -> H2D -> "
                          "widen on the device -> lookup -> insert -> D2H, host wall clock",
                   "bound": {"what": "PCIe host->device copy of the step's inputs",
                             "h2d_gbps_achieved": hb / e2e_s / 1e9,
                             "h2d_gbps_plain_copy": copy_gbps,
                             "frac": (hb / copy_gbps / 1e9) / e2e_s},
                   "u32_tokens": e2e_u32}

    activator = None
    if rank == 0 and world == 1 and not args.profile and not args.no_activator:
        activator = measure_activator(dev, args)

    hash2 = None
    if rank == 0 and world == 1 and not args.profile:
        hash2 = measure_hash2(dev, args, d, stream_np)

    btab = None
    if rank == 0 and world == 1 and not args.profile:
        btab = measure_block_table(dev, args, d, stream_np)

    lru = None
    if rank == 0 and world == 1 and not args.profile and not args.no_evict:
        lru = measure_evict(dev, args)

    other = None
    if rank == 0 and world == 1 and not args.profile and not args.no_configs:
        other = measure_configs(dev, args)
        if not args.no_c5:
            try:
                other["c5"] = measure_c5(dev, args)
            except Exception as e:   # reported, never silently dropped
                other["c5"] = {"error": f"{type(e).__name__}: {e}"}

    peval = None
    if rank == 0 and world == 1 and not args.profile and not args.no_policy_eval:
        peval = measure_policy_eval(dev, args)

    cpu, parity = None, {"status": "not checked (--no-cpu)"}
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        cpu, exp_res, exp_dump = cpu_baseline(stream_np, args.cpu_sample)
        if len(exp_res) == N:
            parity = parity_of_timed_step(res, timed_dump, exp_res, exp_dump)
        else:
            parity = {"status": f"not checked (oracle sample {len(exp_res)} < {N} requests)"}

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "requests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic",
            "blocks_per_s": nblk * world * args.steps / (tot_ms / 1000.0),
            "config": config_n1(desc, N, nblk, stream_np.n_tokens),
            "roofline": roofline,
            "resolver_roofline": resolver_roofline,
            "cpu_baseline": cpu,
            "parity": parity,
            "activator": activator,
            "lru_eviction": lru,
            "hash_components_2": hash2,
            "block_table": btab,
            "policy_eval": peval,
            "other_configs": other,
            "e2e": e2e,
            "gpu_launches": int(sum(launches)),
            "clocks": clocks,
            "phases_ms_median": {k: statistics.median(v) for k, v in phase.items() if v},
            "resolver_rounds": rounds[-1] if rounds else None,
            "resolver_round_us": [round(x, 1) for x in stats["round_us"]],
            "step_ms": ms,
            "result_summary": {"reused_blocks": int(res["reused"].sum()),
                               "diverted": int(((res["bits"] & 4) > 0).sum()),
                               "flagged": int(((res["bits"] & 16) > 0).sum()),
                               "entries": int(stats["live_entries"])},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
