/*
 * solid.h — C ABI of the B200-native CacheSolidarity hot path.
 *
 * One context = one GPU-resident prefix index (open addressing, 16-byte slots {key, owner,
 * sharer}) plus per-batch scratch.  A batch of requests is admitted with solid_lookup_batch
 * (hash -> chained keys -> longest cached prefix -> Detector decision)
 * followed by solid_insert_batch (new entries tagged with the requester, and
 * AttackFlag/sharer writes).  The pair equals admitting the batch's requests one at a time
 * in sequence order (R1): results never depend on how a stream is cut into batches.
 *
 * Conventions
 *   - All functions return solid_status.  Invalid arguments -> SOLID_ERR_INVALID with no side
 *     effect on the index.  Capacity overflow -> SOLID_ERR_CAPACITY with no mutation (R9).
 *     A CUDA failure -> SOLID_ERR_CUDA and the context is poisoned (later calls return
 *     SOLID_ERR_STATE).  solid_last_error() returns a message for the last failure.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Work is
 *     enqueued on it.  solid_lookup_batch is asynchronous (the resolver loops on the device,
 *     DESIGN.md §4.4); solid_insert_batch synchronises `stream` once (capacity check, status).
 *     Batch errors detected on the device (token >= 2^20, user == NONE, bad offsets, request >
 *     max_blocks) are therefore returned by solid_insert_batch, and nothing is committed.
 *   - Device pointers are caller-owned and must stay valid until solid_insert_batch returns.
 *   - A context is single-writer (SPEC S:148 single stream); distinct contexts are independent.
 */
#ifndef SOLID_H
#define SOLID_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SOLID_ABI_VERSION 7u
#define SOLID_USER_NONE 0xFFFFFFFFu   /* "no user": sharer of an unflagged entry */

typedef enum {
  SOLID_OK = 0,
  SOLID_ERR_INVALID = 1,   /* bad argument / batch (token >= 2^20, user == NONE, offsets ...)  */
  SOLID_ERR_CAPACITY = 2,  /* index or scratch would overflow; nothing was mutated             */
  SOLID_ERR_STATE = 3,     /* call order violated, or context poisoned by an earlier failure  */
  SOLID_ERR_CUDA = 4,      /* CUDA runtime error (context poisoned)                           */
  SOLID_ERR_NCCL = 5,      /* sharded index: the record transport failed (a peer did not post
                              its exchange within 60 s, or a collective failed); nothing of
                              the batch was committed on this shard                        */
  SOLID_ERR_OOM = 6        /* device allocation failed in solid_init                          */
} solid_status;

typedef enum {
  SOLID_POLICY_APC = 0,            /* Prefix Caching baseline: full reuse, no flags    */
  SOLID_POLICY_USER_ISOLATION = 1, /* User Cache Isolation baseline (reading R4)   */
  SOLID_POLICY_SOLIDARITY = 2      /* CacheSolidarity: Detector + selective isolation */
} solid_policy;

typedef struct {
  uint32_t block_size;         /* tokens per cache entry; must be 16 (reading R13)       */
  uint32_t max_blocks;         /* max full blocks per request (power tables); e.g. 8192          */
  uint64_t capacity_blocks;    /* max live entries in the index (no eviction, R9)               */
  uint64_t max_batch_tokens;   /* scratch sizing: max tokens per batch                           */
  uint64_t max_batch_requests; /* scratch sizing: max requests per batch                         */
  uint64_t hash_seed;          /* H-def v2 seed; secret per deployment          */
  int32_t policy;              /* solid_policy                                                   */
  int32_t device;              /* CUDA device ordinal                                            */
  uint32_t world;              /* shards of the key-hash-partitioned index (1 = single GPU)      */
  uint32_t rank;               /* this context's shard, < world                                  */
  uint32_t evict;              /* 0: a batch that would exceed capacity_blocks fails with
                                  SOLID_ERR_CAPACITY (R9).  1: LRU eviction (SPEC evict_lru
                                  S:117-125): after each request's inserts, while
                                  more than capacity_blocks entries are live, the entry with the
                                  smallest (last_used, key) is removed — last_used = the global
                                  sequence number of the last request served it or inserted it
                                  (R22-R25).  Single GPU only (world == 1); capacity_blocks >=
                                  max_blocks.                                                     */
  uint32_t hash_components;    /* 0 or 1: H-def v2 keys (one 61-bit polynomial chain).  2: H-def
                                  v3: a second independent chain (base
                                  B2) mixed into every key — the chain collision bound drops from
                                  ~L/2^61 to ~L^2/2^122 per pair (L = tokens), below the 64-bit
                                  key's 2^-64.  Decisions are unchanged (absent collisions); keys
                                  differ.  Also with the sharded index (world > 1).              */
  uint32_t block_table;        /* 1: physical KV blocks and per-request block tables (SURVEY f4,
                                  P:733 "vLLM" block manager, R26-R28).  A pool of
                                  capacity_blocks physical block ids; a FIFO of free ids (initially
                                  0..capacity_blocks-1); per request, its evictions return their
                                  blocks first, then its new entries take blocks in block order.
                                  See solid_block_table / solid_dump_phys.  Single GPU only;
                                  solid_admit_batch admits at submission (see there).            */
  uint32_t pin;                /* 1 (needs block_table = 1): in-flight pinning (R38; the
                                  reference count of vLLM's KVCacheBlock beneath P:733).  Every
                                  admitted request holds one pin on each entry of its block-table
                                  row until the caller releases that row (solid_release); a pinned
                                  entry is never evicted — the LRU victim is the smallest
                                  (last_used, key) among unpinned entries — so its physical block
                                  is never reclaimed while a running request reads it.  A batch
                                  one of whose requests would need more victims than there are
                                  unpinned entries it does not use itself fails with
                                  SOLID_ERR_CAPACITY, nothing mutated (split it: a single such
                                  request is refused until pins are released).                   */
} solid_config;

typedef struct solid_ctx solid_ctx;

/* One batch in global sequence order (CSR).  Pointers are DEVICE memory for
 * solid_lookup_batch and HOST memory for solid_admit_host. */
typedef struct {
  uint64_t n_requests;
  const uint32_t* tokens;   /* concatenated token ids, each < 2^20 (R15); 4-byte aligned.
                               Loads may touch up to 12 bytes past a request's last full block
                               within the same 16-byte granule.                                  */
  const uint64_t* offsets;  /* n_requests+1, offsets[0] == 0, non-decreasing; request j =
                               tokens[offsets[j], offsets[j+1]); its floor(len/16) full blocks are
                               hashed, the tail is never cached                  */
  const uint32_t* users;    /* requester ids, != SOLID_USER_NONE                                */
  const uint8_t* enforce;   /* per-request isolation-active bit (Activator output); NULL
                               = all 1.  enforce=0 still updates metadata (R11)   */
} solid_batch;

/* Per-request result, 24 bytes. */
typedef struct {
  uint32_t n_blocks;     /* floor(len / 16)                                                    */
  uint32_t shared_hits;  /* k: Shared hit-chain length (USER_ISOLATION: 0)                    */
  uint32_t reused;       /* r: blocks whose cached content is served                          */
  int32_t divert_at;     /* f: depth where reuse left the Shared chain, -1 none (USER_ISO: 0) */
  uint32_t flag_depth;   /* depth of the entry this request flagged, 0 = none                 */
  uint32_t bits;         /* HIT=1 (r>0) FULL=2 (n>0,r==n) DIVERTED=4 TRUNCATED=8 (f<k) FLAGGED=16 */
} solid_result;

enum { SOLID_HIT = 1, SOLID_FULL = 2, SOLID_DIVERTED = 4, SOLID_TRUNCATED = 8, SOLID_FLAGGED = 16 };

typedef struct {
  uint64_t key;      /* block key (H-def v2)                                                  */
  uint32_t owner;    /* OwnerID: set once at allocation                              */
  uint32_t sharer;   /* user that flagged it; AttackFlag <=> sharer != SOLID_USER_NONE (R5)  */
} solid_entry;

typedef struct {         /* solid_dump_ex (evict mode)                                        */
  uint64_t key;
  uint32_t owner;
  uint32_t sharer;
  uint64_t last_used;    /* LRU clock: global sequence number of the last request served it or
                            that inserted it (R22)                                               */
} solid_entry_ex;

typedef struct {
  /* cumulative over all committed batches */
  uint64_t batches, requests, blocks, reused_blocks, inserted, flagged, diverted, truncated;
  uint64_t live_entries;
  /* last batch */
  uint32_t last_rounds;          /* resolver rounds until the sequential fixed point         */
  uint32_t last_distinct_keys;   /* scratch keys registered (Shared + isolated) last batch   */
  uint64_t last_requests, last_blocks, last_inserted, last_flagged;
  float ms_hash, ms_resolve, ms_commit;    /* device time per phase of the last batch       */
  uint64_t algorithmic_bytes;    /* DESIGN.md §5 formula for the last batch                  */
  uint64_t last_kernel_launches; /* kernels this library launched for the last batch         */
  float ms_hash_kernel;          /* device time of k_hash_register alone (last batch)        */
  float ms_round_first;          /* device time of the resolver kernel (last batch)          */
  float round_us[8];             /* device time of resolver rounds 1..8 (globaltimer)        */
  /* evict mode */
  uint64_t evicted;              /* entries evicted, cumulative                              */
  uint64_t last_evicted;         /* entries evicted by the last batch                        */
  uint32_t last_evict_iters;     /* resolver / eviction-time iterations of the last batch    */
  uint32_t last_window_keys;     /* batch keys in the eviction window (last batch)           */
  uint64_t window_evicted;       /* cumulative: batch keys evicted by their own batch        */
  uint32_t max_evict_iters;      /* max resolver / eviction-time iterations of any batch     */
  uint32_t rebuilds;             /* index rebuilds (tombstone clean-up), cumulative          */
  uint32_t compactions;          /* LRU log compactions, cumulative                          */
  uint32_t last_shared_keys;     /* distinct keys registered (and probed in the index) by the
                                    hash kernel K_A, last batch: its snapshot probes (§8(d))  */
} solid_stats_t;

uint32_t solid_abi_version(void);

/* Allocate the index (2^ceil(log2(2*capacity)) slots) and scratch on cfg->device. */
solid_status solid_init(const solid_config* cfg, solid_ctx** out);
solid_status solid_destroy(solid_ctx* ctx);

/* Lookup + Detector for one batch (device pointers).  Writes out[n_requests] (DEVICE memory)
 * and stages every mutation (new entries, new flags); the persistent index is only read.
 * Request i of the batch has global sequence position (earlier batches) + i.
 * Must be followed by solid_insert_batch before the next lookup (else SOLID_ERR_STATE). */
solid_status solid_lookup_batch(solid_ctx* ctx, const solid_batch* batch, solid_result* out,
                                void* stream);

/* Commit the staged admissions of the last lookup: 128-bit CAS claims {key, owner, sharer}
 * for new entries and sharer writes on flagged existing entries.  Checks capacity first: the
 * batch's new entries are counted on the device (k_stats) before any claim, and a batch with
 * live + new > capacity_blocks claims nothing and fails with SOLID_ERR_CAPACITY.
 * Evict mode: also removes the batch's LRU victims (tombstones) and appends the LRU records of
 * every entry the batch touched; a batch that would have to evict an entry it touched itself
 * (it inserts more entries than the index holds untouched ones) fails with SOLID_ERR_CAPACITY
 * and nothing is mutated — split it.  In evict mode solid_lookup_batch synchronises `stream`
 * (the joint resolver / eviction-time iteration runs on the device in chunks of iterations; the
 * host waits once per chunk to decide whether another chunk is needed). */
solid_status solid_insert_batch(solid_ctx* ctx, void* stream);

/* Asynchronous admission (lookup + insert with no host synchronisation), for a pipelined caller.
 * The capacity check (R9) runs on the device before any claim (an over-capacity batch claims
 * nothing), so every batch is still all-or-nothing and batches apply in submission order; a failed batch
 * leaves the index exactly as before it, and later batches see that state.  Up to
 * SOLID_MAX_INFLIGHT batches may be outstanding; each must be collected, oldest first, by
 * solid_batch_status, which waits for it and returns ITS status (SOLID_OK, SOLID_ERR_INVALID,
 * SOLID_ERR_CAPACITY, SOLID_ERR_STATE) and folds it into solid_stats.  With none outstanding
 * solid_batch_status returns SOLID_OK.  solid_admit_batch itself fails with SOLID_ERR_STATE when
 * SOLID_MAX_INFLIGHT batches are outstanding or a solid_lookup_batch is pending;
 * solid_lookup_batch, solid_dump, solid_checkpoint and solid_restore fail with SOLID_ERR_STATE
 * while any is outstanding.  solid_reset may be called with batches outstanding: it is then
 * enqueued behind them on their stream without blocking, and the older batches, when
 * collected, report their status but no longer count in solid_stats.  `out` is written when
 * the stream reaches the batch (read it after solid_batch_status or a stream synchronisation).
 * Evict-mode and block_table contexts: the same calls and rules, but the batch is admitted
 * during solid_admit_batch (their lookup waits on the host and their commit reads counts back),
 * so it returns when the batch is committed (or failed) and `out` is final; its status waits
 * for solid_batch_status like an asynchronous batch's. */
#define SOLID_MAX_INFLIGHT 4
solid_status solid_admit_batch(solid_ctx* ctx, const solid_batch* batch, solid_result* out,
                               void* stream);
solid_status solid_batch_status(solid_ctx* ctx);

/* lookup + insert with HOST buffers: copies the batch to the device, admits it, copies the
 * results back to out_host (HOST memory; page-locked memory makes that copy a DMA) and
 * synchronises `stream`.  Large batches are copied in 4 pieces (the last one half the size of
 * the others) on a second stream, each hashed as soon as it has arrived; the commit and the
 * result copy share one host wait.  On failure the index is untouched and out_host is
 * unspecified. */
solid_status solid_admit_host(solid_ctx* ctx, const solid_batch* host_batch,
                              solid_result* out_host, void* stream);

/* The same with 16-bit token ids (vocabularies up to 65 536 — Llama-2's 32 000, the paper's
 * models): half the host->device bytes; the ids are widened on the device (k_widen16) before
 * the admission.  Offsets, users and enforce as in solid_batch (HOST memory). */
typedef struct {
  uint64_t n_requests;
  const uint16_t* tokens;
  const uint64_t* offsets;
  const uint32_t* users;
  const uint8_t* enforce;
} solid_batch_u16;
solid_status solid_admit_host_u16(solid_ctx* ctx, const solid_batch_u16* host_batch,
                                  solid_result* out_host, void* stream);

solid_status solid_stats(solid_ctx* ctx, solid_stats_t* out);

/* Test hook: set the batch-scratch epoch (tags restart, with a scratch re-initialisation, after
 * ~2^20 batches; tests jump close to the limit).  SOLID_ERR_STATE with a batch in flight. */
solid_status solid_debug_set_epoch(solid_ctx* ctx, uint32_t epoch);

/* Test hook: the resolver's round limit (2..4093, default 4093).  Requests
 * before round t are final after round t, so a batch of <= limit - 1 requests always converges.
 * A batch that does not converge is committed in consecutive parts (halves, recursively; the
 * results equal one admission by R1) by solid_insert_batch / solid_admit_host; through
 * solid_admit_batch it fails with SOLID_ERR_STATE and commits nothing (later batches in flight
 * see the index without it), and the caller resubmits it in parts.  Block tables / block keys
 * are not produced for a batch committed in parts (SOLID_ERR_STATE), and a block_table context
 * does not split (SOLID_ERR_STATE).  SOLID_ERR_STATE with a batch in flight. */
solid_status solid_debug_set_max_rounds(solid_ctx* ctx, uint32_t rounds);

/* Block table of the last admitted batch (paged-KV integration; call after
 * solid_insert_batch, or after solid_batch_status collected the last solid_admit_batch, and
 * before the next lookup): for request j and its block b < n_j,
 *   keys_out[offsets[j] / 16 + b] = the key of the index entry that holds that block's KV —
 * the Shared key K[b] when the request stayed in the Shared namespace (served or inserted), the
 * requester's isolated key I_f[b] for b >= f when it was diverted at f (R3), U[b] under
 * USER_ISOLATION.  A paged-KV manager maps these keys to physical blocks.  keys_out: DEVICE
 * memory, ceil(total tokens / 16) entries; positions no request's full block covers are not
 * written.  Enqueued on `stream`.  Single-GPU contexts only. */
solid_status solid_block_keys(solid_ctx* ctx, unsigned long long* keys_out, void* stream);

/* Block table of the last committed batch (block_table = 1, R27): DEVICE array
 * indexed like solid_block_keys (offsets[j]/16 + b); entry = the physical block id of the entry
 * holding request j's block b as the request used it (Shared before the divert point, isolated
 * from it), SOLID_USER_NONE if that entry did not survive the request (evict mode: an entry the
 * request referenced without being served it and then evicted).  Positions no request's full
 * block covers are not written.  The batch's offsets must still be valid.  Enqueued on stream. */
solid_status solid_block_table(solid_ctx* ctx, uint32_t* table_out, void* stream);

/* Release one pin on the entry holding each of the n physical block ids in phys (DEVICE array,
 * e.g. a finished request's block-table row; SOLID_USER_NONE entries are skipped).  pin = 1
 * contexts only.  Synchronises `stream`; SOLID_ERR_INVALID if some block holds no pinned entry
 * (those are left unchanged, the others released). */
solid_status solid_release(solid_ctx* ctx, const uint32_t* phys, uint64_t n, void* stream);

/* Pin count of every physical block (HOST array of capacity_blocks entries; 0 for free blocks).
 * pin = 1 contexts only. */
solid_status solid_pins(solid_ctx* ctx, uint32_t* pins_out);

/* Live entries' physical blocks sorted by key (HOST arrays, capacity cap); *n_out = live
 * entries.  block_table = 1 contexts only. */
solid_status solid_dump_phys(solid_ctx* ctx, uint64_t* keys_out, uint32_t* phys_out, uint64_t cap,
                             uint64_t* n_out);

/* Copy live entries to host_out (HOST memory, capacity `cap` entries) sorted by key; *n_out =
 * number of live entries (may exceed cap; then only cap are written). */
solid_status solid_dump(solid_ctx* ctx, solid_entry* host_out, uint64_t cap, uint64_t* n_out);

/* Evict mode: live entries with their LRU clock, sorted by key (as solid_dump).  Fails with
 * SOLID_ERR_STATE on a context created with evict = 0. */
solid_status solid_dump_ex(solid_ctx* ctx, solid_entry_ex* host_out, uint64_t cap, uint64_t* n_out);

/* Empty the index (keeps allocations).  Synchronous, unless asynchronous batches are outstanding
 * (then ordered behind them on their stream, see solid_admit_batch). */
solid_status solid_reset(solid_ctx* ctx);

/* Save / restore the index contents into / from a ctx-owned device buffer (warm-state reuse). */
solid_status solid_checkpoint(solid_ctx* ctx);
solid_status solid_restore(solid_ctx* ctx);

/* ---- Activator -------------------------------------------
 * per request, selective isolation is enforced iff the hit and miss TTFT distributions
 * of the most recent sliding window are distinguishable, i.e. their KDE overlap (the integral of
 * the minimum of the two densities, P:§2.2) is below theta.  Estimator per SPEC S:245-268:
 * per-token TTFT = ttft_ms / prompt_tokens; Hit if reuse_fraction >= hit_hi, Miss if <= hit_lo,
 * else excluded; each class keeps its window_len most recent values; Gaussian kernels with
 * Silverman bandwidth 0.9 min(sd, IQR/1.34) n^-1/5 (sd with ddof 1, linear-interpolation
 * quartiles, floor 1e-9); trapezoid on `grid` uniform points over [min - 3 h_max, max + 3 h_max];
 * clamp to [0, 1]; fewer than max(min_samples, 2) values in either class -> enforce (fail-safe).
 * All arithmetic fp64.  Its enforce[] output is solid_batch.enforce. */
typedef struct {
  double theta;            /* overlap threshold in [0, 1]                                  */
  double hit_hi;           /* reuse fraction >= hit_hi -> Hit sample                       */
  double hit_lo;           /* reuse fraction <= hit_lo -> Miss sample (hit_lo < hit_hi)    */
  uint32_t window_len;     /* samples kept per class, 2..4096                              */
  uint32_t min_samples;    /* per class, below it the decision is "enforce"                */
  uint32_t grid;           /* trapezoid points, 2..8192 (SPEC: 512)                        */
  int32_t device;          /* CUDA device ordinal                                          */
  uint64_t max_samples;    /* capacity of one call's sample stream (< 2^32)                */
  uint64_t max_queries;    /* capacity of one call's query list                            */
} solid_activator_config;

typedef struct solid_activator solid_activator;

solid_status solid_activator_init(const solid_activator_config* cfg, solid_activator** out);
solid_status solid_activator_destroy(solid_activator* act);

/* Device pointers.  ttft_ms[n_samples] (> 0, finite), prompt_tokens[n_samples] (>= 1),
 * reuse_fraction[n_samples]: the completed requests in completion order.  cuts[n_queries]:
 * for query j (a request being admitted, sequence order) the number of samples recorded before
 * it — non-decreasing, <= n_samples.  Writes overlap_out[j] (NaN when fail-safe) and
 * enforce_out[j] (1 = isolation enforced).  Synchronises `stream` once; invalid samples or cuts
 * -> SOLID_ERR_INVALID (outputs undefined). */
solid_status solid_activator_run(solid_activator* act, const double* ttft_ms,
                                 const uint32_t* prompt_tokens, const double* reuse_fraction,
                                 uint64_t n_samples, const uint64_t* cuts, uint64_t n_queries,
                                 double* overlap_out, uint8_t* enforce_out, void* stream);
const char* solid_activator_last_error(const solid_activator* act);

const char* solid_last_error(const solid_ctx* ctx);

/* ---------------------------------------------------------------------------------------------
 * Sharded index.  world > 1: each context owns the keys with
 * owner(key) = ((key >> 32) * world) >> 32 == rank, and admits its own contiguous slice of the
 * global batch (requests seq_base .. seq_base + n - 1 in global sequence order; slices ordered
 * by rank).  The caller moves the exchange records between the contexts — all-to-all-v over
 * NCCL (torch.distributed) across GPUs, or a loopback in one process — in this order:
 *
 *   solid_dist_begin                       (hash, local registration; packs REG records)
 *   exchange REG -> solid_dist_owner_ingest(phase 0)     (owner registration; packs PULL)
 *   for t = 1, 2, ...:
 *     exchange PULL -> solid_dist_round(t)   (mirror, Detector round; packs INT records)
 *     exchange INT  -> solid_dist_owner_ingest(phase t)  (reduce intents; packs PULL)
 *     changed = max over ranks of solid_dist_round's flag; stop when t >= 2 and !changed
 *                (APC / USER_ISOLATION: stop after t = 1)
 *   solid_dist_commit(mode 1); if any rank reports overflow: solid_dist_commit(mode 2)
 *     (mode 1 counts the shard's new entries first and claims nothing when they would exceed
 *     capacity_blocks, returning SOLID_ERR_CAPACITY; mode 2 then rolls back the shards that
 *     did commit and is a no-op on the others)
 *
 * Records are 24 bytes.  Send region for peer d starts at record d * cap_records of the send
 * buffer; receive region for peer s at record s * cap_records of the receive buffer.  Counts
 * are in records; solid_dist_counts returns the counts of the last pack (per peer).
 * --------------------------------------------------------------------------------------------- */
solid_status solid_dist_buffers(solid_ctx* ctx, void** send_dev, void** recv_dev,
                                uint64_t* cap_records);
solid_status solid_dist_counts(solid_ctx* ctx, uint64_t* counts_host /* [world] */);
solid_status solid_dist_begin(solid_ctx* ctx, const solid_batch* local, solid_result* out,
                              uint64_t seq_base, void* stream);
solid_status solid_dist_owner_ingest(solid_ctx* ctx, uint32_t phase,
                                     const uint64_t* recv_counts_host, void* stream);
solid_status solid_dist_round(solid_ctx* ctx, uint32_t t, const uint64_t* recv_counts_host,
                              uint32_t* changed, void* stream);
solid_status solid_dist_commit(solid_ctx* ctx, int mode, uint64_t* new_entries, void* stream);

/* ---- Peer-memory exchange for the sharded index ---------------------------
 * Replaces the caller-driven all-to-all-v: each rank exports a ctx-owned device region (mailbox +
 * two receive buffers) as a CUDA IPC handle, every rank maps every peer's region, and one
 * solid_dist_p2p_exchange moves the last pack's records straight into the peers' receive
 * buffers (NVLink / NVSwitch peer stores) and signals them through the mailbox — one push and
 * one wait kernel, no collective library.  All ranks must be processes on one node. */
/* 64-byte cudaIpcMemHandle_t of this shard's region into handle_out (allocated on first call). */
solid_status solid_dist_p2p_export(solid_ctx* ctx, void* handle_out);
/* Map the peers' regions; handles = world x 64 bytes in rank order (own entry ignored).  Every
 * rank must have exported first (the caller all-gathers the handles). */
solid_status solid_dist_p2p_connect(solid_ctx* ctx, const void* handles);
/* Exchange the last pack (the counts of solid_dist_counts): recv_counts_out[world] = records
 * received from each source, ready for the next solid_dist_owner_ingest / solid_dist_round;
 * flag = this rank's "decision changed" bit, *gflag_out (may be NULL) = max over all ranks.
 * Every rank must call it the same number of times.  Synchronises `stream`. */
solid_status solid_dist_p2p_exchange(solid_ctx* ctx, uint32_t flag, uint64_t* recv_counts_out,
                                     uint32_t* gflag_out, void* stream);
/* Device-counts mode (on = 1; between batches, after connect): solid_dist_owner_ingest and
 * solid_dist_round then accept recv_counts = NULL and no longer synchronise (their send counts
 * and errors stay on the device); solid_dist_p2p_exchange_dev moves the last pack reading its
 * counts — and, after a round, that round's changed flag — on the device, and writes the
 * received counts straight into the next call's input.  sync = 1: wait for the stream, return
 * the global changed flag in *gflag_out and report a batch error (use it for each round's INT
 * exchange); sync = 0: fully asynchronous (REG / PULL).  solid_dist_commit checks errors. */
solid_status solid_dist_p2p_device_counts(solid_ctx* ctx, uint32_t on);
solid_status solid_dist_p2p_exchange_dev(solid_ctx* ctx, uint32_t sync, uint32_t* gflag_out,
                                         void* stream);

/* ---- The sharded admission as one call -------------
 * Runs the whole protocol above inside the library over the peer-memory exchange: every rank
 * calls it once per batch with its own slice (after solid_dist_p2p_export / _connect on every
 * rank; the caller only all-gathers the 64-byte handles once).  Steps:
 *   1. agreement: every rank posts (seq_base, n) and a "slice rejected" bit (null pointers,
 *      n > max_batch_requests, misaligned tokens, sequence beyond 32 bits); slices must be
 *      contiguous in rank order (seq_base[r] = seq_base[r-1] + n[r-1]).  Every rank sees the
 *      same values, so every rank returns the same verdict: SOLID_ERR_INVALID (the rejecting
 *      rank, or all ranks for non-contiguous slices) / SOLID_ERR_STATE (the other ranks);
 *   2. begin -> REG -> owner registration -> PULL -> rounds t = 1, 2, ...: Detector round ->
 *      INT (carries each rank's changed flag and device-error bit) -> intent reduction; stop at
 *      the first t >= 2 with no change anywhere (APC / USER_ISOLATION: t = 1).  A device error
 *      on any rank (invalid batch, scratch / exchange overflow) abandons the batch on every rank
 *      at that round's INT exchange (the failing rank returns its own code, the others
 *      SOLID_ERR_STATE); nothing is committed;
 *   3. commit: each shard counts its new entries; a capacity overflow (or error) on any shard is
 *      voted through one more exchange and every shard that claimed rolls back (SOLID_ERR_CAPACITY
 *      on every rank; the index is as before the batch).
 * A peer that does not post within 60 s -> SOLID_ERR_NCCL on the waiting ranks.
 * Device pointers as in solid_dist_begin; out[n] = this slice's results.  `timing` (may be NULL)
 * receives the rounds and the exchange figures of this call.  Synchronises `stream`. */
typedef struct {
  uint32_t rounds;               /* resolver rounds                                          */
  uint32_t exchanges;            /* record exchanges (REG, PULL, INT)                        */
  float exchange_ms;             /* device time in the exchange waits (post -> every peer
                                    posted; includes waiting for the slowest rank)           */
  uint32_t record_bytes;         /* bytes per record (24)                                    */
  uint64_t recv_records_remote;  /* records received from other ranks over the whole batch  */
  uint64_t recv_records_local;   /* records this rank sent itself                            */
} solid_dist_timing;

solid_status solid_dist_admit(solid_ctx* ctx, const solid_batch* local, solid_result* out,
                              uint64_t seq_base, solid_dist_timing* timing, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SOLID_H */
