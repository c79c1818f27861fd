// solid.cu — B200 (sm_100a) kernels + host runtime behind include/solid.h.
//
// Hot path of one batch:
//   K_A  k_hash_register   tokens -> per-block hash (a2) -> chained-prefix scan (a3) -> key ->
//                          register in the batch key table (a4; the index is probed once per
//                          distinct key) -> APC first-occurrence guess
//   K_B  k_eval<POLICY>    per-request first miss (a5, warp ballot), barrier scan, isolated walk,
//                          flag decision, seq-min scatter of staged inserts/flags — repeated
//                          (Jacobi rounds) until no decision changes = the sequential answer (R1)
//   K_C  k_commit          128-bit CAS claims {key, owner, sharer} + sharer writes (a6);
//                          the same kernel rolls a batch back exactly on capacity overflow
//   K_D  k_stats           per-batch sums
//
// Batch key table ("scratch"): open addressing over 16-byte slots {key ^ salt(E), id | E << 32}
// written by one 128-bit CAS.  A slot is live only for the batch epoch E that wrote it, so the
// table is never cleared.  Each distinct key gets a dense id; its staged state lives in Hot[id]
// (32 bytes = one sector) and its index snapshot in Cold[id].
//
// Sequence tags.  Every staged value is a u64 (tag << 32 | seq') with tag = ~(E*4096 + sub),
// seq' = batch position + 1, sub = 0 (round-0 guess), t (round t), 4095 (index snapshot).  atomicMin
// keeps the EARLIEST request of the newest tag, so stale rounds and batches never need clearing.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cub/cub.cuh>   // device radix sort / scan (LRU eviction mode, solid_evict.inc)

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

#include "solid.h"
#include "solid_math.cuh"

namespace solid {

namespace cg = cooperative_groups;

constexpr int kNSeg = 128;            // id-allocation segments (spread the allocation atomics)
struct alignas(128) SegCounter {       // one id counter per 128-byte line: atomics on counters
  uint32_t v;                          // sharing a line serialise in one L2 slice
  uint32_t pad[31];
};
constexpr uint32_t kSubSnap = 4095;
constexpr uint32_t kLongBlocks = 128;   // K_A: longer requests are hashed by a whole CTA
constexpr uint64_t kLongMaxBatch = 148 * 32;   // ... in batches of at most this many requests
constexpr int kIsoG = 4;                         // resolver: isolated-walk groups in flight
constexpr uint32_t kMaxRounds = 4093;
constexpr uint32_t kStampWaitNs = 12000;    // resolver main pass: longest wait for a stamp
constexpr uint32_t kMaxEpoch = (0xFFFFFFFFu / 4096u) - 1;

enum : uint32_t {
  ERR_OFFSETS = 1, ERR_TOKEN = 2, ERR_USER = 4, ERR_BLOCKS = 8, ERR_SCRATCH = 16, ERR_SLOTCAP = 32,
  ERR_TIMEOUT = 64   // sharded: a peer never posted its exchange (peer-memory transport)
};

struct __align__(32) Hot {            // staged state of one key, ping-pong by round parity P:
  unsigned long long v[4];            // v[2P] first inserter, v[2P+1] first flagger (tag<<32|seq')
};
struct Cold {                         // the key and its index snapshot at batch start
  unsigned long long key;
  uint32_t snap_owner;                // kNone = absent from the index
  uint32_t snap_sharer;
  uint32_t psl;                       // index slot (snapshot entry, or the slot claimed at commit)
  uint32_t win;                       // evict mode: eviction-window index, kNone = not in it
};
static_assert(sizeof(Hot) == 32 && sizeof(Cold) == 24, "layout");

struct DevStatus {
  uint32_t err;
  uint32_t conv;                         // converged round (0 = not converged)
  unsigned long long new_entries;        // entries claimed by k_commit
  unsigned long long new_flags;          // sharer writes on index (snapshot) entries
  uint32_t overflow;                     // asynchronous admission: capacity exceeded, rolled back
  uint32_t blocks_done;                  // k_stats last-block detection
  uint32_t long_cnt;                     // K_A: requests handed to the CTA-per-request path
  uint32_t long_head;                    // its work counter
  unsigned long long live_after;         // asynchronous admission: live entries after this batch
  unsigned long long ids_after_hash;     // distinct keys registered by K_A (its snapshot probes)
  unsigned long long sums[6];            // blocks, reused, flagged, diverted, truncated, requests
  uint32_t packed;                       // K_A: the packed kernel took this batch (short requests)
  uint32_t fast_commit;                  // k_stats: live + registered ids <= capacity, so the
                                         // batch cannot overflow: k_commit counts and updates live
  uint32_t grab[4];                      // resolver: round t's dynamic-tail counter (t & 3)
  unsigned long long round_ns[17];       // globaltimer at resolver start and after rounds 1..16
  uint32_t seg[kNSeg];                   // id counts per segment (gathered by k_stats)
#ifdef SOLID_COUNTERS
  unsigned long long cnt[16][12];        // profiling build only: per-round path counters
#endif
  // last: round t's "some decision changed" holds the batch epoch (never reset; a stale value
  // can only cost one certifying round), so a batch clears and copies only the head above
  uint32_t changed[kMaxRounds + 2];
};
constexpr size_t kStHead = offsetof(DevStatus, changed);

struct KParams {
  int policy;
  uint32_t klo[kBS], khi[kBS];     // K_i = B^i split in 32-bit limbs
  unsigned long long ksum_lo, ksum_hi;   // sum_i K_lo, sum_i K_hi (the "+1" of x = token + 1)
  const unsigned long long* mpow;  // M^i, i < max_blocks
  const unsigned long long* gtab;  // G[d] = sum_{t<d} M^t, d <= max_blocks
  // H-def v3 second component (nc == 2): same layout for base B2
  int nc;
  uint32_t klo2[kBS], khi2[kBS];
  unsigned long long ksum_lo2, ksum_hi2;
  const unsigned long long* mpow2;
  const unsigned long long* gtab2;
  ulonglong2* cs;                  // nc == 2: per key id, its chain values {S, S2}
  uint64_t seed;
  const uint32_t* tokens;
  const uint64_t* offsets;
  const uint32_t* users;
  const uint8_t* enforce;
  uint64_t n;
  uint64_t j_lo;                   // resolver / stats: requests [j_lo, n) (a split batch's part)
  uint32_t max_blocks;
  uint32_t epoch;
  unsigned long long salt;         // per-epoch key salt of the batch key table
  ulonglong2* stab;                // batch key table
  uint64_t smask;
  Hot* hot;
  Cold* cold;
  ulonglong2* tab;                 // the index {key, owner | sharer << 32}
  uint64_t tmask;
  uint32_t* id_of_block;           // per block: id of its Shared (USER_ISOLATION: U) key
  uint32_t* iso_id;                // per block: id of its isolated key (valid for dec.f)
  uint64_t slot_cap;
  uint4* dec;
  int stamp;                       // inserter-stamp rule on (SOLID_STAMP=0 turns it off for A/B)
  int tail;                        // resolver: last sweeps handed out dynamically (SOLID_TAIL, 0: off)
  uint32_t stamp_wait_ns;          // its wait bound in the main pass (kStampWaitNs)
  uint32_t* dlist;                 // requests deferred by the main pass of a round (stale stamp)
  uint32_t* dcnt;                  // [2]: their count, by round parity
  unsigned long long* fst;         // per request: tag(round) << 32 | divert depth f of its latest
                                   // evaluation (single GPU; read by later requests)
  solid_result* out;
  SegCounter* seg_cnt;
  uint32_t seg_cap;
  DevStatus* st;
  // sharded mode: global sequence base of this rank's requests; the local table
  // holds a mirror of each referenced key's staged state pulled from its owner shard
  uint64_t seq_base;
  int dist;
  unsigned long long* int_ins;     // per local id: this round's earliest local inserter (seq'<<32|user)
  unsigned long long* int_flg;     // per local id: this round's earliest local flagger
  uint32_t* mown;                  // per local id: owner user of the mirrored first inserter
  ulonglong2* lint;                // per local id: the intents last sent to its owner (delta INT)
  uint32_t* long_q;                // K_A: requests longer than kLongBlocks (CTA path)
  // packed K_A for short requests (solid_pack.inc): on for whole-batch launches only
  int pack;
  uint32_t* pk_pre;                // [n + 1] packed full-block prefix Bp[j]
  uint32_t* pk_ctot;               // [grid] per-CTA chunk totals
  uint32_t* pk_cpre;               // [grid + 1] their exclusive prefix
  uint32_t* pk_wfirst;             // [warps + 2] first request starting in each warp's span
  uint32_t* pool_cnt;              // block_table: k_commit counts each request's new entries
  uint32_t* seg_new;               // [kNSeg][2] fast_commit: k_commit's new entries / sharers
  // LRU eviction mode (solid_evict.inc): keys of the batch whose LRU record lies
  // in the eviction window get a window index w (their index snapshot is then visible only up
  // to their eviction time win_ev[w]); winfo[id] = epoch << 32 | w publishes an id's creation
  int evict;
  unsigned long long* winfo;
  const uint32_t* lpos;            // per index slot: position of its valid LRU record
  const uint32_t* lbits;           // LRU log valid bitmap
  const uint32_t* lpc;             // exclusive prefix popcount of lbits words (batch start)
  const unsigned long long* sum_blocks;   // sum of n_j over the batch (device)
  unsigned long long ev_live0, ev_cap;
  uint32_t* win_cnt;
  uint32_t* win_id;
  uint32_t* win_rank;
  uint32_t* win_ev;                // seq' of the evicting request, kNone = not evicted
  unsigned long long* win_oflg;    // [w][2] old-incarnation flagger (tagged, ping-pong)
  uint32_t* win_tau;               // first request served the key (post-pass)
  uint8_t* win_skip;               // k_window's skip flag per window index (0 at creation)
  uint32_t* win_dense;             // [rank] = window index + 1 (0 = no window key of that rank)
  uint32_t* ins_cnt;               // per request: entries it inserts (final round)
  uint32_t* ins_scan;              // merged joint step: their inclusive prefix (resolver tail)
  uint32_t* lt;                    // per id: last request served it (final)
};

#define POLICY_IS_SOLIDARITY(kp) ((kp).policy == SOLID_POLICY_SOLIDARITY)

__host__ __device__ __forceinline__ uint32_t tag_of(uint32_t epoch, uint32_t sub) {
  return 0xFFFFFFFFu - (epoch * 4096u + sub);
}

__device__ __forceinline__ void set_err(DevStatus* st, uint32_t bits) { atomicOr(&st->err, bits); }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Weak (L1-cacheable) loads kept in program order.  Used where a stale value is safe: table
// slots only move stale -> live within a batch, staged values only decrease, and L1 is
// invalidated at every kernel launch.
__device__ __forceinline__ ulonglong2 ldw128(const void* p) {
  ulonglong2 r;
  asm volatile("ld.global.v2.u64 {%0,%1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ unsigned long long ldw64(const void* p) {
  unsigned long long r;
  asm volatile("ld.global.u64 %0, [%1];" : "=l"(r) : "l"(p));
  return r;
}
// Single-copy-atomic 64-bit accesses at gpu scope (the per-request round stamps, fst[]).
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long r;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// 128-bit compare-and-swap (ATOMG.E.CAS.128 on sm_90+).
__device__ __forceinline__ ulonglong2 atomic_cas128(ulonglong2* addr, ulonglong2 cmp,
                                                    ulonglong2 val) {
  ulonglong2 old;
  asm volatile(
      "{\n\t.reg .b128 c, v, d;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.global.cas.b128 d, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(old.x), "=l"(old.y)
      : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(addr)
      : "memory");
  return old;
}

__device__ __forceinline__ void atomic_min_u64(unsigned long long* a, unsigned long long v) {
  // read-before-atomic: values only ever decrease, so a stale read is >= the true value.
  if (ldw64(a) > v) atomicMin(a, v);
}

// Round-t view of a ping-pong pair {P0, P1} of one key: the earliest request (seq' >= 1, or 0 for
// the index snapshot) visible to request seqp, reading round t-1's complete values (tagR in P[R])
// and the round-t values already published in P[W] (Gauss-Seidel).  kNone if none is visible.
// Mixing in partial round-t values never breaks exactness: a round whose decisions all equal the
// previous round's certifies the sequential fixed point, and requests < t are final after round t.
__device__ __forceinline__ uint32_t gs_first(unsigned long long p0, unsigned long long p1, int R,
                                             uint32_t seqp, uint32_t tagR, uint32_t tagW,
                                             uint32_t tagS) {
  const unsigned long long a = R ? p1 : p0, b = R ? p0 : p1;
  const uint32_t ta = (uint32_t)(a >> 32), tb = (uint32_t)(b >> 32);
  if (ta == tagS || tb == tagS) return 0;
  uint32_t s = kNone;
  if (ta == tagR && (uint32_t)a < seqp) s = (uint32_t)a;
  if (tb == tagW && (uint32_t)b < seqp) s = min(s, (uint32_t)b);
  return s;
}

// ---------------------------------------------------------------------------------------------
// Index probe: linear probing over 16-byte slots {key, owner | sharer << 32}; 0 = empty.
// ---------------------------------------------------------------------------------------------
// Continues a probe whose home slot `e` (at `pos`) was already loaded.
__device__ __forceinline__ bool index_find_from(const KParams& kp, uint64_t key, ulonglong2 e,
                                                uint32_t& owner, uint32_t& sharer, uint64_t& pos) {
  for (;;) {
    if (e.x == key) {
      owner = (uint32_t)e.y;
      sharer = (uint32_t)(e.y >> 32);
      return true;
    }
    if (e.x == 0 && e.y == 0) return false;   // EMPTY; {0, ~0} is a tombstone (evict mode)
    pos = (pos + 1) & kp.tmask;
    e = ldw128(&kp.tab[pos]);
  }
}

__device__ __forceinline__ bool index_find(const KParams& kp, uint64_t key, uint32_t& owner,
                                           uint32_t& sharer, uint64_t& pos) {
  pos = key & kp.tmask;
  return index_find_from(kp, key, ldw128(&kp.tab[pos]), owner, sharer, pos);
}

__device__ __forceinline__ uint64_t scratch_home(uint64_t key, uint64_t mask) {
  return (key ^ (key >> 29)) & mask;
}

// The creator of an id records the key and its index snapshot, and seeds both ping-pong states
// with it (the snapshot tag is the smallest tag of the batch, so it is never displaced).
__device__ __forceinline__ bool init_id_at(const KParams& kp, uint32_t id, uint64_t key,
                                           bool present, uint32_t owner, uint32_t sharer,
                                           uint64_t ipos) {
  Cold c;
  c.key = key;
  c.snap_owner = present ? owner : kNone;
  c.snap_sharer = present ? sharer : kNone;
  c.psl = present ? (uint32_t)ipos : kNone;
  c.win = kNone;
  if (kp.evict && present) {
    // eviction window: the entry's LRU rank among the live entries at batch start
    // (valid records before its own); only ranks below ebound can be evicted by this batch
    // ranks count the EVICTABLE records only (pin mode: pinned entries are not in lbits, R38)
    const uint32_t p = kp.lpos[ipos];
    const uint32_t rank = kp.lpc[p >> 5] + __popc(kp.lbits[p >> 5] & ((1u << (p & 31)) - 1u));
    const unsigned long long tot = kp.ev_live0 + *kp.sum_blocks;
    const unsigned long long ebound = tot > kp.ev_cap ? tot - kp.ev_cap : 0ull;
    if (rank < ebound && ((kp.lbits[p >> 5] >> (p & 31)) & 1u)) {
      const uint32_t w = atomicAdd(kp.win_cnt, 1u);
      kp.win_id[w] = id;
      kp.win_rank[w] = rank;
      kp.win_ev[w] = kNone;
      kp.win_oflg[2 * w] = ~0ull;
      kp.win_oflg[2 * w + 1] = ~0ull;
      kp.win_skip[w] = 0;
      kp.win_dense[rank] = w + 1;    // ranks are unique: the window in rank order, unsorted
      c.win = w;
    }
  }
  kp.cold[id] = c;
  if (present && c.win == kNone) {
    Hot* h = kp.hot + id;
    const unsigned long long v = (unsigned long long)tag_of(kp.epoch, kSubSnap) << 32;
    atomicMin(&h->v[0], v);
    atomicMin(&h->v[2], v);
    if (sharer != kNone) {
      atomicMin(&h->v[1], v);
      atomicMin(&h->v[3], v);
    }
  }
  if (kp.evict) {              // publish: readers wait for epoch << 32 | w before reading state
    __threadfence();
    atomicExch(&kp.winfo[id], ((unsigned long long)kp.epoch << 32) | c.win);
  }
  return present;
}

__device__ bool init_id(const KParams& kp, uint32_t id, uint64_t key, uint64_t s1 = 0,
                        uint64_t s2 = 0) {
  if (kp.nc == 2) kp.cs[id] = make_ulonglong2(s1, s2);   // published with the id (below)
  uint32_t owner = kNone, sharer = kNone;
  uint64_t ipos = 0;
  // sharded mode: a local table entry may belong to another shard; its state comes from there
  const bool present = !kp.dist && index_find(kp, key, owner, sharer, ipos);
  return init_id_at(kp, id, key, present, owner, sharer, ipos);
}

// A tile of TW lanes (32: the warp; 16: half a warp) that works on one request.  Its collective
// operations use the tile's own lane mask, so the two halves of a warp may take different paths
// (each evaluates its own request).  ballot() returns the tile's bits in the low TW positions.
template <int TW>
struct Tile {
  uint32_t mask;
  int base;
  __device__ __forceinline__ Tile() {
    if (TW == 32) {
      mask = 0xffffffffu;
      base = 0;
    } else {
      base = (int)(threadIdx.x & 31) & ~(TW - 1);
      mask = ((1u << (TW & 31)) - 1u) << base;
    }
  }
  __device__ __forceinline__ uint32_t ballot(bool p) const {
    return TW == 32 ? __ballot_sync(0xffffffffu, p) : (__ballot_sync(mask, p) >> base);
  }
  template <class T>
  __device__ __forceinline__ T shfl(T v, int src) const { return __shfl_sync(mask, v, src, TW); }
  template <class T>
  __device__ __forceinline__ T shfl_up(T v, unsigned d) const {
    return __shfl_up_sync(mask, v, d, TW);
  }
  __device__ __forceinline__ bool all(bool p) const { return __all_sync(mask, p); }
};

// Tile-cooperative (TW lanes) find-or-insert of one key per active lane.  Returns the key's id (0 only on
// scratch overflow); `created` is set for the lane whose CAS published the key.  New ids are
// allocated with one atomic per warp and probe step (segment `seg`).
template <int TW = 32>
__device__ __forceinline__ uint32_t scratch_register(const KParams& kp, bool active, uint64_t key,
                                                     uint32_t seg, int lane, bool& created,
                                                     bool* snap_present = nullptr,
                                                     uint64_t s1 = 0, uint64_t s2 = 0) {
  const unsigned long long kx = key ^ kp.salt;
  const uint32_t E = kp.epoch;
  uint64_t pos = scratch_home(key, kp.smask);
  uint32_t id = 0;
  bool done = !active;
  bool have_e = false;           // e holds the slot's current value from a failed CAS
  ulonglong2 e = make_ulonglong2(0, 0);
  created = false;
  const Tile<TW> T;
  for (uint64_t probes = 0;; ++probes) {
    bool want = false;
    if (!done) {
      if (!have_e) e = ldw128(&kp.stab[pos]);
      have_e = false;
      if ((uint32_t)(e.y >> 32) == E) {            // live in this batch
        if (e.x == kx) {
          id = (uint32_t)e.y;
          done = true;
        } else {
          pos = (pos + 1) & kp.smask;
        }
      } else {
        want = true;                                // stale or never used: claim it
      }
    }
    const uint32_t wm = T.ballot(want);
    if (wm) {
      uint32_t base = 0;
      if (lane == __ffs(wm) - 1) base = atomicAdd(&kp.seg_cnt[seg].v, (uint32_t)__popc(wm));
      base = T.shfl(base, __ffs(wm) - 1);
      if (want) {
        const uint32_t idx = base + __popc(wm & ((1u << lane) - 1u));
        if (idx >= kp.seg_cap) {
          set_err(kp.st, ERR_SCRATCH);
          done = true;
        } else {
          const uint32_t mine = seg * kp.seg_cap + idx + 1;
          if (kp.dist) {      // sharded: a fresh local id has no mirrored state and no intents
            kp.hot[mine].v[0] = ~0ull;
            kp.hot[mine].v[1] = ~0ull;
            kp.int_ins[mine] = ~0ull;
            kp.int_flg[mine] = ~0ull;
            kp.mown[mine] = kNone;
            kp.lint[mine] = make_ulonglong2(~0ull, ~0ull);
            __threadfence();  // visible before the CAS publishes the id
          }
          const ulonglong2 nv =
              make_ulonglong2(kx, (unsigned long long)mine | ((unsigned long long)E << 32));
          const ulonglong2 old = atomic_cas128(&kp.stab[pos], e, nv);
          if (old.x == e.x && old.y == e.y) {
            id = mine;
            created = true;
            done = true;
            const bool pr = init_id(kp, id, key, s1, s2);
            if (snap_present) *snap_present = pr;
          } else {
            e = old;                                // authoritative current value: re-examine
            have_e = true;                          // without trusting a possibly stale L1 line
          }
        }
      }
    }
    if (T.all(done)) break;
    if (probes > kp.smask) {
      if (!done) set_err(kp.st, ERR_SCRATCH);
      break;
    }
  }
  return id;
}

// Find-only lookup (0 = not registered in this batch).
__device__ __forceinline__ uint32_t scratch_find(const KParams& kp, uint64_t key) {
  const unsigned long long kx = key ^ kp.salt;
  uint64_t pos = scratch_home(key, kp.smask);
  for (uint64_t probes = 0; probes <= kp.smask; ++probes) {
    const ulonglong2 e = ldw128(&kp.stab[pos]);
    if ((uint32_t)(e.y >> 32) != kp.epoch) return 0;
    if (e.x == kx) return (uint32_t)e.y;
    pos = (pos + 1) & kp.smask;
  }
  return 0;
}

// ---------------------------------------------------------------------------------------------
// K_A (round 0): hash + chained-prefix scan + registration.  One warp per request; lane = block
// within a 32-block group; the next group's tokens are in flight while this group registers.
// Forward-exponent chain:
//   S[b] = sum_{t<=b} M^(t-1) * (h_t + sigma)   — a prefix SUM: warp shfl scan + scalar carry.
// ---------------------------------------------------------------------------------------------
// Token loads: each lane loads its own 64-byte block with 16-byte non-coherent loads (4 when
// the request is 16-byte aligned, the aligned 20-word window when it is not; SH is warp-uniform),
// one group ahead: the next group's loads are in flight while this group hashes and registers.
// (A cp.async staging through bank-conflict-free shared rows measured slower: 323 vs 290 us on
// C2 — this kernel is bound by the registration latency, not by the token loads.)
__device__ __forceinline__ uint4 ldg_v4(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// The same without L1 allocation (packed K_A: the token stream does not evict the key-table and
// key-state lines its probes hit in L1; C4 hash 1.33 -> 1.26 ms.  The warp-per-request K_A is
// slower with it, 0.314 -> 0.330 ms on C2: profiles/r02/experiments_r2.md).
__device__ __forceinline__ uint4 ldg_v4_na(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// 32-byte loads (LDG.E.256) of a 32-byte-aligned block: two per block, each covering whole
// 32-byte sectors.
__device__ __forceinline__ void ldg_v8(const uint32_t* p, uint32_t* r) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}

// SH: the request's token offset mod 4 (16-byte loads of the aligned window); V8 (SH = 0 and
// the request 32-byte aligned): two 32-byte loads per block.
template <int SH, bool V8 = false>
struct BlockWords {
  static constexpr int W = SH ? 20 : 16;
  uint32_t w[W];
  __device__ __forceinline__ void load(const uint32_t* p) {
    if (V8) {
      ldg_v8(p, w);
      ldg_v8(p + 8, w + 8);
      return;
    }
    const uint32_t* a = p - SH;
#pragma unroll
    for (int q = 0; q < W / 4; ++q) {
      const uint4 v = ldg_v4(a + 4 * q);
      w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
  }
  // h = sum_i (tok_i + 1) K_i mod p; the "+1" is folded into kp.ksum_*.
  __device__ __forceinline__ uint64_t hash(const KParams& kp, uint32_t& bad) const {
    uint64_t lo = kp.ksum_lo, hi = kp.ksum_hi;
    uint32_t orv = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t t = w[i + SH];
      orv |= t;
      lo += (uint64_t)t * kp.klo[i];
      hi += (uint64_t)t * kp.khi[i];
    }
    bad |= orv >> 20;
    // lo + hi*2^32 mod p, with hi*2^32 = (hi mod 2^29)*2^32 + (hi >> 29)*2^61 == ... + (hi >> 29);
    // partially folded (< 2^61 + 7): it only feeds mulmod
    return fold61_lazy(lo + ((hi & 0x1FFFFFFFull) << 32) + (hi >> 29));
  }
  // second component (base B2), same limb scheme
  __device__ __forceinline__ uint64_t hash2(const KParams& kp) const {
    uint64_t lo = kp.ksum_lo2, hi = kp.ksum_hi2;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t t = w[i + SH];
      lo += (uint64_t)t * kp.klo2[i];
      hi += (uint64_t)t * kp.khi2[i];
    }
    return fold61_lazy(lo + ((hi & 0x1FFFFFFFull) << 32) + (hi >> 29));
  }
};

template <int POLICY, int SH, int NC, bool V8 = false>
__device__ __forceinline__ uint32_t hash_register_request(const KParams& kp, uint64_t j, int lane,
                                                          const uint32_t* base, uint32_t n,
                                                          uint64_t blk0, uint32_t u,
                                                          uint32_t seg) {
  const uint64_t sig = (POLICY == SOLID_POLICY_USER_ISOLATION) ? sigma_of(kp.seed, u) : 0;
  const uint64_t sig2 =
      (NC == 2 && POLICY == SOLID_POLICY_USER_ISOLATION) ? sigma2_of(kp.seed, u) : 0;
  const unsigned long long guess =
      ((unsigned long long)tag_of(kp.epoch, 0) << 32) | (unsigned long long)(kp.seq_base + j + 1);
  uint64_t carry = 0, carry2 = 0;
  uint32_t bad = 0;
  BlockWords<SH, V8> cur, nxt;
  if ((uint32_t)lane < n) cur.load(base + (uint64_t)kBS * lane);
  for (uint32_t g = 0; g < n; g += 32) {
    const uint32_t i = g + lane;
    const bool valid = i < n;
    if (i + 32 < n) nxt.load(base + (uint64_t)kBS * (i + 32));       // prefetch next group
    uint64_t term = 0, term2 = 0;
    if (valid) {
      term = mulmod(cur.hash(kp, bad) + sig, kp.mpow[i]);     // < 2^62 + 7: a mulmod operand
      if (NC == 2) term2 = mulmod(cur.hash2(kp) + sig2, kp.mpow2[i]);
    }
    const uint64_t S = addmod(warp_scan_addmod(term, lane), carry);
    carry = __shfl_sync(0xffffffffu, S, 31);
    uint64_t S2 = 0;
    if (NC == 2) {
      S2 = addmod(warp_scan_addmod(term2, lane), carry2);
      carry2 = __shfl_sync(0xffffffffu, S2, 31);
    }
    bool created = false;
    const uint32_t id = scratch_register(kp, valid, NC == 2 ? key2_of(S, S2) : key_of(S), seg,
                                         lane, created, nullptr, S, S2);
    if (valid && id) {
      kp.id_of_block[blk0 + i] = id;
      // Round-0 state: the exact first occurrence (seq-min over all occurrences).  APC and
      // USER_ISOLATION finish from it in one pass; for SOLIDARITY it is the Jacobi starting
      // point (a worse start, e.g. the creator's seq', costs extra heavy rounds on C2).
      if (created) atomicMin(&kp.hot[id].v[0], guess);
      else atomic_min_u64(&kp.hot[id].v[0], guess);
    }
    cur = nxt;
  }
  return bad;
}

__device__ __forceinline__ bool pack_chosen(const KParams& kp);

template <int POLICY, int NC>
__global__ void __launch_bounds__(256, 4) k_hash_register(KParams kp, uint64_t j_lo, uint64_t j_hi) {
  if (pack_chosen(kp)) return;           // short requests: k_hash_packed registers the batch
  const int lane = threadIdx.x & 31;
  const uint64_t j = j_lo + (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (j >= j_hi) return;
  const uint32_t seg = (uint32_t)(j & (kNSeg - 1));
  const uint64_t o0 = kp.offsets[j], o1 = kp.offsets[j + 1];
  const uint32_t u = kp.users[j];
  if (lane == 0) {
    if ((j == 0 && o0 != 0) || o1 < o0) set_err(kp.st, ERR_OFFSETS);
    if (u == kNone) set_err(kp.st, ERR_USER);
  }
  if (o1 < o0) return;
  const uint64_t nb = (o1 - o0) >> 4;
  if (nb > kp.max_blocks) {
    if (lane == 0) set_err(kp.st, ERR_BLOCKS);
    return;
  }
  const uint32_t n = (uint32_t)nb;
  const uint64_t blk0 = o0 >> 4;
  if (n && blk0 + n > kp.slot_cap) {
    if (lane == 0) set_err(kp.st, ERR_SLOTCAP);
    return;
  }
  if (n > kLongBlocks && kp.long_q) {   // hashed by a whole CTA (k_hash_register_long)
    if (lane == 0) kp.long_q[atomicAdd(&kp.st->long_cnt, 1u)] = (uint32_t)j;
    return;
  }
  const uint32_t* base = kp.tokens + o0;
  uint32_t bad;
  switch (((uintptr_t)base >> 2) & 3) {
    case 0:
      bad = ((uintptr_t)base & 31)
                ? hash_register_request<POLICY, 0, NC>(kp, j, lane, base, n, blk0, u, seg)
                : hash_register_request<POLICY, 0, NC, true>(kp, j, lane, base, n, blk0, u, seg);
      break;
    case 1: bad = hash_register_request<POLICY, 1, NC>(kp, j, lane, base, n, blk0, u, seg); break;
    case 2: bad = hash_register_request<POLICY, 2, NC>(kp, j, lane, base, n, blk0, u, seg); break;
    default: bad = hash_register_request<POLICY, 3, NC>(kp, j, lane, base, n, blk0, u, seg); break;
  }
  if (__any_sync(0xffffffffu, bad != 0) && lane == 0) set_err(kp.st, ERR_TOKEN);
}

// K_A for long requests: one CTA (8 warps) per request, 8 groups of 32 blocks at a time — each
// warp hashes and locally scans its group, the chain carry crosses the warps through shared
// memory (two barriers per 256 blocks), then the 8 groups register in parallel.  A request
// longer than kLongBlocks would otherwise keep one warp walking its groups in sequence.

template <int POLICY, int SH, int NC>
__device__ __forceinline__ uint32_t hash_register_long(const KParams& kp, uint64_t j, int lane,
                                                       int wl, const uint32_t* base, uint32_t n,
                                                       uint64_t blk0, uint32_t u, uint32_t seg,
                                                       uint64_t* s_tot, uint64_t* s_tot2) {
  const uint64_t sig = (POLICY == SOLID_POLICY_USER_ISOLATION) ? sigma_of(kp.seed, u) : 0;
  const uint64_t sig2 =
      (NC == 2 && POLICY == SOLID_POLICY_USER_ISOLATION) ? sigma2_of(kp.seed, u) : 0;
  const unsigned long long guess =
      ((unsigned long long)tag_of(kp.epoch, 0) << 32) | (unsigned long long)(kp.seq_base + j + 1);
  uint64_t carry = 0, carry2 = 0;                 // chain value before this CTA step
  uint32_t bad = 0;
  for (uint32_t g0 = 0; g0 < n; g0 += 256) {
    const uint32_t g = g0 + 32u * (uint32_t)wl;
    const uint32_t i = g + lane;
    const bool valid = i < n;
    uint64_t term = 0, term2 = 0;
    if (valid) {
      BlockWords<SH> blk;
      blk.load(base + (uint64_t)kBS * i);
      term = mulmod(blk.hash(kp, bad) + sig, kp.mpow[i]);
      if (NC == 2) term2 = mulmod(blk.hash2(kp) + sig2, kp.mpow2[i]);
    }
    const uint64_t loc = warp_scan_addmod(term, lane);
    const uint64_t loc2 = NC == 2 ? warp_scan_addmod(term2, lane) : 0;
    if (lane == 31) {
      s_tot[wl] = loc;
      if (NC == 2) s_tot2[wl] = loc2;
    }
    __syncthreads();
    uint64_t c = carry, c2 = carry2;
    for (int w = 0; w < wl; ++w) {
      c = addmod(c, s_tot[w]);
      if (NC == 2) c2 = addmod(c2, s_tot2[w]);
    }
    for (int w = 0; w < 8; ++w) {
      carry = addmod(carry, s_tot[w]);
      if (NC == 2) carry2 = addmod(carry2, s_tot2[w]);
    }
    __syncthreads();                                // s_tot free for the next step
    if (g < n) {                                    // warp-uniform
      const uint64_t S = addmod(loc, c);
      const uint64_t S2 = NC == 2 ? addmod(loc2, c2) : 0;
        bool created = false;
      const uint32_t id = scratch_register(kp, valid, NC == 2 ? key2_of(S, S2) : key_of(S), seg,
                                           lane, created, nullptr, S, S2);
      if (valid && id) {
        kp.id_of_block[blk0 + i] = id;
        if (created) atomicMin(&kp.hot[id].v[0], guess);
        else atomic_min_u64(&kp.hot[id].v[0], guess);
      }
    }
  }
  return bad;
}

template <int POLICY, int NC>
__global__ void __launch_bounds__(256, 4) k_hash_register_long(KParams kp) {
  __shared__ uint64_t s_tot[8], s_tot2[8];
  __shared__ uint32_t s_j;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) {
      const uint32_t q = atomicAdd(&kp.st->long_head, 1u);
      s_j = q < *(volatile uint32_t*)&kp.st->long_cnt ? kp.long_q[q] : 0xFFFFFFFFu;
    }
    __syncthreads();
    const uint32_t jj = s_j;
    __syncthreads();
    if (jj == 0xFFFFFFFFu) return;
    const uint64_t j = jj;
    const uint64_t o0 = kp.offsets[j];
    const uint32_t n = (uint32_t)((kp.offsets[j + 1] - o0) >> 4);   // validated by k_hash_register
    const uint64_t blk0 = o0 >> 4;
    const uint32_t u = kp.users[j];
    const uint32_t seg = (uint32_t)(j & (kNSeg - 1));
    const uint32_t* base = kp.tokens + o0;
    uint32_t bad;
    switch (((uintptr_t)base >> 2) & 3) {
      case 0: bad = hash_register_long<POLICY, 0, NC>(kp, j, lane, wl, base, n, blk0, u, seg, s_tot, s_tot2); break;
      case 1: bad = hash_register_long<POLICY, 1, NC>(kp, j, lane, wl, base, n, blk0, u, seg, s_tot, s_tot2); break;
      case 2: bad = hash_register_long<POLICY, 2, NC>(kp, j, lane, wl, base, n, blk0, u, seg, s_tot, s_tot2); break;
      default: bad = hash_register_long<POLICY, 3, NC>(kp, j, lane, wl, base, n, blk0, u, seg, s_tot, s_tot2); break;
    }
    if (__any_sync(0xffffffffu, bad != 0) && lane == 0) set_err(kp.st, ERR_TOKEN);
  }
}

// K_A on stream s (single GPU and sharded paths), for requests [lo, hi) of the batch (host
// admission hashes each sub-range as soon as its tokens have arrived).
template <int NC>
static void launch_hash_nc(const KParams& kp, unsigned grid, unsigned B, uint64_t lo, uint64_t hi,
                           cudaStream_t s) {
  const unsigned lg = 148 * 4;   // persistent CTAs for the long requests (none: they exit at once)
  switch (kp.policy) {
    case SOLID_POLICY_APC:
      k_hash_register<SOLID_POLICY_APC, NC><<<grid, B, 0, s>>>(kp, lo, hi);
      if (kp.long_q) k_hash_register_long<SOLID_POLICY_APC, NC><<<lg, 256, 0, s>>>(kp);
      break;
    case SOLID_POLICY_USER_ISOLATION:
      k_hash_register<SOLID_POLICY_USER_ISOLATION, NC><<<grid, B, 0, s>>>(kp, lo, hi);
      if (kp.long_q) k_hash_register_long<SOLID_POLICY_USER_ISOLATION, NC><<<lg, 256, 0, s>>>(kp);
      break;
    default:
      k_hash_register<SOLID_POLICY_SOLIDARITY, NC><<<grid, B, 0, s>>>(kp, lo, hi);
      if (kp.long_q) k_hash_register_long<SOLID_POLICY_SOLIDARITY, NC><<<lg, 256, 0, s>>>(kp);
      break;
  }
}
// K_A threads per CTA: 256 (8 requests per CTA), or 64 when the batch is expected to take the
// warp-per-request path (a CTA releases its slot as soon as its 2 requests are done: C2 hash
// 0.296 -> 0.282 ms, C3 1.36 -> 1.34; a batch that the packed K_A takes would pay for 4x more
// CTAs that exit at once: C4 1.26 -> 1.46 ms) — profiles/r02/ka_block_ab.txt
static cudaError_t launch_hash(const KParams& kp, cudaStream_t s, uint64_t lo, uint64_t hi,
                               unsigned B = 256) {
  if (hi <= lo) return cudaSuccess;
  const unsigned grid = (unsigned)(((hi - lo) * 32 + B - 1) / B);
  if (kp.nc == 2) launch_hash_nc<2>(kp, grid, B, lo, hi, s);
  else launch_hash_nc<1>(kp, grid, B, lo, hi, s);
  return cudaGetLastError();
}
static cudaError_t launch_hash(const KParams& kp, cudaStream_t s, unsigned B = 256) {
  return launch_hash(kp, s, 0, kp.n, B);
}

#include "solid_pack.inc"

// ---------------------------------------------------------------------------------------------
// K_B: one resolver round t (t >= 1) — the per-request Detector of P:454-459 evaluated against
// "the state as of this request", reconstructed from round t-1's staged values.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t owner_from(const KParams& kp, uint32_t id, uint32_t first) {
  return first == 0 ? kp.cold[id].snap_owner : kp.users[first - 1u];
}

__device__ __forceinline__ uint64_t iso_key(const KParams& kp, uint64_t blk, uint32_t i,
                                            uint64_t sig, uint64_t gf, uint64_t sig2 = 0,
                                            uint64_t gf2 = 0) {
  const uint32_t sid = kp.id_of_block[blk];
  const uint64_t d = submod(kp.gtab[i + 1], gf);   // G[b] - G[f], b = i + 1
  if (kp.nc == 2) {   // chain values stored at registration (a 64-bit key cannot hold both)
    const ulonglong2 c = kp.cs[sid];
    const uint64_t d2 = submod(kp.gtab2[i + 1], gf2);
    return key2_of(addmod(c.x, mulmod(sig, d)), addmod(c.y, mulmod(sig2, d2)));
  }
  const uint64_t S = chain_of(kp.cold[sid].key);
  return key_of(addmod(S, mulmod(sig, d)));
}

// Gauss-Seidel visibility of an isolated key: round t-1's value (P[R]) or a value already
// published this round (P[W], whose tags are snapshot, t, or older-and-larger).
__device__ __forceinline__ bool iso_visible(const KParams& kp, uint32_t id, int R,
                                            unsigned long long limR, unsigned long long limW) {
  const Hot* h = kp.hot + id;
  return ldw64(&h->v[2 * R]) < limR || ldw64(&h->v[2 - 2 * R]) < limW;
}

// Evaluates request j in round t with a tile of TW lanes (lane = the lane within the tile);
// returns true (tile-uniform) if its decision differs from the previous round's (always true in
// round 1).  TW = 16: two requests per warp, each half walking 4 x 16 blocks per step — twice
// the requests in flight per SM at the same register count (the rounds are latency-bound).
template <int POLICY, bool DIST, int TW = 32, bool DEFER = false>
__device__ __forceinline__ int eval_request(const KParams& kp, uint32_t t, uint64_t j, int lane) {
  constexpr bool may_defer = DEFER;
  const Tile<TW> T;
  constexpr uint32_t STEP = 4 * TW;          // blocks per walk step (4 groups in flight)
  const uint32_t seg = (uint32_t)(j & (kNSeg - 1));
  const uint64_t o0 = kp.offsets[j], o1 = kp.offsets[j + 1];
  const uint32_t u = kp.users[j];
  const bool enf = (POLICY == SOLID_POLICY_SOLIDARITY) && (kp.enforce ? kp.enforce[j] != 0 : true);
  const uint4 prev =
      (POLICY == SOLID_POLICY_SOLIDARITY && t >= 2) ? kp.dec[j] : make_uint4(0, ~0u, 0, 0);
  if (o1 < o0) return 0;
  const uint64_t nb = (o1 - o0) >> 4;
  if (nb > kp.max_blocks) return 0;
  const uint32_t n = (uint32_t)nb;
  const uint64_t blk0 = o0 >> 4;
  if (n && blk0 + n > kp.slot_cap) return 0;
  const uint32_t* sh_ids = kp.id_of_block + blk0;       // this request's blocks (32-bit indexing)
  uint32_t* iso_ids = kp.iso_id + blk0;
  const uint32_t seqp = (uint32_t)(kp.seq_base + j + 1);
  // single GPU: ping-pong by round parity.  Sharded: the pulled mirror always sits in P0 with the
  // fixed mirror tag (round 1's), and nothing is staged locally (intents go to int_ins/int_flg).
  const int R = DIST ? 0 : (int)((t - 1) & 1), W = DIST ? 1 : (int)(t & 1);
  const uint32_t tagR = tag_of(kp.epoch, DIST ? 1 : t - 1), tagW = tag_of(kp.epoch, DIST ? 0 : t),
                 tagS = tag_of(kp.epoch, kSubSnap);
  // speculation: last round's divert depth; its isolated ids are cached in iso_id[]
  const int32_t fprev = (int32_t)prev.y;
  uint32_t iso_pre_id = 0;
  if (POLICY == SOLID_POLICY_SOLIDARITY && fprev >= 1 && (uint32_t)fprev + lane < n)
    iso_pre_id = iso_ids[(uint32_t)fprev + lane];

  // ---- a5: first miss k (warp ballot) and barrier scan f over the Shared chain ----
  // During round t, P[R] holds only the snapshot tag, round t-1's tag and older (numerically
  // larger) tags, so "visible to request seqp" is one 64-bit compare v < limR = tagR<<32 | seqp
  // (snapshot values carry the smallest tag and always pass); likewise "flagged".  Blocks are
  // walked STEP at a time: ids and P[R] pairs of 4 groups of TW are in flight together.
  const unsigned long long limR = ((unsigned long long)tagR << 32) | seqp;
  const unsigned long long limW = DIST ? 0ull : ((unsigned long long)tagW << 32) | seqp;
  uint32_t k = n;
  int32_t f = -1;
  bool carry_flag = false;    // flagged(index g-1) from the previous group
  bool walked = false;
  bool iso_pre_vis = false;
  uint32_t idq[4];            // ids of the last walked STEP blocks (from wbase), kept for the scatter
  uint32_t wbase = 0;
  for (uint32_t base = 0; base <= n && !walked; base += STEP) {
    wbase = base;
    ulonglong2 pq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t i = base + TW * q + lane;
      idq[q] = i < n ? sh_ids[i] : 0u;
    }
    if (POLICY == SOLID_POLICY_SOLIDARITY && base == 0 && fprev >= 1 && (uint32_t)fprev + lane < n)
      iso_pre_vis = iso_visible(kp, iso_pre_id, R, limR, limW);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t i = base + TW * q + lane;
      pq[q] = make_ulonglong2(~0ull, ~0ull);
      if (i < n) pq[q] = ldw128(&kp.hot[idq[q]].v[2 * R]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t g = base + TW * q;
      if (g > n) break;
      const bool vis = pq[q].x < limR;                  // invalid lanes hold ~0: not visible
      const bool fl = POLICY == SOLID_POLICY_SOLIDARITY && pq[q].y < limR;
        const uint32_t inv = T.ballot(!vis);
      int L = inv ? __ffs(inv) - 1 : TW;          // first invisible lane in this group
      if (POLICY == SOLID_POLICY_SOLIDARITY && enf && f < 0) {
        // lane evaluates the barrier condition for index m = i - 1 (needs flagged(m) and the
        // owner of the NEXT entry i): stop at m iff flagged(m) and not (i visible and
        // owned by the requester).  Groups without flagged entries skip it (the common case).
        const uint32_t flm = T.ballot(fl);
        if (flm || carry_flag) {
          bool pf = T.shfl_up(fl, 1);
          if (lane == 0) pf = carry_flag;
          bool cond = false, gone = false, stale = false;
          if (pf && lane <= L && !(g == 0 && lane == 0)) {
            const uint32_t first =
                ((uint32_t)(pq[q].x >> 32) == tagS) ? 0u : (uint32_t)pq[q].x;
            bool pass = vis && (DIST ? kp.mown[idq[q]] : owner_from(kp, idq[q], first)) == u;
            if (!DIST && pass && first != 0u && kp.stamp) {
              // Inserter stamp: entry i passes the barrier because round t-1
              // says an earlier request of this user inserted it.  If that request has already
              // been evaluated in THIS round and now diverts at a depth <= i, it no longer
              // inserts the Shared key: take the entry as absent (stop here, divert at m).  A
              // guess like any Gauss-Seidel value; a request evaluated earlier in this round is
              // waited for (it is < j, so the wait chain ends).  Sound for certification: in a
              // round without changes the rule cannot fire (round t-1's inserter would not
              // have inserted the key either).
              const uint64_t ir = (uint64_t)first - 1u - kp.seq_base;
              if (ir >= kp.j_lo && ir < j) {
                unsigned long long v = ld_relaxed64(&kp.fst[ir]);
                if (may_defer && (uint32_t)(v >> 32) != tagW) {
                  // main pass (long requests): a short bounded wait (the inserter is being
                  // evaluated right now, typically in the round's first wave), then defer the
                  // request to the round's second pass, after a grid barrier.  Unbounded waits
                  // would chain (each request depending on the previous one) and serialise the
                  // round.  Short requests (two per warp) and the deferred pass never wait:
                  // a stale stamp is simply no information (the Jacobi value is used).
                  const unsigned long long t0 = globaltimer_ns();
                  while ((uint32_t)(v >> 32) != tagW && globaltimer_ns() - t0 < kp.stamp_wait_ns) {
                    __nanosleep(64);
                    v = ld_relaxed64(&kp.fst[ir]);
                  }
                  stale = (uint32_t)(v >> 32) != tagW;
                }
                const int32_t fi = (int32_t)(uint32_t)v;
                if ((uint32_t)(v >> 32) == tagW && fi >= 1 && (uint32_t)fi <= g + (uint32_t)lane) {
                  pass = false;
                  gone = true;
                }
#ifdef SOLID_COUNTERS
                if (t < 16) {
                  atomicAdd(&kp.st->cnt[t][8], gone ? 1ull : 0ull);
                  atomicAdd(&kp.st->cnt[t][9], 1ull);

                }
#endif
              }
            }
            cond = !pass;
          }
          const uint32_t cm = T.ballot(cond);
          if (cm) f = (int32_t)(g + (uint32_t)(__ffs(cm) - 1));   // 1-based depth = m + 1 = i
          if (!DIST) {
            if (T.ballot(stale)) {                     // nothing written yet: evaluate it later
              if (lane == 0) kp.dlist[atomicAdd(&kp.dcnt[t & 1], 1u)] = (uint32_t)j;
              return 2;
            }
            const uint32_t gm = T.ballot(gone);
            if (gm) L = min(L, __ffs(gm) - 1);         // the entry taken as absent ends the walk
          }
        }
        carry_flag = (flm >> (TW - 1)) & 1u;
      }
      if (L < TW) {
        k = g + (uint32_t)L;
        walked = true;
        break;
      }
    }
  }
  if (POLICY == SOLID_POLICY_USER_ISOLATION) f = 0;

  // ---- selective isolation: continue in Iso(u) rooted at S[f] (R3) ----
  uint32_t r = k, flagd = 0;
  if (POLICY == SOLID_POLICY_SOLIDARITY && f >= 1) {
    uint32_t m = n - (uint32_t)f;
    if (f == fprev) {
      // same divert depth as last round: the isolated keys of blocks f..n-1 are registered and
      // their ids cached in iso_id[] (created in an earlier round, so the staged state already
      // carries their index snapshot); the first group was prefetched above
      // kIsoG groups with their id and state loads in flight together (long isolated walks)
      bool stop = false;
      for (uint32_t g0 = (uint32_t)f; g0 < n && !stop; g0 += TW * kIsoG) {
        uint32_t idv[kIsoG];
        unsigned long long va[kIsoG], vb[kIsoG];
#pragma unroll
        for (int q = 0; q < kIsoG; ++q) {
          const uint32_t i = g0 + TW * q + lane;
          idv[q] = (i < n && !(q == 0 && g0 == (uint32_t)f)) ? iso_ids[i] : 0u;
        }
#pragma unroll
        for (int q = 0; q < kIsoG; ++q) {
          va[q] = vb[q] = ~0ull;
          if (idv[q]) {
            const Hot* h = kp.hot + idv[q];
            va[q] = ldw64(&h->v[2 * R]);
            vb[q] = ldw64(&h->v[2 - 2 * R]);
          }
        }
#pragma unroll
        for (int q = 0; q < kIsoG; ++q) {
          const uint32_t g = g0 + TW * q;
          if (g >= n) break;
          const uint32_t i = g + lane;
          const bool vis = (q == 0 && g0 == (uint32_t)f) ? (i < n && iso_pre_vis)
                                                          : (idv[q] && (va[q] < limR || vb[q] < limW));
          const uint32_t inv = T.ballot(!vis);
          if (inv) {
            m = g + (uint32_t)(__ffs(inv) - 1) - (uint32_t)f;
            stop = true;
            break;
          }
        }
      }
    } else {
      // new divert depth: derive I_f[b] = S[b] + sigma_u (G[b] - G[f]) for b > f, register every
      // key (find-or-insert) and cache its id; visibility = staged (earlier batch requests) or
      // present in the index snapshot
      const uint64_t sig = sigma_of(kp.seed, u);
      const uint64_t gf = kp.gtab[f];
      const uint64_t sig2 = kp.nc == 2 ? sigma2_of(kp.seed, u) : 0;
      const uint64_t gf2 = kp.nc == 2 ? kp.gtab2[f] : 0;
      bool found = false;
      for (uint32_t g = (uint32_t)f; g < n; g += TW) {
        const uint32_t i = g + lane;
        const bool valid = i < n;
        uint64_t key = 0;
        if (valid) key = iso_key(kp, blk0 + i, i, sig, gf, sig2, gf2);
        bool created, snap = false;
        const uint32_t id = scratch_register<TW>(kp, valid, key, seg, lane, created, &snap);
        bool bvis = false;
        if (valid) {
          iso_ids[i] = id;
          bvis = iso_visible(kp, id, R, limR, limW);
        }
        // lanes not visible through the staged state may still be in the index snapshot; probe
        // them in order, only until the first key that is absent (the walk stops there)
        uint32_t cand = T.ballot(valid && !bvis);
        while (!found && cand) {
          const int L = __ffs(cand) - 1;
          bool present = false;
          if (lane == L && !DIST) {   // sharded: unknown until pulled next round (invisible)
            if (created) {
              present = snap;
            } else {
              uint32_t ow, sr;
              uint64_t ip;
              present = index_find(kp, key, ow, sr, ip);
            }
          }
          present = T.shfl(present, L);
          if (present) {
            cand &= cand - 1;
          } else {
            m = g + (uint32_t)L - (uint32_t)f;
            found = true;
          }
        }
      }
    }
    r = (uint32_t)f + m;
  } else if (POLICY == SOLID_POLICY_SOLIDARITY && k >= 1) {
    // flag rule (R2): e_r = K[k] gets flagged iff owner != u and unflagged; applies with
    // isolation on or off (R11)
    if (lane == 0) {
      const uint32_t id = sh_ids[k - 1];
      const Hot* h = kp.hot + id;
      const ulonglong2 p0 = ldw128(&h->v[0]), p1 = ldw128(&h->v[2]);
      const uint32_t first = gs_first(p0.x, DIST ? ~0ull : p1.x, R, seqp, tagR, tagW, tagS);
      const bool flagged =
          gs_first(p0.y, DIST ? ~0ull : p1.y, R, seqp, tagR, tagW, tagS) != kNone;
      const uint32_t own = DIST ? kp.mown[id] : owner_from(kp, id, first);
      if (!flagged && own != u) {
        flagd = k;
        if (DIST)
          atomicMin(&kp.int_flg[id], ((unsigned long long)seqp << 32) | (unsigned long long)u);
        else
          atomic_min_u64(&kp.hot[id].v[2 * W + 1],
                         ((unsigned long long)tagW << 32) | (unsigned long long)seqp);
      }
    }
    flagd = T.shfl(flagd, 0);
  }

  // ---- staged inserts (seq-min scatter); APC / USER_ISOLATION are exact from round 0 ----
  if (POLICY == SOLID_POLICY_SOLIDARITY) {
    const unsigned long long mine = ((unsigned long long)tagW << 32) | (unsigned long long)seqp;
    const uint32_t* ids = (f >= 1) ? iso_ids : sh_ids;
    // fire-and-forget RED: within a round, concurrent inserters of one key are rare (a request
    // only inserts keys invisible to it), unlike the hot keys of K_A
    if (DIST) {
      const unsigned long long pk = ((unsigned long long)seqp << 32) | (unsigned long long)u;
      for (uint32_t i = r + lane; i < n; i += TW) atomicMin(&kp.int_ins[ids[i]], pk);
    } else {
      // ids already in registers need no dependent load: a request diverting at an unchanged
      // depth has blocks f..f+TW-1 in iso_pre_id (lane l = block f + l); a Shared one has the
      // last walked STEP blocks in idq (lane l of idq[q] = block wbase + TW q + l)
      const bool pre = POLICY == SOLID_POLICY_SOLIDARITY && f >= 1 && f == fprev;
      const bool shr = f < 0;
      for (uint32_t i0 = r; i0 < n; i0 += TW) {
        const uint32_t i = i0 + lane;
        uint32_t id = 0;
        if (pre && i0 < (uint32_t)f + TW) {
          const uint32_t v = T.shfl(iso_pre_id, (int)((i - (uint32_t)f) & (TW - 1)));
          if (i < n) id = i < (uint32_t)f + TW ? v : ids[i];
        } else if (shr && i0 >= wbase && i0 < wbase + STEP) {
          const uint32_t src = (i - wbase) & (TW - 1), q = (i - wbase) / TW;
          const uint32_t v0 = T.shfl(idq[0], (int)src);
          const uint32_t v1 = T.shfl(idq[1], (int)src);
          const uint32_t v2 = T.shfl(idq[2], (int)src);
          const uint32_t v3 = T.shfl(idq[3], (int)src);
          const uint32_t v = q == 0 ? v0 : q == 1 ? v1 : q == 2 ? v2 : v3;
          if (i < n) id = i < wbase + STEP ? v : ids[i];
        } else if (i < n) {
          id = ids[i];
        }
        if (i < n) atomicMin(&kp.hot[id].v[2 * W], mine);
      }
    }
  }

  const uint4 d = make_uint4(k, (uint32_t)f, r, flagd);
  const bool changed =
      t == 1 || prev.x != d.x || prev.y != d.y || prev.z != d.z || prev.w != d.w;
  if (!DIST && POLICY == SOLID_POLICY_SOLIDARITY && lane == 0)   // this round's stamp (every round)
    st_relaxed64(&kp.fst[j], ((unsigned long long)tagW << 32) | (uint32_t)f);
#ifdef SOLID_COUNTERS
  if (lane == 0 && t < 16) {
    unsigned long long* c = kp.st->cnt[t];
    atomicAdd(c + 0, 1ull);
    if (changed) atomicAdd(c + 1, 1ull);
    if (f >= 1 && f != fprev) atomicAdd(c + 2, 1ull);
    if (f >= 1 && f == fprev) atomicAdd(c + 3, 1ull);
    if (flagd) atomicAdd(c + 4, 1ull);
    atomicAdd(c + 5, (unsigned long long)(n - r));
    atomicAdd(c + 6, (unsigned long long)k);
    if (f >= 1) atomicAdd(c + 7, (unsigned long long)(r - (uint32_t)f));
  }
#endif
  if (lane == 0 && changed) {   // an unchanged decision already holds its result
    kp.dec[j] = d;
    const uint32_t kk = (POLICY == SOLID_POLICY_USER_ISOLATION) ? 0u : k;   // no Shared chain
    solid_result res;
    res.n_blocks = n;
    res.shared_hits = kk;
    res.reused = r;
    res.divert_at = f;
    res.flag_depth = flagd;
    res.bits = (r > 0 ? 1u : 0u) | ((n > 0 && r == n) ? 2u : 0u) | (f >= 0 ? 4u : 0u) |
               ((f >= 0 && (uint32_t)f < kk) ? 8u : 0u) | (flagd > 0 ? 16u : 0u);
    kp.out[j] = res;
  }
  return changed ? 1 : 0;
}

// A round's requests: all but the last `tail` sweeps (1) statically strided over the tiles
// (tile w takes w, w + nw, ...), the rest handed out one at a time from a per-round counter, so
// tiles whose requests ran long do not hold the whole grid at the round's barrier.
// (32-bit positions: a batch holds < 2^32 requests, max_batch_requests is checked at init.)
template <int TW, class F>
__device__ __forceinline__ void for_requests(const KParams& kp, uint32_t t, uint64_t w0,
                                             uint64_t nw, int tl, F&& eval) {
  if (TW == 16) {          // two requests per warp (short requests): plain strided loop (the
                           // dynamic tail measured neutral there and its state spills)
    for (uint64_t j = kp.j_lo + w0; j < kp.n; j += nw) eval(j);
    return;
  }
  const uint32_t total = (uint32_t)(kp.n - kp.j_lo), w = (uint32_t)w0, step = (uint32_t)nw;
  const uint32_t sweeps = total / step;
  const uint32_t dyn = (uint32_t)kp.tail;           // sweeps handed out dynamically (0: none)
  const uint32_t stat = !dyn ? total : sweeps > dyn ? (sweeps - dyn) * step : 0;
  for (uint32_t q = w; q < stat; q += step) eval(kp.j_lo + q);
  const Tile<TW> T;
  for (;;) {
    uint32_t q = 0;
    if (tl == 0) q = stat + atomicAdd(&kp.st->grab[t & 3], 1u);
    q = T.shfl(q, 0);
    if (q >= total) break;
    eval(kp.j_lo + q);
  }
}

// The resolver: all rounds in one persistent cooperative launch (grid = resident CTAs).  Tiles
// of TW lanes stride over the requests; between rounds a grid-wide barrier (which also
// invalidates L1, so the next round sees every atomic of this one).  Stops at the first round
// t >= 2 whose decisions all equal round t-1's, or after t_max.
template <int POLICY, int TW>
__device__ __forceinline__ void resolve_rounds(const KParams& kp, uint32_t t_max,
                                               uint32_t* s_changed) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int tl = lane & (TW - 1);                 // lane within the request's tile
  constexpr int LOG = TW == 32 ? 5 : 4;
  const uint64_t w0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> LOG;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> LOG;
  for (uint32_t t = 1; t <= t_max; ++t) {
    if (threadIdx.x == 0) *s_changed = 0;
    __syncthreads();
    bool any = false;
    // (long requests only: with two short requests per warp, C4, moving every new divert into
    // one round measured slower than the Jacobi order — 3.25 vs 2.18 ms for rounds 2 + 3)
    const bool stamps = POLICY == SOLID_POLICY_SOLIDARITY && kp.stamp && TW == 32;
    // main pass: every request; with the stamp rule, a deferred pass follows for the requests
    // whose inserter stamp was stale in the main pass, after a grid barrier,
    // when every main-pass stamp is published
    if (grid.thread_rank() == 0) {
      kp.st->grab[(t + 2) & 3] = 0;      // round t + 2's counter
      kp.dcnt[(t + 1) & 1] = 0;          // round t + 1's deferred list (last read in round t - 1)
    }
    bool synced = false;                 // the round's closing barrier was already passed
    if (stamps) {
      for_requests<TW>(kp, t, w0, nw, tl, [&](uint64_t j) {
        any |= eval_request<POLICY, false, TW, true>(kp, t, j, tl) == 1;
      });
      // the main pass's changes are published before the barrier: with nothing deferred it
      // closes the round (one grid barrier per round instead of two)
      if (tl == 0 && any) *s_changed = 1;
      __syncthreads();
      if (threadIdx.x == 0 && *s_changed) kp.st->changed[t] = kp.epoch;
      grid.sync();
      const uint32_t nd = *(volatile uint32_t*)&kp.dcnt[t & 1];
      synced = nd == 0;
#ifdef SOLID_COUNTERS
      const unsigned long long td0 = globaltimer_ns();
#endif
      for (uint64_t q = w0; q < nd; q += nw)
        any |= eval_request<POLICY, false, TW, false>(kp, t, kp.dlist[q], tl) == 1;
#ifdef SOLID_COUNTERS
      if (tl == 0 && t < 16) atomicMax(&kp.st->cnt[t][10], globaltimer_ns() - td0);
      if (grid.thread_rank() == 0 && t < 16) kp.st->cnt[t][11] = nd;
#endif
    } else {
      for_requests<TW>(kp, t, w0, nw, tl, [&](uint64_t j) {
        any |= eval_request<POLICY, false, TW, false>(kp, t, j, tl) == 1;
      });
    }
    // one store per CTA (100k same-address stores would serialise on one L2 slice)
    if (!synced) {
      if (tl == 0 && any) *s_changed = 1;
      __syncthreads();
      if (threadIdx.x == 0 && *s_changed) kp.st->changed[t] = kp.epoch;
    }
    if (POLICY != SOLID_POLICY_SOLIDARITY) {         // exact in one pass
      if (grid.thread_rank() == 0) kp.st->conv = 1;
      return;
    }
    // grid.sync(): bar.sync + release/acquire at gpu scope; the acquire path also invalidates
    // L1 (CCTL.IVALL in SASS), so the next round's weak loads see every write of this one
    if (!synced) grid.sync();
    if (grid.thread_rank() == 0 && t <= 16) kp.st->round_ns[t] = globaltimer_ns();
    // one L2 read per CTA, broadcast through shared memory
    __shared__ uint32_t s_ch, s_er;
    if (threadIdx.x == 0) {
      s_ch = *(volatile uint32_t*)&kp.st->changed[t] == kp.epoch;
      s_er = *(volatile uint32_t*)&kp.st->err;
    }
    __syncthreads();
    const uint32_t ch = s_ch, er = s_er;
    if ((t >= 2 && ch == 0) || er) {
      if (grid.thread_rank() == 0) kp.st->conv = (t >= 2 && ch == 0) ? t : 0;
      return;
    }
  }
}

// Tile width per batch, decided on the device (the host does not know the batch's tokens in the
// asynchronous paths): short requests (<= 64 blocks on average, e.g. C4) are resolved two per
// warp (TW = 16: twice the requests in flight at the same registers, -23 % on C4), long ones a
// warp each (a 16-lane tile needs twice the dependent walk steps: +20 % on C2 / C3).
template <int POLICY>
__global__ void __launch_bounds__(256, 4) k_resolve(KParams kp, uint32_t t_max, int tile) {
  if (blockIdx.x == 0 && threadIdx.x == 0) kp.st->round_ns[0] = globaltimer_ns();
  if (blockIdx.x == 0 && threadIdx.x < 32) {     // K_A's distinct keys (its index probes)
    const int lane = threadIdx.x;
    unsigned long long c = 0;
#pragma unroll
    for (int q = 0; q < kNSeg / 32; ++q) c += min(kp.seg_cnt[lane + 32 * q].v, kp.seg_cap);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) kp.st->ids_after_hash = c;
  }
  __shared__ uint32_t s_changed;
  bool half = tile == 16;
  if (tile == 0) {                                // auto: average full blocks per request
    const uint64_t T = kp.offsets[kp.n] - kp.offsets[kp.j_lo];
    half = T <= (uint64_t)64 * 16 * (kp.n - kp.j_lo);
  }
  if (half) resolve_rounds<POLICY, 16>(kp, t_max, &s_changed);
  else resolve_rounds<POLICY, 32>(kp, t_max, &s_changed);
}

// ---------------------------------------------------------------------------------------------
// K_C: commit, one thread per registered key (dense ids, coalesced).  In the converged state a
// key carrying the final round's tag was inserted by the request in its low 32 bits (the
// earliest one, "set exactly once"): it claims an index slot with one 128-bit CAS
// {key, owner, sharer}.  A snapshot entry whose flag carries the final tag gets its sharer
// written (a6).  k_stats ran first and counted the batch's new entries: on a capacity overflow
// (R9) it set st->overflow and nothing is claimed — so live + new <= capacity <= tcap / 2 holds
// for every claim and the linear probe always meets an EMPTY slot.  mode 2 rolls a committed
// batch back exactly (every claimed slot was EMPTY before: emptying it restores the chains).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t final_round(const KParams& kp) {
  return kp.st->conv == 0 ? 0 : (POLICY_IS_SOLIDARITY(kp) ? kp.st->conv : 0);
}

__global__ void __launch_bounds__(256, 5) k_commit(KParams kp, int mode) {
  constexpr int U = 4;                 // ids per thread, staged so all loads are in flight at once
  uint32_t n_ins = 0, n_flg = 0;       // fast_commit: this thread's new entries / sharer writes
  // the converged round is read on the device (lookup never waits for the host); an invalid,
  // unconverged or over-capacity batch commits nothing
  if (kp.st->err || (kp.n && kp.st->conv == 0)) return;
  if (mode == 1 && kp.st->overflow) return;
  const uint32_t tf = final_round(kp);
  const uint32_t seg = blockIdx.y;
  const uint32_t cnt = min(kp.seg_cnt[seg].v, kp.seg_cap);
  const int W = (int)(tf & 1);
  const uint32_t tag = tag_of(kp.epoch, tf), tagS = tag_of(kp.epoch, kSubSnap);
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t x0 = blockIdx.x * blockDim.x + threadIdx.x; x0 < cnt; x0 += U * stride) {
    ulonglong2 pw[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const uint32_t x = x0 + q * stride;
      pw[q] = x < cnt ? ldw128(&kp.hot[seg * kp.seg_cap + x + 1].v[2 * W])
                      : make_ulonglong2(~0ull, ~0ull);
    }
    uint64_t key[U];
    uint32_t who[U], sharer[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const uint32_t id = seg * kp.seg_cap + x0 + q * stride + 1;
      const uint32_t itag = (uint32_t)(pw[q].x >> 32);
      const bool ins = itag == tag, flg = itag == tagS && (uint32_t)(pw[q].y >> 32) == tag;
      key[q] = 0;
      who[q] = kNone;
      sharer[q] = kNone;
      if (ins) {
        key[q] = kp.cold[id].key;
        who[q] = kp.users[(uint32_t)pw[q].x - 1u];
        if ((uint32_t)(pw[q].y >> 32) == tag) sharer[q] = kp.users[(uint32_t)pw[q].y - 1u];
      } else if (flg) {
        who[q] = kp.users[(uint32_t)pw[q].y - 1u];
      }
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const uint32_t id = seg * kp.seg_cap + x0 + q * stride + 1;
      const uint32_t itag = (uint32_t)(pw[q].x >> 32);
      if (itag == tag) {
        Cold* c = kp.cold + id;
        ++n_ins;
        if (mode == 1 && kp.pool_cnt) atomicAdd(&kp.pool_cnt[(uint32_t)pw[q].x - 1u], 1u);
        if (mode == 1) {
          const ulonglong2 val =
              make_ulonglong2(key[q], (unsigned long long)who[q] | ((unsigned long long)sharer[q] << 32));
          uint64_t p = key[q] & kp.tmask;
          for (;;) {   // terminates: at most capacity <= tcap / 2 slots are live (k_stats)
            const ulonglong2 old = atomic_cas128(&kp.tab[p], make_ulonglong2(0ull, 0ull), val);
            if (old.x == 0 || old.x == key[q]) break;
            p = (p + 1) & kp.tmask;
          }
          c->psl = (uint32_t)p;
        } else {
          kp.tab[c->psl] = make_ulonglong2(0ull, 0ull);
        }
      } else if (itag == tagS && (uint32_t)(pw[q].y >> 32) == tag) {
        uint32_t* sharer_word = reinterpret_cast<uint32_t*>(&kp.tab[kp.cold[id].psl].y) + 1;
        ++n_flg;
        if (mode == 1) atomicCAS(sharer_word, kNone, who[q]);
        else atomicCAS(sharer_word, who[q], kNone);
      }
    }
  }
  // fast_commit (k_stats skipped its count: this batch cannot overflow): the commit counts the
  // batch's new entries and sharer writes itself (k_live then advances the live count)
  if (mode != 1 || !kp.st->fast_commit) return;
  for (int o = 16; o; o >>= 1) {       // one reduction per warp (no CTA barrier: registers)
    n_ins += __shfl_xor_sync(0xffffffffu, n_ins, o);
    n_flg += __shfl_xor_sync(0xffffffffu, n_flg, o);
  }
  if ((threadIdx.x & 31) == 0) {       // per-segment counters: no hot same-address atomics
    if (n_ins) atomicAdd(&kp.seg_new[2 * seg], n_ins);
    if (n_flg) atomicAdd(&kp.seg_new[2 * seg + 1], n_flg);
  }
}

// After k_commit, fast_commit only: the batch's new entries / sharer writes from k_commit's
// per-segment counts; live += new entries.
__global__ void k_live(DevStatus* st, unsigned long long* live, const uint32_t* seg_new) {
  if (!st->fast_commit) return;
  const int q = threadIdx.x;           // kNSeg threads
  unsigned long long a = seg_new[2 * q], b = seg_new[2 * q + 1];
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __shared__ unsigned long long s_a[kNSeg / 32], s_b[kNSeg / 32];
  if ((q & 31) == 0) {
    s_a[q >> 5] = a;
    s_b[q >> 5] = b;
  }
  __syncthreads();
  if (q) return;
  a = b = 0;
  for (int w = 0; w < kNSeg / 32; ++w) {
    a += s_a[w];
    b += s_b[w];
  }
  st->new_entries = a;
  st->new_flags = b;
  *live += a;
  st->live_after = *live;
}

// K_D, before the commit: per-batch sums over the results (block-weighted hit rate) and
// the batch's new entries / new flags counted from the converged staged state (one 16-byte read
// per key id).  With `live` set, the last CTA takes the capacity decision (R9): live + new >
// capacity -> st->overflow (k_commit then claims nothing, the batch fails with
// SOLID_ERR_CAPACITY), else live += new.  The live count stays resident on the device.
__global__ void __launch_bounds__(256) k_stats(const solid_result* out, uint64_t n,
                                               DevStatus* st, unsigned long long* live,
                                               unsigned long long cap, const SegCounter* seg,
                                               KParams kp) {
  if (blockIdx.x == 0 && threadIdx.x < kNSeg) {
    st->seg[threadIdx.x] = seg[threadIdx.x].v;
    if (kp.seg_new) {
      kp.seg_new[2 * threadIdx.x] = 0;   // k_commit's per-segment counts (fast_commit)
      kp.seg_new[2 * threadIdx.x + 1] = 0;
    }
  }
  unsigned long long a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const solid_result r = out[j];
    a[0] += r.n_blocks;
    a[1] += r.reused;
    a[2] += (r.bits >> 4) & 1;
    a[3] += (r.bits >> 2) & 1;
    a[4] += (r.bits >> 3) & 1;
    a[5] += 1;
  }
  const bool ok = live && !st->err && !(n && st->conv == 0);
  bool fast = false;
  if (ok) {                            // new entries (a[6]) and new sharer writes (a[7])
    // flat index over every registered id: segment prefix sums in shared memory, so each thread
    // handles ~ids / threads ids with independent loads (no per-segment serial loop)
    __shared__ uint32_t s_pre[kNSeg + 1];
    if (threadIdx.x < kNSeg) s_pre[threadIdx.x + 1] = min(seg[threadIdx.x].v, kp.seg_cap);
    if (threadIdx.x == 0) s_pre[0] = 0;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int q = 1; q <= kNSeg; ++q) s_pre[q] += s_pre[q - 1];
    __syncthreads();
    const uint32_t tf = final_round(kp);
    const int W = (int)(tf & 1);
    const uint32_t tag = tag_of(kp.epoch, tf), tagS = tag_of(kp.epoch, kSubSnap);
    const uint32_t total = s_pre[kNSeg];
    // every new entry has a registered id: when even all of them fit, the batch cannot
    // overflow — skip this counting pass; k_commit counts while it claims (fast_commit)
    fast = *(volatile unsigned long long*)live + total <= cap;
    constexpr int UQ = 4;                    // ids per thread per step, loads in flight together
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t g0 = blockIdx.x * blockDim.x + threadIdx.x; g0 < (fast ? 0u : total);
         g0 += UQ * stride) {
      ulonglong2 pw[UQ];
#pragma unroll
      for (int q = 0; q < UQ; ++q) {
        const uint32_t g = g0 + q * stride;
        pw[q] = make_ulonglong2(0ull, 0ull);
        if (g < total) {
          uint32_t lo = 0, hi = kNSeg;       // segment: s_pre[lo] <= g < s_pre[lo + 1]
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (s_pre[mid] <= g) lo = mid; else hi = mid;
          }
          pw[q] = ldw128(&kp.hot[lo * kp.seg_cap + (g - s_pre[lo]) + 1].v[2 * W]);
        }
      }
#pragma unroll
      for (int q = 0; q < UQ; ++q) {
        const uint32_t itag = (uint32_t)(pw[q].x >> 32);
        a[6] += itag == tag;
        a[7] += itag == tagS && (uint32_t)(pw[q].y >> 32) == tag;
      }
    }
  }
  __shared__ unsigned long long s_a[8];
  if (threadIdx.x < 8) s_a[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    for (int o = 16; o; o >>= 1) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
    if ((threadIdx.x & 31) == 0 && a[q]) atomicAdd(&s_a[q], a[q]);
  }
  __syncthreads();
  if (threadIdx.x < 6 && s_a[threadIdx.x]) atomicAdd(&st->sums[threadIdx.x], s_a[threadIdx.x]);
  if (threadIdx.x == 6 && s_a[6]) atomicAdd(&st->new_entries, s_a[6]);
  if (threadIdx.x == 7 && s_a[7]) atomicAdd(&st->new_flags, s_a[7]);
  if (!live) return;
  __shared__ bool s_last;
  __threadfence();                     // this CTA's sums are visible before it is counted done
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&st->blocks_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  if (ok && fast) {
    st->fast_commit = 1;               // k_commit counts (seg_new), k_live advances live
  } else if (ok) {
    const unsigned long long l = *live, add = *(volatile unsigned long long*)&st->new_entries;
    if (l + add > cap) st->overflow = 1;
    else *live = l + add;
  }
  st->live_after = *live;
}

// Compact the live index slots (dump): warp-aggregated append.
__global__ void __launch_bounds__(256) k_compact(const ulonglong2* tab, uint64_t tcap,
                                                 ulonglong2* out, unsigned long long* cnt,
                                                 unsigned long long cap) {
  const int lane = threadIdx.x & 31;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < tcap;
       base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    ulonglong2 e = make_ulonglong2(0, 0);
    if (i < tcap) e = tab[i];
    const uint32_t m = __ballot_sync(0xffffffffu, e.x != 0);
    if (!m) continue;
    unsigned long long b = 0;
    if (lane == __ffs(m) - 1) b = atomicAdd(cnt, (unsigned long long)__popc(m));
    b = __shfl_sync(0xffffffffu, b, __ffs(m) - 1);
    if (e.x) {
      const unsigned long long o = b + __popc(m & ((1u << lane) - 1u));
      if (o < cap) out[o] = e;
    }
  }
}

__global__ void k_fill_u64(unsigned long long* p, uint64_t n, unsigned long long v) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace solid

// =============================================================================================
// Host runtime
// =============================================================================================
using namespace solid;

constexpr uint32_t kRing = SOLID_MAX_INFLIGHT;   // asynchronous batches in flight per context
constexpr uint32_t kHostChunks = 4;              // host admission: sub-batches of a large batch
constexpr uint32_t kHostChunksMax = 16;          // (SOLID_HOST_CHUNKS, A/B only)
struct HostSlot {               // pinned host mirror of one batch's status
  DevStatus st;
};
struct Flight {                 // one batch in flight: events hash|resolve|commit|done
  cudaEvent_t ev[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  uint64_t n = 0, launches = 0, gen = 0;
};

struct solid_ctx {
  solid_config cfg{};
  int dev = 0;
  bool poisoned = false;
  bool pending = false;
  std::string err;
  // index
  ulonglong2* tab = nullptr;
  uint64_t tcap = 0;
  uint64_t live = 0;
  ulonglong2* tab_ckpt = nullptr;
  uint64_t live_ckpt = 0;
  // batch scratch
  ulonglong2* stab = nullptr;
  uint64_t scap = 0;
  Hot* hot = nullptr;
  Cold* cold = nullptr;
  uint64_t idcap = 0;
  uint32_t* id_of_block = nullptr;
  uint32_t* iso_id = nullptr;
  uint64_t slot_cap = 0;
  uint4* dec = nullptr;
  unsigned long long* fst = nullptr;
  int stamp_rule = 1;
  int tail = 1;                  // resolver: sweeps handed out dynamically per round (SOLID_TAIL)
  unsigned commit_gx = 16;       // k_commit CTAs per id segment (SOLID_COMMIT_GX)
  uint32_t stamp_wait_ns = kStampWaitNs;
  uint32_t* dlist = nullptr;
  uint32_t* dcnt = nullptr;
  int pack = 1;                          // packed K_A for short requests (SOLID_PACK=0: off)
  uint32_t* pk_pre = nullptr;
  uint32_t* pk_ctot = nullptr;
  uint32_t* pk_cpre = nullptr;
  uint32_t* pk_wfirst = nullptr;
  uint32_t pk_grid = 0;                  // its cooperative grid (resident CTAs)
  int pack_hint = 1;                     // the last collected batch took the packed K_A
  uint32_t pack_probe = 0;               // batches since the packed kernel was last launched
  uint64_t pack_last_n = 0;              // batch size at the last launch decision
  SegCounter* seg_cnt = nullptr;
  uint32_t seg_cap = 0;
  DevStatus* st = nullptr;
  DevStatus* st_host = nullptr;   // pinned mirror (the current slot's)
  uint32_t* seg_host = nullptr;   // pinned per-segment id counts (the current slot's)
  cudaEvent_t* ev = nullptr;      // the current slot's events
  unsigned long long* mpow = nullptr;
  unsigned long long* gtab = nullptr;
  uint32_t klo[kBS], khi[kBS];
  // H-def v3 second component (hash_components == 2)
  int nc = 1;
  unsigned long long* mpow2 = nullptr;
  unsigned long long* gtab2 = nullptr;
  ulonglong2* cs = nullptr;
  uint32_t klo2[kBS], khi2[kBS];
  uint32_t epoch = 0;
  // pending batch
  KParams kp{};
  uint32_t tf = 0;
  uint32_t rounds = 0;
  uint32_t max_rounds = kMaxRounds;      // resolver round limit (solid_debug_set_max_rounds)
  int resolve_tw = 0;                    // resolver lanes per request: 0 auto (SOLID_RESOLVE_TILE)
  bool split_last = false;               // the last batch was committed in parts (non-convergence)
  cudaStream_t stream = nullptr;
  // host-buffer admission staging
  uint32_t* h_tokens = nullptr;
  uint16_t* h_tokens16 = nullptr;
  cudaStream_t s_copy = nullptr;               // host admission: token copies of later chunks
  cudaEvent_t ev_chunk[kHostChunksMax + 1] = {};
  uint32_t host_chunks = kHostChunks;
  uint64_t* h_offsets = nullptr;
  uint32_t* h_users = nullptr;
  uint8_t* h_enforce = nullptr;
  solid_result* h_out = nullptr;
  // stats
  solid_stats_t stats{};
  uint64_t launches = 0;
  uint64_t resolve_ctas = 0;
  unsigned long long* live_dev = nullptr;   // live count for the asynchronous admission path
  uint32_t* seg_new = nullptr;               // [kNSeg][2] fast-commit counts (k_commit)
  // batches in flight: a ring of kRing status slots (pinned host mirrors + events); the
  // asynchronous ones wait in [head, head + outstanding) for solid_batch_status
  HostSlot* slots = nullptr;
  Flight fl[kRing];
  uint32_t head = 0, outstanding = 0, cur = 0;
  // evict-mode / block-table contexts: solid_admit_batch admits at submission (lookup + insert,
  // the host-driven parts of those paths included); the statuses wait here, oldest first, for
  // solid_batch_status (same ring limit and collection rules as the asynchronous batches)
  std::deque<std::pair<solid_status, std::string>> done_q;
  uint64_t gen = 0;                         // reset generation
  // sharded mode (solid_dist.inc)
  struct Dist* dist = nullptr;
  struct P2P* p2p = nullptr;       // sharded: peer-memory exchange (solid_p2p.inc)
  uint64_t last_add = 0;
  // LRU eviction mode (solid_evict.inc)
  struct Evict* ev_state = nullptr;
  struct Pool* pool = nullptr;     // block_table: physical blocks + block tables (solid_pool.inc)
  uint32_t* pool_cnt = nullptr;    // its per-request new-entry counts (filled by k_commit)
  uint32_t* long_q = nullptr;      // K_A long-request queue (max_batch_requests entries)
};

static void set_slot(solid_ctx* c, uint32_t i) {
  c->cur = i;
  c->st_host = &c->slots[i].st;
  c->seg_host = c->slots[i].st.seg;
  c->ev = c->fl[i].ev;
}

static uint64_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

static solid_status fail(solid_ctx* c, solid_status s, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (s == SOLID_ERR_CUDA) c->poisoned = true;
  }
  return s;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, SOLID_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

extern "C" uint32_t solid_abi_version(void) { return SOLID_ABI_VERSION; }

extern "C" const char* solid_last_error(const solid_ctx* ctx) {
  return ctx ? ctx->err.c_str() : "null context";
}

static void evict_free(solid_ctx* ctx);
static solid_status evict_init(solid_ctx* ctx);
static solid_status evict_lookup(solid_ctx* ctx, cudaStream_t s);
static solid_status evict_insert(solid_ctx* ctx, cudaStream_t s);
static solid_status evict_reset(solid_ctx* ctx, cudaStream_t s);
static solid_status evict_scratch_reset(solid_ctx* ctx, cudaStream_t s);
static solid_status evict_checkpoint(solid_ctx* ctx);
static solid_status evict_restore(solid_ctx* ctx);
static void pool_free(solid_ctx* ctx);
static void p2p_free(solid_ctx* ctx);
static void p2p_direct_targets(solid_ctx* ctx);
static solid_status pool_init(solid_ctx* ctx);
static solid_status pool_reset(solid_ctx* ctx, cudaStream_t s);
static solid_status pool_pre(solid_ctx* ctx, cudaStream_t s, uint32_t tf);
static solid_status pool_commit(solid_ctx* ctx, cudaStream_t s, uint32_t tf, uint64_t new_entries,
                                uint64_t evicted, uint64_t ebound);
static solid_status pool_checkpoint(solid_ctx* ctx);
static void pool_invalidate(solid_ctx* ctx);
static solid_status pool_restore(solid_ctx* ctx);

static void free_all(solid_ctx* c) {
  p2p_free(c);
  evict_free(c);
  pool_free(c);
  cudaFree(c->tab);
  cudaFree(c->tab_ckpt);
  cudaFree(c->stab);
  cudaFree(c->hot);
  cudaFree(c->cold);
  cudaFree(c->id_of_block);
  cudaFree(c->iso_id);
  cudaFree(c->dec);
  cudaFree(c->fst);
  cudaFree(c->dlist);
  cudaFree(c->dcnt);
  cudaFree(c->pk_pre);
  cudaFree(c->pk_ctot);
  cudaFree(c->pk_cpre);
  cudaFree(c->pk_wfirst);
  cudaFree(c->seg_cnt);
  cudaFree(c->st);
  cudaFree(c->live_dev);
  cudaFree(c->seg_new);
  cudaFree(c->mpow);
  cudaFree(c->gtab);
  cudaFree(c->long_q);
  cudaFree(c->mpow2);
  cudaFree(c->gtab2);
  cudaFree(c->cs);
  cudaFree(c->h_tokens);
  cudaFree(c->h_tokens16);
  for (auto& e : c->ev_chunk)
    if (e) cudaEventDestroy(e);
  if (c->s_copy) cudaStreamDestroy(c->s_copy);
  cudaFree(c->h_offsets);
  cudaFree(c->h_users);
  cudaFree(c->h_enforce);
  cudaFree(c->h_out);
  if (c->slots) cudaFreeHost(c->slots);
  for (auto& f : c->fl)
    for (auto& e : f.ev)
      if (e) cudaEventDestroy(e);
}

// (Re)initialise the batch scratch: key table stale, staged states at +inf.
static solid_status init_scratch(solid_ctx* ctx, cudaStream_t s) {
  CK(cudaMemsetAsync(ctx->stab, 0, ctx->scap * sizeof(ulonglong2), s));
  k_fill_u64<<<4096, 256, 0, s>>>(reinterpret_cast<unsigned long long*>(ctx->hot),
                                  ctx->idcap * (sizeof(Hot) / 8), ~0ull);
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(ctx->seg_cnt, 0, kNSeg * sizeof(SegCounter), s));
  if (ctx->st) CK(cudaMemsetAsync(ctx->st, 0, sizeof(DevStatus), s));   // changed[] is epoch-tagged
  if (ctx->ev_state) {                       // id publication words carry the epoch
    solid_status rc = evict_scratch_reset(ctx, s);
    if (rc != SOLID_OK) return rc;
  }
  ctx->epoch = 0;
  return SOLID_OK;
}

static void dist_free(solid_ctx* ctx);
static solid_status dist_init(solid_ctx* ctx, uint32_t world, uint32_t rank);

extern "C" solid_status solid_init(const solid_config* cfg, solid_ctx** out) {
  solid_ctx* ctx = nullptr;
  if (!cfg || !out) return SOLID_ERR_INVALID;
  *out = nullptr;
  if (cfg->block_size != kBS || cfg->max_blocks == 0 || cfg->max_blocks > (1u << 24) ||
      cfg->capacity_blocks == 0 || cfg->max_batch_requests == 0 ||
      cfg->max_batch_requests >= 0xFFFFFFF0ull || cfg->policy < 0 || cfg->policy > 2)
    return SOLID_ERR_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev)
    return SOLID_ERR_INVALID;
  const uint32_t world = cfg->world ? cfg->world : 1;
  if (world > 64 || cfg->rank >= world) return SOLID_ERR_INVALID;
  if (cfg->evict > 1 || (cfg->evict && (world != 1 || cfg->capacity_blocks < cfg->max_blocks)))
    return SOLID_ERR_INVALID;
  if (cfg->hash_components > 2) return SOLID_ERR_INVALID;
  if (cfg->block_table > 1 || (cfg->block_table && world != 1)) return SOLID_ERR_INVALID;
  if (cfg->pin > 1 || (cfg->pin && !cfg->block_table)) return SOLID_ERR_INVALID;
  ctx = new solid_ctx();
  ctx->cfg = *cfg;
  ctx->cfg.world = world;
  ctx->dev = cfg->device;
  if (const char* e = getenv("SOLID_STAMP")) ctx->stamp_rule = atoi(e) != 0;
  if (const char* e = getenv("SOLID_TAIL")) ctx->tail = std::max(0, atoi(e));
  if (const char* e = getenv("SOLID_COMMIT_GX")) {
    const int v = atoi(e);
    if (v >= 1 && v <= 64) ctx->commit_gx = (unsigned)v;
  }
  if (const char* e = getenv("SOLID_HOST_CHUNKS")) {
    const int v = atoi(e);
    if (v >= 1 && v <= (int)kHostChunksMax) ctx->host_chunks = (uint32_t)v;
  }
  if (const char* e = getenv("SOLID_PACK")) ctx->pack = atoi(e) != 0;
  if (const char* e = getenv("SOLID_STAMP_WAIT")) ctx->stamp_wait_ns = (uint32_t)atoi(e);
  if (const char* e = getenv("SOLID_RESOLVE_TILE")) {
    const int v = atoi(e);
    ctx->resolve_tw = (v == 16 || v == 32) ? v : 0;
  }
  CK(cudaSetDevice(ctx->dev));
  // evict mode: 4x headroom so the tombstones of ~C/4 evictions fit between rebuilds
  ctx->tcap = next_pow2(std::max<uint64_t>((cfg->evict ? 4 : 2) * cfg->capacity_blocks, 1024));
  ctx->slot_cap = cfg->max_batch_tokens / kBS + 1;
  // distinct keys per batch <= Shared keys + isolated keys of every divert depth tried; ids are
  // allocated from kNSeg segments chosen by request (j mod kNSeg), each with headroom over an
  // even share: 2x for small batches, 1.25x once a segment's share is large (the requests of a
  // big batch spread evenly; C5's 4e9 tokens would otherwise need 60 GB of id state)
  ctx->idcap = std::max<uint64_t>(2 * ctx->slot_cap, 1u << 16);
  const uint64_t share = ctx->idcap / kNSeg;
  ctx->seg_cap = (uint32_t)std::min<uint64_t>(
      (share >= (1u << 20) ? share + share / 4 : 2 * share) + 1024, 0x7FFFFFFFull);
  ctx->idcap = (uint64_t)kNSeg * ctx->seg_cap + 1;
  ctx->scap = next_pow2(2 * ctx->idcap);
  if (ctx->tcap > (1ull << 32) || ctx->idcap > (1ull << 32)) {   // 32-bit slot / id indices
    delete ctx;
    return SOLID_ERR_INVALID;
  }
  const uint64_t mb = cfg->max_blocks;
  auto alloc = [&](void** p, size_t bytes) -> bool { return cudaMalloc(p, bytes) == cudaSuccess; };
  bool ok = alloc((void**)&ctx->tab, ctx->tcap * sizeof(ulonglong2)) &&
            alloc((void**)&ctx->stab, ctx->scap * sizeof(ulonglong2)) &&
            alloc((void**)&ctx->hot, ctx->idcap * sizeof(Hot)) &&
            alloc((void**)&ctx->cold, ctx->idcap * sizeof(Cold)) &&
            alloc((void**)&ctx->id_of_block, ctx->slot_cap * sizeof(uint32_t)) &&
            alloc((void**)&ctx->iso_id, ctx->slot_cap * sizeof(uint32_t)) &&
            alloc((void**)&ctx->dec, cfg->max_batch_requests * sizeof(uint4)) &&
            alloc((void**)&ctx->fst, std::max<uint64_t>(cfg->max_batch_requests, 1) * sizeof(unsigned long long)) &&
            alloc((void**)&ctx->dlist, std::max<uint64_t>(cfg->max_batch_requests, 1) * sizeof(uint32_t)) &&
            alloc((void**)&ctx->dcnt, 2 * sizeof(uint32_t)) &&
            alloc((void**)&ctx->pk_pre, (cfg->max_batch_requests + 2) * sizeof(uint32_t)) &&
            alloc((void**)&ctx->pk_ctot, 8192 * sizeof(uint32_t)) &&
            alloc((void**)&ctx->pk_cpre, 8193 * sizeof(uint32_t)) &&
            alloc((void**)&ctx->pk_wfirst, (ctx->slot_cap / kPackSpan + 4) * sizeof(uint32_t)) &&
            alloc((void**)&ctx->seg_cnt, kNSeg * sizeof(SegCounter)) &&
            alloc((void**)&ctx->st, sizeof(DevStatus)) &&
            alloc((void**)&ctx->live_dev, sizeof(unsigned long long)) &&
            alloc((void**)&ctx->seg_new, 2 * kNSeg * sizeof(uint32_t)) &&
            alloc((void**)&ctx->mpow, mb * sizeof(unsigned long long)) &&
            alloc((void**)&ctx->gtab, (mb + 1) * sizeof(unsigned long long)) &&
            alloc((void**)&ctx->long_q, (cfg->max_batch_requests + 1) * sizeof(uint32_t)) &&
            cudaMallocHost((void**)&ctx->slots, kRing * sizeof(HostSlot)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    free_all(ctx);
    delete ctx;
    return SOLID_ERR_OOM;
  }
  // H-def v2 constants, computed by this library's own host code.
  const uint64_t B = (1ull << 32) + splitmix64(cfg->hash_seed) % (kP - (1ull << 33));
  uint64_t pw = 1;
  for (uint32_t i = 0; i < kBS; ++i) {
    ctx->klo[i] = (uint32_t)pw;
    ctx->khi[i] = (uint32_t)(pw >> 32);
    pw = mulmod_host(pw, B);
  }
  const uint64_t M = pw;
  std::vector<unsigned long long> mp(mb), g(mb + 1);
  uint64_t x = 1;
  g[0] = 0;
  for (uint64_t i = 0; i < mb; ++i) {
    mp[i] = x;
    g[i + 1] = addmod(g[i], x);
    x = mulmod_host(x, M);
  }
  CK(cudaMemcpy(ctx->mpow, mp.data(), mb * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->gtab, g.data(), (mb + 1) * 8, cudaMemcpyHostToDevice));
  if (cfg->hash_components == 2) {   // H-def v3 second component: base B2, its own tables
    ctx->nc = 2;
    const uint64_t B2 = (1ull << 32) + splitmix64(cfg->hash_seed ^ kSeed2Salt) % (kP - (1ull << 33));
    uint64_t p2 = 1;
    for (uint32_t i = 0; i < kBS; ++i) {
      ctx->klo2[i] = (uint32_t)p2;
      ctx->khi2[i] = (uint32_t)(p2 >> 32);
      p2 = mulmod_host(p2, B2);
    }
    const uint64_t M2 = p2;
    uint64_t y = 1;
    g[0] = 0;
    for (uint64_t i = 0; i < mb; ++i) {
      mp[i] = y;
      g[i + 1] = addmod(g[i], y);
      y = mulmod_host(y, M2);
    }
    CK(cudaMalloc(&ctx->mpow2, mb * 8));
    CK(cudaMalloc(&ctx->gtab2, (mb + 1) * 8));
    CK(cudaMalloc(&ctx->cs, ctx->idcap * sizeof(ulonglong2)));
    CK(cudaMemcpy(ctx->mpow2, mp.data(), mb * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->gtab2, g.data(), (mb + 1) * 8, cudaMemcpyHostToDevice));
  }
  CK(cudaMemset(ctx->tab, 0, ctx->tcap * sizeof(ulonglong2)));
  solid_status rc = init_scratch(ctx, 0);
  if (rc != SOLID_OK) return rc;
  CK(cudaMemset(ctx->st, 0, sizeof(DevStatus)));
  CK(cudaMemset(ctx->live_dev, 0, sizeof(unsigned long long)));
  for (auto& f : ctx->fl)
    for (auto& e : f.ev) CK(cudaEventCreate(&e));
  set_slot(ctx, 0);
  if (cfg->evict) {
    rc = evict_init(ctx);
    if (rc != SOLID_OK) {
      free_all(ctx);
      delete ctx;
      return rc;
    }
  }
  if (cfg->block_table) {
    rc = pool_init(ctx);
    if (rc != SOLID_OK) {
      free_all(ctx);
      delete ctx;
      return rc;
    }
  }
  if (world > 1) {
    rc = dist_init(ctx, world, cfg->rank);
    if (rc != SOLID_OK) {
      dist_free(ctx);
      free_all(ctx);
      delete ctx;
      return rc;
    }
  }
  CK(cudaDeviceSynchronize());
  *out = ctx;
  return SOLID_OK;
}

extern "C" solid_status solid_destroy(solid_ctx* ctx) {
  if (!ctx) return SOLID_ERR_INVALID;
  cudaSetDevice(ctx->dev);
  cudaDeviceSynchronize();
  p2p_free(ctx);
  dist_free(ctx);
  free_all(ctx);
  delete ctx;
  return SOLID_OK;
}

static unsigned grid_for_warps(uint64_t warps) {
  return (unsigned)((warps * 32 + 255) / 256);
}

// Persistent cooperative launch of the resolver: one CTA per resident slot (all co-resident).
static solid_status launch_resolve(solid_ctx* ctx, cudaStream_t s) {
  const void* fn;
  switch (ctx->cfg.policy) {
    case SOLID_POLICY_APC: fn = (const void*)k_resolve<SOLID_POLICY_APC>; break;
    case SOLID_POLICY_USER_ISOLATION: fn = (const void*)k_resolve<SOLID_POLICY_USER_ISOLATION>; break;
    default: fn = (const void*)k_resolve<SOLID_POLICY_SOLIDARITY>; break;
  }
  if (!ctx->resolve_ctas) {           // co-resident CTAs (queried once per context)
    int per_sm = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->dev));
    ctx->resolve_ctas = (uint64_t)per_sm * sms;
  }
  const uint64_t need = ((ctx->kp.n - ctx->kp.j_lo) * 32 + 255) / 256;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ctx->resolve_ctas, need));
  uint32_t tmax = ctx->max_rounds;
  int tile = ctx->resolve_tw;
  void* args[] = {(void*)&ctx->kp, (void*)&tmax, (void*)&tile};
  CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), args, 0, s));
  return SOLID_OK;
}

static void launch_commit(solid_ctx* c, int mode, cudaStream_t s) {
  // 16 CTAs per id segment (SOLID_COMMIT_GX): fewer CTAs looked faster when the index is
  // restored from a checkpoint before each batch (scripts/ab_resolve.py) but are slower in the
  // bench, whose index is reset (C2 commit 0.079 ms with 16, 0.090-0.092 with 6 or 8,
  // profiles/r02/commit_grid_bench_ab.txt)
  k_commit<<<dim3(c->commit_gx, kNSeg), 256, 0, s>>>(c->kp, mode);   // 4 staged ids per thread
  if (mode == 1) k_live<<<1, kNSeg, 0, s>>>(c->st, c->live_dev, c->seg_new);
}

// Validates the batch and prepares the kernel parameters of a lookup (no kernel launched yet).
static solid_status admit_range(solid_ctx* ctx, uint64_t lo, uint64_t hi, cudaStream_t s);
static solid_status lookup_resolve(solid_ctx* ctx, cudaStream_t s);

static solid_status lookup_setup(solid_ctx* ctx, const solid_batch* b, solid_result* out,
                                 void* stream) {
  if (ctx->poisoned) return fail(ctx, SOLID_ERR_STATE, "context poisoned by an earlier failure");
  if (ctx->pending) return fail(ctx, SOLID_ERR_STATE, "lookup_batch twice without insert_batch");
  if (ctx->dist) return fail(ctx, SOLID_ERR_STATE, "sharded context: use the solid_dist_* calls");
  if (!b || (b->n_requests && (!b->tokens || !b->offsets || !b->users || !out)) || !b->offsets)
    return fail(ctx, SOLID_ERR_INVALID, "null batch pointer");
  if (b->n_requests > ctx->cfg.max_batch_requests)
    return fail(ctx, SOLID_ERR_INVALID, "n_requests > max_batch_requests");
  if (((uintptr_t)b->tokens & 3) != 0) return fail(ctx, SOLID_ERR_INVALID, "tokens not 4-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(ctx->dev));
  ctx->stream = s;
  if (ctx->epoch + 1 > kMaxEpoch) {     // tag space exhausted: re-initialise the scratch
    solid_status rc = init_scratch(ctx, s);
    if (rc != SOLID_OK) return rc;
  }
  ++ctx->epoch;
  KParams& kp = ctx->kp;
  memcpy(kp.klo, ctx->klo, sizeof(kp.klo));
  memcpy(kp.khi, ctx->khi, sizeof(kp.khi));
  kp.ksum_lo = kp.ksum_hi = 0;
  for (uint32_t i = 0; i < kBS; ++i) {
    kp.ksum_lo += ctx->klo[i];
    kp.ksum_hi += ctx->khi[i];
  }
  kp.mpow = ctx->mpow;
  kp.gtab = ctx->gtab;
  kp.seed = ctx->cfg.hash_seed;
  kp.nc = ctx->nc;
  memcpy(kp.klo2, ctx->klo2, sizeof(kp.klo2));
  memcpy(kp.khi2, ctx->khi2, sizeof(kp.khi2));
  kp.ksum_lo2 = kp.ksum_hi2 = 0;
  for (uint32_t i = 0; i < kBS && ctx->nc == 2; ++i) {
    kp.ksum_lo2 += ctx->klo2[i];
    kp.ksum_hi2 += ctx->khi2[i];
  }
  kp.mpow2 = ctx->mpow2;
  kp.gtab2 = ctx->gtab2;
  kp.cs = ctx->cs;
  kp.tokens = b->tokens;
  kp.offsets = b->offsets;
  kp.users = b->users;
  kp.enforce = b->enforce;
  kp.n = b->n_requests;
  kp.j_lo = 0;
  ctx->split_last = false;
  kp.policy = ctx->cfg.policy;
  kp.seq_base = 0;
  kp.dist = 0;
  kp.max_blocks = ctx->cfg.max_blocks;
  kp.epoch = ctx->epoch;
  kp.salt = splitmix64(0x5A17ull ^ ((unsigned long long)ctx->epoch << 20));
  kp.stab = ctx->stab;
  kp.smask = ctx->scap - 1;
  kp.hot = ctx->hot;
  kp.cold = ctx->cold;
  kp.tab = ctx->tab;
  kp.tmask = ctx->tcap - 1;
  kp.id_of_block = ctx->id_of_block;
  kp.iso_id = ctx->iso_id;
  kp.slot_cap = ctx->slot_cap;
  kp.dec = ctx->dec;
  kp.fst = ctx->fst;
  kp.stamp = ctx->stamp_rule;
  kp.tail = ctx->tail;
  kp.stamp_wait_ns = ctx->stamp_wait_ns;
  kp.dlist = ctx->dlist;
  kp.dcnt = ctx->dcnt;
  kp.out = out;
  // the CTA-per-request path pays only when the batch has fewer requests than the GPU has
  // resident warps (148 SMs x 32): with more, warp-per-request already fills the machine and
  // the per-step CTA barriers cost more than they parallelise (C3: 1.64 vs 1.34 ms)
  kp.long_q = b->n_requests <= kLongMaxBatch ? ctx->long_q : nullptr;
  kp.pack = 0;                     // set by do_lookup for its whole-batch K_A launch only
  kp.pool_cnt = ctx->pool_cnt;
  kp.seg_new = ctx->seg_new;
  kp.seg_cnt = ctx->seg_cnt;
  kp.seg_cap = ctx->seg_cap;
  kp.st = ctx->st;
  CK(cudaMemsetAsync(ctx->st, 0, kStHead, s));
  CK(cudaMemsetAsync(ctx->seg_cnt, 0, kNSeg * sizeof(SegCounter), s));
  CK(cudaMemsetAsync(ctx->dcnt, 0, 2 * sizeof(uint32_t), s));
  // the block table describes the last COMMITTED batch; this lookup replaces the batch arrays it
  // is built from, so it is unavailable until this batch commits
  pool_invalidate(ctx);
  ctx->launches = 0;
  return SOLID_OK;
}

// After K_A: the resolver; the lookup is then pending (solid_insert_batch commits it).
static solid_status lookup_resolve(solid_ctx* ctx, cudaStream_t s) {
  CK(cudaEventRecord(ctx->ev[1], s));
  CK(cudaEventRecord(ctx->ev[4], s));
  if (ctx->kp.n) {
    solid_status rc = launch_resolve(ctx, s);
    if (rc != SOLID_OK) return rc;
    ctx->launches += 1;
  }
  CK(cudaEventRecord(ctx->ev[5], s));
  CK(cudaEventRecord(ctx->ev[2], s));
  ctx->pending = true;
  return SOLID_OK;
}

static solid_status launch_hash_packed(solid_ctx* ctx, cudaStream_t s) {
  KParams& kp = ctx->kp;
  const void* fn;
  const bool two = kp.nc == 2;
  switch (ctx->cfg.policy) {
    case SOLID_POLICY_APC:
      fn = two ? (const void*)k_hash_packed<SOLID_POLICY_APC, 2>
               : (const void*)k_hash_packed<SOLID_POLICY_APC, 1>;
      break;
    case SOLID_POLICY_USER_ISOLATION:
      fn = two ? (const void*)k_hash_packed<SOLID_POLICY_USER_ISOLATION, 2>
               : (const void*)k_hash_packed<SOLID_POLICY_USER_ISOLATION, 1>;
      break;
    default:
      fn = two ? (const void*)k_hash_packed<SOLID_POLICY_SOLIDARITY, 2>
               : (const void*)k_hash_packed<SOLID_POLICY_SOLIDARITY, 1>;
      break;
  }
  if (!ctx->pk_grid) {
    int per_sm = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->dev));
    ctx->pk_grid = (uint32_t)std::min<int64_t>(std::max(per_sm, 1) * (int64_t)sms, 8192);
  }
  kp.pack = 1;
  kp.pk_pre = ctx->pk_pre;
  kp.pk_ctot = ctx->pk_ctot;
  kp.pk_cpre = ctx->pk_cpre;
  kp.pk_wfirst = ctx->pk_wfirst;
  void* args[] = {(void*)&kp};
  CK(cudaLaunchCooperativeKernel(fn, dim3(ctx->pk_grid), dim3(256), args, 0, s));
  return SOLID_OK;
}

// K_A CTA size for this context's next batch: 64 unless the last collected batch took the
// packed K_A (SOLID_KA_BLOCK = 64 / 128 / 256 fixes it)
static unsigned ka_block(const solid_ctx* ctx) {
  static const int fixed = [] {
    const char* e = getenv("SOLID_KA_BLOCK");
    const int v = e ? atoi(e) : 0;
    return (v == 32 || v == 64 || v == 128 || v == 256) ? v : 0;
  }();
  if (fixed) return (unsigned)fixed;
  return ctx->pack_hint ? 256u : 64u;
}

static solid_status do_lookup(solid_ctx* ctx, const solid_batch* b, solid_result* out,
                              void* stream) {
  solid_status rc = lookup_setup(ctx, b, out, stream);
  if (rc != SOLID_OK) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (ctx->ev_state) return evict_lookup(ctx, s);
  CK(cudaEventRecord(ctx->ev[0], s));
  if (ctx->kp.n) {
    // packed K_A (solid_pack.inc): taken on the device when requests are short; the
    // warp-per-request K_A launched next exits at once then (and vice versa).  While collected
    // batches do not take it, it is launched only when the batch size changed by more than 1.5x
    // or every 64th batch (its early exit costs a cooperative launch; without it the
    // warp-per-request K_A handles any batch by itself)
    const uint64_t nn = ctx->kp.n;
    const bool resized = nn * 2 < ctx->pack_last_n * 3 ? nn * 3 < ctx->pack_last_n * 2 : true;
    const bool try_pack = ctx->pack_hint || resized || ++ctx->pack_probe >= 64;
    ctx->pack_last_n = nn;
    if (ctx->pack && ctx->kp.n >= 2 && try_pack) {
      ctx->pack_probe = 0;
      solid_status rc = launch_hash_packed(ctx, s);
      if (rc != SOLID_OK) return rc;
      ctx->launches += 1;
    }
    CK(launch_hash(ctx->kp, s, ka_block(ctx)));
    ctx->kp.pack = 0;                    // later launches of this batch (splits) are per range
    ctx->launches += 1;
  }
  return lookup_resolve(ctx, s);
}

static solid_status require_collected(solid_ctx* ctx, const char* what) {
  if (ctx->outstanding || !ctx->done_q.empty())
    return fail(ctx, SOLID_ERR_STATE,
                std::string(what) + " with asynchronous batches outstanding (collect them with "
                                    "solid_batch_status)");
  return SOLID_OK;
}

extern "C" solid_status solid_lookup_batch(solid_ctx* ctx, const solid_batch* b, solid_result* out,
                                           void* stream) {
  if (!ctx) return SOLID_ERR_INVALID;
  solid_status rc = require_collected(ctx, "lookup_batch");
  if (rc != SOLID_OK) return rc;
  if (!ctx->pending) set_slot(ctx, ctx->head);
  return do_lookup(ctx, b, out, stream);
}

// Enqueue the commit of the pending lookup (+ stats and the status copies).  The capacity check
// runs on the device before any claim (k_stats), for the synchronous and asynchronous paths.
static solid_status enqueue_commit(solid_ctx* ctx, cudaStream_t s) {
  const uint64_t n = ctx->kp.n - ctx->kp.j_lo;
  if (n) {
    if (ctx->kp.pool_cnt) CK(cudaMemsetAsync(ctx->kp.pool_cnt, 0, ctx->kp.n * 4, s));
    // counts and the capacity decision first (device-resident live count), then the claims
    k_stats<<<296, 256, 0, s>>>(    // 148 SMs x 2: the id count spans every registered key
                                    // (more CTAs only add same-address atomics)
        ctx->kp.out + ctx->kp.j_lo, n, ctx->st, ctx->live_dev, ctx->cfg.capacity_blocks,
        ctx->seg_cnt, ctx->kp);
    CK(cudaGetLastError());
    launch_commit(ctx, 1, s);
    CK(cudaGetLastError());
    ctx->launches += 3;
  }
  CK(cudaEventRecord(ctx->ev[3], s));
  CK(cudaMemcpyAsync(ctx->st_host, ctx->st, kStHead, cudaMemcpyDeviceToHost, s));
  CK(cudaEventRecord(ctx->ev[6], s));
  Flight& f = ctx->fl[ctx->cur];
  f.n = n;
  f.launches = ctx->launches;
  f.gen = ctx->gen;
  return SOLID_OK;
}

// After the stream passed slot i's status copies: report that batch and update the counters.
// A batch admitted before the last solid_reset only reports its status and per-batch figures.
static solid_status finish_batch(solid_ctx* ctx, uint32_t i, cudaStream_t s, bool async_mode) {
  const Flight& f = ctx->fl[i];
  const DevStatus& h = ctx->slots[i].st;
  const uint64_t n = f.n;
  if (h.err) {                             // detected on the device during lookup: nothing committed
    const uint32_t e = h.err;
    std::string m = "invalid batch:";
    if (e & ERR_OFFSETS) m += " offsets";
    if (e & ERR_TOKEN) m += " token>=2^20";
    if (e & ERR_USER) m += " user==NONE";
    if (e & ERR_BLOCKS) m += " request>max_blocks";
    if (e & ERR_SLOTCAP) m += " tokens>max_batch_tokens";
    if (e & ERR_SCRATCH) return fail(ctx, SOLID_ERR_CAPACITY, "batch scratch overflow");
    return fail(ctx, SOLID_ERR_INVALID, m);
  }
  if (n && h.conv == 0)
    return fail(ctx, SOLID_ERR_STATE, "resolver did not converge within the round limit "
                                      "(nothing committed; resubmit the batch in parts)");
  const bool current = f.gen == ctx->gen;
  if (h.overflow)
    return fail(ctx, SOLID_ERR_CAPACITY, "index capacity exceeded (no eviction, R9); nothing committed");
  if (ctx->pool && current && !async_mode) {   // physical blocks (solid_pool.inc)
    solid_status rc = pool_commit(ctx, s, ctx->cfg.policy == SOLID_POLICY_SOLIDARITY ? h.conv : 0u,
                                  h.new_entries, 0, 0);
    if (rc != SOLID_OK) return rc;
  }
  solid_stats_t& S = ctx->stats;
  ctx->rounds = (ctx->cfg.policy == SOLID_POLICY_SOLIDARITY) ? h.conv : (n ? 1u : 0u);
  if (current) {
    S.batches += 1;
    S.requests += n;
    S.blocks += h.sums[0];
    S.reused_blocks += h.sums[1];
    S.flagged += h.sums[2];
    S.diverted += h.sums[3];
    S.truncated += h.sums[4];
    S.inserted += h.new_entries;
    if (n) ctx->live = h.live_after;
    S.live_entries = ctx->live;
  }
  S.last_rounds = ctx->rounds;
  ctx->pack_hint = h.packed ? 1 : (f.n ? 0 : ctx->pack_hint);
  for (int q = 0; q < 8; ++q)
    S.round_us[q] = (q < (int)ctx->rounds && q < 16 && h.round_ns[q + 1] > h.round_ns[0])
                        ? (float)((h.round_ns[q + 1] - h.round_ns[q]) * 1e-3)
                        : 0.f;
  uint64_t distinct = 0;
  for (int q = 0; q < kNSeg; ++q)
    distinct += std::min<uint32_t>(ctx->slots[i].st.seg[q], ctx->seg_cap);
  S.last_distinct_keys = (uint32_t)std::min<uint64_t>(distinct, 0xFFFFFFFFull);
  S.last_shared_keys = (uint32_t)std::min<unsigned long long>(h.ids_after_hash, 0xFFFFFFFFull);
  S.last_kernel_launches = f.launches;
  S.last_requests = n;
  S.last_blocks = h.sums[0];
  S.last_inserted = h.new_entries;
  S.last_flagged = h.sums[2];
  S.algorithmic_bytes = 64ull * h.sums[0] + 37ull * n + 16ull * distinct + 16ull * h.new_entries +
                        4ull * h.new_flags;
  // phase times (the copies behind ev[6] completed, so every event of the batch did)
  cudaEventElapsedTime(&S.ms_hash, f.ev[0], f.ev[1]);
  cudaEventElapsedTime(&S.ms_resolve, f.ev[1], f.ev[2]);
  cudaEventElapsedTime(&S.ms_commit, f.ev[2], f.ev[3]);
  cudaEventElapsedTime(&S.ms_hash_kernel, f.ev[0], f.ev[1]);
  cudaEventElapsedTime(&S.ms_round_first, f.ev[4], f.ev[5]);
  return SOLID_OK;
}

static solid_status admit_range(solid_ctx* ctx, uint64_t lo, uint64_t hi, cudaStream_t s);

// Commit of the pending lookup (not evict mode) and one host wait.  `d2h_bytes` > 0: the batch's
// results are copied to host memory in the same wait (host admission; they are copied again
// after a split), so a converged batch costs a single synchronisation.
static solid_status insert_sync(solid_ctx* ctx, cudaStream_t s, void* d2h_dst,
                                const void* d2h_src, size_t d2h_bytes) {
  solid_status rc = enqueue_commit(ctx, s);
  if (rc != SOLID_OK) return rc;
  if (d2h_bytes) CK(cudaMemcpyAsync(d2h_dst, d2h_src, d2h_bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  ctx->pending = false;
  const DevStatus& h = ctx->slots[ctx->cur].st;
  if (ctx->kp.n > ctx->kp.j_lo && h.conv == 0 && h.err == 0 && !ctx->pool) {
    // the resolver hit its round limit: nothing was committed.  Requests
    // before round t_max are final, so admitting the batch as consecutive parts (R1: results
    // do not depend on the cut) always ends: a part of <= t_max - 1 requests converges.
    const uint64_t lo = ctx->kp.j_lo, hi = ctx->kp.n;
    if (hi - lo < 2) return fail(ctx, SOLID_ERR_STATE, "resolver did not converge");
    const uint64_t mid = lo + (hi - lo) / 2;
    rc = admit_range(ctx, lo, mid, s);
    if (rc == SOLID_OK) rc = admit_range(ctx, mid, hi, s);
    ctx->split_last = true;
    if (rc == SOLID_OK && d2h_bytes) {
      CK(cudaMemcpyAsync(d2h_dst, d2h_src, d2h_bytes, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    return rc;
  }
  return finish_batch(ctx, ctx->cur, s, false);
}

extern "C" solid_status solid_insert_batch(solid_ctx* ctx, void* stream) {
  if (!ctx) return SOLID_ERR_INVALID;
  if (ctx->poisoned) return fail(ctx, SOLID_ERR_STATE, "context poisoned by an earlier failure");
  if (!ctx->pending) return fail(ctx, SOLID_ERR_STATE, "insert_batch without a pending lookup");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(ctx->dev));
  if (ctx->ev_state) return evict_insert(ctx, s);
  return insert_sync(ctx, s, nullptr, nullptr, 0);
}

// Admit requests [lo, hi) of the pending batch's arrays as a batch of their own (a part of a
// batch whose resolver did not converge; R1: admitting a stream in consecutive parts gives the
// same results).  Synchronous; splits again if the part does not converge either.
static solid_status admit_range(solid_ctx* ctx, uint64_t lo, uint64_t hi, cudaStream_t s) {
  if (ctx->epoch + 1 > kMaxEpoch) {
    solid_status rc = init_scratch(ctx, s);
    if (rc != SOLID_OK) return rc;
  }
  ++ctx->epoch;
  KParams& kp = ctx->kp;
  kp.epoch = ctx->epoch;
  kp.salt = splitmix64(0x5A17ull ^ ((unsigned long long)ctx->epoch << 20));
  kp.j_lo = lo;
  kp.n = hi;
  CK(cudaMemsetAsync(ctx->st, 0, kStHead, s));
  CK(cudaMemsetAsync(ctx->seg_cnt, 0, kNSeg * sizeof(SegCounter), s));
  CK(cudaMemsetAsync(ctx->dcnt, 0, 2 * sizeof(uint32_t), s));
  CK(cudaEventRecord(ctx->ev[0], s));
  CK(launch_hash(kp, s, lo, hi));
  ctx->launches = 1;
  solid_status rc = lookup_resolve(ctx, s);
  if (rc != SOLID_OK) return rc;
  return solid_insert_batch(ctx, s);
}

extern "C" solid_status solid_admit_batch(solid_ctx* ctx, const solid_batch* batch,
                                          solid_result* out, void* stream) {
  if (!ctx) return SOLID_ERR_INVALID;
  if (ctx->ev_state || ctx->pool) {
    // LRU eviction / block tables: their lookup waits on the host (joint resolver / eviction-time
    // iteration) and their commit reads counts back, so the batch is admitted here,
    // in submission order, and its status queued for solid_batch_status.  Same contract as the
    // asynchronous path: a failed batch leaves the index as before it, later batches see that
    // state; argument errors are returned at once.
    if (ctx->pending) return fail(ctx, SOLID_ERR_STATE, "admit_batch with a pending lookup");
    if (ctx->done_q.size() >= kRing)
      return fail(ctx, SOLID_ERR_STATE,
                  "SOLID_MAX_INFLIGHT batches outstanding (collect one with solid_batch_status)");
    CK(cudaSetDevice(ctx->dev));
    set_slot(ctx, ctx->head);
    solid_status rc = do_lookup(ctx, batch, out, stream);
    if (rc != SOLID_OK && !ctx->pending) return rc;       // rejected before anything was staged
    if (rc == SOLID_OK) rc = solid_insert_batch(ctx, stream);
    ctx->pending = false;
    if (rc == SOLID_ERR_CUDA) return rc;                   // context poisoned: reported now
    ctx->done_q.emplace_back(rc, rc == SOLID_OK ? std::string() : ctx->err);
    return SOLID_OK;
  }
  if (ctx->pending) return fail(ctx, SOLID_ERR_STATE, "admit_batch with a pending lookup");
  if (ctx->outstanding == kRing)
    return fail(ctx, SOLID_ERR_STATE,
                "SOLID_MAX_INFLIGHT asynchronous batches outstanding (collect one with "
                "solid_batch_status)");
  CK(cudaSetDevice(ctx->dev));
  set_slot(ctx, (ctx->head + ctx->outstanding) % kRing);
  solid_status rc = do_lookup(ctx, batch, out, stream);
  if (rc != SOLID_OK) return rc;
  rc = enqueue_commit(ctx, (cudaStream_t)stream);
  ctx->pending = false;
  if (rc != SOLID_OK) return rc;
  ++ctx->outstanding;
  return SOLID_OK;
}

extern "C" solid_status solid_batch_status(solid_ctx* ctx) {
  if (!ctx) return SOLID_ERR_INVALID;
  if (!ctx->done_q.empty()) {                // admitted at submission (evict / block-table)
    const auto d = ctx->done_q.front();
    ctx->done_q.pop_front();
    if (d.first != SOLID_OK) ctx->err = d.second;
    return d.first;
  }
  if (!ctx->outstanding) return SOLID_OK;
  CK(cudaSetDevice(ctx->dev));
  const uint32_t i = ctx->head;
  CK(cudaEventSynchronize(ctx->fl[i].ev[6]));
  ctx->head = (ctx->head + 1) % kRing;
  --ctx->outstanding;
  return finish_batch(ctx, i, ctx->stream, true);
}

// 16-bit token ids widened to the library's 32-bit layout (8 tokens per thread, 16-byte loads
// when the source is aligned).
__global__ void __launch_bounds__(256) k_widen16(const uint16_t* in, uint32_t* out, uint64_t T) {
  const uint64_t n8 = T / 8;
  const bool al = ((uintptr_t)in & 15) == 0;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n8;
       q += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t w[4];
    if (al) {
      const uint4 v = reinterpret_cast<const uint4*>(in)[q];
      w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else {
      for (int k = 0; k < 4; ++k) w[k] = (uint32_t)in[8 * q + 2 * k] | ((uint32_t)in[8 * q + 2 * k + 1] << 16);
    }
    uint4 a = make_uint4(w[0] & 0xFFFFu, w[0] >> 16, w[1] & 0xFFFFu, w[1] >> 16);
    uint4 b = make_uint4(w[2] & 0xFFFFu, w[2] >> 16, w[3] & 0xFFFFu, w[3] >> 16);
    reinterpret_cast<uint4*>(out)[2 * q] = a;
    reinterpret_cast<uint4*>(out)[2 * q + 1] = b;
  }
  if (blockIdx.x == 0 && threadIdx.x < (T & 7)) out[8 * n8 + threadIdx.x] = in[8 * n8 + threadIdx.x];
}

// Host-buffer admission: batch arrays copied in (tokens as 32- or 16-bit ids), lookup + insert,
// results copied out; synchronises the stream.  The batch is validated on the host first
// (offsets, sizes), so a rejected batch never starts; it is admitted as ONE batch (all or
// nothing, R9) — only K_A is split: the tokens are copied in kHostChunks pieces on a second
// stream and each piece's requests are hashed as soon as their tokens have arrived, so the
// copies overlap the hashing; one resolver and one commit follow.
static solid_status admit_host_common(solid_ctx* ctx, uint64_t n, const void* tokens,
                                      int token_bytes, const uint64_t* offsets,
                                      const uint32_t* users, const uint8_t* enforce,
                                      solid_result* out_host, void* stream) {
  if (!ctx) return SOLID_ERR_INVALID;
  if (ctx->poisoned) return fail(ctx, SOLID_ERR_STATE, "context poisoned by an earlier failure");
  if (ctx->pending) return fail(ctx, SOLID_ERR_STATE, "admit_host with a pending lookup");
  solid_status rc = require_collected(ctx, "admit_host");
  if (rc != SOLID_OK) return rc;
  if (!offsets || (n && (!tokens || !users || !out_host)))
    return fail(ctx, SOLID_ERR_INVALID, "null batch pointer");
  if (n > ctx->cfg.max_batch_requests)
    return fail(ctx, SOLID_ERR_INVALID, "n_requests > max_batch_requests");
  if (offsets[0] != 0) return fail(ctx, SOLID_ERR_INVALID, "invalid batch: offsets[0] != 0");
  for (uint64_t j = 0; j < n; ++j)
    if (offsets[j + 1] < offsets[j]) return fail(ctx, SOLID_ERR_INVALID, "invalid batch: offsets");
  const uint64_t T = offsets[n];
  if (T > ctx->cfg.max_batch_tokens) return fail(ctx, SOLID_ERR_INVALID, "tokens > max_batch_tokens");
  CK(cudaSetDevice(ctx->dev));
  cudaStream_t s = (cudaStream_t)stream;
  if (!ctx->h_tokens) {
    const uint64_t R = ctx->cfg.max_batch_requests;
    CK(cudaMalloc(&ctx->h_tokens, (ctx->cfg.max_batch_tokens + 4) * 4));
    CK(cudaMalloc(&ctx->h_offsets, (R + 1) * 8));
    CK(cudaMalloc(&ctx->h_users, R * 4 + 4));
    CK(cudaMalloc(&ctx->h_enforce, R + 1));
    CK(cudaMalloc(&ctx->h_out, R * sizeof(solid_result) + 32));
  }
  if (token_bytes == 2 && !ctx->h_tokens16)
    CK(cudaMalloc(&ctx->h_tokens16, (ctx->cfg.max_batch_tokens + 8) * 2));
  CK(cudaMemcpyAsync(ctx->h_offsets, offsets, (n + 1) * 8, cudaMemcpyHostToDevice, s));
  if (n) CK(cudaMemcpyAsync(ctx->h_users, users, n * 4, cudaMemcpyHostToDevice, s));
  if (n && enforce) CK(cudaMemcpyAsync(ctx->h_enforce, enforce, n, cudaMemcpyHostToDevice, s));
  const uint32_t HC = ctx->host_chunks;
  const uint32_t K = (T * (uint64_t)token_bytes >= (64ull << 20) && n >= 4 * HC &&
                      !ctx->ev_state) ? HC : 1u;
  if (K > 1 && !ctx->s_copy) {
    CK(cudaStreamCreateWithFlags(&ctx->s_copy, cudaStreamNonBlocking));
    for (auto& e : ctx->ev_chunk) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t sc = K > 1 ? ctx->s_copy : s;
  if (K > 1) {                       // the copy stream starts after the small copies were enqueued
    CK(cudaEventRecord(ctx->ev_chunk[kHostChunksMax], s));
    CK(cudaStreamWaitEvent(sc, ctx->ev_chunk[kHostChunksMax], 0));
  }
  // chunk boundaries (requests): K - 1 equal chunks and a last one of half their size, so the
  // hashing left after the last copy is short
  auto cut = [&](uint32_t k) -> uint64_t {
    if (k >= K) return n;
    return K == 1 ? 0 : n * k * (2 * K - 1) / (2ull * K * (K - 1));
  };
  for (uint32_t k = 0; k < K; ++k) {
    const uint64_t a = offsets[cut(k)], b = offsets[cut(k + 1)];
    if (b > a)
      CK(cudaMemcpyAsync(token_bytes == 2 ? (void*)(ctx->h_tokens16 + a) : (void*)(ctx->h_tokens + a),
                         (const char*)tokens + a * token_bytes, (b - a) * token_bytes,
                         cudaMemcpyHostToDevice, sc));
    if (K > 1) CK(cudaEventRecord(ctx->ev_chunk[k], sc));
  }
  solid_batch db;
  db.n_requests = n;
  db.tokens = ctx->h_tokens;
  db.offsets = ctx->h_offsets;
  db.users = ctx->h_users;
  db.enforce = enforce ? ctx->h_enforce : nullptr;
  set_slot(ctx, ctx->head);
  rc = lookup_setup(ctx, &db, ctx->h_out, stream);
  if (rc == SOLID_OK && ctx->ev_state) {          // evict mode: one piece (K == 1)
    if (token_bytes == 2 && T)
      k_widen16<<<(unsigned)std::min<uint64_t>((T / 8 + 255) / 256 + 1, 8192), 256, 0, s>>>(
          ctx->h_tokens16, ctx->h_tokens, T);
    rc = evict_lookup(ctx, s);
  } else if (rc == SOLID_OK) {
    CK(cudaEventRecord(ctx->ev[0], s));
    for (uint32_t k = 0; k < K; ++k) {
      const uint64_t lo = cut(k), hi = cut(k + 1);
      const uint64_t a = offsets[lo], b = offsets[hi];
      if (K > 1) CK(cudaStreamWaitEvent(s, ctx->ev_chunk[k], 0));
      if (token_bytes == 2 && b > a) {   // widen from an 8-aligned start (earlier ids: same values)
        const uint64_t a8 = a & ~7ull;
        k_widen16<<<(unsigned)std::min<uint64_t>(((b - a8) / 8 + 255) / 256 + 1, 8192), 256, 0, s>>>(
            ctx->h_tokens16 + a8, ctx->h_tokens + a8, b - a8);
        CK(cudaGetLastError());
      }
      CK(launch_hash(ctx->kp, s, lo, hi, ka_block(ctx)));
      ++ctx->launches;
    }
    rc = lookup_resolve(ctx, s);
  }
  if (rc == SOLID_OK) {
    if (ctx->ev_state) {
      rc = solid_insert_batch(ctx, stream);
      if (rc == SOLID_OK && n)
        CK(cudaMemcpyAsync(out_host, ctx->h_out, n * sizeof(solid_result), cudaMemcpyDeviceToHost, s));
    } else {         // commit + result copy, one host wait (the results are unspecified on failure)
      rc = insert_sync(ctx, s, out_host, ctx->h_out, n * sizeof(solid_result));
    }
  }
  if (K > 1) cudaStreamSynchronize(sc);       // no copy may outlive a failed call
  if (rc != SOLID_OK) return rc;
  CK(cudaStreamSynchronize(s));
  return SOLID_OK;
}

extern "C" solid_status solid_admit_host(solid_ctx* ctx, const solid_batch* hb,
                                         solid_result* out_host, void* stream) {
  if (!hb) return ctx ? fail(ctx, SOLID_ERR_INVALID, "null batch pointer") : SOLID_ERR_INVALID;
  return admit_host_common(ctx, hb->n_requests, hb->tokens, 4, hb->offsets, hb->users,
                           hb->enforce, out_host, stream);
}

extern "C" solid_status solid_admit_host_u16(solid_ctx* ctx, const solid_batch_u16* hb,
                                             solid_result* out_host, void* stream) {
  if (!hb) return ctx ? fail(ctx, SOLID_ERR_INVALID, "null batch pointer") : SOLID_ERR_INVALID;
  return admit_host_common(ctx, hb->n_requests, hb->tokens, 2, hb->offsets, hb->users,
                           hb->enforce, out_host, stream);
}

// Profiling build (-DSOLID_COUNTERS) only: the last collected batch's per-round path counters.
// Test hook: move the scratch epoch (the tag space restarts after kMaxEpoch batches, ~1 M; a
// long-running server crosses it, so the restart is tested by jumping close to it).
extern "C" solid_status solid_debug_set_epoch(solid_ctx* ctx, uint32_t epoch) {
  if (!ctx || epoch > kMaxEpoch) return SOLID_ERR_INVALID;
  if (ctx->pending || ctx->outstanding) return fail(ctx, SOLID_ERR_STATE, "batch in flight");
  ctx->epoch = epoch;
  return SOLID_OK;
}

// Test hook: the resolver's round limit (default 4093).  A batch that does not converge within
// it is admitted in parts by the synchronous paths (solid_insert_batch, solid_admit_host).
extern "C" solid_status solid_debug_set_max_rounds(solid_ctx* ctx, uint32_t rounds) {
  if (!ctx || rounds < 2 || rounds > kMaxRounds) return SOLID_ERR_INVALID;
  if (ctx->pending || ctx->outstanding) return fail(ctx, SOLID_ERR_STATE, "batch in flight");
  ctx->max_rounds = rounds;
  return SOLID_OK;
}

extern "C" solid_status solid_debug_counters(solid_ctx* ctx, unsigned long long* out) {
#ifdef SOLID_COUNTERS
  if (!ctx || !out) return SOLID_ERR_INVALID;
  memcpy(out, ctx->slots[ctx->cur].st.cnt, sizeof(ctx->slots[0].st.cnt));
  return SOLID_OK;
#else
  (void)ctx;
  (void)out;
  return SOLID_ERR_STATE;
#endif
}

// Block table of the last batch: the key of the entry that holds each block's KV.
template <int POLICY>
__global__ void __launch_bounds__(256) k_block_keys(KParams kp, unsigned long long* keys_out) {
  const int lane = threadIdx.x & 31;
  const uint64_t j = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= kp.n) return;
  const uint64_t o0 = kp.offsets[j], o1 = kp.offsets[j + 1];
  if (o1 < o0) return;
  const uint32_t n = (uint32_t)min((o1 - o0) >> 4, (uint64_t)kp.max_blocks);
  const uint64_t blk0 = o0 >> 4;
  const int32_t f = POLICY == SOLID_POLICY_SOLIDARITY ? (int32_t)kp.dec[j].y : -1;
  for (uint32_t b = lane; b < n; b += 32) {
    const uint32_t id = (f >= 1 && b >= (uint32_t)f) ? kp.iso_id[blk0 + b] : kp.id_of_block[blk0 + b];
    keys_out[blk0 + b] = kp.cold[id].key;
  }
}

extern "C" solid_status solid_block_keys(solid_ctx* ctx, unsigned long long* keys_out,
                                         void* stream) {
  if (!ctx || !keys_out) return SOLID_ERR_INVALID;
  if (ctx->dist) return fail(ctx, SOLID_ERR_STATE, "block_keys: not available on a shard");
  if (ctx->pending) return fail(ctx, SOLID_ERR_STATE, "block_keys with a pending lookup");
  if (ctx->split_last)
    return fail(ctx, SOLID_ERR_STATE, "block_keys: the last batch was committed in parts");
  if (ctx->poisoned) return fail(ctx, SOLID_ERR_STATE, "context poisoned by an earlier failure");
  CK(cudaSetDevice(ctx->dev));
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t n = ctx->kp.n;
  if (!n) return SOLID_OK;
  const unsigned grid = (unsigned)((n * 32 + 255) / 256);
  switch (ctx->cfg.policy) {
    case SOLID_POLICY_APC: k_block_keys<SOLID_POLICY_APC><<<grid, 256, 0, s>>>(ctx->kp, keys_out); break;
    case SOLID_POLICY_USER_ISOLATION:
      k_block_keys<SOLID_POLICY_USER_ISOLATION><<<grid, 256, 0, s>>>(ctx->kp, keys_out); break;
    default: k_block_keys<SOLID_POLICY_SOLIDARITY><<<grid, 256, 0, s>>>(ctx->kp, keys_out); break;
  }
  CK(cudaGetLastError());
  return SOLID_OK;
}

extern "C" solid_status solid_stats(solid_ctx* ctx, solid_stats_t* out) {
  if (!ctx || !out) return SOLID_ERR_INVALID;
  *out = ctx->stats;
  return SOLID_OK;
}

extern "C" solid_status solid_dump(solid_ctx* ctx, solid_entry* host_out, uint64_t cap,
                                   uint64_t* n_out) {
  if (!ctx || !n_out || (cap && !host_out)) return SOLID_ERR_INVALID;
  solid_status rc0 = require_collected(ctx, "dump");
  if (rc0 != SOLID_OK) return rc0;
  if (ctx->poisoned) return fail(ctx, SOLID_ERR_STATE, "context poisoned by an earlier failure");
  CK(cudaSetDevice(ctx->dev));
  if (ctx->stream) CK(cudaStreamSynchronize(ctx->stream));
  // compact the live slots on the device, copy only those
  const unsigned long long cap_e = ctx->live + 1024;
  ulonglong2* dbuf = nullptr;
  unsigned long long* dcnt = nullptr;
  CK(cudaMalloc(&dbuf, cap_e * sizeof(ulonglong2)));
  CK(cudaMalloc(&dcnt, sizeof(unsigned long long)));
  CK(cudaMemset(dcnt, 0, sizeof(unsigned long long)));
  k_compact<<<2048, 256>>>(ctx->tab, ctx->tcap, dbuf, dcnt, cap_e);
  CK(cudaGetLastError());
  unsigned long long hc = 0;
  CK(cudaMemcpy(&hc, dcnt, sizeof(hc), cudaMemcpyDeviceToHost));
  std::vector<ulonglong2> h(std::min<unsigned long long>(hc, cap_e));
  if (!h.empty())
    CK(cudaMemcpy(h.data(), dbuf, h.size() * sizeof(ulonglong2), cudaMemcpyDeviceToHost));
  cudaFree(dbuf);
  cudaFree(dcnt);
  if (hc > cap_e) return fail(ctx, SOLID_ERR_STATE, "dump: index holds more entries than tracked");
  std::vector<solid_entry> v;
  v.reserve(h.size());
  for (const auto& e : h) v.push_back(solid_entry{e.x, (uint32_t)e.y, (uint32_t)(e.y >> 32)});
  std::sort(v.begin(), v.end(), [](const solid_entry& a, const solid_entry& b) { return a.key < b.key; });
  *n_out = v.size();
  const uint64_t m = std::min<uint64_t>(cap, v.size());
  if (m) memcpy(host_out, v.data(), m * sizeof(solid_entry));
  return SOLID_OK;
}

extern "C" solid_status solid_reset(solid_ctx* ctx) {
  if (!ctx) return SOLID_ERR_INVALID;
  CK(cudaSetDevice(ctx->dev));
  cudaStream_t s = ctx->stream;
  if (ctx->poisoned || !ctx->outstanding) {      // synchronous unless batches are in flight
    if (s) CK(cudaStreamSynchronize(s));
    CK(cudaDeviceSynchronize());
  }
  CK(cudaMemsetAsync(ctx->tab, 0, ctx->tcap * sizeof(ulonglong2), s));
  if (ctx->poisoned) {
    solid_status rc = init_scratch(ctx, s);
    if (rc != SOLID_OK) return rc;
  }
  if (ctx->ev_state) {
    solid_status rc = evict_reset(ctx, s);
    if (rc != SOLID_OK) return rc;
  }
  if (ctx->pool) {
    solid_status rc = pool_reset(ctx, s);
    if (rc != SOLID_OK) return rc;
  }
  CK(cudaMemsetAsync(ctx->live_dev, 0, sizeof(unsigned long long), s));
  if (!ctx->outstanding) CK(cudaStreamSynchronize(s));
  if (ctx->poisoned) ctx->head = ctx->outstanding = 0;   // their results are lost with the state
  ++ctx->gen;
  ctx->live = 0;
  ctx->pending = false;
  ctx->poisoned = false;
  ctx->stats = solid_stats_t{};
  return SOLID_OK;
}

extern "C" solid_status solid_checkpoint(solid_ctx* ctx) {
  if (!ctx) return SOLID_ERR_INVALID;
  if (ctx->pending) return fail(ctx, SOLID_ERR_STATE, "checkpoint with a pending batch");
  solid_status rc0 = require_collected(ctx, "checkpoint");
  if (rc0 != SOLID_OK) return rc0;
  CK(cudaSetDevice(ctx->dev));
  if (ctx->stream) CK(cudaStreamSynchronize(ctx->stream));
  ctx->live_ckpt = ctx->live;
  if (ctx->pool) {
    solid_status rc = pool_checkpoint(ctx);
    if (rc != SOLID_OK) return rc;
  }
  if (ctx->ev_state) return evict_checkpoint(ctx);
  if (!ctx->tab_ckpt) CK(cudaMalloc(&ctx->tab_ckpt, ctx->tcap * sizeof(ulonglong2)));
  CK(cudaMemcpy(ctx->tab_ckpt, ctx->tab, ctx->tcap * sizeof(ulonglong2), cudaMemcpyDeviceToDevice));
  ctx->live_ckpt = ctx->live;
  return SOLID_OK;
}

extern "C" solid_status solid_restore(solid_ctx* ctx) {
  if (!ctx) return SOLID_ERR_INVALID;
  if (!ctx->tab_ckpt && !ctx->ev_state) return fail(ctx, SOLID_ERR_STATE, "restore without checkpoint");
  if (ctx->pending) return fail(ctx, SOLID_ERR_STATE, "restore with a pending batch");
  solid_status rc0 = require_collected(ctx, "restore");
  if (rc0 != SOLID_OK) return rc0;
  CK(cudaSetDevice(ctx->dev));
  if (ctx->stream) CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->pool) {
    solid_status rc = pool_restore(ctx);
    if (rc != SOLID_OK) return rc;
  }
  if (ctx->ev_state) {
    solid_status rc = evict_restore(ctx);
    if (rc != SOLID_OK) return rc;
    ctx->live = ctx->live_ckpt;
    CK(cudaMemcpy(ctx->live_dev, &ctx->live, sizeof(unsigned long long), cudaMemcpyHostToDevice));
    return SOLID_OK;
  }
  CK(cudaMemcpy(ctx->tab, ctx->tab_ckpt, ctx->tcap * sizeof(ulonglong2), cudaMemcpyDeviceToDevice));
  ctx->live = ctx->live_ckpt;
  CK(cudaMemcpy(ctx->live_dev, &ctx->live, sizeof(unsigned long long), cudaMemcpyHostToDevice));
  return SOLID_OK;
}

namespace solid {
// runs f with the policy as a compile-time constant
template <typename F>
static void by_policy(int policy, F&& f) {
  switch (policy) {
    case SOLID_POLICY_APC: f(std::integral_constant<int, SOLID_POLICY_APC>()); break;
    case SOLID_POLICY_USER_ISOLATION:
      f(std::integral_constant<int, SOLID_POLICY_USER_ISOLATION>()); break;
    default: f(std::integral_constant<int, SOLID_POLICY_SOLIDARITY>()); break;
  }
}

}  // namespace solid

#include "solid_dist.inc"
#include "solid_p2p.inc"
#include "solid_pool.inc"
#include "solid_evict.inc"
