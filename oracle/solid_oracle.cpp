// ============================================================================================
//  CacheSolidarity ORACLE — TEST INFRASTRUCTURE ONLY.
//
//  A plain, slow, sequential CPU implementation of what the hot path computes:
//  a dict-based prefix cache (std::unordered_map) plus the per-request selective-isolation state
//  machine of PAPER.md "System Design > KV Cache Extension and Detector".
//
//  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
//  load this library.  It shares NO code, header, table or constant generator with the CUDA path
//  (paper_2603_10726_b200/csrc); both implement DESIGN.md §2 (semantics) independently.
//
//  Requests are processed strictly one at a time in global sequence order (reading R1:
//  sequential semantics).  There is no notion of a batch here.
//
//  Pins (tests/test_oracle_*.py): worked example t1-t4 (golden/p1_example.json),
//  attacker experiment (golden/p2_attack.json), the §5 guarantee by brute force
//  (P:560-603), APC == brute-force longest common prefix, user isolation == per-user LCP,
//  enforce=0 == APC, an independent content-keyed trie reference, splitmix64 published vector,
//  and the chain value against a closed-form big-integer polynomial.  LRU eviction (capacity > 0,
//  SPEC evict_lru S:117-125): the SPEC examples, Mattson's stack-distance theorem, the cyclic
//  thrash closed form, a brute-force trie LRU (tests/test_oracle_eviction.py).  Two-component keys
//  (H-def v3): both chains against their closed forms, exhaustive no-collision, decision
//  invariance (tests/test_oracle_hash2.py).  Physical block pool and block tables (R26-R28): the
//  first-insertion and cyclic-thrash closed forms, a brute-force min-stamp allocator over the
//  trie, lifetime invariants (tests/test_oracle_pool.py).
//  "parity unpinned": fmix64 outputs (an arbitrary finaliser; pinned only by bijectivity and by
//  agreement with the independent CUDA implementation), and likewise the H-def v3 combination
//  key2_of (its chains S, S2 are pinned; the mixing of the two is not).
// ============================================================================================
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <deque>
#include <set>
#include <unordered_map>
#include <utility>
#include <vector>

namespace {

typedef unsigned __int128 u128;

// ---- DESIGN.md §2.1 "H-def v2" (the paper is silent on hashing, P:937 is the only "hash") ----
const uint64_t P61 = (1ULL << 61) - 1;            // p = 2^61 - 1
const uint64_t NONE = 0xFFFFFFFFULL;              // "no user" (sharer unset)
const uint64_t KEY_OFFSET = 0x9E3779B97F4A7C15ULL; // key = fmix64(S + KEY_OFFSET)
const uint64_t SIGMA_SALT = 0xD1B54A32D192ED03ULL;

uint64_t mulmod(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * (u128)b) % P61); }
uint64_t addmod(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a + (u128)b) % P61); }

// splitmix64 (Vigna): one output for state x (the generator adds the golden gamma first).
uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// MurmurHash3 64-bit finaliser.
uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

uint64_t key_of(uint64_t S) {
  uint64_t k = fmix64(S + KEY_OFFSET);
  return k == 0 ? 1 : k;   // never taken (S < 2^61 keeps S+offset away from 0); kept per H-def
}

struct Entry {
  uint32_t owner;     // OwnerID: set exactly once at allocation
  uint32_t sharer;    // user that flagged the entry; AttackFlag <=> sharer != NONE (R5)
  uint64_t last_used; // LRU clock (R22): global sequence number of the last request
                      // that was served this entry or inserted it
  uint32_t phys;      // physical KV block holding the entry's content (R26); NONE = pool off
  uint32_t pins;      // requests holding the entry's block (R38); > 0: not evictable
};

struct Ctx {
  uint32_t bs;
  uint64_t seed;
  int policy;        // 0 = APC, 1 = USER_ISOLATION, 2 = SOLIDARITY
  uint64_t B, M;
  std::vector<uint64_t> K;   // K_i = B^i mod p
  // H-def v3 second component (SURVEY f4 hardening): an independent polynomial
  // chain with base B2 and salts sigma2; the key then depends on both 61-bit chain values
  int components;            // 1 (H-def v2) or 2
  uint64_t B2, M2;
  std::vector<uint64_t> K2;
  std::unordered_map<uint64_t, Entry> table;
  uint64_t next_seq;
  // LRU eviction (SPEC evict_lru S:117-125; R22-R25).  capacity 0 = unbounded (no
  // eviction, R9).  lru orders the live entries by (last_used, key): the first element is the
  // victim ("smallest last_used; ties broken by smaller hash value").
  uint64_t capacity;
  std::set<std::pair<uint64_t, uint64_t>> lru;
  uint64_t evictions;
  // Physical block pool (the vLLM block manager beneath the prefix index, P:733;
  // DESIGN.md R26-R28).  pool 0 = off.  A FIFO of free physical block ids, initially 0..pool-1:
  // an evicted entry's block goes to the back; a request's new entries take blocks from the
  // front, in block order, after the request's own evictions returned theirs (R26).
  uint64_t pool;
  std::deque<uint32_t> freeq;
  std::vector<uint64_t> fresh;        // keys the current request inserted, in block order
  std::vector<uint32_t> btab;         // block table of the last oracle_process call (R27)
  // In-flight pinning (R38, the vLLM KVCacheBlock reference count beneath P:733): with pin on,
  // every admitted request pins the entries of its block-table row until oracle_release; the
  // LRU victim is the smallest (last_used, key) among UNPINNED entries, and a request whose
  // eviction step would find too few of them (other than the entries it uses itself) is
  // refused before it mutates anything.
  bool pin;
  std::vector<uint64_t> key_of_phys;  // physical block -> key of the live entry holding it
  uint64_t admitted;                  // requests admitted by the last oracle_process call
};

uint64_t sigma_of(const Ctx& c, uint32_t user) {
  // sigma(Iso(u)) = 1 + (splitmix64(seed ^ SALT ^ u) mod (p - 1))   in [1, p-1]
  return 1 + splitmix64(c.seed ^ SIGMA_SALT ^ (uint64_t)user) % (P61 - 1);
}

// second component (H-def v3): same construction with its own seed constants
const uint64_t SEED2_SALT = 0xA0761D6478BD642FULL;
const uint64_t SIGMA2_SALT = 0xE7037ED1A0B428DBULL;
const uint64_t MIX2 = 0x9E3779B97F4A7C15ULL;
uint64_t sigma2_of(const Ctx& c, uint32_t user) {
  return 1 + splitmix64(c.seed ^ SIGMA2_SALT ^ (uint64_t)user) % (P61 - 1);
}

// key of a chain position: H-def v2 key_of(S) with one component; with two,
// key = fmix64((S ^ (S2 * MIX2 mod 2^64)) + KEY_OFFSET), 0 -> 1
uint64_t key2_of(uint64_t S, uint64_t S2) {
  uint64_t k = fmix64((S ^ (S2 * MIX2)) + KEY_OFFSET);
  return k == 0 ? 1 : k;
}

// h(block) = sum_i x_i * K_i mod p, x_i = token_i + 1
uint64_t block_hash(const Ctx& c, const uint32_t* tok) {
  uint64_t h = 0;
  for (uint32_t i = 0; i < c.bs; ++i) h = addmod(h, mulmod((uint64_t)tok[i] + 1, c.K[i]));
  return h;
}
uint64_t block_hash2(const Ctx& c, const uint32_t* tok) {
  uint64_t h = 0;
  for (uint32_t i = 0; i < c.bs; ++i) h = addmod(h, mulmod((uint64_t)tok[i] + 1, c.K2[i]));
  return h;
}

// One chain step (SPEC chain_hash(parent, block, ns), with the block's depth b made
// explicit):  S[b] = S[b-1] + M^(b-1) * (h_b + sigma_ns)  (mod p).
uint64_t chain_step(uint64_t parent, uint64_t Mpow_bm1, uint64_t h, uint64_t sigma) {
  return addmod(parent, mulmod(Mpow_bm1, addmod(h, sigma)));
}

bool present(const Ctx& c, uint64_t key) { return c.table.count(key) != 0; }
bool flagged(const Ctx& c, uint64_t key) { return c.table.at(key).sharer != NONE; }
uint32_t owner_of(const Ctx& c, uint64_t key) { return c.table.at(key).owner; }

// "On a cache miss, a new cache entry is created and tagged with the user's ID",
// with last_used = the request's clock.  Inserting a key that is already present leaves
// it unchanged — owner, flag and last_used (R8, R23).
void insert_if_absent(Ctx& c, uint64_t key, uint32_t user, uint64_t seq) {
  if (present(c, key)) return;
  c.table.emplace(key, Entry{user, (uint32_t)NONE, seq, (uint32_t)NONE, 0});
  if (c.capacity) c.lru.insert(std::make_pair(seq, key));
  if (c.pool) c.fresh.push_back(key);
}

// An entry whose cached content is served to the request refreshes its last_used (R23).
void touch(Ctx& c, uint64_t key, uint64_t seq) {
  Entry& e = c.table.at(key);
  if (c.capacity) {
    c.lru.erase(std::make_pair(e.last_used, key));
    c.lru.insert(std::make_pair(seq, key));
  }
  e.last_used = seq;
}

// evict_lru: while the table holds more than `capacity` entries, remove the entry
// with the smallest last_used, ties broken by the smaller key; its owner and flag die with it
// (S:120).  Applied after the request's inserts ("if capacity exceeded, evict_lru is
// applied until the invariant holds"; R24).
void evict_to_capacity(Ctx& c) {
  if (!c.capacity) return;
  auto victim = c.lru.begin();
  while (c.table.size() > c.capacity) {
    while (c.table.at(victim->second).pins) ++victim;    // pinned: not evictable (R38)
    if (c.pool) c.freeq.push_back(c.table.at(victim->second).phys);   // its block is free again
    c.table.erase(victim->second);
    victim = c.lru.erase(victim);
    ++c.evictions;
  }
}

// Pinning (R38): can this request's eviction step find enough victims?  It needs size + new -
// capacity of them among the UNPINNED entries it does not use itself (its served entries and its
// new ones are the most recent and pinned by it after admission).  Checked before the request
// mutates anything; a refused request is not admitted at all.
bool pin_feasible(const Ctx& c, const std::vector<uint64_t>& served,
                  const std::vector<uint64_t>& ins) {
  if (!c.pin || !c.capacity) return true;
  int64_t fresh = 0;
  for (uint64_t k : ins) fresh += !present(c, k);
  const int64_t need = (int64_t)c.table.size() + fresh - (int64_t)c.capacity;
  if (need <= 0) return true;
  std::unordered_map<uint64_t, int> own;
  for (uint64_t k : served) own[k] = 1;
  int64_t avail = 0;
  for (auto& kv : c.table) avail += kv.second.pins == 0 && !own.count(kv.first);
  return avail >= need;
}

}  // namespace

extern "C" {

struct oracle_result {        // same field meaning as DESIGN.md §2.4 (24 bytes)
  uint32_t n_blocks;          // floor(len / bs)
  uint32_t shared_hits;       // k
  uint32_t reused;            // r
  int32_t divert_at;          // f or -1
  uint32_t flag_depth;        // depth of the entry this request flagged, 0 = none
  uint32_t bits;              // HIT=1 FULL=2 DIVERTED=4 TRUNCATED=8 FLAGGED=16
};

struct oracle_entry {
  uint64_t key;
  uint32_t owner;
  uint32_t sharer;
};

void* oracle_create(uint32_t block_size, uint64_t seed, int policy) {
  if (block_size == 0 || policy < 0 || policy > 2) return nullptr;
  Ctx* c = new Ctx();
  c->bs = block_size;
  c->seed = seed;
  c->policy = policy;
  // B = 2^32 + (splitmix64(seed) mod (p - 2^33))
  c->B = (1ULL << 32) + splitmix64(seed) % (P61 - (1ULL << 33));
  c->K.resize(block_size);
  uint64_t pw = 1;
  for (uint32_t i = 0; i < block_size; ++i) { c->K[i] = pw; pw = mulmod(pw, c->B); }
  c->M = pw;                  // M = B^bs
  c->components = 1;
  c->B2 = (1ULL << 32) + splitmix64(seed ^ SEED2_SALT) % (P61 - (1ULL << 33));
  c->K2.resize(block_size);
  pw = 1;
  for (uint32_t i = 0; i < block_size; ++i) { c->K2[i] = pw; pw = mulmod(pw, c->B2); }
  c->M2 = pw;
  c->next_seq = 0;
  c->capacity = 0;
  c->evictions = 0;
  c->pool = 0;
  c->pin = false;
  c->admitted = 0;
  return c;
}

// In-flight pinning (R38).  Needs the block pool (physical block ids name what is released).
int oracle_set_pin(void* h, int on) {
  Ctx* c = (Ctx*)h;
  if (!c->table.empty() || (on && !c->pool)) return 1;
  c->pin = on != 0;
  return 0;
}

// Release one pin on the entry holding each listed physical block (NONE entries skipped), e.g.
// a finished request's block-table row.  1 if a block holds no live pinned entry (the other
// blocks are still released).
int oracle_release(void* h, const uint32_t* phys, uint64_t n) {
  Ctx& c = *(Ctx*)h;
  int err = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (phys[i] == (uint32_t)NONE) continue;
    if (phys[i] >= c.key_of_phys.size()) { err = 1; continue; }
    auto it = c.table.find(c.key_of_phys[phys[i]]);
    if (it == c.table.end() || it->second.phys != phys[i] || it->second.pins == 0) { err = 1; continue; }
    --it->second.pins;
  }
  return err;
}

uint64_t oracle_admitted(void* h) { return ((Ctx*)h)->admitted; }

// Pin counts of the live entries, sorted by key (as oracle_dump).
uint64_t oracle_dump_pins(void* h, uint64_t* keys, uint32_t* pins, uint64_t cap) {
  Ctx& c = *(Ctx*)h;
  std::vector<std::pair<uint64_t, uint32_t>> v;
  for (auto& kv : c.table) v.push_back(std::make_pair(kv.first, kv.second.pins));
  std::sort(v.begin(), v.end());
  for (uint64_t i = 0; i < std::min<uint64_t>(cap, v.size()); ++i) {
    keys[i] = v[i].first;
    pins[i] = v[i].second;
  }
  return v.size();
}

// LRU capacity in entries (0 = unbounded).  Must be set on an empty table.
int oracle_set_capacity(void* h, uint64_t capacity) {
  Ctx* c = (Ctx*)h;
  if (!c->table.empty()) return 1;
  c->capacity = capacity;
  return 0;
}

uint64_t oracle_evictions(void* h) { return ((Ctx*)h)->evictions; }

// Physical block pool of `pool` blocks (R26-R28; 0 = off).  Must be set on an empty table.
int oracle_set_pool(void* h, uint64_t pool) {
  Ctx* c = (Ctx*)h;
  if (!c->table.empty() || pool >= NONE) return 1;
  c->pool = pool;
  c->freeq.clear();
  for (uint64_t i = 0; i < pool; ++i) c->freeq.push_back((uint32_t)i);
  c->key_of_phys.assign(pool, 0);
  return 0;
}

// Block table of the last oracle_process call: entry offsets[j]/bs + b-1 = the physical block of
// request j's block b (R27); positions no request's full block covers hold NONE.  Returns the
// number of positions (writes at most cap).
uint64_t oracle_block_table(void* h, uint32_t* out, uint64_t cap) {
  Ctx* c = (Ctx*)h;
  const uint64_t n = std::min<uint64_t>(cap, c->btab.size());
  if (n) std::memcpy(out, c->btab.data(), n * sizeof(uint32_t));
  return c->btab.size();
}

// Live entries' physical blocks, sorted by key.
uint64_t oracle_dump_phys(void* h, uint64_t* keys, uint32_t* phys, uint64_t cap) {
  Ctx& c = *(Ctx*)h;
  std::vector<std::pair<uint64_t, uint32_t>> v;
  for (auto& kv : c.table) v.push_back(std::make_pair(kv.first, kv.second.phys));
  std::sort(v.begin(), v.end());
  for (uint64_t i = 0; i < std::min<uint64_t>(cap, v.size()); ++i) {
    keys[i] = v[i].first;
    phys[i] = v[i].second;
  }
  return v.size();
}

// H-def components (1 or 2).  Must be set on an empty table.
int oracle_set_components(void* h, int components) {
  Ctx* c = (Ctx*)h;
  if (!c->table.empty() || components < 1 || components > 2) return 1;
  c->components = components;
  return 0;
}

void oracle_params2(void* h, uint64_t* B2, uint64_t* M2) {
  Ctx* c = (Ctx*)h;
  *B2 = c->B2;
  *M2 = c->M2;
}
uint64_t oracle_next_seq(void* h) { return ((Ctx*)h)->next_seq; }

void oracle_destroy(void* h) { delete (Ctx*)h; }

uint64_t oracle_size(void* h) { return ((Ctx*)h)->table.size(); }

void oracle_params(void* h, uint64_t* B, uint64_t* M) {
  Ctx* c = (Ctx*)h;
  *B = c->B;
  *M = c->M;
}

uint64_t oracle_sigma(void* h, uint32_t user) { return sigma_of(*(Ctx*)h, user); }

uint64_t oracle_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t oracle_fmix64(uint64_t x) { return fmix64(x); }

// Chain values and keys of one prompt of n_blocks full blocks: blocks 1..f are Shared, blocks
// f+1..n in Iso(user) (f = -1 -> all Shared; f = 0 -> USER_ISOLATION chain from the root).
void oracle_chain2(void* h, const uint32_t* tokens, uint32_t n_blocks, uint32_t user,
                   int32_t divert_at, uint64_t* S_out, uint64_t* S2_out, uint64_t* keys_out) {
  Ctx* c = (Ctx*)h;
  uint64_t S = 0, Mp = 1, S2 = 0, Mp2 = 1;
  const uint64_t sg = sigma_of(*c, user), sg2 = sigma2_of(*c, user);
  for (uint32_t b = 1; b <= n_blocks; ++b) {
    const uint32_t* blk = tokens + (uint64_t)(b - 1) * c->bs;
    const bool iso = divert_at >= 0 && (int64_t)b > (int64_t)divert_at;
    S = chain_step(S, Mp, block_hash(*c, blk), iso ? sg : 0);
    Mp = mulmod(Mp, c->M);
    S2 = chain_step(S2, Mp2, block_hash2(*c, blk), iso ? sg2 : 0);
    Mp2 = mulmod(Mp2, c->M2);
    if (S_out) S_out[b - 1] = S;
    if (S2_out) S2_out[b - 1] = S2;
    if (keys_out) keys_out[b - 1] = c->components == 2 ? key2_of(S, S2) : key_of(S);
  }
}

// Chain values and keys of one prompt of n_blocks full blocks: blocks 1..f are Shared, blocks
// f+1..n in Iso(user) (f = -1 -> all Shared; f = 0 -> USER_ISOLATION chain from the root).
void oracle_chain(void* h, const uint32_t* tokens, uint32_t n_blocks, uint32_t user,
                  int32_t divert_at, uint64_t* S_out, uint64_t* keys_out) {
  oracle_chain2(h, tokens, n_blocks, user, divert_at, S_out, nullptr, keys_out);
}

// Validate a whole batch first; no side effects on error.
//   1: offsets not monotone / offsets[0] != 0   2: token >= 2^20   3: user == NONE
int oracle_validate(const uint32_t* tokens, const uint64_t* offsets, uint64_t n_req,
                    const uint32_t* users) {
  if (offsets[0] != 0) return 1;
  for (uint64_t j = 0; j < n_req; ++j) {
    if (offsets[j + 1] < offsets[j]) return 1;
    if (users[j] == NONE) return 3;
  }
  for (uint64_t t = 0; t < offsets[n_req]; ++t)
    if (tokens[t] >= (1u << 20)) return 2;
  return 0;
}

// Admit n_req requests, one at a time, in order.  enforce may be NULL (= all 1,
// P:726 "detector ... always active").  Returns 0 or a validation error (nothing admitted).
int oracle_process(void* h, uint64_t n_req, const uint32_t* tokens, const uint64_t* offsets,
                   const uint32_t* users, const uint8_t* enforce, oracle_result* out) {
  Ctx& c = *(Ctx*)h;
  int err = oracle_validate(tokens, offsets, n_req, users);
  if (err) return err;
  std::vector<uint64_t> hsh, hsh2, S, S2, Kk, I;
  const bool two = c.components == 2;
  if (c.pool) c.btab.assign(n_req ? (offsets[n_req] + c.bs - 1) / c.bs : 0, (uint32_t)NONE);
  c.admitted = 0;
  std::vector<uint64_t> sv, iv;       // pinning check: the request's served / inserted keys
  for (uint64_t j = 0; j < n_req; ++j, ++c.next_seq, c.admitted = j) {
    const uint32_t u = users[j];
    const bool e = enforce ? enforce[j] != 0 : true;
    const uint32_t* tok = tokens + offsets[j];
    const uint32_t n = (uint32_t)((offsets[j + 1] - offsets[j]) / c.bs);   // partial tail never
    // hashed or cached ("block size of 16")
    hsh.assign(n + 1, 0);
    for (uint32_t b = 1; b <= n; ++b) hsh[b] = block_hash(c, tok + (uint64_t)(b - 1) * c.bs);
    hsh2.assign(n + 1, 0);
    if (two)
      for (uint32_t b = 1; b <= n; ++b) hsh2[b] = block_hash2(c, tok + (uint64_t)(b - 1) * c.bs);

    uint32_t k = 0, r = 0, flagd = 0;
    int32_t f = -1;
    c.fresh.clear();

    if (c.policy == 1) {
      // USER_ISOLATION baseline: a per-user namespace from the root.
      const uint64_t sg = sigma_of(c, u), sg2 = sigma2_of(c, u);
      I.assign(n + 1, 0);
      uint64_t T = 0, Mp = 1, T2 = 0, Mp2 = 1;
      for (uint32_t b = 1; b <= n; ++b) {
        T = chain_step(T, Mp, hsh[b], sg);
        Mp = mulmod(Mp, c.M);
        if (two) {
          T2 = chain_step(T2, Mp2, hsh2[b], sg2);
          Mp2 = mulmod(Mp2, c.M2);
        }
        I[b] = two ? key2_of(T, T2) : key_of(T);
      }
      while (r < n && present(c, I[r + 1])) ++r;
      if (c.pin) {
        sv.assign(I.begin() + 1, I.begin() + 1 + r);
        iv.assign(I.begin() + 1 + r, I.begin() + 1 + n);
        if (!pin_feasible(c, sv, iv)) return 5;
      }
      for (uint32_t b = 1; b <= r; ++b) touch(c, I[b], c.next_seq);
      for (uint32_t b = r + 1; b <= n; ++b) insert_if_absent(c, I[b], u, c.next_seq);
      f = 0;
    } else {
      // Shared chain S[b] and keys K[b]
      S.assign(n + 1, 0);
      S2.assign(n + 1, 0);
      Kk.assign(n + 1, 0);
      uint64_t Mp = 1, Mp2 = 1;
      for (uint32_t b = 1; b <= n; ++b) {
        S[b] = chain_step(S[b - 1], Mp, hsh[b], 0);
        Mp = mulmod(Mp, c.M);
        if (two) {
          S2[b] = chain_step(S2[b - 1], Mp2, hsh2[b], 0);
          Mp2 = mulmod(Mp2, c.M2);
        }
        Kk[b] = two ? key2_of(S[b], S2[b]) : key_of(S[b]);
      }
      // APC lookup: longest present prefix ("partial hits, starting from the beginning of the
      // prompt"; SPEC lookup_longest_prefix S:99-107).
      while (k < n && present(c, Kk[k + 1])) ++k;

      if (c.policy == 0) {
        // Prefix Caching baseline: full reuse, new entries tagged with owner, no flags.
        r = k;
        if (c.pin) {
          sv.assign(Kk.begin() + 1, Kk.begin() + 1 + k);
          iv.assign(Kk.begin() + 1 + k, Kk.begin() + 1 + n);
          if (!pin_feasible(c, sv, iv)) return 5;
        }
        for (uint32_t b = 1; b <= k; ++b) touch(c, Kk[b], c.next_seq);
        for (uint32_t b = k + 1; b <= n; ++b) insert_if_absent(c, Kk[b], u, c.next_seq);
      } else {
        // Detector.  Enforcement scan, only while isolation is active:
        // a hit on a flagged prefix continues only if the NEXT prefix belongs to the requester
        // (P:458); otherwise reuse stops there (R6, R7).  Flags as of before this request (R10).
        if (e) {
          for (uint32_t b = 1; b <= k; ++b) {
            if (flagged(c, Kk[b]) && !(b < k && owner_of(c, Kk[b + 1]) == u)) {
              f = (int32_t)b;
              break;
            }
          }
        }
        if (f < 0) {
          // Reuse proceeds.  Hit on an unflagged prefix owned by another user:
          // "the Detector flags this prefix" — the last reused entry e_r (R2/D2).
          // Metadata is updated even when isolation is deactivated (R11).
          r = k;
          if (c.pin) {
            sv.assign(Kk.begin() + 1, Kk.begin() + 1 + k);
            iv.assign(Kk.begin() + 1 + k, Kk.begin() + 1 + n);
            if (!pin_feasible(c, sv, iv)) return 5;
          }
          if (k >= 1 && owner_of(c, Kk[k]) != u && !flagged(c, Kk[k])) {
            c.table.at(Kk[k]).sharer = u;
            flagd = k;
          }
          // the served chain K[1..k] (incl. the entry just flagged) refreshes (R23)
          for (uint32_t b = 1; b <= k; ++b) touch(c, Kk[b], c.next_seq);
          for (uint32_t b = k + 1; b <= n; ++b) insert_if_absent(c, Kk[b], u, c.next_seq);
        } else {
          // Selective isolation: reuse stops at the flagged prefix f; the
          // remaining blocks continue in the requester's isolated namespace rooted at S[f]
          // (R3): the chain is re-derived step by step with sigma(Iso(u)).
          const uint64_t sg = sigma_of(c, u), sg2 = sigma2_of(c, u);
          I.assign(n + 1, 0);
          uint64_t T = S[f], T2 = S2[f];
          uint64_t Mpf = 1, Mpf2 = 1;
          for (uint32_t b = 1; b <= (uint32_t)f; ++b) {   // M^f (per component)
            Mpf = mulmod(Mpf, c.M);
            Mpf2 = mulmod(Mpf2, c.M2);
          }
          for (uint32_t b = (uint32_t)f + 1; b <= n; ++b) {
            T = chain_step(T, Mpf, hsh[b], sg);
            Mpf = mulmod(Mpf, c.M);
            if (two) {
              T2 = chain_step(T2, Mpf2, hsh2[b], sg2);
              Mpf2 = mulmod(Mpf2, c.M2);
            }
            I[b] = two ? key2_of(T, T2) : key_of(T);
          }
          uint32_t m = 0;
          while ((uint32_t)f + m < n && present(c, I[(uint32_t)f + m + 1])) ++m;
          r = (uint32_t)f + m;
          if (c.pin) {
            sv.assign(Kk.begin() + 1, Kk.begin() + 1 + f);
            sv.insert(sv.end(), I.begin() + 1 + f, I.begin() + 1 + r);
            iv.assign(I.begin() + 1 + r, I.begin() + 1 + n);
            if (!pin_feasible(c, sv, iv)) return 5;
          }
          // served: Shared K[1..f] (the flagged entry included; SPEC S:157 open question) and
          // Iso I[f+1..r].  Truncated Shared entries K[f+1..k] are not served (R23).
          for (uint32_t b = 1; b <= (uint32_t)f; ++b) touch(c, Kk[b], c.next_seq);
          for (uint32_t b = (uint32_t)f + 1; b <= r; ++b) touch(c, I[b], c.next_seq);
          for (uint32_t b = r + 1; b <= n; ++b) insert_if_absent(c, I[b], u, c.next_seq);
        }
      }
    }
    evict_to_capacity(c);
    if (c.pool) {
      // R26: the request's new entries take free blocks in block order (after its evictions)
      for (uint64_t key : c.fresh) {
        if (c.freeq.empty()) return 4;                       // pool exhausted (no eviction)
        c.table.at(key).phys = c.freeq.front();
        c.key_of_phys[c.freeq.front()] = key;
        c.freeq.pop_front();
      }
      // R27: block table = the physical block of the entry holding each block's key as the
      // request used it (Shared K[b] before the divert point, isolated I[b] from it, per-user
      // I[b] under USER_ISOLATION), NONE if that entry is not live after the request
      const uint64_t bt0 = offsets[j] / c.bs;
      for (uint32_t b = 1; b <= n; ++b) {
        const uint64_t key = (c.policy == 1 || (f >= 0 && (int64_t)b > (int64_t)f)) ? I[b] : Kk[b];
        auto it = c.table.find(key);
        c.btab[bt0 + b - 1] = it == c.table.end() ? (uint32_t)NONE : it->second.phys;
        if (c.pin && it != c.table.end()) ++it->second.pins;   // R38: held until released
      }
    }
    oracle_result& o = out[j];
    o.n_blocks = n;
    o.shared_hits = (c.policy == 1) ? 0 : k;
    o.reused = r;
    o.divert_at = f;
    o.flag_depth = flagd;
    o.bits = (r > 0 ? 1u : 0u) | ((n > 0 && r == n) ? 2u : 0u) | (f >= 0 ? 4u : 0u) |
             ((f >= 0 && (uint32_t)f < k) ? 8u : 0u) | (flagd > 0 ? 16u : 0u);
  }
  return 0;
}

// Table dump sorted by key.  Returns the number of entries (writes at most cap).
uint64_t oracle_dump(void* h, oracle_entry* out, uint64_t cap) {
  Ctx& c = *(Ctx*)h;
  std::vector<oracle_entry> v;
  v.reserve(c.table.size());
  for (auto& kv : c.table) v.push_back(oracle_entry{kv.first, kv.second.owner, kv.second.sharer});
  std::sort(v.begin(), v.end(),
            [](const oracle_entry& a, const oracle_entry& b) { return a.key < b.key; });
  uint64_t n = std::min<uint64_t>(cap, v.size());
  if (n) std::memcpy(out, v.data(), n * sizeof(oracle_entry));
  return v.size();
}

struct oracle_entry_ex {
  uint64_t key;
  uint32_t owner;
  uint32_t sharer;
  uint64_t last_used;
};

// Table dump with the LRU clock, sorted by key.
uint64_t oracle_dump_ex(void* h, oracle_entry_ex* out, uint64_t cap) {
  Ctx& c = *(Ctx*)h;
  std::vector<oracle_entry_ex> v;
  v.reserve(c.table.size());
  for (auto& kv : c.table)
    v.push_back(oracle_entry_ex{kv.first, kv.second.owner, kv.second.sharer, kv.second.last_used});
  std::sort(v.begin(), v.end(),
            [](const oracle_entry_ex& a, const oracle_entry_ex& b) { return a.key < b.key; });
  uint64_t n = std::min<uint64_t>(cap, v.size());
  if (n) std::memcpy(out, v.data(), n * sizeof(oracle_entry_ex));
  return v.size();
}

// Copy the table state (and clock, LRU order) of one ctx into another (warm-state reuse).
void oracle_copy_table(void* dst, void* src) {
  Ctx* d = (Ctx*)dst;
  const Ctx* s = (const Ctx*)src;
  d->table = s->table;
  d->lru = s->lru;
  d->capacity = s->capacity;
  d->evictions = s->evictions;
  d->next_seq = s->next_seq;
  d->components = s->components;
  d->pool = s->pool;
  d->freeq = s->freeq;
  d->pin = s->pin;
  d->key_of_phys = s->key_of_phys;
}

void oracle_reserve(void* h, uint64_t n) { ((Ctx*)h)->table.reserve(n); }

}  // extern "C"
