// solid_math.cuh — device arithmetic for H-def v2, written for the GPU path only
// (the oracle has its own, unrelated implementation; the two share nothing).
//
// Field: GF(p), p = 2^61 - 1 (Mersenne).  Products are reduced by folding (2^61 == 1, 2^64 == 8
// mod p) instead of division; the per-block hash uses 32-bit limbs of the position constants so
// each token costs two IMAD.WIDE.U32 (x < 2^20+1, K_lo < 2^32, K_hi < 2^29: 16 terms fit in 64 bits).
#pragma once
#include <cstdint>

namespace solid {

constexpr uint64_t kP = (1ull << 61) - 1;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint64_t kKeyOffset = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kSigmaSalt = 0xD1B54A32D192ED03ull;
constexpr uint32_t kBS = 16;

__host__ __device__ __forceinline__ uint64_t fold61(uint64_t v) {   // v < 2^64 -> [0, p)
  v = (v & kP) + (v >> 61);
  return v >= kP ? v - kP : v;
}

// Partial fold: v < 2^64 -> a congruent value < 2^61 + 7 (not canonical; a valid mulmod operand).
__host__ __device__ __forceinline__ uint64_t fold61_lazy(uint64_t v) {
  return (v & kP) + (v >> 61);
}

__host__ __device__ __forceinline__ uint64_t addmod(uint64_t a, uint64_t b) {   // a, b < p
  uint64_t s = a + b;
  return s >= kP ? s - kP : s;
}

__host__ __device__ __forceinline__ uint64_t submod(uint64_t a, uint64_t b) {   // a, b < p
  return a >= b ? a - b : a + kP - b;
}

// a < 2^63 (need not be canonical), b < 2^61 -> canonical [0, p)
__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b) {
  uint64_t lo = a * b;
  uint64_t hi = __umul64hi(a, b);              // < 2^60: (hi << 3) + 2^61 + 7 < 2^64
  uint64_t r = (lo & kP) + (lo >> 61) + (hi << 3);
  return fold61(r);
}

__host__ __forceinline__ uint64_t mulmod_host(uint64_t a, uint64_t b) {
  unsigned __int128 pr = (unsigned __int128)a * b;
  uint64_t lo = (uint64_t)pr, hi = (uint64_t)(pr >> 64);
  return fold61((lo & kP) + (lo >> 61) + (hi << 3));
}

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// MurmurHash3 finaliser and its inverse (x ^= x >> 33 is an involution; the multipliers are odd).
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}
__host__ __device__ __forceinline__ uint64_t unfmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0x9cb4b2f8129337dbull;   // inverse of 0xc4ceb9fe1a85ec53 mod 2^64
  k ^= k >> 33;
  k *= 0x4f74430c22a54005ull;   // inverse of 0xff51afd7ed558ccd mod 2^64
  k ^= k >> 33;
  return k;
}

__host__ __device__ __forceinline__ uint64_t key_of(uint64_t S) {
  uint64_t k = fmix64(S + kKeyOffset);
  return k ? k : 1;
}
// Chain value back from a key (exact: key_of never remaps because S + offset != 0 for S < 2^61).
__host__ __device__ __forceinline__ uint64_t chain_of(uint64_t key) {
  return unfmix64(key) - kKeyOffset;
}

__host__ __device__ __forceinline__ uint64_t sigma_of(uint64_t seed, uint32_t user) {
  return 1 + splitmix64(seed ^ kSigmaSalt ^ (uint64_t)user) % (kP - 1);
}

// H-def v3: second component — its own base seed and salts; the key mixes both
// 61-bit chain values before the finaliser.
constexpr uint64_t kSeed2Salt = 0xA0761D6478BD642Full;
constexpr uint64_t kSigma2Salt = 0xE7037ED1A0B428DBull;
constexpr uint64_t kMix2 = 0x9E3779B97F4A7C15ull;
__host__ __device__ __forceinline__ uint64_t sigma2_of(uint64_t seed, uint32_t user) {
  return 1 + splitmix64(seed ^ kSigma2Salt ^ (uint64_t)user) % (kP - 1);
}
__host__ __device__ __forceinline__ uint64_t key2_of(uint64_t S, uint64_t S2) {
  uint64_t k = fmix64((S ^ (S2 * kMix2)) + kKeyOffset);
  return k ? k : 1;
}

// Inclusive warp scan of values in [0, p) under addition mod p, canonical result.  Lazy
// reduction: the first three steps add at most 8 terms (< 8p < 2^64) with plain 64-bit adds,
// one partial fold (< 2^61 + 7), the last two steps add at most 4 such values (< 2^64), then
// one canonical fold.
__device__ __forceinline__ uint64_t warp_scan_addmod(uint64_t x, int lane) {
#pragma unroll
  for (int d = 1; d < 8; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  x = fold61_lazy(x);
#pragma unroll
  for (int d = 8; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  return fold61(x);
}

}  // namespace solid
