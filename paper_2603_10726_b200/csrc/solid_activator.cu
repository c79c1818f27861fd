// solid_activator.cu — the Activator on sm_100a.
//
// P:521-531 (§4.3): per request, selective isolation is enforced iff the hit and miss TTFT
// distributions of the most recent sliding window are distinguishable — their KDE overlap
// (P:§2.2, "the integral of the minimum of their density functions") is below θ.  The estimator
// is SPEC S:245-268's (readings R17-R21): per-token TTFT, hit/miss cutoffs on the reuse
// fraction, per-class FIFO windows, Gaussian kernels with Silverman bandwidth, a trapezoid over
// a uniform grid spanning the samples ± 3·h_max, clamp to [0, 1], fail-safe "active".
//
// Data-parallel form: a stream of completed-request samples and, per query (a request being
// admitted), the number of samples recorded before it.  Queries are non-decreasing in that count
// (sequence order), so each distinct window is computed once:
//   K_act1  per-tile class counts                (one CTA per 1024 samples)
//   K_act2  exclusive scan of the tile counts   (one CTA)
//   K_act3  per-sample ranks -> per-class compacted per-token values and prefix counts
//   K_act4  one CTA per distinct window: gather both windows into shared memory, bitonic sort
//           (quartiles), mean / sample deviation, Silverman bandwidths, KDE on the grid
//           (fp64 exp), trapezoid -> overlap and the enforce bit
//   K_act5  every query copies its window's result (binary search for the window's first query)
// All arithmetic is fp64 (the oracle's precision), so the decision overlap < θ is taken in the
// same precision on both sides.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "solid.h"

namespace solid_act {

constexpr int kTile = 1024;           // samples per K_act1/K_act3 tile (256 threads x 4)
constexpr int kThreads = 256;
constexpr uint32_t kMaxWindow = 4096;
constexpr uint32_t kMaxGrid = 8192;
constexpr uint32_t ERR_CUTS = 1u, ERR_SAMPLE = 2u;

struct Params {
  const double* ttft;
  const uint32_t* ptok;
  const double* reuse;
  uint64_t ns;
  const uint64_t* cuts;
  uint64_t nq;
  double theta, hi, lo;
  uint32_t window, min_samples, grid, p2;
  uint32_t* tile_cnt;          // [2 * tiles]: hits, misses per tile (then exclusive offsets)
  uint32_t* ph;                // [ns + 1] hits among samples [0, i)
  uint32_t* pm;                // [ns + 1] misses among samples [0, i)
  double* hv;                  // hit per-token values in sample order
  double* mv;                  // miss per-token values in sample order
  double* overlap;
  uint8_t* enforce;
  uint32_t* err;
};

__device__ __forceinline__ int klass(const Params& p, uint64_t i) {
  const double r = p.reuse[i];
  if (r >= p.hi) return 0;    // Hit
  if (r <= p.lo) return 1;    // Miss
  return 2;                   // Excluded
}

__device__ __forceinline__ uint32_t block_sum_u32(uint32_t v, uint32_t* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  uint32_t s = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  return s;
}

// Deterministic fp64 block sum (fixed tree), result broadcast to every thread.
__device__ __forceinline__ double block_sum_f64(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  return s;
}

// K_act1: per-tile counts (and sample validation: prompt_tokens >= 1, TTFT finite and > 0).
__global__ void __launch_bounds__(kThreads) k_act_tiles(Params p) {
  __shared__ uint32_t sh[kThreads / 32];
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  uint32_t h = 0, m = 0;
  for (int q = 0; q < kTile / kThreads; ++q) {
    const uint64_t i = t0 + q * kThreads + threadIdx.x;
    if (i >= p.ns) break;
    const double v = p.ttft[i];
    if (p.ptok[i] == 0 || !(v > 0.0) || !isfinite(v)) atomicOr(p.err, ERR_SAMPLE);
    const int c = klass(p, i);
    h += c == 0;
    m += c == 1;
  }
  const uint32_t H = block_sum_u32(h, sh);
  const uint32_t M = block_sum_u32(m, sh);
  if (threadIdx.x == 0) {
    p.tile_cnt[2 * blockIdx.x] = H;
    p.tile_cnt[2 * blockIdx.x + 1] = M;
  }
}

// K_act2: exclusive scan of the tile counts (one CTA; tiles processed 256 at a time).
__global__ void __launch_bounds__(kThreads) k_act_tilescan(Params p, uint32_t tiles) {
  __shared__ uint32_t sh[2][kThreads];
  uint32_t carry_h = 0, carry_m = 0;
  for (uint32_t b = 0; b < tiles; b += kThreads) {
    const uint32_t t = b + threadIdx.x;
    const uint32_t h = t < tiles ? p.tile_cnt[2 * t] : 0u, m = t < tiles ? p.tile_cnt[2 * t + 1] : 0u;
    sh[0][threadIdx.x] = h;
    sh[1][threadIdx.x] = m;
    __syncthreads();
    for (int o = 1; o < kThreads; o <<= 1) {      // Hillis-Steele inclusive scan
      const uint32_t a0 = threadIdx.x >= o ? sh[0][threadIdx.x - o] : 0u;
      const uint32_t a1 = threadIdx.x >= o ? sh[1][threadIdx.x - o] : 0u;
      __syncthreads();
      sh[0][threadIdx.x] += a0;
      sh[1][threadIdx.x] += a1;
      __syncthreads();
    }
    if (t < tiles) {
      p.tile_cnt[2 * t] = carry_h + sh[0][threadIdx.x] - h;
      p.tile_cnt[2 * t + 1] = carry_m + sh[1][threadIdx.x] - m;
    }
    carry_h += sh[0][kThreads - 1];
    carry_m += sh[1][kThreads - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.ph[p.ns] = carry_h;
    p.pm[p.ns] = carry_m;
  }
}

// K_act3: per-sample exclusive ranks within the class -> compacted values and prefix counts.
__global__ void __launch_bounds__(kThreads) k_act_compact(Params p) {
  __shared__ uint32_t sh[2][kThreads];
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  uint32_t base_h = p.tile_cnt[2 * blockIdx.x], base_m = p.tile_cnt[2 * blockIdx.x + 1];
  for (int q = 0; q < kTile / kThreads; ++q) {
    const uint64_t i = t0 + q * kThreads + threadIdx.x;
    const int c = i < p.ns ? klass(p, i) : 2;
    const uint32_t h = c == 0, m = c == 1;
    sh[0][threadIdx.x] = h;
    sh[1][threadIdx.x] = m;
    __syncthreads();
    for (int o = 1; o < kThreads; o <<= 1) {
      const uint32_t a0 = threadIdx.x >= o ? sh[0][threadIdx.x - o] : 0u;
      const uint32_t a1 = threadIdx.x >= o ? sh[1][threadIdx.x - o] : 0u;
      __syncthreads();
      sh[0][threadIdx.x] += a0;
      sh[1][threadIdx.x] += a1;
      __syncthreads();
    }
    const uint32_t rh = base_h + sh[0][threadIdx.x] - h, rm = base_m + sh[1][threadIdx.x] - m;
    if (i < p.ns) {
      p.ph[i] = rh;
      p.pm[i] = rm;
      if (c != 2) {
        const double v = p.ttft[i] / (double)max(p.ptok[i], 1u);   // per-token TTFT
        if (c == 0) p.hv[rh] = v;
        else p.mv[rm] = v;
      }
    }
    base_h += sh[0][kThreads - 1];
    base_m += sh[1][kThreads - 1];
    __syncthreads();
  }
}

// In-place ascending bitonic sort of two arrays of n (power of two) doubles in shared memory.
__device__ void bitonic2(double* a, double* b, uint32_t n) {
  for (uint32_t k = 2; k <= n; k <<= 1) {
    for (uint32_t s = k >> 1; s > 0; s >>= 1) {
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t l = i ^ s;
        if (l > i) {
          const bool up = (i & k) == 0;
          double x = a[i], y = a[l];
          if ((x > y) == up) { a[i] = y; a[l] = x; }
          x = b[i]; y = b[l];
          if ((x > y) == up) { b[i] = y; b[l] = x; }
        }
      }
      __syncthreads();
    }
  }
}

// Linear-interpolation percentile of sorted x[0..n) (R20; numpy's default method and lerp).
__device__ __forceinline__ double percentile(const double* x, uint32_t n, double q) {
  const double pos = (double)(n - 1) * q;
  const double f = floor(pos);
  const uint32_t i = (uint32_t)f;
  const double t = pos - f;
  const double a = x[i], b = x[min(i + 1, n - 1)];
  const double d = b - a;
  return t >= 0.5 ? b - d * (1.0 - t) : a + d * t;
}

__device__ double silverman(const double* x, uint32_t n, double* red) {
  double s = 0.0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  const double mean = block_sum_f64(s, red) / (double)n;
  double q = 0.0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = x[i] - mean;
    q += d * d;
  }
  const double sigma = sqrt(block_sum_f64(q, red) / (double)(n - 1));   // ddof = 1 (R19)
  const double iqr = percentile(x, n, 0.75) - percentile(x, n, 0.25);
  const double h = 0.9 * fmin(sigma, iqr / 1.34) * pow((double)n, -0.2);
  return fmax(h, 1e-9);
}

// K_act4: one CTA per distinct window (the first query of each run of equal counts).
__global__ void __launch_bounds__(kThreads) k_act_window(Params p) {
  extern __shared__ double sm[];        // A[p2] | B[p2] | m[grid]
  __shared__ double red[kThreads / 32];
  const uint64_t j = blockIdx.x + (uint64_t)blockIdx.y * gridDim.x;
  if (j >= p.nq) return;
  const uint64_t c = p.cuts[j];
  if (j > 0) {
    const uint64_t cp = p.cuts[j - 1];
    if (cp > c && threadIdx.x == 0) atomicOr(p.err, ERR_CUTS);
    if (cp == c) return;                // same window as the previous query
  }
  if (c > p.ns) {
    if (threadIdx.x == 0) atomicOr(p.err, ERR_CUTS);
    return;
  }
  const uint32_t nh = p.ph[c], nm = p.pm[c];
  const uint32_t wh = min(nh, p.window), wm = min(nm, p.window);
  const uint32_t need = max(p.min_samples, 2u);
  if (wh < need || wm < need) {         // fail-safe: active
    if (threadIdx.x == 0) {
      p.overlap[j] = __longlong_as_double(0x7ff8000000000000ll);
      p.enforce[j] = 1;
    }
    return;
  }
  double* A = sm;
  double* B = sm + p.p2;
  double* M = sm + 2 * p.p2;
  for (uint32_t i = threadIdx.x; i < p.p2; i += blockDim.x) {
    A[i] = i < wh ? p.hv[nh - wh + i] : INFINITY;
    B[i] = i < wm ? p.mv[nm - wm + i] : INFINITY;
  }
  __syncthreads();
  bitonic2(A, B, p.p2);
  const double ha = silverman(A, wh, red), hb = silverman(B, wm, red);
  const double hmax = fmax(ha, hb);
  // grid exactly as the oracle's linspace (no FMA contraction: x_k = k*step + lo, last = hi)
  const double lo = __dsub_rn(fmin(A[0], B[0]), __dmul_rn(3.0, hmax));
  const double hi = __dadd_rn(fmax(A[wh - 1], B[wm - 1]), __dmul_rn(3.0, hmax));
  const uint32_t G = p.grid;
  const double step = __ddiv_rn(__dsub_rn(hi, lo), (double)(G - 1));
  const double na = 1.0 / ((double)wh * ha * 2.5066282746310002),   // 1 / (n h sqrt(2 pi))
               nb = 1.0 / ((double)wm * hb * 2.5066282746310002);
  const double ia = 1.0 / ha, ib = 1.0 / hb;
  for (uint32_t k = threadIdx.x; k < G; k += blockDim.x) {
    const double x = k == G - 1 ? hi : __dadd_rn(__dmul_rn((double)k, step), lo);
    double fa = 0.0, fb = 0.0;
    for (uint32_t i = 0; i < wh; ++i) {
      const double d = __dsub_rn(x, A[i]) * ia;
      fa += exp(-0.5 * d * d);
    }
    for (uint32_t i = 0; i < wm; ++i) {
      const double d = __dsub_rn(x, B[i]) * ib;
      fb += exp(-0.5 * d * d);
    }
    M[k] = fmin(fa * na, fb * nb);
  }
  __syncthreads();
  double s = 0.0;
  for (uint32_t k = threadIdx.x; k + 1 < G; k += blockDim.x) {
    const double x0 = __dadd_rn(__dmul_rn((double)k, step), lo);
    const double x1 = k + 1 == G - 1 ? hi : __dadd_rn(__dmul_rn((double)(k + 1), step), lo);
    s += (x1 - x0) * (M[k] + M[k + 1]) / 2.0;
  }
  const double ov = fmin(fmax(block_sum_f64(s, red), 0.0), 1.0);
  if (threadIdx.x == 0) {
    p.overlap[j] = ov;
    p.enforce[j] = ov < p.theta ? 1 : 0;
  }
}

// K_act5: every query takes its window's result (first query with the same count).
__global__ void k_act_fill(Params p) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p.nq) return;
  const uint64_t c = p.cuts[j];
  uint64_t lo = 0, hi = j;              // lower_bound of c in cuts[0..j] (non-decreasing)
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (p.cuts[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  if (lo != j) {
    p.overlap[j] = p.overlap[lo];
    p.enforce[j] = p.enforce[lo];
  }
}

}  // namespace solid_act

using namespace solid_act;

struct solid_activator {
  solid_activator_config cfg;
  int dev = 0;
  std::string err;
  uint32_t* tile_cnt = nullptr;
  uint32_t* ph = nullptr;
  uint32_t* pm = nullptr;
  double* hv = nullptr;
  double* mv = nullptr;
  uint32_t* derr = nullptr;
  uint32_t* herr = nullptr;    // pinned
  uint32_t p2 = 0;
  size_t smem = 0;
};

static void act_free(solid_activator* a) {
  cudaFree(a->tile_cnt);
  cudaFree(a->ph);
  cudaFree(a->pm);
  cudaFree(a->hv);
  cudaFree(a->mv);
  cudaFree(a->derr);
  if (a->herr) cudaFreeHost(a->herr);
}

#define ACK(call)                                                                   \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      a->err = std::string(#call) + ": " + cudaGetErrorString(e_);                  \
      return SOLID_ERR_CUDA;                                                        \
    }                                                                               \
  } while (0)

extern "C" solid_status solid_activator_init(const solid_activator_config* cfg,
                                             solid_activator** out) {
  if (!cfg || !out) return SOLID_ERR_INVALID;
  *out = nullptr;
  if (!(cfg->theta >= 0.0 && cfg->theta <= 1.0) || !(cfg->hit_lo < cfg->hit_hi) ||
      cfg->window_len < 2 || cfg->window_len > kMaxWindow || cfg->grid < 2 ||
      cfg->grid > kMaxGrid || cfg->max_samples == 0 || cfg->max_samples >= 0xFFFFFFFFull ||
      cfg->max_queries == 0)
    return SOLID_ERR_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev)
    return SOLID_ERR_INVALID;
  solid_activator* a = new solid_activator();
  a->cfg = *cfg;
  a->dev = cfg->device;
  uint32_t p2 = 1;
  while (p2 < cfg->window_len) p2 <<= 1;
  a->p2 = p2;
  a->smem = (2 * (size_t)p2 + cfg->grid) * sizeof(double);
  const uint64_t ns = cfg->max_samples, tiles = (ns + kTile - 1) / kTile;
  bool ok = cudaSetDevice(a->dev) == cudaSuccess &&
            cudaMalloc(&a->tile_cnt, 2 * tiles * sizeof(uint32_t)) == cudaSuccess &&
            cudaMalloc(&a->ph, (ns + 1) * sizeof(uint32_t)) == cudaSuccess &&
            cudaMalloc(&a->pm, (ns + 1) * sizeof(uint32_t)) == cudaSuccess &&
            cudaMalloc(&a->hv, ns * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&a->mv, ns * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&a->derr, sizeof(uint32_t)) == cudaSuccess &&
            cudaMallocHost(&a->herr, sizeof(uint32_t)) == cudaSuccess &&
            cudaFuncSetAttribute(k_act_window, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)a->smem) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    act_free(a);
    delete a;
    return SOLID_ERR_OOM;
  }
  *out = a;
  return SOLID_OK;
}

extern "C" solid_status solid_activator_destroy(solid_activator* a) {
  if (!a) return SOLID_ERR_INVALID;
  cudaSetDevice(a->dev);
  cudaDeviceSynchronize();
  act_free(a);
  delete a;
  return SOLID_OK;
}

extern "C" const char* solid_activator_last_error(const solid_activator* a) {
  return a ? a->err.c_str() : "null activator";
}

extern "C" solid_status solid_activator_run(solid_activator* a, const double* ttft_ms,
                                            const uint32_t* prompt_tokens,
                                            const double* reuse_fraction, uint64_t n_samples,
                                            const uint64_t* cuts, uint64_t n_queries,
                                            double* overlap_out, uint8_t* enforce_out,
                                            void* stream) {
  if (!a) return SOLID_ERR_INVALID;
  if (n_samples > a->cfg.max_samples || n_queries > a->cfg.max_queries ||
      (n_samples && (!ttft_ms || !prompt_tokens || !reuse_fraction)) ||
      (n_queries && (!cuts || !overlap_out || !enforce_out))) {
    a->err = "invalid arguments (null pointer or size above the configured maximum)";
    return SOLID_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  ACK(cudaSetDevice(a->dev));
  Params p;
  p.ttft = ttft_ms;
  p.ptok = prompt_tokens;
  p.reuse = reuse_fraction;
  p.ns = n_samples;
  p.cuts = cuts;
  p.nq = n_queries;
  p.theta = a->cfg.theta;
  p.hi = a->cfg.hit_hi;
  p.lo = a->cfg.hit_lo;
  p.window = a->cfg.window_len;
  p.min_samples = a->cfg.min_samples;
  p.grid = a->cfg.grid;
  p.p2 = a->p2;
  p.tile_cnt = a->tile_cnt;
  p.ph = a->ph;
  p.pm = a->pm;
  p.hv = a->hv;
  p.mv = a->mv;
  p.overlap = overlap_out;
  p.enforce = enforce_out;
  p.err = a->derr;
  ACK(cudaMemsetAsync(a->derr, 0, sizeof(uint32_t), s));
  const uint32_t tiles = (uint32_t)((n_samples + kTile - 1) / kTile);
  if (tiles) k_act_tiles<<<tiles, kThreads, 0, s>>>(p);
  k_act_tilescan<<<1, kThreads, 0, s>>>(p, tiles);
  if (tiles) k_act_compact<<<tiles, kThreads, 0, s>>>(p);
  ACK(cudaGetLastError());
  if (n_queries) {
    const uint64_t gx = std::min<uint64_t>(n_queries, 65535), gy = (n_queries + gx - 1) / gx;
    k_act_window<<<dim3((unsigned)gx, (unsigned)gy), kThreads, a->smem, s>>>(p);
    k_act_fill<<<(unsigned)((n_queries + 255) / 256), 256, 0, s>>>(p);
    ACK(cudaGetLastError());
  }
  ACK(cudaMemcpyAsync(a->herr, a->derr, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  ACK(cudaStreamSynchronize(s));
  if (*a->herr & ERR_SAMPLE) {
    a->err = "invalid sample (prompt_tokens == 0, or TTFT not finite and > 0)";
    return SOLID_ERR_INVALID;
  }
  if (*a->herr & ERR_CUTS) {
    a->err = "cuts must be non-decreasing and <= n_samples";
    return SOLID_ERR_INVALID;
  }
  return SOLID_OK;
}
