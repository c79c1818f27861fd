// Micro-benchmark: throughput of random-slot CAS128 / CAS64 / 16-byte stores on a 64 MB table.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ ulonglong2 cas128(ulonglong2* a, ulonglong2 c, ulonglong2 v) {
  ulonglong2 o;
  asm volatile("{\n\t.reg .b128 c, v, d;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 v, {%4, %5};\n\t"
               "atom.global.cas.b128 d, [%6], c, v;\n\tmov.b128 {%0, %1}, d;\n\t}"
               : "=l"(o.x), "=l"(o.y) : "l"(c.x), "l"(c.y), "l"(v.x), "l"(v.y), "l"(a) : "memory");
  return o;
}
__device__ uint64_t mix(uint64_t x) { x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; return x; }
__global__ void k(ulonglong2* t, uint64_t mask, int n, int mode, unsigned long long* sink) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t key = mix(i + 1) | 1;
  uint64_t p = key & mask;
  unsigned long long acc = 0;
  if (mode == 0) { ulonglong2 o = cas128(&t[p], make_ulonglong2(0, 0), make_ulonglong2(key, 7)); acc = o.x; }
  else if (mode == 1) { acc = atomicCAS((unsigned long long*)&t[p].x, 0ull, key); }
  else if (mode == 2) { t[p] = make_ulonglong2(key, 7); }
  else { ulonglong2 o = cas128(&t[p], make_ulonglong2(0, 0), make_ulonglong2(key, 7));
         if (o.x != 0) acc = 1; }
  if (acc == 12345) *sink = acc;
}
int main() {
  const uint64_t slots = 1 << 22;   // 64 MB
  ulonglong2* t; cudaMalloc(&t, slots * 16);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"cas128", "cas64", "store16", "cas128(again)"};
  for (int n : {250000, 1000000}) for (int mode = 0; mode < 4; ++mode) for (int blk : {256}) {
    cudaMemset(t, 0, slots * 16);
    k<<<(n + blk - 1) / blk, blk>>>(t, slots - 1, n, mode, sink);   // warm
    cudaMemset(t, 0, slots * 16);
    cudaEventRecord(a);
    k<<<(n + blk - 1) / blk, blk>>>(t, slots - 1, n, mode, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-14s n=%8d  %8.1f us  %.2f Gop/s\n", names[mode], n, ms * 1e3, n / (ms * 1e6));
  }
  return 0;
}
