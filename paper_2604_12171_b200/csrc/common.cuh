// Device helpers shared by the kernels: fingerprint arithmetic, the parity
// byte expansion, 128-bit streaming loads/stores.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pl {

// engine.py:259-261: cell = (seed * 0x9E3779B97F4A7C15 + pos * 0xBF58476D1CE4E5B9) mod 2^64,
// masked to 63 bits.  Unsigned wraparound is exactly "mod 2^64".
__host__ __device__ __forceinline__ uint64_t cell_fingerprint(uint64_t seed, uint64_t pos) {
  return (seed * 0x9E3779B97F4A7C15ull + pos * 0xBF58476D1CE4E5B9ull) & 0x7FFFFFFFFFFFFFFFull;
}

// splitmix64 finaliser; the parity-mode KV byte expansion:
// 8-byte word w of layer j of a cell with fingerprint fp = splitmix64(fp ^ (j << 32 | w)).
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t expand_word(uint64_t fp, uint32_t layer, uint32_t w) {
  return splitmix64(fp ^ (((uint64_t)layer << 32) | (uint64_t)w));
}

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// plain (coherent) 128-bit load: used where the source may be written by the
// same kernel's other CTAs or is peer memory
__device__ __forceinline__ int4 ld_plain(const int4* p) {
  int4 r;
  asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ int find_item(const int64_t* offs, int n_items, int64_t t) {
  // largest i with offs[i] <= t  (offs has n_items+1 entries, offs[0] = 0)
  int lo = 0, hi = n_items - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (offs[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace pl
