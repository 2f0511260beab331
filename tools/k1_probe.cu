// K1 expansion variants: write n_cells 4096-B cells whose 8-byte words are
// splitmix64(fp ^ (j << 32 | w)) (the parity expansion, csrc/common.cuh), one warp per
// cell, and time them; checks every variant is bit-identical to V0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/k1p tools/k1_probe.cu && /tmp/k1p
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
// z ^ (z >> s) with the shifted halves from the FMA pipe (multiply-high / shift-left)
template <int S>
__device__ __forceinline__ uint64_t xorshift_fma(uint64_t z, uint32_t one) {
  const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
  const uint32_t m = one << (32 - S);            // 2^(32-S), opaque to ptxas
  const uint32_t hs = __umulhi(hi, m);           // hi >> S
  const uint32_t ls = __umulhi(lo, m) + hi * m;  // (lo >> S) | (hi << (32-S))
  return z ^ (((uint64_t)hs << 32) | ls);
}
__device__ __forceinline__ uint64_t splitmix64_fma(uint64_t x, uint32_t one, int stages) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (stages & 1 ? xorshift_fma<30>(z, one) : (z ^ (z >> 30))) * 0xBF58476D1CE4E5B9ull;
  z = (stages & 2 ? xorshift_fma<27>(z, one) : (z ^ (z >> 27))) * 0x94D049BB133111EBull;
  return stages & 4 ? xorshift_fma<31>(z, one) : (z ^ (z >> 31));
}

constexpr int K = 4, CELL = 4096, VEC = CELL / 16;

__global__ void v0(uint8_t* out, const uint64_t* fps, int64_t n) {
  const int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint64_t fp = fps[t];
    for (int j = 0; j < K; ++j) {
      int4* cell = reinterpret_cast<int4*>(out + (t * K + j) * CELL);
      for (int64_t v = lane; v < VEC; v += 32) {
        uint64_t a = splitmix64(fp ^ (((uint64_t)j << 32) | (uint32_t)(2 * v)));
        uint64_t b = splitmix64(fp ^ (((uint64_t)j << 32) | (uint32_t)(2 * v + 1)));
        st_stream(cell + v, make_int4((int)(uint32_t)a, (int)(uint32_t)(a >> 32), (int)(uint32_t)b,
                                      (int)(uint32_t)(b >> 32)));
      }
    }
  }
}
// unrolled, constant store offsets; `stages` picks which xorshifts use the FMA pipe
__global__ void v1(uint8_t* out, const uint64_t* fps, int64_t n, uint32_t one, int stages) {
  const int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint64_t fp = fps[t];
#pragma unroll 1
    for (int j = 0; j < K; ++j) {
      int4* cell = reinterpret_cast<int4*>(out + (t * K + j) * CELL) + lane;
      const uint64_t base = fp ^ ((uint64_t)j << 32) ^ (uint32_t)(2 * lane);
#pragma unroll
      for (int u = 0; u < VEC / 32; ++u) {
        const uint64_t xa = base ^ (uint32_t)(64 * u);
        uint64_t a = splitmix64_fma(xa, one, stages);
        uint64_t b = splitmix64_fma(xa ^ 1u, one, stages);
        st_stream(cell + 32 * u, make_int4((int)(uint32_t)a, (int)(uint32_t)(a >> 32),
                                           (int)(uint32_t)b, (int)(uint32_t)(b >> 32)));
      }
    }
  }
}

int main() {
  const int64_t n = 2 * 256 * 2048;  // keys of the bench step: 17.2 GB of cells
  std::vector<uint64_t> h(n);
  for (int64_t i = 0; i < n; ++i) h[i] = (0x9E3779B97F4A7C15ull * (i + 7)) & 0x7fffffffffffffffull;
  uint64_t* fps;
  uint8_t *o0, *o1;
  cudaMalloc(&fps, 8 * n);
  cudaMemcpy(fps, h.data(), 8 * n, cudaMemcpyHostToDevice);
  const size_t bytes = (size_t)n * K * CELL;
  if (cudaMalloc(&o0, bytes) != cudaSuccess || cudaMalloc(&o1, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    return best;
  };
  for (int waves : {8, 16}) {
    const int grid = sms * waves;
    float t0 = timeit([&] { v0<<<grid, 256>>>(o0, fps, n); });
    printf("grid %d waves: V0 %.3f ms (%.2f TB/s)\n", waves, t0, bytes / t0 / 1e9);
    for (int stages : {0, 4, 2, 6, 7}) {
      float t1 = timeit([&] { v1<<<grid, 256>>>(o1, fps, n, 1u, stages); });
      // bit-exact against V0 (sampled words across the buffer)
      std::vector<uint64_t> a(1 << 16), b(1 << 16);
      bool ok = true;
      for (size_t off : {(size_t)0, bytes / 2, bytes - (8 << 16)}) {
        cudaMemcpy(a.data(), o0 + off, 8 << 16, cudaMemcpyDeviceToHost);
        cudaMemcpy(b.data(), o1 + off, 8 << 16, cudaMemcpyDeviceToHost);
        ok = ok && a == b;
      }
      printf("  V1 stages=%d %.3f ms (%.2f TB/s) %s\n", stages, t1, bytes / t1 / 1e9, ok ? "exact" : "MISMATCH");
    }
  }
  return 0;
}
