// Bulk-round copy: 4 KiB cells moved pool -> pool, LDG/STG (the push kernels' way) vs
// TMA bulk copies (cp.async.bulk global -> shared -> global, mbarrier-tracked), to see
// whether the copy engine of the SM beats 128-bit loads/stores at the bulk round's shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tcp tools/tma_copy_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int CELL = 4096;

__device__ __forceinline__ int4 ldcs(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stcs(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// one warp per cell pair, 2 cells in flight (as push_batched_kernel)
__global__ void __launch_bounds__(256) ldst(const uint8_t* src, uint8_t* dst, const int32_t* map,
                                            int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = 2 * w0; c < n; c += 2 * nw) {
    int4 b[2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (c + h < n) {
        const int4* s = reinterpret_cast<const int4*>(src + (c + h) * CELL);
#pragma unroll
        for (int u = 0; u < 8; ++u) b[h][u] = ldcs(s + lane + 32 * u);
      }
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (c + h < n) {
        int4* d = reinterpret_cast<int4*>(dst + (int64_t)map[c + h] * CELL);
#pragma unroll
        for (int u = 0; u < 8; ++u) stcs(d + lane + 32 * u, b[h][u]);
      }
  }
}

// TMA bulk: each warp owns S shared-memory stages of one cell; lane 0 drives them
template <int S>
__global__ void __launch_bounds__(256) tma(const uint8_t* src, uint8_t* dst, const int32_t* map,
                                           int64_t n) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[8][S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* buf = smem + (size_t)warp * S * CELL;
  if (lane == 0)
    for (int s = 0; s < S; ++s) {
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;");
  if (lane != 0) return;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t phase[S] = {};
  int64_t items[S];
  int k = 0;
  // prologue: S loads in flight
  int64_t c = w0;
  for (int s = 0; s < S; ++s, c += nw) {
    items[s] = c;
    if (c >= n) continue;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
    const uint32_t sm = (uint32_t)__cvta_generic_to_shared(buf + s * CELL);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CELL));
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sm), "l"(src + c * CELL), "r"(CELL), "r"(b) : "memory");
  }
  for (;;) {
    const int s = k % S;
    const int64_t cur = items[s];
    if (cur >= n) break;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
    const uint32_t sm = (uint32_t)__cvta_generic_to_shared(buf + s * CELL);
    // wait for the load of stage s
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 ::"r"(b), "r"(phase[s]));
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst + (int64_t)map[cur] * CELL), "r"(sm), "r"(CELL) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    // the stage's buffer is reused once its store has read it
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0));
    const int64_t nxt = cur + (int64_t)S * nw;
    items[s] = nxt;
    if (nxt < n) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CELL));
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sm), "l"(src + nxt * CELL), "r"(CELL), "r"(b) : "memory");
    }
    ++k;
  }
  asm volatile("cp.async.bulk.wait_group 0;");
}

int main() {
  const int64_t n = 4 << 20;  // 4 M cells = 17.2 GB, the bulk round's payload
  const size_t bytes = (size_t)n * CELL;
  uint8_t *src, *dst;
  int32_t* map;
  if (cudaMalloc(&src, bytes) || cudaMalloc(&dst, bytes) || cudaMalloc(&map, 4 * n)) {
    printf("alloc failed\n");
    return 1;
  }
  // destination order: 16-cell runs (a 64 KiB block layer) permuted, as fresh chains
  std::vector<int32_t> h(n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t run = i / 16, off = i % 16;
    h[i] = (int32_t)(((run * 7919) % (n / 16)) * 16 + off);
  }
  cudaMemcpy(map, h.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemset(src, 1, bytes);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto f) {
    f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      f();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    return best;
  };
  float t = timeit([&] { cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice); });
  printf("cudaMemcpy D2D      %.3f ms  %.2f TB/s (read+write)\n", t, 2 * bytes / t / 1e9);
  for (int waves : {4, 8, 16}) {
    t = timeit([&] { ldst<<<sms * waves, 256>>>(src, dst, map, n); });
    printf("LDG/STG  %2d waves   %.3f ms  %.2f TB/s\n", waves, t, 2 * bytes / t / 1e9);
  }
  for (int per : {1, 2}) {
    const size_t sm2 = 8 * 2 * CELL, sm4 = 8 * 4 * CELL;
    cudaFuncSetAttribute(tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    cudaFuncSetAttribute(tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
    t = timeit([&] { tma<2><<<sms * per, 256, sm2>>>(src, dst, map, n); });
    printf("TMA S=2  %d CTA/SM   %.3f ms  %.2f TB/s  err=%s\n", per, t, 2 * bytes / t / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    t = timeit([&] { tma<4><<<sms * per, 256, sm4>>>(src, dst, map, n); });
    printf("TMA S=4  %d CTA/SM   %.3f ms  %.2f TB/s  err=%s\n", per, t, 2 * bytes / t / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
