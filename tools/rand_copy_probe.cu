// Floor of a sparse patch round on B200: copy N random 4 KiB cells (k = 4 layers of a key,
// 64 KiB apart inside a 256 KiB unit, as the store layout) from one pool to another, one
// warp per cell, everything in flight in ONE launch.  Pools from cudaMalloc or from VMM
// (cuMemCreate, 2 MiB granularity, as csrc/vmm.cu); the key set either fixed across reps
// (warm TLBs / L2) or redrawn every rep (cold).  Prints us per launch and payload GB/s.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rcp tools/rand_copy_probe.cu -lcuda
//   /tmp/rcp [pool_GiB=2] [keys...]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)
#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { printf("%s: %d\n", #x, (int)r); exit(1); } } while (0)

constexpr int64_t kUnit = 256 << 10, kCell = 4096, kLayers = 4, kStride = 64 << 10;

__global__ void copy_cells(const uint8_t* src, uint8_t* dst, const int32_t* su, const int32_t* du,
                           int n_items) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n_items) return;
  const int key = w / kLayers, j = w % kLayers;
  const int4* s = reinterpret_cast<const int4*>(src + (int64_t)su[key] * kUnit + j * kStride);
  int4* d = reinterpret_cast<int4*>(dst + (int64_t)du[key] * kUnit + j * kStride);
  int4 b[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) b[u] = __ldcs(s + lane + 32 * u);
#pragma unroll
  for (int u = 0; u < 8; ++u) __stcs(d + lane + 32 * u, b[u]);
}

// the fused kernel's structure without the scan / resolve: a persistent grid of 2 CTAs per
// SM, each warp loops over its items with PAIR cells in flight (registers)
template <int PAIR>
__global__ void __launch_bounds__(256, 2) copy_cells_pairs(const uint8_t* src, uint8_t* dst,
                                                           const int32_t* su, const int32_t* du,
                                                           int n_items) {
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int w = w0; w < n_items; w += nw * PAIR) {
    int4 b[PAIR][8];
    int4* d[PAIR];
#pragma unroll
    for (int h = 0; h < PAIR; ++h) {
      const int it = w + h * nw;
      d[h] = nullptr;
      if (it >= n_items) continue;
      const int key = it / kLayers, j = it % kLayers;
      const int4* s = reinterpret_cast<const int4*>(src + (int64_t)su[key] * kUnit + j * kStride);
      d[h] = reinterpret_cast<int4*>(dst + (int64_t)du[key] * kUnit + j * kStride);
#pragma unroll
      for (int u = 0; u < 8; ++u) b[h][u] = __ldcs(s + lane + 32 * u);
    }
#pragma unroll
    for (int h = 0; h < PAIR; ++h)
      if (d[h])
#pragma unroll
        for (int u = 0; u < 8; ++u) __stcs(d[h] + lane + 32 * u, b[h][u]);
  }
}

// as copy_cells_pairs, but every CTA copies only the keys of its own slice of the source
// pool (as the fused kernel, whose CTAs copy the keys their bitmap chunk holds): the keys
// sorted by source unit, CTA b takes [off[b], off[b+1])
__global__ void __launch_bounds__(256, 2) copy_cells_sliced(const uint8_t* src, uint8_t* dst,
                                                            const int32_t* su, const int32_t* du,
                                                            const int32_t* off) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int a = off[blockIdx.x] * kLayers, b = off[blockIdx.x + 1] * kLayers;
  for (int w = a + warp; w < b; w += 8 * 2) {
    int4 buf[2][8];
    int4* d[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int it = w + h * 8;
      d[h] = nullptr;
      if (it >= b) continue;
      const int key = it / kLayers, j = it % kLayers;
      const int4* s = reinterpret_cast<const int4*>(src + (int64_t)su[key] * kUnit + j * kStride);
      d[h] = reinterpret_cast<int4*>(dst + (int64_t)du[key] * kUnit + j * kStride);
#pragma unroll
      for (int u = 0; u < 8; ++u) buf[h][u] = __ldcs(s + lane + 32 * u);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (d[h])
#pragma unroll
        for (int u = 0; u < 8; ++u) __stcs(d[h] + lane + 32 * u, buf[h][u]);
  }
}

// TMA bulk copies through shared memory: each warp's lane 0 keeps up to SLOTS cells in
// flight (cp.async.bulk global -> shared, mbarrier; then shared -> global, bulk group)
template <int SLOTS>
__global__ void __launch_bounds__(256, 2) copy_cells_tma(const uint8_t* src, uint8_t* dst,
                                                         const int32_t* su, const int32_t* du,
                                                         int n_items) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[8 * SLOTS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane != 0) return;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint8_t* buf = smem + (size_t)warp * SLOTS * kCell;
  for (int i = 0; i < SLOTS; ++i) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp * SLOTS + i]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  }
  asm volatile("fence.mbarrier_init.release.cluster;");
  uint32_t phase = 0;
  for (int base = w0; base < n_items; base += nw * SLOTS) {
    int4* dsts[SLOTS];
    int n = 0;
    for (int h = 0; h < SLOTS; ++h) {
      const int it = base + h * nw;
      if (it >= n_items) break;
      const int key = it / kLayers, j = it % kLayers;
      const uint8_t* s = src + (int64_t)su[key] * kUnit + j * kStride;
      dsts[h] = reinterpret_cast<int4*>(dst + (int64_t)du[key] * kUnit + j * kStride);
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp * SLOTS + h]);
      const uint32_t sm = (uint32_t)__cvta_generic_to_shared(buf + (size_t)h * kCell);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"((int)kCell));
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sm), "l"(s), "r"((int)kCell), "r"(b) : "memory");
      ++n;
    }
    for (int h = 0; h < n; ++h) {
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp * SLOTS + h]);
      asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                   ::"r"(b), "r"(phase));
      const uint32_t sm = (uint32_t)__cvta_generic_to_shared(buf + (size_t)h * kCell);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(dsts[h]), "r"(sm), "r"((int)kCell) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    phase ^= 1;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static uint8_t* vmm_alloc(size_t bytes) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = 0;
  size_t g = 0;
  CU(cuMemGetAllocationGranularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  bytes = (bytes + g - 1) / g * g;
  CUdeviceptr va;
  CU(cuMemAddressReserve(&va, bytes, 0, 0, 0));
  const size_t chunk = 64ull << 20;  // many chunks, like the store's pools
  for (size_t off = 0; off < bytes; off += chunk) {
    CUmemGenericAllocationHandle h;
    const size_t n = std::min(chunk, bytes - off);
    CU(cuMemCreate(&h, n, &p, 0));
    CU(cuMemMap(va + off, n, 0, h, 0));
  }
  CUmemAccessDesc a = {};
  a.location = p.location;
  a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(cuMemSetAccess(va, bytes, &a, 1));
  return reinterpret_cast<uint8_t*>(va);
}

static const char* kModes[] = {"warp-per-cell ", "2/SM x PAIR 2", "tma 2/SM x 3 ", "tma 1/SM x 6 ",
                               "sliced PAIR 2"};

int main(int argc, char** argv) {
  CU(cuInit(0));
  CK(cudaSetDevice(0));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(copy_cells_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 3 * (int)kCell));
  CK(cudaFuncSetAttribute(copy_cells_tma<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 6 * (int)kCell));
  const double gib = argc > 1 ? atof(argv[1]) : 2.0;
  std::vector<int> keys_list;
  for (int i = 2; i < argc; ++i) keys_list.push_back(atoi(argv[i]));
  if (keys_list.empty()) keys_list = {128, 2621, 13107, 65536};
  const size_t bytes = (size_t)(gib * (1ull << 30)) / kUnit * kUnit;
  const int units = (int)(bytes / kUnit);
  std::mt19937 rng(1);
  for (int vmm = 1; vmm < 2; ++vmm) {
    uint8_t *src, *dst;
    if (vmm) { src = vmm_alloc(bytes); dst = vmm_alloc(bytes); }
    else { CK(cudaMalloc(&src, bytes)); CK(cudaMalloc(&dst, bytes)); }
    CK(cudaMemset(src, 1, bytes));
    CK(cudaMemset(dst, 0, bytes));
    int32_t *su, *du, *off;
    const int max_keys = 1 << 18;
    CK(cudaMalloc(&off, 4 * (2 * sms + 1)));
    CK(cudaMalloc(&su, 4 * max_keys));
    CK(cudaMalloc(&du, 4 * max_keys));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int mode : {0, 1, 4, 2})
    for (int keys : keys_list) {
      if (keys > units) continue;
      for (int fresh = 0; fresh < 2; ++fresh) {
        std::vector<int32_t> hs(keys), hd(keys);
        float tot = 0;
        const int reps = 20;
        for (int r = 0; r < reps + 3; ++r) {
          if (r == 0 || fresh) {
            // distinct random units (a key per unit), sorted like a bitmap scan emits them
            std::vector<int32_t> perm(units);
            for (int i = 0; i < units; ++i) perm[i] = i;
            for (int i = 0; i < keys; ++i) std::swap(perm[i], perm[i + rng() % (units - i)]);
            std::sort(perm.begin(), perm.begin() + keys);   // bitmap order (by source unit)
            for (int i = 0; i < keys; ++i) { hs[i] = perm[i]; hd[i] = perm[(i * 7919 + 13) % keys]; }
            // slice offsets: CTA b owns source units [b*units/grid, (b+1)*units/grid)
            std::vector<int32_t> ho(2 * sms + 1, 0);
            for (int b = 0, i = 0; b <= 2 * sms; ++b) {
              const int64_t lim = (int64_t)b * units / (2 * sms);
              while (i < keys && hs[i] < lim) ++i;
              ho[b] = b == 2 * sms ? keys : i;
            }
            CK(cudaMemcpy(off, ho.data(), 4 * ho.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(su, hs.data(), 4 * keys, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(du, hd.data(), 4 * keys, cudaMemcpyHostToDevice));
          }
          const int items = keys * kLayers;
          CK(cudaEventRecord(a));
          if (mode == 0) copy_cells<<<(items + 7) / 8, 256>>>(src, dst, su, du, items);
          else if (mode == 1) copy_cells_pairs<2><<<2 * sms, 256>>>(src, dst, su, du, items);
          else if (mode == 4) copy_cells_sliced<<<2 * sms, 256>>>(src, dst, su, du, off);
          else if (mode == 2) copy_cells_tma<3><<<2 * sms, 256, 8 * 3 * kCell>>>(src, dst, su, du, items);
          else copy_cells_tma<6><<<sms, 256, 8 * 6 * kCell>>>(src, dst, su, du, items);
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          if (r >= 3) tot += ms;
        }
        const double us = tot / reps * 1e3;
        const double payload = (double)keys * kLayers * kCell;
        printf("%s %s pool %.1f GiB keys %6d %s: %8.2f us  payload %7.1f GB/s  hbm %7.1f GB/s\n",
               kModes[mode], vmm ? "vmm " : "cuda", gib, keys, fresh ? "fresh" : "fixed", us,
               payload / us / 1e3, 2 * payload / us / 1e3);
      }
    }
  }
  return 0;
}
