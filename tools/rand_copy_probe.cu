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

int main(int argc, char** argv) {
  CU(cuInit(0));
  CK(cudaSetDevice(0));
  const double gib = argc > 1 ? atof(argv[1]) : 2.0;
  std::vector<int> keys_list;
  for (int i = 2; i < argc; ++i) keys_list.push_back(atoi(argv[i]));
  if (keys_list.empty()) keys_list = {128, 2621, 13107, 65536};
  const size_t bytes = (size_t)(gib * (1ull << 30)) / kUnit * kUnit;
  const int units = (int)(bytes / kUnit);
  std::mt19937 rng(1);
  for (int vmm = 0; vmm < 2; ++vmm) {
    uint8_t *src, *dst;
    if (vmm) { src = vmm_alloc(bytes); dst = vmm_alloc(bytes); }
    else { CK(cudaMalloc(&src, bytes)); CK(cudaMalloc(&dst, bytes)); }
    CK(cudaMemset(src, 1, bytes));
    CK(cudaMemset(dst, 0, bytes));
    int32_t *su, *du;
    const int max_keys = 1 << 18;
    CK(cudaMalloc(&su, 4 * max_keys));
    CK(cudaMalloc(&du, 4 * max_keys));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
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
            for (int i = 0; i < keys; ++i) { hs[i] = perm[i]; hd[i] = perm[(i * 7919 + 13) % keys]; }
            CK(cudaMemcpy(su, hs.data(), 4 * keys, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(du, hd.data(), 4 * keys, cudaMemcpyHostToDevice));
          }
          const int items = keys * kLayers;
          CK(cudaEventRecord(a));
          copy_cells<<<(items + 7) / 8, 256>>>(src, dst, su, du, items);
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          if (r >= 3) tot += ms;
        }
        const double us = tot / reps * 1e3;
        const double payload = (double)keys * kLayers * kCell;
        printf("%s pool %.1f GiB keys %6d %s: %8.2f us  payload %7.1f GB/s  hbm %7.1f GB/s\n",
               vmm ? "vmm " : "cuda", gib, keys, fresh ? "fresh" : "fixed", us, payload / us / 1e3,
               2 * payload / us / 1e3);
      }
    }
  }
  return 0;
}
