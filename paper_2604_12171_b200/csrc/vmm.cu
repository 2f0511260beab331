// VMM-backed pool arenas.  A KV pool of one layer group is a reserved virtual
// range; physical HBM is mapped in chunks at its tail, so KvStore.resize
// (kvstore.py:259-282) grows/shrinks real memory without moving live KV: the
// base address (and every resolved block address) stays put.  Driver entry
// points come from cudaGetDriverEntryPoint so the library links only cudart.
#include <mutex>

#include "internal.h"

namespace pl {

namespace {

struct Driver {
  decltype(&cuMemAddressReserve) AddressReserve = nullptr;
  decltype(&cuMemAddressFree) AddressFree = nullptr;
  decltype(&cuMemCreate) Create = nullptr;
  decltype(&cuMemRelease) Release = nullptr;
  decltype(&cuMemMap) Map = nullptr;
  decltype(&cuMemUnmap) Unmap = nullptr;
  decltype(&cuMemSetAccess) SetAccess = nullptr;
  decltype(&cuMemGetAllocationGranularity) Granularity = nullptr;
};

template <class F>
void load(F& fn, const char* name) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || p == nullptr)
    fail(PL_E_CUDA, std::string("driver entry point missing: ") + name);
  fn = reinterpret_cast<F>(p);
}

Driver& drv() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    load(d.AddressReserve, "cuMemAddressReserve");
    load(d.AddressFree, "cuMemAddressFree");
    load(d.Create, "cuMemCreate");
    load(d.Release, "cuMemRelease");
    load(d.Map, "cuMemMap");
    load(d.Unmap, "cuMemUnmap");
    load(d.SetAccess, "cuMemSetAccess");
    load(d.Granularity, "cuMemGetAllocationGranularity");
  });
  return d;
}

CUmemAllocationProp prop_for(int device) {
  CUmemAllocationProp p{};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  return p;
}

void set_access(CUdeviceptr va, size_t bytes, int device, const std::vector<int>& peers) {
  std::vector<CUmemAccessDesc> desc(1 + peers.size());
  for (size_t i = 0; i < desc.size(); ++i) {
    desc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    desc[i].location.id = i == 0 ? device : peers[i - 1];
    desc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  cu_check(drv().SetAccess(va, bytes, desc.data(), desc.size()), "cuMemSetAccess");
}

}  // namespace

size_t vmm_granularity(int device) {
  CUmemAllocationProp p = prop_for(device);
  size_t g = 0;
  cu_check(drv().Granularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM),
           "cuMemGetAllocationGranularity");
  return g;
}

void Arena::ensure(size_t bytes) {
  if (bytes <= mapped_bytes()) return;
  Driver& d = drv();
  size_t want_chunks = (bytes + chunk_bytes - 1) / chunk_bytes;
  size_t want_va = want_chunks * chunk_bytes;
  if (want_va > va_bytes) {
    // grow the reservation: new range (2x headroom), remap existing chunks there
    size_t new_va_bytes = std::max(want_va, va_bytes * 2);
    CUdeviceptr nva = 0;
    CUresult rr = d.AddressReserve(&nva, new_va_bytes, 0, 0, 0);
    if (rr != CUDA_SUCCESS)
      fail(PL_E_CUDA, "cuMemAddressReserve(" + std::to_string(new_va_bytes) + " B) failed with "
                          "CUresult " + std::to_string((int)rr) + " (chunk " +
                          std::to_string(chunk_bytes) + " B)");
    for (size_t i = 0; i < chunks.size(); ++i) {
      cu_check(d.Map(nva + i * chunk_bytes, chunk_bytes, 0, chunks[i], 0), "cuMemMap");
      set_access(nva + i * chunk_bytes, chunk_bytes, device, peer_devices);
    }
    if (va) {
      for (size_t i = 0; i < chunks.size(); ++i)
        cu_check(d.Unmap(va + i * chunk_bytes, chunk_bytes), "cuMemUnmap");
      cu_check(d.AddressFree(va, va_bytes), "cuMemAddressFree");
    }
    va = nva;
    va_bytes = new_va_bytes;
  }
  CUmemAllocationProp p = prop_for(device);
  size_t first = chunks.size();
  while (chunks.size() < want_chunks) {
    CUmemGenericAllocationHandle h;
    CUresult r = d.Create(&h, chunk_bytes, &p, 0);
    if (r != CUDA_SUCCESS) {
      // roll back the chunks created by this call
      for (size_t i = first; i < chunks.size(); ++i) {
        d.Unmap(va + i * chunk_bytes, chunk_bytes);
        d.Release(chunks[i]);
      }
      chunks.resize(first);
      cu_check(r, "cuMemCreate (device out of memory?)");
    }
    cu_check(d.Map(va + chunks.size() * chunk_bytes, chunk_bytes, 0, h, 0), "cuMemMap");
    set_access(va + chunks.size() * chunk_bytes, chunk_bytes, device, peer_devices);
    chunks.push_back(h);
  }
}

void Arena::trim(size_t bytes) {
  size_t keep = (bytes + chunk_bytes - 1) / chunk_bytes;
  if (keep >= chunks.size()) return;
  Driver& d = drv();
  for (size_t i = keep; i < chunks.size(); ++i) {
    cu_check(d.Unmap(va + i * chunk_bytes, chunk_bytes), "cuMemUnmap");
    cu_check(d.Release(chunks[i]), "cuMemRelease");
  }
  chunks.resize(keep);
}

void Arena::release() {
  if (!va) return;
  Driver& d = drv();
  for (size_t i = 0; i < chunks.size(); ++i) {
    d.Unmap(va + i * chunk_bytes, chunk_bytes);
    d.Release(chunks[i]);
  }
  chunks.clear();
  d.AddressFree(va, va_bytes);
  va = 0;
  va_bytes = 0;
}

void Arena::grant_peer(int dev) {
  for (int p : peer_devices)
    if (p == dev) return;
  peer_devices.push_back(dev);
  for (size_t i = 0; i < chunks.size(); ++i)
    set_access(va + i * chunk_bytes, chunk_bytes, device, peer_devices);
}

}  // namespace pl
