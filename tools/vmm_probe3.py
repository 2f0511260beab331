"""Does a range-wide cuMemUnmap over several mapped chunks leave the sub-ranges
re-mappable one chunk at a time?"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from vmm_probe2 import acc, cu, prop  # noqa: E402

size, n = 2 << 20, 4
va = C.c_uint64()
print("reserve", cu.cuMemAddressReserve(C.byref(va), C.c_size_t(size * n), C.c_size_t(0), C.c_uint64(0), C.c_ulonglong(0)))
hs = []
for i in range(n):
    h = C.c_uint64()
    cu.cuMemCreate(C.byref(h), C.c_size_t(size), C.byref(prop), C.c_ulonglong(0))
    hs.append(h)
    print("map", i, cu.cuMemMap(C.c_uint64(va.value + i * size), C.c_size_t(size), C.c_size_t(0), h, C.c_ulonglong(0)))
print("access", cu.cuMemSetAccess(C.c_uint64(va.value), C.c_size_t(size * n), C.byref(acc), C.c_size_t(1)))
print("range unmap 1..3", cu.cuMemUnmap(C.c_uint64(va.value + size), C.c_size_t(size * (n - 1))))
for i in range(1, n):
    print("remap old handle at", i, cu.cuMemMap(C.c_uint64(va.value + i * size), C.c_size_t(size), C.c_size_t(0), hs[i], C.c_ulonglong(0)))
print("unmap 1..3 individually", [cu.cuMemUnmap(C.c_uint64(va.value + i * size), C.c_size_t(size)) for i in range(1, n)])
h = C.c_uint64()
cu.cuMemCreate(C.byref(h), C.c_size_t(size), C.byref(prop), C.c_ulonglong(0))
print("map new at 1", cu.cuMemMap(C.c_uint64(va.value + size), C.c_size_t(size), C.c_size_t(0), h, C.c_ulonglong(0)))
print("access 1", cu.cuMemSetAccess(C.c_uint64(va.value + size), C.c_size_t(size), C.byref(acc), C.c_size_t(1)))
print("unmap 0..1 range", cu.cuMemUnmap(C.c_uint64(va.value), C.c_size_t(2 * size)))
print("free", cu.cuMemAddressFree(va, C.c_size_t(size * n)))
