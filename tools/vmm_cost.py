"""Per-call cost of the CUDA VMM driver API on this GPU (informs pool chunk sizing)."""
import ctypes as C, time
cu = C.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = C.c_int(); cu.cuDeviceGet(C.byref(dev), 0)
ctx = C.c_void_p(); cu.cuDevicePrimaryCtxRetain(C.byref(ctx), dev); cu.cuCtxSetCurrent(ctx)
class Loc(C.Structure): _fields_ = [("type", C.c_int), ("id", C.c_int)]
class AllocFlags(C.Structure): _fields_ = [("compressionType", C.c_ubyte), ("gpuDirectRDMACapable", C.c_ubyte), ("usage", C.c_ushort), ("reserved", C.c_ubyte * 4)]
class Prop(C.Structure): _fields_ = [("type", C.c_int), ("requestedHandleTypes", C.c_int), ("location", Loc), ("win32HandleMetaData", C.c_void_p), ("allocFlags", AllocFlags)]
class Access(C.Structure): _fields_ = [("location", Loc), ("flags", C.c_int)]
prop = Prop(); prop.type = 1; prop.location.type = 1; prop.location.id = 0
acc = Access(); acc.location.type = 1; acc.location.id = 0; acc.flags = 3
for mb, n in [(2, 64), (32, 32), (128, 16), (512, 8)]:
    size = mb << 20
    va = C.c_uint64()
    assert cu.cuMemAddressReserve(C.byref(va), C.c_size_t(size * n), C.c_size_t(0), C.c_uint64(0), C.c_ulonglong(0)) == 0
    hs = []
    t = [0.0] * 5
    for i in range(n):
        h = C.c_uint64()
        t0 = time.perf_counter(); r = cu.cuMemCreate(C.byref(h), C.c_size_t(size), C.byref(prop), C.c_ulonglong(0)); t[0] += time.perf_counter() - t0
        assert r == 0, r
        t0 = time.perf_counter(); assert cu.cuMemMap(C.c_uint64(va.value + i * size), C.c_size_t(size), C.c_size_t(0), h, C.c_ulonglong(0)) == 0; t[1] += time.perf_counter() - t0
        t0 = time.perf_counter(); assert cu.cuMemSetAccess(C.c_uint64(va.value + i * size), C.c_size_t(size), C.byref(acc), C.c_size_t(1)) == 0; t[2] += time.perf_counter() - t0
        hs.append(h)
    for i, h in enumerate(hs):
        t0 = time.perf_counter(); assert cu.cuMemUnmap(C.c_uint64(va.value + i * size), C.c_size_t(size)) == 0; t[3] += time.perf_counter() - t0
        t0 = time.perf_counter(); assert cu.cuMemRelease(h) == 0; t[4] += time.perf_counter() - t0
    cu.cuMemAddressFree(va, C.c_size_t(size * n))
    print(f"chunk {mb:4d} MiB: create {t[0]/n*1e3:.3f} map {t[1]/n*1e3:.3f} access {t[2]/n*1e3:.3f} unmap {t[3]/n*1e3:.3f} release {t[4]/n*1e3:.3f} ms/call")
