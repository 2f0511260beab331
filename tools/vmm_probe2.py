"""VMM driver-call costs that shape the resize path: range-wide unmap / set-access over
many mapped chunks in one call, and whether cuMemRelease on a helper thread stalls
launches on the main thread."""
import ctypes as C
import threading
import time

import torch

torch.cuda.init()
torch.zeros(1, device="cuda")
cu = C.CDLL("libcuda.so.1")
ctx = C.c_void_p()
cu.cuCtxGetCurrent(C.byref(ctx))


class Loc(C.Structure):
    _fields_ = [("type", C.c_int), ("id", C.c_int)]


class AllocFlags(C.Structure):
    _fields_ = [("compressionType", C.c_ubyte), ("gpuDirectRDMACapable", C.c_ubyte),
                ("usage", C.c_ushort), ("reserved", C.c_ubyte * 4)]


class Prop(C.Structure):
    _fields_ = [("type", C.c_int), ("requestedHandleTypes", C.c_int), ("location", Loc),
                ("win32HandleMetaData", C.c_void_p), ("allocFlags", AllocFlags)]


class Access(C.Structure):
    _fields_ = [("location", Loc), ("flags", C.c_int)]


prop = Prop(); prop.type = 1; prop.location.type = 1; prop.location.id = 0
acc = Access(); acc.location.type = 1; acc.location.id = 0; acc.flags = 3


def ms(t0):
    return (time.perf_counter() - t0) * 1e3


def setup(size, n):
    va = C.c_uint64()
    assert cu.cuMemAddressReserve(C.byref(va), C.c_size_t(size * n), C.c_size_t(0), C.c_uint64(0), C.c_ulonglong(0)) == 0
    hs = []
    t0 = time.perf_counter()
    for i in range(n):
        h = C.c_uint64()
        assert cu.cuMemCreate(C.byref(h), C.c_size_t(size), C.byref(prop), C.c_ulonglong(0)) == 0
        hs.append(h)
    tc = ms(t0)
    t0 = time.perf_counter()
    for i, h in enumerate(hs):
        assert cu.cuMemMap(C.c_uint64(va.value + i * size), C.c_size_t(size), C.c_size_t(0), h, C.c_ulonglong(0)) == 0
    tm = ms(t0)
    return va, hs, tc, tm



if __name__ == "__main__":
    for mb, n, touch in [(2, 256, 0), (128, 64, 0), (512, 16, 0), (128, 64, 1), (512, 16, 1)]:
        size = mb << 20
        va, hs, tc, tm = setup(size, n)
        t0 = time.perf_counter()
        r = cu.cuMemSetAccess(C.c_uint64(va.value), C.c_size_t(size * n), C.byref(acc), C.c_size_t(1))
        ta = ms(t0)
        if touch:
            assert cu.cuMemsetD8_v2(C.c_uint64(va.value), C.c_ubyte(1), C.c_size_t(size * n)) == 0
            torch.cuda.synchronize()
        x = torch.empty(0)
        t0 = time.perf_counter()
        r2 = cu.cuMemUnmap(C.c_uint64(va.value), C.c_size_t(size * n))
        tu = ms(t0)
        t0 = time.perf_counter()
        for h in hs:
            cu.cuMemRelease(h)
        tr = ms(t0)
        cu.cuMemAddressFree(va, C.c_size_t(size * n))
        print(f"touch={touch} {mb:4d} MiB x {n:3d}: create {tc:8.2f} map {tm:7.2f} setaccess(range,1 call) rc={r} {ta:7.2f} "
              f"unmap(range,1 call) rc={r2} {tu:7.2f} release(all) {tr:8.2f} ms", flush=True)

    # helper-thread release vs main-thread launch latency
    size, n = 128 << 20, 64
    va, hs, _, _ = setup(size, n)
    cu.cuMemSetAccess(C.c_uint64(va.value), C.c_size_t(size * n), C.byref(acc), C.c_size_t(1))
    cu.cuMemUnmap(C.c_uint64(va.value), C.c_size_t(size * n))
    a = torch.randn(1 << 20, device="cuda")


    def launches(k=2000):
        torch.cuda.synchronize()
        lat = []
        for _ in range(k):
            t0 = time.perf_counter()
            a.add_(1.0)
            lat.append(ms(t0))
        torch.cuda.synchronize()
        lat.sort()
        return lat[len(lat) // 2], lat[-1], sum(lat)


    base = launches()
    done = []


    def rel():
        cu.cuCtxSetCurrent(ctx)
        t0 = time.perf_counter()
        for h in hs:
            cu.cuMemRelease(h)
        done.append(ms(t0))


    th = threading.Thread(target=rel)
    th.start()
    during = launches()
    th.join()
    cu.cuMemAddressFree(va, C.c_size_t(size * n))
    print(f"launch latency median/max/total ms: idle {base[0]:.4f}/{base[1]:.3f}/{base[2]:.1f}; "
          f"during helper-thread release of {n}x128MiB ({done[0]:.1f} ms) {during[0]:.4f}/{during[1]:.3f}/{during[2]:.1f}")
