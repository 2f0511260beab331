import ctypes as C
cu = C.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = C.c_int(); cu.cuDeviceGet(C.byref(dev), 0)
ctx = C.c_void_p(); cu.cuDevicePrimaryCtxRetain(C.byref(ctx), dev); cu.cuCtxSetCurrent(ctx)
for size_mb, align in [(8448, 2), (8448, 0), (132*64, 2), (132*64, 0), (130*66, 2), (130*66, 0), (8192, 2), (16384, 2), (128*64, 128)]:
    p = C.c_uint64()
    r = cu.cuMemAddressReserve(C.byref(p), C.c_size_t(size_mb << 20), C.c_size_t(align << 20), C.c_uint64(0), C.c_ulonglong(0))
    print(size_mb, "MiB align", align, "MiB ->", r, hex(p.value))
    if r == 0:
        cu.cuMemAddressFree(p, C.c_size_t(size_mb << 20))
