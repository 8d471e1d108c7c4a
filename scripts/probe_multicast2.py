"""Probe: cuMulticastCreate / AddDevice / BindMem with one device (driver API via ctypes)."""
import ctypes
c = ctypes.CDLL("libcuda.so.1")
print("cuInit", c.cuInit(0))
dev = ctypes.c_int(); print("cuDeviceGet", c.cuDeviceGet(ctypes.byref(dev), 0))
ctx = ctypes.c_void_p(); print("cuDevicePrimaryCtxRetain", c.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev)); print("cuCtxSetCurrent", c.cuCtxSetCurrent(ctx))
class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong), ("flags", ctypes.c_ulonglong)]
for ht in (0, 1, 8):  # none, POSIX fd, fabric
    p = Prop(1, 2 << 20, ht, 0)
    g = ctypes.c_size_t()
    r1 = c.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 1)
    p.size = max(g.value, 2 << 20)
    h = ctypes.c_ulonglong()
    r2 = c.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
    r3 = c.cuMulticastAddDevice(h, dev) if r2 == 0 else None
    print("handleTypes", ht, "gran rc", r1, g.value, "create rc", r2, "add rc", r3)
