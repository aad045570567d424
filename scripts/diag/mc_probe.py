import ctypes
cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuInit(0)
dev = ctypes.c_int()
cuda.cuDeviceGet(ctypes.byref(dev), 0)
val = ctypes.c_int()
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
r = cuda.cuDeviceGetAttribute(ctypes.byref(val), 132, dev)
print("multicast supported:", r, val.value)
for a, n in ((128, "HANDLE_TYPE_FABRIC?"), (111, "VIRTUAL_MEMORY_MANAGEMENT"), (102, "POSIX_FD?")):
    r = cuda.cuDeviceGetAttribute(ctypes.byref(val), a, dev); print(n, a, r, val.value)
