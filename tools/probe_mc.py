import ctypes, os
cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
n = ctypes.c_int()
cu.cuDeviceGetCount(ctypes.byref(n))
for d in range(n.value):
    dev = ctypes.c_int()
    cu.cuDeviceGet(ctypes.byref(dev), d)
    v = ctypes.c_int()
    # CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132, HANDLE_TYPE_POSIX_FD supported = 102? (VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED=102)
    for name, attr in (("MULTICAST_SUPPORTED", 132), ("VMM_SUPPORTED", 102), ("HANDLE_TYPE_POSIX_FD", 103), ("HANDLE_TYPE_FABRIC", 128)):
        r = cu.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
        print(d, name, r, v.value)
