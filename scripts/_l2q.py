import ctypes, torch
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so.12") if True else None
v = ctypes.c_int()
for name, attr in [("MaxPersistingL2CacheSize", 108), ("MaxAccessPolicyWindowSize", 109), ("L2CacheSize", 89)]:
    rt.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0)
    print(name, v.value)
sz = ctypes.c_size_t()
rt.cudaDeviceGetLimit(ctypes.byref(sz), 0x06)
print("persisting limit now", sz.value)
