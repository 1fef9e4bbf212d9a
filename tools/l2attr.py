import ctypes, torch
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so.12") if False else None
import cuda.bindings.runtime as cr
for name in ["cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrL2CacheSize"]:
    err, v = cr.cudaDeviceGetAttribute(getattr(cr.cudaDeviceAttr, name), 0)
    print(name, err, v)
