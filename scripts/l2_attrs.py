"""Print the device's L2 size and persistence limits."""
from cuda.bindings import runtime as rt
for name in ("cudaDevAttrL2CacheSize", "cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize"):
    err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, name), 0)
    print(name, err, v)
