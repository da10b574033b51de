from cuda.bindings import runtime as rt
err, v1 = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
err, v2 = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0)
err, v3 = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0)
print("max persisting L2", v1/2**20, "MiB; max window", v2/2**20, "MiB; L2", v3/2**20, "MiB")
