"""Does SetPreferredLocation = {HostNuma, id} take on this box? cudaMemAdvise_v2 on fresh
managed ranges, then cudaMemRangeGetAttribute(PreferredLocationType = 5 / Id = 6); the Device
and Host forms as controls. Prints one JSON line per case."""
import ctypes
import glob
import json
import os
import time

import torch

torch.cuda.init()
lib = os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so.12")
rt = ctypes.CDLL(lib)


class Loc(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("id", ctypes.c_int)]


rt.cudaMallocManaged.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_uint]
rt.cudaMemAdvise_v2.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, Loc]
rt.cudaMemRangeGetAttribute.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
rt.cudaFree.argtypes = [ctypes.c_void_p]
rt.cudaGetErrorName.restype = ctypes.c_char_p
PREF = 3   # cudaMemAdviseSetPreferredLocation


def query(p, n):
    t, i = ctypes.c_int(-9), ctypes.c_int(-9)
    e1 = rt.cudaMemRangeGetAttribute(ctypes.byref(t), 4, 5, p, n)
    e2 = rt.cudaMemRangeGetAttribute(ctypes.byref(i), 4, 6, p, n)
    return e1, e2, t.value, i.value


print(json.dumps({"nodes": sorted(os.path.basename(x) for x in glob.glob("/sys/devices/system/node/node*")),
                  "numa_attr": torch.cuda.get_device_properties(0).name}))
for name, loc in [("device0", Loc(1, 0)), ("host", Loc(2, 0)), ("hostnuma0", Loc(3, 0)),
                  ("hostnuma1", Loc(3, 1)), ("hostnuma_current", Loc(4, 0))]:
    p = ctypes.c_void_p()
    n = 64 << 20
    assert rt.cudaMallocManaged(ctypes.byref(p), n, 1) == 0
    t0 = time.perf_counter()
    e = rt.cudaMemAdvise_v2(p, n, PREF, loc)
    dt = time.perf_counter() - t0
    q = query(p, n)
    # touch on the host, then query again (placement happens at population)
    ctypes.memset(p, 1, n)
    q2 = query(p, n)
    print(json.dumps({"case": name, "advise_rc": e, "advise_err": rt.cudaGetErrorName(e).decode(),
                      "advise_us": round(dt * 1e6, 1), "after_advise": q, "after_touch": q2}))
    rt.cudaFree(p)
