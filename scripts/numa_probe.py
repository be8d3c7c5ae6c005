"""ut_numa_interleave on a papers-sized managed table: how long the striping takes and whether
every stripe's preferred location took (cudaMemRangeGetAttribute)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2101_07956_b200 as ut  # noqa: E402


def _preferred(addr: int, nbytes: int):
    """(type, id) of the range's preferred location (cudaMemRangeGetAttribute 5 and 6)."""
    import ctypes
    import os
    lib = os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                       "libcudart.so.12")
    rt = ctypes.CDLL(lib if os.path.exists(lib) else "libcudart.so.12")
    f = rt.cudaMemRangeGetAttribute
    f.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    typ, loc = ctypes.c_int(-1), ctypes.c_int(-1)
    assert f(ctypes.byref(typ), 4, 5, addr, nbytes) == 0
    assert f(ctypes.byref(loc), 4, 6, addr, nbytes) == 0
    return {2: "cudaMemLocationTypeHost", 3: "cudaMemLocationTypeHostNuma"}.get(typ.value, typ.value), loc.value


rows, rb = 111_000_000, 512
torch.cuda.set_device(0)
for chunk in (0, 64 << 20):
    with ut.Table.create(rows, rb, "managed") as t:
        t0 = time.perf_counter()
        try:
            t.numa_interleave(1, chunk)
            err = None
        except ut.UTError as e:
            err = str(e)
        dt = time.perf_counter() - t0
        bad = 0
        step = max(chunk, 2 << 20)
        nstripes = (rows * rb + step - 1) // step
        for k in range(0, nstripes, max(1, nstripes // 997)):
            bad += int(_preferred(t.host_addr + k * step, 4096) != ("cudaMemLocationTypeHostNuma", 0))
        print(json.dumps({"table_gb": rows * rb / 1e9, "chunk": chunk, "stripes": nstripes,
                          "advise_s": round(dt, 4), "us_per_stripe": round(dt / nstripes * 1e6, 3),
                          "sampled_not_hostnuma": bad, "error": err}))
