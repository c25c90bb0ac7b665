"""Wall-clock variants of cpb_run_host_models at config-5 size (diagnostic)."""
import ctypes
import sys
import time

import numpy as np

import paper_2407_18015_b200 as cpb
from paper_2407_18015_b200 import _lib

H = W = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
M = 64
lib = _lib.load()
n_ens = M * H * W
p_ens, p_out = ctypes.c_void_p(), ctypes.c_void_p()
_lib.check(lib.cpb_host_alloc(ctypes.byref(p_ens), n_ens * 4))
_lib.check(lib.cpb_host_alloc(ctypes.byref(p_out), 9 * H * W * 8 + H * W))
host = np.ctypeslib.as_array((ctypes.c_float * n_ens).from_address(p_ens.value)).reshape(M, H, W)
chunk = max(1, (1 << 30) // (M * W * 4))
for r in range(0, H, chunk):
    n = min(chunk, H - r)
    host[:, r:r + n] = cpb.synthetic_rows(r, n, W, H, M).cpu().numpy()


def run(models, with_out, reps=2):
    nm = len(models)
    outs = (ctypes.c_void_p * (3 * nm))(*[(p_out.value + q * H * W * 8) if with_out else None
                                          for q in range(3 * nm)])
    kinds = (ctypes.c_int32 * nm)(*[_lib.KIND_CODES[k] for k in models])
    binsv = (ctypes.c_int32 * nm)(*([5] * nm))
    ks = (ctypes.c_double * nm)(*[float(cpb.ModelSpec(k).k) for k in models])
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        _lib.check(lib.cpb_run_host_models(p_ens.value, M, H, W, nm, kinds, binsv, ks, 0, 0, 0, 7,
                                           outs, None))
        ts.append(time.perf_counter() - t)
    print(f"{'+'.join(models):40s} out={with_out} ms={[round(x * 1e3, 1) for x in ts]}", flush=True)


run(["uniform"], True, 1)
for models in (["uniform"], ["epanechnikov"], ["histogram"], ["uniform", "epanechnikov", "histogram"]):
    run(models, False)
    run(models, True)
t = time.perf_counter()
lib.cpb_host_free(p_ens)
lib.cpb_host_free(p_out)
print("host free ms", round((time.perf_counter() - t) * 1e3, 1))
