"""Raw pinned H2D bandwidth over a config-5-sized buffer, repeated (diagnostic)."""
import ctypes
import time

import numpy as np
import torch

from paper_2407_18015_b200 import _lib

lib = _lib.load()
nbytes = 64 * 16384 * 16384 * 4
p = ctypes.c_void_p()
_lib.check(lib.cpb_host_alloc(ctypes.byref(p), nbytes))
host = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(p.value))
host[::4096] = 1  # touch
t_host = torch.from_numpy(host)
chunk = 256 << 20
dev = [torch.empty(chunk, dtype=torch.uint8, device="cuda") for _ in range(2)]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
for rep in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for j, off in enumerate(range(0, nbytes, chunk)):
        with torch.cuda.stream(streams[j & 1]):
            dev[j & 1].copy_(t_host[off:off + chunk], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"rep {rep}: {nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.0f} ms)", flush=True)
out = torch.empty(9 * 16384 * 16384 * 8 // 8, dtype=torch.float64, device="cuda")
q = ctypes.c_void_p()
_lib.check(lib.cpb_host_alloc(ctypes.byref(q), out.numel() * 8))
hq = torch.from_numpy(np.ctypeslib.as_array((ctypes.c_uint8 * (out.numel() * 8)).from_address(q.value)))
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    hq.view(torch.float64).copy_(out, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"d2h rep {rep}: {out.numel() * 8 / dt / 1e9:.1f} GB/s", flush=True)
import subprocess
print(subprocess.run("nvidia-smi topo -m; numactl -H 2>/dev/null | head -5; nproc; free -g", shell=True, capture_output=True, text=True).stdout)
