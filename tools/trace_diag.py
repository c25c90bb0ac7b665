"""Summarise CPB_HOST_TRACE timelines (diagnostic): reads stderr lines from e2e_diag."""
import sys

import numpy as np

for line in open(sys.argv[1]):
    if not line.startswith("cpb_trace_ms"):
        continue
    v = np.array([float(x) for x in line.split()[1:]])
    print(f"n={len(v)} last={v[-1]:.0f} ms  first10={np.round(v[:10], 1).tolist()}")
    d = np.diff(v)
    big = np.argsort(d)[-8:][::-1]
    print("  largest gaps:", [(int(i), round(float(d[i]), 1)) for i in big])
