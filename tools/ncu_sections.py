"""Warp-stall samples of one kernel split into address ranges (prologue / loops / epilogue).

    python tools/ncu_sections.py REPORT KERNEL_SUBSTR

Backward branches delimit the loops; every sample is attributed to the
innermost loop that contains its address, else to 'straight-line'.
Prints per section: samples, instructions executed, top stall reasons.
"""
import csv
import io
import re
import subprocess
import sys

path, filt = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for blk in raw.split('"Kernel Name",')[1:]:
    lines = blk.splitlines()
    if filt not in lines[0]:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    ia, isrc, isamp, iexe = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                     "Instructions Executed"))
    stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    addr = [int(r[ia], 16) for r in data]
    loops = []
    for r, a in zip(data, addr):
        m = re.search(r"BRA (0x[0-9a-f]+)", r[isrc])
        if m and int(m.group(1), 16) < a:
            loops.append((int(m.group(1), 16), a))
    def section(a):
        best = None
        for lo, hi in loops:
            if lo <= a <= hi and (best is None or hi - lo < best[1] - best[0]):
                best = (lo, hi)
        return best
    agg = {}
    for r, a in zip(data, addr):
        s = section(a)
        key = f"loop {s[0] - addr[0]:#x}-{s[1] - addr[0]:#x}" if s else "straight-line"
        d = agg.setdefault(key, {"samples": 0, "inst": 0, "stall": {}})
        d["samples"] += int(r[isamp] or 0)
        d["inst"] += int(r[iexe] or 0)
        for i in stalls:
            d["stall"][hdr[i]] = d["stall"].get(hdr[i], 0) + int(r[i] or 0)
    tot_s = sum(d["samples"] for d in agg.values())
    tot_i = sum(d["inst"] for d in agg.values())
    print(f"== {lines[0][:100]}")
    for k, d in sorted(agg.items(), key=lambda kv: -kv[1]["samples"]):
        top = sorted(d["stall"].items(), key=lambda kv: -kv[1])[:5]
        print(f"  {k:22s} samples {100 * d['samples'] / tot_s:5.1f}%  inst {100 * d['inst'] / tot_i:5.1f}%  "
              + ", ".join(f"{n[6:]} {100 * v / max(d['samples'], 1):.0f}%" for n, v in top))
