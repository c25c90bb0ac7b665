"""Top SASS lines by warp-stall samples for each kernel in an ncu report."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
filt = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = raw.split('"Kernel Name",')
for blk in blocks[1:]:
    lines = blk.splitlines()
    name = lines[0].strip().strip(",").strip('"')
    if filt and filt not in name:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[1:] if len(r) > i_s]
    total = sum(int(r[i_s] or 0) for r in data)
    print(f"== {name[:90]}  samples={total}")
    for r in sorted(data, key=lambda r: -int(r[i_s] or 0))[:top]:
        print(f"  {int(r[i_s]):7d} {100*int(r[i_s])/max(total,1):5.1f}%  {r[i_src].strip()[:90]}")
