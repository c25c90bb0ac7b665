"""Extract FP64 work and pipe utilisation per kernel from an ncu --set full report.

    python tools/ncu_fp64.py gpurun_out/prof_full_r1b.ncu-rep > profiles/ncu_fp64.json

Per kernel: DADD / DMUL / DFMA thread instructions per cycle (GPU total), the
peak DFMA rate ncu reports (thread ops per cycle), the FP64 instruction
fraction of that peak, the FLOP rate (DFMA = 2) at the kernel's clock, and
ncu's FP64 pipe-active percentage.
"""

import csv
import io
import json
import subprocess
import sys


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}

    def get(r, name):
        return float(r[col[name]].replace(",", "")) if name in col and r[col[name]] else None

    out = {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "").split("::")[-1]
        per_cycle = {op: get(r, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
                     for op in ("dadd", "dmul", "dfma")}
        peak = get(r, "sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained")
        # the .sum peak is already the whole GPU (148 SMs x 64 DFMA lanes); the
        # cycles-per-second metric is reported in cycles per nanosecond
        clk = get(r, "smsp__cycles_elapsed.avg.per_second") or get(r, "gpc__cycles_elapsed.avg.per_second")
        clk = clk * 1e9 if clk and clk < 1e6 else clk
        if None in per_cycle.values() or peak is None:
            continue
        inst = sum(per_cycle.values())
        flops = per_cycle["dadd"] + per_cycle["dmul"] + 2 * per_cycle["dfma"]
        gpu_peak = peak
        out[short] = {
            "fp64_thread_inst_per_cycle": round(inst, 1),
            "peak_dfma_per_cycle": gpu_peak,
            "fp64_inst_frac": round(inst / gpu_peak, 4),
            "flop_frac": round(flops / (2 * gpu_peak), 4),
            "achieved_tflops": round(flops * clk / 1e12, 2) if clk else None,
            "peak_tflops": round(2 * gpu_peak * clk / 1e12, 2) if clk else None,
            "fp64_pipe_active_pct": get(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "clock_hz": clk,
            "ms": get(r, "gpu__time_duration.sum"),
        }
    out["_source"] = f"ncu --set full report {path}; tools/ncu_fp64.py"
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
