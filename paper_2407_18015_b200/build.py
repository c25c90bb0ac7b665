"""Build libcritprob_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2407_18015_b200.build        (or __graft_entry__.build())

Each translation unit is compiled separately so the bit-exact ones (fit,
Monte Carlo) can be built with -fmad=false on top of their explicit
round-to-nearest intrinsics.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libcritprob_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
UNITS = {
    "cpb_fit.cu": ["-fmad=false"],
    "cpb_mc.cu": ["-fmad=false"],
    "cpb_cases.cu": ["-fmad=false"],
    "cpb_closed.cu": [],
    "cpb_capi.cu": [],
}


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out: str, deps: list) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    headers.append(os.path.join(ROOT, "include", "critprob_b200.h"))
    objs = []
    logs = []
    for unit, extra in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(BUILD, unit.replace(".cu", ".o"))
        objs.append(obj)
        if not force and not _stale(obj, [src, __file__] + headers):
            continue
        # CPB_NVCC_EXTRA: extra -D flags for developer A/B builds (tools/build_variant.sh)
        dev = os.environ.get("CPB_NVCC_EXTRA", "").split()
        cmd = [nvcc(), *ARCH, *COMMON, *extra, *dev, "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(res.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {unit}:\n{res.stderr}\n{res.stdout}")
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    if logs:
        with open(os.path.join(BUILD, "ptxas.log"), "w") as fh:
            fh.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
