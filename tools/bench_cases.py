"""Per-case batch benchmark: the reference's acceptance #2 as GPU batches.

Workload (test_acceptance.py:75-97): for each bounded model (uniform,
Epanechnikov, histogram(5)) 500 seeded random_case neighbourhoods, the closed
form of each and a Monte Carlo estimate from 1e6 joint draws -- 1500 cases,
1.5e9 joint draws (7.5e9 keyed uniforms).  The reference runs it one case at a
time in numpy (~200 s of its 213 s test suite).

Prints one JSON line:
  value     joint draws per second, device time (batch resident, CUDA events)
  e2e       the same through the public API from case objects (packing, H2D,
            kernels, D2H inside the timed region), wall clock
  cpu_baseline  the CPU oracle (numpy port of mc_all_patterns + closed form)
            on a bounded sample, 1 thread, extrapolated per draw
  parity    acceptance fraction within 4 SE and oracle spot checks
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    import torch

    import paper_2407_18015_b200 as cpb
    from paper_2407_18015_b200.cases import CaseBatch

    n = int(os.environ.get("CASES_N", 1_000_000))
    per_model = int(os.environ.get("CASES_PER_MODEL", 500))
    models = ("uniform", "epanechnikov", "histogram")
    cases = {k: [cpb.random_case(1000 * i + j, model=k, neighborhood=4) for j in range(per_model)]
             for i, k in enumerate(models)}
    batches = {k: CaseBatch.pack(v) for k, v in cases.items()}
    px = np.arange(per_model, dtype=np.uint64)
    for k in models:  # warm-up (module load, smem attributes)
        batches[k].closed()
        batches[k].monte_carlo(1000, 0, px)

    # ---- device time: resident batches, closed form + 1e6-draw MC per model
    lib_stream = torch.cuda.current_stream()
    reps = 3
    times = []
    results = {}
    for _ in range(reps):
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(lib_stream)
        for k in models:
            results[k] = (batches[k].closed(), batches[k].monte_carlo(n, 0, px))
        t1.record(lib_stream)
        torch.cuda.synchronize()
        times.append(t0.elapsed_time(t1) / 1e3)
    dev_s = min(times)
    draws = len(models) * per_model * n

    # ---- end to end from case objects
    t = time.perf_counter()
    e2e_res = {}
    for k in models:
        b = CaseBatch.pack(cases[k])
        e2e_res[k] = (b.closed(), b.monte_carlo(n, 0, px))
    e2e_s = time.perf_counter() - t

    # ---- acceptance: >= 99 % of checks within 4 binomial SE
    fr = {}
    for k in models:
        closed, mc = results[k]
        se = np.sqrt(closed * (1.0 - closed) / n)
        fr[k] = float((np.abs(closed - mc) <= 4.0 * se).mean(axis=0).min())

    # ---- CPU oracle on a bounded sample (1 thread)
    from oracle import cases_oracle as co

    sample_n = int(os.environ.get("CASES_CPU_N", 200_000))
    sample_cases = 2
    t = time.perf_counter()
    spot = 0.0
    for k in models:
        for j in range(sample_cases):
            _, kind, a, b, bins, w = cpb.cases.pack_arrays([cases[k][j]])
            oc = co.unpack(kind, a, b, bins, w)[0]
            ref_closed = np.array(co.closed_triple(oc))
            ref_mc = np.array(co.mc_triple(oc, sample_n, 0, j))
            spot = max(spot, float(np.max(np.abs(ref_closed - results[k][0][j]))))
            got = batches[k].monte_carlo(sample_n, 0, px)[j] if j == 0 else None
            if got is not None and k != "epanechnikov":
                assert np.array_equal(got, ref_mc), (k, got, ref_mc)
    cpu_s = time.perf_counter() - t
    cpu_rate = len(models) * sample_cases * sample_n / cpu_s

    line = {
        "metric": "joint draws/s, acceptance #2 (closed form + MC(1e6) for 3 x 500 random cases)",
        "value": round(draws / dev_s / 1e9, 3), "unit": "Gdraws/s", "higher_is_better": True,
        "ms_total": round(dev_s * 1e3, 2), "draws": draws, "dtype": "f64",
        "data": "synthetic (seeded random_case, synth.py:124-151)",
        "config": {"workload": "test_acceptance.py:75-97 as three GPU batches", "cases": 3 * per_model,
                   "n": n},
        "e2e": {"value": round(draws / e2e_s / 1e9, 3), "unit": "Gdraws/s", "ms_total": round(e2e_s * 1e3, 1),
                "path": "paper_2407_18015_b200.cases: CaseBatch.pack -> cpb_cases_closed + cpb_cases_mc -> host"},
        "cpu_baseline": {"value": round(cpu_rate / 1e9, 6), "unit": "Gdraws/s", "cores": 1, "kind": "port",
                         "sample": f"{sample_cases} cases per model x {sample_n} draws + closed form, numpy oracle",
                         "extrapolated_total_s": round(draws / cpu_rate, 1)},
        "parity": {"within_4se_min_fraction": fr, "closed_vs_oracle_max_abs": spot,
                   "mc_vs_oracle": "bit-identical (uniform, histogram sample)"},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
