#!/usr/bin/env python
"""Benchmark: Mvertices/s of the min/max/saddle probability fields (BASELINE.json metric).

Workload (BASELINE.json configs[4], the north_star target): a 16384 x 16384
grid, 64-member synthetic ensemble resident in HBM (68.7 GB float32, larger
than L2), closed-form probabilities for all three bounded models.  One STEP
= for each of uniform, epanechnikov, histogram(bins=5): fit over the members
+ closed-form min/max/saddle stencil over every interior vertex, including
the global-eps all-reduce, the halo exchange and the per-type expected-count
all-reduce when N > 1.  value = (models x interior vertices) / step time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun as row slabs (strong scaling: the grid is fixed and
split across ranks); the step time is the max over ranks.

Reported beside `value`:
  e2e          same metric through the C ABI with HOST buffers
               (cpb_run_host_models): every step copies the pinned host ensemble
               in once (fitted for every model while resident) and every model's
               three float64 planes out; N > 1 uses the slab pipeline with host
               copies
  roofline     the dominant kernel's algorithmic bytes / its CUDA-event time
               vs MEASURED_PEAKS.json hbm_gbs, plus the whole-step figure
  cpu_baseline the numpy oracle (a restatement of the reference algorithm,
               test infrastructure) on one host thread, on rows of the same
               ensemble regenerated bit-identically on the host; the same rows
               of the GPU result are checked against it (parity spot-check)
  clocks       nvidia-smi SM clocks and throttle reasons sampled during the
               timed region
`--impl reference` times the oracle port on all host cores (process pool),
rank 0 only, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODELS = ("uniform", "epanechnikov", "histogram")
METRIC = "Mvertices/sec of min/max/saddle probability fields"
PARAM_BYTES = {"uniform": 8, "epanechnikov": 16}  # compact params per pixel; histogram 8 + bins


def param_bytes(kind, bins):
    return PARAM_BYTES.get(kind, 8 + bins)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--height", type=int, default=16384)
    p.add_argument("--width", type=int, default=16384)
    p.add_argument("--members", type=int, default=64)
    p.add_argument("--bins", type=int, default=5)
    p.add_argument("--models", default=",".join(MODELS))
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--serial", action="store_true", help="no fit/stencil overlap (one stream)")
    p.add_argument("--precision", choices=("fp64", "mixed"), default="fp64",
                   help="closed form: fp64 (reference parity ~1e-15) or mixed (FP32 GL evaluation "
                        "for uniform / Epanechnikov, stated bound 1e-6)")
    p.add_argument("--fit-priority", choices=("high", "low"), default="high",
                   help="stream priority of the (overlapped) fit relative to the stencils")
    p.add_argument("--concurrent-stencils", action="store_true",
                   help="run the models' stencils on separate streams (one output buffer each)")
    p.add_argument("--fit", choices=("fused", "separate"), default="fused",
                   help="fused: one cpb_fit_multi pass over the ensemble for all models per step; "
                        "separate: one cpb_fit per model")
    p.add_argument("--fit-ctas", type=int, default=0,
                   help="persistent fit CTAs per SM while overlapping (0 = occupancy maximum)")
    p.add_argument("--profile", action="store_true", help="one short pass, for ncu")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi polling during the timed region: SM clock (median of the busy
    samples), max SM clock and the throttle reasons seen."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = f"/tmp/cpb_clocks_{os.getpid()}.csv"
        self.window = None

    def start(self):
        """Start polling every 100 ms and wait for the first sample, so that even a
        short timed region right after this call is covered."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        deadline = time.time() + 10.0
        while time.time() < deadline and self.proc.poll() is None and os.path.getsize(self.path) == 0:
            time.sleep(0.05)

    def mark(self, begin, end):
        """Wall-clock window of the timed region; samples outside it are dropped."""
        self.window = (begin, end)

    def stop(self):
        import datetime

        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)  # one more polling period past the window's end
        self.proc.terminate()
        self.proc.wait(timeout=10)
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                t = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                t = None
            rows.append((t, f))
        keep = rows
        if self.window and rows:
            b, e = self.window
            inside = [r for r in rows if r[0] is not None and b - 0.1 <= r[0] <= e + 0.1]
            keep = inside or rows
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for _, f in keep:
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        busy = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class KernelTimer:
    """CUDA events around each fit / classify launch, on the launching stream."""

    def __init__(self):
        import torch

        self.torch = torch
        self.pending = []
        self.kind = None
        self.open = None

    def __call__(self, what, begin):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self.torch.cuda.current_stream())
        if begin:
            self.open = ev
        else:
            self.pending.append((self.kind, what, self.open, ev))

    def collect(self):
        self.torch.cuda.synchronize()
        out = {}
        for kind, what, a, b in self.pending:
            out.setdefault((kind, what), []).append(a.elapsed_time(b))
        self.pending = []
        return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2407_18015_b200 as cpb
    from paper_2407_18015_b200 import distributed as D

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    H, W, M, bins = args.height, args.width, args.members, args.bins
    models = [m for m in args.models.split(",") if m]
    slab = D.slab_rows(H, rank, world)
    ens = cpb.synthetic_rows(slab.row_begin, slab.owned, W, H, M, noise_amp=0.3, seed=0)
    torch.cuda.synchronize()
    out = torch.zeros((3, slab.local_height, W), dtype=torch.float64, device=device)
    est = cpb.EstimatorSpec(precision=args.precision)
    timer = KernelTimer()
    sums = {}
    overlap = not args.serial
    if overlap and args.fit_ctas:
        from paper_2407_18015_b200 import _lib

        _lib.check(_lib.load().cpb_set_option(b"fit_ctas_per_sm", args.fit_ctas))
    # stream priorities (lower = higher priority); --fit-priority low lets the
    # stencils keep the SMs and the next step's fit fill the gaps
    fit_hi = args.fit_priority == "high"
    s_fit = torch.cuda.Stream(device=device, priority=-1 if fit_hi else 0)
    s_cls = torch.cuda.Stream(device=device, priority=0 if fit_hi else -1)
    fused = args.fit == "fused" and len(models) > 1
    if fused:
        # all models fitted in ONE pass over the ensemble (cpb_fit_multi); two
        # sets of halo-padded planes alternate between steps, so the next
        # step's fit (HBM-bound, high-priority stream) runs under this step's
        # stencils (FP64-bound, low-priority stream)
        nsets = 2 if overlap else 1
        sets = [{k: D.SlabField(cpb.ModelSpec(kind=k, bins=bins), slab, W, M, device) for k in models}
                for _ in range(nsets)]
        fitted = [torch.cuda.Event() for _ in range(nsets)]
        consumed = [torch.cuda.Event() for _ in range(nsets)]
        counter = [0]
        conc = args.concurrent_stencils
        if conc:
            s_model = {k: torch.cuda.Stream(device=device, priority=0) for k in models}
            outs = {k: torch.zeros((3, slab.local_height, W), dtype=torch.float64, device=device)
                    for k in models}

        def step():
            b = counter[0] % nsets
            counter[0] += 1
            fs = sets[b]
            timer.kind = "fused"
            with torch.cuda.stream(s_fit if overlap else torch.cuda.current_stream()):
                if overlap:
                    s_fit.wait_event(consumed[b])
                D.fit_slab_fields([fs[k] for k in models], ens, timer=timer)
                fitted[b].record()
            if conc:
                # each model's stencil on its own stream: the load-latency-bound
                # uniform and the FP64-bound stencils share the SMs
                for kind in models:
                    sk = s_model[kind]
                    sk.wait_event(fitted[b])
                    with torch.cuda.stream(sk):
                        timer.kind = kind
                        _, sums[kind] = D.classify_slab(fs[kind].dev, slab, est, out=outs[kind],
                                                        sums=True, timer=timer)
                    s_cls.wait_stream(sk)
                s_cls.record_event(consumed[b])
            else:
                with torch.cuda.stream(s_cls if overlap else torch.cuda.current_stream()):
                    if overlap:
                        s_cls.wait_event(fitted[b])
                    for kind in models:
                        timer.kind = kind
                        _, sums[kind] = D.classify_slab(fs[kind].dev, slab, est, out=out, sums=True,
                                                        timer=timer)
                    consumed[b].record()
            if overlap or conc:
                torch.cuda.current_stream().wait_stream(s_cls)
    else:
        # one reusable halo-padded field per model; eps stays on the device, so the
        # fits (HBM-bound, high-priority stream) run ahead and overlap the previous
        # model's stencil (FP64-bound, low-priority stream)
        fields = {k: D.SlabField(cpb.ModelSpec(kind=k, bins=bins), slab, W, M, device) for k in models}
        fitted = {k: torch.cuda.Event() for k in models}
        consumed = {k: torch.cuda.Event() for k in models}

        def step():
            for kind in models:
                timer.kind = kind
                with torch.cuda.stream(s_fit if overlap else torch.cuda.current_stream()):
                    if overlap:
                        s_fit.wait_event(consumed[kind])  # last step's stencil is done with the planes
                    fields[kind].fit(ens, timer=timer)
                    fitted[kind].record()
                with torch.cuda.stream(s_cls if overlap else torch.cuda.current_stream()):
                    if overlap:
                        s_cls.wait_event(fitted[kind])
                    _, sums[kind] = D.classify_slab(fields[kind].dev, slab, est, out=out, sums=True,
                                                    timer=timer)
                    consumed[kind].record()
            if overlap:
                torch.cuda.current_stream().wait_stream(s_cls)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 0 if args.profile else 3)):
        step()
    timer.collect()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    t0.record()
    for _ in range(args.steps):
        step()
    t1.record()
    torch.cuda.synchronize()
    clocks.mark(wall0, time.time())
    barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    per_kernel = timer.collect()
    ms_step = ms / args.steps
    verts = (H - 2) * (W - 2)
    value = len(models) * verts / (ms_step / 1e3) / 1e6
    expected = {k: [float(x) for x in v.cpu()] for k, v in sums.items()}

    # ---- roofline of the dominant kernel (this rank's launches)
    hbm, peak_kind = peaks()
    owned_px = slab.owned * W
    a, b = slab.stencil_rows()
    st_verts = (b - a) * (W - 2)
    kern = {}
    for (kind, what), times in per_kernel.items():
        t = statistics.mean(times)
        if what == "fit" and kind == "fused":
            nbytes = owned_px * (4 * M + sum(param_bytes(k, bins) for k in models))
            name = "fit_tma_multi_kernel"
        elif what == "fit":
            nbytes = owned_px * (4 * M + param_bytes(kind, bins))
            name = f"fit_tma_kernel<{kind}>"
        else:
            nbytes = st_verts * (param_bytes(kind, bins) + 24)
            name = {"uniform": "closed_uniform_kernel", "epanechnikov": "closed_pp_kernel<epanechnikov>",
                    "histogram": "closed_hist_tab_kernel"}[kind]
        kern[(kind, what)] = {"kernel": name, "ms": t, "bytes": nbytes, "gbs": nbytes / (t / 1e3) / 1e9}
    dom = max(kern.values(), key=lambda r: r["ms"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom["kernel"])
        except Exception:
            traffic = None
    # the stencils are FP64-bound: their pipe-level figures from the committed
    # ncu capture (profiles/ncu_fp64.json, tools/ncu_fp64.py)
    compute = None
    fpath = os.path.join(ROOT, "profiles", "ncu_fp64.json")
    if os.path.exists(fpath):
        try:
            fp = json.load(open(fpath))
            key = next((k for k in fp if k.split("<")[0] == dom["kernel"].split("<")[0]), None)
            if key:
                r = fp[key]
                compute = {"bound": "fp64", "kernel": key, "achieved": r["achieved_tflops"],
                           "peak": r["peak_tflops"], "unit": "TFLOP/s", "frac": r["flop_frac"],
                           "fp64_inst_frac": r["fp64_inst_frac"],
                           "fp64_pipe_active_pct": r["fp64_pipe_active_pct"],
                           "source": "ncu --set full (profiles/ncu_fp64.json); peak = ncu DFMA "
                                     "peak_sustained x 2 x SM clock"}
        except Exception:
            compute = None
    # 4M + 24 bytes per vertex per model (the ensemble read once
    # per model); the fused step reads it once for all models, so its minimal
    # traffic is the ensemble once + the compact planes written and read + outputs
    step_bytes = len(models) * (owned_px * 4 * M + st_verts * 24)
    planes = sum(param_bytes(k, bins) for k in models)
    min_bytes = owned_px * (4 * M + planes) + st_verts * (planes + 24 * len(models))
    roofline = {"bound": "hbm", "kernel": dom["kernel"], "achieved": round(dom["gbs"], 1),
                "peak": hbm, "peak_source": peak_kind, "unit": "GB/s",
                "frac": round(dom["gbs"] / hbm, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": dom["bytes"],
                "step": {"bytes": step_bytes,
                         "achieved": round(step_bytes / (ms_step / 1e3) / 1e9, 1),
                         "frac": round(step_bytes / (ms_step / 1e3) / 1e9 / hbm, 4),
                         "note": "e2e algorithmic bytes 4M+24 per vertex per model (SURVEY 8d)",
                         "fused_minimal_bytes": min_bytes,
                         "fused_minimal_frac": round(min_bytes / (ms_step / 1e3) / 1e9 / hbm, 4)},
                "kernels": {f"{k}/{w}": {"ms": round(r["ms"], 3), "GB/s": round(r["gbs"], 1)}
                            for (k, w), r in kern.items()},
                "compute": compute}
    # our kernels per step: range init, fit(s), weight table (histogram),
    # range->pair, pair->eps per field, one stencil per model and (closed form)
    # the two expected-count reduction kernels per model
    hist = 1 if "histogram" in models else 0
    per_model_counts = 2 if est.method == "closed_form" else 0
    if fused:
        launches_per_step = 1 + 1 + hist + 1 + (2 + per_model_counts) * len(models)
    else:
        launches_per_step = sum(5 + per_model_counts + (1 if k == "histogram" else 0) for k in models)

    # ---- parity spot-check + CPU baseline (rank 0, N = 1)
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        cpu, parity = cpu_baseline_and_parity(args, models, ens, out, est, slab)

    # ---- end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e and not args.profile:
        del ens
        torch.cuda.empty_cache()
        e2e = run_e2e(args, models, slab, rank, world, device)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "Mvertices/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f64 (histogram) / mixed f64-f32 (uniform, epanechnikov)",
            "data": "synthetic (device-generated bowl + keyed-splitmix noise, host-reproducible)",
            "config": {"workload": f"config5: {H}x{W} grid, {M} members, closed form, one step = "
                                   f"fit + min/max/saddle for {'+'.join(models)} (bins={bins})",
                       "height": H, "width": W, "members": M, "bins": bins, "models": models,
                       "vertices_per_model": verts, "parallelism": f"row-slab x{world}",
                       "fit": "one fused pass over the ensemble for all models" if fused else
                              "one pass per model",
                       "l2": "inputs (68.7 GB ensemble) larger than L2; no flush needed"},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "parity": parity,
            "clocks": clk, "gpu_launches": launches_per_step * args.steps,
            "expected_counts": expected,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline_and_parity(args, models, ens, out_unused, est, slab):
    # fp64: the reference's own grid-vs-case tolerance; mixed: the north_star's stated bound
    tol = 1e-12 if est.precision == "fp64" else 1e-6
    """Oracle on rows [r0, r0+6) of the same ensemble (host twin), 1 thread; GPU rows compared."""
    import torch

    from oracle import critprob_oracle as orc
    from paper_2407_18015_b200 import distributed as D

    try:
        from threadpoolctl import threadpool_limits
        limit = threadpool_limits(1)
    except Exception:  # pragma: no cover
        limit = None
    H, W, M, bins = args.height, args.width, args.members, args.bins
    r0, nr = H // 2 - 3, 6
    host = orc.synthetic_rows(r0, nr, W, H, M, noise_amp=0.3, seed=0)
    dev_rows = ens[:, r0:r0 + nr].cpu().numpy()
    bit_identical_input = bool(np.array_equal(host, dev_rows))
    times, errs = {}, {}
    verts = (nr - 2) * (W - 2)
    out = torch.zeros((3, slab.local_height, W), dtype=torch.float64, device=ens.device)
    for kind in models:
        model_eps = None
        dev = D.fit_slab(ens, __import__("paper_2407_18015_b200").ModelSpec(kind=kind, bins=bins), slab, W)
        model_eps = dev.eps
        D.classify_slab(dev, slab, est, out=out)
        gpu = out[:, r0 + 1:r0 + nr - 1].cpu().numpy()
        t = time.perf_counter()
        params = orc.fit(host, kind, bins, eps=model_eps)
        ref = orc.classify(params, kind)
        times[kind] = time.perf_counter() - t
        errs[kind] = max(float(np.max(np.abs(gpu[i][:, 1:-1] - ref[ch][1:-1, 1:-1])))
                         for i, ch in enumerate(("min", "max", "saddle")))
    if limit is not None:
        limit.unregister() if hasattr(limit, "unregister") else None
    total = sum(times.values())
    cpu = {"value": round(len(models) * verts / total / 1e6, 5), "unit": "Mvertices/s", "cores": 1,
           "kind": "port",
           "sample": f"rows [{r0},{r0 + nr}) of the config-5 ensemble ({verts} interior vertices "
                     f"per model, all {len(models)} models), numpy oracle, 1 thread, fit+classify",
           "seconds": {k: round(v, 3) for k, v in times.items()}}
    parity = {"rows": [r0 + 1, r0 + nr - 1], "input_bit_identical": bit_identical_input,
              "max_abs_err_vs_oracle": errs, "tolerance": tol,
              "ok": bit_identical_input and all(e <= tol for e in errs.values())}
    return cpu, parity


def run_e2e(args, models, slab, rank, world, device):
    """Same metric through host buffers: H2D of the ensemble + fit + classify + D2H, every step."""
    import torch

    import paper_2407_18015_b200 as cpb
    from paper_2407_18015_b200 import _lib
    from paper_2407_18015_b200 import distributed as D

    H, W, M, bins = args.height, args.width, args.members, args.bins
    lib = _lib.load()
    steps = max(1, min(args.steps, 2))
    if world == 1:
        n_ens = M * H * W
        p_ens = ctypes.c_void_p()
        p_out = ctypes.c_void_p()
        nm = len(models)
        _lib.check(lib.cpb_host_alloc(ctypes.byref(p_ens), n_ens * 4))
        _lib.check(lib.cpb_host_alloc(ctypes.byref(p_out), nm * 3 * H * W * 8 + H * W))
        try:
            host = np.ctypeslib.as_array((ctypes.c_float * n_ens).from_address(p_ens.value))
            host = host.reshape(M, H, W)
            chunk = max(1, (1 << 30) // (M * W * 4))
            for r in range(0, H, chunk):  # fill from the device generator, untimed
                n = min(chunk, H - r)
                host[:, r:r + n] = cpb.synthetic_rows(r, n, W, H, M).cpu().numpy()
            outs = (ctypes.c_void_p * (3 * nm))(*[p_out.value + q * H * W * 8 for q in range(3 * nm)])
            valid = p_out.value + 3 * nm * H * W * 8
            kinds = (ctypes.c_int32 * nm)(*[_lib.KIND_CODES[k] for k in models])
            binsv = (ctypes.c_int32 * nm)(*([bins] * nm))
            ks = (ctypes.c_double * nm)(*[float(cpb.ModelSpec(k).k) for k in models])

            def one():  # the reference workflow: one stack, every model (one upload)
                _lib.check(lib.cpb_run_host_models(p_ens.value, M, H, W, nm, kinds, binsv, ks, 0, 0,
                                                   0, 7, outs, valid))
            one()  # warm-up (pools, module load)
            t = time.perf_counter()
            for _ in range(steps):
                one()
            sec = (time.perf_counter() - t) / steps
            # raw pinned H2D bandwidth of this host, for context
            dev_buf = torch.empty(1 << 28, dtype=torch.float32, device=device)
            hb = torch.from_numpy(host.reshape(-1)[: 1 << 28])
            torch.cuda.synchronize()
            t = time.perf_counter()
            dev_buf.copy_(hb, non_blocking=True)
            torch.cuda.synchronize()
            h2d_gbs = (1 << 30) / (time.perf_counter() - t) / 1e9
            del dev_buf
        finally:
            lib.cpb_host_free(p_ens)
            lib.cpb_host_free(p_out)
        verts = (H - 2) * (W - 2)
        return {"value": round(nm * verts / sec / 1e6, 2), "unit": "Mvertices/s",
                "h2d_bytes_per_step": n_ens * 4,
                "d2h_bytes_per_step": nm * (3 * H * W * 8),
                "steps": steps, "ms_per_step": round(sec * 1e3, 1),
                "host_h2d_gbs": round(h2d_gbs, 1),
                "path": "cpb_run_host_models (C ABI, pinned host buffers; the ensemble crosses "
                        "PCIe once per step and is fitted for all models while resident)"}
    # N > 1: per-rank slab pipeline with host copies
    import torch.distributed as dist

    host = torch.empty((M, slab.owned, W), dtype=torch.float32).pin_memory()
    host.copy_(cpb.synthetic_rows(slab.row_begin, slab.owned, W, H, M))
    res = torch.empty((3, slab.local_height, W), dtype=torch.float64).pin_memory()
    est = cpb.EstimatorSpec()

    def one():  # one upload of the slab per step, every model fitted from it
        ens = host.to(device, non_blocking=True)
        for kind in models:
            dev = D.fit_slab(ens, cpb.ModelSpec(kind=kind, bins=bins), slab, W)
            out, _ = D.classify_slab(dev, slab, est, sums=True)
            res.copy_(out, non_blocking=True)
            torch.cuda.synchronize()
    one()
    dist.barrier()
    t = time.perf_counter()
    for _ in range(steps):
        one()
    dist.barrier()
    sec = torch.tensor([(time.perf_counter() - t) / steps], dtype=torch.float64, device=device)
    dist.all_reduce(sec, op=dist.ReduceOp.MAX)
    verts = (H - 2) * (W - 2)
    return {"value": round(len(models) * verts / float(sec[0]) / 1e6, 2), "unit": "Mvertices/s",
            "h2d_bytes_per_step": M * H * W * 4,
            "d2h_bytes_per_step": len(models) * 3 * H * W * 8, "steps": steps,
            "path": "row-slab pipeline with pinned host copies per rank"}


# ---------------------------------------------------------------------------
# reference arm: the oracle port on all host cores
# ---------------------------------------------------------------------------
_CACHE = {}


def _ref_init(counter, W, H, M, rows, stride):
    """Pool initializer: each worker regenerates its own row slab once (untimed)."""
    from oracle import critprob_oracle as orc

    with counter.get_lock():
        wid = counter.value
        counter.value += 1
    r0 = min(wid * stride, H - rows - 2)
    _CACHE["slab"] = orc.synthetic_rows(r0, rows + 2, W, H, M, noise_amp=0.3, seed=0)


def _ref_work(task):
    from oracle import critprob_oracle as orc

    models, bins, eps = task
    slab = _CACHE["slab"]
    n = 0
    for kind in models:
        ref = orc.classify(orc.fit(slab, kind, bins, eps=eps), kind)
        n += (slab.shape[1] - 2) * (slab.shape[2] - 2)
        assert ref["min"].shape == slab.shape[1:]
    return n


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp

    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    H, W, M, bins = args.height, args.width, args.members, args.bins
    models = [m for m in args.models.split(",") if m]
    cores = os.cpu_count() or 1
    total_steps = args.steps + args.warmup
    rows = 4 if total_steps <= 10 else (2 if total_steps <= 20 else 1)
    # eps of the full ensemble (distributions.py:30-36): the bowl spans [0, 5] and the noise
    # +-0.3; eps only affects degenerate pixels, of which the synthetic ensemble has none
    eps = max(1e-12, 1e-9 * (5.3 - (-0.3)))
    stride = max(rows + 2, (H - 2) // cores)
    ctx = mp.get_context("fork")
    counter = ctx.Value("i", 0)
    with ctx.Pool(cores, initializer=_ref_init, initargs=(counter, W, H, M, rows, stride)) as pool:
        work = [(models, bins, eps)] * cores
        for _ in range(args.warmup):
            pool.map(_ref_work, work, chunksize=1)
        t = time.perf_counter()
        done = 0
        for _ in range(args.steps):
            done += sum(pool.map(_ref_work, work, chunksize=1))
        sec = time.perf_counter() - t
    value = done / sec / 1e6
    sample = (f"{cores} worker processes x {rows} interior rows x {W - 2} columns of the config-5 "
              f"ensemble ({M} members) per step, fit + closed form for {'+'.join(models)}")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "Mvertices/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sec / args.steps * 1e3, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (host twin of the device generator)",
            "config": {"workload": f"config5: {H}x{W} grid, {M} members, closed form, "
                                   f"{'+'.join(models)} (bins={bins}) -- bounded row sample",
                       "height": H, "width": W, "members": M, "bins": bins, "models": models},
            "cpu_baseline": {"value": round(value, 5), "unit": "Mvertices/s", "cores": cores,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(value, 5), "unit": "Mvertices/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
