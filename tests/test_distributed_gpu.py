"""The CUDA row-slab pipeline as several PROCESSES (one rank each).

The round's GPU boxes have one GPU, so the ranks share cuda:0 and talk over
gloo, which stages the device tensors through host copies
(distributed._host_staged); on an 8 x B200 node the same code runs over NCCL
with device tensors.  Each rank runs the real kernels on its own slab:
the fused fit (SlabField / fit_slab_fields), the {-min, max} pair MAX
all-reduce -> global eps on the device, ONE packed halo exchange per
neighbour for all fields, the stencil rows (closed form and Monte Carlo with
global pixel keys) and the SUM all-reduce of the expected per-type counts.
The gathered rows must be bit-identical to one process over the whole grid
(the reference's worker-count invariance, engine.py:724-727, test_acceptance.py:219-231).
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

H, W, M = 29, 45, 12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ensemble():
    from oracle import critprob_oracle as orc

    vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=9)
    vals[:, 13, 7] = 0.5   # degenerate pixels: their result needs the GLOBAL eps
    vals[:, 3, 20] = vals[0, 3, 20]
    vals[4, 25, 30] = 40.0  # the last slab widens the global range
    return np.ascontiguousarray(vals)


def _rank_job(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        import paper_2407_18015_b200 as cpb
        from paper_2407_18015_b200 import distributed as D

        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        vals = _ensemble()
        slab = D.slab_rows(H, rank, world)
        ens = torch.as_tensor(vals[:, slab.row_begin:slab.row_end].copy(), device=dev)
        models = [cpb.ModelSpec("uniform"), cpb.ModelSpec("epanechnikov"), cpb.ModelSpec("histogram", bins=5)]
        fields = [D.SlabField(m, slab, W, M, dev) for m in models]
        D.fit_slab_fields(fields, ens)  # fused fit + MAX all-reduce + one packed halo exchange
        a, b = slab.stencil_rows()
        res = {}
        for m, f in zip(models, fields):
            out, sums = D.classify_slab(f.dev, slab, cpb.EstimatorSpec(), sums=True)
            outm, _ = D.classify_slab(f.dev, slab, cpb.EstimatorSpec("monte_carlo", n_samples=257, seed=4))
            res[m.kind] = (out[:, a:b].cpu().numpy(), outm[:, a:b].cpu().numpy(), sums.cpu().numpy(),
                           slab.local_row0 + a)
        # the synchronous path (host eps, separate fits) as well
        d = D.fit_slab(ens, cpb.ModelSpec("histogram", bins=4), slab, W)
        out, _ = D.classify_slab(d, slab, cpb.EstimatorSpec())
        res["hist4"] = (out[:, a:b].cpu().numpy(), None, None, slab.local_row0 + a)
        q.put((rank, res))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback

        q.put((rank, traceback.format_exc() + repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_ranks_as_processes_match_single_gpu(world):
    import paper_2407_18015_b200 as cpb

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_job, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(world):
        assert isinstance(got[r], dict), got[r]
    stack = cpb.EnsembleStack(_ensemble())
    for kind, bins in (("uniform", 5), ("epanechnikov", 5), ("histogram", 5), ("hist4", 4)):
        model = cpb.ModelSpec("histogram" if kind == "hist4" else kind, bins=bins)
        full = cpb.UncertainField.from_ensemble(stack, model)
        ref_c = cpb.classify_field(full)
        ref_m = cpb.classify_field(full, cpb.EstimatorSpec("monte_carlo", n_samples=257, seed=4))
        for r in range(world):
            closed, mc, sums, g0 = got[r][kind]
            n = closed.shape[1]
            for c, ch in enumerate(("min", "max", "saddle")):
                assert np.array_equal(closed[c], ref_c.channel(ch)[g0:g0 + n]), (world, kind, ch, r)
                if mc is not None:
                    assert np.array_equal(mc[c], ref_m.channel(ch)[g0:g0 + n]), (world, kind, ch, r)
            if sums is not None:
                # every rank holds the SUM all-reduced expected counts
                want = [ref_c.channel(ch).sum() for ch in ("min", "max", "saddle")]
                assert np.allclose(sums, want, rtol=1e-12, atol=1e-9), (kind, sums, want)


def test_bench_multirank_dry_run(tmp_path):
    """bench.py --gpus 2 end to end (self-launch under torch.distributed.run,
    per-rank slabs, max-over-ranks timing, rank-0 parity bands, the N > 1 e2e
    pipeline) with the test-only gloo / shared-GPU switches; the measured run
    is the same flow over NCCL with one GPU per rank."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CPB_BENCH_BACKEND="gloo", CPB_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--height", "1026",
                        "--width", "1024", "--members", "8", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, env=env, cwd=root, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["parity"]["ok"], line["parity"]
