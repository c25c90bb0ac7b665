"""Multi-rank row-slab logic on CPU (gloo, world_size 2 and 3).

The GPU pipeline (paper_2407_18015_b200.distributed.fit_slab/classify_slab)
uses exactly these helpers around the CUDA calls; here the per-rank compute
is the CPU oracle (test infrastructure), so the test checks the
decomposition itself: slab bookkeeping, the global-eps all-reduce, the halo
exchange and global Monte Carlo keys give results bit-identical to one
process over the whole grid.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_18015_b200.distributed import (allreduce_range, allreduce_sums,
                                               exchange_halo_rows, slab_rows)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(world, fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


def test_slab_rows_partition():
    for H in (3, 7, 64, 1000):
        for G in (1, 2, 3, 4, 8):
            if G > 1 and H < 2 * G:  # every rank needs two rows
                with pytest.raises(ValueError):
                    slab_rows(H, 0, G)
                continue
            slabs = [slab_rows(H, g, G) for g in range(G)]
            assert slabs[0].row_begin == 0 and slabs[-1].row_end == H
            for a, b in zip(slabs, slabs[1:]):
                assert a.row_end == b.row_begin
            sizes = [s.owned for s in slabs]
            assert max(sizes) - min(sizes) <= 1
            rows = set()
            for s in slabs:
                a, b = s.stencil_rows()
                rows |= {s.local_row0 + r for r in range(a, b)}
            assert rows == set(range(1, H - 1))


def _halo_job(rank, world):
    H, W = 11, 5
    s = slab_rows(H, rank, world)
    plane = torch.full((s.local_height, W), -1.0, dtype=torch.float64)
    stack = torch.full((2, s.local_height, W), -1, dtype=torch.int16)
    for lr in range(s.local_height):
        g = s.local_row0 + lr
        if s.row_begin <= g < s.row_end:
            plane[lr] = g
            stack[0, lr] = g
            stack[1, lr] = 100 + g
    exchange_halo_rows([plane, stack], s)
    lo, hi = allreduce_range(float(rank), float(10 * rank), torch.device("cpu"))
    sums = allreduce_sums(torch.tensor([1.0, rank, 2.0], dtype=torch.float64))
    return plane.numpy(), stack.numpy(), (lo, hi), sums.numpy(), s.local_row0


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_and_allreduce(world):
    res = _run(world, _halo_job)
    for rank, (plane, stack, rng, sums, row0) in enumerate(res):
        for lr in range(plane.shape[0]):
            assert (plane[lr] == row0 + lr).all()
            assert (stack[0, lr] == row0 + lr).all() and (stack[1, lr] == 100 + row0 + lr).all()
        assert rng == (0.0, 10.0 * (world - 1))
        assert sums.tolist() == [world, sum(range(world)), 2.0 * world]


def _slab_job(rank, world):
    from oracle import critprob_oracle as orc

    H, W, M = 13, 9, 12
    vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=3)
    s = slab_rows(H, rank, world)
    mine = vals[:, s.row_begin:s.row_end]
    lo, hi = allreduce_range(float(mine.min()), float(mine.max()), torch.device("cpu"))
    eps = orc.epsilon_from_range(lo, hi)
    results = {}
    for kind, bins in (("uniform", 5), ("histogram", 4), ("epanechnikov", 5)):
        params = orc.fit(mine, kind, bins, eps=eps)
        padded = {}
        for name, arr in params.items():
            t = torch.zeros((s.local_height,) + arr.shape[1:], dtype=torch.float64)
            t[s.halo_top:s.halo_top + s.owned] = torch.from_numpy(arr)
            padded[name] = t
        planes = [padded[n] if padded[n].dim() == 2 else padded[n].permute(2, 0, 1).contiguous()
                  for n in padded]
        exchange_halo_rows(planes, s)
        for n, p in zip(list(padded), planes):
            padded[n] = p if p.dim() == 2 else p.permute(1, 2, 0)
        local = {n: t.numpy() for n, t in padded.items()}
        closed = orc.classify(local, kind)
        mc = orc.classify(local, kind, method="monte_carlo", n_samples=300, seed=5,
                          row0=s.local_row0, global_width=W)
        a, b = s.stencil_rows()
        results[kind] = ({c: closed[c][a:b] for c in ("min", "max", "saddle")},
                         {c: mc[c][a:b] for c in ("min", "max", "saddle")},
                         s.local_row0 + a)
    return results


@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_matches_single_process(world):
    from oracle import critprob_oracle as orc

    H, W, M = 13, 9, 12
    vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=3)
    res = _run(world, _slab_job)
    for kind, bins in (("uniform", 5), ("histogram", 4), ("epanechnikov", 5)):
        params = orc.fit(vals, kind, bins)
        full_c = orc.classify(params, kind)
        full_m = orc.classify(params, kind, method="monte_carlo", n_samples=300, seed=5)
        for part in res:
            closed, mc, g0 = part[kind]
            n = closed["min"].shape[0]
            for ch in ("min", "max", "saddle"):
                assert np.array_equal(closed[ch], full_c[ch][g0:g0 + n]), (kind, ch)
                assert np.array_equal(mc[ch], full_m[ch][g0:g0 + n]), (kind, ch)
