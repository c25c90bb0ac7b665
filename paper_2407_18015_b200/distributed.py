"""Row-slab decomposition of the grid over one process per GPU.

The reference parallelises only over flat pixel chunks in one process pool
(engine.py:757-779) and every chunk carries pre-shifted copies of all five
stencil positions, so it never exchanges anything.  Here the grid is split
into G contiguous row slabs, one per rank (torchrun, NCCL over NVLink):

1. each rank fits its own rows (cpb_fit) and gets its local value range;
2. one all-reduce (MAX over [-min, max]) gives the GLOBAL range, hence the
   same eps on every rank (distributions.py:30-36 is global, fields.py:136);
3. one halo exchange sends the first / last owned row of every fitted plane
   to the rank above / below, packed into one byte buffer per neighbour (one
   send + one receive per neighbour per step, whatever the planes and bins);
4. each rank runs the stencil (closed form or Monte Carlo) on its rows --
   Monte Carlo keys use GLOBAL pixel indices (engine.py:752-754), so the
   result is bit-identical for every G;
5. optionally one all-reduce (SUM) of the per-type expected counts
   E[#min], E[#max], E[#saddle] = sum over vertices of p.

The helpers below (``slab_rows``, ``exchange_halo_rows``,
``allreduce_range``, ``allreduce_sums``) are plain torch.distributed code.
With NCCL they move device tensors directly; with gloo they stage device
tensors through host copies, so the whole CUDA slab pipeline also runs as
several processes sharing one GPU (tests/test_distributed_gpu.py) and the
pure-host logic runs on CPU (tests/test_distributed_cpu.py).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Slab:
    """Rows [row_begin, row_end) of a height-row grid owned by one rank."""

    rank: int
    world: int
    height: int
    row_begin: int
    row_end: int

    @property
    def halo_top(self) -> int:
        return 1 if self.row_begin > 0 else 0

    @property
    def halo_bottom(self) -> int:
        return 1 if self.row_end < self.height else 0

    @property
    def owned(self) -> int:
        return self.row_end - self.row_begin

    @property
    def local_height(self) -> int:
        """Rows of the local field planes: owned rows plus one halo row per neighbour."""
        return self.owned + self.halo_top + self.halo_bottom

    @property
    def local_row0(self) -> int:
        """Global row of local row 0."""
        return self.row_begin - self.halo_top

    def stencil_rows(self) -> tuple[int, int]:
        """Local rows [a, b) whose vertices this rank computes (global interior only)."""
        g0 = max(self.row_begin, 1)
        g1 = min(self.row_end, self.height - 1)
        if g1 <= g0:
            return (0, 0)
        return g0 - self.local_row0, g1 - self.local_row0


def slab_rows(height: int, rank: int, world: int) -> Slab:
    """Contiguous, balanced row slabs (the first height % world ranks get one extra row).

    Every rank must own at least two rows (one halo row is sent each way, and an
    interior rank's first and last owned rows must differ from its halo rows),
    so ``world`` may not exceed ``height // 2``.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if world > 1 and height < 2 * world:
        raise ValueError(f"{height} rows cannot be split into {world} slabs of at least two rows")
    base, extra = divmod(height, world)
    r0 = rank * base + min(rank, extra)
    r1 = r0 + base + (1 if rank < extra else 0)
    return Slab(rank, world, height, r0, r1)


def _group_world(group):
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _host_staged(t, group=None) -> bool:
    """True when ``t`` lives on a GPU but the group's backend only moves host
    tensors (gloo): the collective then runs on a host copy.  NCCL groups move
    device tensors directly (over NVLink / NVSwitch)."""
    import torch.distributed as dist

    return t.is_cuda and dist.get_backend(group) == "gloo"


def _all_reduce(t, op, group=None) -> None:
    import torch.distributed as dist

    if _host_staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)


def allreduce_range(vmin: float, vmax: float, device, group=None) -> tuple[float, float]:
    """Global (min, max) over ranks: one MAX all-reduce of [-min, max]."""
    import torch
    import torch.distributed as dist

    _, world = _group_world(group)
    if world == 1:
        return vmin, vmax
    t = torch.tensor([-vmin, vmax], dtype=torch.float64, device=device)
    _all_reduce(t, dist.ReduceOp.MAX, group)
    return -float(t[0]), float(t[1])


def _row_views(planes, row):
    """Row ``row`` of every plane as byte views: (local_height, W) planes give a
    (W,) row, (k, local_height, W) stacks a (k, W) block."""
    import torch

    out = []
    for t in planes:
        v = t[row] if t.dim() == 2 else t[:, row]
        out.append(v)
    return out


def _pack(rows):
    import torch

    return torch.cat([r.contiguous().reshape(-1).view(torch.uint8) for r in rows])


def _unpack(buf, rows) -> None:
    off = 0
    for r in rows:
        n = r.numel() * r.element_size()
        r.copy_(buf[off:off + n].view(r.dtype).view(r.shape))
        off += n


def exchange_halo_rows(planes, slab: Slab, group=None) -> None:
    """Fill the halo rows of every plane from the neighbouring ranks.

    ``planes``: tensors shaped (local_height, W) or (k, local_height, W), any
    dtypes; local row ``halo_top`` is the first owned row.  The first owned row
    of every plane goes up and the last one down, PACKED into one contiguous
    byte buffer per neighbour (one send + one receive per neighbour, however
    many planes and bins), and is unpacked into row 0 / the last row.
    """
    import torch
    import torch.distributed as dist

    rank, world = _group_world(group)
    if world == 1 or not planes:
        return
    if slab.owned < 1:
        raise ValueError("a rank with no rows cannot exchange halo rows")
    first = slab.halo_top
    last = slab.halo_top + slab.owned - 1
    staged = _host_staged(planes[0], group)

    def dev(t):
        return t.cpu() if staged else t

    ops, recv = [], []
    if slab.halo_top:
        send = dev(_pack(_row_views(planes, first)))
        buf = torch.empty_like(send)
        ops += [dist.P2POp(dist.isend, send, rank - 1, group), dist.P2POp(dist.irecv, buf, rank - 1, group)]
        recv.append((buf, _row_views(planes, 0)))
    if slab.halo_bottom:
        send = dev(_pack(_row_views(planes, last)))
        buf = torch.empty_like(send)
        ops += [dist.P2POp(dist.isend, send, rank + 1, group), dist.P2POp(dist.irecv, buf, rank + 1, group)]
        recv.append((buf, _row_views(planes, last + 1)))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    for buf, rows in recv:
        _unpack(buf.to(planes[0].device) if staged else buf, rows)


def allreduce_sums(sums, group=None):
    """SUM all-reduce of the per-type expected counts (a small float64 tensor)."""
    import torch.distributed as dist

    _, world = _group_world(group)
    if world > 1:
        _all_reduce(sums, dist.ReduceOp.SUM, group)
    return sums


# ---------------------------------------------------------------------------
# device pipeline for one rank
# ---------------------------------------------------------------------------

def _plane_views(dev):
    """(local_height, W)-shaped views of a fitted field's planes, by dtype."""
    import torch

    H, W = dev.height, dev.width
    out = []
    t = dev.tensors
    if "lo" in t:
        out += [t["lo"].view(torch.float32).view(H, W), t["hi"].view(torch.float32).view(H, W)]
    if "mean" in t:
        out += [t["mean"].view(torch.float64).view(H, W), t["spread"].view(torch.float64).view(H, W)]
    if "weights" in t:
        dt = torch.uint8 if dev.members <= 255 else torch.int16
        out.append(t["weights"].view(dt).view(dev.bins, H, W))
    return out


class SlabField:
    """Halo-padded fitted planes of one rank's slab, reusable across refits.

    ``dev`` is the DeviceField over all local rows (halo rows included);
    ``view`` a cpb_field over the owned rows only (offset base pointers and
    the full-height bin-plane stride), which is what cpb_fit writes through.
    With ``device_eps`` the global eps never visits the host: the fit's range
    words become a {-min, max} pair on the device, the pair is MAX-all-reduced
    across ranks (NCCL), and cpb_pair_to_eps writes eps where the stencil
    kernels read it (cpb_field.eps_device).
    """

    def __init__(self, model, slab: Slab, width: int, members: int, device, device_eps: bool = True):
        import torch

        from . import _lib
        from .fields import DeviceField

        self.model, self.slab, self.width, self.members = model, slab, width, members
        dev = DeviceField(model.kind, model.bins, members, slab.local_height, width,
                          row0=slab.local_row0, global_width=width, k=model.k, device=device)
        dev.allocate_fitted()
        view = _lib.CpbField.from_buffer_copy(dev.struct)
        off = slab.halo_top * width
        for name, esz in (("lo", 4), ("hi", 4), ("mean", 8), ("spread", 8)):
            base = getattr(dev.struct, name)
            if base:
                setattr(view, name, base + off * esz)
        if dev.struct.weights:
            view.weights = dev.struct.weights + off * (1 if members <= 255 else 2)
            view.plane_stride = slab.local_height * width
        view.height = slab.owned
        self.dev, self.view = dev, view
        self.device_eps = device_eps
        self.pair = torch.zeros(2, dtype=torch.float64, device=device)
        self.eps_t = torch.zeros(1, dtype=torch.float64, device=device)
        if device_eps:
            dev.struct.eps_device = self.eps_t.data_ptr()

    def fit(self, ens_slab, group=None, timer=None):
        """Fit the owned rows, make the global eps, exchange the halo rows."""
        import ctypes

        from . import _lib

        lib = _lib.load()
        s = _lib.stream_ptr()
        rng = self.dev.tensors["range"].data_ptr()
        if timer:
            timer("fit", True)
        _lib.check(lib.cpb_fit(ens_slab.data_ptr(), self.slab.owned * self.width,
                               ctypes.byref(self.view), rng, 0, s))
        if timer:
            timer("fit", False)
        st = self.dev.struct
        st.bounds, st.weights_mode, st.plane_stride = self.view.bounds, self.view.weights_mode, 0
        if self.device_eps:
            _lib.check(lib.cpb_range_to_pair(rng, self.pair.data_ptr(), s))
            _, world = _group_world(group)
            if world > 1:
                import torch.distributed as dist

                _all_reduce(self.pair, dist.ReduceOp.MAX, group)
            _lib.check(lib.cpb_pair_to_eps(self.pair.data_ptr(), self.eps_t.data_ptr(), s))
        else:
            gmin, gmax = ctypes.c_double(), ctypes.c_double()
            _lib.check(lib.cpb_read_range(rng, ctypes.byref(gmin), ctypes.byref(gmax), s))
            gmin, gmax = allreduce_range(gmin.value, gmax.value, ens_slab.device, group)
            self.dev.eps = lib.cpb_epsilon(gmin, gmax)
        exchange_halo_rows(_plane_views(self.dev), self.slab, group)
        return self.dev


def fit_slab_fields(fields, ens_slab, group=None, timer=None, finish: bool = True):
    """Fit several SlabFields of one slab in a single pass over the ensemble
    (cpb_fit_multi); then (``finish``) the shared global eps and each field's
    halo exchange (finish_slab_fields)."""
    import ctypes

    from . import _lib

    lib = _lib.load()
    s = _lib.stream_ptr()
    f0 = fields[0]
    rng = f0.dev.tensors["range"].data_ptr()
    views = (ctypes.POINTER(_lib.CpbField) * len(fields))(*[ctypes.pointer(f.view) for f in fields])
    if timer:
        timer("fit", True)
    _lib.check(lib.cpb_fit_multi(ens_slab.data_ptr(), f0.slab.owned * f0.width, views, len(fields),
                                 rng, 0, s))
    if timer:
        timer("fit", False)
    for f in fields:
        st = f.dev.struct
        st.bounds, st.weights_mode, st.plane_stride = f.view.bounds, f.view.weights_mode, 0
    if all(f.device_eps for f in fields):
        # this slab's {-min, max} pair, on the device
        _lib.check(lib.cpb_range_to_pair(rng, f0.pair.data_ptr(), s))
    if finish:
        finish_slab_fields(fields, group)
    return [f.dev for f in fields]


def finish_slab_fields(fields, group=None):
    """Second half of fit_slab_fields: MAX all-reduce of the {-min, max} pair
    (NCCL), the global eps written where the stencils read it, and the halo
    rows of every plane from the neighbouring ranks."""
    import ctypes

    from . import _lib

    lib = _lib.load()
    s = _lib.stream_ptr()
    f0 = fields[0]
    if all(f.device_eps for f in fields):
        _, world = _group_world(group)
        if world > 1:
            import torch.distributed as dist

            _all_reduce(f0.pair, dist.ReduceOp.MAX, group)
        for f in fields:
            _lib.check(lib.cpb_pair_to_eps(f0.pair.data_ptr(), f.eps_t.data_ptr(), s))
    else:
        rng = f0.dev.tensors["range"].data_ptr()
        gmin, gmax = ctypes.c_double(), ctypes.c_double()
        _lib.check(lib.cpb_read_range(rng, ctypes.byref(gmin), ctypes.byref(gmax), s))
        gmin, gmax = allreduce_range(gmin.value, gmax.value, f0.pair.device, group)
        for f in fields:
            f.dev.eps = lib.cpb_epsilon(gmin, gmax)
    # every field's boundary rows in ONE packed exchange per neighbour
    exchange_halo_rows([v for f in fields for v in _plane_views(f.dev)], f0.slab, group)


def fit_slab(ens_slab, model, slab: Slab, width: int, group=None, timer=None):
    """Fit a rank's owned rows into halo-padded planes; global eps; halo exchange.

    ``ens_slab``: (M, owned, W) float32 CUDA tensor of rows [row_begin, row_end).
    Returns the DeviceField (local_height rows; local row 0 is global row
    ``slab.local_row0``); its eps is a host value (synchronous path).
    """
    sf = SlabField(model, slab, width, int(ens_slab.shape[0]), ens_slab.device, device_eps=False)
    return sf.fit(ens_slab, group, timer)


def classify_slab(dev, slab: Slab, estimator, channels=("min", "max", "saddle"), out=None,
                  group=None, sums: bool = False, timer=None):
    """Run the estimator on the rank's stencil rows; returns ((3, Hl, W) planes, sums or None)."""
    import torch

    from .engine import run_rows

    H, W = dev.height, dev.width
    if out is None:
        out = torch.zeros((3, H, W), dtype=torch.float64, device=dev.device)
    a, b = slab.stencil_rows()
    # closed form: the per-type sums come out of the stencil kernels' epilogue
    fused = sums and estimator.method == "closed_form" and set(channels) == {"min", "max", "saddle"}
    total = torch.zeros(3, dtype=torch.float64, device=dev.device) if fused else None
    if timer:
        timer("classify", True)
    if b > a:
        run_rows(dev, estimator, channels, a, b, {"min": out[0], "max": out[1], "saddle": out[2]},
                 type_sums=total)
    if timer:
        timer("classify", False)
    if sums:
        if not fused:
            total = out[:, a:b].sum(dim=(1, 2)) if b > a else torch.zeros(3, dtype=torch.float64,
                                                                            device=dev.device)
        allreduce_sums(total, group)
    return out, total


def fit_classify(fields, ens_slab, slab: Slab, out, group=None, timer=None, work=None):
    """One pass over the slab's ensemble: every field of ``fields`` is fitted
    (cpb_fit_multi_classify; one of them uniform) and the uniform one is
    stencilled in the same kernel over the rows that have both neighbours
    locally; then the shared global eps (MAX all-reduce), ONE packed halo
    exchange for every field, the slab's first / last rows of the uniform
    field (ordinary stencil, after the exchange) and the rows left for the
    final eps (cpb_fit_classify_finish).  Returns (the SUM-all-reduced expected
    per-type counts of the uniform field, 3 device doubles; the work buffer).

    ``out``: (3, local_height, W) float64 planes of the uniform field;
    ``work``: a reusable uint8 device buffer (allocated if None)."""
    import ctypes

    import torch

    from . import _lib
    from .engine import EstimatorSpec, run_rows

    fields = list(fields)
    uni = next(f for f in fields if f.model.kind == "uniform")
    lib = _lib.load()
    s = _lib.stream_ptr()
    W = uni.width
    h0, n = slab.halo_top, slab.owned
    rb, re_ = 1, max(1, n - 1)  # vertex rows of the owned view with both neighbours local
    nb = ctypes.c_size_t()
    _lib.check(lib.cpb_fit_classify_work_bytes(W, rb, re_, ctypes.byref(nb)))
    if work is None or work.numel() < nb.value:
        work = torch.empty(nb.value, dtype=torch.uint8, device=ens_slab.device)
    planes = [out[c, h0:].data_ptr() for c in range(3)]
    f0 = fields[0]
    rng = f0.dev.tensors["range"].data_ptr()
    views = (ctypes.POINTER(_lib.CpbField) * len(fields))(*[ctypes.pointer(f.view) for f in fields])
    if timer:
        timer("fit+classify", True)
    _lib.check(lib.cpb_fit_multi_classify(ens_slab.data_ptr(), n * W, views, len(fields), rng, 0, rb, re_,
                                          *planes, work.data_ptr(), s))
    if timer:
        timer("fit+classify", False)
    for f in fields:
        st = f.dev.struct
        st.bounds, st.weights_mode, st.plane_stride = f.view.bounds, f.view.weights_mode, 0
    uni.view.eps_device = uni.eps_t.data_ptr()
    _lib.check(lib.cpb_range_to_pair(rng, f0.pair.data_ptr(), s))
    finish_slab_fields(fields, group)  # MAX all-reduce -> eps (device), one packed halo exchange
    total = torch.zeros(3, dtype=torch.float64, device=ens_slab.device)
    est = EstimatorSpec()
    chans = {"min": out[0], "max": out[1], "saddle": out[2]}
    # the owned rows next to a neighbouring slab, now that the halo rows are in
    a, b = slab.stencil_rows()
    edge_rows = sorted({r for r in (h0, h0 + n - 1) if a <= r < b and not (h0 + rb <= r < h0 + re_)})
    for r in edge_rows:
        run_rows(uni.dev, est, CH3, r, r + 1, chans, type_sums=total)
    _lib.check(lib.cpb_fit_classify_finish(ctypes.byref(uni.view), rb, re_, *planes, total.data_ptr(),
                                           work.data_ptr(), s))
    allreduce_sums(total, group)
    return total, work


def fit_classify_uniform(field: SlabField, ens_slab, slab: Slab, out, group=None, timer=None, work=None):
    """fit_classify for a uniform field alone."""
    return fit_classify([field], ens_slab, slab, out, group, timer, work)


CH3 = ("min", "max", "saddle")
