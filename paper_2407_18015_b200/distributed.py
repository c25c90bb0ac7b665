"""Row-slab decomposition of the grid over one process per GPU.

The reference parallelises only over flat pixel chunks in one process pool
(engine.py:757-779) and every chunk carries pre-shifted copies of all five
stencil positions, so it never exchanges anything.  Here the grid is split
into G contiguous row slabs, one per rank (torchrun, NCCL over NVLink):

1. each rank fits its own rows (cpb_fit) and gets its local value range;
2. one all-reduce (MAX over [-min, max]) gives the GLOBAL range, hence the
   same eps on every rank (distributions.py:30-36 is global, fields.py:136);
3. one halo exchange sends the first / last owned row of every fitted plane
   to the rank above / below (batched send/recv);
4. each rank runs the stencil (closed form or Monte Carlo) on its rows --
   Monte Carlo keys use GLOBAL pixel indices (engine.py:752-754), so the
   result is bit-identical for every G;
5. optionally one all-reduce (SUM) of the per-type expected counts
   E[#min], E[#max], E[#saddle] = sum over vertices of p.

The helpers below (``slab_rows``, ``exchange_halo_rows``,
``allreduce_range``, ``allreduce_sums``) are plain torch.distributed code so
the multi-rank logic is tested on CPU with the gloo backend.
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
    """Contiguous, balanced row slabs (the first height % world ranks get one extra row)."""
    base, extra = divmod(height, world)
    r0 = rank * base + min(rank, extra)
    r1 = r0 + base + (1 if rank < extra else 0)
    return Slab(rank, world, height, r0, r1)


def _group_world(group):
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def allreduce_range(vmin: float, vmax: float, device, group=None) -> tuple[float, float]:
    """Global (min, max) over ranks: one MAX all-reduce of [-min, max]."""
    import torch
    import torch.distributed as dist

    _, world = _group_world(group)
    if world == 1:
        return vmin, vmax
    t = torch.tensor([-vmin, vmax], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return -float(t[0]), float(t[1])


def exchange_halo_rows(planes, slab: Slab, group=None) -> None:
    """Fill the halo rows of every plane from the neighbouring ranks.

    ``planes``: tensors shaped (local_height, W) or (k, local_height, W);
    local row ``halo_top`` is the first owned row.  Sends the first owned row
    up and the last owned row down, receives into row 0 / the last row.
    """
    import torch.distributed as dist

    rank, world = _group_world(group)
    if world == 1:
        return
    ops = []
    first = slab.halo_top
    last = slab.halo_top + slab.owned - 1
    for t in planes:
        views = [t] if t.dim() == 2 else [t[i] for i in range(t.shape[0])]
        for v in views:
            if slab.halo_top:
                ops.append(dist.P2POp(dist.isend, v[first].contiguous(), rank - 1, group))
                ops.append(dist.P2POp(dist.irecv, v[0], rank - 1, group))
            if slab.halo_bottom:
                ops.append(dist.P2POp(dist.isend, v[last].contiguous(), rank + 1, group))
                ops.append(dist.P2POp(dist.irecv, v[last + 1], rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def allreduce_sums(sums, group=None):
    """SUM all-reduce of the per-type expected counts (a small float64 tensor)."""
    import torch.distributed as dist

    _, world = _group_world(group)
    if world > 1:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
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

                dist.all_reduce(self.pair, op=dist.ReduceOp.MAX, group=group)
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

            dist.all_reduce(f0.pair, op=dist.ReduceOp.MAX, group=group)
        for f in fields:
            _lib.check(lib.cpb_pair_to_eps(f0.pair.data_ptr(), f.eps_t.data_ptr(), s))
    else:
        rng = f0.dev.tensors["range"].data_ptr()
        gmin, gmax = ctypes.c_double(), ctypes.c_double()
        _lib.check(lib.cpb_read_range(rng, ctypes.byref(gmin), ctypes.byref(gmax), s))
        gmin, gmax = allreduce_range(gmin.value, gmax.value, f0.pair.device, group)
        for f in fields:
            f.dev.eps = lib.cpb_epsilon(gmin, gmax)
    for f in fields:
        exchange_halo_rows(_plane_views(f.dev), f.slab, group)


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
