"""Grid containers with the reference's API, backed by device-resident planes.

Mirrors critprob.fields (/root/reference/pkg/src/critprob/fields.py):

- ``ModelSpec``       fields.py:25-39  (same fields, defaults and ValueErrors)
- ``EnsembleStack``   fields.py:42-83  (numpy input as in the reference; a CUDA
                                        torch tensor is also accepted and stays
                                        on the device)
- ``UncertainField``  fields.py:86-178 (``from_ensemble`` / ``from_scalar`` run on
                                        the GPU; ``params`` materialises the
                                        reference's float64 dict on demand)
- ``ProbabilityField`` fields.py:181-212

The fitted parameters live on the device in compact form (float32 min/max,
uint8 bin counts, float64 mean/std; see include/critprob_b200.h), and
``params`` reproduces the reference arrays bit for bit from them.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

MODEL_KINDS = ("uniform", "epanechnikov", "histogram", "gaussian")
CHANNELS = ("min", "max", "saddle")

_device_index: int | None = None


def set_device(index: int | None) -> None:
    """Select the CUDA device new fields are placed on (None = current device)."""
    global _device_index
    _device_index = index


def _device():
    import torch

    _lib.load()
    return torch.device("cuda", _device_index if _device_index is not None else torch.cuda.current_device())


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


@dataclass(frozen=True)
class ModelSpec:
    """Which distribution family to fit, plus its shape parameters (fields.py:25-39)."""

    kind: str
    bins: int = 5
    k: float = math.sqrt(5.0)

    def __post_init__(self) -> None:
        if self.kind not in MODEL_KINDS:
            raise ValueError(f"unknown model kind {self.kind!r}")
        if self.bins < 1:
            raise ValueError("bins must be at least 1")
        if not self.k > 0.0:
            raise ValueError("k must be positive")


class _PinnedBlock:
    """Page-locked host memory from cpb_host_alloc, freed with its last array."""

    def __init__(self, nbytes: int) -> None:
        self.ptr = None
        p = ctypes.c_void_p()
        _lib.check(_lib.load(require_device=False).cpb_host_alloc(ctypes.byref(p), max(1, nbytes)))
        self.ptr = p.value

    def __del__(self) -> None:
        if self.ptr and _lib._lib is not None:
            _lib._lib.cpb_host_free(self.ptr)
            self.ptr = None


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """An uninitialised numpy array in page-locked host memory (exact size).

    Ensembles and results kept in pinned memory cross PCIe by DMA at full
    bandwidth (EnsembleStack upload, copy-outs); the memory is released when
    the last array viewing it is garbage-collected.
    """
    shape = tuple(int(x) for x in (shape if np.iterable(shape) else (shape,)))
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
    block = _PinnedBlock(nbytes)
    raw = (ctypes.c_char * max(1, nbytes)).from_address(block.ptr)
    raw._cpb_block = block  # keeps the allocation alive as long as any view
    return np.frombuffer(raw, dtype=dt, count=nbytes // dt.itemsize).reshape(shape)


@dataclass
class EnsembleStack:
    """Member rasters, shape (members, height, width), float32 (fields.py:42-83).

    ``values`` may be a numpy array (validated like the reference) or a CUDA
    torch tensor, which stays in HBM; its finiteness is then checked by the
    fit kernel, and a NaN/Inf raises the same ValueError at fit time.

    A numpy stack is uploaded to HBM ONCE and the device copy is kept, so the
    reference workflow ``for model: classify_field(from_ensemble(stack, model))``
    moves the ensemble over PCIe once, not once per model.  Stacks of
    ``_DEVICE_CHECK_BYTES`` or more are uploaded at construction and checked for
    NaN/Inf in HBM (cpb_check_finite; the same ValueError as the reference's
    host isfinite pass, fields.py:54-55); smaller ones are checked on the host
    and uploaded on first use.  A stack in pinned host memory (``pinned_empty``)
    crosses PCIe at full DMA bandwidth.  The device copy is a snapshot:
    in-place writes to ``values`` after construction are not seen by the fits.
    """

    values: object

    _DEVICE_CHECK_BYTES = 256 << 20

    def __post_init__(self) -> None:
        self._dev = None
        if _is_tensor(self.values) and self.values.is_cuda:
            t = self.values
            if t.dim() != 3:
                raise ValueError("ensemble values must be 3-D (members, height, width)")
            if t.shape[0] < 1 or t.shape[1] < 1 or t.shape[2] < 1:
                raise ValueError("ensemble needs at least one member and one pixel")
            import torch

            self.values = t.to(torch.float32).contiguous()
            return
        arr = np.asarray(self.values.cpu().numpy() if _is_tensor(self.values) else self.values)
        if arr.ndim != 3:
            raise ValueError("ensemble values must be 3-D (members, height, width)")
        if arr.shape[0] < 1 or arr.shape[1] < 1 or arr.shape[2] < 1:
            raise ValueError("ensemble needs at least one member and one pixel")
        if arr.nbytes >= self._DEVICE_CHECK_BYTES and arr.dtype == np.float32:
            self.values = np.ascontiguousarray(arr)
            dev = self._upload()
            _lib.check(_lib.load().cpb_check_finite(dev.data_ptr(), dev.numel(), _lib.stream_ptr()))
            self._dev = dev
            return
        if not np.isfinite(arr).all():
            raise ValueError("ensemble values must be finite")
        self.values = np.ascontiguousarray(arr, dtype=np.float32)

    def _upload(self):
        import torch

        dev = torch.empty(self.values.shape, dtype=torch.float32, device=_device())
        dev.copy_(torch.from_numpy(self.values))
        return dev

    @property
    def on_device(self) -> bool:
        return _is_tensor(self.values)

    @property
    def members(self) -> int:
        return int(self.values.shape[0])

    @property
    def height(self) -> int:
        return int(self.values.shape[1])

    @property
    def width(self) -> int:
        return int(self.values.shape[2])

    def device_values(self):
        """The stack as a contiguous float32 CUDA tensor (a host stack is uploaded once)."""
        if self.on_device:
            return self.values
        if self._dev is None:
            self._dev = self._upload()
        return self._dev

    def normalized(self) -> tuple["EnsembleStack", float, float]:
        """Affine copy rescaled to [0, 1]; returns (stack, scale, offset) (fields.py:70-83)."""
        if self.on_device:
            import torch

            vmin = float(self.values.min())
            vmax = float(self.values.max())
            if vmax <= vmin:
                return EnsembleStack(self.values.clone()), 1.0, 0.0
            scale = 1.0 / (vmax - vmin)
            offset = -vmin * scale
            rescaled = (self.values.to(torch.float64) - vmin) * scale
            return EnsembleStack(rescaled.to(torch.float32)), scale, offset
        vmin = float(self.values.min())
        vmax = float(self.values.max())
        if vmax <= vmin:
            return EnsembleStack(self.values.copy()), 1.0, 0.0
        scale = 1.0 / (vmax - vmin)
        offset = -vmin * scale
        rescaled = (self.values.astype(np.float64) - vmin) * scale
        return EnsembleStack(rescaled.astype(np.float32)), scale, offset


class DeviceField:
    """Device planes of one fitted field plus the ``cpb_field`` describing them."""

    def __init__(self, kind: str, bins: int, members: int, height: int, width: int, *,
                 row0: int = 0, global_width: int | None = None, k: float = math.sqrt(5.0),
                 eps: float = 0.0, device=None):
        import torch

        self.device = device if device is not None else _device()
        self.kind, self.bins, self.members = kind, int(bins), int(members)
        self.height, self.width = int(height), int(width)
        self.tensors: dict = {}
        st = _lib.CpbField()
        st.kind = _lib.KIND_CODES[kind]
        st.bins = self.bins
        st.members = self.members
        st.height, st.width = self.height, self.width
        st.row0 = int(row0)
        st.global_width = int(global_width if global_width is not None else width)
        st.k = float(k)
        st.eps = float(eps)
        self.struct = st
        self._torch = torch

    # -- allocation ---------------------------------------------------------
    def allocate_fitted(self) -> None:
        """Allocate the compact planes cpb_fit writes (cpb_field_plane_bytes)."""
        torch = self._torch
        lib = _lib.load()
        out = (ctypes.c_size_t * 7)()
        _lib.check(lib.cpb_field_plane_bytes(self.struct.kind, self.bins, self.members,
                                             self.height, self.width, out))
        names = ("lo", "hi", "mean", "spread", "weights", "weight_table", "range")
        for name, nbytes in zip(names, out):
            if nbytes:
                self.tensors[name] = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        self._bind()

    def set_planes(self, **planes) -> None:
        """Attach caller-built planes (user-given float64 params)."""
        self.tensors.update(planes)
        self._bind()

    def _bind(self) -> None:
        st = self.struct
        for name in ("lo", "hi", "mean", "spread", "weights", "weight_table"):
            t = self.tensors.get(name)
            setattr(st, name, t.data_ptr() if t is not None else None)

    @property
    def eps(self) -> float:
        return self.struct.eps

    @eps.setter
    def eps(self, value: float) -> None:
        self.struct.eps = float(value)

    def ref(self):
        return ctypes.byref(self.struct)


class UncertainField:
    """One fitted distribution per pixel (fields.py:86-121).

    ``params`` holds the reference's (height, width) float64 arrays
    (uniform: lo, hi; epanechnikov: mean, halfwidth; histogram: lo, hi,
    weights (h, w, bins); gaussian: mean, stddev).  Fields produced on the
    GPU keep compact device planes and materialise ``params`` lazily.
    """

    def __init__(self, model: ModelSpec, params: dict | None = None, *, _device_field=None) -> None:
        self.model = model
        self._params = dict(params) if params is not None else None
        self._dev = _device_field
        if self._params is not None:
            first = next(iter(self._params.values()))
            self.height = int(first.shape[0])
            self.width = int(first.shape[1])
        else:
            self.height = _device_field.height
            self.width = _device_field.width

    @property
    def shape(self) -> tuple[int, int]:
        return self.height, self.width

    # -- parameters ------------------------------------------------------------
    @property
    def params(self) -> dict:
        if self._params is None:
            self._params = self._materialize()
        return self._params

    def _materialize(self) -> dict:
        import torch

        dev = self._dev
        lib = _lib.load()
        H, W = self.shape
        a = torch.empty((H, W), dtype=torch.float64, device=dev.device)
        b = torch.empty((H, W), dtype=torch.float64, device=dev.device)
        w = None
        if self.model.kind == "histogram":
            w = torch.empty((H, W, dev.bins), dtype=torch.float64, device=dev.device)
        _lib.check(lib.cpb_materialize(dev.ref(), a.data_ptr(), b.data_ptr(), _lib.ptr(w),
                                       _lib.stream_ptr()))
        a, b = a.cpu().numpy(), b.cpu().numpy()
        kind = self.model.kind
        if kind == "uniform":
            return {"lo": a, "hi": b}
        if kind == "histogram":
            return {"lo": a, "hi": b, "weights": w.cpu().numpy()}
        if kind == "epanechnikov":
            return {"mean": a, "halfwidth": b}
        return {"mean": a, "stddev": b}

    def device_field(self) -> DeviceField:
        """Device planes of this field (uploads a user-built params dict once)."""
        if self._dev is None:
            self._dev = self._upload(self._params)
        return self._dev

    def _upload(self, params: dict) -> DeviceField:
        import torch

        kind = self.model.kind
        H, W = self.shape
        dev = DeviceField(kind, self.model.bins, 1, H, W, k=1.0, eps=0.0)

        def f64(x):
            return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)),
                                   device=dev.device)

        st = dev.struct
        st.bounds = _lib.BOUNDS_F64
        st.weights_mode = _lib.WEIGHTS_F64
        if kind in ("uniform", "histogram"):
            planes = {"lo": f64(params["lo"]), "hi": f64(params["hi"])}
            if kind == "histogram":
                wts = np.asarray(params["weights"], dtype=np.float64)
                st.bins = dev.bins = int(wts.shape[-1])
                planes["weights"] = f64(np.moveaxis(wts, -1, 0))
            dev.set_planes(**planes)
        elif kind == "epanechnikov":
            dev.set_planes(mean=f64(params["mean"]), spread=f64(params["halfwidth"]))
        else:
            dev.set_planes(mean=f64(params["mean"]), spread=f64(params["stddev"]))
        return dev

    # -- fitting -----------------------------------------------------------
    @classmethod
    def from_ensemble(cls, stack: EnsembleStack, model: ModelSpec) -> "UncertainField":
        """Fit the chosen model independently at every pixel (fields.py:125-158), on the GPU."""
        vals = stack.device_values()
        M, H, W = (int(s) for s in vals.shape)
        if M < 2 and model.kind in ("epanechnikov", "gaussian"):
            raise ValueError(f"{model.kind} fit needs at least two members")
        dev = fit_device(vals, model)
        return cls(model, _device_field=dev)

    def dist_at(self, row: int, col: int):
        """Materialize the pixel's distribution (fields.py:109-121) as a per-case object."""
        from .cases import dist_at

        return dist_at(self, row, col)

    @classmethod
    def from_ensemble_models(cls, stack: EnsembleStack, models) -> list:
        """``[from_ensemble(stack, m) for m in models]`` in one pass over the
        ensemble (cpb_fit_multi): the reference workflow of fitting one stack
        with several models, with the stack read from HBM once."""
        models = list(models)
        vals = stack.device_values()
        M = int(vals.shape[0])
        for model in models:
            if M < 2 and model.kind in ("epanechnikov", "gaussian"):
                raise ValueError(f"{model.kind} fit needs at least two members")
        return [cls(m, _device_field=d) for m, d in zip(models, fit_device_models(vals, models))]

    @classmethod
    def from_scalar(cls, values, error_bound: float) -> "UncertainField":
        """Uniform field from a plain raster with a +/- error_bound / 2 band (fields.py:160-178)."""
        import torch

        if error_bound < 0.0:
            raise ValueError("error bound must be nonnegative")
        if _is_tensor(values):
            arr = values.to(_device(), torch.float64)
            if arr.dim() != 2:
                raise ValueError("scalar field must be 2-D")
            if not bool(torch.isfinite(arr).all()):
                raise ValueError("scalar field values must be finite")
        else:
            host = np.asarray(values, dtype=np.float64)
            if host.ndim != 2:
                raise ValueError("scalar field must be 2-D")
            if not np.isfinite(host).all():
                raise ValueError("scalar field values must be finite")
            arr = torch.as_tensor(np.ascontiguousarray(host), device=_device())
        arr = arr.contiguous()
        H, W = (int(s) for s in arr.shape)
        eps = 0.0
        if 0.5 * error_bound <= 0.0:
            lo_v, hi_v = torch.aminmax(arr)
            eps = _lib.load().cpb_epsilon(float(lo_v), float(hi_v))
        lo = torch.empty_like(arr)
        hi = torch.empty_like(arr)
        lib = _lib.load()
        _lib.check(lib.cpb_from_scalar(arr.data_ptr(), H, W, float(error_bound), eps, lo.data_ptr(),
                                       hi.data_ptr(), _lib.stream_ptr()))
        dev = DeviceField("uniform", 5, 1, H, W, k=1.0, eps=0.0)
        dev.struct.bounds = _lib.BOUNDS_F64
        dev.set_planes(lo=lo, hi=hi)
        return cls(ModelSpec("uniform"), _device_field=dev)


def fit_device(vals, model: ModelSpec, *, row0: int = 0, global_width: int | None = None,
               eps: float | None = None, range_out: list | None = None) -> DeviceField:
    """Run cpb_fit on a (M, H, W) float32 CUDA tensor; returns the device field.

    ``eps`` overrides the field's epsilon (row slabs pass the GLOBAL one); by
    default it comes from this tensor's own range like distributions.py:30-36.
    ``range_out`` receives [min, max] of the values read.
    """
    M, H, W = (int(s) for s in vals.shape)
    lib = _lib.load()
    dev = DeviceField(model.kind, model.bins, M, H, W, row0=row0, global_width=global_width,
                      k=model.k, device=vals.device)
    dev.allocate_fitted()
    s = _lib.stream_ptr()
    _lib.check(lib.cpb_fit(vals.data_ptr(), H * W, dev.ref(), dev.tensors["range"].data_ptr(), 0, s))
    gmin, gmax = ctypes.c_double(), ctypes.c_double()
    _lib.check(lib.cpb_read_range(dev.tensors["range"].data_ptr(), ctypes.byref(gmin),
                                  ctypes.byref(gmax), s))
    if range_out is not None:
        range_out[:] = [gmin.value, gmax.value]
    dev.eps = lib.cpb_epsilon(gmin.value, gmax.value) if eps is None else eps
    return dev


def fit_device_models(vals, models, *, row0: int = 0, global_width: int | None = None,
                      eps: float | None = None, range_out: list | None = None) -> list:
    """cpb_fit_multi over a (M, H, W) float32 CUDA tensor: one DeviceField per model."""
    M, H, W = (int(s) for s in vals.shape)
    lib = _lib.load()
    devs = []
    for model in models:
        dev = DeviceField(model.kind, model.bins, M, H, W, row0=row0, global_width=global_width,
                          k=model.k, device=vals.device)
        dev.allocate_fitted()
        devs.append(dev)
    s = _lib.stream_ptr()
    rng = devs[0].tensors["range"].data_ptr()
    arr = (ctypes.POINTER(_lib.CpbField) * len(devs))(*[ctypes.pointer(d.struct) for d in devs])
    _lib.check(lib.cpb_fit_multi(vals.data_ptr(), H * W, arr, len(devs), rng, 0, s))
    gmin, gmax = ctypes.c_double(), ctypes.c_double()
    _lib.check(lib.cpb_read_range(rng, ctypes.byref(gmin), ctypes.byref(gmax), s))
    if range_out is not None:
        range_out[:] = [gmin.value, gmax.value]
    e = lib.cpb_epsilon(gmin.value, gmax.value) if eps is None else eps
    for dev in devs:
        dev.eps = e
    return devs


@dataclass
class ProbabilityField:
    """Per-pixel probabilities of each critical-point type (fields.py:181-212).

    The one-pixel border has no full neighborhood and is marked invalid
    (``valid`` False, probabilities zero).  Arrays are numpy (host) unless
    produced with ``output="device"``, in which case they are CUDA tensors.
    """

    p_min: object
    p_max: object
    p_saddle: object
    valid: object

    def __post_init__(self) -> None:
        shape = tuple(self.p_min.shape)
        for arr in (self.p_max, self.p_saddle, self.valid):
            if tuple(arr.shape) != shape:
                raise ValueError("all channels must share one shape")

    @property
    def shape(self) -> tuple[int, int]:
        return tuple(self.p_min.shape)

    def channel(self, name: str):
        if name not in CHANNELS:
            raise ValueError(f"unknown channel {name!r}")
        return {"min": self.p_min, "max": self.p_max, "saddle": self.p_saddle}[name]

    @classmethod
    def empty(cls, height: int, width: int) -> "ProbabilityField":
        zero = np.zeros((height, width), dtype=np.float64)
        return cls(zero, zero.copy(), zero.copy(), np.zeros((height, width), dtype=bool))
