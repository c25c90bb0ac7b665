"""UCVF / CSV / P5 I/O around the B200 path.

Same container and API as critprob.field_io (field_io.py:1-169):

    UCVF  = ASCII header "UCVF1 <width> <height> <channels>\\n" followed by
            channels * height * width little-endian float32, channel-major
            (one channel per ensemble member; probability files carry
            min, max, saddle, mask)
    CSV   = x,y,p_min,p_max,p_saddle,valid with 17 significant digits
    P5    = 8-bit grayscale heatmap, gray = round(255 * clip(p)^gamma)

The UCVF payload already has the ensemble's (M, H, W) float32 layout, so
``load_ensemble(path, device=True)`` streams it from disk through a pinned
staging buffer straight into HBM (no full host copy) and checks finiteness
on the device; ``export_heatmap`` quantises on the device (cpb_heatmap) when
the probability planes are CUDA tensors.  Error classes and messages follow
the reference (UcvfFormatError / UcvfPayloadError / UcvfValueError).
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from .fields import CHANNELS, EnsembleStack, ProbabilityField, UncertainField

UCVF_MAGIC = "UCVF1"


class UcvfError(Exception):
    """Base for UCVF parsing failures."""


class UcvfFormatError(UcvfError):
    """Header is not a UCVF header."""


class UcvfPayloadError(UcvfError):
    """Header and payload length disagree."""


class UcvfValueError(UcvfError):
    """Payload holds non-finite values."""


# ---------------------------------------------------------------------------
# container
# ---------------------------------------------------------------------------

def _header(width: int, height: int, channels: int) -> bytes:
    return f"{UCVF_MAGIC} {width} {height} {channels}\n".encode("ascii")


def _write(path, width: int, height: int, planes) -> None:
    data = np.ascontiguousarray(planes, dtype="<f4")
    with open(path, "wb") as fh:
        fh.write(_header(width, height, data.shape[0]))
        fh.write(memoryview(data).cast("B"))


def _parse_header(fh) -> tuple[int, int, int, int]:
    """(width, height, channels, payload offset); validates like field_io.py:43-62."""
    head = fh.read(256)
    nl = head.find(b"\n")
    if nl < 0:
        raise UcvfFormatError("missing header line")
    try:
        parts = head[:nl].decode("ascii").split()
    except UnicodeDecodeError as exc:
        raise UcvfFormatError("header is not ASCII") from exc
    if len(parts) != 4 or parts[0] != UCVF_MAGIC:
        raise UcvfFormatError(f"expected '{UCVF_MAGIC} <w> <h> <c>' header")
    try:
        width, height, channels = (int(v) for v in parts[1:])
    except ValueError as exc:
        raise UcvfFormatError("header dimensions are not integers") from exc
    if width < 1 or height < 1 or channels < 1:
        raise UcvfFormatError("header dimensions must be positive")
    return width, height, channels, nl + 1


def _open_checked(path):
    fh = open(path, "rb")
    try:
        width, height, channels, off = _parse_header(fh)
        size = os.fstat(fh.fileno()).st_size - off
        expected = 4 * width * height * channels
        if size != expected:
            raise UcvfPayloadError(f"payload holds {size} bytes, header implies {expected}")
        fh.seek(off)
    except Exception:
        fh.close()
        raise
    return fh, width, height, channels


def _read_host(path) -> tuple[int, int, np.ndarray]:
    fh, width, height, channels = _open_checked(path)
    with fh:
        planes = np.empty((channels, height, width), dtype="<f4")
        fh.readinto(memoryview(planes).cast("B"))
    if not np.isfinite(planes).all():
        raise UcvfValueError("payload holds non-finite values")
    return width, height, planes


def _read_device(path, chunk_bytes: int = 256 << 20):
    """Stream the payload through a pinned buffer into a CUDA tensor."""
    import torch

    from .fields import _device

    fh, width, height, channels = _open_checked(path)
    with fh:
        dev = torch.empty((channels, height, width), dtype=torch.float32, device=_device())
        flat = dev.view(-1)
        n = flat.numel()
        step = max(1, chunk_bytes // 4)
        stage = [torch.empty(min(step, n), dtype=torch.float32).pin_memory() for _ in range(2)]
        done = [None, None]
        bad = torch.zeros((), dtype=torch.bool, device=dev.device)
        for k, start in enumerate(range(0, n, step)):
            cnt = min(step, n - start)
            buf = stage[k & 1]
            if done[k & 1] is not None:
                done[k & 1].synchronize()   # the previous copy out of this buffer finished
            fh.readinto(memoryview(buf.numpy()[:cnt]).cast("B"))
            dst = flat[start:start + cnt]
            dst.copy_(buf[:cnt], non_blocking=True)
            bad |= ~torch.isfinite(dst).all()
            ev = torch.cuda.Event()
            ev.record()
            done[k & 1] = ev
        if bool(bad):
            raise UcvfValueError("payload holds non-finite values")
    return width, height, dev


# ---------------------------------------------------------------------------
# ensembles and scalar fields
# ---------------------------------------------------------------------------

def save_ensemble(stack: EnsembleStack, path) -> None:
    vals = stack.values.cpu().numpy() if stack.on_device else stack.values
    _write(path, stack.width, stack.height, vals)


def load_ensemble(path, device: bool = False) -> EnsembleStack:
    """UCVF ensemble (field_io.py:77-79); ``device=True`` streams it into HBM."""
    if device:
        _, _, planes = _read_device(path)
        return EnsembleStack(planes)
    _, _, planes = _read_host(path)
    return EnsembleStack(np.array(planes, dtype=np.float32))


def save_scalar_field(values, path) -> None:
    arr = np.asarray(values, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError("scalar field must be a 2-D raster")
    _write(path, arr.shape[1], arr.shape[0], arr[None].astype(np.float32))


def load_scalar_field(path) -> np.ndarray:
    _, _, planes = _read_host(path)
    if planes.shape[0] != 1:
        raise UcvfFormatError("scalar fields carry exactly 1 channel")
    return np.array(planes[0], dtype=np.float64)


def uniform_field_from_scalar(values, error_bound: float) -> UncertainField:
    """Per-pixel uniform model on [v - eb/2, v + eb/2] (fields.py:160-178)."""
    return UncertainField.from_scalar(values, error_bound)


# ---------------------------------------------------------------------------
# probability fields
# ---------------------------------------------------------------------------

def _host(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def save_probability_field(field: ProbabilityField, path, format: str = "ucvf") -> None:
    """(min, max, saddle, mask) as UCVF float32 planes, or a CSV table (field_io.py:82-108)."""
    pm, pM, ps, ok = (_host(a) for a in (field.p_min, field.p_max, field.p_saddle, field.valid))
    height, width = pm.shape
    if format == "ucvf":
        _write(path, width, height, np.stack([pm, pM, ps, ok.astype(np.float64)]))
        return
    if format == "csv":
        ys, xs = np.mgrid[0:height, 0:width]
        with open(path, "w", encoding="ascii") as fh:
            fh.write("x,y,p_min,p_max,p_saddle,valid\n")
            for x, y, a, b, c, v in zip(xs.ravel(), ys.ravel(), pm.ravel(), pM.ravel(),
                                        ps.ravel(), ok.ravel()):
                fh.write(f"{x},{y},{a:.17g},{b:.17g},{c:.17g},{int(v)}\n")
        return
    raise ValueError(f"unknown format {format!r}")


def load_probability_field(path, format: str = "ucvf") -> ProbabilityField:
    if format == "ucvf":
        width, height, planes = _read_host(path)
        if planes.shape[0] != 4:
            raise UcvfFormatError("probability fields carry exactly 4 channels")
        out = ProbabilityField.empty(height, width)
        for dst, src in zip((out.p_min, out.p_max, out.p_saddle), planes[:3]):
            dst[:] = src
        out.valid[:] = planes[3] >= 0.5
        return out
    if format == "csv":
        table = np.atleast_2d(np.genfromtxt(path, delimiter=",", skip_header=1))
        xs, ys = table[:, 0].astype(int), table[:, 1].astype(int)
        out = ProbabilityField.empty(int(ys.max()) + 1, int(xs.max()) + 1)
        out.p_min[ys, xs] = table[:, 2]
        out.p_max[ys, xs] = table[:, 3]
        out.p_saddle[ys, xs] = table[:, 4]
        out.valid[ys, xs] = table[:, 5] >= 0.5
        return out
    raise ValueError(f"unknown format {format!r}")


def heatmap_bytes(field: ProbabilityField, channel: str, gamma: float = 1.0) -> np.ndarray:
    """The P5 pixel bytes of one channel, quantised on the device (cpb_heatmap)."""
    import torch

    from .fields import _device

    if channel not in CHANNELS:
        raise ValueError(f"unknown channel {channel!r}")
    if gamma <= 0:
        raise ValueError("gamma must be positive")
    dev = _device()
    p = torch.as_tensor(field.channel(channel), dtype=torch.float64, device=dev).contiguous()
    ok = torch.as_tensor(field.valid, device=dev).to(torch.uint8).contiguous()
    out = torch.empty(p.shape, dtype=torch.uint8, device=dev)
    lib = _lib.load()
    _lib.check(lib.cpb_heatmap(p.data_ptr(), ok.data_ptr(), p.numel(), float(gamma),
                               out.data_ptr(), _lib.stream_ptr()))
    return out.cpu().numpy()


def export_heatmap(field: ProbabilityField, channel: str, path, gamma: float = 1.0) -> None:
    """8-bit grayscale P5 image of one channel; masked pixels are black (field_io.py:138-150)."""
    gray = heatmap_bytes(field, channel, gamma)
    height, width = gray.shape
    with open(path, "wb") as fh:
        fh.write(f"P5 {width} {height} 255\n".encode("ascii"))
        fh.write(gray.tobytes())
