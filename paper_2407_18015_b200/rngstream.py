"""The keyed splitmix64 uniform stream, evaluated on the device.

Mirrors critprob.rngstream (rngstream.py:33-53): draws are a pure function
of (seed, pixel, plane, sample index), which is what makes the Monte Carlo
grid results independent of how pixels are split across blocks, slabs or
GPUs.  ``unit_block`` returns a numpy array like the reference.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def unit_block(seed: int, pixels, planes: int, n: int, start: int = 0, *, output: str = "host"):
    """Uniform [0, 1) draws of shape (len(pixels), planes, n) (rngstream.py:33-48)."""
    import torch

    from .fields import _device

    px = np.asarray(pixels, dtype=np.uint64).reshape(-1)
    d_px = torch.as_tensor(px.view(np.int64), device=_device())
    out = torch.empty((px.size, planes, n), dtype=torch.float64, device=d_px.device)
    lib = _lib.load()
    _lib.check(lib.cpb_unit_block(int(seed) & ((1 << 64) - 1), d_px.data_ptr(), px.size, planes,
                                  start, n, out.data_ptr(), _lib.stream_ptr()))
    return out if output == "device" else out.cpu().numpy()


def unit_planes(seed: int, pixel: int, planes: int, n: int) -> np.ndarray:
    """Uniform [0, 1) draws of shape (planes, n) for a single pixel key (rngstream.py:51-53)."""
    return unit_block(seed, np.asarray([pixel], dtype=np.uint64), planes, n)[0]
