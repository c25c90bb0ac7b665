"""Device-side synthetic ensembles (the config-5 input, synthesised in HBM).

value(m, r, c) = f32(bowl(r, c) + noise_amp * (2u - 1)) with u the keyed
splitmix64 draw (seed, pixel r*W + c, plane m, sample 0) and bowl a
transcendental-free quadratic surface, so any row slab can be regenerated
bit for bit on the host (oracle.critprob_oracle.synthetic_rows) for parity
checks.  The reference's own generator (synth.ackley_ensemble, synth.py:54-65)
draws numpy PCG64 noise, which has no device twin; configs 1-4 therefore use
host-generated Ackley ensembles copied to the device.
"""

from __future__ import annotations

from . import _lib
from .fields import EnsembleStack, _device


def synthetic_rows(row0: int, nrows: int, width: int, height: int, members: int,
                   noise_amp: float = 0.3, seed: int = 0, out=None):
    """(members, nrows, width) float32 CUDA tensor of rows [row0, row0 + nrows)."""
    import torch

    if out is None:
        out = torch.empty((members, nrows, width), dtype=torch.float32, device=_device())
    lib = _lib.load()
    _lib.check(lib.cpb_synth_ensemble(out.data_ptr(), members, row0, nrows, width, height,
                                      float(noise_amp), int(seed) & ((1 << 64) - 1),
                                      _lib.stream_ptr()))
    return out


def synthetic_ensemble(width: int, height: int, members: int, noise_amp: float = 0.3,
                       seed: int = 0) -> EnsembleStack:
    """A whole synthetic ensemble, resident on the device."""
    return EnsembleStack(synthetic_rows(0, height, width, height, members, noise_amp, seed))
