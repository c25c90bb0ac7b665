"""ctypes binding of libcritprob_b200.so (include/critprob_b200.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every entry point raises instead of computing anything.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcritprob_b200.so")

CPB_OK, CPB_EINVAL, CPB_ECUDA, CPB_ENOMEM, CPB_ENONFINITE = 0, 1, 2, 4, 5
KIND_CODES = {"uniform": 0, "epanechnikov": 1, "histogram": 2, "gaussian": 3}
CH_MIN, CH_MAX, CH_SADDLE = 1, 2, 4
RNG_CODES = {"splitmix64": 0, "philox": 1}
BOUNDS_F32_FITTED, BOUNDS_F64 = 0, 1
WEIGHTS_U8, WEIGHTS_U16, WEIGHTS_F64 = 0, 1, 2
FLAG_MIXED = 1

c_i32, c_i64, c_u32, c_u64, c_dbl, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                            ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p)


class CpbField(ctypes.Structure):
    """Mirror of `struct cpb_field` (include/critprob_b200.h)."""

    _fields_ = [
        ("kind", c_i32), ("bins", c_i32), ("members", c_i32), ("bounds", c_i32),
        ("weights_mode", c_i32), ("flags", c_i32),
        ("height", c_i64), ("width", c_i64), ("row0", c_i64), ("global_width", c_i64),
        ("plane_stride", c_i64), ("eps_device", c_vp),
        ("eps", c_dbl), ("k", c_dbl),
        ("lo", c_vp), ("hi", c_vp), ("mean", c_vp), ("spread", c_vp),
        ("weights", c_vp), ("weight_table", c_vp),
    ]


class CpbCaseBatch(ctypes.Structure):
    """Mirror of `struct cpb_case_batch` (include/critprob_b200.h)."""

    _fields_ = [
        ("n_cases", c_i64), ("neighbors", c_i32), ("max_bins", c_i32),
        ("kind", c_vp), ("a", c_vp), ("b", c_vp), ("bins", c_vp), ("woff", c_vp), ("weights", c_vp),
    ]


_SIGNATURES = {
    "cpb_abi_version": (c_i32, []),
    "cpb_last_error": (ctypes.c_char_p, []),
    "cpb_set_option": (c_i32, [ctypes.c_char_p, c_i64]),
    "cpb_epsilon": (c_dbl, [c_dbl, c_dbl]),
    "cpb_field_plane_bytes": (c_i32, [c_i32, c_i32, c_i32, c_i64, c_i64, ctypes.POINTER(ctypes.c_size_t)]),
    "cpb_fit": (c_i32, [c_vp, c_i64, ctypes.POINTER(CpbField), c_vp, c_i32, c_vp]),
    "cpb_fit_multi": (c_i32, [c_vp, c_i64, ctypes.POINTER(ctypes.POINTER(CpbField)), c_i32, c_vp, c_i32,
                              c_vp]),
    "cpb_check_finite": (c_i32, [c_vp, c_i64, c_vp]),
    "cpb_fit_classify_work_bytes": (c_i32, [c_i64, c_i64, c_i64, ctypes.POINTER(ctypes.c_size_t)]),
    "cpb_fit_classify": (c_i32, [c_vp, c_i64, ctypes.POINTER(CpbField), c_vp, c_i32, c_i64, c_i64, c_vp, c_vp,
                                 c_vp, c_vp, c_vp]),
    "cpb_fit_multi_classify": (c_i32, [c_vp, c_i64, ctypes.POINTER(ctypes.POINTER(CpbField)), c_i32, c_vp,
                                       c_i32, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "cpb_fit_classify_finish": (c_i32, [ctypes.POINTER(CpbField), c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                                        c_vp, c_vp]),
    "cpb_read_range": (c_i32, [c_vp, ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl), c_vp]),
    "cpb_range_to_pair": (c_i32, [c_vp, c_vp, c_vp]),
    "cpb_pair_to_eps": (c_i32, [c_vp, c_vp, c_vp]),
    "cpb_from_scalar": (c_i32, [c_vp, c_i64, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_vp]),
    "cpb_classify_closed": (c_i32, [ctypes.POINTER(CpbField), c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "cpb_classify_closed_counts": (c_i32, [ctypes.POINTER(CpbField), c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                                           c_vp]),
    "cpb_classify_mc": (c_i32, [ctypes.POINTER(CpbField), c_i64, c_i64, c_u64, c_i64, c_i32,
                                c_vp, c_vp, c_vp, c_vp, c_vp]),
    "cpb_classify_semi": (c_i32, [ctypes.POINTER(CpbField), c_i64, c_i64, c_u64, c_i64, c_vp, c_vp,
                                  c_vp, c_vp]),
    "cpb_classify_combinatorial": (c_i32, [ctypes.POINTER(CpbField), c_i64, c_i64, c_vp, c_vp, c_vp,
                                           c_vp]),
    "cpb_materialize": (c_i32, [ctypes.POINTER(CpbField), c_vp, c_vp, c_vp, c_vp]),
    "cpb_unit_block": (c_i32, [c_u64, c_vp, c_i64, c_i32, c_i64, c_i64, c_vp, c_vp]),
    "cpb_synth_ensemble": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_dbl, c_u64, c_vp]),
    "cpb_run_host": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_i32, c_i32, c_dbl, c_i32, c_u64, c_i64,
                             c_u32, c_vp, c_vp, c_vp, c_vp]),
    "cpb_run_host_models": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_i32, ctypes.POINTER(c_i32),
                                    ctypes.POINTER(c_i32), ctypes.POINTER(c_dbl), c_i32, c_u64,
                                    c_i64, c_u32, ctypes.POINTER(c_vp), c_vp]),
    "cpb_heatmap": (c_i32, [c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp]),
    "cpb_cases_closed": (c_i32, [ctypes.POINTER(CpbCaseBatch), c_vp, c_vp]),
    "cpb_cases_mc": (c_i32, [ctypes.POINTER(CpbCaseBatch), c_u64, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "cpb_cases_semi": (c_i32, [ctypes.POINTER(CpbCaseBatch), c_u64, c_vp, c_i64, c_vp, c_vp]),
    "cpb_cases_combinatorial": (c_i32, [ctypes.POINTER(CpbCaseBatch), c_vp, c_vp]),
    "cpb_host_alloc": (c_i32, [ctypes.POINTER(c_vp), ctypes.c_size_t]),
    "cpb_host_free": (c_i32, [c_vp]),
    "cpb_release_workspace": (c_i32, [ctypes.POINTER(ctypes.c_size_t)]),
}

EXPORTED = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


class CudaPathError(RuntimeError):
    """The CUDA library could not run (missing build, no device, CUDA error)."""


def load(require_device: bool = True) -> ctypes.CDLL:
    """Load the shared library (once).  Raises if it is absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise CudaPathError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2407_18015_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise CudaPathError("critprob_b200 needs a CUDA device (there is no CPU fallback)")
    return _lib


def check(status: int) -> None:
    """Map a cpb_status to the reference's exception types."""
    if status == CPB_OK:
        return
    msg = _lib.cpb_last_error().decode(errors="replace") if _lib is not None else ""
    if status in (CPB_EINVAL, CPB_ENONFINITE):
        raise ValueError(msg)
    if status == CPB_ENOMEM:
        raise MemoryError(msg)
    raise CudaPathError(msg or f"critprob_b200 status {status}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
