"""ctypes binding of libhoib200.so (the C ABI in include/hoi_b200.h).

Device memory and streams come from PyTorch (plumbing only); every numeric
stage of the hot path runs in the library's sm_100a kernels.  There is no
CPU fallback: if the library or a CUDA device is missing, the entry points
raise ``BackendUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import (HoiError, InsufficientSamples, InvalidData, NotPositiveDefinite)

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libhoib200.so"

OK, INVALID_ARG, INSUFFICIENT_SAMPLES, NOT_PD, CUDA_ERROR, CAPACITY, FALLBACK = range(7)

_lock = threading.Lock()
_lib = None


class BackendUnavailable(HoiError):
    """The CUDA library or a CUDA device is not available."""


_vp, _i32, _i64, _sz, _dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t, C.c_double
_SIGS = {
    "hoi_version": ([], C.c_int),
    "hoi_last_error": ([], C.c_char_p),
    "hoi_launch_count": ([], _i64),
    "hoi_rank_copula": ([_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, C.POINTER(_sz), _vp], C.c_int),
    "hoi_covariance": ([_vp, _i64, _i32, _i32, _vp, _vp], C.c_int),
    "hoi_rank_copula_cols": ([_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, C.POINTER(_sz), _vp],
                             C.c_int),
    "hoi_covariance_cols": ([_vp, _i64, _i32, _i32, _vp, _vp], C.c_int),
    "hoi_correlation": ([_vp, _i32, _i32, _vp, _vp, _vp], C.c_int),
    "hoi_eval_indices": ([_vp, _vp, _vp, _i32, _i32, _i32, _vp, _i64, _i32, _vp, _vp, _vp, _vp,
                          _vp, _i32, _vp], C.c_int),
    "hoi_eval_indices_into": ([_vp, _vp, _vp, _i32, _i32, _i32, _vp, _i64, _i32, _vp, _i64, _vp,
                               _vp, _i32, _vp], C.c_int),
    "hoi_eval_indices_fp32": ([_vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _i64, _i32, _vp, _vp,
                               _vp, _i32, _vp], C.c_int),
    "hoi_eval_masks": ([_vp, _vp, _vp, _i32, _i32, _i32, _vp, _i32, _i64, _vp, _vp, _vp, _vp,
                        _vp, _i32, _vp], C.c_int),
    "hoi_logdet_invdiag": ([_vp, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _vp], C.c_int),
    "hoi_unrank": ([_i32, _i32, _i32, _i64, _i64, _vp, _vp, _vp], C.c_int),
    "hoi_unrank_list": ([_i32, _i32, _i32, _vp, _i64, _vp, _vp, _vp], C.c_int),
    "hoi_scan_full": ([_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i64, _i64, _i32, _vp, _vp,
                       _vp, _i32, _vp, C.POINTER(_sz), _vp], C.c_int),
    "hoi_lattice_table": ([_vp, _i32, _i32, _i32, _vp, _sz, _vp], C.c_int),
    "hoi_lattice_status": ([_vp, _i32, _vp], C.c_int),
    "hoi_lattice_shard": ([_vp, _i32, _i32, _i32, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp,
                           _sz, _vp], C.c_int),
    "hoi_lattice_shard_filter": ([_vp, _i32, _i32, _i32, _vp, _i32, _i32, _i32, _i32, _i32, _i32,
                                  _i32, _dbl, _vp, _vp, _i64, _vp, _i32, _vp, _sz, _vp], C.c_int),
    "hoi_lattice_shard_set": ([_vp, _i32, _i32, _i32, _vp, _i32, _i32, _i32, C.c_uint64, _i32,
                               _vp, _vp, _sz, _vp], C.c_int),
    "hoi_lattice_shard_set_filter": ([_vp, _i32, _i32, _i32, _vp, _i32, _i32, _i32, C.c_uint64,
                                      _i32, _i32, _i32, _dbl, _vp, _vp, _i64, _vp, _i32, _vp, _sz,
                                      _vp], C.c_int),
    "hoi_lattice_filter": ([_vp, _i32, _i32, _i32, _vp, _i32, _i32, _i32, _i32, _dbl, _i32, _vp,
                            _vp, _i64, _vp, _vp], C.c_int),
    "hoi_lattice_measures": ([_vp, _i32, _i32, _i32, _vp, _i32, _i32, _i32, _i64, _i64, _vp,
                              _vp], C.c_int),
    "hoi_lattice_shard_local": ([_vp, _i32, _i32, _i32, _vp, _i32, _i32, _i32, C.c_uint64, _i32,
                                 _vp, _i64, _vp, _vp, _vp, _sz, _vp], C.c_int),
    "hoi_lattice_local_scatter": ([_vp, _i64, _vp, _vp, _i32, _i32, _i32, _i32, _i64, _i64, _vp,
                                   _vp], C.c_int),
    "hoi_topk_select": ([_vp, _i64, _i32, _i32, _dbl, _i64, _i64, _vp, _i64, C.POINTER(_i64),
                         _vp, _vp], C.c_int),
    "hoi_topk_select_multi": ([_vp, _i64, _i32, _dbl, _i64, _i64, _vp, _i64, C.POINTER(_i64),
                               _vp, _vp], C.c_int),
    "hoi_features": ([_vp, _i64, _i32, _i64, _i64, _i64, _vp, _vp, _i64, _vp], C.c_int),
    "hoi_objective": ([_vp, _i64, _i32, _i32, _vp, _vp, _i32, _dbl, _vp, _vp, _vp], C.c_int),
    "hoi_topk_order": ([_vp, _i32, _dbl, _vp, _i64, _vp, _vp, _i32, _i64, _vp, _vp], C.c_int),
    "hoi_topk_threshold": ([_vp, _i64, _i32, _i32, _dbl, _i64, _vp, _vp, _vp], C.c_int),
    "hoi_topk_bound": ([_vp, _i64, _i32, _i32, _dbl, _i64, _i32, _vp, _vp, _vp], C.c_int),
    "hoi_topk_filter": ([_vp, _i64, _i32, _i32, _dbl, _vp, _vp, _vp, _i64, _vp], C.c_int),
    "hoi_histogram": ([_vp, _i64, _i32, _i32, _dbl, _dbl, _vp, _vp, _vp], C.c_int),
    "hoi_fp64_probe": ([_vp, _i64, _i32, _vp], C.c_int),
}


def exported_symbols():
    return tuple(_SIGS)


def load(path: Path | None = None):
    """Load (without touching the GPU) and bind every exported symbol."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path or os.environ.get("HOI_B200_LIB", LIB_PATH))
        if not p.exists():
            raise BackendUnavailable(f"{p} is missing: run `python -m paper_2501_03381_b200._build` "
                                     "(or __graft_entry__.build())")
        lib = C.CDLL(str(p))
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if path is None:
            _lib = lib
        return lib


def torch_cuda():
    """Import torch and require a CUDA device (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device: the B200 engine has no CPU fallback")
    return torch


def lib():
    return _lib if _lib is not None else load()


def last_error() -> str:
    return lib().hoi_last_error().decode(errors="replace")


def check(status: int, what: str = ""):
    if status == OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == INVALID_ARG:
        raise InvalidData(msg)
    if status == INSUFFICIENT_SAMPLES:
        raise InsufficientSamples(msg)
    if status == NOT_PD:
        raise NotPositiveDefinite(msg)
    raise HoiError(f"CUDA backend error ({status}): {msg}")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle(torch):
    return torch.cuda.current_stream().cuda_stream


def launch_count() -> int:
    return int(lib().hoi_launch_count())


def traced(name: str):
    """Decorator: an NVTX range named `name` around a public entry point, so
    nsys / ncu timelines show the pipeline's stages (copula, covariance,
    scan, batch evaluation, TopK, shard) by the reference's names.  The push
    and pop are host calls of a few hundred nanoseconds; without a CUDA
    device the call runs unwrapped (its own checks raise as before)."""
    import functools

    def wrap(fn):
        @functools.wraps(fn)
        def run(*args, **kwargs):
            import torch
            if not torch.cuda.is_available():
                return fn(*args, **kwargs)
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*args, **kwargs)
            finally:
                torch.cuda.nvtx.range_pop()
        return run
    return wrap
