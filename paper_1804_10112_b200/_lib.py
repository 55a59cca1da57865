"""ctypes binding of the sm_100a kernel library (include/sl_abi.h).

The library is built in-tree by paper_1804_10112_b200.build.  There is no CPU
fallback: if the library is missing or no CUDA device is present, every
compute entry point raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

from . import errors as E

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "_lib" / "libsl_b200.so"
HEADER = PKG.parent / "include" / "sl_abi.h"

SL_OK = 0
_STATUS_EXC = {
    1: ValueError,
    2: E.UnsupportedCapabilityError,
    3: E.AssemblyError,
    4: E.HashSegmentFullError,
    5: E.UnsupportedMergeError,
    6: E.UnsupportedOutputError,
    7: OverflowError,
    8: ValueError,
    9: E.DeviceError,
}

# level kinds / function ids (sl_abi.h)
KIND_ID = {"dense": 0, "range": 1, "compressed": 2, "singleton": 3, "offset": 4, "hashed": 5}
FN_ID = {"coord_bounds": 0, "coord_access": 1, "pos_bounds": 2, "pos_access": 3, "locate": 4,
         "size": 5}


class SlLevel(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("crd_stride", ctypes.c_int32),
                ("crd_base", ctypes.c_int32), ("noffset", ctypes.c_int32),
                ("n", ctypes.c_int64), ("m", ctypes.c_int64), ("w", ctypes.c_int64),
                ("range_n", ctypes.c_int64), ("pos", ctypes.c_void_p),
                ("crd", ctypes.c_void_p), ("offset", ctypes.c_void_p)]


_i32, _i64, _p, _sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
SIGNATURES = {
    "sl_version": ([], ctypes.c_int),
    "sl_status_string": ([ctypes.c_int], ctypes.c_char_p),
    "sl_last_cuda_error": ([], ctypes.c_int),
    "sl_device_sm_count": ([_p], ctypes.c_int),
    "sl_level_query": ([ctypes.POINTER(SlLevel), _i32, _i64, _p, _p, _p, _p, _p], ctypes.c_int),
    "sl_hashed_locate": ([_i64, _p, _p, _i64, _p, _p, _p, _i32, _p], ctypes.c_int),
    "sl_hashed_insert_init": ([_i64, _p, _p], ctypes.c_int),
    "sl_hashed_insert": ([_i64, _p, _p, _i64, _p, _p, _p], ctypes.c_int),
    "sl_hashed_insert_ordered_workspace_bytes": ([_i64, _i64], _sz),
    "sl_hashed_insert_ordered": ([_i64, _p, _p, _i64, _i64, _p, _p, _p, _sz, _p], ctypes.c_int),
    "sl_spmv_coo_f64": ([_i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _sz, _p], ctypes.c_int),
    "sl_spmv_coo_workspace_bytes": ([_i64], _sz),
    "sl_build_features": ([], ctypes.c_int),
    "sl_spmv_csr_peers_f64": ([_i64, _i64, _i64, _p, _p, _p, _p, _p, _i32, _p], ctypes.c_int),
    "sl_spmv_csr_workspace_bytes": ([_i64, _i64, _i32], _sz),
    "sl_spmv_csr_f64": ([_i64, _i64, _i64, _p, _p, _p, _p, _p, _i32, _p, _sz, _p], ctypes.c_int),
    "sl_spmv_ell_f64": ([_i64, _i64, _i32, _p, _p, _p, _p, _p], ctypes.c_int),
    "sl_spmv_dia_f64": ([_i64, _i64, _i32, _p, _i32, _p, _p, _p, _p], ctypes.c_int),
    "sl_spmv_dia_rows_f64": ([_i64, _i64, _i64, _i32, _p, _i32, _p, _p, _p, _p], ctypes.c_int),
    "sl_spmv_csr_hashx_f64": ([_i64, _p, _p, _p, _i64, _p, _p, _p, _p], ctypes.c_int),
    "sl_add_csr_workspace_bytes": ([_i64, _i64], _sz),
    "sl_add_csr_count": ([_i64, _p, _p, _i64, _p, _p, _p, _p, _p, _sz, _p], ctypes.c_int),
    "sl_add_csr_fill": ([_i64, _p, _p, _p, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p],
                        ctypes.c_int),
    "sl_add_csr_f64": ([_i64, _p, _p, _p, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p],
                       ctypes.c_int),
    "sl_mttkrp_workspace_bytes": ([_i64, _i32], _sz),
    "sl_mttkrp_coo3_f64": ([_i64, _i64, _i64, _i32, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _sz,
                            _p], ctypes.c_int),
    "sl_mttkrp_csf_f64": ([_i64, _i64, _i64, _i32, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _p,
                           _p, _p, _p, _sz, _p], ctypes.c_int),
    "sl_convert_coo_to_csr": ([_i64, _i64, _p, _p, _p], ctypes.c_int),
    "sl_convert_coo_to_csr_exact_workspace_bytes": ([_i64, _i64], _sz),
    "sl_convert_coo_to_csr_exact": ([_i64, _i64, _p, _p, _p, _p, _p, _p, _p, _sz, _p],
                                    ctypes.c_int),
    "sl_csr_max_row_length": ([_i64, _p, _p, _p, _p], ctypes.c_int),
    "sl_convert_csr_to_ell": ([_i64, _i32, _p, _p, _p, _p, _p, _p], ctypes.c_int),
    "sl_convert_coo_to_dia_workspace_bytes": ([_i64, _i64], _sz),
    "sl_convert_coo_to_dia_offsets": ([_i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _sz, _p],
                                      ctypes.c_int),
    "sl_convert_coo_to_dia_values": ([_i64, _i64, _i64, _i32, _p, _p, _p, _p, _p, _sz, _p],
                                     ctypes.c_int),
    "sl_hashed_slot_map_workspace_bytes": ([_i64, _i64], _sz),
    "sl_hashed_slot_map": ([_i64, _i64, _p, _p, _sz, _p], ctypes.c_int),
    "sl_spmv_csr_hashx_map_workspace_bytes": ([_i64, _i64], _sz),
    "sl_spmv_csr_hashx_map_f64": ([_i64, _i64, _i64, _p, _p, _p, _i64, _p, _p, _p, _p, _sz, _p],
                                  ctypes.c_int),
    "sl_spmv_csr_spx_workspace_bytes": ([_i64], _sz),
    "sl_spmv_csr_spx_f64": ([_i64, _i64, _i64, _p, _p, _p, _i64, _p, _p, _p, _p, _sz, _p],
                            ctypes.c_int),
    "sl_spmm_csr_f64": ([_i64, _i64, _i64, _p, _p, _p, _p, _p, _p], ctypes.c_int),
    "sl_spmm_csr_nnz_f64": ([_i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p], ctypes.c_int),
    "sl_spmm_csr_split_workspace_bytes": ([_i64, _i64, ctypes.c_int32], _i64),
    "sl_spmm_csr_split_f64": ([_i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, ctypes.c_int32, _p,
                               _i64, _p], ctypes.c_int),
    "sl_csf_fiber_scatter_f64": ([_i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p],
                                 ctypes.c_int),
    "sl_csf_fiber_rowptr": ([_i64, _i64, _p, _p, _p, _p], ctypes.c_int),
    "sl_inner_coo3_workspace_bytes": ([_i64], _sz),
    "sl_inner_coo3_f64": ([_i64, _i64, _i64, _i64, _p, _p, _p, _p, _i64, _p, _p, _p, _p, _p, _p,
                           _sz, _p], ctypes.c_int),
    "sl_csr_row_indices": ([_i64, _p, _p, _p], ctypes.c_int),
    "sl_l2_flush": ([_p, _sz, _p], ctypes.c_int),
    "sl_l2_read": ([_p, _sz, _p, _p], ctypes.c_int),
}

_LIB = None


def header_symbols():
    """Function names declared in include/sl_abi.h."""
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sl_[a-z0-9_]+)\s*\(", text)))


def load(path: Path = LIB_PATH):
    """Load the library (no CUDA context is created)."""
    global _LIB
    if _LIB is None:
        # SL_LIB_PATH: load another build of the same ABI (A/B timing of two builds)
        override = "SL_LIB_PATH" in os.environ
        path = Path(os.environ.get("SL_LIB_PATH", str(path)))
        if not path.exists():
            raise E.DeviceError(
                f"kernel library {path} is missing: run `python -m paper_1804_10112_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(path))
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None and override:   # an older build under A/B: bind what it has
                continue
            if fn is None:
                raise E.DeviceError(f"{path} does not export {name}: rebuild the library")
            fn.argtypes = args
            fn.restype = res
        _LIB = L
    return _LIB


def check(status: int, what: str = "") -> None:
    if status == SL_OK:
        return
    msg = load().sl_status_string(status).decode()
    exc = _STATUS_EXC.get(status, E.DeviceError)
    raise exc(f"{what}: {msg}" if what else msg)


def require_device(t, what="tensor"):
    """Every array handed to a kernel must already be a CUDA tensor."""
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise E.DeviceError(f"{what} must be a CUDA tensor (no CPU fallback)")
    return t


def ptr(t):
    return None if t is None else t.data_ptr()


def stream_handle(stream=None):
    """cudaStream_t of `stream`, else of the current device's current stream
    (the raw query: torch.cuda.current_stream() costs several microseconds of
    Python per launch, which the e2e step pays on every call)."""
    import torch

    if stream is not None:
        return stream.cuda_stream
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
