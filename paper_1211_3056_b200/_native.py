"""ctypes binding of libhrb200.so (include/hrb200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every entry point raises.  Device memory comes from torch
(plumbing only); pointers cross the ABI as plain integers.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .build import LIB

HRB_OK = 0
HRB_ERR_RUNTIME = 1
HRB_ERR_CONFIG = 2
HRB_ERR_OVERFLOW = 4
HRB_ERR_CAPACITY = 8

ALGO_CODES = {"lefevre": 0, "lefevre_swap": 1, "regular": 2, "regular_unrolled": 3}

EXPORTS = (
    "hrb_version",
    "hrb_last_error",
    "hrb_device_info",
    "hrb_search_batch",
    "hrb_search_trace",
    "hrb_search_verdicts",
    "hrb_domain_coefficients",
    "hrb_phase1",
    "hrb_phase2",
    "hrb_phase3",
    "hrb_run_slice",
    "hrb_run_slice_host",
    "hrb_run_slice_resident",
    "hrb_wrun_slice",
    "hrb_wrun_slice_host",
    "hrb_wdomain_coefficients",
    "hrb_confirm_exp",
    "hrb_pack_blocks",
)


class HrbSlice(C.Structure):
    _fields_ = [
        ("n_super", C.c_int64),
        ("n_total", C.c_int64),
        ("max_dom_n", C.c_uint32),
        ("coef_limbs", C.c_int32),
        ("frac_bits", C.c_int32),
        ("word_bits", C.c_int32),
        ("delta", C.c_int32),
        ("coef", C.c_void_p),
        ("G", C.c_void_p),
        ("s2abs", C.c_void_p),
        ("n_dom", C.c_void_p),
        ("dom_n", C.c_void_p),
        ("last_n", C.c_void_p),
        ("dom_base", C.c_void_p),
        ("m0", C.c_void_p),
    ]


class HrbWSlice(C.Structure):
    _fields_ = [
        ("n_super", C.c_int64),
        ("n_total", C.c_int64),
        ("max_dom_n", C.c_uint32),
        ("degree", C.c_int32),
        ("frac_limbs", C.c_int32),
        ("word_bits", C.c_int32),
        ("coef", C.c_void_p),
        ("padg", C.c_void_p),
        ("s2b", C.c_void_p),
        ("win", C.c_void_p),
        ("n_dom", C.c_void_p),
        ("dom_n", C.c_void_p),
        ("last_n", C.c_void_p),
        ("dom_base", C.c_void_p),
        ("m0", C.c_void_p),
    ]


class HrbRunOut(C.Structure):
    _fields_ = [
        ("fail_ids", C.c_void_p),
        ("fail_cap", C.c_uint64),
        ("sub_keys", C.c_void_p),
        ("sub_cap", C.c_uint64),
        ("cand_index", C.c_void_p),
        ("cand_dist", C.c_void_p),
        ("cand_dom", C.c_void_p),
        ("cand_cap", C.c_uint64),
        ("counts", C.c_void_p),
    ]


class NativeError(RuntimeError):
    """A libhrb200 call returned a non-zero status."""

    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed with status {code}: {msg}")
        self.code = code


_lib = None
_lock = threading.Lock()


def _declare(lib) -> None:
    P, I, I64, U64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
    lib.hrb_version.restype = I
    lib.hrb_last_error.restype = C.c_char_p
    lib.hrb_device_info.argtypes = [I, C.c_char_p, I]
    lib.hrb_search_batch.argtypes = [I, I, I, I64, P, P, P, P, P, P, P, P, P, P]
    lib.hrb_search_verdicts.argtypes = [I, I, I64, P, P, P, P, P, P, P, P]
    lib.hrb_search_trace.argtypes = [I, I, I, I64, P, P, P, P, P, P, P, P, P, P, I64, P, P]
    lib.hrb_domain_coefficients.argtypes = [C.POINTER(HrbSlice), P, P]
    lib.hrb_phase1.argtypes = [C.POINTER(HrbSlice), I, I, P, P, U64, P, P]
    lib.hrb_phase2.argtypes = [C.POINTER(HrbSlice), I, I, I, P, P, U64, P, P, U64, P]
    lib.hrb_phase3.argtypes = [C.POINTER(HrbSlice), I, P, P, U64, P, P, P, P, U64, P]
    lib.hrb_run_slice.argtypes = [C.POINTER(HrbSlice), I, I, I, C.POINTER(HrbRunOut), P]
    lib.hrb_run_slice_host.argtypes = [C.POINTER(HrbSlice), I, I, I, P, P, U64, P, P, P, U64,
                                       C.POINTER(C.c_float)]
    lib.hrb_run_slice_resident.argtypes = [C.POINTER(HrbSlice), I, I, I, P, P, P, P, U64, C.POINTER(C.c_float), P]
    lib.hrb_wrun_slice.argtypes = [C.POINTER(HrbWSlice), I, I, C.POINTER(HrbRunOut), P]
    lib.hrb_wrun_slice_host.argtypes = [C.POINTER(HrbWSlice), I, I, P, P, P, P, U64, C.POINTER(C.c_float)]
    lib.hrb_wdomain_coefficients.argtypes = [C.POINTER(HrbWSlice), P, P]
    lib.hrb_confirm_exp.argtypes = [I, I, I, I64, P, P, P, P, P]
    lib.hrb_pack_blocks.argtypes = [P, I64, P, P, P, P, P, P, P, P, P, P, P]
    for name in EXPORTS:
        if name not in ("hrb_version", "hrb_last_error"):
            getattr(lib, name).restype = I


def load(path: str | None = None):
    """Load libhrb200.so (building it first if the sources are newer)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = path or os.environ.get("HRB_LIB")
        if path is None:
            from .build import build

            path = build()  # recompiles only when the sources' content hash changed
        lib = C.CDLL(path)
        _declare(lib)
        _lib = lib
        return lib


def check(fn: str, rc: int) -> None:
    if rc != HRB_OK:
        msg = load().hrb_last_error().decode(errors="replace")
        raise NativeError(fn, rc, msg)


def require_cuda():
    """The device path only: fail loudly instead of falling back to the CPU."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("hardround-b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    return torch


def stream_ptr(stream=None) -> int:
    torch = require_cuda()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
