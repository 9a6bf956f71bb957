"""Native host half of the hybrid split (include/hrb_host.h, libhrbhost.so).

For exp on binades <= 0 with delta <= 2 -- the north-star workload -- the
per-super-domain host work of the reference (taylor_approx, polygen.py:
193-252; hierarchical_split 113-131; the MPInt / eps'' / pad checks of
phase 1, pipeline.py:141-184) and the candidate confirmation (decide_hr,
evalf.py:286-327, as pipeline.py:446-461 calls it) run in C++ over all host
threads, bit-identical to the reference: the interval exp these read
(mpmath 1.3.0 iv.exp) is restated exactly in csrc/host/mpexp.h.

Anything the library does not cover -- other functions, binades > 0, a
budget ceiling, or an item where the reference raises -- comes back flagged
and goes through the exact Python path (slices.py / enclosure.py), which
raises the reference's exception where the reference does.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .build import HOST_LIB, build_host

HRBH_OK = 0
HRBH_FALLBACK = 1
FN_CODES = {"exp": 0}

_lib = None
_lock = threading.Lock()


class HrbhCfg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("fn", "precision", "eps_bits", "binade", "frac_bits", "guard", "limbs",
                                         "delta", "word_bits")]


def load():
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("HRB_HOST_LIB") or build_host()
            lib = C.CDLL(path)
            P, I, I64 = C.c_void_p, C.c_int, C.c_int64
            lib.hrbh_version.restype = I
            lib.hrbh_pack_blocks.argtypes = [C.POINTER(HrbhCfg), I64, P, P, P, P, P, P, P, P, P, P, I]
            lib.hrbh_pack_blocks.restype = I
            lib.hrbh_confirm.argtypes = [C.POINTER(HrbhCfg), I64, P, P, P, P, I]
            lib.hrbh_confirm.restype = I
            lib.hrbh_wide_blocks.argtypes = [C.POINTER(HrbhCfg), I, I, I64, P, P, P, P, P, P, P, P, P, P, I]
            lib.hrbh_wide_blocks.restype = I
            lib.hrbh_exp_enclose.argtypes = [C.c_uint64, I, I, P, P, P, P, P]
            lib.hrbh_exp_enclose.restype = I
            _lib = lib
        return _lib


def covers(fn: str, binade: int, fmt, pg, budget_ceiling=None) -> bool:
    """Whether the native generator handles this configuration at all."""
    return (fn in FN_CODES and binade <= 0 and pg.delta in (1, 2) and budget_ceiling is None
            and 2 <= fmt.precision <= 64 and 1 <= pg.limbs <= 16)


def make_cfg(fn: str, fmt, pg, binade: int, word_bits: int) -> HrbhCfg:
    return HrbhCfg(FN_CODES[fn], fmt.precision, fmt.eps_bits, binade, pg.frac_bits, pg.guard, pg.limbs, pg.delta,
                   word_bits)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def pack_columns(cfg: HrbhCfg, index_start, count, n_p, tau, e_out, workers: int = 0):
    """Run hrbh_pack_blocks over S blocks; returns (coef, G, s2abs, status,
    shift_ok) as numpy arrays (columns of fallback items are zero)."""
    lib = load()
    S = len(index_start)
    cl = cfg.limbs + 1
    cols = [np.ascontiguousarray(index_start, dtype=np.uint64), np.ascontiguousarray(count, dtype=np.uint64),
            np.ascontiguousarray(n_p, dtype=np.uint32), np.ascontiguousarray(tau, dtype=np.uint32),
            np.ascontiguousarray(e_out, dtype=np.int32)]
    coef = np.zeros((6, cl, S), dtype=np.uint32)
    G = np.zeros((2, S), dtype=np.uint64)
    s2 = np.zeros((2, S), dtype=np.uint64)
    status = np.zeros(S, dtype=np.uint8)
    ok2 = np.zeros(S, dtype=np.uint8)
    rc = lib.hrbh_pack_blocks(C.byref(cfg), S, *(_ptr(a) for a in cols), _ptr(coef), _ptr(G), _ptr(s2),
                              _ptr(status), _ptr(ok2), int(workers))
    if rc:
        raise ValueError(f"hrbh_pack_blocks rejected the configuration (status {rc})")
    return coef, G, s2, status, ok2


def wide_columns(cfg: HrbhCfg, degree: int, frac_limbs: int, index_start, count, n_p, tau, e_out,
                 workers: int = 0):
    """hrbh_wide_blocks over S blocks: (coef [(D+1)(D+2)/2, NL, S] u32,
    padg [2, S], s2b [2, S], win [NL, S] u32, status [S])."""
    lib = load()
    S = len(index_start)
    cols = [np.ascontiguousarray(index_start, dtype=np.uint64), np.ascontiguousarray(count, dtype=np.uint64),
            np.ascontiguousarray(n_p, dtype=np.uint32), np.ascontiguousarray(tau, dtype=np.uint32),
            np.ascontiguousarray(e_out, dtype=np.int32)]
    ncoef = (degree + 1) * (degree + 2) // 2
    coef = np.zeros((ncoef, frac_limbs, S), dtype=np.uint32)
    padg = np.zeros((2, S), dtype=np.uint64)
    s2b = np.zeros((2, S), dtype=np.uint64)
    win = np.zeros((frac_limbs, S), dtype=np.uint32)
    status = np.zeros(S, dtype=np.uint8)
    rc = lib.hrbh_wide_blocks(C.byref(cfg), degree, frac_limbs, S, *(_ptr(a) for a in cols), _ptr(coef),
                              _ptr(padg), _ptr(s2b), _ptr(win), _ptr(status), int(workers))
    if rc:
        raise ValueError(f"hrbh_wide_blocks rejected the configuration (status {rc})")
    return coef, padg, s2b, win, status


def confirm(cfg: HrbhCfg, index: np.ndarray, workers: int = 0):
    """(is_hr, dist_raw, status) for candidates given by binade index."""
    lib = load()
    idx = np.ascontiguousarray(index, dtype=np.uint64)
    n = len(idx)
    is_hr = np.zeros(n, dtype=np.uint8)
    dist = np.zeros(n, dtype=np.uint64)
    status = np.zeros(n, dtype=np.uint8)
    rc = lib.hrbh_confirm(C.byref(cfg), n, _ptr(idx), _ptr(is_hr), _ptr(dist), _ptr(status), int(workers))
    if rc:
        raise ValueError(f"hrbh_confirm rejected the configuration (status {rc})")
    return is_hr, dist, status


def exp_enclose(M: int, xe: int, prec: int):
    """Native enclosure of exp(M 2^xe) as two Fractions (tests)."""
    from fractions import Fraction

    lib = load()
    lo = np.zeros(16, dtype=np.uint64)
    hi = np.zeros(16, dtype=np.uint64)
    le, he, nw = C.c_int32(), C.c_int32(), C.c_int32()
    rc = lib.hrbh_exp_enclose(M, xe, prec, _ptr(lo), C.byref(le), _ptr(hi), C.byref(he), C.byref(nw))
    if rc:
        return None
    lm = sum(int(lo[i]) << (64 * i) for i in range(nw.value))
    hm = sum(int(hi[i]) << (64 * i) for i in range(nw.value))
    return Fraction(lm) * Fraction(2) ** le.value, Fraction(hm) * Fraction(2) ** he.value
