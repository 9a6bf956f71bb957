"""CPU oracle for the HR-search hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package, and only as the checker or
the timed CPU baseline; the product path (paper_1211_3056_b200) never does.

It wraps hr_oracle.c, a plain-C restatement of the reference algorithms
(/root/reference/pkg/src/hardround/lowerbound.py:88-308,
polygen.py:134-158 + 255-280, pipeline.py:141-293; see that file's
header), compiled with gcc + OpenMP into oracle/_build/libhroracle.so.
The oracle is pinned against golden vectors produced by the reference
itself (tests/golden/make_golden.py, tests/test_oracle_golden.py).  There
is no oracle/_ref: the reference is a pure-Python package (nothing to
compile), and it cannot travel to the GPU box, so its outputs are committed
as fixtures instead.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libhroracle.so")

ALGO = {"lefevre": 0, "lefevre_swap": 1, "regular": 2, "regular_unrolled": 3}

_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "hr_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(src) > os.path.getmtime(LIB):
        subprocess.run(["make", "-s", "-C", HERE, "-B" if force else "all"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        P, I, I64, U64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
        L.or_search_batch.argtypes = [I, I, U64, U64, I64, P, P, P, P, P, P, P, P, P]
        L.or_set_threads.argtypes = [I]
        L.or_get_threads.restype = I
        slice_args = [I64, I, I, I, I, I, P, P, P, P, P, P, P, P, P]
        L.or_phase1_flat.argtypes = slice_args + [I, I, P, I64, P, I64]
        L.or_phase1_flat.restype = I64
        L.or_phase2_flat.argtypes = slice_args + [I, I, I, P, I64, P, P, P, P, P, I64]
        L.or_phase2_flat.restype = I64
        L.or_phase3_flat.argtypes = slice_args + [I64, P, P, P, P, P, P, P, I64]
        L.or_phase3_flat.restype = I64
        L.or_boolean_problem.argtypes = [U64] * 9 + [I, I, P]
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def threads() -> int:
    return int(lib().or_get_threads())


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def search_batch(algo: str, mode: int, one: int, a, b, eps, count):
    """The four reference cores over arrays (general modulus one <= 2^64).
    Returns (ok u8, d u64, it u64, points as python-int-capable (lo, hi))."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    e = np.ascontiguousarray(eps, dtype=np.uint64)
    n = np.ascontiguousarray(count, dtype=np.uint64)
    m = len(a)
    ok = np.zeros(m, np.uint8)
    d = np.zeros(m, np.uint64)
    it = np.zeros(m, np.uint64)
    pl = np.zeros(m, np.uint64)
    ph = np.zeros(m, np.uint64)
    lib().or_search_batch(ALGO[algo], int(mode), one & (2**64 - 1), one >> 64, m, _p(a), _p(b), _p(e), _p(n),
                          _p(ok), _p(d), _p(it), _p(pl), _p(ph))
    return ok, d, it, pl, ph


def _slice_args(batch):
    arrs = [np.ascontiguousarray(x) for x in (batch.coef, batch.G, batch.s2abs, batch.n_dom, batch.dom_n,
                                              batch.last_n)]
    nu = np.ascontiguousarray(batch.nus, dtype=np.uint32)
    dom_id0 = np.ascontiguousarray((batch.dom_base[:-1] + np.uint64(batch.id0)).astype(np.uint64))
    m0 = np.ascontiguousarray(batch.m0)
    keep = arrs + [nu, dom_id0, m0]
    args = [batch.n_super, batch.coef_limbs, batch.limbs, batch.frac_bits, batch.word_bits, batch.delta,
            *(_p(x) for x in keep)]
    return args, keep


def phase1(batch, algo: str, mode: int, with_coeffs: bool = False):
    """Failing GLOBAL domain ids (ascending) of a packed slice, following the
    reference's MPInt packet walk; optionally the per-domain residues
    (3 x 2 x n_total u64: s_j mod 2^128 as lo/hi)."""
    args, keep = _slice_args(batch)
    n_total = batch.n_total
    out = np.zeros(max(n_total, 1), np.uint64)
    coef = np.zeros((3, 2, max(n_total, 1)), np.uint64) if with_coeffs else None
    r = lib().or_phase1_flat(*args, ALGO[algo], int(mode), _p(out), n_total,
                             _p(coef) if with_coeffs else None, n_total)
    if r == -1:
        raise OverflowError("MPInt overflow in the coefficient walk")
    if r < 0:
        raise RuntimeError(f"or_phase1 failed ({r})")
    return (out[:r], coef) if with_coeffs else out[:r]


def phase2(batch, algo: str, mode: int, split: int, fail_ids):
    """Rows (global id, j, start, cnt) and shifted residues (rows x 6 u64)."""
    args, keep = _slice_args(batch)
    ids = np.ascontiguousarray(fail_ids, dtype=np.uint64)
    cap = max(len(ids) * 2 * split, 1)
    oid = np.zeros(cap, np.uint64)
    oj = np.zeros(cap, np.uint32)
    ost = np.zeros(cap, np.uint32)
    ocnt = np.zeros(cap, np.uint32)
    ores = np.zeros((cap, 6), np.uint64)
    r = lib().or_phase2_flat(*args, ALGO[algo], int(mode), int(split), _p(ids), len(ids), _p(oid), _p(oj), _p(ost),
                             _p(ocnt), _p(ores), cap)
    if r == -1:
        raise OverflowError("MPInt overflow in the phase-2 shift")
    if r < 0:
        raise RuntimeError(f"or_phase2 failed ({r})")
    return oid[:r], oj[:r], ost[:r], ocnt[:r], ores[:r]


def phase3(batch, rows):
    """Candidates (binade index, dist64, global domain id) from phase-2 rows."""
    oid, oj, ost, ocnt, ores = rows
    args, keep = _slice_args(batch)
    n = len(oid)
    cap = max(int(ocnt.astype(np.int64).sum()) if n else 1, 1)
    cap = min(cap, 1 << 26)
    om = np.zeros(cap, np.uint64)
    od = np.zeros(cap, np.uint64)
    oi = np.zeros(cap, np.uint64)
    ins = [np.ascontiguousarray(x) for x in (oid, ost, ocnt, ores)]
    r = lib().or_phase3_flat(*args, n, *(_p(x) for x in ins), _p(om), _p(od), _p(oi), cap)
    if r < 0:
        raise RuntimeError(f"or_phase3 failed ({r})")
    return om[:r], od[:r], oi[:r]


def boolean_problem(s0: int, s1: int, G: int, s2abs: int, n: int, F: int, W: int):
    """(a, b, eps) of the closed-form pad (pinned against Fractions in tests)."""
    out = np.zeros(4, np.uint64)
    m = 2**64 - 1
    s0 %= 1 << 128
    s1 %= 1 << 128
    lib().or_boolean_problem(s0 & m, s0 >> 64, s1 & m, s1 >> 64, G & m, G >> 64, s2abs & m, s2abs >> 64, n, F, W,
                             _p(out))
    return int(out[0]), int(out[1]), int(out[2]) | (int(out[3]) << 64)
