"""Lower-bound searches for min{(b - a*x) mod 1 : x < N}, served by the GPU.

Drop-in for /root/reference/pkg/src/hardround/lowerbound.py: the same
Verdict / Algorithm / SearchProblem / SearchOutcome types (36-77) and the
SEARCHES registry (321-381), every call executed by hrb_search_batch
(include/hrb200.h) with bit-identical (verdict, d, iterations,
points_placed).  `search_many` is the batched form the pipeline uses; the
per-problem callables exist for API completeness (one launch per call).

The optional `trace` list of the reference (branch decisions, consumed by
its warp simulator) is served by hrb_search_trace, which records the same
decision stream on the device.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np

from .arith import MODE_CODE, DivisionMode, UFrac


class Verdict(Enum):
    SUCCESS = "success"
    FAILURE = "failure"


class Algorithm(Enum):
    LEFEVRE = "lefevre"
    LEFEVRE_SWAP = "lefevre_swap"
    REGULAR = "regular"
    REGULAR_UNROLLED = "regular_unrolled"


ALGO_CODE = {Algorithm.LEFEVRE: 0, Algorithm.LEFEVRE_SWAP: 1, Algorithm.REGULAR: 2, Algorithm.REGULAR_UNROLLED: 3}


@dataclass(frozen=True, slots=True)
class SearchProblem:
    a: UFrac
    b: UFrac
    eps: UFrac
    count: int

    def __post_init__(self) -> None:
        if self.count < 1:
            raise ValueError("count must be >= 1")
        if self.b.width != self.a.width or self.eps.width != self.a.width:
            raise ValueError("mixed word widths in problem")
        if self.eps.raw >= 1 << (self.a.width - 1):
            raise ValueError("eps must be < 1/2")


@dataclass(frozen=True, slots=True)
class SearchOutcome:
    verdict: Verdict
    d: UFrac
    iterations: int
    points_placed: int

    @property
    def success(self) -> bool:
        return self.verdict is Verdict.SUCCESS


def search_arrays(algo: Algorithm | str, word_bits: int, a, b, eps, count,
                  mode: DivisionMode = DivisionMode.HYBRID):
    """Raw batched form on uint64 arrays -> (ok, d, iterations, points_lo,
    points_hi); points_placed = points_lo + 2^64 points_hi."""
    from .device import search_batch_arrays

    algo = Algorithm(algo)
    ok, d, it, pl, ph = search_batch_arrays(ALGO_CODE[algo], MODE_CODE[mode], word_bits, a, b, eps, count)
    return ok.astype(bool), d, it, pl, ph


def search_many(problems: Sequence[SearchProblem], algo: Algorithm | str = Algorithm.REGULAR,
                mode: DivisionMode = DivisionMode.HYBRID) -> list[SearchOutcome]:
    """One device launch for the whole batch (all problems share a width)."""
    problems = list(problems)
    if not problems:
        return []
    w = problems[0].a.width
    if any(p.a.width != w for p in problems):
        raise ValueError("mixed word widths in batch")
    a = np.array([p.a.raw for p in problems], dtype=np.uint64)
    b = np.array([p.b.raw for p in problems], dtype=np.uint64)
    e = np.array([p.eps.raw for p in problems], dtype=np.uint64)
    n = np.array([p.count for p in problems], dtype=np.uint64)
    ok, d, it, pl, ph = search_arrays(algo, w, a, b, e, n, mode)
    return [SearchOutcome(Verdict.SUCCESS if ok[k] else Verdict.FAILURE, UFrac(int(d[k]), w), int(it[k]),
                          int(pl[k]) | (int(ph[k]) << 64)) for k in range(len(problems))]


def _single(algo: Algorithm):
    def run(problem: SearchProblem, mode: DivisionMode = DivisionMode.HYBRID, trace: list | None = None):
        if trace is None:
            return search_many([problem], algo, mode)[0]
        from .device import search_trace_arrays

        p = problem
        ok, d, it, pl, ph, paths = search_trace_arrays(ALGO_CODE[algo], MODE_CODE[mode], p.a.width, [p.a.raw],
                                                       [p.b.raw], [p.eps.raw], [p.count])
        trace.extend(paths[0])
        return SearchOutcome(Verdict.SUCCESS if ok[0] else Verdict.FAILURE, UFrac(int(d[0]), p.a.width), int(it[0]),
                             int(pl[0]) | (int(ph[0]) << 64))

    run.__name__ = f"{algo.value}_lb"
    return run


lefevre_lb = _single(Algorithm.LEFEVRE)
lefevre_swap_lb = _single(Algorithm.LEFEVRE_SWAP)
regular_lb = _single(Algorithm.REGULAR)
regular_unrolled_lb = _single(Algorithm.REGULAR_UNROLLED)

SEARCHES = {
    Algorithm.LEFEVRE: lefevre_lb,
    Algorithm.LEFEVRE_SWAP: lefevre_swap_lb,
    Algorithm.REGULAR: regular_lb,
    Algorithm.REGULAR_UNROLLED: regular_unrolled_lb,
}
