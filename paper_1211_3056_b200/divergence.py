"""Warp divergence of the searches, measured on the device.

Drop-in for /root/reference/pkg/src/hardround/divergence.py.  The reference
*simulates* SIMT warps: it replays each search with a `trace` list and
groups consecutive problems into warps of 32 lanes.  Here the same
quantities come from the real kernels.  hrb_search_trace returns every
lane's outcome, iteration count and branch-decision stream (bit-identical to
the reference cores' traces), and hrb_search_batch gives the iteration counts
alone for large batches (measure_warps).

Definitions kept from the reference: MDM = max(l) - mean(l) and
NMDM = 1 - mean(l)/max(l) per warp (divergence.py:96-110), the static
branch-cost table BRANCH_WEIGHTS (139-144) and its serialization estimate
(113-122, 185-201).  linear_problem_batch (32-93) is the config-2 problem
generator, restated on this package's host enclosures.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Iterable, Sequence

import numpy as np

from .arith import DivisionMode, MODE_CODE, UFrac
from .search import ALGO_CODE, Algorithm, SearchOutcome, SearchProblem, Verdict

WARP_WIDTH = 32


# ----------------------------------------------------------- problem batches


def _slope(fn: str, x: Fraction, value: Fraction, prec: int) -> Fraction:
    from .enclosure import enclose, is_polynomial, poly_value

    if fn == "exp":
        return value
    if fn == "exp2":
        lo, hi = enclose("log", Fraction(2), prec)
        return value * (lo + hi) / 2
    if fn == "log":
        return 1 / x
    if fn == "identity":
        return Fraction(1)
    if is_polynomial(fn):
        return poly_value(fn, x, 1)
    raise ValueError(f"unsupported function {fn!r}")


def _linear_problems(args) -> list[SearchProblem]:
    from .enclosure import enclose, value_exponent
    from .fpformat import Domain

    fn, fmt, binade, domain_size, total, starts, word_bits, eps = args
    half = 1 << (fmt.precision - 1)
    prec = word_bits + 32
    ulp = Fraction(1, 1 << (fmt.precision - 1 - binade))
    out = []
    for start in starts:
        x = Domain(half + start, binade + 1, 1, 0).x_at(0, fmt)
        scale = Fraction(2) ** (fmt.precision - value_exponent(fn, x))
        lo, hi = enclose(fn, x, prec)
        mid = (lo + hi) / 2
        a = (_slope(fn, x, mid, prec) * ulp * scale) % 1
        out.append(SearchProblem(UFrac.from_fraction(a, word_bits), UFrac.from_fraction((mid * scale) % 1, word_bits),
                                 UFrac.from_fraction(2 * eps, word_bits), min(domain_size, total - start)))
    return out


def linear_problem_batch(fn: str, fmt, binade: int, domain_size: int, domain_count: int | None = None,
                         word_bits: int = 64, eps: Fraction | None = None, workers: int = 1) -> list[SearchProblem]:
    """One linearised problem per subdomain of `domain_size` consecutive
    arguments of the binade: b = {2^(p-e) f(x0)}, a = {f'(x0) ulp 2^(p-e)},
    eps = 2 eps_fmt, count = the subdomain size (divergence.py:32-93).
    `workers` > 1 spreads the (independent) enclosures over host processes."""
    if domain_size < 1:
        raise ValueError("domain_size must be >= 1")
    half = 1 << (fmt.precision - 1)
    total = half if domain_count is None else domain_count * domain_size
    if not 1 <= total <= half:
        raise ValueError("batch does not fit in one binade")
    eps = fmt.eps if eps is None else eps
    starts = list(range(0, total, domain_size))
    if workers <= 1 or len(starts) < 2 * workers:
        return _linear_problems((fn, fmt, binade, domain_size, total, starts, word_bits, eps))
    import multiprocessing as mp

    chunk = -(-len(starts) // (workers * 4))
    jobs = [(fn, fmt, binade, domain_size, total, starts[k:k + chunk], word_bits, eps)
            for k in range(0, len(starts), chunk)]
    with mp.get_context("fork").Pool(workers) as pool:
        return [p for part in pool.map(_linear_problems, jobs) for p in part]


def problem_arrays(problems: Sequence[SearchProblem]):
    """SoA uint64 arrays (a, b, eps, count) and the common word width."""
    w = problems[0].a.width
    a = np.array([p.a.raw for p in problems], dtype=np.uint64)
    b = np.array([p.b.raw for p in problems], dtype=np.uint64)
    e = np.array([p.eps.raw for p in problems], dtype=np.uint64)
    n = np.array([p.count for p in problems], dtype=np.uint64)
    return a, b, e, n, w


# ---------------------------------------------------------------- metrics


def mdm(lane_iterations: Sequence[int]) -> Fraction:
    """Mean deviation to the maximum, exact: max(l) - mean(l)."""
    lanes = list(lane_iterations)
    if not lanes:
        raise ValueError("empty lane vector")
    return max(lanes) - Fraction(sum(lanes), len(lanes))


def nmdm(lane_iterations: Sequence[int]) -> Fraction:
    """Normalised MDM, exact: 1 - mean(l)/max(l); 0 for an all-zero warp."""
    lanes = list(lane_iterations)
    if not lanes:
        raise ValueError("empty lane vector")
    top = max(lanes)
    return Fraction(0) if top == 0 else 1 - Fraction(sum(lanes), len(lanes) * top)


def branch_serialization_estimate(n_then: int, n_else: int, diverged: bool, taken: bool = True) -> int:
    """Instructions one conditional issues: both bodies when the warp
    diverged, else the one body every lane took."""
    if min(n_then, n_else) < 0:
        raise ValueError("negative instruction count")
    if diverged:
        return n_then + n_else
    return n_then if taken else n_else


@dataclass(frozen=True, slots=True)
class BranchWeights:
    """Static then/else body sizes of an algorithm's main conditional;
    unified bodies pay only a predicated fixup when lanes disagree."""

    then_cost: int
    else_cost: int
    unified: bool = False
    fixup_cost: int = 1


BRANCH_WEIGHTS = {
    Algorithm.LEFEVRE: BranchWeights(7, 9),
    Algorithm.LEFEVRE_SWAP: BranchWeights(9, 9, unified=True, fixup_cost=2),
    Algorithm.REGULAR: BranchWeights(6, 6),
    Algorithm.REGULAR_UNROLLED: BranchWeights(3, 1, unified=True),
}


@dataclass(frozen=True, slots=True)
class WarpTrace:
    lane_iterations: tuple
    lane_branch_counts: tuple
    branch_paths: tuple
    outcomes: tuple


@dataclass(frozen=True, slots=True)
class WarpStats:
    mdm: Fraction
    nmdm: Fraction
    serialized_iterations: int
    branch_serialized_instructions: int

    def __post_init__(self) -> None:
        if not 0 <= self.nmdm < 1:
            raise ValueError("nmdm out of [0, 1)")


@dataclass(frozen=True, slots=True)
class DivergenceReport:
    algorithm: Algorithm
    traces: tuple
    warps: tuple
    min_iterations: int
    max_iterations: int
    mean_iterations: Fraction
    mean_nmdm: Fraction


def _serialized(paths: Sequence[Sequence[bool]], w: BranchWeights) -> int:
    total = 0
    for step in range(max((len(p) for p in paths), default=0)):
        live = [p[step] for p in paths if len(p) > step]
        then_any, else_any = any(live), not all(live)
        split = then_any and else_any
        if w.unified:
            total += max(w.then_cost, w.else_cost) + (w.fixup_cost if split else 0)
        else:
            total += branch_serialization_estimate(w.then_cost, w.else_cost, split, taken=then_any)
    return total


def simulate_warps(problems: Iterable[SearchProblem], algo: Algorithm | str = Algorithm.REGULAR,
                   div_mode: DivisionMode = DivisionMode.HYBRID, warp_width: int = WARP_WIDTH) -> DivergenceReport:
    """Group the ordered batch into warps of `warp_width` lanes; every lane's
    search runs on the device with its decision stream recorded
    (hrb_search_trace), and the per-warp statistics are the reference's."""
    from .device import search_trace_arrays

    algo = Algorithm(algo)
    if warp_width < 1:
        raise ValueError("warp_width must be >= 1")
    batch = list(problems)
    if not batch:
        raise ValueError("empty problem batch")
    a, b, e, n, w = problem_arrays(batch)
    if any(p.a.width != w for p in batch):
        raise ValueError("mixed word widths in batch")
    ok, d, it, pl, ph, paths = search_trace_arrays(ALGO_CODE[algo], MODE_CODE[div_mode], w, a, b, e, n)
    weights = BRANCH_WEIGHTS[algo]
    traces, stats = [], []
    for base in range(0, len(batch), warp_width):
        lanes = range(base, min(base + warp_width, len(batch)))
        iters = tuple(int(it[k]) for k in lanes)
        lp = tuple(tuple(paths[k]) for k in lanes)
        outs = tuple(SearchOutcome(Verdict.SUCCESS if ok[k] else Verdict.FAILURE, UFrac(int(d[k]), w), int(it[k]),
                                   int(pl[k]) | (int(ph[k]) << 64)) for k in lanes)
        counts = tuple((sum(p), len(p) - sum(p)) for p in lp)
        t = WarpTrace(iters, counts, lp, outs)
        traces.append(t)
        stats.append(WarpStats(mdm(iters), nmdm(iters), max(iters), _serialized(lp, weights)))
    all_it = [int(x) for x in it]
    return DivergenceReport(algo, tuple(traces), tuple(stats), min(all_it), max(all_it),
                            Fraction(sum(all_it), len(all_it)), Fraction(sum(s.nmdm for s in stats), len(stats)))


def report_rows(report: DivergenceReport) -> list[tuple[int, int, float, float, float]]:
    """(warp_id, max_iter, mean_iter, mdm, nmdm) per warp, for CSV."""
    return [(k, s.serialized_iterations, float(Fraction(sum(t.lane_iterations), len(t.lane_iterations))),
             float(s.mdm), float(s.nmdm)) for k, (t, s) in enumerate(zip(report.traces, report.warps))]


# ------------------------------------------------- large batches (config 2)


@dataclass
class WarpSummary:
    """Per-warp iteration statistics of a large batch (float, vectorised)."""

    lane_iterations: np.ndarray   # uint64 [n]
    warp_max: np.ndarray          # [n_warps]
    warp_mean: np.ndarray
    warp_nmdm: np.ndarray

    @property
    def mean_nmdm(self) -> float:
        return float(self.warp_nmdm.mean())

    def spread_ok_fraction(self, spread: int = 2) -> float:
        """Share of warps whose lanes' iteration counts span <= `spread`."""
        n = len(self.warp_max)
        lanes = self.lane_iterations[: n * WARP_WIDTH].reshape(n, -1) if n else self.lane_iterations
        return float(((lanes.max(axis=1) - lanes.min(axis=1)) <= spread).mean()) if n else 1.0


def warp_summary(iterations: np.ndarray, warp_width: int = WARP_WIDTH) -> WarpSummary:
    it = np.asarray(iterations, dtype=np.uint64)
    n = len(it) // warp_width
    lanes = it[: n * warp_width].reshape(n, warp_width).astype(np.float64)
    mx = lanes.max(axis=1)
    mean = lanes.mean(axis=1)
    nm = np.where(mx > 0, 1.0 - mean / np.where(mx > 0, mx, 1.0), 0.0)
    return WarpSummary(it, mx, mean, nm)


def measure_warps(a, b, eps, count, algo: Algorithm | str = Algorithm.REGULAR,
                  div_mode: DivisionMode = DivisionMode.HYBRID, word_bits: int = 64) -> WarpSummary:
    """Per-lane iteration counts of a (large) SoA batch from one
    hrb_search_batch launch, summarised per warp of 32 consecutive lanes."""
    from .device import search_batch_arrays

    algo = Algorithm(algo)
    ok, d, it, pl, ph = search_batch_arrays(ALGO_CODE[algo], MODE_CODE[div_mode], word_bits, a, b, eps, count)
    return warp_summary(it)
