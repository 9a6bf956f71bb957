"""Super-domain generation and packing into the device slice layout.

Host half of the hybrid split (PAPER.md "CPU-GPU" polynomial generation):
for an argument-index range of one binade this module reproduces the
super-domain schedule of /root/reference/pkg/src/hardround/pipeline.py:374-409
(_build_tasks: output-exponent pieces 296-347, adaptive domain size 350-371,
tau*N blocks, taylor_approx + hierarchical_split per block), then packs the
per-block r_j polynomials, the eps' budget and the domain geometry into the
structure-of-arrays layout of include/hrb200.h (hrb_slice).

It also performs every check that makes the reference raise on this path --
MPInt limb overflow in the coefficient walk (fixedpoint.py:136), the eps''
< 1/4 budget (fpmodel.py:224-225), the configured budget ceiling
(pipeline.py:225-226) and the SearchProblem eps < 1/2 rule
(lowerbound.py:64-65) -- exactly, so the device never sees a slice the
reference would have rejected.
"""

from __future__ import annotations

import functools

import math
import os
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Sequence

import numpy as np

from .arith import LIMB_BITS, MPInt, MPOverflowError, as_int
from .enclosure import derivative_bound, is_polynomial, value_exponent
from .fpformat import Domain, ErrorBudget, FpFormat
from .taylor import BinomialPoly, PolyGenConfig, hierarchical_split, straightforward_shift, taylor_approx


@dataclass(frozen=True, slots=True)
class SuperDomain:
    """One Taylor block: `tau` domains of `n_p` arguments (the last may be
    shorter) starting at binade index `index_start`."""

    index_start: int
    count: int
    n_p: int
    tau: int
    mu: int
    nu: int
    e_out: int
    dom_id0: int
    r_polys: tuple          # BinomialPoly per j = 0..delta (hierarchical_split)
    eps_prime: Fraction     # eps + eps_approx of this block

    @property
    def last_count(self) -> int:
        return self.count - (self.tau - 1) * self.n_p

    def domain_count(self, i: int) -> int:
        return self.last_count if i == self.tau - 1 else self.n_p


# ---------------------------------------------------------------- schedule


def output_binade_pieces(fn: str, binade: int, fmt: FpFormat) -> list[tuple[int, int, int]]:
    """Maximal runs (start, count, e_out) of constant output exponent over
    the binade's argument indices (pipeline.py:296-347)."""
    return list(_output_binade_pieces(fn, binade, fmt))


@functools.lru_cache(maxsize=256)
def _output_binade_pieces(fn: str, binade: int, fmt: FpFormat) -> tuple[tuple[int, int, int], ...]:
    # a pure function of its arguments (rigorous exponent enclosures), planned
    # once per (fn, binade, format) instead of once per slice / interval
    count = 1 << (fmt.precision - 1)
    base = Domain(1 << (fmt.precision - 1), binade + 1, count)

    def e_at(i: int) -> int:
        return value_exponent(fn, base.x_at(i, fmt))

    if is_polynomial(fn):
        pieces, run_start, run_e = [], None, None
        for i in range(count):
            try:
                e_i = e_at(i)
            except ValueError:  # fn(x) == 0
                e_i = None
            if e_i != run_e:
                if run_e is not None:
                    pieces.append((run_start, i - run_start, run_e))
                run_start, run_e = i, e_i
        if run_e is not None:
            pieces.append((run_start, count - run_start, run_e))
        return tuple(pieces)
    start = 1 if (fn == "log" and binade == 0) else 0
    pieces = []
    while start < count:
        e0 = e_at(start)
        if e_at(count - 1) == e0:
            pieces.append((start, count - start, e0))
            break
        lo, hi = start, count - 1  # e is monotone: binary search the last index with e0
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if e_at(mid) == e0:
                lo = mid
            else:
                hi = mid - 1
        pieces.append((start, lo - start + 1, e0))
        start = lo + 1
    return tuple(pieces)


def piece_domain_size(fn: str, piece: Domain, e_out: int, fmt: FpFormat, n_max: int) -> int:
    """Largest power of two N <= n_max with |c2| (N-1)^2 < 1/8 on the piece
    (pipeline.py:350-371)."""
    norm = Fraction(2) ** (fmt.precision - e_out)
    ulp = Fraction(2) ** (piece.exponent - fmt.precision)
    c2 = norm * ulp**2 * derivative_bound(fn, 2, piece.x_at(0, fmt), piece.x_at(piece.count - 1, fmt))
    n = n_max
    while n > 1 and c2 * (n - 1) ** 2 >= Fraction(1, 8):
        n //= 2
    return n


@dataclass(frozen=True, slots=True)
class _Block:
    fn: str
    binade: int
    fmt: FpFormat
    bcfg: PolyGenConfig
    bstart: int
    bcount: int
    n_p: int
    e_out: int
    dom_id0: int


def _make_super(b: _Block) -> SuperDomain:
    m_base = 1 << (b.fmt.precision - 1)
    sup = Domain(m_base + b.bstart, b.binade + 1, b.bcount, b.dom_id0)
    r_t, eps_approx = taylor_approx(b.fn, sup, b.bcfg, b.fmt)
    r_polys = hierarchical_split(r_t, b.n_p, b.bcfg.delta)
    return SuperDomain(b.bstart, b.bcount, b.n_p, b.bcfg.tau, b.bcfg.mu, b.bcfg.nu, b.e_out, b.dom_id0,
                       tuple(r_polys), b.fmt.eps + eps_approx)


def plan_blocks(fn: str, binade: int, fmt: FpFormat, pg: PolyGenConfig, start: int, count: int,
                id0: int = 0) -> list[_Block]:
    """The super-domain schedule of _build_tasks restricted to indices
    [start, start + count); with the whole binade it is _build_tasks'."""
    blocks, next_id = [], id0
    for p_start, p_count, e_out in output_binade_pieces(fn, binade, fmt):
        lo, hi = max(p_start, start), min(p_start + p_count, start + count)
        if lo >= hi:
            continue
        piece = Domain((1 << (fmt.precision - 1)) + lo, binade + 1, hi - lo, 0)
        n_p = piece_domain_size(fn, piece, e_out, fmt, pg.N)
        block = pg.tau * n_p
        for bstart in range(lo, hi, block):
            bcount = min(block, hi - bstart)
            if bcount == block and n_p == pg.N:
                bcfg = pg
            else:
                tau_t = -(-bcount // n_p)
                bcfg = PolyGenConfig(tau=tau_t, N=n_p, mu=1, nu=tau_t, delta=pg.delta,
                                     limbs=pg.limbs, frac_bits=pg.frac_bits, guard=pg.guard)
            blocks.append(_Block(fn, binade, fmt, bcfg, bstart, bcount, n_p, e_out, next_id))
            next_id += bcfg.tau
    return blocks


def build_super_domains(fn: str, binade: int, fmt: FpFormat, pg: PolyGenConfig, start: int = 0,
                        count: int | None = None, workers: int = 1, id0: int = 0) -> list[SuperDomain]:
    """taylor_approx + hierarchical_split for every block of the range.
    workers > 1 fans the (independent) blocks out to a process pool: the
    mpmath host work, not the GPU, bounds large slices."""
    if count is None:
        count = (1 << (fmt.precision - 1)) - start
    return supers_of_blocks(plan_blocks(fn, binade, fmt, pg, start, count, id0), workers)


def supers_of_blocks(blocks: Sequence[_Block], workers: int = 1) -> list[SuperDomain]:
    """Taylor model + hierarchical split of planned blocks, in block order."""
    blocks = list(blocks)
    if workers > 1 and len(blocks) > 1:
        import multiprocessing as mp

        ctx = mp.get_context("fork")
        with ctx.Pool(workers) as pool:
            return pool.map(_make_super, blocks, chunksize=max(1, len(blocks) // (workers * 8)))
    return [_make_super(b) for b in blocks]


# ---------------------------------------------------------------- checks


def _walk_bound(sd: SuperDomain) -> int:
    """max over j of sum_l |c_l| tau^l: bounds every value the reference's
    packet walk (straightforward_shift seeds + tabulated steps) produces."""
    best = 0
    for rp in sd.r_polys:
        best = max(best, sum(abs(as_int(c)) * sd.tau**l for l, c in enumerate(rp.coeffs)))
    return best


def _emulate_walk(sd: SuperDomain, limbs: int) -> None:
    """Exact replay of generate_packets (polygen.py:255-271) with MPInt
    semantics; raises MPOverflowError where the reference would."""
    for rp in sd.r_polys:
        mp = BinomialPoly(tuple(MPInt.from_int(as_int(c), limbs) for c in rp.coeffs), rp.scale)
        for u in range(sd.mu):
            col = list(straightforward_shift(mp, u * sd.nu).coeffs)
            for i in range(1, sd.nu):
                for l in range(len(col) - 1):
                    col[l] = col[l] + col[l + 1]


def domain_poly(sd: SuperDomain, i: int) -> tuple[int, ...]:
    """(s_0..s_delta) of domain i: r_j(i) by exact evaluation (equals the walk)."""
    return tuple(as_int(BinomialPoly(tuple(as_int(c) for c in rp.coeffs)).evaluate(i)) for rp in sd.r_polys)


def eps_dprime(sd: SuperDomain, count: int, frac_bits: int) -> Fraction:
    s2 = abs(as_int(sd.r_polys[2].coeffs[0])) if len(sd.r_polys) > 2 else 0
    return sd.eps_prime + Fraction(s2 * (count - 1) ** 2, 1 << frac_bits)


def check_super(sd: SuperDomain, fmt: FpFormat, pg: PolyGenConfig, word_bits: int,
                budget_ceiling: Fraction | None) -> bool:
    """Raise exactly where the reference's phase 1 would for this block;
    return whether phase-2 shifts are overflow-free by bound."""
    limbs = pg.limbs
    bound = _walk_bound(sd)
    if bound >> (LIMB_BITS * limbs) or (sd.tau * sd.tau) >> (LIMB_BITS * limbs):
        _emulate_walk(sd, limbs)
    # phase-1 budget at the largest count of the block (eps'' grows with count)
    n = max(sd.n_p if sd.tau > 1 else sd.last_count, sd.last_count)
    e_dp = eps_dprime(sd, n, pg.frac_bits)
    ErrorBudget(fmt.eps, sd.eps_prime - fmt.eps, e_dp - sd.eps_prime, Fraction(0))  # raises >= 1/4
    if budget_ceiling is not None and e_dp > budget_ceiling:
        raise ValueError("domain budget exceeds the configured ceiling")
    pad = -((-e_dp.numerator << word_bits) // e_dp.denominator) + n + 1
    if 2 * pad >= 1 << (word_bits - 1):
        raise ValueError("eps must be < 1/2")
    # phase-2 shift bound: |s_l| <= bound, shift by < n_p
    b2 = sum(bound * sd.n_p**l for l in range(len(sd.r_polys)))
    return not (b2 >> (LIMB_BITS * limbs))


def check_phase2_exact(sd: SuperDomain, i: int, split: int, limbs: int) -> None:
    """Exact MPInt replay of phase 2's straightforward_shift for one failing
    domain (used only when the cheap bound could not rule overflow out)."""
    s = domain_poly(sd, i)
    poly = BinomialPoly(tuple(MPInt.from_int(v, limbs) for v in s))
    n = sd.domain_count(i)
    step = max(n // split, 1)
    for start in range(0, n, step):
        straightforward_shift(poly, start)


# ---------------------------------------------------------------- packing


@dataclass
class SliceBatch:
    """Host-side hrb_slice (include/hrb200.h) plus the metadata the host
    needs to map results back (domain ids, argument indices)."""

    supers: list
    fmt: FpFormat
    binade: int
    frac_bits: int
    word_bits: int
    delta: int
    limbs: int
    coef: np.ndarray        # uint32 [6, CL, S]
    G: np.ndarray           # uint64 [2, S]
    s2abs: np.ndarray       # uint64 [2, S]
    n_dom: np.ndarray       # uint32 [S]
    dom_n: np.ndarray       # uint32 [S]
    last_n: np.ndarray      # uint32 [S]
    dom_base: np.ndarray    # uint64 [S+1]
    m0: np.ndarray          # uint64 [S]
    id0: int = 0
    shift_bound_ok: np.ndarray = field(default=None)  # bool [S]
    counts: np.ndarray = field(default=None)  # uint64 [S] arguments per super-domain
    nus: np.ndarray = field(default=None)     # uint32 [S] packet length nu (the reference's packet walk)
    # device copies of coef / G / s2abs still being downloaded into the
    # arrays above (pack_plan(resident=True)); None once they are final
    resident: object = field(default=None, repr=False, compare=False)

    def __post_init__(self) -> None:
        if self.counts is None:
            self.counts = np.array([s.count for s in self.supers], dtype=np.uint64)
        if self.nus is None:
            self.nus = np.array([s.nu for s in self.supers], dtype=np.uint32)

    @property
    def n_super(self) -> int:
        return len(self.n_dom)

    @property
    def n_total(self) -> int:
        return int(self.dom_base[-1])

    @property
    def coef_limbs(self) -> int:
        return self.coef.shape[1]

    @property
    def max_dom_n(self) -> int:
        return int(max(self.dom_n.max(), self.last_n.max()))

    @property
    def arguments(self) -> int:
        return int(self.counts.sum())

    def locate(self, local_ids: np.ndarray):
        """(super index, domain index within it) of slice-local ids."""
        t = np.searchsorted(self.dom_base, local_ids, side="right") - 1
        return t, local_ids - self.dom_base[t]

    def domain_sizes(self, local_ids: np.ndarray) -> np.ndarray:
        t, i = self.locate(np.asarray(local_ids, dtype=np.uint64))
        return np.where(i == self.n_dom[t].astype(np.uint64) - 1, self.last_n[t], self.dom_n[t]).astype(np.uint64)

    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.coef, self.G, self.s2abs, self.n_dom, self.dom_n, self.last_n,
                                      self.dom_base, self.m0))


def _limbs_of(v: int, cl: int) -> list[int]:
    v &= (1 << (32 * cl)) - 1  # two's complement over cl limbs
    return [(v >> (32 * l)) & 0xFFFFFFFF for l in range(cl)]


COEF_SLOTS = ((0, 0), (0, 1), (0, 2), (1, 0), (1, 1), (2, 0))  # (j, l) of coef rows


def _pack_rows(supers: Sequence[SuperDomain], fmt: FpFormat, pg: PolyGenConfig, word_bits: int,
               budget_ceiling: Fraction | None, check: bool):
    """The packed columns of a run of super-domains (and their checks, which
    raise exactly where the reference would)."""
    F = pg.frac_bits
    S = len(supers)
    cl = pg.limbs + 1  # MPInt magnitude < 2^(32 L) fits L+1 two's complement limbs
    coef = np.zeros((6, cl, S), dtype=np.uint32)
    G = np.zeros((2, S), dtype=np.uint64)
    s2 = np.zeros((2, S), dtype=np.uint64)
    meta = np.zeros((4, S), dtype=np.uint64)  # n_dom, dom_n, last_n, m0
    ok2 = np.ones(S, dtype=bool)
    m128 = (1 << 64) - 1
    for t, sd in enumerate(supers):
        if check:
            ok2[t] = check_super(sd, fmt, pg, word_bits, budget_ceiling)
        for row, (j, l) in enumerate(COEF_SLOTS):
            if j < len(sd.r_polys) and l < len(sd.r_polys[j].coeffs):
                coef[row, :, t] = _limbs_of(as_int(sd.r_polys[j].coeffs[l]), cl)
        g = -((-sd.eps_prime.numerator << F) // sd.eps_prime.denominator)  # ceil(eps' 2^F)
        G[0, t], G[1, t] = g & m128, g >> 64
        if len(sd.r_polys) > 2:
            a = min(abs(as_int(sd.r_polys[2].coeffs[0])), (1 << 128) - 1)
            s2[0, t], s2[1, t] = a & m128, a >> 64
        meta[:, t] = (sd.tau, sd.n_p, sd.last_count, sd.index_start)
    return coef, G, s2, meta, ok2


_PACK_JOB = None  # (supers, fmt, pg, word_bits, ceiling, check): inherited by forked workers
PACK_PARALLEL_MIN = 1024  # super-domains below which packing stays in-process (a fork costs more)


def _pack_range(rng):
    supers, fmt, pg, word_bits, ceiling, check = _PACK_JOB
    return _pack_rows(supers[rng[0]:rng[1]], fmt, pg, word_bits, ceiling, check)


def pack_slice(supers: Sequence[SuperDomain], fmt: FpFormat, pg: PolyGenConfig, word_bits: int,
               binade: int, budget_ceiling: Fraction | None = None, check: bool = True,
               workers: int = 1) -> SliceBatch:
    """hrb_slice columns of the super-domains, after the host checks.
    workers > 1 packs runs of super-domains in forked processes (the exact
    Fraction / MPInt checks dominate at 2^16 super-domains); a check that
    fails raises the error of the first failing super-domain, as the
    sequential loop does."""
    global _PACK_JOB
    if not supers:
        raise ValueError("empty slice")
    F = pg.frac_bits
    if not word_bits <= F <= 128:
        raise ValueError(f"the B200 path needs word_bits <= frac_bits <= 128 (got F={F}, W={word_bits})")
    S = len(supers)
    if workers > 1 and S >= max(4 * workers, PACK_PARALLEL_MIN):
        import multiprocessing as mp

        per = -(-S // (4 * workers))
        ranges = [(a, min(a + per, S)) for a in range(0, S, per)]
        _PACK_JOB = (list(supers), fmt, pg, word_bits, budget_ceiling, check)
        try:
            with mp.get_context("fork").Pool(workers) as pool:
                parts = pool.map(_pack_range, ranges, chunksize=1)
        finally:
            _PACK_JOB = None
        coef, G, s2, meta, ok2 = (np.concatenate([p[k] for p in parts], axis=-1) for k in range(5))
    else:
        coef, G, s2, meta, ok2 = _pack_rows(supers, fmt, pg, word_bits, budget_ceiling, check)
    n_dom, dom_n, last_n = (meta[k].astype(np.uint32) for k in range(3))
    m0 = meta[3].copy()
    dom_base = np.zeros(S + 1, dtype=np.uint64)
    np.cumsum(n_dom, out=dom_base[1:])
    return SliceBatch(list(supers), fmt, binade, F, word_bits, pg.delta, pg.limbs, coef, G, s2, n_dom, dom_n,
                      last_n, dom_base, m0, id0=supers[0].dom_id0, shift_bound_ok=ok2)


def slice_view(batch: SliceBatch, t0: int, t1: int) -> SliceBatch:
    """Contiguous sub-slice of super-domains [t0, t1) (a shard)."""
    db = batch.dom_base[t0:t1 + 1] - batch.dom_base[t0]
    return SliceBatch(batch.supers[t0:t1], batch.fmt, batch.binade, batch.frac_bits, batch.word_bits,
                      batch.delta, batch.limbs, np.ascontiguousarray(batch.coef[:, :, t0:t1]),
                      np.ascontiguousarray(batch.G[:, t0:t1]), np.ascontiguousarray(batch.s2abs[:, t0:t1]),
                      batch.n_dom[t0:t1].copy(), batch.dom_n[t0:t1].copy(), batch.last_n[t0:t1].copy(),
                      db, batch.m0[t0:t1].copy(), id0=batch.id0 + int(batch.dom_base[t0]),
                      shift_bound_ok=batch.shift_bound_ok[t0:t1].copy(), counts=batch.counts[t0:t1].copy(),
                      nus=batch.nus[t0:t1].copy())


def default_workers() -> int:
    return max(1, min(os.cpu_count() or 1, 64))


# ------------------------------------------------- vectorised plan + native


@dataclass
class BlockPlan:
    """The super-domain schedule of plan_blocks as columns (one entry per
    block), so that a 2^40-argument range (65,536 blocks) is planned without
    a Python object per block.  block(i) gives plan_blocks' _Block."""

    fn: str
    binade: int
    fmt: FpFormat
    pg: PolyGenConfig
    bstart: np.ndarray    # uint64 binade index of the first argument
    bcount: np.ndarray    # uint64 arguments
    n_p: np.ndarray       # uint32 domain size
    tau: np.ndarray       # uint32 domains
    mu: np.ndarray        # uint32 packets
    nu: np.ndarray        # uint32 domains per packet
    e_out: np.ndarray     # int32 output exponent
    dom_id0: np.ndarray   # uint64 first domain id

    def __len__(self) -> int:
        return len(self.bstart)

    def __getitem__(self, sl: slice) -> "BlockPlan":
        if not isinstance(sl, slice):
            raise TypeError("BlockPlan slices only; use block(i)")
        return BlockPlan(self.fn, self.binade, self.fmt, self.pg, *(getattr(self, k)[sl] for k in _PLAN_COLS))

    @property
    def sizes(self) -> np.ndarray:
        return self.bcount

    def block(self, i: int) -> _Block:
        pg = self.pg
        n_p, tau = int(self.n_p[i]), int(self.tau[i])
        if int(self.bcount[i]) == pg.tau * n_p and n_p == pg.N:
            bcfg = pg
        else:
            bcfg = PolyGenConfig(tau=tau, N=n_p, mu=1, nu=tau, delta=pg.delta, limbs=pg.limbs,
                                 frac_bits=pg.frac_bits, guard=pg.guard)
        return _Block(self.fn, self.binade, self.fmt, bcfg, int(self.bstart[i]), int(self.bcount[i]), n_p,
                      int(self.e_out[i]), int(self.dom_id0[i]))


_PLAN_COLS = ("bstart", "bcount", "n_p", "tau", "mu", "nu", "e_out", "dom_id0")


def plan_arrays(fn: str, binade: int, fmt: FpFormat, pg: PolyGenConfig, start: int, count: int,
                id0: int = 0) -> BlockPlan:
    """plan_blocks as columns: the same blocks, sizes and domain ids."""
    cols = {k: [] for k in _PLAN_COLS}
    next_id = id0
    for p_start, p_count, e_out in output_binade_pieces(fn, binade, fmt):
        lo, hi = max(p_start, start), min(p_start + p_count, start + count)
        if lo >= hi:
            continue
        piece = Domain((1 << (fmt.precision - 1)) + lo, binade + 1, hi - lo, 0)
        n_p = piece_domain_size(fn, piece, e_out, fmt, pg.N)
        block = pg.tau * n_p
        # every block of a piece is full-sized but its last: constant columns
        # with the last row patched (a block is "full" -- the tau/mu/nu
        # schedule -- when it holds `block` arguments and n_p == N)
        nb = -(-(hi - lo) // block)
        last = hi - lo - (nb - 1) * block
        tau_last = -(-last // n_p)
        mid_full = n_p == pg.N
        bst = np.arange(nb, dtype=np.uint64)
        bst *= np.uint64(block)
        bst += np.uint64(lo)
        bcnt = np.full(nb, block, dtype=np.uint64)
        bcnt[-1] = last
        tau = np.full(nb, pg.tau, dtype=np.uint32)
        tau[-1] = tau_last
        mu = np.full(nb, pg.mu if mid_full else 1, dtype=np.uint32)
        nu = np.full(nb, pg.nu, dtype=np.uint32) if mid_full else tau.copy()
        if not (mid_full and last == block):
            mu[-1], nu[-1] = 1, tau_last
        ids = np.arange(nb, dtype=np.uint64)
        ids *= np.uint64(pg.tau)
        ids += np.uint64(next_id)
        cols["bstart"].append(bst)
        cols["bcount"].append(bcnt)
        cols["n_p"].append(np.full(nb, n_p, dtype=np.uint32))
        cols["tau"].append(tau)
        cols["mu"].append(mu)
        cols["nu"].append(nu)
        cols["e_out"].append(np.full(nb, e_out, dtype=np.int32))
        cols["dom_id0"].append(ids)
        next_id += pg.tau * (nb - 1) + tau_last
    dt = {"bstart": np.uint64, "bcount": np.uint64, "n_p": np.uint32, "tau": np.uint32, "mu": np.uint32,
          "nu": np.uint32, "e_out": np.int32, "dom_id0": np.uint64}

    def column(k):  # no copy for the usual one-piece range
        c = cols[k]
        if not c:
            return np.zeros(0, dt[k])
        return (c[0] if len(c) == 1 else np.concatenate(c)).astype(dt[k], copy=False)

    return BlockPlan(fn, binade, fmt, pg, *(column(k) for k in _PLAN_COLS))


def _signed_limbs(col: np.ndarray) -> int:
    """Integer value of a two's-complement column of 32-bit limbs."""
    v = 0
    for k, w in enumerate(col.tolist()):
        v |= int(w) << (32 * k)
    bits = 32 * len(col)
    return v - (1 << bits) if v >> (bits - 1) else v


class PackedSupers:
    """Sequence view of a natively packed slice's super-domains: SuperDomain
    objects built on demand from the plan and the packed limbs (r_polys are
    exact: L+1 two's-complement limbs hold every MPInt-valid coefficient).
    eps_prime is not kept (the device reads G = ceil(eps' 2^F))."""

    def __init__(self, plan: BlockPlan, coef: np.ndarray, delta: int):
        self.plan, self.coef, self.delta = plan, coef, delta

    def __len__(self) -> int:
        return len(self.plan)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return PackedSupers(self.plan[i], self.coef[:, :, i], self.delta)
        if i < 0:
            i += len(self)
        pl = self.plan
        vals = [_signed_limbs(self.coef[row, :, i]) for row in range(6)]
        rows = [[vals[0], vals[1], vals[2]], [vals[3], vals[4]], [vals[5]]]
        rp = tuple(BinomialPoly(tuple(rows[j][:self.delta - j + 1]), pl.pg.frac_bits) for j in range(self.delta + 1))
        return SuperDomain(int(pl.bstart[i]), int(pl.bcount[i]), int(pl.n_p[i]), int(pl.tau[i]), int(pl.mu[i]),
                           int(pl.nu[i]), int(pl.e_out[i]), int(pl.dom_id0[i]), rp, None)

    def __iter__(self):
        return (self[i] for i in range(len(self)))


DEVICE_GEN_MIN = 256  # super-domains from which the device generation pays for its launch and copies


def _device_gen_ok(pg: PolyGenConfig, n: int) -> bool:
    if n < DEVICE_GEN_MIN or pg.limbs > 12 or pg.frac_bits + pg.guard > 224:
        return False
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pack_plan(plan: BlockPlan, word_bits: int, budget_ceiling: Fraction | None = None,
              workers: int = 1, native: bool | None = None, device: bool | None = None,
              resident: bool = False) -> SliceBatch:
    """Taylor models + split + checks + packing of planned blocks.

    With the native generation (exp on binades <= 0, delta <= 2, no budget
    ceiling) every block runs in compiled code, bit-identical to the Python
    path: on the GPU (hrb_pack_blocks, one thread per block) when CUDA is
    there and the slice has DEVICE_GEN_MIN blocks or more (device=True /
    False forces the choice), else in libhrbhost.so over `workers` host
    threads.  Blocks it flags go through the exact Python path one by one
    (raising the reference's error where the reference raises).
    native=False forces the Python path; otherwise the native path runs
    wherever it covers the configuration.  resident=True (run_range): with
    the device generation the columns also stay on the device
    (batch.resident, device.ResidentColumns) and the host copies of coef /
    G / s2abs are filled behind the search -- valid after
    batch.resident.wait(), which funnel.execute_batch_host calls."""
    from . import hostgen

    fmt, pg = plan.fmt, plan.pg
    F = pg.frac_bits
    if not len(plan):
        raise ValueError("empty slice")
    if not word_bits <= F <= 128:
        raise ValueError(f"the B200 path needs word_bits <= frac_bits <= 128 (got F={F}, W={word_bits})")
    use_native = native is not False and hostgen.covers(plan.fn, plan.binade, fmt, pg, budget_ceiling)
    if not use_native:
        blocks = [plan.block(i) for i in range(len(plan))]
        return pack_slice(supers_of_blocks(blocks, workers), fmt, pg, word_bits, plan.binade,
                          budget_ceiling=budget_ceiling, workers=workers)
    cfg = hostgen.make_cfg(plan.fn, fmt, pg, plan.binade, word_bits)
    if device is None:
        device = _device_gen_ok(pg, len(plan))
    sizes = []

    def size_columns():  # n_dom, dom_n, last_n, dom_base, m0
        n_dom = plan.tau.copy()
        last_n = (plan.bcount - (plan.tau.astype(np.uint64) - np.uint64(1)) * plan.n_p.astype(np.uint64)).astype(
            np.uint32)
        dom_base = np.zeros(len(plan) + 1, dtype=np.uint64)
        np.cumsum(n_dom.astype(np.int64), out=dom_base[1:].view(np.int64))  # numpy's int64 scan: ~3x its uint64 one
        sizes[:] = [n_dom, plan.n_p.copy(), last_n, dom_base, plan.bstart.copy()]
        return sizes

    res = None
    if device:
        from .device import pack_columns_device

        if resident:
            # the size columns are computed and uploaded while the kernel runs
            coef, G, s2, status, ok2, res = pack_columns_device(cfg, plan.bstart, plan.bcount, plan.n_p, plan.tau,
                                                                plan.e_out, resident=True, during=size_columns)
        else:
            coef, G, s2, status, ok2 = pack_columns_device(cfg, plan.bstart, plan.bcount, plan.n_p, plan.tau,
                                                           plan.e_out)
    else:
        coef, G, s2, status, ok2 = hostgen.pack_columns(cfg, plan.bstart, plan.bcount, plan.n_p, plan.tau,
                                                        plan.e_out, workers)
    fallback = np.flatnonzero(status != hostgen.HRBH_OK).tolist()
    if fallback and res is not None:
        res.wait()  # the host columns are patched below, then sent back
    for t in fallback:
        sd = _make_super(plan.block(t))  # exact Python path; raises where the reference raises
        c1, g1, s21, _, k1 = _pack_rows([sd], fmt, pg, word_bits, budget_ceiling, True)
        coef[:, :, t], G[:, t], s2[:, t], ok2[t] = c1[:, :, 0], g1[:, 0], s21[:, 0], k1[0]
    if fallback and res is not None:
        res.upload(coef, G, s2)
    n_dom, dom_n, last_n, dom_base, m0 = sizes or size_columns()
    return SliceBatch(PackedSupers(plan, coef, pg.delta), fmt, plan.binade, F, word_bits, pg.delta, pg.limbs, coef,
                      G, s2, n_dom, dom_n, last_n, dom_base, m0, id0=int(plan.dom_id0[0]),
                      shift_bound_ok=ok2.astype(bool), counts=plan.bcount.copy(), nus=plan.nu.copy(),
                      resident=res)
