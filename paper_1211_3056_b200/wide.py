"""High-degree (delta_R >= 3) super-domains: the paper's large super-domain
polynomial generation, as an extension of the
reference, which rejects delta >= 3 (polygen.py:81-82).

One Taylor polynomial R_t of degree delta_R covers a super-domain of up to
2^25 domains (2^40 arguments at N = 2^15): the host (libhrbhost.so,
hrbh_wide_blocks) builds it with its rigorous error budget and splits it
hierarchically into r_j(i) = Delta^j R_t(i N) of degree delta_R - j in the
domain index; the device (libhrb200.so, hrb_wrun_slice) walks r_0 and r_1
with multi-limb add-with-carry difference tables (F = 32 max(4, delta_R)
bits), tests every domain, refines the failures and walks the survivors
exactly at degree delta_R.  The specification is oracle/wide.py.

Parity: UNPINNED for the tabulated values and the phase flags (no
reference exists for delta >= 3); the confirmed HR records are pinned to
the reference's exhaustive_hr_search (oracle.py:77-113) and equal the
delta = 2 pipeline's, because every filter is sound.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import hostgen
from .fpformat import FpFormat, HrCaseRecord, index_bits
from .arith import UFrac
from .taylor import PolyGenConfig

# super-domain size (log2 arguments) per degree at which eps_approx stays
# below ~2^-50 for exp on [1, 2) (oracle/wide.py sizing; Lagrange term)
DEFAULT_LOG2_SUPER = {3: 27, 4: 33, 5: 36, 6: 40, 7: 40, 8: 40}


@dataclass(frozen=True, slots=True)
class WideGenConfig:
    """delta_R in 3..8; tau domains of N arguments per super-domain; guard
    bits of the enclosures (as PolyGenConfig.guard)."""

    delta: int = 4
    tau: int = 1 << 18
    N: int = 1 << 15
    guard: int = 32

    def __post_init__(self) -> None:
        if not 3 <= self.delta <= 8:
            raise ValueError("the high-degree path takes delta in 3..8 (delta <= 2: PolyGenConfig)")
        if self.N < 1 or self.N & (self.N - 1) or self.N > 1 << 16:
            raise ValueError("N must be a power of two <= 2^16")
        if self.tau < 1 or self.tau > 1 << 32:
            raise ValueError("tau outside [1, 2^32]")

    @property
    def frac_limbs(self) -> int:
        return max(4, self.delta)

    @property
    def frac_bits(self) -> int:
        return 32 * self.frac_limbs

    @staticmethod
    def for_degree(delta: int, N: int = 1 << 15, guard: int = 32) -> "WideGenConfig":
        lg = DEFAULT_LOG2_SUPER[delta]
        return WideGenConfig(delta, max(1, (1 << lg) // N), N, guard)

    def planning_config(self) -> PolyGenConfig:
        """The block planner's view (plan_arrays reads tau, N, mu, nu)."""
        return PolyGenConfig(tau=self.tau, N=self.N, mu=1, nu=self.tau, delta=2, limbs=16,
                             frac_bits=min(self.frac_bits, 512), guard=self.guard)


@dataclass
class WideSliceBatch:
    """Host-side hrb_wslice (include/hrb200.h) plus the metadata to map
    results back."""

    fmt: FpFormat
    binade: int
    wcfg: WideGenConfig
    coef: np.ndarray      # uint32 [(D+1)(D+2)/2, NL, S]
    padg: np.ndarray      # uint64 [2, S]
    s2b: np.ndarray       # uint64 [2, S]
    win: np.ndarray       # uint32 [NL, S]
    n_dom: np.ndarray
    dom_n: np.ndarray
    last_n: np.ndarray
    dom_base: np.ndarray
    m0: np.ndarray
    counts: np.ndarray
    id0: int = 0
    keep: list = field(default_factory=list)

    @property
    def n_super(self) -> int:
        return len(self.n_dom)

    @property
    def n_total(self) -> int:
        return int(self.dom_base[-1])

    @property
    def max_dom_n(self) -> int:
        return int(max(self.dom_n.max(), self.last_n.max()))

    @property
    def arguments(self) -> int:
        return int(self.counts.sum())

    @property
    def delta(self) -> int:
        return self.wcfg.delta

    @property
    def frac_limbs(self) -> int:
        return self.wcfg.frac_limbs

    def desc(self, ptrs=None) -> "nat.HrbWSlice":
        p = ptrs or {k: getattr(self, k).ctypes.data for k in WIDE_INPUTS}
        return nat.HrbWSlice(n_super=self.n_super, n_total=self.n_total, max_dom_n=self.max_dom_n,
                             degree=self.delta, frac_limbs=self.frac_limbs, word_bits=64, **p)


WIDE_INPUTS = ("coef", "padg", "s2b", "win", "n_dom", "dom_n", "last_n", "dom_base", "m0")


def plan_wide(fn: str, binade: int, fmt: FpFormat, wcfg: WideGenConfig, start: int, count: int, id0: int = 0):
    from .slices import plan_arrays

    return plan_arrays(fn, binade, fmt, wcfg.planning_config(), start, count, id0)


def pack_wide(plan, wcfg: WideGenConfig, workers: int = 0) -> WideSliceBatch:
    """Native high-degree Taylor models of the planned blocks, packed."""
    if plan.fn not in hostgen.FN_CODES or plan.binade > 0:
        raise ValueError("the high-degree path covers exp on binades <= 0")
    fmt = plan.fmt
    cfg = hostgen.make_cfg(plan.fn, fmt, PolyGenConfig(guard=wcfg.guard), plan.binade, 64)
    coef, padg, s2b, win, status = hostgen.wide_columns(cfg, wcfg.delta, wcfg.frac_limbs, plan.bstart, plan.bcount,
                                                        plan.n_p, plan.tau, plan.e_out, workers)
    bad = np.flatnonzero(status != hostgen.HRBH_OK)
    if len(bad):
        t = int(bad[0])
        raise ValueError(f"high-degree super-domain {t} (index {int(plan.bstart[t])}, {int(plan.bcount[t])} args, "
                         f"delta {wcfg.delta}) is out of range: eps'' >= 1/4 or pad too wide; use smaller super-domains")
    dom_base = np.zeros(len(plan) + 1, dtype=np.uint64)
    np.cumsum(plan.tau, out=dom_base[1:])
    last_n = (plan.bcount - (plan.tau.astype(np.uint64) - np.uint64(1)) * plan.n_p.astype(np.uint64)).astype(np.uint32)
    return WideSliceBatch(fmt, plan.binade, wcfg, coef, padg, s2b, win, plan.tau.copy(), plan.n_p.copy(), last_n,
                          dom_base, plan.bstart.copy(), plan.bcount.copy(), id0=int(plan.dom_id0[0]))


def prepare_wide(fn: str, binade: int, start: int, count: int, fmt: FpFormat, wcfg: WideGenConfig,
                 workers: int = 0, id0: int = 0) -> WideSliceBatch:
    return pack_wide(plan_wide(fn, binade, fmt, wcfg, start, count, id0), wcfg, workers)


@dataclass
class WideResult:
    counts: np.ndarray      # [6] fails, survivors, candidates, iterations, phase-2 args, phase-3 args
    cand_index: np.ndarray
    cand_dist: np.ndarray
    cand_dom: np.ndarray
    device_ms: float


def run_wide_host(batch: WideSliceBatch, algo_code: int = 2, split: int = 8, cand_cap: int = 1 << 16) -> WideResult:
    """hrb_wrun_slice_host: one call, host buffers in and out."""
    nat.require_cuda()
    lib = nat.load()
    arrs = {k: np.ascontiguousarray(getattr(batch, k)) for k in WIDE_INPUTS}
    desc = batch.desc({k: v.ctypes.data for k, v in arrs.items()})
    counts = np.zeros(6, dtype=np.uint64)
    ms = C.c_float(0)
    while True:
        cm, cd, cdom = (np.zeros(max(cand_cap, 1), dtype=np.uint64) for _ in range(3))
        rc = lib.hrb_wrun_slice_host(C.byref(desc), algo_code, split, counts.ctypes.data, cm.ctypes.data,
                                     cd.ctypes.data, cdom.ctypes.data, cand_cap, C.byref(ms))
        if rc == nat.HRB_ERR_CAPACITY and int(counts[2]) > cand_cap:
            cand_cap = int(counts[2])
            continue
        nat.check("hrb_wrun_slice_host", rc)
        break
    nc = int(counts[2])
    return WideResult(counts, cm[:nc], cd[:nc], cdom[:nc], ms.value)


class WideDeviceSlice:
    """A WideSliceBatch resident in HBM (the bench's inputs-resident step)."""

    def __init__(self, batch: WideSliceBatch):
        torch = nat.require_cuda()
        self.torch = torch
        self.batch = batch
        dev = torch.device("cuda", torch.cuda.current_device())
        self.t = {}
        for k in WIDE_INPUTS:
            a = np.ascontiguousarray(getattr(batch, k))
            view = a.view(np.int32) if a.dtype == np.uint32 else a.view(np.int64)
            self.t[k] = torch.from_numpy(view).to(dev)
        self.desc = batch.desc({k: v.data_ptr() for k, v in self.t.items()})
        self.device = dev

    def empty64(self, n: int):
        return self.torch.empty(max(int(n), 1), dtype=self.torch.int64, device=self.device)


class WideRunner:
    """hrb_wrun_slice on persistent device buffers (no host sync per step)."""

    def __init__(self, ds: WideDeviceSlice, algo_code: int = 2, split: int = 8, sub_cap: int | None = None,
                 cand_cap: int = 1 << 16):
        self.ds, self.algo, self.split = ds, algo_code, split
        b = ds.batch
        self.fail = ds.empty64(b.n_total)
        self.sub_cap = sub_cap if sub_cap is not None else max(1 << 16, b.n_total // 4)
        self.cand_cap = cand_cap
        self.subs = ds.empty64(self.sub_cap)
        self.cm, self.cd, self.cdom = ds.empty64(cand_cap), ds.empty64(cand_cap), ds.empty64(cand_cap)
        self.counts = ds.empty64(6)
        self.out = nat.HrbRunOut(fail_ids=self.fail.data_ptr(), fail_cap=b.n_total, sub_keys=self.subs.data_ptr(),
                                 sub_cap=self.sub_cap, cand_index=self.cm.data_ptr(), cand_dist=self.cd.data_ptr(),
                                 cand_dom=self.cdom.data_ptr(), cand_cap=cand_cap, counts=self.counts.data_ptr())

    def launch(self, stream=None) -> None:
        lib = nat.load()
        nat.check("hrb_wrun_slice", lib.hrb_wrun_slice(C.byref(self.ds.desc), self.algo, self.split,
                                                        C.byref(self.out), nat.stream_ptr(stream)))

    def counts_host(self) -> np.ndarray:
        return self.counts.cpu().numpy().view(np.uint64)

    def result(self):
        c = self.counts_host()
        nf, ns, nc = int(c[0]), min(int(c[1]), self.sub_cap), min(int(c[2]), self.cand_cap)
        u = lambda t, n: t[:n].cpu().numpy().view(np.uint64)  # noqa: E731
        return c, u(self.fail, nf), u(self.subs, ns), u(self.cm, nc), u(self.cd, nc), u(self.cdom, nc)


def wide_domain_coefficients(batch: WideSliceBatch) -> np.ndarray:
    """hrb_wdomain_coefficients -> uint32 [D+1, NL, n_total]: every domain's
    (s_0..s_D) mod 2^F through the device's multi-limb packet walk."""
    ds = WideDeviceSlice(batch)
    torch = ds.torch
    lib = nat.load()
    D, NL = batch.delta, batch.frac_limbs
    out = torch.empty((D + 1) * NL * max(batch.n_total, 1), dtype=torch.int32, device=ds.device)
    nat.check("hrb_wdomain_coefficients", lib.hrb_wdomain_coefficients(C.byref(ds.desc), out.data_ptr(),
                                                                       nat.stream_ptr()))
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32).reshape(D + 1, NL, -1)[:, :, : batch.n_total]


def candidates_of(batch: WideSliceBatch, res: WideResult) -> list:
    fmt = batch.fmt
    return [HrCaseRecord(index_bits(batch.binade, int(m), fmt), UFrac(int(d), 64), batch.id0 + int(dm))
            for m, d, dm in zip(res.cand_index.tolist(), res.cand_dist.tolist(), res.cand_dom.tolist())]
