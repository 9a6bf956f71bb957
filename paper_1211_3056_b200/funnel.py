"""Three-phase HR-case funnel with the phases on the GPU.

Drop-in for /root/reference/pkg/src/hardround/pipeline.py: the same config
types (PhaseConfig 48-69, PipelineConfig 72-86), statistics (PhaseRow /
PhaseStats 89-112), task types (DomainTask / SubdomainTask 115-134),
algorithm auto-selection (select_algorithm 187-197), the per-phase entry
points (phase1 213-231, phase2 234-257, phase3_exhaustive 260-293) and the
binade driver (run_pipeline 412-463).  `run_slice` is the same driver over
an argument-index range (the reference runs only whole binades).

Host: output-exponent pieces, Taylor models, hierarchical split and the
final rigorous confirmation (decide_hr).  Device (include/hrb200.h): the
tabulated coefficient walk, Boolean problems, both search families,
subdomain refinement, the exhaustive walk, and all compaction.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Sequence

import numpy as np

from . import _native as nat
from .arith import LIMB_BITS, MODE_CODE, DivisionMode, MPInt, UFrac, as_int
from .enclosure import decide_hr
from .fpformat import Domain, ErrorBudget, FpFormat, HrCaseRecord, bits_float, index_bits
from .records import RecordSet
from .search import ALGO_CODE, Algorithm
from .slices import (SliceBatch, SuperDomain, build_super_domains, check_phase2_exact, domain_poly,
                     output_binade_pieces, pack_slice)
from .taylor import BinomialPoly, PolyGenConfig, straightforward_shift

ALGORITHMS = ("lefevre", "regular", "auto")
SELECT_THRESHOLD = 1e-3


@dataclass(frozen=True, slots=True)
class PhaseConfig:
    algorithm: str = "auto"
    div_mode: DivisionMode = DivisionMode.HYBRID
    phase2_split: int = 8
    budgets: ErrorBudget | None = None
    N1: int = 1 << 6
    parallel_width: int = 1  # host workers for Taylor generation (the device needs none)

    def __post_init__(self) -> None:
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"algorithm must be one of {ALGORITHMS}")
        if not 2 <= self.phase2_split <= 64:
            raise ValueError("phase2_split outside {2..64}")
        if self.N1 % self.phase2_split:
            raise ValueError("phase2_split must divide N1")
        if not 1 <= self.parallel_width <= 64:
            raise ValueError("parallel_width outside [1, 64]")


@dataclass(frozen=True, slots=True)
class PipelineConfig:
    fn: str
    fmt: FpFormat
    polygen: PolyGenConfig = PolyGenConfig()
    phase: PhaseConfig = PhaseConfig()
    word_bits: int = 64

    def __post_init__(self) -> None:
        if self.phase.N1 != self.polygen.N:
            raise ValueError("phase N1 and polygen N must agree")
        if self.word_bits not in (32, 64):
            raise ValueError("word_bits must be 32 or 64")
        if self.polygen.frac_bits > self.polygen.limbs * LIMB_BITS:
            raise ValueError("difference registers would not fit the limb budget")


@dataclass(frozen=True, slots=True)
class PhaseRow:
    phase: str
    domains_in: int
    domains_out: int
    arguments_covered: int
    wall_ms: float


@dataclass(slots=True)
class PhaseStats:
    rows: list = field(default_factory=list)
    algorithm_choices: list = field(default_factory=list)

    def row(self, phase: str) -> PhaseRow:
        for r in self.rows:
            if r.phase == phase:
                return r
        raise KeyError(phase)

    def phase3_phase1_ratio(self) -> float:
        p1 = self.row("phase1").domains_in
        return self.row("phase3").domains_in / p1 if p1 else 0.0


@dataclass(frozen=True, slots=True)
class DomainTask:
    domain: Domain
    coeffs: tuple
    frac_bits: int
    eps_prime: Fraction
    e_out: int


@dataclass(frozen=True, slots=True)
class SubdomainTask:
    parent: DomainTask
    sub_index: int
    start: int
    count: int
    coeffs: tuple


def select_algorithm(prev_interval_stats: PhaseStats | None, threshold: float = SELECT_THRESHOLD) -> str:
    """Heavy funnels (phase3/phase1 > threshold) pick the classic walk."""
    if prev_interval_stats is None:
        return "regular"
    try:
        ratio = prev_interval_stats.phase3_phase1_ratio()
    except KeyError:
        return "regular"
    return "lefevre" if ratio > threshold else "regular"


def _resolve(cfg: PipelineConfig, algo: str | None) -> str:
    return algo or (cfg.phase.algorithm if cfg.phase.algorithm != "auto" else "regular")


# ------------------------------------------------------------------ slices


@dataclass
class SliceOutput:
    """Everything one slice produced, in the reference's types and order.
    The per-domain outputs stay numpy arrays (a 2^40 slice fails millions of
    domains); failing_ids / sub_rows give the reference's list forms."""

    batch: SliceBatch
    fail_global: np.ndarray    # uint64 phase-1 failing global domain ids (ascending)
    sub_table: tuple           # uint64 arrays (parent id, sub index, start, count), ascending
    candidates: object         # RecordSet of phase-3 candidates (argument order; a Sequence of HrCaseRecord)
    records: object            # RecordSet of confirmed HR records (sorted)
    stats: PhaseStats
    iterations: int            # phase-1 quotient steps (SearchOutcome.iterations)

    @property
    def failing_ids(self) -> list:
        return self.fail_global.tolist()

    @property
    def sub_rows(self) -> list:
        return list(zip(*(a.tolist() for a in self.sub_table)))


def _sub_geometry(n: np.ndarray, j: np.ndarray, split: int):
    step = np.maximum(n // np.uint64(split), np.uint64(1))
    start = j * step
    cnt = np.minimum(step, n - start)
    return start, cnt


def execute_batch(batch: SliceBatch, cfg: PipelineConfig, algo: str, fn: str | None = None,
                  confirm: bool = True, workers: int | None = None) -> SliceOutput:
    """Run phases 1-3 of a packed slice on the current CUDA device, then
    confirm the candidates on the host (pipeline.py:447-462)."""
    from .device import DeviceSlice, run_phases

    fmt = cfg.fmt
    split = cfg.phase.phase2_split
    ds = DeviceSlice(batch)
    res = run_phases(ds, ALGO_CODE[Algorithm(algo)], MODE_CODE[cfg.phase.div_mode], split)
    id0 = batch.id0
    # phase-2 MPInt replay for blocks whose shift bound was inconclusive
    if batch.shift_bound_ok is not None and not batch.shift_bound_ok.all():
        t_idx, i_idx = batch.locate(res.fail_ids)
        for t, i in zip(t_idx.tolist(), i_idx.tolist()):
            if not batch.shift_bound_ok[t]:
                check_phase2_exact(batch.supers[t], i, split, cfg.polygen.limbs)
    stats = PhaseStats()
    fail_sizes = batch.domain_sizes(res.fail_ids)
    stats.rows.append(PhaseRow("phase1", batch.n_total, len(res.fail_ids), batch.arguments, res.phase_ms[0]))
    sub_local = res.sub_keys >> np.uint64(8)
    sub_j = res.sub_keys & np.uint64(255)
    sub_n = batch.domain_sizes(sub_local)
    sub_start, sub_cnt = _sub_geometry(sub_n, sub_j, split)
    stats.rows.append(PhaseRow("phase2", len(res.fail_ids), len(res.sub_keys), int(fail_sizes.sum()),
                               res.phase_ms[1]))
    cand = RecordSet(fmt.precision, batch.binade, res.cand_index, res.cand_dist, res.cand_dom + np.uint64(id0))
    stats.rows.append(PhaseRow("phase3", len(res.sub_keys), len(cand), int(sub_cnt.sum()), res.phase_ms[2]))
    t4 = time.perf_counter()
    records = confirm_set(fn or cfg.fn, cand, fmt, workers if workers is not None else cfg.phase.parallel_width) \
        if confirm else RecordSet(fmt.precision, batch.binade, [], [], [])
    stats.rows.append(PhaseRow("confirm", len(cand), len(records), len(cand), (time.perf_counter() - t4) * 1e3))
    table = (sub_local + np.uint64(id0), sub_j, sub_start, sub_cnt)
    return SliceOutput(batch, res.fail_ids + np.uint64(id0), table, cand, records, stats, res.iterations)


def execute_batch_host(batch: SliceBatch, cfg: PipelineConfig, algo: str, fn: str | None = None,
                       confirm: bool = True, workers: int | None = None) -> SliceOutput:
    """execute_batch through ONE host-buffer ABI call (hrb_run_slice_host:
    streamed upload behind phase 1, all phases, counts and candidates back)
    -- the path run_range takes.  The per-domain lists (failing ids,
    subdomain rows) are not brought back: fail_global / sub_table are None;
    the statistics (counts and arguments covered per phase) come from the
    device.  The phase-1 row's wall_ms is the device time of all three
    phases (the call does not split it)."""
    from .device import run_slice_host, run_slice_resident

    fmt = cfg.fmt
    args = (batch, ALGO_CODE[Algorithm(algo)], MODE_CODE[cfg.phase.div_mode], cfg.phase.phase2_split)
    r = batch.resident
    if r is not None and r.device.index != _current_cuda_device():
        r.wait()  # generated on another device: the host-buffer path below
        batch.resident = r = None
    if r is not None:
        # generated on the device (pack_plan(resident=True)): search the
        # columns where they are; their host copies land meanwhile
        try:
            res = run_slice_resident(*args)
        finally:
            r.wait()
            batch.resident = None
    else:
        res = run_slice_host(*args)
    n_fail, n_sub, n_cand, iters, a2, a3 = (int(x) for x in res.counts)
    if batch.shift_bound_ok is not None and not batch.shift_bound_ok.all():
        # the MPInt replay needs the failing ids: rare (narrow limb budgets)
        return execute_batch(batch, cfg, algo, fn, confirm, workers)
    id0 = batch.id0
    stats = PhaseStats()
    stats.rows.append(PhaseRow("phase1", batch.n_total, n_fail, batch.arguments, res.device_ms))
    stats.rows.append(PhaseRow("phase2", n_fail, n_sub, a2, 0.0))
    cand = RecordSet(fmt.precision, batch.binade, res.cand_index, res.cand_dist, res.cand_dom + np.uint64(id0))
    stats.rows.append(PhaseRow("phase3", n_sub, n_cand, a3, 0.0))
    t4 = time.perf_counter()
    records = confirm_set(fn or cfg.fn, cand, fmt, workers if workers is not None else cfg.phase.parallel_width) \
        if confirm else RecordSet(fmt.precision, batch.binade, [], [], [])
    stats.rows.append(PhaseRow("confirm", len(cand), len(records), len(cand), (time.perf_counter() - t4) * 1e3))
    return SliceOutput(batch, None, None, cand, records, stats, iters)


def _confirm_chunk(job) -> list:
    fn, fmt, cands = job
    guard = 2 * (fmt.precision + fmt.eps_bits) + 16
    out = []
    for c in cands:
        dec = decide_hr(fn, bits_float(c.argument, fmt), fmt, start_prec=guard)
        if dec.is_hr:
            out.append(HrCaseRecord(c.argument, UFrac.from_fraction(dec.distance_lo), c.domain_id))
    return out


CONFIRM_CHUNK = 64


def _confirm_native(fn: str, cand: list, fmt: FpFormat, workers: int):
    """hostgen.confirm on the candidates it covers; returns (records, rest)
    where rest are the candidates for the exact Python path."""
    from . import hostgen
    from .fpformat import EXP_BIAS

    p = fmt.precision
    if fn not in hostgen.FN_CODES or not cand:
        return [], cand
    e = {c.argument >> (p - 1) for c in cand}
    if len(e) != 1:
        return [], cand
    binade = e.pop() - EXP_BIAS - 1
    if binade > 0:
        return [], cand
    pg = PolyGenConfig(delta=2)  # only precision / eps / binade matter to the confirmation
    cfg = hostgen.make_cfg(fn, fmt, pg, binade, 64)
    idx = np.array([c.argument & ((1 << (p - 1)) - 1) for c in cand], dtype=np.uint64)
    is_hr, dist, status = hostgen.confirm(cfg, idx, workers)
    records, rest = [], []
    for c, h, d, st in zip(cand, is_hr.tolist(), dist.tolist(), status.tolist()):
        if st != hostgen.HRBH_OK:
            rest.append(c)
        elif h:
            records.append(HrCaseRecord(c.argument, UFrac(int(d), 64), c.domain_id))
    return records, rest


DEVICE_CONFIRM_MIN = 4096  # candidates from which the device confirmation pays for its copies


def _current_cuda_device():
    """The calling thread's CUDA device index, or None without CUDA."""
    try:
        import torch

        return torch.cuda.current_device() if torch.cuda.is_available() else None
    except Exception:  # pragma: no cover
        return None


def _cuda_ready() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def confirm_on_device(fmt: FpFormat, binade: int, index: np.ndarray):
    """hrb_confirm_exp over host arrays: (is_hr, dist_raw, status), the
    device running the same exact decide_hr restatement as the host
    library (csrc/host/decide.h)."""
    import ctypes as C

    torch = nat.require_cuda()
    lib = nat.load()
    n = len(index)
    dev = torch.device("cuda", torch.cuda.current_device())
    idx = torch.from_numpy(np.ascontiguousarray(index, dtype=np.uint64).view(np.int64)).to(dev)
    is_hr = torch.empty(n, dtype=torch.uint8, device=dev)
    st = torch.empty(n, dtype=torch.uint8, device=dev)
    dist = torch.empty(n, dtype=torch.int64, device=dev)
    nat.check("hrb_confirm_exp", lib.hrb_confirm_exp(fmt.precision, fmt.eps_bits, binade, n, idx.data_ptr(),
                                                     is_hr.data_ptr(), dist.data_ptr(), st.data_ptr(),
                                                     nat.stream_ptr()))
    return (is_hr.cpu().numpy(), dist.cpu().numpy().view(np.uint64).copy(), st.cpu().numpy())


def confirm_set(fn: str, cand: RecordSet, fmt: FpFormat, workers: int = 1) -> RecordSet:
    """confirm_candidates on a RecordSet of candidates, staying in arrays:
    the native decide_hr (hostgen) runs on the index column and only the
    candidates it hands back (and functions it does not cover) go through
    the Python decide_hr.  Same records, sorted."""
    from . import hostgen

    p, binade = fmt.precision, cand.binade
    if fn in hostgen.FN_CODES and binade <= 0 and len(cand):
        if len(cand) >= DEVICE_CONFIRM_MIN and _cuda_ready():
            is_hr, dist, status = confirm_on_device(fmt, binade, cand.index)
            if status.any():  # whatever the device left goes to the host library
                rest = np.flatnonzero(status != 0)
                cfg = hostgen.make_cfg(fn, fmt, PolyGenConfig(delta=2), binade, 64)
                h_is, h_d, h_st = hostgen.confirm(cfg, cand.index[rest], workers)
                is_hr[rest], dist[rest], status[rest] = h_is, h_d, h_st
        else:
            cfg = hostgen.make_cfg(fn, fmt, PolyGenConfig(delta=2), binade, 64)
            is_hr, dist, status = hostgen.confirm(cfg, cand.index, workers)
        ok = status == hostgen.HRBH_OK
        keep = ok & (is_hr != 0)
        recs = RecordSet(p, binade, cand.index[keep], dist[keep], cand.dom[keep])
        if ok.all():
            return recs
        rest = [cand[int(k)] for k in np.flatnonzero(~ok)]
        more = confirm_candidates(fn, rest, fmt, workers, native=False)
        return recs.merged(RecordSet.of(more, p, binade))
    return RecordSet.of(confirm_candidates(fn, list(cand), fmt, workers), p, binade)


def confirm_candidates(fn: str, cand: Sequence[HrCaseRecord], fmt: FpFormat, workers: int = 1,
                       native: bool | None = None) -> list:
    """Rigorous confirmation of phase-3 candidates (pipeline.py:447-462):
    decide_hr at rising precision per candidate, records sorted.  exp on
    binades <= 0 runs natively (hostgen, bit-identical decisions and
    distances) over `workers` threads; everything else -- and any candidate
    the native path hands back -- runs the Python decide_hr, spread over
    host processes when workers > 1 (the result is sorted, so
    order-independent)."""
    cand = list(cand)
    native_recs = []
    if native is not False:
        native_recs, cand = _confirm_native(fn, cand, fmt, workers)
    if workers > 1 and len(cand) > 2 * CONFIRM_CHUNK:
        import multiprocessing as mp

        jobs = [(fn, fmt, cand[k:k + CONFIRM_CHUNK]) for k in range(0, len(cand), CONFIRM_CHUNK)]
        with mp.get_context("fork").Pool(workers) as pool:
            records = [r for part in pool.map(_confirm_chunk, jobs) for r in part]
    else:
        records = _confirm_chunk((fn, fmt, cand))
    records.extend(native_recs)
    records.sort()
    return records


def prepare_slice(fn: str, binade: int, start: int, count: int, cfg: PipelineConfig, workers: int | None = None,
                  id0: int = 0, native: bool | None = None) -> SliceBatch:
    """Host half: Taylor blocks of the range, packed and checked (natively
    where hostgen covers the configuration, else the exact Python path)."""
    from .slices import pack_plan, plan_arrays

    w = workers if workers is not None else cfg.phase.parallel_width
    ceiling = cfg.phase.budgets.eps_dprime if cfg.phase.budgets is not None else None
    plan = plan_arrays(fn, binade, cfg.fmt, cfg.polygen, start, count, id0)
    return pack_plan(plan, cfg.word_bits, budget_ceiling=ceiling, workers=w, native=native)


def run_slice(fn: str, binade: int, start: int, count: int, cfg: PipelineConfig, algo: str | None = None,
              workers: int | None = None) -> SliceOutput:
    """The funnel over argument indices [start, start+count) of one binade."""
    batch = prepare_slice(fn, binade, start, count, cfg, workers)
    return execute_batch(batch, cfg, _resolve(cfg, algo), fn, workers=workers)


def run_pipeline(binade: int, cfg: PipelineConfig, prev_stats: PhaseStats | None = None):
    """Full funnel over one binade -> (records ascending, PhaseStats)."""
    algo = cfg.phase.algorithm
    if algo == "auto":
        algo = select_algorithm(prev_stats)
    out = run_slice(cfg.fn, binade, 0, 1 << (cfg.fmt.precision - 1), cfg, algo)
    out.stats.algorithm_choices.append((binade, algo))
    return list(out.records), out.stats


@dataclass
class RangeOutput:
    """run_range's result: records of the whole range (ascending) and one
    PhaseStats per interval, with the algorithm each interval used."""

    records: object   # RecordSet (a Sequence of HrCaseRecord), ascending
    interval_stats: list
    choices: list  # (first argument index, algorithm) per interval


# ------------------------------------------------ resumable range manifest
#
# A JSON-lines file: a header naming the run (a hash of everything that
# determines its results), then one line per finished interval with its
# records, phase stats and algorithm.  run_range(manifest=path) appends a line
# (flushed and fsynced) after every interval and, when the file already
# exists, restores the finished intervals instead of recomputing them: a long
# range resumes at interval granularity after a crash (SURVEY.md 2,
# checkpoint / resume).  A line torn by a crash is ignored.


MANIFEST_VERSION = 2  # bump when the interval-line format or the results of a config change


def manifest_key(fn: str, binade: int, start: int, count: int, cfg: PipelineConfig, interval_args: int,
                 confirm: bool = True, wide=None) -> str:
    """Hash of everything that determines a run's results.  The host worker
    count (PhaseConfig.parallel_width) does not change results, so it is
    normalised out: a run may resume on a machine with other core counts."""
    import dataclasses
    import hashlib

    norm = dataclasses.replace(cfg, phase=dataclasses.replace(cfg.phase, parallel_width=1))
    ident = (MANIFEST_VERSION, fn, binade, start, count, norm, interval_args, confirm) + ((wide,) if wide else ())
    return hashlib.sha256(repr(ident).encode()).hexdigest()[:32]


def interval_line(k: int, bstart: int, algo: str, records, stats: PhaseStats) -> str:
    import json

    return json.dumps({"kind": "interval", "k": k, "bstart": bstart, "algo": algo,
                       "records": [[hex(r.argument), r.distance.raw, r.distance.width, r.domain_id, r.undecided]
                                   for r in records],
                       "rows": [[r.phase, r.domains_in, r.domains_out, r.arguments_covered, r.wall_ms]
                                for r in stats.rows],
                       "choices": [list(c) for c in stats.algorithm_choices]})


def _manifest_has_header(path: str) -> bool:
    import json
    import os

    if not os.path.exists(path):
        return False
    with open(path) as fh:
        for line in fh:
            try:
                return json.loads(line).get("kind") == "header"
            except ValueError:
                return False  # the header itself was torn by a crash
    return False


def read_manifest(path: str, key: str) -> dict:
    """Finished intervals of a manifest: {k: (bstart, algo, records, stats)}.
    Raises ValueError when the file belongs to a different run.  A file
    without a valid header (a crash tore it) holds no finished interval."""
    import json
    import os

    done = {}
    if not os.path.exists(path) or not _manifest_has_header(path):
        return done
    with open(path) as fh:
        lines = fh.read().splitlines()
    header = False
    for line in lines:
        try:
            d = json.loads(line)
        except ValueError:
            continue  # a line torn by a crash
        if d.get("kind") == "header":
            if d.get("key") != key:
                raise ValueError(f"manifest {path} belongs to another run (key {d.get('key')} != {key})")
            header = True
            continue
        if not header:
            raise ValueError(f"manifest {path} has no header")
        recs = [HrCaseRecord(int(a, 16), UFrac(raw, width), dom, bool(und)) for a, raw, width, dom, und in d["records"]]
        st = PhaseStats([PhaseRow(*r) for r in d["rows"]], [tuple(c) for c in d["choices"]])
        done[int(d["k"])] = (int(d["bstart"]), d["algo"], recs, st)
    return done


def execute_wide(batch, cfg: PipelineConfig, algo: str, fn: str | None = None, confirm: bool = True,
                 workers: int | None = None) -> SliceOutput:
    """A high-degree slice (wide.WideSliceBatch) through ONE host-buffer ABI
    call (hrb_wrun_slice_host), then the rigorous confirmation; statistics
    as execute_batch_host.  The wide kernels run the regular family."""
    from .wide import run_wide_host

    if algo not in ("regular", "regular_unrolled"):
        raise ValueError("high-degree slices run the regular search family")
    res = run_wide_host(batch, ALGO_CODE[Algorithm(algo)], cfg.phase.phase2_split)
    n_fail, n_sub, n_cand, iters, a2, a3 = (int(x) for x in res.counts)
    stats = PhaseStats()
    stats.rows.append(PhaseRow("phase1", batch.n_total, n_fail, batch.arguments, res.device_ms))
    stats.rows.append(PhaseRow("phase2", n_fail, n_sub, a2, 0.0))
    cand = RecordSet(cfg.fmt.precision, batch.binade, res.cand_index, res.cand_dist,
                     res.cand_dom + np.uint64(batch.id0))
    stats.rows.append(PhaseRow("phase3", n_sub, n_cand, a3, 0.0))
    t4 = time.perf_counter()
    records = confirm_set(fn or cfg.fn, cand, cfg.fmt, workers if workers is not None else
                          cfg.phase.parallel_width) if confirm else RecordSet(cfg.fmt.precision, batch.binade, [],
                                                                              [], [])
    stats.rows.append(PhaseRow("confirm", len(cand), len(records), len(cand), (time.perf_counter() - t4) * 1e3))
    return SliceOutput(batch, None, None, cand, records, stats, iters)


def run_range(fn: str, binade: int, start: int, count: int, cfg: PipelineConfig, interval_args: int = 1 << 36,
              workers: int | None = None, confirm: bool = True, manifest: str | None = None,
              native: bool | None = None, wide=None) -> RangeOutput:
    """A long argument range as consecutive intervals, the way the paper walks
    a binade: the block schedule of the WHOLE range is
    planned once (so blocks, domain ids and results are exactly those of a
    single run_slice), cut into intervals of about `interval_args`
    arguments, and with algorithm "auto" each interval's search family is
    chosen from the previous interval's funnel (select_algorithm,
    pipeline.py:187-197).  The host Taylor generation of interval i+1 runs in
    a background thread while the device and the host confirmation work on
    interval i.  manifest: a path that makes the run resumable (see
    read_manifest); finished intervals are restored, not recomputed.
    wide: a wide.WideGenConfig switches to the high-degree path (delta_R
    3..8, one Taylor model per large super-domain; the regular family; an
    extension of the reference, see wide.py) -- same records."""
    import contextlib
    from concurrent.futures import Future, ThreadPoolExecutor

    from .shard import partition_blocks
    from .slices import pack_plan, plan_arrays

    w = workers if workers is not None else cfg.phase.parallel_width
    if wide is not None:
        from .wide import pack_wide, plan_wide

        if cfg.phase.algorithm == "lefevre":
            raise ValueError("high-degree slices run the regular search family")
        plan = plan_wide(fn, binade, cfg.fmt, wide, start, count)
    else:
        plan = plan_arrays(fn, binade, cfg.fmt, cfg.polygen, start, count)
    sizes = plan.sizes
    n_int = max(1, -(-int(sizes.sum()) // max(1, interval_args)))
    parts = [p for p in partition_blocks(sizes, n_int) if p[1] > p[0]]
    ceiling = cfg.phase.budgets.eps_dprime if cfg.phase.budgets is not None else None
    bstart_of = [int(plan.bstart[p[0]]) for p in parts]

    # the generation runs in a worker thread: give it the caller's CUDA device
    # (a new thread starts on device 0, which under torchrun is another
    # rank's GPU)
    dev = _current_cuda_device()

    def prepare(part):
        if dev is not None:
            import torch

            torch.cuda.set_device(dev)
        if wide is not None:
            return pack_wide(plan[part[0]:part[1]], wide, w)
        return pack_plan(plan[part[0]:part[1]], cfg.word_bits, budget_ceiling=ceiling, workers=w, native=native,
                         resident=True)

    done, sink = {}, None
    if manifest is not None:
        import json
        import os

        key = manifest_key(fn, binade, start, count, cfg, interval_args, confirm, wide)
        done = read_manifest(manifest, key)
        # no valid header (absent, empty, or torn by a crash before its
        # newline was durable): start the file over
        fresh = not _manifest_has_header(manifest)
        torn = False
        if not fresh:
            with open(manifest, "rb") as fh:
                fh.seek(-1, os.SEEK_END)
                torn = fh.read(1) != b"\n"
        sink = open(manifest, "w" if fresh else "a")
        if torn:
            sink.write("\n")  # end a line torn by a crash; read_manifest skips it
        if fresh:
            sink.write(json.dumps({"kind": "header", "key": key, "version": MANIFEST_VERSION, "fn": fn,
                                   "binade": binade, "start": start, "count": count,
                                   "intervals": len(parts)}) + "\n")
            sink.flush()
            os.fsync(sink.fileno())
    todo = [k for k in range(len(parts)) if k not in done]
    records, stats_list, choices = [], [], []
    prev = None
    try:
        # the first interval is prepared inline (nothing to overlap it with);
        # a worker thread only exists when there is a next interval to prepare
        # behind the current one (a thread's start and join cost milliseconds
        # against a one-interval range's few)
        with ThreadPoolExecutor(max_workers=1) if len(todo) > 1 else contextlib.nullcontext() as ex:
            futs = {todo[0]: prepare(parts[todo[0]])} if todo else {}
            for k, part in enumerate(parts):
                if k in done:  # restored from the manifest
                    bstart, algo, recs, st = done[k]
                    records.append(recs)
                    stats_list.append(st)
                    choices.append((bstart, algo))
                    prev = st
                    continue
                batch = futs.pop(k)
                if isinstance(batch, Future):
                    batch = batch.result()
                i = todo.index(k)
                if i + 1 < len(todo):
                    futs[todo[i + 1]] = ex.submit(prepare, parts[todo[i + 1]])
                algo = cfg.phase.algorithm
                if algo == "auto":
                    algo = select_algorithm(prev) if wide is None else "regular"
                if wide is not None:
                    out = execute_wide(batch, cfg, algo, fn, confirm=confirm, workers=w)
                else:
                    out = execute_batch_host(batch, cfg, algo, fn, confirm=confirm, workers=w)
                out.stats.algorithm_choices.append((bstart_of[k], algo))
                records.append(out.records)
                stats_list.append(out.stats)
                choices.append((bstart_of[k], algo))
                prev = out.stats
                if sink is not None:
                    sink.write(interval_line(k, bstart_of[k], algo, out.records, out.stats) + "\n")
                    sink.flush()
                    os.fsync(sink.fileno())
    finally:
        if sink is not None:
            sink.close()
    return RangeOutput(RecordSet.concat(records, cfg.fmt.precision, binade).sorted(), stats_list, choices)


# --------------------------------------------------- per-phase drop-ins


def _task_slice(items, cfg: PipelineConfig, binade: int) -> SliceBatch:
    """Pack explicit (coeffs, count, eps', index) items as one-domain
    super-domains: r_0 = (s0, 0, 0), r_1 = (s1, 0), r_2 = (s2,).  A missing
    s2 (delta = 1) packs as 0, which is exactly the reference's
    len(coeffs) < 3 truncation rule (pipeline.py:144-145)."""
    supers = []
    for k, (coeffs, count, eps_prime, index) in enumerate(items):
        c = [as_int(x) for x in coeffs] + [0] * (3 - len(coeffs))
        rp = (BinomialPoly((c[0], 0, 0)), BinomialPoly((c[1], 0)), BinomialPoly((c[2],)))
        supers.append(SuperDomain(index, count, count, 1, 1, 1, 0, k, rp, eps_prime))
    pg = cfg.polygen
    one = PolyGenConfig(tau=1, N=1, mu=1, nu=1, delta=2, limbs=pg.limbs, frac_bits=pg.frac_bits, guard=pg.guard)
    ceiling = cfg.phase.budgets.eps_dprime if cfg.phase.budgets is not None else None
    return pack_slice(supers, cfg.fmt, one, cfg.word_bits, binade, budget_ceiling=ceiling)


def _binade_of(dom: Domain, fmt: FpFormat) -> int:
    return dom.exponent - 1


def phase1(tasks: Sequence[DomainTask], cfg: PipelineConfig, algo: str | None = None) -> list[int]:
    """Failing domain ids of explicit DomainTasks (one device launch)."""
    tasks = list(tasks)
    if not tasks:
        return []
    from .device import DeviceSlice, run_phases

    m_base = 1 << (cfg.fmt.precision - 1)
    batch = _task_slice([(t.coeffs, t.domain.count, t.eps_prime, t.domain.m_start - m_base) for t in tasks], cfg,
                        _binade_of(tasks[0].domain, cfg.fmt))
    res = _phase1_only(batch, cfg, _resolve(cfg, algo))
    return [tasks[int(i)].domain.domain_id for i in res]


def _phase1_only(batch: SliceBatch, cfg: PipelineConfig, algo: str) -> np.ndarray:
    import ctypes as C

    from .device import DeviceSlice

    ds = DeviceSlice(batch)
    lib = nat.load()
    fail = ds.empty64(batch.n_total)
    cnt = ds.empty64(4)
    cnt.zero_()
    nat.check("hrb_phase1", lib.hrb_phase1(C.byref(ds.desc), ALGO_CODE[Algorithm(algo)], MODE_CODE[cfg.phase.div_mode],
                                           fail.data_ptr(), cnt.data_ptr(), batch.n_total, None, nat.stream_ptr()))
    n = int(cnt[0].item())
    return fail[:n].cpu().numpy().view(np.uint64)


def phase2(tasks: Sequence[DomainTask], cfg: PipelineConfig, algo: str | None = None) -> list[SubdomainTask]:
    """Split each task s ways, shift, re-test; survivors in task order."""
    tasks = list(tasks)
    if not tasks:
        return []
    import ctypes as C

    from .device import DeviceSlice

    m_base = 1 << (cfg.fmt.precision - 1)
    batch = _task_slice([(t.coeffs, t.domain.count, t.eps_prime, t.domain.m_start - m_base) for t in tasks], cfg,
                        _binade_of(tasks[0].domain, cfg.fmt))
    split = cfg.phase.phase2_split
    ds = DeviceSlice(batch)
    lib = nat.load()
    torch = ds.torch
    ids = torch.arange(len(tasks), dtype=torch.int64, device=ds.device)
    cnt = ds.empty64(4)
    cnt.zero_()
    cnt[0] = len(tasks)
    cap = len(tasks) * 2 * split
    subs = ds.empty64(cap)
    nat.check("hrb_phase2", lib.hrb_phase2(C.byref(ds.desc), ALGO_CODE[Algorithm(_resolve(cfg, algo))],
                                           MODE_CODE[cfg.phase.div_mode], split, ids.data_ptr(), cnt.data_ptr(),
                                           len(tasks), subs.data_ptr(), cnt[1:].data_ptr(), cap, nat.stream_ptr()))
    n = int(cnt[1].item())
    keys = subs[:n].cpu().numpy().view(np.uint64)
    out = []
    for key in keys.tolist():
        t, j = key >> 8, key & 255
        task = tasks[t]
        n_t = task.domain.count
        step = max(n_t // split, 1)
        start = j * step
        cnt_j = min(step, n_t - start)
        poly = BinomialPoly(tuple(task.coeffs), task.frac_bits)
        out.append(SubdomainTask(task, j, start, cnt_j, straightforward_shift(poly, start).coeffs))
    return out


def phase3_exhaustive(tasks: Sequence[SubdomainTask], cfg: PipelineConfig) -> list[HrCaseRecord]:
    """Window test of every argument of the subdomains (device walk)."""
    tasks = list(tasks)
    if not tasks:
        return []
    import ctypes as C

    from .device import DeviceSlice

    fmt = cfg.fmt
    m_base = 1 << (fmt.precision - 1)
    binade = _binade_of(tasks[0].parent.domain, fmt)
    batch = _task_slice([(s.coeffs, s.count, s.parent.eps_prime, s.parent.domain.m_start - m_base + s.start)
                         for s in tasks], cfg, binade)
    ds = DeviceSlice(batch)
    lib = nat.load()
    torch = ds.torch
    keys = torch.arange(len(tasks), dtype=torch.int64, device=ds.device) << 8
    cnt = ds.empty64(4)
    cnt.zero_()
    cnt[1] = len(tasks)
    cap = 1 << 12
    while True:
        cm, cd, cdom = ds.empty64(cap), ds.empty64(cap), ds.empty64(cap)
        nat.check("hrb_phase3", lib.hrb_phase3(C.byref(ds.desc), 1, keys.data_ptr(), cnt[1:].data_ptr(), len(tasks),
                                               cm.data_ptr(), cd.data_ptr(), cdom.data_ptr(), cnt[2:].data_ptr(), cap,
                                               nat.stream_ptr()))
        n = int(cnt[2].item())
        if n <= cap:
            break
        cap = n
    m = cm[:n].cpu().numpy().view(np.uint64).tolist()
    d = cd[:n].cpu().numpy().view(np.uint64).tolist()
    dom = cdom[:n].cpu().numpy().view(np.uint64).tolist()
    return [HrCaseRecord(index_bits(binade, mi, fmt), UFrac(di, 64), tasks[ti].parent.domain.domain_id)
            for mi, di, ti in zip(m, d, dom)]
