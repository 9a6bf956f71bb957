"""Device-side execution of a packed slice through libhrb200 (C-ABI).

torch supplies device memory and the stream; every computation is a call
into include/hrb200.h.  There is no CPU fallback (see _native.require_cuda).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .slices import SliceBatch


def _t(torch, arr: np.ndarray, device):
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device, non_blocking=False)


class DeviceSlice:
    """A SliceBatch resident in HBM plus its hrb_slice descriptor."""

    def __init__(self, batch: SliceBatch, device=None):
        torch = nat.require_cuda()
        self.torch = torch
        self.batch = batch
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        u32 = lambda a: _t(torch, a.view(np.int32), self.device)  # noqa: E731  (torch lacks uint32 ops)
        u64 = lambda a: _t(torch, a.view(np.int64), self.device)  # noqa: E731
        self.coef = u32(batch.coef)
        self.G = u64(batch.G)
        self.s2abs = u64(batch.s2abs)
        self.n_dom = u32(batch.n_dom)
        self.dom_n = u32(batch.dom_n)
        self.last_n = u32(batch.last_n)
        self.dom_base = u64(batch.dom_base)
        self.m0 = u64(batch.m0)
        self.desc = nat.HrbSlice(
            n_super=batch.n_super, n_total=batch.n_total, max_dom_n=batch.max_dom_n,
            coef_limbs=batch.coef_limbs, frac_bits=batch.frac_bits, word_bits=batch.word_bits, delta=batch.delta,
            coef=self.coef.data_ptr(), G=self.G.data_ptr(), s2abs=self.s2abs.data_ptr(),
            n_dom=self.n_dom.data_ptr(), dom_n=self.dom_n.data_ptr(), last_n=self.last_n.data_ptr(),
            dom_base=self.dom_base.data_ptr(), m0=self.m0.data_ptr())

    def empty64(self, n: int):
        return self.torch.empty(max(int(n), 1), dtype=self.torch.int64, device=self.device)


@dataclass
class SliceResult:
    """Device outputs of one slice, on the host (slice-local ids)."""

    fail_ids: np.ndarray      # uint64, ascending
    sub_keys: np.ndarray      # uint64 (local id << 8 | j), ascending
    cand_index: np.ndarray    # uint64 binade argument index, ascending
    cand_dist: np.ndarray     # uint64 distance floored to 2^-64
    cand_dom: np.ndarray      # uint64 slice-local domain id
    iterations: int           # phase-1 SearchOutcome.iterations sum
    phase_ms: tuple = (0.0, 0.0, 0.0)


def _u64(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def run_phases(ds: DeviceSlice, algo_code: int, mode_code: int, split: int, cand_hint: int = 4096,
               timed: bool = True) -> SliceResult:
    """Phase 1, 2, 3 as separate ABI calls with the counts read back between
    them (sizes the next phase's buffers; wall times per phase like the
    reference's PhaseRow)."""
    torch = ds.torch
    lib = nat.load()
    b = ds.batch
    st = nat.stream_ptr()
    stream = torch.cuda.current_stream()
    n_total = b.n_total
    cnt = ds.empty64(4)
    cnt.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    # phase 1
    fail = ds.empty64(n_total)
    ev[0].record(stream)
    nat.check("hrb_phase1", lib.hrb_phase1(C.byref(ds.desc), algo_code, mode_code, fail.data_ptr(),
                                           cnt.data_ptr(), n_total, cnt[3:].data_ptr(), st))
    ev[1].record(stream)
    n_fail = int(cnt[0].item())
    # phase 2
    jmax = 2 * split
    sub_cap = max(n_fail * jmax, 1)
    subs = ds.empty64(sub_cap)
    nat.check("hrb_phase2", lib.hrb_phase2(C.byref(ds.desc), algo_code, mode_code, split, fail.data_ptr(),
                                           cnt[0:].data_ptr(), n_total, subs.data_ptr(), cnt[1:].data_ptr(),
                                           sub_cap, st))
    ev[2].record(stream)
    n_sub = int(cnt[1].item())
    # phase 3 (grow the candidate buffer once if the hint was too small)
    cap = max(cand_hint, 1)
    while True:
        cm, cdist, cdom = ds.empty64(cap), ds.empty64(cap), ds.empty64(cap)
        nat.check("hrb_phase3", lib.hrb_phase3(C.byref(ds.desc), split, subs.data_ptr(), cnt[1:].data_ptr(),
                                               sub_cap, cm.data_ptr(), cdist.data_ptr(), cdom.data_ptr(),
                                               cnt[2:].data_ptr(), cap, st))
        n_c = int(cnt[2].item())
        if n_c <= cap:
            break
        cap = n_c
    ev[3].record(stream)
    torch.cuda.synchronize()
    ms = tuple(ev[k].elapsed_time(ev[k + 1]) for k in range(3)) if timed else (0.0, 0.0, 0.0)
    return SliceResult(_u64(fail[:n_fail]), _u64(subs[:n_sub]), _u64(cm[:n_c]), _u64(cdist[:n_c]),
                       _u64(cdom[:n_c]), int(cnt[3].item()), ms)


class FusedRunner:
    """hrb_run_slice with persistent device buffers: the bench hot path
    (inputs resident in HBM, no host synchronisation inside a step)."""

    def __init__(self, ds: DeviceSlice, algo_code: int, mode_code: int, split: int, sub_cap: int,
                 cand_cap: int):
        self.ds = ds
        self.algo, self.mode, self.split = algo_code, mode_code, split
        n_total = ds.batch.n_total
        self.fail = ds.empty64(n_total)
        self.subs = ds.empty64(sub_cap)
        self.cm, self.cd, self.cdom = ds.empty64(cand_cap), ds.empty64(cand_cap), ds.empty64(cand_cap)
        self.counts = ds.empty64(4)
        self.out = nat.HrbRunOut(fail_ids=self.fail.data_ptr(), fail_cap=n_total, sub_keys=self.subs.data_ptr(),
                                 sub_cap=sub_cap, cand_index=self.cm.data_ptr(), cand_dist=self.cd.data_ptr(),
                                 cand_dom=self.cdom.data_ptr(), cand_cap=cand_cap, counts=self.counts.data_ptr())
        self.sub_cap, self.cand_cap = sub_cap, cand_cap

    def launch(self, stream=None) -> None:
        lib = nat.load()
        nat.check("hrb_run_slice", lib.hrb_run_slice(C.byref(self.ds.desc), self.algo, self.mode, self.split,
                                                     C.byref(self.out), nat.stream_ptr(stream)))

    def counts_host(self) -> np.ndarray:
        return self.counts.cpu().numpy().view(np.uint64)

    def result(self) -> SliceResult:
        c = self.counts_host()
        if c[1] > self.sub_cap or c[2] > self.cand_cap:
            raise nat.NativeError("hrb_run_slice", nat.HRB_ERR_CAPACITY, f"counts {c.tolist()} exceed capacity")
        nf, ns, nc = int(c[0]), int(c[1]), int(c[2])
        return SliceResult(_u64(self.fail[:nf]), _u64(self.subs[:ns]), _u64(self.cm[:nc]), _u64(self.cd[:nc]),
                           _u64(self.cdom[:nc]), int(c[3]))


def run_host(batch: SliceBatch, algo_code: int, mode_code: int, split: int, cand_cap: int = 1 << 16,
             with_fail_ids: bool = True):
    """hrb_run_slice_host straight from the packed (pageable) host arrays:
    streamed upload, phases 1-3, counts and candidates back (the e2e path).
    Returns (counts[6], fail_ids, cand_index, cand_dist, cand_dom,
    device_ms); with_fail_ids=False leaves the failing-domain list on the
    device (fail_cap 0) and returns an empty array for it."""
    nat.require_cuda()
    lib = nat.load()
    arrs = [np.ascontiguousarray(a) for a in (batch.coef, batch.G, batch.s2abs, batch.n_dom, batch.dom_n,
                                               batch.last_n, batch.dom_base, batch.m0)]
    p = [a.ctypes.data for a in arrs]
    desc = nat.HrbSlice(n_super=batch.n_super, n_total=batch.n_total, max_dom_n=batch.max_dom_n,
                        coef_limbs=batch.coef_limbs, frac_bits=batch.frac_bits, word_bits=batch.word_bits,
                        delta=batch.delta, coef=p[0], G=p[1], s2abs=p[2], n_dom=p[3], dom_n=p[4], last_n=p[5],
                        dom_base=p[6], m0=p[7])
    counts = np.zeros(6, dtype=np.uint64)
    fail = np.zeros(max(batch.n_total, 1) if with_fail_ids else 1, dtype=np.uint64)
    while True:
        cm = np.zeros(max(cand_cap, 1), dtype=np.uint64)
        cd = np.zeros(max(cand_cap, 1), dtype=np.uint64)
        cdom = np.zeros(max(cand_cap, 1), dtype=np.uint64)
        ms = C.c_float(0)
        rc = lib.hrb_run_slice_host(C.byref(desc), algo_code, mode_code, split, counts.ctypes.data,
                                    fail.ctypes.data if with_fail_ids else None, fail.size if with_fail_ids else 0,
                                    cm.ctypes.data, cd.ctypes.data, cdom.ctypes.data, cand_cap, C.byref(ms))
        if rc == nat.HRB_ERR_CAPACITY and counts[2] > cand_cap:
            cand_cap = int(counts[2])
            continue
        nat.check("hrb_run_slice_host", rc)
        break
    nf, nc = (int(counts[0]) if with_fail_ids else 0), int(counts[2])
    return counts, fail[:nf], cm[:nc], cd[:nc], cdom[:nc], ms.value


class HostRunner:
    """hrb_run_slice_host with page-locked host buffers allocated once: the
    slice inputs are copied into pinned memory at construction, outputs land
    in pinned arrays.  Each run() is one C-ABI call (H2D of the slice, all
    kernels, D2H of counts + failing ids + candidates, synchronised)."""

    INPUTS = ("coef", "G", "s2abs", "n_dom", "dom_n", "last_n", "dom_base", "m0")

    def __init__(self, batch: SliceBatch, algo_code: int, mode_code: int, split: int, cand_cap: int = 1 << 16):
        torch = nat.require_cuda()
        self.lib = nat.load()
        self.batch, self.algo, self.mode, self.split = batch, algo_code, mode_code, split

        def pinned(shape, dtype):
            n = int(np.prod(shape)) * np.dtype(dtype).itemsize
            t = torch.empty(max(n, 8), dtype=torch.uint8).pin_memory()
            self._keep.append(t)
            return t.numpy()[:n].view(dtype).reshape(shape)

        self._keep = []
        self.inputs = {}
        for name in self.INPUTS:
            src = np.ascontiguousarray(getattr(batch, name))
            dst = pinned(src.shape, src.dtype)
            dst[...] = src
            self.inputs[name] = dst
        p = {k: v.ctypes.data for k, v in self.inputs.items()}
        self.desc = nat.HrbSlice(n_super=batch.n_super, n_total=batch.n_total, max_dom_n=batch.max_dom_n,
                                 coef_limbs=batch.coef_limbs, frac_bits=batch.frac_bits, word_bits=batch.word_bits,
                                 delta=batch.delta, coef=p["coef"], G=p["G"], s2abs=p["s2abs"], n_dom=p["n_dom"],
                                 dom_n=p["dom_n"], last_n=p["last_n"], dom_base=p["dom_base"], m0=p["m0"])
        self.counts = pinned((6,), np.uint64)
        self.fail = pinned((max(batch.n_total, 1),), np.uint64)
        self._alloc_cands(cand_cap)
        self.device_ms = C.c_float(0)

    def _alloc_cands(self, cap: int) -> None:
        import torch

        self.cand_cap = cap
        bufs = [torch.empty(cap * 8, dtype=torch.uint8).pin_memory() for _ in range(3)]
        self._cand_keep = bufs
        self.cm, self.cd, self.cdom = (b.numpy().view(np.uint64) for b in bufs)

    def input_bytes(self) -> int:
        """Bytes hrb_run_slice_host copies host -> device per call (coefficients
        travel as their low four limbs, the residues the phases read)."""
        cl = self.batch.coef_limbs
        coef = self.inputs["coef"].nbytes * min(cl, 4) // cl
        return coef + sum(v.nbytes for k, v in self.inputs.items() if k != "coef")

    def run(self):
        """One end-to-end call; returns (counts, fail_ids, cand_index,
        cand_dist, cand_dom) as views of the pinned buffers."""
        while True:
            rc = self.lib.hrb_run_slice_host(C.byref(self.desc), self.algo, self.mode, self.split,
                                             self.counts.ctypes.data, self.fail.ctypes.data, self.fail.size,
                                             self.cm.ctypes.data, self.cd.ctypes.data, self.cdom.ctypes.data,
                                             self.cand_cap, C.byref(self.device_ms))
            if rc == nat.HRB_ERR_CAPACITY and int(self.counts[2]) > self.cand_cap:
                self._alloc_cands(int(self.counts[2]))
                continue
            nat.check("hrb_run_slice_host", rc)
            break
        nf, nc = int(self.counts[0]), int(self.counts[2])
        return self.counts, self.fail[:nf], self.cm[:nc], self.cd[:nc], self.cdom[:nc]

    def output_bytes(self) -> int:
        """Bytes the last run() copied device -> host."""
        return 48 + 8 * int(self.counts[0]) + 24 * min(int(self.counts[2]), self.cand_cap)


@dataclass
class HostSliceResult:
    """hrb_run_slice_host outputs without the per-domain lists."""

    counts: np.ndarray        # uint64 [6]: fails, survivors, candidates, iterations, phase-2 args, phase-3 args
    cand_index: np.ndarray
    cand_dist: np.ndarray
    cand_dom: np.ndarray
    device_ms: float


def run_slice_host(batch: SliceBatch, algo_code: int, mode_code: int, split: int,
                   cand_cap: int = 1 << 16) -> HostSliceResult:
    """run_host without the failing-domain list: what the end-to-end path
    needs (counts, the arguments each phase covered, the candidates)."""
    counts, _, cm, cd, cdom, ms = run_host(batch, algo_code, mode_code, split, cand_cap, with_fail_ids=False)
    return HostSliceResult(counts, cm, cd, cdom, ms)


def run_slice_resident(batch: SliceBatch, algo_code: int, mode_code: int, split: int,
                       cand_cap: int = 1 << 16) -> HostSliceResult:
    """run_slice_host for a batch whose generated columns are still on the
    device (batch.resident, pack_plan's device generation inside run_range):
    the size columns are uploaded, the columns are not -- one
    hrb_run_slice_resident call on the current stream."""
    torch = nat.require_cuda()
    lib = nat.load()
    r = batch.resident
    # the size columns: uploaded by pack_plan while the generation ran, else now
    keep = r.extra if r.extra is not None else upload_columns(
        torch, [batch.n_dom, batch.dom_n, batch.last_n, batch.dom_base, batch.m0], r.device)
    desc = nat.HrbSlice(n_super=batch.n_super, n_total=batch.n_total, max_dom_n=batch.max_dom_n,
                        coef_limbs=r.coef.shape[1], frac_bits=batch.frac_bits, word_bits=batch.word_bits,
                        delta=batch.delta, coef=r.coef.data_ptr(), G=r.G.data_ptr(), s2abs=r.s2abs.data_ptr(),
                        n_dom=keep[0].data_ptr(), dom_n=keep[1].data_ptr(), last_n=keep[2].data_ptr(),
                        dom_base=keep[3].data_ptr(), m0=keep[4].data_ptr())
    counts = np.zeros(6, dtype=np.uint64)
    while True:
        cm, cd, cdom = (np.zeros(max(cand_cap, 1), dtype=np.uint64) for _ in range(3))
        ms = C.c_float(0)
        rc = lib.hrb_run_slice_resident(C.byref(desc), algo_code, mode_code, split, counts.ctypes.data,
                                        cm.ctypes.data, cd.ctypes.data, cdom.ctypes.data, cand_cap, C.byref(ms),
                                        nat.stream_ptr())
        if rc == nat.HRB_ERR_CAPACITY and counts[2] > cand_cap:
            cand_cap = int(counts[2])
            continue
        nat.check("hrb_run_slice_resident", rc)
        break
    nc = int(counts[2])
    return HostSliceResult(counts, cm[:nc], cd[:nc], cdom[:nc], ms.value)


def domain_coefficients(ds: DeviceSlice) -> np.ndarray:
    """hrb_domain_coefficients -> uint32 [3, CL, n_total] (two's complement)."""
    torch = ds.torch
    lib = nat.load()
    b = ds.batch
    out = torch.empty(3 * b.coef_limbs * max(b.n_total, 1), dtype=torch.int32, device=ds.device)
    nat.check("hrb_domain_coefficients", lib.hrb_domain_coefficients(C.byref(ds.desc), out.data_ptr(),
                                                                     nat.stream_ptr()))
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32).reshape(3, b.coef_limbs, -1)[:, :, : b.n_total]


def search_batch_arrays(algo_code: int, mode_code: int, word_bits: int, a, b, eps, count, device=None):
    """hrb_search_batch over host arrays; returns host arrays
    (ok, d, iterations, points_lo, points_hi)."""
    torch = nat.require_cuda()
    lib = nat.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = len(a)
    ins = [torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.uint64)).view(np.int64)).to(dev)
           for x in (a, b, eps, count)]
    ok = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    d = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    it = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    pl = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    ph = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    nat.check("hrb_search_batch", lib.hrb_search_batch(algo_code, mode_code, word_bits, n, *(x.data_ptr() for x in ins),
                                                       ok.data_ptr(), d.data_ptr(), it.data_ptr(), pl.data_ptr(),
                                                       ph.data_ptr(), nat.stream_ptr()))
    torch.cuda.synchronize()
    return (ok[:n].cpu().numpy(), _u64(d[:n]), _u64(it[:n]), _u64(pl[:n]), ph[:n].cpu().numpy())


def search_trace_arrays(algo_code: int, mode_code: int, word_bits: int, a, b, eps, count, device=None):
    """hrb_search_trace over host arrays: the outcomes of search_batch_arrays
    plus every problem's branch-decision list (the reference cores' `trace`).
    Two passes: the first counts decisions, the second stores them."""
    torch = nat.require_cuda()
    lib = nat.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = len(a)
    ins = [torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.uint64)).view(np.int64)).to(dev)
           for x in (a, b, eps, count)]
    m = max(n, 1)
    ok = torch.empty(m, dtype=torch.uint8, device=dev)
    d, it, pl = (torch.empty(m, dtype=torch.int64, device=dev) for _ in range(3))
    ph = torch.empty(m, dtype=torch.uint8, device=dev)
    tlen = torch.zeros(m, dtype=torch.int32, device=dev)
    wpp = 1
    while True:
        words = torch.zeros(m * wpp, dtype=torch.int64, device=dev)
        nat.check("hrb_search_trace", lib.hrb_search_trace(algo_code, mode_code, word_bits, n,
                                                           *(x.data_ptr() for x in ins), ok.data_ptr(), d.data_ptr(),
                                                           it.data_ptr(), pl.data_ptr(), ph.data_ptr(),
                                                           words.data_ptr(), wpp, tlen.data_ptr(), nat.stream_ptr()))
        torch.cuda.synchronize()
        lens = tlen[:n].cpu().numpy().view(np.uint32).astype(np.int64)
        need = int((lens.max() + 63) // 64) if n else 1
        if need <= wpp:
            break
        wpp = need
    bits = np.unpackbits(words.cpu().numpy().view(np.uint8).reshape(m, wpp * 8), axis=1, bitorder="little")
    traces = [bits[i, : lens[i]].astype(bool).tolist() for i in range(n)]
    return (ok[:n].cpu().numpy(), _u64(d[:n]), _u64(it[:n]), _u64(pl[:n]), ph[:n].cpu().numpy(), traces)


def search_verdict_arrays(algo_code: int, word_bits: int, a, b, eps, count, device=None):
    """hrb_search_verdicts over host arrays (regular family): the lockstep
    throughput form; returns host arrays (ok, d, iterations)."""
    torch = nat.require_cuda()
    lib = nat.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = len(a)
    ins = [torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.uint64)).view(np.int64)).to(dev)
           for x in (a, b, eps, count)]
    ok = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    d = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    it = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    nat.check("hrb_search_verdicts", lib.hrb_search_verdicts(algo_code, word_bits, n, *(x.data_ptr() for x in ins),
                                                             ok.data_ptr(), d.data_ptr(), it.data_ptr(),
                                                             nat.stream_ptr()))
    torch.cuda.synchronize()
    return ok[:n].cpu().numpy(), _u64(d[:n]), _u64(it[:n])


PIN_GEN_MIN = 8192  # super-domains from which pack_columns_device downloads into pinned memory


class ResidentColumns:
    """The device copies of a slice's generated columns (hrb_pack_blocks'
    coef, G, s2abs) kept for hrb_run_slice_resident, while their download to
    the host arrays of the same SliceBatch runs on a side stream: the host
    arrays are valid only after wait()."""

    def __init__(self, coef, G, s2abs, done, device, extra=None):
        self.coef, self.G, self.s2abs, self.done, self.device = coef, G, s2abs, done, device
        self.extra = extra  # device copies of the caller's `during` columns (pack_columns_device)

    def wait(self) -> None:
        self.done.synchronize()

    def upload(self, coef: np.ndarray, G: np.ndarray, s2abs: np.ndarray) -> None:
        """Replace the device columns by the host ones (after host-side patches)."""
        import torch

        self.wait()
        for d, h in ((self.coef, coef.view(np.int32)), (self.G, G.view(np.int64)), (self.s2abs, s2abs.view(np.int64))):
            d.copy_(torch.from_numpy(np.ascontiguousarray(h)))


def upload_columns(torch, arrays, dev, pin: bool = True) -> list:
    """Host 1-D columns -> device tensors of the same dtypes through ONE copy
    (a staging buffer, page-locked when pin; 8-byte aligned segments):
    each small pageable copy costs tens of microseconds on its own."""
    arrays = [np.ascontiguousarray(a) for a in arrays]
    offs, n = [], 0
    for a in arrays:
        offs.append(n)
        n += -(-a.nbytes // 8) * 8
    host = torch.empty(max(n, 8), dtype=torch.uint8, pin_memory=pin)
    h = host.numpy()
    for a, o in zip(arrays, offs):
        h[o:o + a.nbytes] = a.view(np.uint8).reshape(-1)
    dbuf = host.to(dev, non_blocking=pin)
    tdt = {1: torch.uint8, 4: torch.int32, 8: torch.int64}
    return [dbuf[o:o + a.nbytes].view(tdt[a.dtype.itemsize]) for a, o in zip(arrays, offs)]


def pack_columns_device(cfg, index_start, count, n_p, tau, e_out, device=None, resident: bool = False,
                        during=None):
    """hrb_pack_blocks: the native generation (hostgen.pack_columns' Taylor
    models, split, checks and packed columns) with one device thread per
    super-domain, the same source as the host library.  Returns host numpy
    arrays (coef, G, s2abs, status, shift_ok) like hostgen.pack_columns.
    resident=True also returns a ResidentColumns (appended to the tuple):
    the columns stay on the device for the search and their download runs
    behind it -- the returned coef / G / s2abs arrays are filled only once
    its wait() returned (status and shift_ok are final on return).
    during (resident only): a callable run on the host while the kernel
    runs; the 1-D columns it returns are uploaded (one copy) and kept as
    ResidentColumns.extra."""
    torch = nat.require_cuda()
    lib = nat.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is not None and dev.index != torch.cuda.current_device():
        with torch.cuda.device(dev):  # the library launches on the current device's stream
            return pack_columns_device(cfg, index_start, count, n_p, tau, e_out, dev, resident, during)
    S = len(index_start)
    cl = cfg.limbs + 1

    pin = S >= PIN_GEN_MIN or resident
    ins = upload_columns(torch, [np.asarray(index_start, dtype=np.uint64), np.asarray(count, dtype=np.uint64),
                                 np.asarray(n_p, dtype=np.uint32), np.asarray(tau, dtype=np.uint32),
                                 np.asarray(e_out, dtype=np.int32)], dev, pin)
    # every column of every block is written (status decides which are valid)
    coef = torch.empty((6, cl, S), dtype=torch.int32, device=dev)
    G = torch.empty((2, S), dtype=torch.int64, device=dev)
    s2 = torch.empty((2, S), dtype=torch.int64, device=dev)
    status = torch.empty(S, dtype=torch.uint8, device=dev)
    ok2 = torch.empty(S, dtype=torch.uint8, device=dev)
    nat.check("hrb_pack_blocks", lib.hrb_pack_blocks(C.byref(cfg), S, *(t.data_ptr() for t in ins), coef.data_ptr(),
                                                     G.data_ptr(), s2.data_ptr(), status.data_ptr(), ok2.data_ptr(),
                                                     nat.stream_ptr()))
    # download into pinned host memory (torch's caching host allocator): a
    # pageable download of the 16 MB of a 2^40 slice runs at a few GB/s once
    # it has to fault in fresh pages, and the pinned columns also make the
    # later upload of the slice a direct DMA
    # (small slices: pageable; pinning fresh host memory costs more than it saves)
    cur = torch.cuda.current_stream(dev)
    outs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=pin) for t in (coef, G, s2, status, ok2)]
    res = None
    if resident:
        # the flags now (the caller decides on them), the columns behind the
        # search on a side stream
        outs[3].copy_(status, non_blocking=True)
        outs[4].copy_(ok2, non_blocking=True)
        flags = cur.record_event()
        side = torch.cuda.Stream(dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            for h, t in zip(outs[:3], (coef, G, s2)):
                h.copy_(t, non_blocking=True)
                t.record_stream(side)
        extra = upload_columns(torch, during(), dev) if during is not None else None
        res = ResidentColumns(coef, G, s2, side.record_event(), dev, extra)
        flags.synchronize()
    else:
        for h, t in zip(outs, (coef, G, s2, status, ok2)):
            h.copy_(t, non_blocking=pin)
        cur.synchronize()
    cols = (outs[0].numpy().view(np.uint32), outs[1].numpy().view(np.uint64), outs[2].numpy().view(np.uint64),
            outs[3].numpy(), outs[4].numpy())
    return cols + (res,) if resident else cols
