"""Tabulated-differences kernel on its own (hrb_domain_coefficients,
polygen.py:255-280 domain_coefficient_sets): every domain's (s0, s1, s2)
as full-width two's-complement limbs, walked with add-with-carry chains from
the per-super-domain seeds.  Store-bound: reports domains/s and achieved HBM
GB/s (algorithmic bytes = the coefficient output written + the seeds read)
against MEASURED_PEAKS.json.  Prints one JSON line."""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-args", type=int, default=38)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch

    from paper_1211_3056_b200 import _native as nat
    from paper_1211_3056_b200.device import DeviceSlice

    ns = argparse.Namespace(log2_args=a.log2_args, eps_bits=32, algo="regular", log2_super=24, log2_N=15, fn="exp",
                            start=0)
    batch, _ = bench.prepare_rank(ns, 0, 1, os.cpu_count() or 1)
    ds = DeviceSlice(batch)
    cl = batch.coef_limbs
    out = torch.empty(3 * cl * batch.n_total, dtype=torch.int32, device="cuda")
    lib = nat.load()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def launch():
        nat.check("hrb_domain_coefficients", lib.hrb_domain_coefficients(C.byref(ds.desc), out.data_ptr(),
                                                                         nat.stream_ptr()))
    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    ms = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = float(np.mean(ms))
    # the write-only ceiling of this device: torch fills of 1 GiB (the kernel
    # is store-bound; the copy peak in MEASURED_PEAKS.json counts reads too)
    fills = {}
    big = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
    for name, fn in (("fill_i32", lambda: big.fill_(7)), ("zero_i32", lambda: big.zero_())):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        fills[name] = (1 << 30) / (min(ts) / 1e3) / 1e9
    wo = max(fills.values())
    written = out.numel() * 4
    read = batch.coef.nbytes + batch.n_dom.nbytes + batch.dom_base.nbytes
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    gbs = (written + read) / (t / 1e3) / 1e9
    print(json.dumps({"kernel": "tabdiff_full_kernel (hrb_domain_coefficients)", "domains": batch.n_total,
                      "limbs": cl, "ms": t, "domains_per_s": batch.n_total / (t / 1e3),
                      "args_per_s": batch.arguments / (t / 1e3), "bytes_written": written, "bytes_read": read,
                      "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak if peak else None,
                      "write_only_gbs": wo, "write_only_probes": fills, "frac_of_write_only": gbs / wo,
                      "note": "includes the per-launch prep kernels (tile scan); L2 flushed before each launch"}))


if __name__ == "__main__":
    main()
