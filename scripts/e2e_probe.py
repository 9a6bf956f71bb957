"""Where the end-to-end call's time goes: wall time of hrb_run_slice_host
against its own device interval (events e0 -> e1 on the compute stream), the
bare H2D of the same bytes, and the D2H of the failing ids.

    python scripts/e2e_probe.py [--log2-args 40]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1211_3056_b200.device import HostRunner  # noqa: E402


def main():
    args = bench.parse()
    batch, _ = bench.prepare_rank(args, 0, 1, os.cpu_count() or 1)
    host = HostRunner(batch, 2, 1, 8)
    for _ in range(3):
        host.run()
    wall, dev = [], []
    for _ in range(10):
        t0 = time.perf_counter()
        host.run()
        wall.append(1e3 * (time.perf_counter() - t0))
        dev.append(host.device_ms.value)
    nb_in, nb_out = host.input_bytes(), host.output_bytes()
    x = torch.empty(nb_in, dtype=torch.uint8, pin_memory=True)
    y = torch.empty(nb_in, dtype=torch.uint8, device="cuda")
    z = torch.empty(nb_out, dtype=torch.uint8, pin_memory=True)
    w = torch.empty(nb_out, dtype=torch.uint8, device="cuda")
    h2d, d2h = [], []
    for _ in range(10):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        y.copy_(x, non_blocking=True)
        e1.record()
        z.copy_(w, non_blocking=True)
        e2.record()
        torch.cuda.synchronize()
        h2d.append(e0.elapsed_time(e1))
        d2h.append(e1.elapsed_time(e2))
    print({"wall_ms": round(float(np.median(wall)), 4), "device_ms": round(float(np.median(dev)), 4),
           "h2d_ms": round(float(np.median(h2d)), 4), "h2d_bytes": nb_in, "d2h_ms": round(float(np.median(d2h)), 4),
           "d2h_bytes": nb_out})


if __name__ == "__main__":
    main()
