"""Device confirmation throughput: hrb_confirm_exp on N random candidates
(exp p=53, binade 0), wall time and device time, against the host library.

    python scripts/confirm_probe.py --n 2000000 --eps-bits 16
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 21)
    ap.add_argument("--eps-bits", type=int, default=16)
    ap.add_argument("--host", action="store_true")
    a = ap.parse_args()
    import torch

    from paper_1211_3056_b200 import hostgen
    from paper_1211_3056_b200.fpformat import FpFormat
    from paper_1211_3056_b200.funnel import confirm_on_device
    from paper_1211_3056_b200.taylor import PolyGenConfig

    fmt = FpFormat(53, a.eps_bits)
    idx = np.random.default_rng(1).integers(0, 1 << 52, a.n, dtype=np.uint64)
    confirm_on_device(fmt, 0, idx[:1000])
    torch.cuda.synchronize()
    t = time.perf_counter()
    is_hr, d, st = confirm_on_device(fmt, 0, idx)
    torch.cuda.synchronize()
    out = {"n": a.n, "device_wall_s": time.perf_counter() - t, "undecided_on_device": int(st.sum()),
           "hr": int(is_hr.sum())}
    if a.host:
        cfg = hostgen.make_cfg("exp", fmt, PolyGenConfig(), 0, 64)
        t = time.perf_counter()
        h = hostgen.confirm(cfg, idx, 0)
        out["host_wall_s"] = time.perf_counter() - t
        out["equal"] = bool(np.array_equal(h[0], is_hr) and np.array_equal(h[1][h[0] == 1], d[is_hr == 1]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
