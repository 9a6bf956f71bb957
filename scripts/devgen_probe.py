"""Time the device generation (hrb_pack_blocks) against the host library on
the bench workload's plan (exp, 2^40 arguments, 65,536 super-domains);
one JSON line.  HRB_LIB selects a variant library."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1211_3056_b200 import hostgen
    from paper_1211_3056_b200.device import pack_columns_device
    from paper_1211_3056_b200.fpformat import FpFormat
    from paper_1211_3056_b200.slices import plan_arrays
    from paper_1211_3056_b200.taylor import PolyGenConfig

    log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    fmt = FpFormat(53, 32)
    pg = PolyGenConfig(tau=512, N=1 << 15, mu=16, nu=32, delta=2, limbs=8, frac_bits=96, guard=32)
    plan = plan_arrays("exp", 0, fmt, pg, 0, 1 << log2)
    cfg = hostgen.make_cfg("exp", fmt, pg, 0, 64)
    cols = (plan.bstart, plan.bcount, plan.n_p, plan.tau, plan.e_out)
    pack_columns_device(cfg, *cols)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pack_columns_device(cfg, *cols)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"lib": os.environ.get("HRB_LIB", "default"), "supers": len(plan),
                      "device_ms": round(1e3 * float(np.median(ts)), 3), "samples": [round(1e3 * t, 3) for t in ts]}))


if __name__ == "__main__":
    main()
