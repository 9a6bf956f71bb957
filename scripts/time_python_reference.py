"""Time the REFERENCE's own pure-Python path (build container only: it
imports /root/reference/pkg/src, which does not exist on the GPU box) on a
slice of the bench workload: exp p=53, eps=2^-32, N=2^15, super-domains of
2^24, delta=2, F=96, split 8, regular.  Phases are timed separately, single
process (the reference's ThreadPool is GIL-bound).

    python scripts/time_python_reference.py [log2_args] > profiles/r01/python_reference_timing.json
"""
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")

from hardround.fpmodel import Domain, FpFormat  # noqa: E402
from hardround.pipeline import (DomainTask, PhaseConfig, PipelineConfig, phase1, phase2,  # noqa: E402
                                phase3_exhaustive)
from hardround.polygen import PolyGenConfig, domain_coefficient_sets, hierarchical_split, taylor_approx  # noqa: E402


def main():
    log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    N, tau = 1 << 15, 512
    pg = PolyGenConfig(tau=tau, N=N, mu=16, nu=32, delta=2, limbs=8, frac_bits=96, guard=32)
    fmt = FpFormat(53, 32)
    cfg = PipelineConfig("exp", fmt, pg, PhaseConfig("regular", phase2_split=8, N1=N))
    m_base = 1 << 52
    t0 = time.perf_counter()
    tasks, nid = [], 0
    t_taylor = t_tab = 0.0
    for s in range(0, 1 << log2, 1 << 24):
        ta = time.perf_counter()
        sup = Domain(m_base + s, 1, 1 << 24, nid)
        r_t, eps_approx = taylor_approx("exp", sup, pg, fmt)
        r_polys = hierarchical_split(r_t, N, 2)
        tb = time.perf_counter()
        for i, coeffs in enumerate(domain_coefficient_sets(r_polys, pg)):
            tasks.append(DomainTask(Domain(m_base + s + i * N, 1, N, nid), coeffs, 96, fmt.eps + eps_approx, 0))
            nid += 1
        tc = time.perf_counter()
        t_taylor += tb - ta
        t_tab += tc - tb
    t1 = time.perf_counter()
    fails = phase1(tasks, cfg, "regular")
    t2 = time.perf_counter()
    by_id = {t.domain.domain_id: t for t in tasks}
    subs = phase2([by_id[i] for i in fails], cfg, "regular")
    t3 = time.perf_counter()
    cands = phase3_exhaustive(subs, cfg)
    t4 = time.perf_counter()
    args = 1 << log2
    hot = t_tab + (t4 - t1)
    print(json.dumps({
        "what": "reference hardround (pure Python) on its own code path, single process, this build container",
        "host": os.uname().nodename, "cpu_count": os.cpu_count(),
        "workload": f"exp p=53 [1,2) indices [0, 2^{log2}) eps=2^-32 N=2^15 super=2^24 delta=2 F=96 split=8 regular",
        "arguments": args, "domains": len(tasks), "phase1_fail": len(fails), "phase2_survivors": len(subs),
        "candidates": len(cands),
        "seconds": {"taylor_and_split": t_taylor, "domain_coefficient_sets": t_tab, "phase1": t2 - t1,
                    "phase2": t3 - t2, "phase3": t4 - t3},
        "hot_path_args_per_s": args / hot,
        "hot_path": "domain_coefficient_sets + phase1 + phase2 + phase3 (the GPU's part)"}, indent=1))


if __name__ == "__main__":
    main()
