"""Divergence fixtures from the REFERENCE itself (build container only):

    python tests/golden/make_divergence.py

Writes tests/golden/divergence.json: the reference's linear_problem_batch
problems (divergence.py:32-93) for exp at p=33 (the demo / acceptance C5
batch, demos/warp_divergence.py) and p=53 (Table III analogue, SURVEY.md
8d C2), and for every algorithm (and every division mode of the classic
walk) the reference's simulate_warps report: per-lane outcomes, iteration
counts, branch-decision traces, and per-warp MDM / NMDM / serialization.
"""

from __future__ import annotations

import json
import os
import sys
from fractions import Fraction

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from hardround.divergence import linear_problem_batch, simulate_warps  # noqa: E402
from hardround.fixedpoint import DivisionMode  # noqa: E402
from hardround.fpmodel import FpFormat  # noqa: E402
from hardround.lowerbound import Algorithm  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
RUNS = [("regular", "HYBRID"), ("regular_unrolled", "HYBRID"), ("lefevre", "SUBTRACTIVE"), ("lefevre", "HYBRID"),
        ("lefevre", "HARDWARE"), ("lefevre_swap", "HYBRID"), ("lefevre_swap", "SUBTRACTIVE")]


def frac(x: Fraction) -> list[str]:
    return [str(x.numerator), str(x.denominator)]


def bits_hex(path) -> str:
    v = 0
    for k, b in enumerate(path):
        if b:
            v |= 1 << k
    return hex(v)


def case(name, fmt, domain_size, domain_count, warp_width=32):
    batch = linear_problem_batch("exp", fmt, 0, domain_size, domain_count=domain_count)
    out = {"name": name, "p": fmt.precision, "eps_bits": fmt.eps_bits, "domain_size": domain_size,
           "domain_count": domain_count, "warp_width": warp_width,
           "problems": [[p.a.raw, p.b.raw, p.eps.raw, p.count] for p in batch], "runs": []}
    for algo, mode in RUNS:
        rep = simulate_warps(batch, Algorithm(algo), DivisionMode[mode], warp_width)
        lanes = []
        for t in rep.traces:
            for it, path, o in zip(t.lane_iterations, t.branch_paths, t.outcomes):
                lanes.append([int(o.success), o.d.raw, it, o.points_placed, len(path), bits_hex(path)])
        warps = [[frac(w.mdm), frac(w.nmdm), w.serialized_iterations, w.branch_serialized_instructions]
                 for w in rep.warps]
        out["runs"].append({"algo": algo, "mode": mode, "lanes": lanes, "warps": warps,
                            "min": rep.min_iterations, "max": rep.max_iterations,
                            "mean": frac(rep.mean_iterations), "mean_nmdm": frac(rep.mean_nmdm)})
    return out


def main():
    cases = [case("exp_p33_512x1024", FpFormat(33, 22), 512, 1024),
             case("exp_p53_2p15x512", FpFormat(53, 32), 1 << 15, 512),
             case("exp_p33_w8", FpFormat(33, 22), 256, 64, warp_width=8)]
    with open(os.path.join(HERE, "divergence.json"), "w") as fh:
        json.dump(cases, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
