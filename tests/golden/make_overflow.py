"""Golden outcomes of the REFERENCE's host generation under tight limb
budgets (MPInt raises MPOverflowError on carry-out / product overflow,
fixedpoint.py:136-137, 239, 252, 291, 300; reached through taylor_approx's
MPInt.from_int, polygen.py:236, hierarchical_split's MPInt products,
polygen.py:113-131, and the packet walk, polygen.py:255-271).  Build
container only:

    python tests/golden/make_overflow.py

For each configuration: the reference's _build_tasks over the whole binade
(pipeline.py:374-409) either succeeds (the number of domain tasks is
recorded) or raises (the exception class name is recorded).
"""

from __future__ import annotations

import json
import os
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from hardround.fpmodel import FpFormat  # noqa: E402
from hardround.pipeline import PhaseConfig, PipelineConfig, _build_tasks  # noqa: E402
from hardround.polygen import PolyGenConfig  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    out = []
    for fn, p, binade in (("exp", 13, 0), ("exp", 13, -1), ("log", 13, 1)):
        for limbs, F in ((3, 96), (3, 90), (3, 84), (3, 83), (3, 82), (3, 80), (3, 76), (2, 64), (2, 56), (4, 116)):
            if F > 32 * limbs:
                continue
            pg = PolyGenConfig(tau=16, N=64, mu=4, nu=4, delta=2, limbs=limbs, frac_bits=F, guard=32)
            cfg = PipelineConfig(fn=fn, fmt=FpFormat(p, 8), polygen=pg,
                                 phase=PhaseConfig(algorithm="regular", N1=64))
            try:
                tasks = _build_tasks(fn, binade, cfg)
                res = {"ok": True, "tasks": len(tasks)}
            except Exception as e:  # noqa: BLE001 -- the class is the recorded outcome
                res = {"ok": False, "error": type(e).__name__, "message": str(e)[:200]}
            out.append({"fn": fn, "p": p, "eps_bits": 8, "binade": binade, "limbs": limbs, "frac_bits": F,
                        "tau": 16, "N": 64, "mu": 4, "nu": 4, **res})
            print(fn, binade, limbs, F, res, flush=True)
    with open(os.path.join(HERE, "overflow.json"), "w") as fh:
        json.dump(out, fh, indent=0)


if __name__ == "__main__":
    main()
