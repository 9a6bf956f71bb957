"""Golden HR sets from the REFERENCE's exhaustive enumerator
(oracle.py:77-113 exhaustive_hr_search: every argument decided by direct
rigorous evaluation, no polynomial, no filter).  Build container only:

    python tests/golden/make_exhaustive.py

Writes tests/golden/exhaustive.json: for each case the (argument bits,
distance raw 2^-64, undecided) of every HR case in order.  These pin the
end results of paths the reference itself cannot run -- the high-degree
(delta >= 3) pipeline -- and every other path's records.
"""

from __future__ import annotations

import json
import os
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from hardround.fpmodel import Domain, FpFormat  # noqa: E402
from hardround.oracle import exhaustive_hr_search  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (name, fn, p, eps_bits, binade, start index, count)
CASES = [
    ("exp_p53_2p20_e16", "exp", 53, 16, 0, 0, 1 << 20),
    ("exp_p53_2p20_e20", "exp", 53, 20, 0, 0, 1 << 20),
    ("exp_p53_2p20_e16_mid", "exp", 53, 16, 0, 0x5A827999FCEF3, 1 << 20),
    ("exp_p53_2p20_e16_bm1", "exp", 53, 16, -1, 0x3C6EF372FE94F, 1 << 20),
]


def main():
    out = []
    for name, fn, p, eps_bits, binade, start, count in CASES:
        fmt = FpFormat(p, eps_bits)
        dom = Domain((1 << (p - 1)) + start, binade + 1, count, 0)
        recs = exhaustive_hr_search(fn, dom, fmt)
        out.append({"name": name, "fn": fn, "p": p, "eps_bits": eps_bits, "binade": binade, "start": start,
                    "count": count,
                    "records": [[hex(r.argument), r.distance.raw, bool(r.undecided)] for r in recs]})
        print(name, len(recs), flush=True)
    with open(os.path.join(HERE, "exhaustive.json"), "w") as fh:
        json.dump(out, fh, indent=0)


if __name__ == "__main__":
    main()
