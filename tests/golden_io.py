"""Load the reference-generated fixtures of tests/golden/ into this
package's types (SuperDomain, configs) so oracle and GPU runs can be fed
exactly what the reference computed."""

from __future__ import annotations

import json
import os
from fractions import Fraction

import numpy as np

from paper_1211_3056_b200.arith import DivisionMode, MPInt
from paper_1211_3056_b200.fpformat import FpFormat
from paper_1211_3056_b200.funnel import PhaseConfig, PipelineConfig
from paper_1211_3056_b200.slices import SuperDomain, pack_slice
from paper_1211_3056_b200.taylor import BinomialPoly, PolyGenConfig

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MODES = {"sub": DivisionMode.SUBTRACTIVE, "hybrid": DivisionMode.HYBRID, "hw": DivisionMode.HARDWARE}
MODE_CODE = {"sub": 0, "hybrid": 1, "hw": 2}
# column order of the search goldens: lefevre x (sub, hybrid, hw), swap x 3, regular, unrolled
CORE_COLUMNS = [("lefevre", 0), ("lefevre", 1), ("lefevre", 2), ("lefevre_swap", 0), ("lefevre_swap", 1),
                ("lefevre_swap", 2), ("regular", 1), ("regular_unrolled", 1)]

_cases = None


def pipeline_cases() -> list[dict]:
    global _cases
    if _cases is None:
        with open(os.path.join(GOLDEN, "pipeline_cases.json")) as fh:
            _cases = json.load(fh)
    return _cases


def case(name: str) -> dict:
    for c in pipeline_cases():
        if c["name"] == name:
            return c
    raise KeyError(name)


def config_of(c: dict) -> PipelineConfig:
    k = c["cfg"]
    pg = PolyGenConfig(tau=k["tau"], N=k["N"], mu=k["mu"], nu=k["nu"], delta=k["delta"], limbs=k["limbs"],
                       frac_bits=k["frac_bits"], guard=k["guard"])
    ph = PhaseConfig(algorithm=k["algorithm"], div_mode=MODES[k["div_mode"]], phase2_split=k["split"], N1=k["N"])
    return PipelineConfig(fn=c["fn"], fmt=FpFormat(c["p"], c["eps_bits"]), polygen=pg, phase=ph,
                          word_bits=k["word_bits"])


def supers_of(c: dict) -> list[SuperDomain]:
    limbs = c["cfg"]["limbs"]
    out = []
    for s in c["supers"]:
        rp = tuple(BinomialPoly(tuple(MPInt.from_int(int(x, 16), limbs) for x in poly), c["cfg"]["frac_bits"])
                   for poly in s["r_polys"])
        out.append(SuperDomain(s["index_start"], s["count"], s["n_p"], s["tau"], s["mu"], s["nu"], s["e_out"],
                               s["dom_id0"], rp, Fraction(int(s["eps_prime"][0]), int(s["eps_prime"][1]))))
    return out


def batch_of(c: dict):
    cfg = config_of(c)
    return pack_slice(supers_of(c), cfg.fmt, cfg.polygen, cfg.word_bits, c["binade"])


def essence(records) -> list:
    return [[hex(r.argument), r.distance.raw, r.domain_id, r.undecided] for r in records]


def load_search(name: str):
    z = np.load(os.path.join(GOLDEN, name))
    return {k: z[k] for k in z.files}
