"""hardround-b200: B200-native (sm_100a) hard-to-round case search.

A drop-in for the reference `hardround` package's hot path
(/root/reference/pkg/src/hardround/__init__.py:62-114 export list): the same
public names, with the searches, the tabulated coefficient walk, the three
filtering phases and all compaction executed by hand-written CUDA kernels
behind the C-ABI of include/hrb200.h.  Rigorous Taylor models, error
budgets and candidate confirmation stay on the host (mpmath), as in the
paper's hybrid CPU-GPU split.
"""

from .arith import DivisionMode, MPInt, MPOverflowError, UFrac, frac_div
from .divergence import (
    BRANCH_WEIGHTS,
    BranchWeights,
    DivergenceReport,
    WarpStats,
    WarpTrace,
    branch_serialization_estimate,
    linear_problem_batch,
    mdm,
    measure_warps,
    nmdm,
    simulate_warps,
)
from .enclosure import UndecidedError, decide_hr, derivative_bound, enclose, value_exponent
from .fpformat import (
    BinadeDomains,
    Domain,
    ErrorBudget,
    FpFormat,
    HrCaseRecord,
    bits_float,
    dist_p,
    float_bits,
    is_hr_case,
    mantissa_exponent,
    split_binade,
)
from .funnel import (
    DomainTask,
    PhaseConfig,
    PhaseRow,
    PhaseStats,
    PipelineConfig,
    SubdomainTask,
    phase1,
    phase2,
    phase3_exhaustive,
    prepare_slice,
    execute_batch,
    run_pipeline,
    run_range,
    run_slice,
    select_algorithm,
)
from .search import (
    SEARCHES,
    Algorithm,
    SearchOutcome,
    SearchProblem,
    Verdict,
    lefevre_lb,
    lefevre_swap_lb,
    regular_lb,
    regular_unrolled_lb,
    search_many,
)
from .records import emit_records, emit_stats, record_dict, write_records
from .slices import SliceBatch, SuperDomain, build_super_domains, output_binade_pieces, pack_slice
from .taylor import (
    BinomialPoly,
    PolyGenConfig,
    forward_difference,
    hierarchical_split,
    newton_interpolate,
    straightforward_shift,
    tabulated_shift_step,
    taylor_approx,
)

__version__ = "0.1.0"


def domain_coefficient_sets(r_polys, cfg: PolyGenConfig) -> list[tuple]:
    """Drop-in for the reference's domain_coefficient_sets (polygen.py:274-280):
    per-domain coefficient tuples (s_0..s_delta) = (r_0(i), .., r_delta(i))
    of one super-domain, i < cfg.tau, as MPInt with cfg.limbs limbs -- the
    values of the reference's (j, u, i) packet walk (generate_packets,
    polygen.py:255-271).  The walk runs on the GPU (hrb_domain_coefficients:
    add-with-carry chains over L+1 two's-complement limbs, exact while the
    values fit the MPInt budget).  Where the reference's walk would raise
    MPOverflowError (fixedpoint.py:136), the exact host replay raises it
    first; only the walk is involved (FpFormat, eps and the search do not
    enter), so the slice is packed without the phase checks."""
    from fractions import Fraction

    from .arith import as_int
    from .device import DeviceSlice, domain_coefficients
    from .slices import _emulate_walk, _walk_bound

    r_polys = [BinomialPoly(tuple(as_int(c) for c in rp.coeffs), rp.scale) for rp in r_polys]
    delta = len(r_polys) - 1
    if not 0 <= delta <= 2:
        raise ValueError("the device walk takes delta <= 2 (the reference's PolyGenConfig range)")
    sd = SuperDomain(0, cfg.tau * cfg.N, cfg.N, cfg.tau, cfg.mu, cfg.nu, 0, 0, tuple(r_polys), Fraction(0))
    if _walk_bound(sd) >> (32 * cfg.limbs) or (cfg.tau * cfg.tau) >> (32 * cfg.limbs):
        _emulate_walk(sd, cfg.limbs)  # raises MPOverflowError where the reference's walk would
    padded = tuple(r_polys) + (BinomialPoly((0,)),) * (2 - delta)
    # frac_bits / word_bits only feed the search; any legal pair packs the walk
    pg = PolyGenConfig(tau=cfg.tau, N=cfg.N, mu=cfg.mu, nu=cfg.nu, delta=2, limbs=cfg.limbs, frac_bits=64,
                       guard=cfg.guard)
    batch = pack_slice([SuperDomain(0, sd.count, sd.n_p, sd.tau, sd.mu, sd.nu, 0, 0, padded, Fraction(0))],
                       FpFormat(53, 32), pg, 64, 0, check=False)
    raw = domain_coefficients(DeviceSlice(batch))
    cl = raw.shape[1]
    out = []
    for i in range(cfg.tau):
        vals = []
        for j in range(delta + 1):
            v = 0
            for l in range(cl):
                v |= int(raw[j, l, i]) << (32 * l)
            if v >> (32 * cl - 1):
                v -= 1 << (32 * cl)
            vals.append(MPInt.from_int(v, cfg.limbs))
        out.append(tuple(vals))
    return out


__all__ = [
    "emit_records", "emit_stats", "record_dict", "write_records",
    "BRANCH_WEIGHTS", "BranchWeights", "DivergenceReport", "WarpStats", "WarpTrace", "branch_serialization_estimate",
    "linear_problem_batch", "mdm", "measure_warps", "nmdm", "simulate_warps",
    "Algorithm", "BinadeDomains", "BinomialPoly", "DivisionMode", "Domain", "DomainTask", "ErrorBudget",
    "FpFormat", "HrCaseRecord", "MPInt", "MPOverflowError", "PhaseConfig", "PhaseRow", "PhaseStats",
    "PipelineConfig", "PolyGenConfig", "SEARCHES", "SearchOutcome", "SearchProblem", "SliceBatch",
    "SubdomainTask", "SuperDomain", "UFrac", "UndecidedError", "Verdict", "bits_float", "build_super_domains",
    "decide_hr", "derivative_bound", "dist_p", "domain_coefficient_sets", "enclose", "execute_batch",
    "float_bits", "forward_difference", "frac_div", "hierarchical_split", "is_hr_case", "lefevre_lb",
    "lefevre_swap_lb", "mantissa_exponent", "newton_interpolate", "output_binade_pieces", "pack_slice",
    "phase1", "phase2", "phase3_exhaustive", "prepare_slice", "regular_lb", "regular_unrolled_lb",
    "run_pipeline", "run_range", "run_slice", "search_many", "select_algorithm", "split_binade", "straightforward_shift",
    "tabulated_shift_step", "taylor_approx", "value_exponent",
]
