"""GPU parity: the CUDA path (libhrb200 via the C-ABI) against the reference's
golden vectors and the CPU oracle.  Integer work, so every comparison is
bit-exact."""

from fractions import Fraction

import numpy as np
import pytest

import oracle
from golden_io import CORE_COLUMNS, MODE_CODE, batch_of, case, config_of, essence, load_search, pipeline_cases

pytestmark = pytest.mark.gpu

ALGO_CODE = {"lefevre": 0, "lefevre_swap": 1, "regular": 2, "regular_unrolled": 3}


def gpu_search(algo, mode, W, a, b, e, n):
    from paper_1211_3056_b200.device import search_batch_arrays

    return search_batch_arrays(ALGO_CODE[algo], mode, W, a, b, e, n)


@pytest.mark.parametrize("fixture,W", [("search_w64.npz", 64), ("search_w32.npz", 32)])
def test_search_batch_matches_reference_goldens(fixture, W):
    g = load_search(fixture)
    for col, (algo, mode) in enumerate(CORE_COLUMNS):
        ok, d, it, pl, ph = gpu_search(algo, mode, W, g["a"], g["b"], g["eps"], g["count"])
        bad = np.nonzero((ok != g["ok"][:, col]) | (d != g["d"][:, col]) | (it != g["it"][:, col])
                         | (pl != g["pts_lo"][:, col]) | (ph.astype(np.uint64) != g["pts_hi"][:, col]))[0]
        assert bad.size == 0, (fixture, algo, mode, bad[:5].tolist(),
                               [(int(g["a"][k]), int(g["b"][k]), int(g["eps"][k]), int(g["count"][k])) for k in bad[:3]])


@pytest.mark.parametrize("algo,mode", [("regular", 1), ("regular_unrolled", 1), ("lefevre", 0), ("lefevre", 1),
                                       ("lefevre", 2), ("lefevre_swap", 1)])
def test_search_batch_random_vs_oracle(algo, mode):
    rng = np.random.default_rng(1234 + ALGO_CODE[algo] * 3 + mode)
    n = 1 << 20
    a = rng.integers(0, 2**64, n, dtype=np.uint64)
    b = rng.integers(0, 2**64, n, dtype=np.uint64)
    e = rng.integers(1, 2**36, n, dtype=np.uint64)
    N = rng.choice(np.array([1, 2, 3, 17, 1 << 12, 1 << 15, 1 << 16], dtype=np.uint64), n)
    got = gpu_search(algo, mode, 64, a, b, e, N)
    want = oracle.search_batch(algo, mode, 1 << 64, a, b, e, N)
    for k, name in enumerate(("ok", "d", "it", "pts_lo", "pts_hi")):
        assert np.array_equal(got[k].astype(np.uint64), want[k].astype(np.uint64)), (algo, mode, name)


@pytest.mark.parametrize("algo", ["lefevre", "lefevre_swap", "regular", "regular_unrolled"])
def test_criterion2_embedded_grid_sweep(algo):
    """test_acceptance.py:93-163 at full size on the device: every (a, b) on
    the 2^10 grid, N in {16, 256, 1024}, embedded into W=64 words by << 54;
    results must be the grid cores' results shifted, and Success must be
    sound against the exact minimum."""
    grid = 1 << 10
    eps = grid >> 6
    A, B = np.meshgrid(np.arange(grid, dtype=np.uint64), np.arange(grid, dtype=np.uint64), indexing="ij")
    A, B = A.ravel(), B.ravel()
    for n in (16, 256, 1024):
        N = np.full(A.size, n, dtype=np.uint64)
        E = np.full(A.size, eps, dtype=np.uint64)
        ok, d, it, pl, ph = gpu_search(algo, 2, 64, A << np.uint64(54), B << np.uint64(54), E << np.uint64(54), N)
        wok, wd, wit, wpl, wph = oracle.search_batch(algo, 2, grid, A, B, E, N)
        assert np.array_equal(ok, wok)
        assert np.array_equal(d, wd << np.uint64(54))
        assert np.array_equal(it, wit)
        # exact minimum over x < n for every (a, b): soundness of Success
        x = np.arange(n, dtype=np.int64)
        succ = np.nonzero(ok)[0]
        av, bv = A[succ].astype(np.int64), B[succ].astype(np.int64)
        for chunk in range(0, succ.size, 1 << 14):
            sl = slice(chunk, chunk + (1 << 14))
            truth = ((bv[sl, None] - av[sl, None] * x[None, :]) % grid).min(axis=1)
            assert (truth >= eps).all()
            assert ((d[succ][sl] >> np.uint64(54)).astype(np.int64) <= truth).all()


@pytest.mark.parametrize("name", [c["name"] for c in pipeline_cases()])
def test_pipeline_case_matches_reference(name):
    from paper_1211_3056_b200.funnel import execute_batch

    c = case(name)
    cfg = config_of(c)
    batch = batch_of(c)
    out = execute_batch(batch, cfg, c["cfg"]["algorithm"], c["fn"])
    assert out.failing_ids == c["phase1_fail"]
    assert [list(r) for r in out.sub_rows] == [r[:4] for r in c["phase2"]]
    assert [[hex(x.argument), x.distance.raw, x.domain_id] for x in out.candidates] == c["phase3"]
    assert essence(out.records) == c["records"]
    st = {r.phase: r for r in out.stats.rows}
    assert [st["phase1"].domains_in, st["phase1"].domains_out, st["phase1"].arguments_covered] == c["stats"]["phase1"]
    assert [st["phase2"].domains_in, st["phase2"].domains_out, st["phase2"].arguments_covered] == c["stats"]["phase2"]
    assert [st["phase3"].domains_in, st["phase3"].domains_out, st["phase3"].arguments_covered] == c["stats"]["phase3"]


@pytest.mark.parametrize("name", ["p13_exp_b0", "p53_exp_2p20_e16_N12", "p53_exp_ragged", "p53_exp_delta1"])
def test_tabulated_values_match_reference(name):
    """hrb_domain_coefficients (full-width add-with-carry walk) equals the
    reference's domain_coefficient_sets value for value."""
    from paper_1211_3056_b200.device import DeviceSlice, domain_coefficients

    c = case(name)
    batch = batch_of(c)
    raw = domain_coefficients(DeviceSlice(batch))
    cl = raw.shape[1]
    for k, dom in enumerate(c["domains"]):
        for j, hx in enumerate(dom[3:]):
            v = 0
            for l in range(cl):
                v |= int(raw[j, l, k]) << (32 * l)
            if v >> (32 * cl - 1):
                v -= 1 << (32 * cl)
            assert v == int(hx, 16), (name, k, j)


# p13_log_b0 (41 super-domains) and p16_exp_b1 (131) stream their upload in
# 16 chunks through hrb_run_slice_host; the Lefevre cases upload up front
@pytest.mark.parametrize("name", ["p53_exp_2p20_e16_N12", "p53_exp_ragged", "p13_log_b0", "p16_exp_b1",
                                  "p53_exp_delta1", "p13_exp_b0_lefevre", "p53_exp_lef_hw"])
def test_fused_and_host_paths_equal_phase_path(name):
    from paper_1211_3056_b200.device import DeviceSlice, FusedRunner, run_host, run_phases

    c = case(name)
    batch = batch_of(c)
    algo = ALGO_CODE[c["cfg"]["algorithm"]]
    mode = MODE_CODE[c["cfg"]["div_mode"]]
    split = c["cfg"]["split"]
    ds = DeviceSlice(batch)
    ref = run_phases(ds, algo, mode, split)
    fused = FusedRunner(ds, algo, mode, split, sub_cap=batch.n_total * 2 * split, cand_cap=1 << 16)
    for _ in range(2):  # re-launch on the same buffers: no stale state
        fused.launch()
        r = fused.result()
        assert np.array_equal(r.fail_ids, ref.fail_ids)
        assert np.array_equal(r.sub_keys, ref.sub_keys)
        assert np.array_equal(r.cand_index, ref.cand_index)
        assert np.array_equal(r.cand_dist, ref.cand_dist)
        assert r.iterations == ref.iterations
    counts, fail, cm, cd, cdom, ms = run_host(batch, algo, mode, split)
    assert np.array_equal(fail, ref.fail_ids)
    assert np.array_equal(cm, ref.cand_index) and np.array_equal(cd, ref.cand_dist)
    assert np.array_equal(cdom, ref.cand_dom)
    assert ms > 0


def test_run_pipeline_whole_binade_host_polygen():
    """Host Taylor generation (this package) + device phases reproduce the
    reference's run_pipeline records and stats for exp p=13 binade 0."""
    from paper_1211_3056_b200 import run_pipeline

    c = case("p13_exp_b0")
    records, stats = run_pipeline(0, config_of(c))
    assert essence(records) == c["records"]
    assert len(records) == 42
    assert [r.phase for r in stats.rows] == ["phase1", "phase2", "phase3", "confirm"]


def test_per_phase_dropins():
    """phase1 / phase2 / phase3_exhaustive over explicit DomainTasks."""
    from paper_1211_3056_b200 import Domain, DomainTask, phase1, phase2, phase3_exhaustive
    from paper_1211_3056_b200.arith import MPInt

    c = case("p13_exp_b0")
    cfg = config_of(c)
    m_base = 1 << (c["p"] - 1)
    eps_of = {}
    for s in c["supers"]:
        for k in range(s["tau"]):
            eps_of[s["dom_id0"] + k] = (Fraction(int(s["eps_prime"][0]), int(s["eps_prime"][1])), s["e_out"])
    tasks = []
    for dom in c["domains"]:
        did, m_off, cnt = dom[0], dom[1], dom[2]
        ep, e_out = eps_of[did]
        tasks.append(DomainTask(Domain(m_base + m_off, c["binade"] + 1, cnt, did),
                                tuple(MPInt.from_int(int(h, 16), 8) for h in dom[3:]), 96, ep, e_out))
    fails = phase1(tasks, cfg, "regular")
    assert fails == c["phase1_fail"]
    by_id = {t.domain.domain_id: t for t in tasks}
    subs = phase2([by_id[i] for i in fails], cfg, "regular")
    assert [[s.parent.domain.domain_id, s.sub_index, s.start, s.count] for s in subs] == [r[:4] for r in c["phase2"]]
    cands = phase3_exhaustive(subs, cfg)
    assert [[hex(x.argument), x.distance.raw, x.domain_id] for x in cands] == c["phase3"]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_logical_shards_equal_reference(world):
    """G logical shards on one device (the multi-GPU partition and merge)
    reproduce the reference's candidates and records of the whole slice."""
    from paper_1211_3056_b200.shard import run_logical_shards

    c = case("p53_exp_2p20_e16_N12")
    cfg = config_of(c)
    lo, cnt = c["slice"]
    merged, per_rank = run_logical_shards(c["fn"], c["binade"], lo, cnt, cfg, world)
    cand = [[hex((int(h) << 64) | int(l)), int(d), int(i)] for h, l, d, i in merged.cand.tolist()]
    assert cand == c["phase3"]
    assert essence(merged.record_objects()) == c["records"]
    assert int(merged.counters[0]) == len(c["phase1_fail"])
    assert int(per_rank[:, 5].sum()) == cnt


def _big_slice(fn, start, log2_count, eps_bits, algo="regular", N=1 << 15, super_log2=24):
    from paper_1211_3056_b200 import FpFormat, PhaseConfig, PipelineConfig, PolyGenConfig
    from paper_1211_3056_b200.funnel import prepare_slice

    tau = (1 << super_log2) // N
    mu = 1 << ((tau.bit_length() - 1) // 2)
    pg = PolyGenConfig(tau=tau, N=N, mu=mu, nu=tau // mu, delta=2, limbs=8, frac_bits=96, guard=32)
    cfg = PipelineConfig(fn, FpFormat(53, eps_bits), pg, PhaseConfig(algo, phase2_split=8, N1=N))
    import os

    return prepare_slice(fn, 0, start, 1 << log2_count, cfg, workers=os.cpu_count() or 1), cfg


@pytest.mark.parametrize("fn,start,log2_count,eps_bits,algo", [
    ("exp", 0, 36, 24, "regular"),          # C5-shaped: loose eps, many candidates
    ("exp", 1 << 44, 34, 32, "lefevre"),    # classic walk in the fused pipeline
    ("log", 0x6A09E667F3BCD, 34, 28, "regular"),  # C4-shaped: log near sqrt(2)
])
def test_large_slice_fused_equals_oracle(fn, start, log2_count, eps_bits, algo):
    """Full outputs of hrb_run_slice at 2^34-2^36 arguments (thousands of
    super-domains) equal the CPU oracle's: failing ids, surviving
    subdomains, candidates (argument, distance, domain)."""
    from paper_1211_3056_b200.device import DeviceSlice, FusedRunner

    batch, cfg = _big_slice(fn, start, log2_count, eps_bits, algo)
    code = ALGO_CODE[algo]
    fused = FusedRunner(DeviceSlice(batch), code, 1, 8, sub_cap=batch.n_total * 16, cand_cap=1 << 22)
    fused.launch()
    r = fused.result()
    want1 = oracle.phase1(batch, algo, 1)
    assert np.array_equal(r.fail_ids + np.uint64(batch.id0), want1)
    rows = oracle.phase2(batch, algo, 1, 8, want1)
    got_keys = (r.sub_keys >> np.uint64(8)) + np.uint64(batch.id0)
    assert np.array_equal(got_keys, rows[0]) and np.array_equal(r.sub_keys & np.uint64(255), rows[1].astype(np.uint64))
    m, dist, dom = oracle.phase3(batch, rows)
    assert np.array_equal(r.cand_index, m) and np.array_equal(r.cand_dist, dist)
    assert np.array_equal(r.cand_dom + np.uint64(batch.id0), dom)
    assert len(m) > 0 or eps_bits >= 28


def test_large_slice_logical_shards_and_rerun_are_identical():
    """Determinism and shard invariance at 2^36: 4 logical shards merged in
    rank order equal the single run, and a re-launch reproduces it."""
    from paper_1211_3056_b200.device import DeviceSlice, FusedRunner
    from paper_1211_3056_b200.shard import partition_blocks
    from paper_1211_3056_b200.slices import slice_view

    batch, cfg = _big_slice("exp", 0, 36, 20)
    whole = FusedRunner(DeviceSlice(batch), 2, 1, 8, sub_cap=batch.n_total * 16, cand_cap=1 << 22)
    whole.launch()
    a = whole.result()
    whole.launch()
    b = whole.result()
    assert np.array_equal(a.cand_index, b.cand_index) and np.array_equal(a.fail_ids, b.fail_ids)
    parts = partition_blocks([s.count for s in batch.supers], 4)
    fails, cands = [], []
    for t0, t1 in parts:
        sub = slice_view(batch, t0, t1)
        fr = FusedRunner(DeviceSlice(sub), 2, 1, 8, sub_cap=sub.n_total * 16, cand_cap=1 << 22)
        fr.launch()
        rr = fr.result()
        fails.append(rr.fail_ids + np.uint64(sub.id0 - batch.id0))
        cands.append(rr.cand_index)
    assert np.array_equal(np.concatenate(fails), a.fail_ids)
    assert np.array_equal(np.concatenate(cands), a.cand_index)


def _adversarial_problems(rng, n):
    """Inputs that stress the lockstep form's rare paths: huge and
    near-integer continued-fraction quotients (a close to a rational with a
    small denominator, tiny a, a near 1), counts at the 32-bit edge."""
    one = 1 << 64
    rows = []
    for k in range(n):
        kind = k % 8
        if kind == 0:    # a ~ one * p / q: the expansion hits a huge quotient
            q = int(rng.integers(2, 5000))
            p = int(rng.integers(1, q))
            a = (one * p // q + int(rng.integers(-3, 4))) % one
        elif kind == 1:  # tiny slope
            a = int(rng.integers(1, 1 << 20))
        elif kind == 2:  # slope just below one
            a = one - int(rng.integers(1, 1 << 20))
        elif kind == 3:  # near 2^64 / k
            a = one // int(rng.integers(2, 1 << 16)) + int(rng.integers(-2, 3))
        elif kind == 4:  # near 2^63 (S <= 2^63 boundary)
            a = (1 << 63) + int(rng.integers(-1 << 10, 1 << 10))
        else:
            a = int(rng.integers(0, 1 << 63)) * 2 + int(rng.integers(0, 2))
        a %= one
        b = int(rng.integers(0, 1 << 63)) * 2 + int(rng.integers(0, 2))
        e = int(rng.integers(1, 1 << 40))
        N = [1, 2, 3, 1 << 12, 1 << 15, (1 << 32) - 1, 1 << 32, (1 << 32) + 7][int(rng.integers(0, 8))]
        rows.append((a, b, e, N))
    return [np.array([r[i] for r in rows], dtype=np.uint64) for i in range(4)]


@pytest.mark.parametrize("algo", ["regular", "regular_unrolled"])
@pytest.mark.parametrize("kind", ["random", "adversarial", "grid"])
def test_search_verdicts_lockstep_form_vs_oracle(algo, kind):
    """hrb_search_verdicts (the phases' lockstep form: round-down FP32
    quotient estimates, exact path entered by warp vote) equals the oracle
    port of _regular_core / _regular_unrolled_core on (verdict, d, it)."""
    from paper_1211_3056_b200.device import search_verdict_arrays

    rng = np.random.default_rng(99 + (algo == "regular_unrolled") + 7 * ["random", "adversarial", "grid"].index(kind))
    W = 64
    if kind == "random":
        n = 1 << 21
        a = rng.integers(0, 2**64, n, dtype=np.uint64)
        b = rng.integers(0, 2**64, n, dtype=np.uint64)
        e = rng.integers(1, 2**40, n, dtype=np.uint64)
        N = rng.choice(np.array([1, 2, 17, 1 << 12, 1 << 15, 1 << 20, (1 << 31) + 5], dtype=np.uint64), n)
    elif kind == "adversarial":
        a, b, e, N = _adversarial_problems(rng, 1 << 17)
    else:  # criterion-2 grid embedded << 54
        grid = 1 << 10
        A, B = np.meshgrid(np.arange(grid, dtype=np.uint64), np.arange(grid, dtype=np.uint64), indexing="ij")
        a, b = A.ravel() << np.uint64(54), B.ravel() << np.uint64(54)
        e = np.full(a.size, (grid >> 6) << 54, dtype=np.uint64)
        N = np.full(a.size, 1024, dtype=np.uint64)
    ok, d, it = search_verdict_arrays(ALGO_CODE[algo], W, a, b, e, N)
    wok, wd, wit, _, _ = oracle.search_batch(algo, 1, 1 << 64, a, b, e, N)
    bad = np.nonzero((ok != wok) | (d != wd) | (it != wit))[0]
    assert bad.size == 0, [(int(a[k]), int(b[k]), int(e[k]), int(N[k])) for k in bad[:3]]


def test_search_verdicts_w32_vs_reference_goldens():
    from paper_1211_3056_b200.device import search_verdict_arrays

    g = load_search("search_w32.npz")
    for col, (algo, mode) in enumerate(CORE_COLUMNS):
        if not algo.startswith("regular"):
            continue
        ok, d, it = search_verdict_arrays(ALGO_CODE[algo], 32, g["a"], g["b"], g["eps"], g["count"])
        assert np.array_equal(ok, g["ok"][:, col]) and np.array_equal(d, g["d"][:, col])
        assert np.array_equal(it, g["it"][:, col])


def test_full_size_bench_slice_equals_oracle():
    """BASELINE configs[2] at its full per-GPU size (2^40 exp arguments,
    65,536 super-domains, 2^25 domains): the device funnel's counts, failing
    ids and candidates equal the CPU oracle's, and 8 logical shards of the
    same slice reproduce them in order (size-independent properties)."""
    import os

    from paper_1211_3056_b200.device import DeviceSlice, FusedRunner
    from paper_1211_3056_b200.shard import partition_blocks
    from paper_1211_3056_b200.slices import slice_view

    oracle.set_threads(os.cpu_count() or 1)
    batch, cfg = _big_slice("exp", 0, 40, 32)
    run = FusedRunner(DeviceSlice(batch), 2, 1, 8, sub_cap=batch.n_total // 4, cand_cap=1 << 16)
    run.launch()
    r = run.result()
    fails = oracle.phase1(batch, "regular", 1)
    assert np.array_equal(r.fail_ids + np.uint64(batch.id0), fails)
    rows = oracle.phase2(batch, "regular", 1, 8, fails)
    m, dist, dom = oracle.phase3(batch, rows)
    assert len(r.sub_keys) == len(rows[0])
    assert np.array_equal(r.cand_index, m) and np.array_equal(r.cand_dist, dist)
    cands = []
    for t0, t1 in partition_blocks([s.count for s in batch.supers], 8):
        sub = slice_view(batch, t0, t1)
        fr = FusedRunner(DeviceSlice(sub), 2, 1, 8, sub_cap=sub.n_total // 4, cand_cap=1 << 16)
        fr.launch()
        cands.append(fr.result().cand_index)
    assert np.array_equal(np.concatenate(cands), m)


def test_run_range_intervals_equal_one_slice_and_switch_algorithms():
    """run_range cuts the planned block schedule into intervals: records
    equal one run_slice of the whole range (and the reference's golden
    records), and "auto" picks each interval's search from the previous
    interval's funnel."""
    from dataclasses import replace

    from paper_1211_3056_b200.funnel import run_range, run_slice

    c = case("p53_exp_2p20_e16_N12")
    cfg = config_of(c)
    lo, cnt = c["slice"]
    whole = run_slice(c["fn"], c["binade"], lo, cnt, cfg)
    out = run_range(c["fn"], c["binade"], lo, cnt, cfg, interval_args=1 << 18, workers=2)
    assert essence(out.records) == essence(whole.records) == c["records"]
    assert len(out.interval_stats) == 4
    auto = replace(cfg, phase=replace(cfg.phase, algorithm="auto"))
    out2 = run_range(c["fn"], c["binade"], lo, cnt, auto, interval_args=1 << 18, workers=2)
    assert essence(out2.records) == c["records"]
    assert out2.choices[0][1] == "regular"  # no previous interval
    for k in range(1, len(out2.choices)):
        ratio = out2.interval_stats[k - 1].phase3_phase1_ratio()
        assert out2.choices[k][1] == ("lefevre" if ratio > 1e-3 else "regular")


def test_host_path_first_call_in_fresh_process():
    """hrb_run_slice_host as the first call of a process (unsized workspace:
    its allocations happen while the streamed upload is in flight) must
    neither deadlock nor differ from the phase path."""
    import subprocess
    import sys

    code = (
        "import numpy as np\n"
        "from golden_io import batch_of, case\n"
        "from paper_1211_3056_b200.device import DeviceSlice, run_host, run_phases\n"
        "c = case('p16_exp_b1')\n"
        "b = batch_of(c)\n"
        "counts, fail, cm, cd, cdom, ms = run_host(b, 2, 1, c['cfg']['split'])\n"
        "ref = run_phases(DeviceSlice(b), 2, 1, c['cfg']['split'])\n"
        "assert np.array_equal(fail, ref.fail_ids) and np.array_equal(cm, ref.cand_index)\n"
        "assert np.array_equal(cd, ref.cand_dist) and np.array_equal(cdom, ref.cand_dom)\n"
        "print('ok')\n")
    import os

    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.dirname(__file__), os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), os.environ.get("PYTHONPATH", "")]))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("algo", ["lefevre", "regular"])
def test_phase1_iteration_sums_equal_oracle(algo, mode):
    """The fused phase 1's SearchOutcome.iterations sum (per division mode
    for the classic family: the batched-run counting of lowerbound.py:
    170-222) equals the oracle cores' over the same Boolean problems, which
    are rebuilt here from the oracle's own tabulated residues."""
    from paper_1211_3056_b200.device import DeviceSlice, FusedRunner

    batch, _ = _big_slice("exp", 1 << 40, 24, 14, algo, N=1 << 10, super_log2=16)
    fused = FusedRunner(DeviceSlice(batch), ALGO_CODE[algo], mode, 8, sub_cap=batch.n_total * 16, cand_cap=1 << 20)
    fused.launch()
    r = fused.result()
    fails, coef = oracle.phase1(batch, algo, mode, with_coeffs=True)
    n = batch.n_total
    t, _ = batch.locate(np.arange(n, dtype=np.uint64))
    sizes = batch.domain_sizes(np.arange(n, dtype=np.uint64))
    a = np.zeros(n, np.uint64)
    b = np.zeros(n, np.uint64)
    e = np.zeros(n, np.uint64)
    for g in range(n):
        s0 = int(coef[0, 0, g]) | (int(coef[0, 1, g]) << 64)
        s1 = int(coef[1, 0, g]) | (int(coef[1, 1, g]) << 64)
        tt = int(t[g])
        G = int(batch.G[0, tt]) | (int(batch.G[1, tt]) << 64)
        s2 = int(batch.s2abs[0, tt]) | (int(batch.s2abs[1, tt]) << 64)
        a[g], b[g], e[g] = oracle.boolean_problem(s0, s1, G, s2, int(sizes[g]), batch.frac_bits, batch.word_bits)
    ok, _, it, _, _ = oracle.search_batch(algo, mode, 1 << batch.word_bits, a, b, e, sizes)
    if algo == "regular_unrolled":
        it = (it + 1) // 2
    assert np.array_equal(r.fail_ids + np.uint64(batch.id0), fails)
    assert int((~ok.astype(bool)).sum()) == len(fails)
    assert r.iterations == int(it.astype(np.uint64).sum()), (algo, mode)
