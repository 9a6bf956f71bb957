"""Public drop-ins that the phase tests do not reach: the reference-signature
domain_coefficient_sets, the multi-rank run_sharded (two processes sharing
cuda:0 over gloo), and measure_warps."""
import os
import socket

import numpy as np
import pytest

from golden_io import case, config_of, supers_of

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["p13_exp_b0", "p53_exp_2p20_e16_N15", "p53_exp_ragged", "p53_exp_delta1",
                                  "p13_log_b0"])
def test_domain_coefficient_sets_reference_signature(name):
    """domain_coefficient_sets(r_polys, cfg) with the reference's own r_polys
    and a PolyGenConfig of each super-domain equals the values the
    reference's domain_coefficient_sets produced (tests/golden)."""
    from paper_1211_3056_b200 import domain_coefficient_sets
    from paper_1211_3056_b200.taylor import PolyGenConfig

    c = case(name)
    k = c["cfg"]
    by_id = {d[0]: d for d in c["domains"]}
    for sd in supers_of(c):
        pg = PolyGenConfig(tau=sd.tau, N=sd.n_p, mu=sd.mu, nu=sd.nu, delta=k["delta"], limbs=k["limbs"],
                           frac_bits=k["frac_bits"], guard=k["guard"])
        sets = domain_coefficient_sets(sd.r_polys, pg)
        assert len(sets) == sd.tau
        for i, tup in enumerate(sets):
            want = by_id[sd.dom_id0 + i][3:3 + k["delta"] + 1]
            assert [x.to_int() for x in tup] == [int(h, 16) for h in want], (name, sd.dom_id0 + i)
            assert all(x.limb_count == k["limbs"] for x in tup)


def test_domain_coefficient_sets_overflow_raises():
    from paper_1211_3056_b200 import domain_coefficient_sets
    from paper_1211_3056_b200.arith import MPOverflowError
    from paper_1211_3056_b200.taylor import BinomialPoly, PolyGenConfig

    pg = PolyGenConfig(tau=16, N=64, mu=4, nu=4, delta=2, limbs=2, frac_bits=64, guard=0)
    big = (1 << 63) + 12345
    with pytest.raises(MPOverflowError):
        domain_coefficient_sets([BinomialPoly((big, big, big)), BinomialPoly((big, big)), BinomialPoly((big,))], pg)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_worker(rank, world, port, name, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist

    from golden_io import case as _case, config_of as _config_of
    from paper_1211_3056_b200.shard import run_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = _case(name)
        start, count = c["slice"]
        merged, per_rank = run_sharded(c["fn"], c["binade"], start, count, _config_of(c), rank=rank, world=world,
                                       workers=2)
        q.put((rank, merged.counters.tolist(), merged.records.tolist(), per_rank.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("p53_exp_2p20_e16_N12", 2), ("p16_exp_b1", 3)])
def test_run_sharded_two_ranks_on_one_gpu(name, world):
    """run_sharded with `world` processes on cuda:0 (gloo for the end-of-run
    gather): the merged records equal a single run_slice's, and the
    reference's records."""
    import torch.multiprocessing as mp

    from paper_1211_3056_b200.funnel import run_slice

    c = case(name)
    start, count = c["slice"]
    whole = run_slice(c["fn"], c["binade"], start, count, config_of(c), workers=2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = [[r.argument >> 64, r.argument & ((1 << 64) - 1), r.distance.raw, r.domain_id, int(r.undecided)]
            for r in whole.records]
    ref = [[int(a, 16) >> 64, int(a, 16) & ((1 << 64) - 1), d, dom, int(u)] for a, d, dom, u in c["records"]]
    for rank, counters, records, per_rank in got:
        assert records == want == ref
        assert counters[0] == len(whole.fail_global) and counters[2] == len(whole.candidates)
        assert len(per_rank) == world and sum(r[5] for r in per_rank) == count


def test_measure_warps_matches_oracle_iterations():
    """measure_warps (iteration counts from one hrb_search_batch launch,
    summarised per warp) equals the CPU oracle's per-lane iteration counts
    (SearchOutcome.iterations, lowerbound.py) with the reference's exact
    nmdm per warp (divergence.py:96-110)."""
    import oracle
    from paper_1211_3056_b200.divergence import measure_warps, nmdm

    rng = np.random.default_rng(5)
    n = 32 * 64
    a = rng.integers(1, 1 << 63, n, dtype=np.uint64)
    b = rng.integers(0, 1 << 63, n, dtype=np.uint64)
    eps = np.full(n, 1 << 20, dtype=np.uint64)
    N = np.full(n, 1 << 15, dtype=np.uint64)
    for algo in ("regular", "lefevre"):
        s = measure_warps(a, b, eps, N, algo)
        it = oracle.search_batch(algo, 1, 1 << 64, a, b, eps, N)[2].astype(np.int64)
        assert np.array_equal(s.lane_iterations.astype(np.int64), it)
        want = [float(nmdm(it[w * 32:(w + 1) * 32].tolist())) for w in range(n // 32)]
        assert np.allclose(s.warp_nmdm, want, rtol=0, atol=1e-12)
        assert len(s.warp_max) == n // 32


@pytest.mark.parametrize("p,eps_bits,binade", [(53, 16, 0), (53, 32, 0), (53, 20, -1), (24, 12, 0), (13, 6, -2)])
def test_device_confirmation_equals_host_and_decide_hr(p, eps_bits, binade):
    """hrb_confirm_exp (the device running csrc/host/decide.h) gives the
    host library's decisions and distances, which equal decide_hr's; plus
    arguments near HR (from the reference's own candidates) at p = 53."""
    from paper_1211_3056_b200 import hostgen
    from paper_1211_3056_b200.enclosure import decide_hr
    from paper_1211_3056_b200.fpformat import FpFormat, bits_float
    from paper_1211_3056_b200.arith import UFrac
    from paper_1211_3056_b200.funnel import confirm_on_device
    from paper_1211_3056_b200.taylor import PolyGenConfig

    fmt = FpFormat(p, eps_bits)
    rng = np.random.default_rng(p * 100 + eps_bits)
    idx = rng.integers(0, 1 << (p - 1), 20000, dtype=np.uint64)
    if p == 53 and binade == 0:
        c = case("p53_exp_2p20_e16_N15")
        idx = np.concatenate([idx, np.array([int(a, 16) & ((1 << 52) - 1) for a, _, _ in c["phase3"]],
                                            dtype=np.uint64)])
    d_is, d_dist, d_st = confirm_on_device(fmt, binade, idx)
    assert (d_st == 0).all()
    cfg = hostgen.make_cfg("exp", fmt, PolyGenConfig(), binade, 64)
    h_is, h_dist, h_st = hostgen.confirm(cfg, idx, 4)
    assert np.array_equal(d_is, h_is) and np.array_equal(d_dist[d_is == 1], h_dist[h_is == 1])
    for k in list(np.flatnonzero(d_is))[:40] + list(range(0, len(idx), 997)):
        arg = ((binade + 1 + (1 << 15)) << (p - 1)) | int(idx[k])
        dec = decide_hr("exp", bits_float(arg, fmt), fmt, start_prec=2 * (p + eps_bits) + 16)
        assert bool(d_is[k]) == dec.is_hr
        if dec.is_hr:
            assert int(d_dist[k]) == UFrac.from_fraction(dec.distance_lo).raw
