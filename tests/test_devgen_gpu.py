"""Native generation on the device (hrb_pack_blocks): one GPU thread per
super-domain runs csrc/host/polygen.h, the same source as libhrbhost.so's
hrbh_pack_blocks.  Pinned to the reference's own fixtures (the packed
super-domains the reference computed) and, column for column, to the host
library on random configurations, fallback flags included."""
import random

import numpy as np
import pytest

from golden_io import batch_of, case, config_of, pipeline_cases

from paper_1211_3056_b200 import hostgen, slices
from paper_1211_3056_b200.fpformat import FpFormat
from paper_1211_3056_b200.taylor import PolyGenConfig

pytestmark = pytest.mark.gpu

PACKED = ("coef", "G", "s2abs", "n_dom", "dom_n", "last_n", "dom_base", "m0")


@pytest.mark.parametrize("name", [c["name"] for c in pipeline_cases() if c["fn"] == "exp" and c["binade"] <= 0])
def test_device_pack_equals_reference_fixture(name):
    c = case(name)
    cfg = config_of(c)
    want = batch_of(c)
    start, count = c["slice"]
    plan = slices.plan_arrays(c["fn"], c["binade"], cfg.fmt, cfg.polygen, start, count)
    got = slices.pack_plan(plan, cfg.word_bits, workers=1, native=True, device=True)
    for k in PACKED:
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    assert np.array_equal(got.shift_bound_ok, want.shift_bound_ok)


def _random_plan(rng):
    p = rng.choice([24, 32, 53, 53, 64])
    eps_bits = rng.randint(8, 40)
    fmt = FpFormat(p, eps_bits)
    N = 1 << rng.randint(6, 15)
    tau = 1 << rng.randint(1, 9)
    mu = 1 << rng.randint(0, tau.bit_length() - 1)
    delta = rng.choice([1, 2, 2])
    F = rng.choice([48, 64, 96, 112, 128])
    W = rng.choice([32, 64]) if F >= 64 else 32
    pg = PolyGenConfig(tau=tau, N=N, mu=mu, nu=tau // mu, delta=delta, limbs=rng.randint(2, 12), frac_bits=F,
                       guard=rng.choice([0, 8, 32, 64]))
    binade = rng.choice([0, 0, -1, -7, -60])
    span = 1 << (p - 1)
    count = min(span, rng.randint(1, 1 << 12) * N * tau // rng.choice([1, 3, 7]))
    start = rng.randrange(0, span - count + 1)
    return slices.plan_arrays("exp", binade, fmt, pg, start, count), fmt, pg, binade, W


@pytest.mark.parametrize("seed", range(40))
def test_device_columns_equal_host_library(seed):
    from paper_1211_3056_b200.device import pack_columns_device

    rng = random.Random(7000 + seed)
    plan, fmt, pg, binade, W = _random_plan(rng)
    if not len(plan):
        pytest.skip("empty plan")
    cfg = hostgen.make_cfg("exp", fmt, pg, binade, W)
    cols = (plan.bstart, plan.bcount, plan.n_p, plan.tau, plan.e_out)
    host = hostgen.pack_columns(cfg, *cols, 1)
    dev = pack_columns_device(cfg, *cols)
    for name, h, d in zip(("coef", "G", "s2abs", "status", "shift_ok"), host, dev):
        if name in ("coef", "G", "s2abs", "shift_ok"):  # fallback columns are unspecified
            ok = host[3] == hostgen.HRBH_OK
            h, d = h[..., ok], d[..., ok]
        assert np.array_equal(h, d), (seed, name)


def test_device_columns_at_2p36():
    """4,096 super-domains (the C4/C5 slice size) and the 2^40 bench slice's
    first 8,192 blocks: device == host library."""
    from paper_1211_3056_b200.device import pack_columns_device

    fmt = FpFormat(53, 32)
    pg = PolyGenConfig(tau=512, N=1 << 15, mu=16, nu=32, delta=2, limbs=8, frac_bits=96, guard=32)
    for start, count in ((0, 1 << 36), (1 << 45, 1 << 37)):
        plan = slices.plan_arrays("exp", 0, fmt, pg, start, count)
        cfg = hostgen.make_cfg("exp", fmt, pg, 0, 64)
        cols = (plan.bstart, plan.bcount, plan.n_p, plan.tau, plan.e_out)
        host = hostgen.pack_columns(cfg, *cols, 0)
        dev = pack_columns_device(cfg, *cols)
        assert (host[3] == hostgen.HRBH_OK).all()
        for h, d in zip(host, dev):
            assert np.array_equal(h, d)


@pytest.mark.parametrize("seed", [6, 14, 21, 25, 28, 32, 35, 38, 1, 9])
def test_pack_plan_device_raises_like_host(seed):
    """pack_plan on the device hands the blocks it flags to the exact Python
    path, which raises the reference's error where the reference raises
    (MPOverflowError here) -- the same exception and message as the host
    library's pack_plan -- and otherwise returns the same slice."""
    rng = random.Random(7000 + seed)
    plan, fmt, pg, binade, W = _random_plan(rng)

    def run(device):
        try:
            return slices.pack_plan(plan, W, workers=1, native=True, device=device), None
        except Exception as exc:  # noqa: BLE001 - compared below
            return None, (type(exc).__name__, str(exc))

    got, gerr = run(True)
    want, werr = run(False)
    assert gerr == werr
    if want is not None:
        for k in PACKED:
            assert np.array_equal(getattr(got, k), getattr(want, k)), k
        assert np.array_equal(got.shift_bound_ok, want.shift_bound_ok)


@pytest.mark.parametrize("seed,flag_every", [(0, 0), (2, 7), (5, 0), (11, 3), (22, 0), (27, 1)])
def test_pack_plan_resident_columns(seed, flag_every, monkeypatch):
    """pack_plan(resident=True): the device columns it keeps for the search
    equal the host slice, and the host copies landing behind it equal the
    plain pack once waited for.  flag_every > 0 marks every k-th block as a
    fallback (and zeroes its device columns): the exact Python path redoes
    those rows and the patched columns must reach the device too."""
    from paper_1211_3056_b200 import device as devmod

    rng = random.Random(7000 + seed)
    plan, fmt, pg, binade, W = _random_plan(rng)
    want = slices.pack_plan(plan, W, workers=1, native=True, device=False)
    if flag_every:
        real = devmod.pack_columns_device

        def flagged(*a, **k):
            out = real(*a, **k)
            status, res = out[3], out[5]
            status[::flag_every] = hostgen.HRBH_FALLBACK
            res.coef[:, :, ::flag_every] = 0
            res.G[:, ::flag_every] = 0
            res.s2abs[:, ::flag_every] = 0
            return out

        monkeypatch.setattr(devmod, "pack_columns_device", flagged)
    got = slices.pack_plan(plan, W, workers=1, native=True, device=True, resident=True)
    r = got.resident
    assert r is not None
    r.wait()
    for k in PACKED:
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    assert np.array_equal(r.coef.cpu().numpy().view(np.uint32), want.coef)
    assert np.array_equal(r.G.cpu().numpy().view(np.uint64), want.G)
    assert np.array_equal(r.s2abs.cpu().numpy().view(np.uint64), want.s2abs)


@pytest.mark.parametrize("eps_bits,log2_count", [(32, 30), (14, 24), (20, 27)])
def test_resident_run_equals_host_buffer_run(eps_bits, log2_count):
    """hrb_run_slice_resident on the generated device columns (run_range's
    path) == hrb_run_slice_host on the host slice: counts (phases' outputs and
    arguments covered), candidates, records."""
    from paper_1211_3056_b200 import FpFormat, PhaseConfig, PipelineConfig
    from paper_1211_3056_b200.funnel import execute_batch_host

    N = 1 << 12
    pg = PolyGenConfig(tau=64, N=N, mu=8, nu=8, delta=2, limbs=8, frac_bits=96, guard=32)
    cfg = PipelineConfig("exp", FpFormat(53, eps_bits), pg, PhaseConfig("regular", phase2_split=8, N1=N))
    plan = slices.plan_arrays("exp", 0, cfg.fmt, pg, 12345 << 20, 1 << log2_count)
    host = slices.pack_plan(plan, 64, workers=2, device=False)
    res = slices.pack_plan(plan, 64, workers=2, device=True, resident=True)
    a = execute_batch_host(host, cfg, "regular", workers=2)
    b = execute_batch_host(res, cfg, "regular", workers=2)
    assert res.resident is None
    assert a.records == b.records
    assert a.iterations == b.iterations
    assert [(r.phase, r.domains_in, r.domains_out, r.arguments_covered) for r in a.stats.rows] == \
           [(r.phase, r.domains_in, r.domains_out, r.arguments_covered) for r in b.stats.rows]
    assert a.candidates == b.candidates and len(a.candidates) > 0
    for k in PACKED:
        assert np.array_equal(getattr(res, k), getattr(host, k)), k


def test_run_range_resident_intervals_equal_host_generation():
    """run_range over 4 intervals with the device generation (each interval
    prepared in the worker thread behind the previous one's search, searched
    in place) == one host-generated, host-buffer slice of the whole range."""
    from paper_1211_3056_b200 import FpFormat, PhaseConfig, PipelineConfig
    from paper_1211_3056_b200.funnel import execute_batch_host, run_range

    N = 1 << 12
    pg = PolyGenConfig(tau=64, N=N, mu=8, nu=8, delta=2, limbs=8, frac_bits=96, guard=32)
    cfg = PipelineConfig("exp", FpFormat(53, 20), pg, PhaseConfig("regular", phase2_split=8, N1=N))
    start, count = 777 << 30, 1 << 33
    plan = slices.plan_arrays("exp", 0, cfg.fmt, pg, start, count)
    assert len(plan) // 4 >= slices.DEVICE_GEN_MIN
    whole = execute_batch_host(slices.pack_plan(plan, 64, workers=2, device=False), cfg, "regular", workers=2)
    out = run_range("exp", 0, start, count, cfg, interval_args=count // 4, workers=2)
    assert len(out.interval_stats) == 4
    assert out.records == whole.records and len(whole.records) > 0
    for k in range(3):  # phases' domains out and arguments covered add up
        assert sum(st.rows[k].domains_out for st in out.interval_stats) == whole.stats.rows[k].domains_out
        assert sum(st.rows[k].arguments_covered for st in out.interval_stats) == whole.stats.rows[k].arguments_covered
