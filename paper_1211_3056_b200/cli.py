"""Command-line entry point, shaped like the reference's (cli.py:221-271).

    python -m paper_1211_3056_b200.cli search [reference flags]
        [--range START:COUNT] [--gpus N] [--degree D] [--interval LOG2]
        [--manifest PATH]
    python -m paper_1211_3056_b200.cli divergence [reference flags]

`search` keeps the reference's flags, defaults and streams: records as
JSONL / CSV on stdout (or --out), byte-identical to the reference's for the
same records (records.py, cli.py:116-138), phase statistics as CSV on stderr
(cli.py:141-149), exit codes 0 / 1 runtime / 2 configuration (cli.py:261-271).
Without --range it searches the whole binade (run_pipeline); the extensions:
- --range START:COUNT  argument indices [START, START+COUNT) of the binade,
  walked as intervals (funnel.run_range; --interval, resumable --manifest);
- --gpus N            N processes, one per GPU, contiguous shards, NCCL
  gather of records at the end (shard.run_sharded);
- --degree D          the Taylor degree: 1-2 as the reference, 3-8 the
  high-degree path (one model per large super-domain, wide.py).
The reference's oracle-check needs its exhaustive enumerator, which stays in
the test fixtures (tests/golden), not in this package.
"""

from __future__ import annotations

import argparse
import os
import sys

from .records import emit_records, emit_stats

DIV_MODES = ("sub", "hw", "hybrid")


class ConfigError(ValueError):
    pass


def _add_common_flags(sp: argparse.ArgumentParser) -> None:
    """The reference's common flags and defaults (cli.py:67-83)."""
    sp.add_argument("--fn", default="exp", help="exp | log | exp2")
    sp.add_argument("--p", type=int, default=13, help="target precision in bits")
    sp.add_argument("--eps-bits", type=int, default=8, help="HR threshold exponent: eps = 2^-eps_bits")
    sp.add_argument("--binade", type=int, default=0, help="input binade exponent: arguments in [2^b, 2^(b+1))")
    sp.add_argument("--domain-bits", type=int, default=4, help="log2 of the phase-1 domain size N")
    sp.add_argument("--div-mode", choices=sorted(DIV_MODES), default="hybrid")
    sp.add_argument("--word-bits", type=int, choices=(32, 64), default=64)
    sp.add_argument("--out", default=None, help="write records here instead of stdout")
    sp.add_argument("--format", choices=("jsonl", "csv"), default="jsonl")
    sp.add_argument("--seed", type=int, default=0, help="accepted; the search is deterministic")


def _pipeline_config(args):
    """The reference's default block shape (cli.py:86-113)."""
    from .arith import DivisionMode
    from .fpformat import FpFormat
    from .funnel import PhaseConfig, PipelineConfig
    from .taylor import PolyGenConfig

    modes = {"sub": DivisionMode.SUBTRACTIVE, "hw": DivisionMode.HARDWARE, "hybrid": DivisionMode.HYBRID}
    fmt = FpFormat(precision=args.p, eps_bits=args.eps_bits)
    n1 = 1 << args.domain_bits
    half = 1 << (args.p - 1)
    tau = max(1, min(16, half // n1))
    mu, nu = 1, tau
    for cand in (4, 2):
        if tau % cand == 0:
            mu, nu = cand, tau // cand
            break
    delta = min(args.degree, 2)
    pg = PolyGenConfig(tau=tau, N=n1, mu=mu, nu=nu, delta=delta, limbs=8, frac_bits=96, guard=32)
    if n1 % args.phase2_split:
        raise ConfigError(f"--phase2-split {args.phase2_split} must divide the domain size N = {n1}")
    phase = PhaseConfig(algorithm=args.algo, div_mode=modes[args.div_mode], phase2_split=args.phase2_split, N1=n1,
                        parallel_width=max(1, min(64, args.workers)))
    return PipelineConfig(fn=args.fn, fmt=fmt, polygen=pg, phase=phase, word_bits=args.word_bits)


def _range_of(args):
    if args.range is None:
        return 0, 1 << (args.p - 1)
    try:
        a, b = args.range.split(":")
        start, count = int(a, 0), int(b, 0)
    except ValueError:
        raise ConfigError(f"--range {args.range!r}: expected START:COUNT") from None
    if start < 0 or count < 1 or start + count > 1 << (args.p - 1):
        raise ConfigError(f"--range {args.range!r} is outside the binade's {1 << (args.p - 1)} arguments")
    return start, count


def _wide_config(args):
    if args.degree < 3:
        return None
    from .wide import WideGenConfig

    w = WideGenConfig.for_degree(args.degree, N=1 << args.domain_bits)
    if args.super_bits:
        w = WideGenConfig(args.degree, tau=max(1, (1 << args.super_bits) >> args.domain_bits),
                          N=1 << args.domain_bits)
    return w


def _merged_stats(interval_stats):
    from .funnel import PhaseRow, PhaseStats

    rows, order, choices = {}, [], []
    for st in interval_stats:
        for r in st.rows:
            if r.phase not in rows:
                order.append(r.phase)
                rows[r.phase] = [0, 0, 0, 0.0]
            acc = rows[r.phase]
            acc[0] += r.domains_in
            acc[1] += r.domains_out
            acc[2] += r.arguments_covered
            acc[3] += r.wall_ms
        choices.extend(st.algorithm_choices)
    return PhaseStats([PhaseRow(k, *rows[k]) for k in order], choices)


def _write(records, args):
    if args.out:
        with open(args.out, "w", encoding="utf-8", newline="") as fh:
            emit_records(records, args.format, fh)
    else:
        emit_records(records, args.format, sys.stdout)


def cmd_search(args) -> int:
    cfg = _pipeline_config(args)
    wide = _wide_config(args)
    if args.gpus > 1:
        return _search_multi_gpu(args, cfg, wide)
    from .funnel import run_pipeline, run_range

    if args.range is None and wide is None and args.manifest is None:
        records, stats = run_pipeline(args.binade, cfg)  # the reference's search (cli.py:152-161)
    else:
        start, count = _range_of(args)
        out = run_range(cfg.fn, args.binade, start, count, cfg, interval_args=1 << args.interval,
                        workers=args.workers, manifest=args.manifest, wide=wide)
        records, stats = out.records, _merged_stats(out.interval_stats)
    _write(records, args)
    emit_stats(stats, sys.stderr)
    return 0


def _rank_main(rank, world, port, args, q):
    import torch
    import torch.distributed as dist

    from .shard import run_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        cfg = _pipeline_config(args)
        start, count = _range_of(args)
        merged, per_rank = run_sharded(cfg.fn, args.binade, start, count, cfg, rank=rank, world=world,
                                       workers=max(1, args.workers))
        if rank == 0:
            q.put((merged.record_objects(), per_rank.tolist()))
    finally:
        dist.destroy_process_group()


def _search_multi_gpu(args, cfg, wide) -> int:
    import socket

    import torch
    import torch.multiprocessing as mp

    if wide is not None:
        raise ConfigError("--gpus > 1 runs the delta <= 2 path")
    if torch.cuda.device_count() < args.gpus:
        raise ConfigError(f"--gpus {args.gpus}: only {torch.cuda.device_count()} CUDA devices visible")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, args.gpus, port, args, q)) for r in range(args.gpus)]
    for p in procs:
        p.start()
    records, per_rank = q.get()
    for p in procs:
        p.join()
        if p.exitcode != 0:
            raise RuntimeError(f"rank process exited with {p.exitcode}")
    _write(records, args)
    import csv

    w = csv.writer(sys.stderr, lineterminator="\n")
    w.writerow(["rank", "phase1_fail", "phase2_survivors", "candidates", "records", "quotient_steps", "arguments"])
    for r, row in enumerate(per_rank):
        w.writerow([r, *row])
    return 0


def cmd_divergence(args) -> int:
    """The reference's divergence report (cli.py:188-218), with every
    lane's search run on the device (divergence.simulate_warps)."""
    import csv

    from .arith import DivisionMode
    from .divergence import linear_problem_batch, report_rows, simulate_warps
    from .fpformat import FpFormat
    from .search import Algorithm

    modes = {"sub": DivisionMode.SUBTRACTIVE, "hw": DivisionMode.HARDWARE, "hybrid": DivisionMode.HYBRID}
    fmt = FpFormat(precision=args.p, eps_bits=args.eps_bits)
    try:
        algo = Algorithm(args.algo)
    except ValueError:
        raise ConfigError(f"--algo {args.algo!r}: divergence needs one concrete algorithm, not auto") from None
    problems = linear_problem_batch(args.fn, fmt, args.binade, 1 << args.domain_bits, domain_count=args.count,
                                    word_bits=args.word_bits)
    report = simulate_warps(problems, algo, modes[args.div_mode], warp_width=args.warp_width)
    sink = open(args.out, "w", encoding="utf-8", newline="") if args.out else sys.stdout
    try:
        writer = csv.writer(sink, lineterminator="\n")
        writer.writerow(["warp_id", "max_iter", "mean_iter", "mdm", "nmdm"])
        for row in report_rows(report):
            writer.writerow([row[0], row[1], f"{row[2]:.6f}", f"{row[3]:.6f}", f"{row[4]:.6f}"])
    finally:
        if args.out:
            sink.close()
    summary = csv.writer(sys.stderr, lineterminator="\n")
    summary.writerow(["algorithm", "min_iterations", "max_iterations", "mean_iterations", "mean_nmdm"])
    summary.writerow([report.algorithm.value, report.min_iterations, report.max_iterations,
                      f"{float(report.mean_iterations):.6f}", f"{float(report.mean_nmdm):.6f}"])
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="hardround-b200",
                                     description="hard-to-round case search for elementary functions (B200)")
    sub = parser.add_subparsers(dest="command", required=True)
    sp = sub.add_parser("search", help="run the filtering pipeline on a binade or an argument range")
    _add_common_flags(sp)
    sp.add_argument("--phase2-split", type=int, default=8, help="subdomains per domain in phase 2")
    sp.add_argument("--algo", choices=("lefevre", "regular", "auto"), default="regular")
    sp.add_argument("--workers", type=int, default=os.cpu_count() or 1, help="host threads / processes")
    sp.add_argument("--range", default=None, help="START:COUNT argument indices of the binade (default: all)")
    sp.add_argument("--gpus", type=int, default=1, help="one process per GPU, contiguous shards")
    sp.add_argument("--degree", type=int, default=2, choices=range(1, 9), metavar="1..8",
                    help="Taylor degree: 1-2 as the reference, 3-8 the high-degree path")
    sp.add_argument("--super-bits", type=int, default=0, help="high-degree super-domain size (log2 arguments)")
    sp.add_argument("--interval", type=int, default=38, help="log2 arguments per run_range interval")
    sp.add_argument("--manifest", default=None, help="resumable JSON-lines manifest of finished intervals")
    sp.set_defaults(func=cmd_search)
    sp = sub.add_parser("divergence", help="warp divergence of the lower-bound searches (device traces)")
    _add_common_flags(sp)
    sp.add_argument("--algo", choices=("lefevre", "lefevre_swap", "regular", "regular_unrolled"), default="regular")
    sp.add_argument("--count", type=int, default=None, help="number of consecutive subdomains")
    sp.add_argument("--warp-width", type=int, default=32)
    sp.set_defaults(func=cmd_divergence)
    return parser


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    try:
        return args.func(args)
    except (ConfigError, ValueError) as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2
    except Exception as exc:  # noqa: BLE001 -- CLI boundary
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    raise SystemExit(main())
