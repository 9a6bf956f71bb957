"""Multi-GPU sharding of an argument range: one process per GPU.

The reference has no distributed layer (its only
parallelism is the order-preserving ThreadPool of pipeline.py:204-210; the
paper's CPU baseline used MPI with a cyclic interval distribution,
PAPER.md:2155-2160).  Here the argument range is cut into contiguous runs of
the reference's super-domain blocks -- the _build_tasks schedule of
pipeline.py:374-409, planned ONCE for the whole range on every rank so that
block boundaries and global domain ids are exactly those of a single-process
run -- and every rank runs its run of blocks on its own GPU with no
communication.  At the end one collective gathers the per-rank counters and
the (small) candidate / record lists in rank order, which is argument order
because the shards are contiguous.  With an NCCL process
group that gather runs over NVLink/NVSwitch; the CPU tests drive the same
code with gloo.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from .arith import UFrac
from .fpformat import HrCaseRecord

M64 = (1 << 64) - 1
N_COUNTERS = 6  # phase-1 fails, phase-2 survivors, candidates, records, quotient steps, arguments


def partition_blocks(block_sizes: Sequence[int], world: int) -> list[tuple[int, int]]:
    """Contiguous [b0, b1) block ranges per rank, balanced by arguments:
    rank r ends at the first block boundary at or past r+1 of `world` equal
    shares.  Ranks may get an empty range when there are fewer blocks than
    ranks."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    sizes = np.asarray(block_sizes, dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(sizes)])
    total = cum[-1]
    out, b0 = [], 0
    for r in range(world):
        if r == world - 1:
            b1 = len(sizes)
        else:
            target = total * (r + 1) / world
            b1 = int(np.searchsorted(cum, target, side="left"))
            b1 = min(max(b1, b0), len(sizes))
        out.append((b0, b1))
        b0 = b1
    return out


@dataclass
class ShardResult:
    """What one rank contributes to the end-of-run gather.  Candidate and
    record arguments are float_bits patterns (fpmodel.py:126-137; up to 80
    bits for binary64, so carried as hi/lo words), distances raw 2^-64
    units, domain ids global."""

    counters: np.ndarray                      # int64 [N_COUNTERS]
    cand: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), np.uint64))  # (arg hi, arg lo, dist, dom)
    records: np.ndarray = field(default_factory=lambda: np.zeros((0, 5), np.uint64))  # + undecided

    @staticmethod
    def rows(records, with_flag: bool) -> np.ndarray:
        k = 5 if with_flag else 4
        out = [[r.argument >> 64, r.argument & M64, r.distance.raw, r.domain_id] + ([int(r.undecided)] if with_flag
                                                                                     else []) for r in records]
        return np.array(out, dtype=np.uint64).reshape(-1, k)

    @staticmethod
    def of(fails: int, subs: int, cands, records, iterations: int, arguments: int) -> "ShardResult":
        c = ShardResult.rows(cands, False)
        rec = ShardResult.rows(records, True)
        ctr = np.array([fails, subs, len(c), len(rec), iterations, arguments], dtype=np.int64)
        return ShardResult(ctr, c, rec)

    def record_objects(self) -> list[HrCaseRecord]:
        return [HrCaseRecord((int(h) << 64) | int(lo), UFrac(int(d), 64), int(i), bool(u))
                for h, lo, d, i, u in self.records.tolist()]

    def candidate_objects(self) -> list[HrCaseRecord]:
        return [HrCaseRecord((int(h) << 64) | int(lo), UFrac(int(d), 64), int(i))
                for h, lo, d, i in self.cand.tolist()]


def _gather_rows(dist, rows: np.ndarray, counts: list[int], device, group) -> np.ndarray:
    """All-gather a [n_r, k] uint64 array of variable length per rank (padded
    to the max count), concatenated in rank order."""
    import torch

    k = rows.shape[1]
    world = len(counts)
    m = max(max(counts), 1)
    pad = np.zeros((m, k), dtype=np.uint64)
    pad[: len(rows)] = rows
    t = torch.from_numpy(pad.view(np.int64)).to(device)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    parts = [b.cpu().numpy().view(np.uint64)[: counts[r]] for r, b in enumerate(bufs)]
    return np.concatenate(parts, axis=0) if parts else np.zeros((0, k), np.uint64)


def gather_shards(local: ShardResult, group=None, device=None) -> tuple[ShardResult, np.ndarray]:
    """End-of-run collective: counters, then candidates and records, all
    gathered to every rank in rank (= argument) order.  Returns the merged
    result (summed counters) and the per-rank counter matrix [world, K]."""
    import torch
    import torch.distributed as dist

    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
            else torch.device("cpu")
    world = dist.get_world_size(group)
    ctr = torch.from_numpy(local.counters.astype(np.int64)).to(device)
    allc = [torch.empty_like(ctr) for _ in range(world)]
    dist.all_gather(allc, ctr, group=group)
    per_rank = np.stack([c.cpu().numpy() for c in allc])
    cand = _gather_rows(dist, local.cand, per_rank[:, 2].astype(int).tolist(), device, group)
    rec = _gather_rows(dist, local.records, per_rank[:, 3].astype(int).tolist(), device, group)
    return ShardResult(per_rank.sum(axis=0), cand, rec), per_rank


def merge_shards(parts: Sequence[ShardResult]) -> ShardResult:
    """Rank-ordered merge (what gather_shards computes, without a process
    group): summed counters, concatenated candidate and record rows."""
    return ShardResult(np.sum([p.counters for p in parts], axis=0),
                       np.concatenate([p.cand for p in parts], axis=0),
                       np.concatenate([p.records for p in parts], axis=0))


def _run_rank(plan, rank, world, fn, binade, cfg, algo, workers, confirm) -> ShardResult:
    from .funnel import _resolve, execute_batch
    from .slices import pack_plan

    b0, b1 = partition_blocks(plan.sizes, world)[rank]
    if b1 <= b0:
        return ShardResult(np.zeros(N_COUNTERS, np.int64))
    ceiling = cfg.phase.budgets.eps_dprime if cfg.phase.budgets is not None else None
    batch = pack_plan(plan[b0:b1], cfg.word_bits, budget_ceiling=ceiling, workers=workers)
    out = execute_batch(batch, cfg, _resolve(cfg, algo), fn, confirm=confirm, workers=workers)
    return ShardResult.of(len(out.fail_global), len(out.sub_table[0]), out.candidates, out.records,
                          out.iterations, batch.arguments)


def run_logical_shards(fn: str, binade: int, start: int, count: int, cfg, world: int, algo: str | None = None,
                       workers: int = 1, confirm: bool = True) -> tuple[ShardResult, np.ndarray]:
    """Single-GPU stand-in for a `world`-rank run: the same partition, the
    shards run one after another on the current device, merged in rank
    order (tests the shard boundaries without 8 GPUs)."""
    from .slices import plan_arrays

    plan = plan_arrays(fn, binade, cfg.fmt, cfg.polygen, start, count)
    parts = [_run_rank(plan, r, world, fn, binade, cfg, algo, workers, confirm) for r in range(world)]
    return merge_shards(parts), np.stack([p.counters for p in parts])


def run_sharded(fn: str, binade: int, start: int, count: int, cfg, algo: str | None = None, rank: int = 0,
                world: int = 1, workers: int = 1, group=None, confirm: bool = True):
    """The funnel over [start, start+count) of one binade, split across the
    ranks of `group`; this rank runs its contiguous share on the current
    CUDA device.  Returns (merged ShardResult, per-rank counters) on every
    rank; records are confirmed on the rank that found them."""
    from .slices import plan_arrays

    plan = plan_arrays(fn, binade, cfg.fmt, cfg.polygen, start, count)
    local = _run_rank(plan, rank, world, fn, binade, cfg, algo, workers, confirm)
    if world == 1:
        return local, local.counters[None, :]
    return gather_shards(local, group)
