"""Multi-rank sharding on CPU (gloo, world size 2): the partition of the
reference's block schedule and the end-of-run gather.  Each rank computes
its shard with the CPU oracle (test infrastructure standing in for the GPU,
which these CPU tests do not have); the merged, rank-ordered result must
equal the single-process result of the whole range and the reference's
golden candidates."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from golden_io import case, config_of, supers_of
from paper_1211_3056_b200.fpformat import index_bits
from paper_1211_3056_b200.shard import N_COUNTERS, ShardResult, gather_shards, partition_blocks
from paper_1211_3056_b200.slices import pack_slice


def test_partition_is_contiguous_and_balanced():
    sizes = [1 << 24] * 65536
    parts = partition_blocks(sizes, 8)
    assert parts[0][0] == 0 and parts[-1][1] == len(sizes)
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    assert {p[1] - p[0] for p in parts} == {8192}
    ragged = [5, 1, 1, 1, 9, 2, 2]
    parts = partition_blocks(ragged, 3)
    assert parts[0][0] == 0 and parts[-1][1] == len(ragged)
    assert sum(p[1] - p[0] for p in parts) == len(ragged)
    assert partition_blocks([3], 4) == [(0, 1), (1, 1), (1, 1), (1, 1)]
    with pytest.raises(ValueError):
        partition_blocks(sizes, 0)


def _oracle_shard(c, supers, p):
    cfg = config_of(c)
    if not supers:
        return ShardResult(np.zeros(N_COUNTERS, np.int64))
    batch = pack_slice(supers, cfg.fmt, cfg.polygen, cfg.word_bits, c["binade"])
    algo = c["cfg"]["algorithm"]
    mode = {"sub": 0, "hybrid": 1, "hw": 2}[c["cfg"]["div_mode"]]
    fails = oracle.phase1(batch, algo, mode)
    rows = oracle.phase2(batch, algo, mode, c["cfg"]["split"], fails)
    m, dist, dom = oracle.phase3(batch, rows)
    bits = [index_bits(c["binade"], int(x), cfg.fmt) for x in m]
    cand = np.array([[b >> 64, b & ((1 << 64) - 1), int(d), int(i)] for b, d, i in zip(bits, dist, dom)],
                    dtype=np.uint64).reshape(-1, 4)
    ctr = np.array([len(fails), len(rows[0]), len(cand), 0, 0, batch.arguments], dtype=np.int64)
    return ShardResult(ctr, cand)


def _worker(rank, world, port, name, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = case(name)
        supers = supers_of(c)
        b0, b1 = partition_blocks([s.count for s in supers], world)[rank]
        local = _oracle_shard(c, supers[b0:b1], None)
        merged, per_rank = gather_shards(local)
        q.put((rank, merged.counters.tolist(), merged.cand.tolist(), per_rank.tolist()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,world", [("p53_exp_2p20_e16_N12", 2), ("p13_exp_b0", 2), ("p53_exp_ragged", 3)])
def test_gloo_sharded_run_equals_single_run(name, world):
    oracle.build()
    c = case(name)
    whole = _oracle_shard(c, supers_of(c), None)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_cand = [[int(h, 16) >> 64, int(h, 16) & ((1 << 64) - 1), d, i] for h, d, i in c["phase3"]]
    for rank, counters, cand, per_rank in got:
        assert counters == whole.counters.tolist()
        assert cand == whole.cand.tolist()
        assert cand == want_cand  # the reference's own phase-3 output, in order
        assert len(per_rank) == world and sum(r[5] for r in per_rank) == c["slice"][1]
