"""Multi-GPU sharding logic, exercised on CPU with torch.distributed/gloo
(world_size 2): contiguous rank ranges cover the space exactly, and the
TopK / Histogram partials merged through the collectives equal the
single-process result (values from the CPU oracle stand in for the per-GPU
device output)."""

import itertools
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2501_03381_b200 import sharding


def test_rank_ranges_partition_the_space():
    for n, lo, hi in [(30, 2, 30), (20, 3, 20), (12, 1, 12)]:
        total = sum(math.comb(n, k) for k in range(lo, hi + 1))
        for world in (1, 2, 3, 4, 8):
            for weight in ("count", "flops"):
                rr = sharding.rank_ranges(n, lo, hi, world, weight)
                assert rr[0][0] == 0 and rr[-1][1] == total
                assert all(a <= b for a, b in rr)
                assert all(rr[i][1] == rr[i + 1][0] for i in range(world - 1))
            counts = [b - a for a, b in sharding.rank_ranges(n, lo, hi, world, "count")]
            assert max(counts) - min(counts) <= 1
    # flops balance: every shard within 1% of the mean cost
    rr = sharding.rank_ranges(30, 2, 30, 8, "flops")
    offs, _ = sharding.order_offsets(30, 2, 30)

    def cost(a, b):
        c, off = 0.0, 0
        for k in range(2, 31):
            n_k = math.comb(30, k)
            ov = max(0, min(b, off + n_k) - max(a, off))
            c += ov * sharding.nplet_flops(k)
            off += n_k
        return c

    costs = [cost(a, b) for a, b in rr]
    assert max(costs) / min(costs) < 1.01


def test_block_shards_partition_the_space():
    """Lattice block shards (top shard_bits prefix variables) partition the
    rank space into equal halves/quarters, and each shard's stencil only
    reads table chunks equal to the shard with at most one bit cleared."""
    from paper_2501_03381_b200.scanner import shard_rows
    n, lo, hi = 14, 2, 14
    total = sum(math.comb(n, k) for k in range(lo, hi + 1))
    for sb in (1, 2):
        parts = [shard_rows(n, lo, hi, r, sb) for r in range(1 << sb)]
        allr = np.sort(np.concatenate(parts))
        np.testing.assert_array_equal(allr, np.arange(total))
        # a subset S of shard r: its leave-one-out neighbours S \ j lie in
        # shard r (j outside the shard bits) or r with one bit cleared
        lo_var = n - 10 - sb
        for r in range(1 << sb):
            need = {r} | {r & ~(1 << t) for t in range(sb) if (r >> t) & 1}
            for c in itertools.islice(itertools.combinations(range(n), 6), 0, 3000, 7):
                pat = sum(1 << (v - lo_var) for v in c if lo_var <= v < n - 10)
                if pat != r:
                    continue
                for j in c:
                    rest = [v for v in c if v != j]
                    p2 = sum(1 << (v - lo_var) for v in rest if lo_var <= v < n - 10)
                    assert p2 in need
    assert sharding.block_shard_bits(30, 8) == 3 and sharding.block_shard_bits(30, 6) is None
    assert sharding.block_shard_bits(17, 2) == 1 and sharding.block_shard_bits(16, 2) is None
    assert sharding.block_shard_bits(11, 2) is None


def _rows(n, lo, hi):
    return [c for k in range(lo, hi + 1) for c in itertools.combinations(range(n), k)]


def _worker(rank, world, port, q, mode="ranges"):
    import sys
    from pathlib import Path
    repo = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(repo / "oracle"))
    import torch.distributed as dist

    import hoi_oracle as ora
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(11)
        a = rng.standard_normal((24, 8))
        sig = a.T @ a / 24 + 0.3 * np.eye(8)
        n, lo, hi, k = 8, 2, 8, 7
        if mode == "ranges":
            g0, g1 = sharding.rank_ranges(n, lo, hi, world, "count")[rank]
            rows = _rows(n, lo, hi)[g0:g1]
        else:   # block-shard membership pattern (variables 1..2 of 8 for 2 bits; model only)
            from paper_2501_03381_b200.scanner import shard_rows
            allrows = _rows(14, lo, 14)
            rows = [r for r in (allrows[i] for i in shard_rows(14, lo, 14, rank, 1))
                    if max(r) < n and len(r) <= hi]
        best = []
        hist = np.zeros((1, 6), dtype=np.int64)
        edges = np.linspace(-0.2, 1.0, 7)
        for kk in sorted({len(r) for r in rows}):
            sel = [r for r in rows if len(r) == kk]
            tc, dtc, o, s, _ = ora.hoi_batch(sig, [0], idx=np.array(sel))
            for i, r in enumerate(sel):
                best.append(((-float(o[i, 0]), r), (r, float(o[i, 0]))))
            hist[0] += np.histogram(np.clip(tc[:, 0], edges[0], edges[-1]), bins=edges)[0]
        best.sort(key=lambda p: p[0])
        parts = sharding.allgather_objects([best[:k]])
        merged = sharding.merge_topk(parts, k)
        counts = sharding.allreduce_counts(hist)
        if rank == 0:
            q.put(([e for _, e in merged[0]], counts.tolist()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", ["ranges", "blocks"])
def test_two_rank_topk_and_histogram_merge(oracle, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    got_top, got_counts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(11)
    a = rng.standard_normal((24, 8))
    sig = a.T @ a / 24 + 0.3 * np.eye(8)
    want = oracle.scan(sig, [0], 2, 8, oracle.TopKR("o", "max", 7))[0]
    assert [tuple(e[0]) for e in got_top] == [tuple(w[0]) for w in want]
    np.testing.assert_allclose([e[1] for e in got_top], [w[1] for w in want], rtol=1e-12)
    _, c = oracle.scan(sig, [0], 2, 8, oracle.HistR("tc", 6, -0.2, 1.0))
    assert got_counts == c.tolist()


def test_block_shard_plan_partitions_and_balances():
    """The per-rank shard sets of block_shard_plan partition the rank space,
    and every rank rebuilds the same number of table chunks at 4 and 8 GPUs."""
    from paper_2501_03381_b200.scanner import shard_set_rows
    n, lo, hi = 22, 2, 9
    total = sum(math.comb(n, k) for k in range(lo, hi + 1))
    for world in (2, 4, 8):
        sb, masks = sharding.block_shard_plan(n, world)
        rows = [shard_set_rows(n, lo, hi, m, sb) for m in masks]
        allr = np.concatenate(rows)
        assert len(allr) == total and len(np.unique(allr)) == total
        if world >= 4:    # (at 2 ranks the pairs {0, 3} / {1, 2} build 4 / 3 chunks)
            assert len({len(sharding.shard_set_chunks(m, sb)) for m in masks}) == 1
    for world in (4, 8):  # the headline N = 30: every rank rebuilds the same number of chunks
        sb, masks = sharding.block_shard_plan(30, world)
        assert sb == world.bit_length() and len({len(sharding.shard_set_chunks(m, sb))
                                                for m in masks}) == 1
    assert sharding.block_shard_plan(17, 2) == (1, [1, 2])    # N - 16 = 1 shard bit at most
    assert sharding.block_shard_plan(14, 2) is None              # table CTAs span every prefix bit

