"""Multi-GPU sharding of the n-plet space (one process per GPU).

Every (n-plet, dataset) is independent, so nothing is exchanged while
computing.  Two partitions:

* lattice engine (12 <= N <= 32, power-of-two world): BLOCK shards -- the
  log-det table blocks are split by their top sb prefix bits into 2^sb
  shards and rank r owns shards r and 2^sb-1-r (block_shard_plan; sb =
  log2(world) + 1, ScanCtx.full_shard_set / hoi_lattice_shard_set).  A rank
  rebuilds only the table chunks its stencil reads (its shards and those
  with one of their bits cleared) and streams only its own blocks, so both
  phases shrink with the world size; rank-range
  shards would each stream nearly every block (a contiguous range of the
  order-major order touches blocks of almost every prefix pattern).
* otherwise: the global order-major lexicographic rank space [0, total)
  cut into contiguous ranges, one per rank, balanced by cost.

The only collectives are the final merges:

* full output -- shards are contiguous slices of the global order, so
  concatenating them in rank order is bit-identical to a one-GPU scan;
* TopK -- every rank's local top-k (value, index tuple, measures) is
  all-gathered and merged with the reference's (sign*value, tuple) key;
* Histogram -- counts are summed (all-reduce).

Collectives go through torch.distributed (NCCL over NVLink on the GPU box,
gloo in the CPU tests).
"""

from __future__ import annotations

import math

import numpy as np


def nplet_flops(k: int) -> float:
    """Algorithmic FP64 flops per (n-plet, dataset) of order k for the
    per-n-plet engine: (k^3-k)/3 (LDL^T) + (k^3-k)/3 (triangular inverse)
    + k(k+1) (inverse-diagonal column norms); one FMA = 2 flops."""
    return 2.0 * (k ** 3 - k) / 3.0 + k * (k + 1)


def order_offsets(n: int, lo: int, hi: int):
    off, acc = [], 0
    for k in range(lo, hi + 1):
        off.append(acc)
        acc += math.comb(n, k)
    return off, acc


def rank_ranges(n: int, lo: int, hi: int, world: int, weight: str = "count"):
    """Contiguous [g0, g1) per rank with (approximately) equal cost.

    weight="count": equal n-plet counts (the lattice engine's cost is flat
    per n-plet); weight="flops": equal sum of nplet_flops(k) (the per-n-plet
    engine's cost grows as k^3).  Cuts may fall inside an order."""
    offs, total = order_offsets(n, lo, hi)
    if weight == "count":
        cuts = [total * r // world for r in range(world + 1)]
        return [(cuts[r], cuts[r + 1]) for r in range(world)]
    ks = list(range(lo, hi + 1))
    cost = [math.comb(n, k) * nplet_flops(k) for k in ks]
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    bounds = [0]
    for r in range(1, world):
        target = cum[-1] * r / world
        i = int(np.searchsorted(cum, target, side="right")) - 1
        i = min(i, len(ks) - 1)
        within = (target - cum[i]) / nplet_flops(ks[i])
        g = offs[i] + int(round(within))
        bounds.append(max(bounds[-1], min(g, total)))
    bounds.append(total)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def merge_topk(partials, k: int):
    """Merge per-rank TopK partial lists (each a list over datasets of
    ((key_value, index_tuple), entry) pairs) deterministically."""
    d_count = max(len(p) for p in partials)
    merged = []
    for d in range(d_count):
        pool = [pair for p in partials for pair in (p[d] if d < len(p) else [])]
        pool.sort(key=lambda pair: pair[0])
        merged.append(pool[:k])
    return merged


def allgather_objects(obj, group=None):
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def allreduce_counts(counts: np.ndarray, group=None, device="cpu") -> np.ndarray:
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(counts, dtype=torch.int64, device=device).clone()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


def block_shard_bits(n: int, world: int):
    """log2(world) when the lattice engine can block-shard N variables over
    `world` ranks (power of two, at most (N-10)/2 shard bits), else None."""
    sb = world.bit_length() - 1
    if world < 1 or (1 << sb) != world or not 12 <= n <= 32 or sb > (n - 10) // 2:
        return None
    return sb


def block_shard_plan(n: int, world: int):
    """(shard_bits, per-rank shard masks) for the lattice engine's block
    shards, or None when N cannot be block-sharded over `world` ranks.

    A rank whose shard has p set bits must build 1 + p table chunks (its
    own and each with one bit cleared), so one shard per rank leaves the
    all-ones rank with half the table to build at 8 GPUs.  With one more
    shard bit each rank owns a complementary pair, shards r and 2^sb-1-r,
    whose popcounts sum to sb: every rank then builds the same number of
    chunks (measured on B200, cfg4, G = 8: slowest rank 4.47 -> 3.92 ms)."""
    sb = block_shard_bits(n, world)
    if sb is None:
        return None
    if world > 1 and sb + 1 <= min(6, (n - 10) // 2):
        sb += 1
        full = (1 << sb) - 1
        return sb, [(1 << r) | (1 << (full - r)) for r in range(world)]
    return sb, [1 << r for r in range(world)]


def shard_set_chunks(mask: int, sb: int) -> list:
    """Table chunks a GPU owning shard `mask` builds: every owned shard and
    every shard one cleared bit below one (host model of lattice_shard)."""
    owned = [c for c in range(1 << sb) if (mask >> c) & 1]
    return [c for c in range(1 << sb)
            if any((c & ~o) == 0 and bin(o ^ c).count("1") <= 1 for o in owned)]


def scan_sharded(covs, lo, hi, reducer, *, bias_correct=False, group=None):
    """Run this rank's shard of an exhaustive scan on its GPU and merge the
    TopK / Histogram result across ranks (all ranks return the same value)."""
    import torch.distributed as dist

    from .nplet_engine import _raise_not_pd
    from .scanner import Histogram, MEASURES, TopK, _ScanCtx, _topk_lattice, _topk_plane
    import torch
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = covs.n_variables
    plan = block_shard_plan(n, world)
    if type(reducer) is TopK and plan is not None:
        sb, masks = plan
        ctx = _ScanCtx(covs, lo, hi, bias_correct)
        ok = ctx.engine == 2 and _topk_lattice(ctx, reducer, MEASURES.index(reducer.measure),
                                               shard_bits=sb, shard_mask=masks[rank])
        if all(allgather_objects(bool(ok), group)):
            parts = allgather_objects(reducer._best, group)
            reducer._best = merge_topk(parts, reducer.k)
            return reducer.finalize()
        reducer._best = None                       # a rank declined: rank-range path
    weight = "count" if n <= 34 else "flops"
    g0, g1 = rank_ranges(n, lo, hi, world, weight)[rank]
    ctx = _ScanCtx(covs, lo, hi, bias_correct)
    out, cnt, coords = ctx.full(g0, g1)
    _raise_not_pd(cnt, coords)
    m = MEASURES.index(reducer.measure)
    if type(reducer) is TopK:
        _topk_plane(ctx, reducer, out, g0, m)
        parts = allgather_objects(reducer._best, group)
        reducer._best = merge_topk(parts, reducer.k)
    elif type(reducer) is Histogram:
        from . import _native as nat
        edges = torch.from_numpy(reducer.edges).cuda()
        c = torch.zeros((ctx.d, len(reducer.edges) - 1), dtype=torch.int64, device="cuda")
        nat.check(nat.lib().hoi_histogram(out[m].data_ptr(), g1 - g0, ctx.d, c.shape[1],
                                          float(reducer.edges[0]), float(reducer.edges[-1]),
                                          edges.data_ptr(), c.data_ptr(),
                                          nat.stream_handle(torch)), "histogram")
        dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
        reducer._counts = c.cpu().numpy()
    else:
        raise TypeError("scan_sharded supports TopK and Histogram reducers")
    return reducer.finalize()
