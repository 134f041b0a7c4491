"""Multi-GPU sharding of the n-plet space (one process per GPU).

Every (n-plet, dataset) is independent, so nothing is exchanged while
computing.  Two partitions (shard_plan):

* lattice engine (power-of-two world, N >= 17): BLOCK shards -- the
  log-det table blocks are split by their top sb prefix bits into 2^sb
  shards and rank r owns shards r and 2^sb-1-r (block_shard_plan; sb =
  log2(world) + 1).  A rank rebuilds only the table chunks its stencil
  reads (its shards and those with one of their bits cleared) and streams
  only its own blocks, so both phases shrink with the world size; rank-range
  shards would each stream nearly every block (a contiguous range of the
  order-major order touches blocks of almost every prefix pattern).  The
  rank's rows land COMPACT, block-major (hoi_lattice_shard_local): no rank
  holds more than its share of the 32 B x n-plets output.
* otherwise: the global order-major lexicographic rank space [0, total)
  cut into contiguous ranges, one per rank, balanced by cost.

The only collectives are the final merges (scan_sharded):

* full output -- ShardedScan.gather(dst): point-to-point transfers to dst,
  rank slices copied in place, block shards scattered to their global rows
  (hoi_lattice_local_scatter); bit-identical to a one-GPU scan;
* TopK -- every rank's local top-k (value, index tuple, measures) is
  all-gathered and merged with the reference's (sign*value, tuple) key;
* Histogram -- counts are summed (all-reduce);
* FeatureAccumulator -- canonical chunks (fixed size, independent of the
  world size) are dealt round-robin, their partials all-gathered and merged
  in enumeration order: the same features, bit for bit, at any world size.

Collectives go through torch.distributed (NCCL over NVLink on the GPU box,
gloo in the CPU tests and the one-GPU two-process test).
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as nat


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
    if world < 1 or (1 << sb) != world or not 12 <= n <= 32 or sb > _max_shard_bits(n):
        return None
    return sb


def _max_shard_bits(n: int) -> int:
    """Shard bits the lattice can split: at most (N-10)/2 (the stencil's two
    passes) and at most N-16 (a table CTA expands prefix variables 0..5, so
    shard chunks are cut above them), at most 6 (a 64-bit shard mask)."""
    return max(0, min(6, (n - 10) // 2, n - 16))


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
    if world > 1 and sb + 1 <= _max_shard_bits(n):
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


def shard_plan(ctx, world):
    """("blocks", sb, masks) when the lattice engine block-shards N over a
    power-of-two world, else ("ranges", per-rank [g0, g1))."""
    n = ctx.n
    plan = block_shard_plan(n, world) if ctx.engine == 2 else None
    if plan is not None:
        return ("blocks",) + plan
    weight = "count" if ctx.engine == 2 else "flops"
    return ("ranges", rank_ranges(n, ctx.lo, ctx.hi, world, weight))


def _is_nccl(group):
    import torch.distributed as dist
    return dist.get_backend(group) == "nccl"


def _send(t, dst, group):
    """Point-to-point send of a device tensor (staged through the host on
    gloo, which moves CPU tensors only)."""
    import torch.distributed as dist
    dist.send(t.contiguous() if _is_nccl(group) else t.cpu(), dst, group=group)


def _recv_into(t, src, group):
    import torch.distributed as dist
    if _is_nccl(group):
        dist.recv(t, src, group=group)
    else:
        h = torch_empty_like_cpu(t)
        dist.recv(h, src, group=group)
        t.copy_(h)


def torch_empty_like_cpu(t):
    import torch
    return torch.empty(t.shape, dtype=t.dtype)


class ShardedScan:
    """One rank's part of an exhaustive FULL-output scan, resident on its
    GPU and compact (no rank holds the full 32 B x n-plets output):

    * kind "blocks" (lattice engine, power-of-two world): the rank's block
      shards, block-major -- local block c holds the 1024 n-plets of table
      block blocks[c] in run order (hoi_lattice_shard_local);
    * kind "ranges": the contiguous global ranks [g0, g1) in order.

    gather(dst) reassembles the single-GPU output, bit for bit, on rank dst
    (NCCL point-to-point over NVLink; the reference's ordered merge,
    ref:scanner.py:290-305): rank slices land straight in place, block
    shards through hoi_lattice_local_scatter."""

    def __init__(self, kind, out, n, lo, hi, total, rank, world, group, plan, blocks=None,
                 nblocks=None):
        self.kind, self.out, self.n, self.lo, self.hi = kind, out, n, lo, hi
        self.total, self.rank, self.world, self.group, self.plan = total, rank, world, group, plan
        self.blocks, self.nblocks = blocks, nblocks

    @property
    def local_rows(self) -> int:
        return int(self.out.shape[1])

    def _local_rows_of(self, r):
        if self.kind == "ranges":
            g0, g1 = self.plan[1][r]
            return g1 - g0
        sb, masks = self.plan[1], self.plan[2]
        return bin(masks[r]).count("1") << (self.n - sb)

    def gather(self, dst: int = 0):
        """The whole scan as a DeviceScan on rank dst (None elsewhere)."""
        import torch
        from . import _native as nat
        from .scanner import DeviceScan
        d = self.out.shape[2]
        if self.rank != dst:
            _send(self.out, dst, self.group)
            if self.kind == "blocks":
                _send(self.blocks, dst, self.group)
                _send(self.nblocks, dst, self.group)
            return None
        full = torch.empty((4, self.total, d), dtype=torch.float64, device="cuda")
        lib = nat.lib()
        for r in range(self.world):
            if self.kind == "ranges":
                g0, g1 = self.plan[1][r]
                if r == self.rank:
                    full[:, g0:g1].copy_(self.out)
                else:
                    stage = torch.empty((4, g1 - g0, d), dtype=torch.float64, device="cuda")
                    _recv_into(stage, r, self.group)
                    full[:, g0:g1].copy_(stage)
                continue
            if r == self.rank:
                loc, blk, nb = self.out, self.blocks, self.nblocks
            else:
                loc = torch.empty((4, self._local_rows_of(r), d), dtype=torch.float64,
                                  device="cuda")
                blk = torch.empty_like(self.blocks)
                nb = torch.empty_like(self.nblocks)
                _recv_into(loc, r, self.group)
                _recv_into(blk, r, self.group)
                _recv_into(nb, r, self.group)
            nat.check(lib.hoi_lattice_local_scatter(loc.data_ptr(), loc.shape[1], blk.data_ptr(),
                                                    nb.data_ptr(), self.n, d, self.lo, self.hi,
                                                    0, self.total, full.data_ptr(),
                                                    nat.stream_handle(torch)), "local_scatter")
        return DeviceScan(full, self.n, self.lo, self.hi, 0, self.total)

    def save(self, path, dst: int = 0):
        """Gather on rank dst and write the binary scan format there."""
        dev = self.gather(dst)
        return dev.save(path) if dev is not None else None


def local_buffers(ctx, plan, rank):
    """Device buffers of this rank's compact full output: (out, blocks,
    nblocks) -- blocks/nblocks None for rank ranges."""
    import torch
    if plan[0] == "ranges":
        g0, g1 = plan[1][rank]
        return torch.empty((4, g1 - g0, ctx.d), dtype=torch.float64, device="cuda"), None, None
    sb, masks = plan[1], plan[2]
    rows = bin(masks[rank]).count("1") << (ctx.n - sb)
    return (torch.empty((4, rows, ctx.d), dtype=torch.float64, device="cuda"),
            torch.empty(1 << (ctx.n - 10), dtype=torch.int32, device="cuda"),
            torch.zeros(1, dtype=torch.int64, device="cuda"))


def full_local_into(ctx, plan, rank, out, blocks=None, nblocks=None):
    """Compute this rank's compact full output into local_buffers()."""
    import torch
    from . import _native as nat
    from .nplet_engine import _raise_not_pd
    if plan[0] == "ranges":
        g0, g1 = plan[1][rank]
        _, cnt, coords = ctx.full(g0, g1, out)
        _raise_not_pd(cnt, coords)
        return
    sb, masks = plan[1], plan[2]
    lib = nat.lib()
    s = nat.stream_handle(torch)
    kst = 0 if ctx.eta is None else ctx.eta.shape[1]
    for d in range(ctx.d):
        nat.check(lib.hoi_lattice_shard_local(ctx.st.corr.data_ptr(), ctx.n, ctx.d, d,
                                              nat.ptr(ctx.eta), kst, ctx.lo, ctx.hi,
                                              int(masks[rank]), sb, out.data_ptr(), out.shape[1],
                                              blocks.data_ptr(), nblocks.data_ptr(),
                                              ctx.ws.data_ptr(), ctx.ws.numel(), s),
                  "lattice_shard_local")
    ctx._table_ok = False


def _full_local(ctx, plan, rank, fill_nan=False):
    """This rank's compact full output (see ShardedScan)."""
    import torch
    out, blocks, nblocks = local_buffers(ctx, plan, rank)
    if fill_nan and blocks is not None:
        out.view(torch.int64).fill_(-1)              # all-ones bits: NaN in the holes
    full_local_into(ctx, plan, rank, out, blocks, nblocks)
    return out, blocks, nblocks


@nat.traced("hoi.scan_sharded")
def scan_sharded(covs, lo, hi, reducer=None, *, bias_correct=False, group=None):
    """This rank's shard of an exhaustive scan on its GPU (one process per
    GPU), merged across the ranks of `group` with the reference's reducer
    semantics (ref:scanner.py:290-365: results as if one ordered scan ran):

    * reducer None       -> ShardedScan (FULL output, compact per rank;
                            .gather() / .save() reassemble it in rank order)
    * TopK               -> the merged lists (every rank returns them)
    * Histogram          -> the summed counts
    * FeatureAccumulator -> the merged features (canonical chunks, so the
                            result does not depend on the world size)
    The reducer's prior state is kept: only this scan's contribution is
    reduced across ranks and then merged into it once."""
    import torch
    import torch.distributed as dist

    from . import _native as nat
    from .nplet_engine import count_nplets
    from .scanner import (FeatureAccumulator, Histogram, MEASURES, TopK, _ScanCtx,
                          _topk_lattice, _topk_plane)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = covs.n_variables
    total = count_nplets(n, lo, hi)
    ctx = _ScanCtx(covs, lo, hi, bias_correct)
    plan = shard_plan(ctx, world)
    if reducer is None:
        out, blocks, nblocks = _full_local(ctx, plan, rank)
        return ShardedScan(plan[0], out, n, lo, hi, total, rank, world, group, plan, blocks,
                           nblocks)
    if type(reducer) is TopK:
        fresh = TopK(reducer.measure, reducer.direction, reducer.k)
        m = MEASURES.index(reducer.measure)
        ok = False
        if plan[0] == "blocks":
            ok = _topk_lattice(ctx, fresh, m, shard_bits=plan[1], shard_mask=plan[2][rank])
            if not all(allgather_objects(bool(ok), group)):
                fresh = TopK(reducer.measure, reducer.direction, reducer.k)
                ok = False
        if not ok:
            g0, g1 = rank_ranges(n, lo, hi, world, "count" if ctx.engine == 2 else "flops")[rank]
            out, cnt, coords = ctx.full(g0, g1)
            from .nplet_engine import _raise_not_pd
            _raise_not_pd(cnt, coords)
            _topk_plane(ctx, fresh, out, g0, m)
        fresh._materialize()
        parts = allgather_objects(fresh._best or [[] for _ in range(ctx.d)], group)
        merged = merge_topk(parts, reducer.k)
        reducer._materialize()
        if reducer._best is None:
            reducer._best = merged
        else:
            for d in range(ctx.d):
                reducer._merge(d, merged[d])
        return reducer.finalize()
    if type(reducer) is Histogram:
        m = MEASURES.index(reducer.measure)
        out, _, _ = _full_local(ctx, plan, rank, fill_nan=True)
        edges = torch.from_numpy(reducer.edges).cuda()
        c = torch.zeros((ctx.d, len(reducer.edges) - 1), dtype=torch.int64, device="cuda")
        nat.check(nat.lib().hoi_histogram(out[m].data_ptr(), out.shape[1], ctx.d, c.shape[1],
                                          float(reducer.edges[0]), float(reducer.edges[-1]),
                                          edges.data_ptr(), c.data_ptr(),
                                          nat.stream_handle(torch)), "histogram")
        del out
        if _is_nccl(group):
            dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
            counts = c.cpu().numpy()
        else:
            counts = allreduce_counts(c.cpu().numpy(), group)
        reducer._counts = counts if reducer._counts is None else reducer._counts + counts
        return reducer.finalize()
    if type(reducer) is FeatureAccumulator and reducer.n == n:
        from .scanner import _feature_chunks, _feature_merge
        chunks = _feature_chunks(ctx, total)
        mine = [c for i, c in enumerate(chunks) if i % world == rank]
        parts = [(g0, _feature_partial_rows(ctx, g0, g1)) for g0, g1 in mine]
        allparts = sorted(p for per in allgather_objects(parts, group) for p in per)
        _feature_merge(ctx, reducer, allparts)
        return reducer.finalize()
    raise TypeError("scan_sharded supports TopK, Histogram, FeatureAccumulator or None "
                    "(full output)")


def _feature_partial_rows(ctx, g0, g1):
    from .scanner import _feature_partial
    return _feature_partial(ctx, g0, g1)
