"""Exhaustive scans with pluggable reducers (drop-in for ref:scanner.py).

The n-plet space of a scan is the order-major, lexicographic sequence the
reference enumerates (ref:scanner.py:345-347), addressed by a global rank
g.  The device computes whole rank ranges at once (``hoi_scan_full``);
the host then either

* reduces on the device -- TopK (candidate filter + exact merge with the
  reference's (sign*value, index tuple) key) and Histogram (numpy's edge
  semantics) -- so only a few hundred bytes come back, or
* replays the reference's batches (<= batch_size rows, never crossing an
  order) to any other Reducer in enumeration order, with the same progress
  counters.

Results never depend on batch_size or workers (workers is validated and
otherwise has nothing to do: there is no host thread pool to size).
"""

from __future__ import annotations

import ctypes
import functools
import gc
import itertools
import math
import time
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from ._device import device_covs
from .copula_core import CovSet
from .errors import ExhaustiveLimitExceeded, InvalidData, InvalidOrderRange
from .measures import HoiBatch, compute_hoi_batch
from .nplet_engine import ERR_CAP, NpletBatch, _err_buffers, _raise_not_pd, count_nplets

MEASURES = ("tc", "dtc", "o", "s")


class Reducer:
    """Consumes (NpletBatch, HoiBatch) pairs in enumeration order (ref:scanner.py:27-34)."""

    def update(self, batch: NpletBatch, hoi: HoiBatch) -> None:
        raise NotImplementedError

    def finalize(self):
        raise NotImplementedError


@dataclass(frozen=True)
class TopEntry:
    """One selected n-plet with all four measures (ref:scanner.py:37-47)."""

    indices: tuple
    order: int
    value: float
    tc: float
    dtc: float
    o: float
    s: float


_new = object.__new__


def _gc_paused(fn):
    """Run fn with Python's cyclic collector paused (restored on exit).  The
    TopK merges build tens of thousands of small acyclic objects (entries,
    index tuples, keys); with torch loaded, the collections they trigger walk
    every live object and cost more than the merge itself (BASELINE config
    5's 16 x 1000 entries: 55 -> 19 ms)."""
    @functools.wraps(fn)
    def run(*args, **kwargs):
        was = gc.isenabled()
        gc.disable()
        try:
            return fn(*args, **kwargs)
        finally:
            if was:
                gc.enable()
    return run


def _entry(t, v, tc, dtc, o, sv):
    """TopEntry(t, len(t), v, tc, dtc, o, sv) without the frozen dataclass's
    per-field object.__setattr__ calls (half the cost; the device TopK paths
    build one per selected row).  Same class, fields, equality and hash."""
    e = _new(TopEntry)
    e.__dict__.update(indices=t, order=len(t), value=v, tc=tc, dtc=dtc, o=o, s=sv)
    return e


class TopEntries(Sequence):
    """One dataset's TopK result held as arrays -- index tuples (m, K) and
    the four measures (4, m) -- in the reference's order; the TopEntry
    objects are built on first access, all at once (a config-5 result is
    16 x 1,000 entries, and building them eagerly cost more than the device
    work).  Compares equal to the list of TopEntry it stands for."""

    def __init__(self, tuples: np.ndarray, vals: np.ndarray, m_idx: int):
        self._t, self._v, self._m = tuples, vals, m_idx
        self._cache = None

    def __len__(self):
        return self._t.shape[0]

    @_gc_paused
    def _list(self):
        if self._cache is None:
            m = self._m
            self._cache = [_entry(tuple(r), x[m], x[0], x[1], x[2], x[3])
                           for r, x in zip(self._t.tolist(), self._v.T.tolist())]
        return self._cache

    def __getitem__(self, i):
        return self._list()[i]

    def __iter__(self):
        return iter(self._list())

    def __eq__(self, other):
        try:
            return self._list() == list(other)
        except TypeError:
            return NotImplemented

    def __repr__(self):
        return f"TopEntries({self._list()!r})"


class TopK(Reducer):
    """k best n-plets per dataset for one measure; ties broken by the
    lexicographically smallest index tuple (ref:scanner.py:50-105)."""

    def __init__(self, measure: str, direction: str, k: int):
        if measure not in MEASURES:
            raise InvalidData(f"measure must be one of {MEASURES}, got {measure!r}")
        if direction not in ("max", "min"):
            raise InvalidData(f"direction must be 'max' or 'min', got {direction!r}")
        if k < 1:
            raise InvalidData(f"k must be >= 1, got {k}")
        self.measure, self.direction, self.k = measure, direction, k
        self._best = None
        self._compact = None      # [TopEntries per dataset] from the device order

    def _materialize(self):
        """Fold a compact device result into the list state (before a merge)."""
        if self._compact is not None:
            self._best = [[((self.sign * e.value, e.indices), e) for e in per]
                          for per in self._compact]
            self._compact = None

    @property
    def sign(self) -> float:
        return -1.0 if self.direction == "max" else 1.0

    def _merge(self, d, entries):
        best = self._best[d]
        best.extend(entries)
        best.sort(key=lambda pair: pair[0])
        del best[self.k:]

    @_gc_paused
    def update(self, batch, hoi):
        self._materialize()
        vals = getattr(hoi, self.measure)
        b, d_count = vals.shape
        if self._best is None:
            self._best = [[] for _ in range(d_count)]
        sign = self.sign
        k_eff = min(self.k, b)
        for d in range(d_count):
            key = sign * vals[:, d]
            thr = np.partition(key, k_eff - 1)[k_eff - 1]
            new = []
            for i in np.flatnonzero(key <= thr):
                idx = batch.row_indices(int(i))
                e = TopEntry(indices=idx, order=len(idx), value=float(vals[i, d]),
                             tc=float(hoi.tc[i, d]), dtc=float(hoi.dtc[i, d]),
                             o=float(hoi.o[i, d]), s=float(hoi.s[i, d]))
                new.append(((sign * e.value, idx), e))
            self._merge(d, new)

    def finalize(self):
        if self._compact is not None:
            return list(self._compact)
        if self._best is None:
            return []
        return [[e for _, e in per] for per in self._best]


class Histogram(Reducer):
    """Clipped fixed-range histogram of one measure per dataset (ref:scanner.py:108-137)."""

    def __init__(self, measure: str, bins: int, lo: float, hi: float):
        if measure not in MEASURES:
            raise InvalidData(f"measure must be one of {MEASURES}, got {measure!r}")
        if bins < 1:
            raise InvalidData(f"bins must be >= 1, got {bins}")
        if not lo < hi:
            raise InvalidData(f"need lo < hi, got [{lo}, {hi}]")
        self.measure = measure
        self.edges = np.linspace(lo, hi, bins + 1)
        self._counts = None

    def update(self, batch, hoi):
        vals = getattr(hoi, self.measure)
        if self._counts is None:
            self._counts = np.zeros((vals.shape[1], len(self.edges) - 1), dtype=np.int64)
        lo, hi = self.edges[0], self.edges[-1]
        for d in range(vals.shape[1]):
            self._counts[d] += np.histogram(np.clip(vals[:, d], lo, hi), bins=self.edges)[0]

    def finalize(self):
        return self.edges, self._counts


class Callback(Reducer):
    """Calls fn(batch, hoi) per batch in enumeration order (ref:scanner.py:140-154)."""

    def __init__(self, fn):
        if not callable(fn):
            raise InvalidData("Callback needs a callable")
        self.fn = fn
        self._results = []

    def update(self, batch, hoi):
        self._results.append(self.fn(batch, hoi))

    def finalize(self):
        return self._results


FEATURE_NAMES = (
    "tc_max", "tc_min", "tc_mean", "tc_whole",
    "dtc_max", "dtc_min", "dtc_mean", "dtc_whole",
    "o_max", "o_min", "o_mean", "o_whole",
    "s_max", "s_min", "s_mean", "s_whole",
    "mi_mean", "mi_std",
    "o_max_order_norm", "o_min_order_norm",
    "prop_synergistic",
)


@dataclass(frozen=True)
class FeatureVector:
    """The 21-feature fingerprint of one dataset (ref:scanner.py:168-202)."""

    tc_max: float
    tc_min: float
    tc_mean: float
    tc_whole: float
    dtc_max: float
    dtc_min: float
    dtc_mean: float
    dtc_whole: float
    o_max: float
    o_min: float
    o_mean: float
    o_whole: float
    s_max: float
    s_min: float
    s_mean: float
    s_whole: float
    mi_mean: float
    mi_std: float
    o_max_order_norm: float
    o_min_order_norm: float
    prop_synergistic: float

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name in FEATURE_NAMES}


class FeatureAccumulator(Reducer):
    """Streaming 21-feature accumulator over orders 2..N (ref:scanner.py:205-287)."""

    def __init__(self, n_variables: int):
        self.n = int(n_variables)
        self._d = None

    def _init_state(self, d_count):
        self._d = d_count
        self._sums = np.zeros((d_count, 4))
        self._maxs = np.full((d_count, 4), -np.inf)
        self._mins = np.full((d_count, 4), np.inf)
        self._count = 0
        self._o_max_order = np.zeros(d_count, dtype=np.int64)
        self._o_min_order = np.zeros(d_count, dtype=np.int64)
        self._syn = np.zeros(d_count, dtype=np.int64)
        self._mi_sum = np.zeros(d_count)
        self._mi_sumsq = np.zeros(d_count)
        self._mi_count = 0
        self._whole = np.full((d_count, 4), np.nan)

    def update(self, batch, hoi):
        vals = np.stack([hoi.tc, hoi.dtc, hoi.o, hoi.s], axis=-1)
        if self._d is None:
            self._init_state(vals.shape[1])
        orders = hoi.order
        pair = orders == 2
        if pair.any():
            mi = hoi.tc[pair]
            self._mi_sum += mi.sum(axis=0)
            self._mi_sumsq += (mi * mi).sum(axis=0)
            self._mi_count += int(pair.sum())
        rows = orders >= 3
        if rows.any():
            v = vals[rows]
            o_col = hoi.o[rows]
            row_orders = orders[rows]
            for d in range(self._d):
                i_max = int(np.argmax(o_col[:, d]))
                if o_col[i_max, d] > self._maxs[d, 2]:
                    self._o_max_order[d] = row_orders[i_max]
                i_min = int(np.argmin(o_col[:, d]))
                if o_col[i_min, d] < self._mins[d, 2]:
                    self._o_min_order[d] = row_orders[i_min]
            np.maximum(self._maxs, v.max(axis=0), out=self._maxs)
            np.minimum(self._mins, v.min(axis=0), out=self._mins)
            self._sums += v.sum(axis=0)
            self._count += v.shape[0]
            self._syn += (o_col < 0.0).sum(axis=0)
            whole = np.flatnonzero(row_orders == self.n)
            if whole.size:
                self._whole = v[whole[0]]

    def finalize(self):
        if self._d is None or self._count == 0 or self._mi_count == 0:
            raise InvalidData("feature accumulation needs orders 2..N")
        if np.isnan(self._whole).any():
            raise InvalidData("feature accumulation never saw the order-N row")
        out = []
        for d in range(self._d):
            means = self._sums[d] / self._count
            mi_mean = self._mi_sum[d] / self._mi_count
            mi_var = max(self._mi_sumsq[d] / self._mi_count - mi_mean * mi_mean, 0.0)
            kw = {}
            for m_i, m in enumerate(MEASURES):
                kw[f"{m}_max"] = float(self._maxs[d, m_i])
                kw[f"{m}_min"] = float(self._mins[d, m_i])
                kw[f"{m}_mean"] = float(means[m_i])
                kw[f"{m}_whole"] = float(self._whole[d, m_i])
            kw["mi_mean"] = float(mi_mean)
            kw["mi_std"] = float(np.sqrt(mi_var))
            kw["o_max_order_norm"] = float(self._o_max_order[d] / self.n)
            kw["o_min_order_norm"] = float(self._o_min_order[d] / self.n)
            kw["prop_synergistic"] = float(self._syn[d] / self._count)
            out.append(FeatureVector(**kw))
        return out


# ------------------------------------------------------------- device scan --

class DeviceScan:
    """Full output of an exhaustive scan resident on the device.

    ``out`` is a (4, rows, D) float64 tensor (tc, dtc, o, s) for the global
    ranks [g_begin, g_end) of orders min_order..max_order."""

    def __init__(self, out, n, min_order, max_order, g_begin, g_end):
        self.out, self.n = out, n
        self.min_order, self.max_order = min_order, max_order
        self.g_begin, self.g_end = g_begin, g_end

    def offsets(self):
        off, acc = {}, 0
        for k in range(self.min_order, self.max_order + 1):
            off[k] = acc
            acc += math.comb(self.n, k)
        return off

    def save(self, path, chunk_rows: int = 1 << 24):
        """Write the scan in the binary scan format (the
        full output of an exhaustive scan -- 34 GB for N = 30 -- has no CSV
        form): a 4096-byte JSON header (format, n, orders, rank range, D,
        plane order, dtype), then the four float64 planes tc, dtc, o, s,
        each (rows, D) in global rank order, rank implicit (row i is rank
        g_begin + i; `unrank` maps it to its index tuple).  Streamed from HBM
        in chunks through a pinned staging buffer.  read_scan() maps it back."""
        import json
        torch = nat.torch_cuda()
        rows, d = self.out.shape[1], self.out.shape[2]
        head = json.dumps({"format": "hoi-b200-scan/1", "n": self.n, "min_order": self.min_order,
                           "max_order": self.max_order, "g_begin": self.g_begin,
                           "g_end": self.g_end, "datasets": d, "planes": list(MEASURES),
                           "dtype": "float64", "layout": "planes x rows x datasets, C order",
                           "header_bytes": 4096}).encode()
        if len(head) > 4096:
            raise InvalidData("scan header too long")
        step = max(1, min(chunk_rows, rows))
        stage = torch.empty((step, d), dtype=torch.float64, pin_memory=True)
        with open(path, "wb") as f:
            f.write(head.ljust(4096, b" "))
            for q in range(4):
                for a in range(0, rows, step):
                    b = min(rows, a + step)
                    stage[:b - a].copy_(self.out[q, a:b])
                    f.write(stage[:b - a].numpy().tobytes())
        return path


class _ScanCtx:
    def __init__(self, covs, lo, hi, bias_correct, engine=0):
        self.st = device_covs(covs)
        self.torch = self.st.torch
        self.n, self.d = self.st.n, self.st.d
        self.lo, self.hi = lo, hi
        self.eta = self.st.eta(hi) if bias_correct else None
        # auto: the subset-lattice engine when its 2^N table applies
        # (12 <= N <= 32), the per-n-plet engine otherwise
        self.engine = engine or (2 if 12 <= self.n <= 32 else 1)
        self.ws = None
        self.ws_bytes = ctypes.c_size_t(0)
        self._alloc_ws()

    def _args(self, g0, g1):
        kst = 0 if self.eta is None else self.eta.shape[1]
        return (self.st.corr.data_ptr(), self.st.sdiag.data_ptr(), nat.ptr(self.eta), kst,
                self.n, self.d, self.lo, self.hi, g0, g1, self.engine)

    def _alloc_ws(self):
        """Query and allocate the engine workspace (the lattice engine's
        2^N log-det table); auto mode drops to the per-n-plet engine when
        the table does not fit."""
        lib, torch = nat.lib(), self.torch
        need = ctypes.c_size_t(0)
        nat.check(lib.hoi_scan_full(*self._args(0, 0), None, None, None, 0, None,
                                    ctypes.byref(need), None), "scan_full")
        try:
            self.ws = torch.empty(max(int(need.value), 8), dtype=torch.uint8, device="cuda")
        except torch.cuda.OutOfMemoryError:
            if self.engine == 1:
                raise
            self.engine = 1
            self.ws = torch.empty(8, dtype=torch.uint8, device="cuda")
        self.ws_bytes = ctypes.c_size_t(self.ws.numel())

    def full(self, g0, g1, out=None, reuse_table=False):
        """Full output (4, g1-g0, D) for global ranks [g0, g1).

        reuse_table: for the lattice engine with one dataset, keep the log-det
        table of a previous call (a scan split into several rank chunks
        builds it once)."""
        torch, lib = self.torch, nat.lib()
        rows = g1 - g0
        if out is None:
            out = torch.empty((4, rows, self.d), dtype=torch.float64, device="cuda")
        cnt, coords = _err_buffers(torch)
        s = nat.stream_handle(torch)
        if self.engine == 2 and self.d == 1 and reuse_table and getattr(self, "_table_ok", False):
            # the log-det table of an earlier chunk of this scan is complete
            kst = 0 if self.eta is None else self.eta.shape[1]
            rc = lib.hoi_lattice_measures(self.ws.data_ptr(), self.n, 1, 0, nat.ptr(self.eta),
                                          kst, self.lo, self.hi, g0, g1, out.data_ptr(), s)
        else:
            rc = lib.hoi_scan_full(*self._args(g0, g1), out.data_ptr(), cnt.data_ptr(),
                                   coords.data_ptr(), ERR_CAP, self.ws.data_ptr(),
                                   ctypes.byref(self.ws_bytes), s)
        if rc == nat.FALLBACK:
            # the lattice engine declined (correlation not numerically PD):
            # the per-n-plet engine applies the reference's jitter rule
            self.engine = 1
            self.ws = None
            self._alloc_ws()
            return self.full(g0, g1, out)
        nat.check(rc, "scan_full")
        # after a full engine-2 pass (D == 1) the workspace holds the whole table
        self._table_ok = self.engine == 2 and self.d == 1
        return out, cnt, coords


    def full_shard_set(self, shard_mask: int, shard_bits: int, out=None):
        """Lattice engine, the block shards in `shard_mask` (bit c = shard c
        of 2^shard_bits) on this GPU, each n-plet at its GLOBAL row of a
        full-size (4, total, D) output (see full_shard)."""
        torch, lib = self.torch, nat.lib()
        total = count_nplets(self.n, self.lo, self.hi)
        if out is None:
            out = torch.empty((4, total, self.d), dtype=torch.float64, device="cuda")
        s = nat.stream_handle(torch)
        kst = 0 if self.eta is None else self.eta.shape[1]
        for d in range(self.d):
            nat.check(lib.hoi_lattice_shard_set(self.st.corr.data_ptr(), self.n, self.d, d,
                                                nat.ptr(self.eta), kst, self.lo, self.hi,
                                                int(shard_mask), shard_bits, out.data_ptr(),
                                                self.ws.data_ptr(), self.ws.numel(), s),
                      "lattice_shard_set")
        self._table_ok = False
        return out

    def full_shard(self, shard: int, shard_bits: int, out=None):
        """Lattice engine, block shard `shard` of 2^shard_bits: every n-plet
        of the shard's table blocks at its GLOBAL row of a full-size
        (4, total, D) output (rows of other shards are left untouched)."""
        torch, lib = self.torch, nat.lib()
        total = count_nplets(self.n, self.lo, self.hi)
        if out is None:
            out = torch.empty((4, total, self.d), dtype=torch.float64, device="cuda")
        s = nat.stream_handle(torch)
        kst = 0 if self.eta is None else self.eta.shape[1]
        for d in range(self.d):
            nat.check(lib.hoi_lattice_shard(self.st.corr.data_ptr(), self.n, self.d, d,
                                            nat.ptr(self.eta), kst, self.lo, self.hi, shard,
                                            shard_bits, out.data_ptr(), self.ws.data_ptr(),
                                            self.ws.numel(), s), "lattice_shard")
        self._table_ok = False
        return out


def shard_set_rows(n: int, lo: int, hi: int, shard_mask: int, shard_bits: int) -> np.ndarray:
    """Global ranks owned by the block shards in `shard_mask` (host model of
    hoi_lattice_shard_set's partition, for tests)."""
    parts = [shard_rows(n, lo, hi, c, shard_bits) for c in range(1 << shard_bits)
             if (shard_mask >> c) & 1]
    return np.sort(np.concatenate(parts)) if parts else np.zeros(0, dtype=np.int64)


def shard_rows(n: int, lo: int, hi: int, shard: int, shard_bits: int) -> np.ndarray:
    """Global ranks owned by block shard `shard` of 2^shard_bits (host
    model of hoi_lattice_shard's partition, for tests): the n-plets whose
    membership pattern over variables n-10-shard_bits .. n-11 equals shard."""
    import itertools
    lo_var = n - 10 - shard_bits
    rows, g = [], 0
    for k in range(lo, hi + 1):
        for c in itertools.combinations(range(n), k):
            pat = sum(1 << (v - lo_var) for v in c if lo_var <= v < n - 10)
            if pat == shard:
                rows.append(g)
            g += 1
    return np.asarray(rows, dtype=np.int64)


def read_scan(path):
    """(header dict, (4, rows, D) float64 memmap) of a file written by
    DeviceScan.save (host only; no device needed)."""
    import json
    with open(path, "rb") as f:
        head = json.loads(f.read(4096).decode())
    if head.get("format") != "hoi-b200-scan/1":
        raise InvalidData(f"{path}: not a hoi-b200 scan file")
    rows = head["g_end"] - head["g_begin"]
    planes = np.memmap(path, dtype=np.float64, mode="r", offset=head["header_bytes"],
                       shape=(4, rows, head["datasets"]))
    return head, planes


@nat.traced("hoi.scan_device")
def scan_device(covs: CovSet, min_order: int, max_order: int, *, bias_correct: bool = False,
                g_begin: int = 0, g_end: int | None = None, engine: int = 0,
                out=None) -> DeviceScan:
    """Exhaustive full-output scan kept on the device (extension of the
    reference API: the equivalent of collecting every batch of
    ``scan(..., Callback(...))`` without leaving HBM)."""
    n = covs.n_variables
    total = count_nplets(n, min_order, max_order)
    g_end = total if g_end is None else g_end
    if not 0 <= g_begin <= g_end <= total:
        raise InvalidData(f"rank range [{g_begin}, {g_end}) outside [0, {total})")
    if n > 64:
        # beyond the device unranking table: host-enumerated index batches
        # (the reference's itertools order), measures computed on the device
        # straight into the resident output
        from .nplet_engine import eval_device
        torch = nat.torch_cuda()
        d = covs.n_datasets
        o = out if out is not None else torch.empty((4, g_end - g_begin, d),
                                                    dtype=torch.float64, device="cuda")
        for r0, k, idx in _host_batches(n, min_order, max_order, 1 << 18, g_begin, g_end):
            h, _, _ = eval_device(covs, NpletBatch(n, indices=idx, check_unique=False),
                                  bias_correct, measures=True)
            o[:, r0 - g_begin:r0 - g_begin + idx.shape[0]] = h
        return DeviceScan(o, n, min_order, max_order, g_begin, g_end)
    ctx = _ScanCtx(covs, min_order, max_order, bias_correct, engine)
    o, cnt, coords = ctx.full(g_begin, g_end, out)
    _raise_not_pd(cnt, coords)
    return DeviceScan(o, n, min_order, max_order, g_begin, g_end)


def _host_batches(n, lo, hi, batch_size, g_begin=0, g_end=None):
    """(global rank of the first row, order, (m, k) int64 indices) for the
    rows [g_begin, g_end) of the order-major lexicographic scan, batches of
    at most batch_size rows never crossing an order, from itertools (the
    reference's enumeration, ref:nplet_engine.py:128-136; used for N > 64)."""
    off = 0
    for k in range(lo, hi + 1):
        c = math.comb(n, k)
        a = max(g_begin - off, 0)
        b = c if g_end is None else min(c, g_end - off)
        if a < b:
            it = itertools.islice(itertools.combinations(range(n), k), a, b)
            g = off + a
            while True:
                flat = np.fromiter(itertools.chain.from_iterable(itertools.islice(it, batch_size)),
                                   dtype=np.int64)
                if flat.size == 0:
                    break
                idx = flat.reshape(-1, k)
                yield g, k, idx
                g += idx.shape[0]
        off += c
        if g_end is not None and off >= g_end:
            return


def _batch_bounds(n, lo, hi, batch_size):
    """The reference's batch sequence as (g_start, g_stop, order)."""
    off = 0
    for k in range(lo, hi + 1):
        c = math.comb(n, k)
        for s in range(0, c, batch_size):
            yield off + s, off + min(s + batch_size, c), k
        off += c


def _chunk_rows(d: int, torch, cap_bytes: int = 64 << 30, extra_per_row: int = 0) -> int:
    """Rows per device chunk: 32 B x D of output per row (+ any per-row
    staging) within 60% of the free device memory, capped at cap_bytes."""
    free, _ = torch.cuda.mem_get_info()
    # memory held in torch's cache is free for our next allocation too
    free += torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
    budget = min(int(free * 0.6), cap_bytes)
    return max(1 << 16, budget // (4 * 8 * d + extra_per_row))


def _unrank_list(n, lo, hi, ranks):
    """Index tuples of the given global ranks (device unranking)."""
    torch = nat.torch_cuda()
    r = torch.as_tensor(np.asarray(ranks, dtype=np.int64), device="cuda")
    m = r.numel()
    if m == 0:
        return []
    idx = torch.empty((m, hi), dtype=torch.int32, device="cuda")
    orders = torch.empty(m, dtype=torch.int32, device="cuda")
    nat.check(nat.lib().hoi_unrank_list(n, lo, hi, r.data_ptr(), m, idx.data_ptr(),
                                        orders.data_ptr(), nat.stream_handle(torch)), "unrank_list")
    hi_idx, ho = idx.cpu().numpy().tolist(), orders.cpu().numpy().tolist()
    return [tuple(row[:k]) for row, k in zip(hi_idx, ho)]


def _scan_stream(ctx, covs, reducer, batch_size, progress, total, t0):
    torch = ctx.torch
    from .nplet_engine import unrank_device
    bounds = list(_batch_bounds(ctx.n, ctx.lo, ctx.hi, batch_size))
    # host-side staging size; unranked indices add 4 B x max order per row
    per_chunk = _chunk_rows(ctx.d, torch, cap_bytes=1 << 30, extra_per_row=4 * ctx.hi)
    i, seen, nb = 0, 0, 0
    while i < len(bounds):
        j, rows = i, 0
        while j < len(bounds) and (rows == 0 or rows + bounds[j][1] - bounds[j][0] <= per_chunk):
            rows += bounds[j][1] - bounds[j][0]
            j += 1
        g0, g1 = bounds[i][0], bounds[j - 1][1]
        out, cnt, coords = ctx.full(g0, g1, reuse_table=i > 0)
        try:
            _raise_not_pd(cnt, coords)
        except Exception as e:  # map to the reference's per-batch coordinates
            if getattr(e, "coords", None):
                r0 = e.coords[0][0]
                bsel = next(b for b in bounds[i:j] if b[0] <= g0 + r0 < b[1])
                e.coords = [(g0 + r - bsel[0], d) for r, d in e.coords if bsel[0] <= g0 + r < bsel[1]]
            raise
        idx, _ = unrank_device(ctx.n, ctx.lo, ctx.hi, g0, g1 - g0)
        host = out.cpu().numpy()
        hidx = idx.cpu().numpy().astype(np.int64)
        for (a, b, k) in bounds[i:j]:
            ra, rb = a - g0, b - g0
            batch = NpletBatch(ctx.n, indices=hidx[ra:rb, :k], check_unique=False)
            hoi = HoiBatch(tc=host[0, ra:rb], dtc=host[1, ra:rb], o=host[2, ra:rb],
                           s=host[3, ra:rb], order=np.full(rb - ra, k, dtype=np.int64))
            reducer.update(batch, hoi)
            nb += 1
            seen += rb - ra
            if progress is not None:
                progress({"batches": nb, "nplets": seen, "total": total, "order": int(k),
                          "elapsed": time.perf_counter() - t0})
        i = j


def _emit_progress(progress, n, lo, hi, batch_size, total, t0):
    if progress is None:
        return
    seen = 0
    for i, (a, b, k) in enumerate(_batch_bounds(n, lo, hi, batch_size)):
        seen += b - a
        progress({"batches": i + 1, "nplets": seen, "total": total, "order": int(k),
                  "elapsed": time.perf_counter() - t0})


@_gc_paused
def _topk_plane(ctx, reducer, out, g0, m_idx, tuples_of=None):
    """Merge one device chunk into the running per-dataset TopK lists.

    The device radix-selects the k smallest keys sign*value (plus the rest
    of the k-th key's final radix bucket, so every tie is present); only
    those candidates reach the host, where the reference's exact key
    (sign*value, index tuple) orders them.  tuples_of(positions) gives the
    index tuples of rows (default: device unranking of the scan ranks)."""
    torch = ctx.torch
    lib = nat.lib()
    rows = out.shape[1]
    sign = reducer.sign
    reducer._materialize()
    if reducer._best is None:
        reducer._best = [[] for _ in range(ctx.d)]
    plane = out[m_idx]
    # the multi-dataset select resolves 8 bits per pass, so it can narrow
    # the k-th key's bucket to a few entries cheaply
    bucket_cap = 64 if ctx.d > 1 else max(4096, reducer.k)
    cap = reducer.k + max(bucket_cap, 4096) + 1
    s = nat.stream_handle(torch)
    if ctx.d > 1:
        # every dataset of the plane in one multi-dataset radix select
        cands = torch.empty((ctx.d, cap), dtype=torch.int64, device="cuda")
        ws = torch.empty(ctx.d * 256 + 5 * ctx.d + 32, dtype=torch.int64, device="cuda")
        hc = (ctypes.c_int64 * ctx.d)()
        nat.check(lib.hoi_topk_select_multi(plane.data_ptr(), rows, ctx.d, sign, reducer.k,
                                            bucket_cap, cands.data_ptr(), cap, hc,
                                            ws.data_ptr(), s), "topk_select_multi")
        counts = [int(hc[d]) for d in range(ctx.d)]
    else:
        cands = torch.empty((1, cap), dtype=torch.int64, device="cuda")
        ws = torch.empty(4096 + 64, dtype=torch.int64, device="cuda")
        cnt = ctypes.c_int64(0)
        nat.check(lib.hoi_topk_select(plane.data_ptr(), rows, 1, 0, sign, reducer.k, bucket_cap,
                                      cands.data_ptr(), cap, ctypes.byref(cnt), ws.data_ptr(), s),
                  "topk_select")
        counts = [int(cnt.value)]
    # every dataset's candidates in one gather and one device->host copy
    ok = [d for d in range(ctx.d) if counts[d] <= cap]
    if ok:
        cnt_t = torch.tensor([counts[d] for d in ok], dtype=torch.int64)
        d_sel = torch.repeat_interleave(torch.tensor(ok, dtype=torch.int64), cnt_t).to("cuda")
        pos_all = torch.cat([cands[d, :counts[d]] for d in ok])
        vals_all = out[:, pos_all, d_sel].cpu().numpy()            # (4, sum c)
        pos_all = pos_all.cpu().numpy()
    a = 0
    for d in range(ctx.d):
        c = counts[d]
        if c > cap:
            # a tie wider than the candidate buffer at the k-th value (e.g.
            # identical covariances): resolve it with the reference's host
            # rule over the chunk, slice by slice
            if tuples_of is None:
                _topk_host_slices(ctx, reducer, out, g0, d)
            else:
                _topk_host_rows(reducer, out, d, tuples_of)
            continue
        vals, pos = vals_all[:, a:a + c], pos_all[a:a + c]
        a += c
        if c > reducer.k:
            # keep the k best keys and every tie at the k-th before building
            # Python objects (the exact tuple tie-break happens in _merge)
            key = sign * vals[m_idx]
            keep = np.flatnonzero(key <= np.partition(key, reducer.k - 1)[reducer.k - 1])
            vals, pos = vals[:, keep], pos[keep]
            c = keep.size
        if tuples_of is not None:
            tuples = tuples_of(pos)
        else:
            tuples = _unrank_list(ctx.n, ctx.lo, ctx.hi, pos + g0) if c else []
        new = []
        for t, (tc, dtc, o, sv) in zip(tuples, vals.T.tolist()):
            v = (tc, dtc, o, sv)[m_idx]
            new.append(((sign * v, t), _entry(t, v, tc, dtc, o, sv)))
        reducer._merge(d, new)


def _topk_host_rows(reducer, out, d, tuples_of):
    """The reference's host TopK rule over one dataset of a device batch."""
    v = out[:, :, d].cpu().numpy()
    rows = v.shape[1]
    sub = TopK(reducer.measure, reducer.direction, reducer.k)
    sign = reducer.sign
    key = sign * v[MEASURES.index(reducer.measure)]
    k_eff = min(reducer.k, rows)
    thr = np.partition(key, k_eff - 1)[k_eff - 1]
    sel = np.flatnonzero(key <= thr)
    tuples = tuples_of(sel)
    new = []
    for i, t in zip(sel, tuples):
        e = TopEntry(indices=t, order=len(t), value=float(v[MEASURES.index(reducer.measure), i]),
                     tc=float(v[0, i]), dtc=float(v[1, i]), o=float(v[2, i]), s=float(v[3, i]))
        new.append(((sign * e.value, t), e))
    sub._best = [[]]
    sub._merge(0, new)
    reducer._merge(d, sub._best[0])


def _topk_host_slices(ctx, reducer, out, g0, d, step=1 << 20):
    from .nplet_engine import unrank_device
    rows = out.shape[1]
    sub = TopK(reducer.measure, reducer.direction, reducer.k)
    for a in range(0, rows, step):
        b = min(rows, a + step)
        idx, orders = unrank_device(ctx.n, ctx.lo, ctx.hi, g0 + a, b - a)
        hidx, ho = idx.cpu().numpy(), orders.cpu().numpy()
        v = out[:, a:b, d:d + 1].cpu().numpy()
        for k in np.unique(ho):
            sel = np.flatnonzero(ho == k)
            batch = NpletBatch(ctx.n, indices=hidx[sel, :k].astype(np.int64), check_unique=False)
            sub.update(batch, HoiBatch(tc=v[0, sel], dtc=v[1, sel], o=v[2, sel], s=v[3, sel],
                                       order=np.full(sel.size, k, dtype=np.int64)))
    reducer._merge(d, sub._best[0])


@_gc_paused
def _topk_lattice(ctx, reducer, m_idx, shard=0, shard_bits=0, shard_mask=None):
    """TopK over an exhaustive scan without writing the full output (lattice
    engine): per dataset, (1) build the log-det table; (2) run the filtered
    stencil over a hash-sampled 1/256 of the table blocks with no threshold
    and take an upper bound of the k-th smallest key of that sample (its
    top 36 bits resolved) -- any subset's k-th smallest key bounds the
    global k-th smallest from above, so every true top-k n-plet passes it;
    (3) one filtered stencil pass over all blocks keeps
    only the n-plets at or under that key; (4) an exact radix select over
    those candidates hands the k best (plus every tie at the k-th key) to
    the reference's host merge (sign*value, index tuple).  Returns False
    when the engine declines (not PD) or the sample is smaller than k; the
    caller then takes the full-output path.  shard_bits > 0: only the
    n-plets of block shard `shard`, or of the shards in `shard_mask`
    (multi-GPU; see ScanCtx.full_shard_set)."""
    mask = (1 << shard) if shard_mask is None else int(shard_mask)
    torch, lib = ctx.torch, nat.lib()
    s = nat.stream_handle(torch)
    n = ctx.n
    kst = 0 if ctx.eta is None else ctx.eta.shape[1]
    k, sign = reducer.k, reducer.sign
    nblocks = 1 << (n - 10)
    every = 256 if nblocks >= (1 << 14) else 1
    ws_sel = torch.empty(4096 + 64, dtype=torch.int64, device="cuda")
    key = torch.empty(1, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    best = [[] for _ in range(ctx.d)]
    for d in range(ctx.d):
        if shard_bits == 0:
            rc = lib.hoi_lattice_table(ctx.st.corr.data_ptr(), n, ctx.d, d, ctx.ws.data_ptr(),
                                       ctx.ws.numel(), s)
            nat.check(rc, "lattice_table")
            rc = lib.hoi_lattice_status(ctx.ws.data_ptr(), n, s)
            if rc == nat.FALLBACK:
                return False
            nat.check(rc, "lattice_status")
        built = [False]

        def filt(every_, cap):
            cand = torch.empty((max(cap, 1), 5), dtype=torch.float64, device="cuda")
            cnt.zero_()
            if shard_bits == 0:
                rc = lib.hoi_lattice_filter(ctx.ws.data_ptr(), n, ctx.d, d, nat.ptr(ctx.eta), kst,
                                            ctx.lo, ctx.hi, m_idx, sign, every_, key.data_ptr(),
                                            cand.data_ptr(), cap, cnt.data_ptr(), s)
            else:
                rc = lib.hoi_lattice_shard_set_filter(
                    ctx.st.corr.data_ptr(), n, ctx.d, d, nat.ptr(ctx.eta), kst, ctx.lo, ctx.hi,
                    mask, shard_bits, every_, m_idx, sign, key.data_ptr(), cand.data_ptr(), cap,
                    cnt.data_ptr(), 0 if built[0] else 1, ctx.ws.data_ptr(), ctx.ws.numel(), s)
                if rc == nat.FALLBACK:
                    return None, -1
                built[0] = True
            nat.check(rc, "lattice_filter")
            return cand, int(cnt.item())

        key.fill_(-1)                                   # all-ones key: no threshold
        if every > 1:
            cap = (nblocks // every + 1) * 1024         # every row of the sampled blocks
            cand, c = filt(every, cap)
            if c <= k:
                return False
            # an upper bound of the sample's k-th key is all the filter needs:
            # 3 synchronous radix rounds (36 bits) instead of 6 for the exact key
            nat.check(lib.hoi_topk_bound(cand.data_ptr(), c, 5, 1 + m_idx, sign, k, 36,
                                         key.data_ptr(), ws_sel.data_ptr(), s),
                      "topk_bound")
            del cand
            cap = max(16 * every * k, 1 << 20)
        else:
            cap = count_nplets(n, ctx.lo, ctx.hi)
        cand, c = filt(1, cap)
        if c < 0:
            return False
        if c > cap:                                     # loose sample: exact size, once more
            cand, c = filt(1, c)
        # exact k best (+ ties at the k-th key) among the candidates
        sel_cap = 2 * k + 4096 + 1
        pos = torch.empty(sel_cap, dtype=torch.int64, device="cuda")
        hc = ctypes.c_int64(0)
        nat.check(lib.hoi_topk_select(cand.data_ptr(), c, 5, 1 + m_idx, sign, k, k + 4096,
                                      pos.data_ptr(), sel_cap, ctypes.byref(hc),
                                      ws_sel.data_ptr(), s), "topk_select")
        h = int(hc.value)
        if h > sel_cap:                                 # a tie wider than the buffer
            pos = torch.arange(c, device="cuda")
            h = c
        rec = cand[pos[:h]].cpu().numpy()
        ranks = rec[:, 0].view(np.int64)
        tuples = _unrank_list(n, ctx.lo, ctx.hi, ranks) if h else []
        for t, r in zip(tuples, rec[:, 1:].tolist()):
            v = r[m_idx]
            best[d].append(((sign * v, t), _entry(t, v, *r)))
    if reducer._best is None:
        reducer._best = [[] for _ in range(ctx.d)]
    for d in range(ctx.d):
        reducer._merge(d, best[d])
    ctx._table_ok = ctx.d == 1
    return True


class _BatchCtx:
    """The fields _topk_plane reads, for a user batch on the device."""

    def __init__(self, d, torch):
        self.d, self.torch = d, torch


@nat.traced("hoi.topk_batch")
def topk_batch(covs: CovSet, batch: NpletBatch, reducer: TopK, *, bias_correct: bool = False,
               precision: str = "fp64"):
    """``reducer.update(batch, compute_hoi_batch(covs, batch, bias_correct))``
    with the selection on the device (ref:scanner.py:75-100 semantics):
    the four measures of the batch stay in HBM, a radix select per dataset
    keeps the k best keys plus every tie, and only those rows reach the
    reference's host merge (sign*value, index tuple).  Extension of the
    reference API for large user batches (the greedy/anneal candidate
    evaluations and BASELINE config 5: 4M order-10 n-plets x 16 datasets)."""
    if not isinstance(reducer, TopK):
        raise InvalidData("topk_batch needs a TopK reducer")
    from .nplet_engine import eval_device
    keep = []
    out, _, _ = eval_device(covs, batch, bias_correct, measures=True, terms=False,
                            precision=precision, keep_idx=keep)
    ctx = _BatchCtx(out.shape[2], nat.torch_cuda())
    if (batch.mode == "fixed" and reducer._best is None and reducer._compact is None
            and keep and 1 <= ctx.d <= 64 and reducer.k <= _ORDER_MAX // 2):
        if _topk_batch_device(ctx, reducer, out, keep[0], batch):
            return reducer

    def tuples_of(pos):
        if batch.mode == "fixed":
            return [tuple(r) for r in batch.indices[np.asarray(pos, dtype=np.int64)].tolist()]
        return [batch.row_indices(int(i)) for i in pos]

    _topk_plane(ctx, reducer, out, 0, MEASURES.index(reducer.measure), tuples_of)
    return reducer


_ORDER_MAX = 8192     # candidates per dataset that hoi_topk_order sorts on chip


def _topk_batch_device(ctx, reducer, out, idx_dev, batch) -> bool:
    """The whole TopK of a fixed-order batch on the device: multi-dataset
    radix select (the k best keys + every tie at the k-th), then
    hoi_topk_order sorts each dataset's candidates by the reference's key
    (sign*value, index tuple) and keeps k; only the (D, k) winners and their
    four measures reach the host, as arrays (TopEntries).  False when a tie
    is wider than the on-chip sort (the caller's host path then decides)."""
    torch = ctx.torch
    lib = nat.lib()
    s = nat.stream_handle(torch)
    rows, d, k = out.shape[1], ctx.d, reducer.k
    m_idx = MEASURES.index(reducer.measure)
    plane = out[m_idx]
    cap = _ORDER_MAX
    bucket = min(64, cap - k - 1)
    cands = torch.empty((d, cap), dtype=torch.int64, device="cuda")
    ws = torch.empty(d * 256 + 5 * d + 32, dtype=torch.int64, device="cuda")
    hc = (ctypes.c_int64 * d)()
    nat.check(lib.hoi_topk_select_multi(plane.data_ptr(), rows, d, reducer.sign, k, bucket,
                                        cands.data_ptr(), cap, hc, ws.data_ptr(), s),
              "topk_select_multi")
    counts = [int(hc[i]) for i in range(d)]
    if max(counts) > cap:
        return False
    cnt = torch.tensor(counts, dtype=torch.int64).to("cuda", non_blocking=True)
    top = torch.empty((d, k), dtype=torch.int64, device="cuda")
    kk = int(idx_dev.shape[1])
    nat.check(lib.hoi_topk_order(plane.data_ptr(), d, reducer.sign, cands.data_ptr(), cap,
                                 cnt.data_ptr(), idx_dev.data_ptr(), kk, k, top.data_ptr(), s),
              "topk_order")
    m = min(k, rows)
    sel = top[:, :m]
    dsel = torch.arange(d, device="cuda")[:, None].expand(d, m)
    vals = out[:, sel, dsel].cpu().numpy()                     # (4, D, m)
    pos = sel.cpu().numpy()
    tuples = batch.indices[pos]                                # (D, m, K)
    reducer._compact = [TopEntries(tuples[i], vals[:, i], m_idx) for i in range(d)]
    return True


def _feature_chunks(ctx, total):
    """Canonical chunks of the feature reduction: a fixed power-of-two row
    count that depends only on D (32 B x D per row, <= 8 GB), so the
    partial sums -- and hence the features, to the last bit -- are the same
    however many ranks share the chunks (sharding.scan_sharded)."""
    rows = 1 << 28
    while rows > (1 << 16) and rows * 32 * ctx.d > (8 << 30):
        rows >>= 1
    return [(g, min(total, g + rows)) for g in range(0, total, rows)]


def _feature_partial(ctx, g0, g1):
    """hoi_features over global ranks [g0, g1): the (D, 19) partials (sums,
    extrema with the first global rank attaining the o extremes, counts) and,
    when the chunk holds it, the whole-system row (D, 4)."""
    torch, lib = ctx.torch, nat.lib()
    n, d_count = ctx.n, ctx.d
    offs, acc = [], 0
    for k in range(ctx.lo, ctx.hi + 1):
        offs.append(acc)
        acc += math.comb(n, k)
    pb = pe = 0
    if ctx.lo <= 2 <= ctx.hi:
        pb = offs[2 - ctx.lo]
        pe = pb + math.comb(n, 2)
    whole_rank = offs[n - ctx.lo] if ctx.lo <= n <= ctx.hi else -1
    feat = torch.empty((d_count, 19), dtype=torch.float64, device="cuda")
    ws_doubles = 8 * 148 * 256 * 19
    ws = torch.empty(ws_doubles, dtype=torch.float64, device="cuda")
    out, cnt, coords = ctx.full(g0, g1, reuse_table=getattr(ctx, "_table_ok", False))
    _raise_not_pd(cnt, coords)
    nat.check(lib.hoi_features(out.data_ptr(), g1 - g0, d_count, g0, pb, pe, feat.data_ptr(),
                               ws.data_ptr(), ws_doubles, nat.stream_handle(torch)), "features")
    whole = None
    if g0 <= whole_rank < g1:
        whole = out[:, whole_rank - g0, :].cpu().numpy().T.copy()
    return feat.cpu().numpy(), whole


def _feature_merge(ctx, reducer, parts):
    """Merge (g0, (partials, whole)) chunks, in enumeration order, into the
    accumulator's own state, so finalize() is the reference's
    (ref:scanner.py:231-287)."""
    n, d_count = ctx.n, ctx.d
    if reducer._d is None:
        reducer._init_state(d_count)
    offs, acc = [], 0
    for k in range(ctx.lo, ctx.hi + 1):
        offs.append(acc)
        acc += math.comb(n, k)
    offs_np = np.asarray(offs, dtype=np.int64)

    def order_of(rank):
        return ctx.lo + int(np.searchsorted(offs_np, rank, side="right")) - 1

    for _, (f, whole) in parts:
        reducer._mi_count += int(f[0, 0])
        reducer._mi_sum += f[:, 1]
        reducer._mi_sumsq += f[:, 2]
        reducer._count += int(f[0, 3])
        reducer._sums += f[:, 4:8]
        reducer._syn += f[:, 18].astype(np.int64)
        for d in range(d_count):
            if f[d, 3] == 0:
                continue
            if f[d, 10] > reducer._maxs[d, 2]:
                reducer._o_max_order[d] = order_of(int(f[d, 16]))
            if f[d, 14] < reducer._mins[d, 2]:
                reducer._o_min_order[d] = order_of(int(f[d, 17]))
        np.maximum(reducer._maxs, f[:, 8:12], out=reducer._maxs)
        np.minimum(reducer._mins, f[:, 12:16], out=reducer._mins)
        if whole is not None:
            reducer._whole = whole


def _scan_device_features(ctx, reducer, batch_size, progress, total, t0):
    """FeatureAccumulator over device full-output chunks: hoi_features
    reduces each canonical chunk to 19 partials per dataset on the device;
    the host merges them in enumeration order into the accumulator's own
    state (ref:scanner.py:231-287)."""
    parts = [(g0, _feature_partial(ctx, g0, g1)) for g0, g1 in _feature_chunks(ctx, total)]
    _feature_merge(ctx, reducer, parts)
    _emit_progress(progress, ctx.n, ctx.lo, ctx.hi, batch_size, total, t0)


def _scan_device_reduce(ctx, reducer, batch_size, progress, total, t0):
    torch = ctx.torch
    if isinstance(reducer, TopK) and ctx.engine == 2 and _topk_lattice(
            ctx, reducer, MEASURES.index(reducer.measure)):
        _emit_progress(progress, ctx.n, ctx.lo, ctx.hi, batch_size, total, t0)
        return
    per_chunk = _chunk_rows(ctx.d, torch)
    hist_counts = None
    if isinstance(reducer, Histogram):
        edges = torch.from_numpy(reducer.edges).cuda()
        hist_counts = torch.zeros((ctx.d, len(reducer.edges) - 1), dtype=torch.int64, device="cuda")
    m_idx = MEASURES.index(reducer.measure)
    g0 = 0
    while g0 < total:
        g1 = min(total, g0 + per_chunk)
        out, cnt, coords = ctx.full(g0, g1, reuse_table=g0 > 0)
        _raise_not_pd(cnt, coords)
        if hist_counts is not None:
            nat.check(nat.lib().hoi_histogram(
                out[m_idx].data_ptr(), g1 - g0, ctx.d, len(reducer.edges) - 1,
                float(reducer.edges[0]), float(reducer.edges[-1]), edges.data_ptr(),
                hist_counts.data_ptr(), nat.stream_handle(torch)), "histogram")
        else:
            _topk_plane(ctx, reducer, out, g0, m_idx)
        g0 = g1
    if hist_counts is not None:
        c = hist_counts.cpu().numpy()
        reducer._counts = c if reducer._counts is None else reducer._counts + c
    _emit_progress(progress, ctx.n, ctx.lo, ctx.hi, batch_size, total, t0)


@nat.traced("hoi.scan")
def scan(covs: CovSet, min_order: int, max_order: int, reducer: Reducer, *,
         batch_size: int = 10000, bias_correct: bool = False, workers: int = 1, progress=None):
    """Visit every n-plet with order in [min_order, max_order] once
    (ref:scanner.py:308-365); returns reducer.finalize()."""
    if not isinstance(reducer, Reducer):
        raise InvalidData("reducer must be a Reducer instance")
    n = covs.n_variables
    total = count_nplets(n, min_order, max_order)
    if workers < 1:
        raise InvalidData(f"workers must be >= 1, got {workers}")
    if batch_size < 1:
        raise InvalidData(f"batch_size must be >= 1, got {batch_size}")
    t0 = time.perf_counter()
    if n > 64:
        # beyond the unranking table: host-enumerated batches, device math
        seen = 0
        nb = 0
        for _, k, idx in _host_batches(n, min_order, max_order, batch_size):
            batch = NpletBatch(n, indices=idx, check_unique=False)
            reducer.update(batch, compute_hoi_batch(covs, batch, bias_correct=bias_correct))
            nb += 1
            seen += batch.batch_size
            if progress is not None:
                progress({"batches": nb, "nplets": seen, "total": total, "order": k,
                          "elapsed": time.perf_counter() - t0})
        return reducer.finalize()
    ctx = _ScanCtx(covs, min_order, max_order, bias_correct)
    if type(reducer) in (TopK, Histogram):
        _scan_device_reduce(ctx, reducer, batch_size, progress, total, t0)
    elif type(reducer) is FeatureAccumulator and reducer.n == n:
        _scan_device_features(ctx, reducer, batch_size, progress, total, t0)
    else:
        _scan_stream(ctx, covs, reducer, batch_size, progress, total, t0)
    return reducer.finalize()


@nat.traced("hoi.extract_features")
def extract_features(covs: CovSet, *, bias_correct: bool = False, limit: int = 20,
                     batch_size: int = 10000, workers: int = 1, progress=None):
    """21 features per dataset from one scan of orders 2..N (ref:scanner.py:368-387)."""
    n = covs.n_variables
    if n > limit:
        raise ExhaustiveLimitExceeded(
            f"N={n} exceeds the exhaustive feature limit ({limit}); use greedy or annealing search")
    if n < 3:
        raise InvalidOrderRange(f"feature extraction needs N >= 3, got {n}")
    return scan(covs, 2, n, FeatureAccumulator(n), batch_size=batch_size,
                bias_correct=bias_correct, workers=workers, progress=progress)
