"""N-plet batches, enumeration and batched entropy terms on the B200.

Drop-in for ref:nplet_engine.py.  NpletBatch keeps the reference's
validation; enumeration is the device unranking kernel (bit-exact with
itertools.combinations order); every log-determinant / inverse diagonal is
computed by the library's per-n-plet LDL^T kernel with the reference's
single jitter retry.
"""

from __future__ import annotations

import ctypes
import itertools
import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from ._device import device_covs
from .copula_core import NORMAL_ENTROPY, CovSet
from .errors import InvalidData, InvalidNplet, InvalidOrderRange, NotPositiveDefinite

ERR_CAP = 1 << 16


def count_nplets(n: int, min_order: int, max_order: int) -> int:
    """Number of subsets with size in [min_order, max_order] (ref:nplet_engine.py:26-33)."""
    if not 1 <= min_order <= max_order <= n:
        raise InvalidOrderRange(
            f"need 1 <= min_order <= max_order <= n, "
            f"got min={min_order}, max={max_order}, n={n}")
    return sum(math.comb(n, k) for k in range(min_order, max_order + 1))


class NpletBatch:
    """B n-plets over N variables, as (B, K) indices or (B, N) masks
    (ref:nplet_engine.py:36-115)."""

    def __init__(self, n_variables: int, indices=None, masks=None, check_unique: bool = True):
        if (indices is None) == (masks is None):
            raise InvalidNplet("provide exactly one of indices or masks")
        if n_variables < 1:
            raise InvalidData(f"n_variables must be >= 1, got {n_variables}")
        self.n_variables = int(n_variables)
        if indices is not None:
            idx = np.asarray(indices, dtype=np.int64)
            if idx.ndim != 2 or idx.shape[0] < 1 or idx.shape[1] < 1:
                raise InvalidNplet(f"indices must be a nonempty 2-D array, got shape {idx.shape}")
            if idx.min() < 0 or idx.max() >= n_variables:
                raise InvalidNplet(f"indices out of range for N={n_variables}")
            if idx.shape[1] > 1 and not (np.diff(idx, axis=1) > 0).all():
                raise InvalidNplet("index rows must be strictly increasing")
            if check_unique and np.unique(idx, axis=0).shape[0] != idx.shape[0]:
                raise InvalidNplet("duplicate n-plets in batch")
            self.mode, self.indices, self.masks = "fixed", idx, None
        else:
            m = np.asarray(masks)
            if m.dtype != np.bool_:
                raise InvalidNplet("masks must be boolean")
            if m.ndim != 2 or m.shape[0] < 1 or m.shape[1] != n_variables:
                raise InvalidNplet(f"masks must have shape (B, {n_variables}), got {m.shape}")
            if not m.any(axis=1).all():
                raise InvalidNplet("every mask must select at least one variable")
            if check_unique and np.unique(m, axis=0).shape[0] != m.shape[0]:
                raise InvalidNplet("duplicate n-plets in batch")
            self.mode, self.indices, self.masks = "mixed", None, m

    @property
    def batch_size(self) -> int:
        return (self.indices if self.mode == "fixed" else self.masks).shape[0]

    @property
    def order(self) -> int:
        if self.mode != "fixed":
            raise InvalidNplet("mixed-order batch has no single order")
        return self.indices.shape[1]

    def orders(self) -> np.ndarray:
        if self.mode == "fixed":
            return np.full(self.batch_size, self.indices.shape[1], dtype=np.int64)
        return self.masks.sum(axis=1).astype(np.int64)

    def row_indices(self, i: int) -> tuple:
        if self.mode == "fixed":
            return tuple(int(v) for v in self.indices[i])
        return tuple(int(v) for v in np.flatnonzero(self.masks[i]))

    def to_masks(self) -> np.ndarray:
        if self.mode == "mixed":
            return self.masks
        out = np.zeros((self.batch_size, self.n_variables), dtype=bool)
        np.put_along_axis(out, self.indices, True, axis=1)
        return out


def unrank_device(n: int, kmin: int, kmax: int, g0: int, count: int):
    """(count, kmax) int32 device tensor of the n-plets at global
    order-major lexicographic ranks [g0, g0+count) plus their orders."""
    torch = nat.torch_cuda()
    idx = torch.empty((max(count, 1), kmax), dtype=torch.int32, device="cuda")
    orders = torch.empty((max(count, 1),), dtype=torch.int32, device="cuda")
    nat.check(nat.lib().hoi_unrank(n, kmin, kmax, g0, count, idx.data_ptr(), orders.data_ptr(),
                                   nat.stream_handle(torch)), "unrank")
    return idx[:count], orders[:count]


def enumerate_order(n: int, k: int, batch_size: int = 10000):
    """Every C(n, k) combination once, lexicographic, in chunks of at most
    batch_size rows (ref:nplet_engine.py:118-136); rows come from the
    device unranking kernel."""
    if not 1 <= k <= n:
        raise InvalidOrderRange(f"need 1 <= k <= n, got k={k}, n={n}")
    if batch_size < 1:
        raise InvalidData(f"batch_size must be >= 1, got {batch_size}")
    total = math.comb(n, k)
    if n > 64:
        # beyond the device unranking table (64-bit binomials, N <= 64): the
        # reference's own itertools walk, same batches
        it = itertools.combinations(range(n), k)
        while True:
            flat = np.fromiter(itertools.chain.from_iterable(itertools.islice(it, batch_size)),
                               dtype=np.int64)
            if flat.size == 0:
                return
            yield NpletBatch(n, indices=flat.reshape(-1, k), check_unique=False)
    chunk = max(batch_size, min(1 << 22, (total // batch_size + 1) * batch_size))
    chunk = (chunk // batch_size) * batch_size
    g = 0
    while g < total:
        m = min(chunk, total - g)
        idx, _ = unrank_device(n, k, k, g, m)
        host = idx.cpu().numpy().astype(np.int64)
        for lo in range(0, m, batch_size):
            yield NpletBatch(n, indices=host[lo:lo + batch_size], check_unique=False)
        g += m


@dataclass
class SubCovBatch:
    """(B, D, K, K) sub-covariances plus identity pad counts (ref:nplet_engine.py:139-151)."""

    matrices: np.ndarray
    pad_counts: np.ndarray


@dataclass
class EntropyTerms:
    """Entropy terms per (n-plet, dataset) in nats (ref:nplet_engine.py:154-181)."""

    h_joint: np.ndarray
    h_singles: np.ndarray
    h_leave_one_out: np.ndarray
    orders: np.ndarray
    excess_joint: np.ndarray | None = None
    excess_singles: np.ndarray | None = None
    excess_leave_one_out: np.ndarray | None = None


def _check_batch(covs, batch):
    if batch.n_variables != covs.n_variables:
        raise InvalidNplet(
            f"batch is over {batch.n_variables} variables, covariances over {covs.n_variables}")


def extract_subcov_batch(covs: CovSet, batch: NpletBatch) -> SubCovBatch:
    """Principal sub-matrices (B, D, K, K), gathered on the device
    (ref:nplet_engine.py:185-201)."""
    if batch.mode != "fixed":
        raise InvalidNplet("extract_subcov_batch needs a fixed-order batch")
    _check_batch(covs, batch)
    st = device_covs(covs)
    torch = st.torch
    idx = torch.from_numpy(batch.indices).cuda()
    sub = st.cov[:, idx[:, :, None], idx[:, None, :]].permute(1, 0, 2, 3)
    return SubCovBatch(matrices=sub.contiguous().cpu().numpy(),
                       pad_counts=np.zeros(batch.batch_size, dtype=np.int64))


def pad_subcov_batch(covs: CovSet, batch: NpletBatch) -> SubCovBatch:
    """Identity-padded (B, D, N, N) mixed-order matrices (ref:nplet_engine.py:204-224)."""
    if batch.mode != "mixed":
        raise InvalidNplet("pad_subcov_batch needs a mixed-order batch")
    _check_batch(covs, batch)
    st = device_covs(covs)
    torch = st.torch
    m = torch.from_numpy(batch.masks).cuda()
    keep = m[:, None, :, None] & m[:, None, None, :]
    eye = torch.eye(covs.n_variables, dtype=torch.float64, device="cuda")
    mats = torch.where(keep, st.cov[None], eye)
    return SubCovBatch(matrices=mats.cpu().numpy(),
                       pad_counts=(batch.n_variables - batch.masks.sum(axis=1)).astype(np.int64))


def _raise_not_pd(err_count, err_coords, unravel=None):
    n = int(err_count.item())
    if n == 0:
        return
    c = err_coords[: 2 * min(n, ERR_CAP)].cpu().numpy().reshape(-1, 2)
    coords = sorted((int(b), int(d)) for b, d in c)
    if unravel is not None:
        coords = sorted(unravel(b) for b, _ in coords)
    raise NotPositiveDefinite(
        f"{n} sub-covariance(s) not positive definite even after jitter, "
        f"first at (batch, dataset)={coords[0]}", coords=coords)


def _err_buffers(torch):
    return (torch.zeros(1, dtype=torch.int32, device="cuda"),
            torch.empty(2 * ERR_CAP, dtype=torch.int64, device="cuda"))


def _batched_logdet_invdiag(mats: np.ndarray):
    """(logdet, inverse diagonal) of a (..., K, K) stack with the
    reference's per-matrix jitter retry (ref:nplet_engine.py:227-281)."""
    torch = nat.torch_cuda()
    mats = np.asarray(mats, dtype=np.float64)
    lead, k = mats.shape[:-2], mats.shape[-1]
    m = int(np.prod(lead)) if lead else 1
    dm = torch.from_numpy(np.ascontiguousarray(mats.reshape(m, k, k))).cuda()
    ld = torch.empty(m, dtype=torch.float64, device="cuda")
    idg = torch.empty((m, k), dtype=torch.float64, device="cuda")
    cnt, coords = _err_buffers(torch)
    nat.check(nat.lib().hoi_logdet_invdiag(dm.data_ptr(), m, k, ld.data_ptr(), idg.data_ptr(),
                                           cnt.data_ptr(), coords.data_ptr(), ERR_CAP,
                                           nat.stream_handle(torch)), "logdet_invdiag")
    _raise_not_pd(cnt, coords, unravel=lambda b: tuple(int(v) for v in np.unravel_index(b, lead)))
    return ld.cpu().numpy().reshape(lead), idg.cpu().numpy().reshape(lead + (k,))


def _indices_to_device(indices, torch):
    """(B, k) host indices -> int32 device tensor: torch's multi-threaded
    int64->int32 conversion into a (cached) pinned buffer, then one async
    copy -- numpy's single-threaded astype plus a pageable copy cost ~55 ms
    for BASELINE config 5's 4M x 10 indices."""
    src = torch.from_numpy(np.ascontiguousarray(indices))
    if src.numel() * 4 > (256 << 20):
        # very large batches: no multi-GB pinned block held by torch's
        # caching host allocator; still a multi-threaded conversion
        return src.to(torch.int32).cuda()
    host = torch.empty(src.shape, dtype=torch.int32, pin_memory=True)
    host.copy_(src)
    return host.to("cuda", non_blocking=True)


_STREAM_ROWS = 1 << 19      # rows per chunk of a streamed index upload
_INT16_N = 1 << 15          # systems up to this size upload int16 variable ids


def index_upload_bytes(b: int, k: int, n: int) -> int:
    """Host-to-device bytes of a streamed (B, k) index batch over N variables."""
    return b * k * (2 if n <= _INT16_N else 4)
_stream_state = {}


def _eval_streamed(st, batch, eta, kstride, out, keep_idx):
    """A large fixed-order host batch, chunk by chunk: while chunk c's kernel
    runs, chunk c+1's indices are narrowed to int32 into a pinned buffer
    (torch's multi-threaded copy) and uploaded on a side stream, so the
    host conversion, the PCIe transfer and the FP64 kernel overlap instead
    of running back to back (BASELINE config 5: 4M x 10 indices, 160 MB)."""
    torch = st.torch
    lib = nat.lib()
    b, k = batch.indices.shape
    d, n = st.d, st.n
    dev = torch.cuda.current_device()
    # variable ids below 2^15 cross PCIe as int16 (half the bytes of the
    # upload that bounds this path) and are widened to the kernel's int32 on
    # the copy stream
    narrow = torch.int16 if n <= _INT16_N else torch.int32
    ss = _stream_state.get(dev)
    if ss is None or ss["pin"][0].shape[1] != k or ss["pin"][0].dtype != narrow:
        ss = {"copy": torch.cuda.Stream(),
              "pin": [torch.empty((_STREAM_ROWS, k), dtype=narrow, pin_memory=True)
                      for _ in range(2)],
              "stage": [torch.empty((_STREAM_ROWS, k), dtype=narrow, device="cuda")
                        for _ in range(2)] if narrow != torch.int32 else None}
        _stream_state[dev] = ss
    src = torch.from_numpy(np.ascontiguousarray(batch.indices))
    idx = torch.empty((b, k), dtype=torch.int32, device="cuda")
    nch = -(-b // _STREAM_ROWS)
    cnt = torch.zeros(nch, dtype=torch.int32, device="cuda")
    coords = torch.zeros((nch, 2 * ERR_CAP), dtype=torch.int64, device="cuda")
    main, copy = torch.cuda.current_stream(), ss["copy"]
    s = nat.stream_handle(torch)
    done = [None, None]                  # the upload that last read each pinned buffer
    plane = b * d
    for c in range(nch):
        r0, r1 = c * _STREAM_ROWS, min(b, (c + 1) * _STREAM_ROWS)
        pin = ss["pin"][c & 1]
        if done[c & 1] is not None:
            done[c & 1].synchronize()
        pin[:r1 - r0].copy_(src[r0:r1])
        with torch.cuda.stream(copy):
            if ss["stage"] is None:
                idx[r0:r1].copy_(pin[:r1 - r0], non_blocking=True)
            else:
                stage = ss["stage"][c & 1]
                stage[:r1 - r0].copy_(pin[:r1 - r0], non_blocking=True)
                idx[r0:r1].copy_(stage[:r1 - r0])
            ev = torch.cuda.Event()
            ev.record(copy)
        done[c & 1] = ev
        main.wait_event(ev)
        nat.check(lib.hoi_eval_indices_into(st.corr.data_ptr(), st.sdiag.data_ptr(), nat.ptr(eta),
                                            kstride, n, d, idx[r0].data_ptr(), r1 - r0, k,
                                            out[0, r0].data_ptr(), plane, cnt[c:].data_ptr(),
                                            coords[c].data_ptr(), ERR_CAP, s), "eval_indices_into")
    idx.record_stream(main)
    if keep_idx is not None:
        keep_idx.append(idx)
    if int(cnt.sum().item()):
        rows = []
        for c in range(nch):
            m = min(int(cnt[c].item()), ERR_CAP)
            pairs = coords[c, :2 * m].cpu().numpy().reshape(-1, 2)
            rows.extend((int(r) + c * _STREAM_ROWS, int(dd)) for r, dd in pairs)
        rows.sort()
        raise NotPositiveDefinite(
            f"{int(cnt.sum().item())} sub-covariance(s) not positive definite even after "
            f"jitter, first at (batch, dataset)={rows[0]}", coords=rows)
    return out


def eval_device(covs: CovSet, batch: NpletBatch, bias_correct: bool, *, measures: bool = True,
                terms: bool = False, precision: str = "fp64", keep_idx: list | None = None):
    """Run the fused per-n-plet kernel on a batch.  Returns device tensors
    (out (4, B, D) or None, logdet (B, D) or None, invdiag or None).
    precision="fp32": the FP32 fast path (index batches, measures only;
    within 1e-4 nats of FP64).  keep_idx (a list): receives the device
    int32 (B, K) index tensor of a fixed-order batch."""
    if precision not in ("fp64", "fp32"):
        raise InvalidData(f"precision must be 'fp64' or 'fp32', got {precision!r}")
    _check_batch(covs, batch)
    st = device_covs(covs)
    torch = st.torch
    lib = nat.lib()
    b, d, n = batch.batch_size, st.d, st.n
    eta = None
    if bias_correct:   # (a fixed-order batch's order without materialising (B,) orders)
        eta = st.eta(batch.order if batch.mode == "fixed" else int(batch.orders().max()))
    kstride = 0 if eta is None else eta.shape[1]
    out = torch.empty((4, b, d), dtype=torch.float64, device="cuda") if measures else None
    cnt, coords = _err_buffers(torch)
    logdet = invdiag = None
    if batch.mode == "fixed":
        k = batch.order
        if terms:
            logdet = torch.empty((b, d), dtype=torch.float64, device="cuda")
            invdiag = torch.empty((b, d, k), dtype=torch.float64, device="cuda")
        if (precision == "fp64" and measures and not terms
                and b >= 2 * _STREAM_ROWS and b * k * 4 > (64 << 20)):
            out = _eval_streamed(st, batch, eta, kstride, out, keep_idx)
            return out, None, None
        idx = _indices_to_device(batch.indices, torch)
        if keep_idx is not None:
            keep_idx.append(idx)
        if precision == "fp32" and measures and not terms:
            nat.check(lib.hoi_eval_indices_fp32(st.corr.data_ptr(), st.corr32.data_ptr(),
                                                st.sdiag.data_ptr(), nat.ptr(eta), kstride, n, d,
                                                idx.data_ptr(), b, k, out.data_ptr(), cnt.data_ptr(),
                                                coords.data_ptr(), ERR_CAP,
                                                nat.stream_handle(torch)), "eval_indices_fp32")
            _raise_not_pd(cnt, coords)
            return out, None, None
        nat.check(lib.hoi_eval_indices(st.corr.data_ptr(), st.sdiag.data_ptr(), nat.ptr(eta),
                                       kstride, n, d, idx.data_ptr(), b, k, nat.ptr(out),
                                       nat.ptr(logdet), nat.ptr(invdiag), cnt.data_ptr(),
                                       coords.data_ptr(), ERR_CAP, nat.stream_handle(torch)),
                  "eval_indices")
    else:
        if terms:
            logdet = torch.empty((b, d), dtype=torch.float64, device="cuda")
            invdiag = torch.zeros((b, d, n), dtype=torch.float64, device="cuda")
        w = (n + 63) // 64
        words = np.zeros((b, w), dtype=np.uint64)
        for j in range(n):
            words[:, j // 64] |= batch.masks[:, j].astype(np.uint64) << np.uint64(j % 64)
        dm = torch.from_numpy(words.view(np.int64)).cuda()
        nat.check(lib.hoi_eval_masks(st.corr.data_ptr(), st.sdiag.data_ptr(), nat.ptr(eta),
                                     kstride, n, d, dm.data_ptr(), w, b, nat.ptr(out),
                                     nat.ptr(logdet), nat.ptr(invdiag), cnt.data_ptr(),
                                     coords.data_ptr(), ERR_CAP, nat.stream_handle(torch)),
                  "eval_masks")
    _raise_not_pd(cnt, coords)
    return out, logdet, invdiag


@nat.traced("hoi.entropy_terms")
def entropy_terms(covs: CovSet, batch: NpletBatch, bias_correct: bool = False) -> EntropyTerms:
    """Joint, marginal and leave-one-out entropies (ref:nplet_engine.py:284-351).

    The device kernel returns log det Sigma_S and the inverse diagonal; the
    excess terms are assembled with the reference's expressions."""
    out, logdet, invdiag = eval_device(covs, batch, bias_correct, measures=False, terms=True)
    st = device_covs(covs)
    sig_diag = st.sdiag.cpu().numpy()                               # (D, N)
    ld = logdet.cpu().numpy()
    idg = invdiag.cpu().numpy()
    orders = batch.orders()
    x_singles = 0.5 * np.log(sig_diag)
    if bias_correct:
        tables = st.eta(int(orders.max())).cpu().numpy()
        x_singles = x_singles - tables[:, 1][:, None]
    if batch.mode == "fixed":
        k = batch.order
        x_joint = 0.5 * ld
        x_loo = 0.5 * (ld[..., None] + np.log(idg))
        x_sing = x_singles[:, batch.indices].transpose(1, 0, 2)
        if bias_correct:
            x_joint = x_joint - tables[:, k][None, :]
            x_loo = x_loo - tables[:, k - 1][None, :, None]
        return EntropyTerms(h_joint=x_joint + k * NORMAL_ENTROPY,
                            h_singles=x_sing + NORMAL_ENTROPY,
                            h_leave_one_out=x_loo + (k - 1) * NORMAL_ENTROPY,
                            orders=orders, excess_joint=x_joint, excess_singles=x_sing,
                            excess_leave_one_out=x_loo)
    ks = orders.astype(np.float64)[:, None]
    in_set = batch.masks[:, None, :]
    x_joint = 0.5 * ld
    with np.errstate(divide="ignore"):
        x_loo = 0.5 * (ld[..., None] + np.log(np.where(in_set, idg, 1.0)))
    if bias_correct:
        x_joint = x_joint - tables[:, orders].T
        x_loo = x_loo - tables[:, orders - 1].T[..., None]
    x_sing = np.where(in_set, x_singles[None], 0.0)
    x_loo = np.where(in_set, x_loo, 0.0)
    return EntropyTerms(
        h_joint=x_joint + ks * NORMAL_ENTROPY,
        h_singles=np.where(in_set, x_sing + NORMAL_ENTROPY, 0.0),
        h_leave_one_out=np.where(in_set, x_loo + (ks[..., None] - 1.0) * NORMAL_ENTROPY, 0.0),
        orders=orders, excess_joint=x_joint, excess_singles=x_sing, excess_leave_one_out=x_loo)
