"""Exact centers on the device (mirrors lshclust.numeric, numeric.py:1-76, and
the center reductions of seeding.py:168-197 / engine.py:299-323, :481-516).

Dense: exact integer column sums (base-2^32 digits in int64 lanes) ->
correctly rounded mean; partial sums from different shards add exactly, so
the engine reduces them with an int64 all-reduce.  Categorical: per
attribute value counts, argmax with ties to the smallest code.  Sparse:
strict-majority membership.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .data import CategoricalData, InvalidInput, SparseData
from .tables import GroupSet

_ND_CHOICES = (3, 4, 5, 6, 8, 12, 20, 40)


def exponent_range(X: torch.Tensor):
    out = np.zeros(2, dtype=np.int32)
    _lib.call("geek_exponent_range", _lib.ptr(X), _lib.dtype_code(X), X.shape[0], X.shape[1], _lib.hptr(out),
              _lib.stream())
    return int(out[0]), int(out[1])


def digit_count(emin: int, emax: int) -> int:
    if emin > emax:
        return _ND_CHOICES[0]
    need = -(-(emax - emin + 33) // 32) + 1
    for c in _ND_CHOICES:
        if c >= need:
            return c
    raise InvalidInput("exponent range too wide for exact sums")


def partial_sums(X: torch.Tensor, groups: GroupSet, emin: int, nd: int, row_lo: int = 0, digits=None,
                 nonfinite=None) -> torch.Tensor:
    """int64 [k, d, nd] exact digit sums over the members that are rows
    [row_lo, row_lo + X.shape[0]) of the global id space (added into
    `digits` when given).  `nonfinite` (int32 [1] on the device) is set to 1
    if a member coordinate is NaN / inf (numeric.py:24-25 raises there)."""
    k, d = groups.count, X.shape[1]
    if digits is None:
        digits = _lib.zeros(max(1, k * d * nd), torch.int64)[: k * d * nd].view(k, d, nd)
    if k:
        _lib.call("geek_exact_sums", _lib.ptr(X), _lib.dtype_code(X), X.shape[0], d, row_lo, _lib.ptr(groups.flat),
                  _lib.ptr(groups.off), k, emin, nd, _lib.ptr(digits), _lib.ptr(nonfinite), _lib.stream())
    return digits


def center_stats_bytes(digits: torch.Tensor, emin: int, out: torch.Tensor):
    """out (int64 [1], device) += the bytes the reference's pack_bigints
    spends on these exact sums (engine.py:488-490 LocalCenters accounting)."""
    k, d, nd = digits.shape
    if k:
        _lib.call("geek_sum_pack_bytes", _lib.ptr(digits.contiguous()), k, d, nd, emin, _lib.ptr(out), _lib.stream())


def round_means(digits: torch.Tensor, counts: torch.Tensor, emin: int, nd: int) -> torch.Tensor:
    k, d, _ = digits.shape
    out = _lib.empty(max(1, k * d), torch.float64)
    if k:
        _lib.call("geek_round_means", _lib.ptr(digits.contiguous()), _lib.ptr(counts.to(torch.int64).contiguous()),
                  k, d, emin, nd, _lib.ptr(out), _lib.stream())
    return out[: k * d].view(k, d)


def dense_centers(X: torch.Tensor, groups: GroupSet) -> torch.Tensor:
    emin, emax = exponent_range(X)
    nd = digit_count(emin, emax)
    bad = _lib.zeros(1, torch.int32)
    digits = partial_sums(X, groups, emin, nd, nonfinite=bad)
    if int(bad.item()):
        raise InvalidInput("non-finite value in exact sum")
    return round_means(digits, groups.sizes(), emin, nd)


def mode_counts(codes: torch.Tensor, code_space: int, groups: GroupSet, row_lo: int = 0) -> torch.Tensor:
    n, d = codes.shape
    k = groups.count
    if k * d * code_space > (1 << 31):
        raise InvalidInput("mode statistics too large for dense counting")
    cnt = _lib.zeros(max(1, k * d * code_space), torch.int64)
    _lib.call("geek_mode_counts", _lib.ptr(codes), n, d, row_lo, code_space, _lib.ptr(groups.flat),
              _lib.ptr(groups.off), k, _lib.ptr(cnt), _lib.stream())
    return cnt[: k * d * code_space].view(k, d, code_space)


def mode_centers(codes: torch.Tensor, code_space: int, groups: GroupSet) -> torch.Tensor:
    """int32 [k, d] per-attribute modes, ties to the smallest code (seeding.py:180-185)."""
    k, d = groups.count, codes.shape[1]
    if k * d * code_space <= (1 << 31):
        # argmax returns the first maximum: ties go to the smallest code
        return torch.argmax(mode_counts(codes, code_space, groups), dim=2).to(torch.int32)
    return sparse_mode_centers(codes, code_space, groups.flat, groups.off)


def sparse_mode_centers(codes: torch.Tensor, code_space: int, flat: torch.Tensor, off: torch.Tensor) -> torch.Tensor:
    """Modes without a dense [k, d, code_space] table (large code spaces, e.g.
    Criteo-like cardinalities): per attribute, the (group, code) pairs of all
    members are counted by a device sort + run-length pass; each group keeps
    its most frequent code, the smallest among equal counts."""
    k = off.numel() - 1
    d = codes.shape[1]
    sizes = off[1:] - off[:-1]
    total = int(off[-1].item())
    ids = flat[:total].to(torch.int64) & 0xFFFFFFFF
    grp = torch.repeat_interleave(torch.arange(k, device=codes.device), sizes)
    out = torch.zeros((k, d), dtype=torch.int32, device=codes.device)
    for c in range(d):
        key = grp * code_space + codes[ids, c].to(torch.int64)
        uk, cnt = torch.unique(key, sorted=True, return_counts=True)
        g = uk // code_space
        top = torch.zeros(k, dtype=cnt.dtype, device=cnt.device).scatter_reduce(0, g, cnt, "amax", include_self=False)
        win = cnt == top[g]
        code = torch.full((k,), code_space, dtype=torch.int64, device=cnt.device)
        code = code.scatter_reduce(0, g[win], (uk - g * code_space)[win], "amin", include_self=True)
        out[:, c] = code.to(torch.int32)
    return out


def sparse_counts(data: SparseData, groups: GroupSet, row_lo: int = 0, csr=None) -> torch.Tensor:
    flat, off = csr if csr is not None else data.csr()
    k, u = groups.count, data.universe
    cnt = _lib.zeros(max(1, k * u), torch.int64)
    _lib.call("geek_sparse_counts", _lib.ptr(flat), _lib.ptr(off), data.n, row_lo, u, _lib.ptr(groups.flat),
              _lib.ptr(groups.off), k, _lib.ptr(cnt), _lib.stream())
    return cnt[: k * u].view(k, u)


def sparse_centers(data: SparseData, groups: GroupSet) -> torch.Tensor:
    cnt = sparse_counts(data, groups)
    return (2 * cnt > groups.sizes()[:, None]).to(torch.int32)


# ---- refinement: statistics keyed by the current labels (assignment.py:110-137) ----

_SORT_RUNS = 8  # mean label-run length below which rows are visited in label order


def label_sums(X: torch.Tensor, labels: torch.Tensor, k: int, emin: int, nd: int, order=None) -> torch.Tensor:
    """int64 [k, d, nd] exact digit sums of the rows with each label (one
    pass over X; shards add their partials exactly).  Rows stream in storage
    order while labels come in runs (cluster-ordered data); otherwise through
    a stable label sort, so every run flushes once instead of once per row."""
    n, d = X.shape
    labels = labels.contiguous()
    digits = _lib.zeros(max(1, k * d * nd), torch.int64)
    if k and n:
        if order is None and n > 1:
            # label changes per row, from 64 windows of 4096 consecutive rows on large inputs (either
            # path is exact; this only picks the faster one)
            W = 4096
            win = labels[: (n // W) * W].view(-1, W)
            win = win[:: max(1, win.shape[0] // 64)] if n >= 64 * W else labels.view(1, -1)
            changes = int((win[:, 1:] != win[:, :-1]).sum().item())
            if changes * _SORT_RUNS > win.numel():
                order = torch.sort(labels, stable=True).indices
        _lib.call("geek_label_sums", _lib.ptr(X), _lib.dtype_code(X), n, d, _lib.ptr(labels),
                  _lib.ptr(order), k, emin, nd, _lib.ptr(digits), _lib.stream())
    return digits[: k * d * nd].view(k, d, nd)


def label_mode_counts(codes: torch.Tensor, code_space: int, labels: torch.Tensor, k: int) -> torch.Tensor:
    n, d = codes.shape
    if k * d * code_space > (1 << 31):
        raise InvalidInput("mode statistics too large for dense counting")
    cnt = _lib.zeros(max(1, k * d * code_space), torch.int64)
    _lib.call("geek_label_mode_counts", _lib.ptr(codes), n, d, _lib.ptr(labels.contiguous()), k, code_space,
              _lib.ptr(cnt), _lib.stream())
    return cnt[: k * d * code_space].view(k, d, code_space)


_DENSE_MODE_LIMIT = 1 << 31


def label_mode_centers(codes: torch.Tensor, code_space: int, labels: torch.Tensor, k: int,
                       keep: torch.Tensor) -> torch.Tensor:
    """int32 [len(keep), d] modes of the clusters `keep` (non-empty, ascending)
    from the labels: dense label-keyed counts when [k, d, code_space] fits,
    else the members grouped by a stable label sort and the sort-based mode."""
    d = codes.shape[1]
    if k * d * code_space <= _DENSE_MODE_LIMIT:
        return torch.argmax(label_mode_counts(codes, code_space, labels, k)[keep], dim=2).to(torch.int32)
    order = torch.sort(labels, stable=True).indices
    sizes = torch.bincount(labels, minlength=k)[keep]
    off = torch.zeros(keep.numel() + 1, dtype=torch.int64, device=labels.device)
    torch.cumsum(sizes, 0, out=off[1:])
    return sparse_mode_centers(codes, code_space, order.to(torch.int32).contiguous(), off)


def label_sparse_counts(flat, off, n: int, universe: int, labels: torch.Tensor, k: int) -> torch.Tensor:
    cnt = _lib.zeros(max(1, k * universe), torch.int64)
    _lib.call("geek_label_sparse_counts", _lib.ptr(flat), _lib.ptr(off), n, _lib.ptr(labels.contiguous()), k,
              universe, _lib.ptr(cnt), _lib.stream())
    return cnt[: k * universe].view(k, universe)


# ---- reference API (numeric.py:19-51) -----------------------------------------

def exact_centroid(vectors) -> np.ndarray:
    """Correctly rounded mean of the rows, identical under any partition."""
    X = _lib.to_dev(np.asarray(vectors) if not isinstance(vectors, torch.Tensor) else vectors)
    if X.dim() != 2 or X.shape[0] == 0:
        raise InvalidInput("expected a non-empty matrix")
    if X.dtype not in (torch.float32, torch.float64):
        X = X.to(torch.float64)
    if not bool(torch.isfinite(X).all().item()):
        raise ValueError("non-finite value in exact sum")
    gs = GroupSet(_lib.to_dev(np.arange(X.shape[0], dtype=np.uint32).view(np.int32)),
                  _lib.to_dev(np.array([0, X.shape[0]], dtype=np.int64)))
    return dense_centers(X.contiguous(), gs).cpu().numpy()[0]
