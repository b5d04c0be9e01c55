"""One-pass assignment (mirrors lshclust.assignment, assignment.py:1-170).

Euclidean: geek_assign_l2 evaluates numpy's float64 direct-difference
distance bit-for-bit (pairwise summation order, no FMA contraction,
correctly rounded sqrt, first-index ties), so labels, best distances and
radii equal the reference exactly; the objective is numpy's pairwise sum of
the best distances, reproduced on the device (geek_pairwise_sum).
Jaccard: categorical 1 - m/(2d - m) and binary sparse intersection/union.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .data import CategoricalData, CentralVector, Clustering, DenseData, InvalidInput, SparseData

__all__ = ["assign", "refine", "distance_matrix", "squared_objective", "CHUNK"]

CHUNK = 8192  # reference chunking (assignment.py:23); results do not depend on it
_METRICS = ("euclidean", "jaccard")


def _check_compat(data, centers, metric):
    if metric not in _METRICS:
        raise InvalidInput(f"unknown metric {metric!r}")
    kinds = {c.kind for c in centers}
    if metric == "euclidean":
        if not isinstance(data, DenseData) or kinds != {"centroid"}:
            raise InvalidInput("euclidean assignment needs dense data and centroids")
    elif not isinstance(data, (CategoricalData, SparseData)) or kinds != {"mode"}:
        raise InvalidInput("jaccard assignment needs categorical or sparse data and modes")


class AssignStats:
    """Device-side statistics of one geek_assign_l2 call (geek_assign_stats_t)
    plus CUDA events around its screen; read them after the stream reaches
    them (`read()` synchronises on the end event)."""

    def __init__(self):
        self.dev = _lib.zeros(4, torch.int64)
        self.ev0 = torch.cuda.Event(enable_timing=True)
        self.ev1 = torch.cuda.Event(enable_timing=True)
        self.ev0.record()  # materialise the events (torch creates them lazily)
        self.ev1.record()

    def read(self) -> dict:
        v = self.dev.cpu().tolist()
        self.ev1.synchronize()
        ms = self.ev0.elapsed_time(self.ev1)
        return dict(assign_rechecked=int(v[0]), assign_full_scans=int(v[1]), screen_mode=int(v[2]),
                    screen_ms=float(ms) if v[2] else 0.0, screen_tiles=int(v[3]))


_LAST = [None]


def last_assign_stats() -> dict:
    """Statistics of this process's last assign_l2_device call (tests, tools)."""
    return _LAST[0].read() if _LAST[0] is not None else {}


def assign_l2_device(X: torch.Tensor, C: torch.Tensor, stats: AssignStats = None):
    """(labels int64, best float64) on the device."""
    n, d = X.shape
    k = C.shape[0]
    labels = _lib.empty(max(1, n), torch.int64)
    best = _lib.empty(max(1, n), torch.float64)
    st = stats if stats is not None else AssignStats()
    _lib.call("geek_assign_l2", _lib.ptr(X), _lib.dtype_code(X), n, d, _lib.ptr(C.contiguous()), k,
              _lib.ptr(labels), _lib.ptr(best), _lib.ptr(st.dev), _lib.C.c_void_p(st.ev0.cuda_event),
              _lib.C.c_void_p(st.ev1.cuda_event), None, 0, _lib.stream())
    _LAST[0] = st
    return labels[:n], best[:n]


def assign_cat_device(codes: torch.Tensor, M: torch.Tensor):
    n, d = codes.shape
    k = M.shape[0]
    labels = _lib.empty(max(1, n), torch.int64)
    best = _lib.empty(max(1, n), torch.float64)
    _lib.call("geek_assign_categorical", _lib.ptr(codes), n, d, _lib.ptr(M.contiguous()), k, _lib.ptr(labels),
              _lib.ptr(best), _lib.stream())
    return labels[:n], best[:n]


def assign_sparse_device(flat, off, n: int, universe: int, M: torch.Tensor):
    k = M.shape[0]
    labels = _lib.empty(max(1, n), torch.int64)
    best = _lib.empty(max(1, n), torch.float64)
    _lib.call("geek_assign_sparse", _lib.ptr(flat), _lib.ptr(off), n, universe, _lib.ptr(M.contiguous()), k,
              _lib.ptr(labels), _lib.ptr(best), _lib.stream())
    return labels[:n], best[:n]


def radii_sizes(labels: torch.Tensor, best: torch.Tensor, k: int):
    radii = _lib.zeros(max(1, k), torch.float64)
    sizes = _lib.zeros(max(1, k), torch.int64)
    _lib.call("geek_radii_sizes", _lib.ptr(labels), _lib.ptr(best), labels.numel(), k, _lib.ptr(radii),
              _lib.ptr(sizes), _lib.stream())
    return radii[:k], sizes[:k]


def pairwise_sum(v: torch.Tensor) -> torch.Tensor:
    out = _lib.empty(1, torch.float64)
    _lib.call("geek_pairwise_sum", _lib.ptr(v.contiguous()), v.numel(), _lib.ptr(out), _lib.stream())
    return out


def center_matrix(centers, metric):
    vals = np.stack([c.values for c in centers])
    if metric == "euclidean":
        return _lib.to_dev(vals.astype(np.float64))
    return _lib.to_dev(vals.astype(np.int32))


def assign_device(data, C: torch.Tensor, metric: str):
    if metric == "euclidean":
        return assign_l2_device(data.device_vectors(), C)
    if isinstance(data, CategoricalData):
        return assign_cat_device(data.device_codes(), C)
    flat, off = data.csr()
    return assign_sparse_device(flat, off, data.n, data.universe, C)


def assign(data, centers, metric) -> Clustering:
    """Nearest center for every object in one pass (assignment.py:81-107)."""
    if not centers:
        raise InvalidInput("cannot assign without centers")
    _check_compat(data, centers, metric)
    k = len(centers)
    C = center_matrix(centers, metric)
    if metric == "jaccard" and C.shape[1] != (data.dim if isinstance(data, CategoricalData) else data.universe):
        raise InvalidInput("mode width does not match the data")
    labels, best = assign_device(data, C, metric)
    radii, sizes = radii_sizes(labels, best, k)
    obj = pairwise_sum(best)
    return Clustering(centers=list(centers), assignment=labels.cpu().numpy(), radii=radii.cpu().numpy(),
                      objective=float(obj.item()), sizes=sizes.cpu().numpy())


def distance_matrix(data, centers, metric, rows=None) -> np.ndarray:
    """Full distance matrix (small-scale API helper, assignment.py:44-78):
    one assignment pass per center on the device."""
    _check_compat(data, centers, metric)
    idx = np.arange(data.n) if rows is None else np.asarray(rows)
    out = np.empty((idx.size, len(centers)))
    for j, c in enumerate(centers):
        C = center_matrix([c], metric)
        _, best = assign_device(data, C, metric)
        out[:, j] = best.cpu().numpy()[idx]
    return out


def _centers_from_assignment(data, assignment, k) -> list:
    """One central vector per non-empty cluster, in label order
    (assignment.py:110-137).  The members of cluster j are the rows labelled
    j, so the statistics come from one pass over the rows keyed by label
    (geek_label_sums / geek_label_mode_counts / geek_label_sparse_counts)
    instead of materialised member lists."""
    from .numeric import digit_count, exponent_range, label_mode_centers, label_sparse_counts, label_sums, \
        round_means

    labels = _lib.to_dev(np.ascontiguousarray(assignment, dtype=np.int64))
    zero = _lib.zeros(max(1, labels.numel()), torch.float64)
    _, sizes = radii_sizes(labels, zero[: labels.numel()], k)
    keep = torch.nonzero(sizes > 0).flatten()
    counts = sizes[keep].contiguous()
    w = counts.cpu().numpy()
    if isinstance(data, DenseData):
        X = data.device_vectors()
        emin, emax = exponent_range(X)
        nd = digit_count(emin, emax)
        C = round_means(label_sums(X, labels, k, emin, nd)[keep].contiguous(), counts, emin, nd).cpu().numpy()
        return [CentralVector("centroid", C[i], int(w[i])) for i in range(len(w))]
    if isinstance(data, CategoricalData):
        M = label_mode_centers(data.device_codes(), data.code_space, labels, k, keep).cpu().numpy()
    else:
        flat, off = data.csr()
        cnt = label_sparse_counts(flat, off, data.n, data.universe, labels, k)[keep]
        M = (2 * cnt > counts[:, None]).to(torch.int32).cpu().numpy()
    return [CentralVector("mode", M[i], int(w[i])) for i in range(len(w))]


def squared_objective(data, clustering: Clustering, metric: str) -> float:
    """Sum of squared assigned distances (assignment.py:140-154)."""
    C = center_matrix(clustering.centers, metric)
    lab = _lib.to_dev(clustering.assignment)
    total = 0.0
    for j in range(len(clustering.centers)):
        _, best = assign_device(data, C[j:j + 1], metric)
        sel = lab == j
        b = best[sel]
        total += float((b * b).sum().item()) if b.numel() else 0.0
    return total


def refine(data, clustering: Clustering, metric: str, passes: int) -> Clustering:
    """Recompute centers (dropping empty clusters) and reassign, `passes` times."""
    if passes < 0:
        raise InvalidInput("passes must be >= 0")
    out = clustering
    for _ in range(passes):
        centers = _centers_from_assignment(data, out.assignment, len(out.centers))
        out = assign(data, centers, metric)
    return out
