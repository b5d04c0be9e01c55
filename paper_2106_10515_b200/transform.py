"""Bucketize: every data type into the unified bucket collection
(mirrors lshclust.transform, transform.py:1-199).

Dense data: float64-accurate projections (K1, geek_project_keys) and the
exact even rank split (K2, geek_rank_split), all on the device.  Mixed and
sparse data: numeric discretisation by the same rank split, DOPH reduction
and (K, L) signature buckets via device MinHash + lexicographic group-by.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .data import CategoricalData, DenseData, InvalidInput, MixedData, SparseData
from .hashing import (DophReducer, PermBatch, ProjectionFunction, SignatureScheme, derive_seed,
                      set_signatures_device)
from .tables import BucketTable

__all__ = ["HomoTransformParams", "MinhashTransformParams", "even_partition_sizes", "transform_homo",
           "discretize_numeric", "transform_hetero", "transform_sparse"]


_DIRECTIONS = {}


@dataclass(frozen=True)
class HomoTransformParams:
    """m projection tables split into t even buckets (transform.py:35-60)."""

    num_tables: int
    buckets_per_table: int
    seed: int = 0
    directions: np.ndarray = None

    def __post_init__(self):
        if self.num_tables < 1:
            raise InvalidInput("need at least one table")
        if self.buckets_per_table < 2:
            raise InvalidInput("need at least two buckets per table")
        if self.directions is not None:
            d = np.asarray(self.directions, dtype=np.float64)
            if d.ndim != 2 or d.shape[0] != self.num_tables:
                raise InvalidInput("directions must be (num_tables, dim)")
            object.__setattr__(self, "directions", d)

    def __hash__(self):
        return hash((self.num_tables, self.buckets_per_table, self.seed))

    def projection(self, table: int, dim: int) -> ProjectionFunction:
        if self.directions is not None:
            return ProjectionFunction(self.directions[table])
        return ProjectionFunction.from_seed(self.seed, table, dim)

    def direction_matrix(self, dim: int) -> np.ndarray:
        if self.directions is not None:
            if self.directions.shape[1] != dim:
                raise InvalidInput(f"dimension mismatch: directions have {self.directions.shape[1]}, data {dim}")
            return self.directions
        key = (self.seed, self.num_tables, dim)
        A = _DIRECTIONS.get(key)
        if A is None:  # the reference's PCG64 draws, once per (seed, tables, dim)
            A = np.stack([self.projection(j, dim).direction for j in range(self.num_tables)])
            _DIRECTIONS[key] = A
        return A


@dataclass(frozen=True)
class MinhashTransformParams:
    """(K, L) signature bucketing; discretisation bins; sparse target dims."""

    num_hashes: int
    num_tables: int
    seed: int = 0
    bins_per_attribute: int = 1024
    target_dims: int = 400
    table_seeds: tuple = None

    def __post_init__(self):
        if self.num_hashes < 1 or self.num_tables < 1:
            raise InvalidInput("need K >= 1 and L >= 1")
        if self.bins_per_attribute < 2:
            raise InvalidInput("need at least two discretization bins")

    def scheme(self, universe: int) -> SignatureScheme:
        return SignatureScheme(self.num_hashes, self.num_tables, universe, seed=self.seed,
                               table_seeds=self.table_seeds)


def even_partition_sizes(n: int, parts: int) -> np.ndarray:
    """First n % parts parts get one extra (transform.py:95-100)."""
    q, r = divmod(n, parts)
    s = np.full(parts, q, dtype=np.int64)
    s[:r] += 1
    return s


# ---------------------------------------------------------------------------
# dense

_DIRS = {}


def directions_device(A: np.ndarray) -> torch.Tensor:
    """The float64 direction matrix on the current device, cached by content
    (the same job's directions are re-used every call)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    key = (A.shape, hash(A.tobytes()), torch.cuda.current_device())
    t = _DIRS.get(key)
    if t is None:
        if len(_DIRS) > 8:
            _DIRS.clear()
        t = _lib.to_dev(A)
        _DIRS[key] = t
    return t


def project_keys(X: torch.Tensor, A: np.ndarray, exprange: torch.Tensor = None) -> torch.Tensor:
    """[m, n] order-preserving uint64 keys (int64 storage) of X @ A.T in float64.
    `exprange` (int32[2] on the device, preset to (2^30, -2^30)) receives the
    exact-sum exponent window of X from the same pass."""
    n, d = X.shape
    m = A.shape[0]
    keys = _lib.empty(max(1, m * n), torch.int64)
    Ad = directions_device(A)
    _lib.call("geek_project_keys", _lib.ptr(X), _lib.dtype_code(X), n, d, _lib.ptr(Ad), m, _lib.ptr(keys),
              _lib.ptr(exprange), _lib.stream())
    return keys[: m * n].view(m, n) if n else keys[:0].view(m, 0)


def rank_split_codes(keys: torch.Tensor, t: int, stats=None) -> torch.Tensor:
    """id-major int32 [n, m] slot codes of the exact even rank split of every table."""
    m, n = keys.shape
    codes = _lib.empty(max(1, n * m), _lib.U32)
    st = np.zeros(4, dtype=np.uint64)
    _lib.call("geek_rank_split", _lib.ptr(keys), n, m, t, _lib.ptr(codes), _lib.hptr(st), _lib.stream())
    if stats is not None:
        stats.update(fine_bins=int(st[0]), straddling=int(st[1]), max_straddle_bin=int(st[2]),
                     sorted_fallback=int(st[3]))
    return codes[: n * m].view(n, m)


def projection_tolerance(A: np.ndarray, xmax_exp: int) -> np.ndarray:
    """Per-table bound on |K1 key - reference key| (transform.py:125 / engine.py:180
    form X @ a with OpenBLAS dgemv; K1 with exact integer tensor-core products
    rounded within 2^-6 of the same bound plus 2 ulps, tc_project.cu, or with
    DMMA FMA chains under GEEK_TCPROJ=0).  Any float64
    summation order of d products is within gamma_d * sum_k |x_k a_k| of the
    exact dot product (gamma_d = d u / (1 - d u), u = 2^-53), and
    sum_k |x_k a_k| <= 2^xmax_exp * |a|_1 when every |x_k| < 2^xmax_exp, so
    the two keys differ by at most twice that."""
    A = np.asarray(A, dtype=np.float64)
    d = A.shape[1]
    u = 2.0 ** -53
    gamma = d * u / (1.0 - d * u)
    return 2.0 * gamma * np.ldexp(1.0, int(xmax_exp)) * np.abs(A).sum(axis=1) * (1.0 + 4 * u)


def split_boundary_stats(keys: torch.Tensor, codes: torch.Tensor, t: int, tol: np.ndarray,
                         rel=(1e-12, 1e-6), cap: int = 4096, tables=None) -> dict:
    """Count the ids whose key lies near a rank-split boundary (north_star's
    tie tolerance): `ambiguous` within the float64 order bound `tol` (their
    code may differ from the reference's; listed as (table, id) in
    `ambiguous_ids`), `within_rel` within rel * |boundary| for each rel."""
    m, n = keys.shape
    L = _lib.lib()
    wsb = int(L.geek_split_boundary_workspace(m, t))
    ws = _lib.empty(max(1, (wsb + 7) // 8), torch.int64)
    tol_d = _lib.to_dev(np.ascontiguousarray(tol, dtype=np.float64))
    counts = _lib.zeros(4, torch.int64)
    lst = _lib.empty(max(2, 2 * cap), torch.int32)
    _lib.call("geek_split_boundary_stats", _lib.ptr(keys), n, m, t, _lib.ptr(codes), codes.shape[1],
              _lib.ptr(tol_d), float(rel[0]), float(rel[1]), _lib.ptr(counts), _lib.ptr(lst), cap, _lib.ptr(ws),
              wsb, _lib.stream())
    c = counts.cpu().numpy()
    k = int(min(c[3], cap))
    ids = lst[: 2 * k].view(k, 2).cpu().numpy().astype(np.int64)
    if tables is not None and k:
        ids[:, 0] = np.asarray(tables)[ids[:, 0]]
    return dict(ambiguous=int(c[0]), within_rel={f"{rel[0]:g}": int(c[1]), f"{rel[1]:g}": int(c[2])},
                ambiguous_ids=ids, tol_max=float(np.max(tol)) if len(tol) else 0.0,
                listed_complete=bool(c[3] <= cap))


def homo_codes(X: torch.Tensor, params: HomoTransformParams, stats=None) -> torch.Tensor:
    n, d = X.shape
    t = params.buckets_per_table
    if t > n:
        raise InvalidInput(f"cannot split {n} objects into {t} buckets")
    keys = project_keys(X, params.direction_matrix(d))
    codes = rank_split_codes(keys, t, stats)
    del keys
    return codes


def transform_homo(data: DenseData, params: HomoTransformParams) -> BucketTable:
    """Project every table, rank-split evenly (transform.py:112-128).

    Returns a device BucketTable that iterates as list[Bucket] in the
    reference order (table-major, slots ascending)."""
    if not isinstance(data, DenseData):
        raise InvalidInput("homogeneous transform expects dense data")
    X = data.device_vectors()
    codes = homo_codes(X, params)
    return BucketTable(codes, data.n, [params.buckets_per_table] * params.num_tables, "rank", even=True)


# ---------------------------------------------------------------------------
# mixed / sparse

def discretize_codes(numeric: torch.Tensor, bins: int, total_cols: int) -> torch.Tensor:
    """int32 [n, total_cols] with the first numeric.shape[1] columns filled by
    the equal-frequency bin of every numeric attribute (transform.py:131-155)."""
    n, dn = numeric.shape
    out = _lib.empty(max(1, n * total_cols), _lib.U32)
    keys = _lib.empty(max(1, n), torch.int64)
    for c in range(dn):
        _lib.call("geek_column_keys", _lib.ptr(numeric), _lib.dtype_code(numeric), n, dn, c, _lib.ptr(keys),
                  _lib.stream())
        _lib.call("geek_rank_split_strided", _lib.ptr(keys), n, bins, _lib.ptr(out), total_cols, c, _lib.stream())
    return out[: n * total_cols].view(n, total_cols)


def discretize_numeric(data, bins_per_attribute: int) -> CategoricalData:
    if isinstance(data, DenseData):
        numeric = data.device_vectors()
        categorical = np.empty((data.n, 0), dtype=np.int32)
    elif isinstance(data, MixedData):
        numeric = _lib.to_dev(data.numeric)
        categorical = data.categorical
    else:
        raise InvalidInput("discretization expects dense or mixed data")
    if numeric.shape[1] == 0:
        raise InvalidInput("no numeric attribute to discretize")
    n = numeric.shape[0]
    if bins_per_attribute > n:
        raise InvalidInput("more discretization bins than objects")
    dn, dc = numeric.shape[1], categorical.shape[1]
    codes = discretize_codes(numeric, bins_per_attribute, dn + dc)
    if dc:
        codes[:, dn:] = _lib.to_dev(categorical, torch.int32)
    return CategoricalData.from_device(codes)  # stays on the device (no host round trip)


def categorical_token_csr(cat: CategoricalData):
    """Token CSR (attr * code_space + code) of every record, on the device."""
    codes = cat.device_codes().to(torch.int64)
    n, d = codes.shape
    base = torch.arange(d, device=codes.device, dtype=torch.int64) * cat.code_space
    flat = (codes + base).reshape(-1)
    if flat.numel() and int(flat.max().item()) >= (1 << 32) - 1:
        raise InvalidInput("token universe must stay below 2^32")
    off = torch.arange(n + 1, device=codes.device, dtype=torch.int64) * d
    return flat.to(torch.int32).contiguous(), off


def signature_rows(scheme: SignatureScheme, flat: torch.Tensor, off: torch.Tensor, n: int) -> torch.Tensor:
    """[n, L*K] MinHash signatures of every set for every table (hashing.py:250-282)."""
    funcs = scheme.all_functions()
    return set_signatures_device(funcs, flat, off, n, PermBatch(funcs))


def group_signature_tables(sig: torch.Tensor, K: int, universe: int):
    """Per table (K consecutive columns of sig [n, T*K]): objects grouped by
    K-signature, slots numbered in sorted signature order (transform.py:158-169,
    np.unique(axis=0)) -> (codes [n, T] int32, tsizes)."""
    n = sig.shape[0]
    T = sig.shape[1] // K
    codes = _lib.empty(max(1, n * T), _lib.U32).view(-1)
    codes = codes[: n * T].view(n, T) if n else codes[:0].view(0, T)
    tsizes = []
    bits = np.full(K, max(1, int(universe - 1).bit_length()), dtype=np.int32)
    perm = _lib.empty(max(1, n), _lib.U32)
    gid = _lib.empty(max(1, n), _lib.U32)
    for tb in range(T):
        rows = sig[:, tb * K:(tb + 1) * K].contiguous()
        ng = np.zeros(1, dtype=np.uint64)
        _lib.call("geek_group_rows", _lib.ptr(rows), n, K, _lib.hptr(bits), _lib.ptr(perm), _lib.ptr(gid),
                  _lib.hptr(ng), _lib.stream())
        col = torch.empty(n, dtype=torch.int32, device=codes.device)
        col[perm[:n].to(torch.int64)] = gid[:n]
        codes[:, tb] = col
        tsizes.append(int(ng[0]))
    return codes.contiguous(), tsizes


def signature_bucket_codes(scheme: SignatureScheme, flat: torch.Tensor, off: torch.Tensor, n: int):
    """Per table, objects grouped by K-signature with slots numbered in sorted
    signature order (transform.py:158-169) -> (codes [n, L] int32, tsizes)."""
    sig = signature_rows(scheme, flat, off, n)  # [n, L*K]
    return group_signature_tables(sig, scheme.num_hashes, scheme.universe)


def transform_hetero(data, params: MinhashTransformParams):
    """(K, L) signature buckets of attribute tokens (transform.py:172-184)."""
    if isinstance(data, (DenseData, MixedData)):
        cat = discretize_numeric(data, params.bins_per_attribute)
    elif isinstance(data, CategoricalData):
        cat = data
    else:
        raise InvalidInput("heterogeneous transform expects mixed or categorical data")
    flat, off = categorical_token_csr(cat)
    scheme = params.scheme(universe=cat.dim * cat.code_space)
    codes, tsizes = signature_bucket_codes(scheme, flat, off, cat.n)
    return BucketTable(codes, cat.n, tsizes, "sig", even=False), cat


def transform_sparse(data: SparseData, params: MinhashTransformParams):
    """DOPH-reduce, then signature-bucket the reduced sets (transform.py:187-199)."""
    if not isinstance(data, SparseData):
        raise InvalidInput("sparse transform expects sparse data")
    if params.target_dims > data.universe:
        reduced = data
        flat, off = data.csr()
    else:
        red = DophReducer(derive_seed(params.seed, 0xD0), data.universe, params.target_dims)
        flat, off = red.reduce_device(*data.csr(), data.n)
        reduced = SparseData.from_csr(flat.to(torch.int64) & 0xFFFFFFFF, off, params.target_dims)
        flat, off = reduced.csr()
    scheme = params.scheme(universe=reduced.universe)
    codes, tsizes = signature_bucket_codes(scheme, flat, off, reduced.n)
    return BucketTable(codes, reduced.n, tsizes, "sig", even=False), reduced
