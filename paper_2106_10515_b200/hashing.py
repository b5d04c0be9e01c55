"""LSH primitives (mirrors lshclust.hashing, hashing.py:1-351).

Seed derivation and permutation *parameters* are computed on the host (they
are O(1) per function, or a <= 4096-entry rank table); every evaluation over
data runs in libgeek (perm_forward / set_minhash / invscan / doph kernels).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from . import _lib
from .errors import InvalidInput

M64 = (1 << 64) - 1
MERSENNE61 = (1 << 61) - 1
RANK_TABLE_MAX = 4096  # hashing.py:25


def splitmix64(z: int) -> int:
    """hashing.py:28-33."""
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return (z ^ (z >> 31)) & M64


def derive_seed(master: int, *path: int) -> int:
    """hashing.py:36-41."""
    z = splitmix64(master & M64)
    for p in path:
        z = splitmix64(z ^ splitmix64((p + 0x632BE59BD9B4E019) & M64))
    return z


def as_index_array(s) -> np.ndarray:
    if isinstance(s, (set, frozenset)):
        s = sorted(s)
    if isinstance(s, torch.Tensor):
        s = s.detach().cpu().numpy()
    return np.asarray(s, dtype=np.int64)


def _mulinv(c: int, w: int) -> int:
    inv = c
    for _ in range(6):
        inv = (inv * (2 - c * inv)) & 0xFFFFFFFF
    return inv & ((1 << w) - 1)


def _rank_table(seed: int, u: int) -> np.ndarray:
    """pi for u <= 4096 as ranks of a 64-bit mix (hashing.py:80-95)."""
    a1 = np.uint64(derive_seed(seed, 3))
    c1 = np.uint64(derive_seed(seed, 1) | 1)
    c2 = np.uint64(derive_seed(seed, 2) | 1)
    with np.errstate(over="ignore"):
        z = np.arange(u, dtype=np.uint64) + a1
        z ^= z >> np.uint64(30)
        z *= c1
        z ^= z >> np.uint64(27)
        z *= c2
        z ^= z >> np.uint64(31)
    out = np.empty(u, dtype=np.uint64)
    out[np.argsort(z, kind="stable")] = np.arange(u, dtype=np.uint64)
    return out


class PermBatch:
    """A batch of permutations as geek_perm_t structs plus a device table pool."""

    def __init__(self, funcs):
        self.funcs = list(funcs)
        self.structs = (_lib.PermT * len(self.funcs))()
        pool = []
        off = 0
        for i, f in enumerate(self.funcs):
            st = self.structs[i]
            st.u = f.universe_size
            if f.table is not None:
                tab = np.asarray(f.table, dtype=np.uint64).astype(np.uint32)
                inv = np.empty_like(tab)
                inv[tab] = np.arange(tab.size, dtype=np.uint32)
                st.table, st.inv_table = off, off + tab.size
                pool += [tab, inv]
                off += 2 * tab.size
                st.mask = st.c1 = st.c2 = st.a1 = st.s1 = st.s2 = st.c1inv = st.c2inv = 0
            else:
                w, mask, c1, c2, a1, s1, s2 = f.params
                st.mask, st.c1, st.c2, st.a1, st.s1, st.s2 = mask, c1, c2, a1, s1, s2
                st.c1inv, st.c2inv = _mulinv(c1, w), _mulinv(c2, w)
                st.table = st.inv_table = _lib.NONE32
        self.tables = _lib.to_dev(np.concatenate(pool).view(np.int32)) if pool else None

    @property
    def n(self) -> int:
        return len(self.funcs)

    def args(self):
        return self.structs, len(self.funcs), _lib.ptr(self.tables)


@dataclass(frozen=True)
class MinHashFunction:
    """Seeded bijection pi over [0, universe); h(S) = min pi(S) (hashing.py:51-147)."""

    seed: int
    universe_size: int
    table: np.ndarray = None

    def __post_init__(self):
        if self.universe_size < 1:
            raise InvalidInput("universe must be positive")
        if self.universe_size >= (1 << 32):
            raise InvalidInput("universe must be below 2^32")
        if self.table is None and self.universe_size <= RANK_TABLE_MAX:
            object.__setattr__(self, "table", _rank_table(self.seed, self.universe_size))
        elif self.table is not None:
            t = np.asarray(self.table, dtype=np.uint64)
            if t.shape != (self.universe_size,):
                raise InvalidInput("permutation table has wrong length")
            object.__setattr__(self, "table", t)

    def __hash__(self):
        return hash((self.seed, self.universe_size))

    def __eq__(self, other):
        return (isinstance(other, MinHashFunction) and self.seed == other.seed
                and self.universe_size == other.universe_size
                and ((self.table is None and other.table is None)
                     or (self.table is not None and other.table is not None
                         and np.array_equal(self.table, other.table))))

    @classmethod
    def identity(cls, universe_size: int) -> "MinHashFunction":
        return cls(0, universe_size, table=np.arange(universe_size, dtype=np.uint64))

    @cached_property
    def params(self):
        """(w, mask, c1, c2, a1, s1, s2), hashing.py:97-113."""
        w = max(1, int(self.universe_size - 1).bit_length())
        mask = (1 << w) - 1
        return (w, mask, (derive_seed(self.seed, 1) | 1) & mask, (derive_seed(self.seed, 2) | 1) & mask,
                derive_seed(self.seed, 3) & mask, max(1, w // 2), max(1, w // 3))

    @cached_property
    def _batch(self) -> PermBatch:
        return PermBatch([self])

    def permute(self, elements) -> np.ndarray:
        a = as_index_array(elements)
        if a.size and (a.min() < 0 or a.max() >= self.universe_size):
            raise InvalidInput("element outside hash universe")
        if a.size == 0:
            return np.zeros(0, dtype=np.uint64)
        x = _lib.to_dev(a.astype(np.uint32).view(np.int32))
        out = _lib.empty(a.size, _lib.U32)
        st, n, tab = self._batch.args()
        _lib.call("geek_perm_forward", st, n, tab, _lib.ptr(x), a.size, _lib.ptr(out), _lib.stream())
        return out.cpu().numpy().view(np.uint32).astype(np.uint64)

    def __call__(self, s) -> int:
        arr = as_index_array(s)
        if arr.size == 0:
            raise InvalidInput("minhash of an empty set is undefined")
        return int(self.permute(arr).min())


def set_signatures_device(funcs, flat: torch.Tensor, offsets: torch.Tensor, nsets: int,
                          batch: PermBatch = None) -> torch.Tensor:
    """[nsets, len(funcs)] uint32 (as int32 storage) segmented-min signatures."""
    batch = batch or PermBatch(funcs)
    sig = _lib.empty(max(1, nsets * batch.n), _lib.U32)
    if nsets:
        st, n, tab = batch.args()
        _lib.call("geek_set_minhash", st, n, tab, _lib.ptr(flat), _lib.ptr(offsets), nsets, _lib.ptr(sig),
                  _lib.stream())
    return sig[: nsets * batch.n].view(nsets, batch.n)


def csr_from_sets(sets):
    """Host list of index arrays -> (flat u32 dev, offsets u64 dev, sizes np)."""
    sets = [as_index_array(s) for s in sets]
    sizes = np.array([s.size for s in sets], dtype=np.int64)
    off = np.zeros(len(sets) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    flat = np.concatenate(sets) if sets else np.zeros(0, np.int64)
    if flat.size and (flat.min() < 0 or flat.max() >= (1 << 32) - 1):
        raise InvalidInput("ids must lie in [0, 2^32 - 1)")
    return (_lib.to_dev(flat.astype(np.uint32).view(np.int32) if flat.size else np.zeros(1, np.int32)),
            _lib.to_dev(off), sizes)


def minhash_collision_matrix(seeds, universe: int, a, b) -> np.ndarray:
    """h(A) == h(B) for many seeds (hashing.py:150-192)."""
    if universe <= RANK_TABLE_MAX:
        raise InvalidInput("batched collisions require a cycle-walking universe")
    seeds = [int(s) for s in np.asarray(seeds, dtype=np.uint64).tolist()]
    funcs = [MinHashFunction(s, universe) for s in seeds]
    out = np.empty(len(seeds), dtype=bool)
    for lo in range(0, len(funcs), 256):
        fs = funcs[lo:lo + 256]
        flat, off, _ = csr_from_sets([as_index_array(a), as_index_array(b)])
        sig = set_signatures_device(fs, flat, off, 2).cpu().numpy().view(np.uint32)
        out[lo:lo + len(fs)] = sig[0] == sig[1]
    return out


@dataclass(frozen=True)
class ProjectionFunction:
    """Inner product with a fixed standard-normal direction (hashing.py:195-219)."""

    direction: np.ndarray

    def __post_init__(self):
        d = np.ascontiguousarray(np.asarray(self.direction, dtype=np.float64))
        if d.ndim != 1:
            raise InvalidInput("direction must be a vector")
        object.__setattr__(self, "direction", d)

    @classmethod
    def from_seed(cls, seed: int, index: int, dim: int) -> "ProjectionFunction":
        # numpy's PCG64 + ziggurat stream is the reference's definition of the
        # directions (hashing.py:210): drawn on the host, 8*dim bytes per table
        return cls(np.random.default_rng([seed & M64, index]).standard_normal(dim))

    def __call__(self, x) -> float:
        xv = np.asarray(x, dtype=np.float64)
        if xv.shape != self.direction.shape:
            raise InvalidInput(f"dimension mismatch: {xv.shape} vs {self.direction.shape}")
        return float(self.direction @ xv)


@dataclass(frozen=True)
class SignatureScheme:
    """(K, L) MinHash signature composition (hashing.py:222-282)."""

    num_hashes: int
    num_tables: int
    universe: int
    seed: int = 0
    table_seeds: tuple = None

    def __post_init__(self):
        if self.num_hashes < 1 or self.num_tables < 1:
            raise InvalidInput("need at least one hash and one table")
        if self.table_seeds is not None:
            ts = tuple(tuple(int(s) for s in row) for row in self.table_seeds)
            if len(ts) != self.num_tables or any(len(r) != self.num_hashes for r in ts):
                raise InvalidInput("table_seeds must be L rows of K seeds")
            object.__setattr__(self, "table_seeds", ts)

    def function_seeds(self, table: int) -> tuple:
        if not 0 <= table < self.num_tables:
            raise InvalidInput("table index out of range")
        if self.table_seeds is not None:
            return self.table_seeds[table]
        return tuple(derive_seed(self.seed, table, j) for j in range(self.num_hashes))

    def functions(self, table: int) -> list:
        return [MinHashFunction(s, self.universe) for s in self.function_seeds(table)]

    def all_functions(self) -> list:
        """Functions of every table, table-major (index = table * K + j)."""
        return [f for tb in range(self.num_tables) for f in self.functions(tb)]

    def signature(self, table: int, s) -> tuple:
        return tuple(int(v) for v in self.signatures_for_sets(table, [s])[0])

    def signatures_for_sets(self, table: int, sets) -> np.ndarray:
        sets = [as_index_array(s) for s in sets]
        if not sets:
            return np.empty((0, self.num_hashes), dtype=np.uint64)
        if any(s.size == 0 for s in sets):
            raise InvalidInput("cannot sign an empty set")
        for s in sets:
            if s.min() < 0 or s.max() >= self.universe:
                raise InvalidInput("element outside hash universe")
        flat, off, _ = csr_from_sets(sets)
        sig = set_signatures_device(self.functions(table), flat, off, len(sets))
        return sig.cpu().numpy().view(np.uint32).astype(np.uint64)


@dataclass(frozen=True)
class DophReducer:
    """One-permutation hashing of sparse sets to [0, target_dims) (hashing.py:285-351)."""

    seed: int
    universe_size: int
    target_dims: int

    def __post_init__(self):
        if not 1 <= self.target_dims <= self.universe_size:
            raise InvalidInput("need 1 <= target_dims <= universe_size")

    @cached_property
    def _perm(self) -> MinHashFunction:
        return MinHashFunction(self.seed, self.universe_size)

    @cached_property
    def _width(self) -> int:
        return -(-self.universe_size // self.target_dims)

    def reduce_device(self, flat: torch.Tensor, offsets: torch.Tensor, nsets: int):
        """Device CSR in -> device CSR out (flat u32 as int32, offsets u64)."""
        batch = self._perm._batch
        st, _, tab = batch.args()
        counts = _lib.empty(max(1, nsets), _lib.U32)
        _lib.call("geek_doph_reduce", st, tab, _lib.ptr(flat), _lib.ptr(offsets), nsets, self.universe_size,
                  self.target_dims, _lib.ptr(counts), None, None, _lib.stream())
        cnt = counts[:nsets].to(torch.int64)
        off = torch.zeros(nsets + 1, dtype=torch.int64, device=flat.device)
        torch.cumsum(cnt, 0, out=off[1:])
        total = int(off[-1].item())
        out = _lib.empty(max(1, total), _lib.U32)
        _lib.call("geek_doph_reduce", st, tab, _lib.ptr(flat), _lib.ptr(offsets), nsets, self.universe_size,
                  self.target_dims, None, _lib.ptr(off), _lib.ptr(out), _lib.stream())
        return out, off

    def reduce(self, s) -> np.ndarray:
        arr = as_index_array(s)
        if arr.size == 0:
            raise InvalidInput("cannot reduce an empty set")
        return self.reduce_dataset([arr])[0]

    def reduce_dataset(self, sets) -> list:
        sets = [as_index_array(s) for s in sets]
        if any(s.size == 0 for s in sets):
            raise InvalidInput("cannot reduce an empty set")
        flat, off, _ = csr_from_sets(sets)
        out, ooff = self.reduce_device(flat, off, len(sets))
        o = ooff.cpu().numpy()
        v = out.cpu().numpy().view(np.uint32).astype(np.int64)
        return [v[o[i]:o[i + 1]] for i in range(len(sets))]

    def _range_mins(self, s):
        arr = as_index_array(s)
        if arr.size == 0:
            raise InvalidInput("cannot reduce an empty set")
        p = self._perm.permute(arr).astype(np.int64)
        bins = p // self._width
        rel = p - bins * self._width
        order = np.argsort(bins, kind="stable")
        bins, rel = bins[order], rel[order]
        uniq, start = np.unique(bins, return_index=True)
        return uniq, np.minimum.reduceat(rel, start)

    def sketch(self, s) -> np.ndarray:
        """Densified length-r vector of range minima (API helper, hashing.py:334-351)."""
        bins, mins = self._range_mins(s)
        r = self.target_dims
        out = np.full(r, -1, dtype=np.int64)
        out[bins] = mins
        carry = -1
        for j in range(2 * r - 1, -1, -1):
            jj = j % r
            if out[jj] >= 0:
                carry = out[jj]
            elif carry >= 0:
                out[jj] = carry
        return out
