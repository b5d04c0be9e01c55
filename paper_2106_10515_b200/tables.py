"""Device-resident bucket and group containers.

`BucketTable` is what the bucketize entry points return: the partition of
ids into buckets held as slot codes, id-major (`codes[i, j]` = slot of id i
in table j), which is the layout the SILK inverse-rank scan reads.  It
behaves like the reference's `list[Bucket]` (transform.py:112-128,
:158-169): len(), indexing and iteration materialise `Bucket` objects in
(table, slot) order on first use.

`GroupSet` is a CSR of sorted id groups (seed groups, bins, vote winners).
"""

from __future__ import annotations

from collections.abc import Sequence

import numpy as np
import torch

from . import _lib
from .data import Bucket, SeedGroup


def csr_gather(flat: torch.Tensor, off: torch.Tensor, idx: torch.Tensor):
    """Sub-CSR of the segments `idx` (device tensors; offsets int64)."""
    idx = idx.to(torch.int64)
    sizes = (off[1:] - off[:-1])[idx]
    noff = torch.zeros(idx.numel() + 1, dtype=torch.int64, device=off.device)
    torch.cumsum(sizes, 0, out=noff[1:])
    total = int(noff[-1].item()) if idx.numel() else 0
    if total == 0:
        return flat[:0], noff
    starts = torch.repeat_interleave(off[:-1][idx], sizes, output_size=total)
    local = torch.arange(total, device=off.device, dtype=torch.int64) - torch.repeat_interleave(
        noff[:-1], sizes, output_size=total)
    return flat[starts + local], noff


class GroupSet:
    """CSR of groups of uint32 ids (stored as int32) with int64 offsets."""

    def __init__(self, flat: torch.Tensor, off: torch.Tensor):
        self.flat = flat
        self.off = off

    @property
    def count(self) -> int:
        return int(self.off.numel() - 1)

    def sizes(self) -> torch.Tensor:
        return self.off[1:] - self.off[:-1]

    def select(self, idx: torch.Tensor) -> "GroupSet":
        f, o = csr_gather(self.flat, self.off, idx)
        return GroupSet(f, o)

    def to_host(self) -> list:
        off = self.off.cpu().numpy()
        flat = self.flat[: int(off[-1])].cpu().numpy().view(np.uint32).astype(np.int64) if off[-1] else \
            np.zeros(0, np.int64)
        return [flat[off[i]:off[i + 1]] for i in range(len(off) - 1)]

    def to_seed_groups(self) -> list:
        return [SeedGroup(g) for g in self.to_host()]

    @classmethod
    def from_host(cls, groups) -> "GroupSet":
        arrs = [np.asarray(g.members if isinstance(g, SeedGroup) else g, dtype=np.int64) for g in groups]
        sizes = np.array([a.size for a in arrs], dtype=np.int64)
        off = np.zeros(len(arrs) + 1, dtype=np.int64)
        np.cumsum(sizes, out=off[1:])
        flat = np.concatenate(arrs).astype(np.uint32) if arrs else np.zeros(0, np.uint32)
        if flat.size == 0:
            flat = np.zeros(1, np.uint32)
        return cls(_lib.to_dev(flat.view(np.int32)), _lib.to_dev(off))

    @classmethod
    def empty(cls) -> "GroupSet":
        return cls(_lib.zeros(1, torch.int32), _lib.zeros(1, torch.int64))


class BucketTable(Sequence):
    """m partitions of [0, n) held as id-major slot codes on the device."""

    def __init__(self, codes: torch.Tensor, n: int, tsizes, kind: str, even: bool):
        self.codes = codes  # int32 [n, m] (uint32 bits)
        self.n = int(n)
        self.tsizes = [int(t) for t in tsizes]
        self.m = len(self.tsizes)
        self.kind = kind  # "rank" (even split) | "sig" (signature buckets)
        self.even = even
        self.stride = max(self.tsizes) if self.tsizes else 0
        self.toff = np.concatenate(([0], np.cumsum(self.tsizes))).astype(np.int64)
        self._buckets = None
        self._csr = None

    # ---- Sequence protocol: list[Bucket] in (table, slot) order ----------
    def __len__(self) -> int:
        return int(self.toff[-1])

    def __getitem__(self, i):
        return self.buckets()[i]

    def __iter__(self):
        return iter(self.buckets())

    def bucket_sizes(self) -> torch.Tensor:
        """int64 sizes of every bucket, (table, slot) order."""
        if self.even:
            q, r = divmod(self.n, self.tsizes[0])
            one = np.full(self.tsizes[0], q, dtype=np.int64)
            one[:r] += 1
            return _lib.to_dev(np.tile(one, self.m))
        _, off = self.member_csr()
        return off[1:] - off[:-1]

    def member_csr(self):
        """(flat ids int32, offsets int64) of all buckets, (table, slot) order,
        members ascending -- a stable device sort of (table, code) pairs."""
        if self._csr is None:
            nm = self.n * self.m
            rows = torch.empty((nm, 2), dtype=torch.int32, device=self.codes.device)
            rows[:, 0] = torch.arange(self.m, device=self.codes.device, dtype=torch.int32).repeat(self.n)
            rows[:, 1] = self.codes.reshape(-1)
            perm = _lib.empty(nm, _lib.U32)
            gid = _lib.empty(nm, _lib.U32)
            ng = np.zeros(1, dtype=np.uint64)
            bits = np.array([max(1, int(self.m - 1).bit_length()), max(1, int(self.stride - 1).bit_length())],
                            dtype=np.int32)
            _lib.call("geek_group_rows", _lib.ptr(rows), nm, 2, _lib.hptr(bits), _lib.ptr(perm), _lib.ptr(gid),
                      _lib.hptr(ng), _lib.stream())
            flat = torch.div(perm.to(torch.int64), self.m, rounding_mode="floor").to(torch.int32)
            counts = torch.bincount(gid.to(torch.int64), minlength=int(ng[0]))
            off = torch.zeros(int(ng[0]) + 1, dtype=torch.int64, device=flat.device)
            torch.cumsum(counts, 0, out=off[1:])
            self._csr = (flat, off)
        return self._csr

    def buckets(self) -> list:
        if self._buckets is None:
            flat, off = self.member_csr()
            f = flat.cpu().numpy().view(np.uint32).astype(np.int64)
            o = off.cpu().numpy()
            out = []
            b = 0
            for j, t in enumerate(self.tsizes):
                for s in range(t):
                    out.append(Bucket(j, s, f[o[b]:o[b + 1]]))
                    b += 1
            self._buckets = out
        return self._buckets

    def codes_host(self) -> np.ndarray:
        """[m, n] int64 slot codes (parity helper)."""
        return self.codes.cpu().numpy().view(np.uint32).astype(np.int64).T.copy()
