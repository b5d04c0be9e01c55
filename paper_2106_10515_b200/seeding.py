"""SILK seeding (mirrors lshclust.seeding, seeding.py:1-197; engine.py:242-295).

Device pipeline:
  bucket signatures  -- inverse-rank scan over the id-major slot codes when
                        the buckets are an even rank split (K3'), else the
                        segmented-min MinHash over member CSR (K3)
  bins               -- per SILK table, lexicographic group-by of
                        (owner, K-signature) rows; groups of >= 2 buckets
  vote               -- (bin, id) membership pairs -> strict majority -> delta
  dedup              -- dedup-table signatures of the groups, group-by, one
                        representative per bin, canonical member-tuple order
`owner` carries the engine's logical-worker semantics: table j belongs to
worker j % g and only same-owner buckets can bin (engine.py:242-283).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .data import Bin, Bucket, CategoricalData, CentralVector, DenseData, InvalidInput, SeedGroup, SparseData
from .errors import EngineError
from .hashing import PermBatch, SignatureScheme, derive_seed, set_signatures_device, csr_from_sets
from .tables import BucketTable, GroupSet, csr_gather

__all__ = ["SeedingParams", "bin_buckets", "majority_vote", "find_seed_groups", "dedup_groups",
           "collect_votes", "seeds_to_centers"]

DEDUP_TAG = 0xDED0  # seeding.py:38


@dataclass(frozen=True)
class SeedingParams:
    """K hashes, L tables, min group size delta (seeding.py:41-80)."""

    num_hashes: int
    num_tables: int
    min_group_size: int = 1
    seed: int = 0
    dedup_tables: int = 1
    table_seeds: tuple = None
    dedup_seeds: tuple = None

    def __post_init__(self):
        if self.num_hashes < 1 or self.num_tables < 1 or self.dedup_tables < 1:
            raise InvalidInput("need K >= 1, L >= 1, dedup_tables >= 1")
        if self.min_group_size < 1:
            raise InvalidInput("minimum group size must be >= 1")

    def scheme(self, universe: int) -> SignatureScheme:
        return SignatureScheme(self.num_hashes, self.num_tables, universe, seed=self.seed,
                               table_seeds=self.table_seeds)

    def dedup_scheme(self, universe: int) -> SignatureScheme:
        return SignatureScheme(self.num_hashes, self.dedup_tables, universe,
                               seed=derive_seed(self.seed, DEDUP_TAG), table_seeds=self.dedup_seeds)


# ---------------------------------------------------------------------------
# bucket signatures

def bucket_signatures_codes(bt: BucketTable, funcs, info=None) -> torch.Tensor:
    """[H, m*t] int32 MinHash minima of every bucket of an even rank split
    via the inverse-rank scan (geek_silk_invscan)."""
    batch = PermBatch(funcs)
    nb = bt.m * bt.stride
    sig = _lib.empty(max(1, batch.n * nb), _lib.U32)
    draws = np.zeros(1, dtype=np.uint64)
    st, n, tab = batch.args()
    _lib.call("geek_silk_invscan", _lib.ptr(bt.codes), bt.n, bt.m, bt.stride, st, n, tab, _lib.ptr(sig), None,
              _lib.hptr(draws), _lib.stream())
    if info is not None:
        info["invscan_draws"] = int(draws[0])
    return sig[: batch.n * nb].view(batch.n, nb)


def bucket_signatures_csr(flat, off, nsets, funcs) -> torch.Tensor:
    """[H, nsets] via segmented-min MinHash over member CSR."""
    sig = set_signatures_device(funcs, flat, off, nsets, PermBatch(funcs))
    return sig.t().contiguous()


def silk_signatures(buckets, scheme: SignatureScheme, info=None):
    """(sig [L*K, nb], nb, csr or None) for a BucketTable or list[Bucket]."""
    funcs = scheme.all_functions()
    if isinstance(buckets, BucketTable):
        if buckets.even and buckets.n == scheme.universe:
            return bucket_signatures_codes(buckets, funcs, info), len(buckets), None
        flat, off = buckets.member_csr()
        return bucket_signatures_csr(flat, off, len(buckets), funcs), len(buckets), (flat, off)
    sets = [b.members for b in buckets]
    for s in sets:
        if s.size and (s.min() < 0 or s.max() >= scheme.universe):
            raise InvalidInput("element outside hash universe")
    flat, off, _ = csr_from_sets(sets)
    return bucket_signatures_csr(flat, off, len(sets), funcs), len(sets), (flat, off)


# ---------------------------------------------------------------------------
# bins

class Bins:
    """All bins of all SILK tables: (bucket, bin) pairs, bin sizes, bin table."""

    def __init__(self, pair_bucket, pair_bin, bin_size, bin_table, bin_sig):
        self.pair_bucket = pair_bucket  # int64 [P] bucket position
        self.pair_bin = pair_bin        # int64 [P] global bin id
        self.bin_size = bin_size        # int32 [B] buckets per bin
        self.bin_table = bin_table      # int64 [B] SILK table of each bin (device)
        self.bin_sig = bin_sig          # int32 [B, K] signature of each bin

    @property
    def count(self) -> int:
        return int(self.bin_size.numel())


def find_bins(sig: torch.Tensor, K: int, L: int, universe: int, owner: torch.Tensor = None,
              tables=None, prune=None) -> Bins:
    """Per SILK table, group buckets by (owner, signature); keep groups of
    >= 2 buckets (seeding.py:83-104, engine.py:270-277).  Bin ids are
    table-major, then in sorted (owner, signature) order."""
    nb = sig.shape[1]
    dev = sig.device
    tables = list(range(L) if tables is None else tables)
    nt = len(tables)
    if nb == 0 or nt == 0:
        z = torch.zeros(0, dtype=torch.int64, device=dev)
        return Bins(z, z, torch.zeros(0, dtype=torch.int32, device=dev), z,
                    torch.zeros((0, K), dtype=torch.int32, device=dev))
    # all SILK tables in one group-by: rows (table, owner, signature), the
    # table column most significant, so groups come out table-major
    width = K + 1 + (1 if owner is not None else 0)
    bits = [max(1, int(nt - 1).bit_length())] + \
        ([max(1, int(int(owner.max().item())).bit_length())] if owner is not None else []) + \
        [max(1, int(universe - 1).bit_length())] * K
    bits = np.array(bits, dtype=np.int32)
    tcol = torch.arange(nt, dtype=torch.int32, device=dev).repeat_interleave(nb)
    cols = [tcol]
    if owner is not None:
        cols.append(owner.to(torch.int32).repeat(nt))
    idx = _lib.to_dev(np.array([st * K for st in tables], dtype=np.int64))
    for j in range(K):
        cols.append(sig.index_select(0, idx + j).reshape(-1).to(torch.int32))
    rows = torch.stack(cols, dim=1).contiguous()
    nr = nt * nb
    perm = _lib.empty(nr, _lib.U32)
    gid = _lib.empty(nr, _lib.U32)
    ng = np.zeros(1, dtype=np.uint64)
    _lib.call("geek_group_rows", _lib.ptr(rows), nr, width, _lib.hptr(bits), _lib.ptr(perm), _lib.ptr(gid),
              _lib.hptr(ng), _lib.stream())
    g = gid.to(torch.int64)
    counts = torch.bincount(g, minlength=int(ng[0]))
    binned = counts >= 2
    newid = torch.cumsum(binned.to(torch.int64), 0) - 1
    sel = binned[g]
    p64 = perm.to(torch.int64)
    psel = p64[sel]
    first = torch.ones_like(sel)
    first[1:] = g[1:] != g[:-1]
    heads = p64[sel & first]
    bt = _lib.to_dev(np.asarray(tables, dtype=np.int64))[rows[heads, 0].to(torch.int64)]
    bins = Bins(psel % nb, newid[g][sel], counts[binned].to(torch.int32), bt, rows[heads][:, -K:])
    return _prune_bins(bins, *prune) if prune is not None else bins


def _prune_bins(bins: Bins, bucket_sizes: torch.Tensor, delta: int) -> Bins:
    """Drop the bins that cannot yield a group of >= delta winners (exact:
    a winner lies in >= need = |bin| // 2 + 1 of the bin's buckets, so
    #winners <= sum of the bin's bucket sizes // need).  Pipeline use only --
    the reference-facing bin_buckets / collect_votes keep every bin.  On
    signature buckets this removes the bins of one id's identical singleton
    buckets across its owner's tables (one winner each)."""
    B = bins.count
    if B == 0:
        return bins
    tot = torch.zeros(B, dtype=torch.int64, device=bins.pair_bin.device).index_add_(
        0, bins.pair_bin, bucket_sizes[bins.pair_bucket].to(torch.int64))
    need = bins.bin_size.to(torch.int64) // 2 + 1
    keep = tot // need >= max(1, int(delta))
    if bool(keep.all().item()):
        return bins
    newid = torch.cumsum(keep.to(torch.int64), 0) - 1
    pk = keep[bins.pair_bin]
    return Bins(bins.pair_bucket[pk], newid[bins.pair_bin[pk]], bins.bin_size[keep], bins.bin_table[keep],
                bins.bin_sig[keep])


# ---------------------------------------------------------------------------
# vote

def membership_pairs(bins: Bins, buckets, csr, bucket_sizes: torch.Tensor):
    """(pair_bin, pair_id) int32 for every id of every binned bucket."""
    if bins.pair_bucket.numel() == 0:
        z = torch.zeros(0, dtype=torch.int32, device=bins.pair_bin.device)
        return z, z
    if csr is not None:
        flat, off = csr
        ids, noff = csr_gather(flat, off, bins.pair_bucket)
        sizes = noff[1:] - noff[:-1]
        pbin = torch.repeat_interleave(bins.pair_bin, sizes, output_size=ids.numel())
        return pbin.to(torch.int32).contiguous(), ids.contiguous()
    # id-major codes: one pass over codes emits (bin, id) for binned buckets
    bt: BucketTable = buckets
    nb = bt.m * bt.stride
    order = torch.argsort(bins.pair_bucket, stable=True)
    pbk = bins.pair_bucket[order]
    pbn = bins.pair_bin[order].to(torch.int32).contiguous()
    # an id's count in a bin is at most the number of distinct tables among the
    # bin's buckets (one bucket per table per id): bins with 2 * that <= |bin|
    # cannot be won by anyone, so their memberships are not emitted at all
    key = pbn.to(torch.int64) * bt.m + pbk // bt.stride
    dt = torch.bincount(torch.unique(key) // bt.m, minlength=bins.count)
    keep = (2 * dt > bins.bin_size.to(torch.int64))[pbn.to(torch.int64)]
    pbk, pbn = pbk[keep], pbn[keep].contiguous()
    cnt = torch.bincount(pbk, minlength=nb)
    bb_off = torch.zeros(nb + 1, dtype=torch.int64, device=pbk.device)
    torch.cumsum(cnt, 0, out=bb_off[1:])
    bb_off = bb_off.to(torch.int32).contiguous()
    cap = int(bucket_sizes[bins.pair_bucket].sum().item())
    out_bin = _lib.empty(max(1, cap), _lib.U32)
    out_id = _lib.empty(max(1, cap), _lib.U32)
    count = np.zeros(1, dtype=np.uint64)
    _lib.call("geek_emit_members_codes", _lib.ptr(bt.codes), bt.n, bt.m, bt.stride, _lib.ptr(bb_off),
              _lib.ptr(pbn), _lib.ptr(out_bin), _lib.ptr(out_id), cap, _lib.hptr(count), _lib.stream())
    c = int(count[0])
    return out_bin[:c], out_id[:c]


def vote(pair_bin, pair_id, bins: Bins, delta: int):
    """Strict-majority winners per bin, bins with < delta winners dropped ->
    (GroupSet ordered by bin id, winning bin ids int64)."""
    npairs = int(pair_bin.numel())
    if npairs == 0 or bins.count == 0:
        return GroupSet.empty(), torch.zeros(0, dtype=torch.int64, device=pair_bin.device)
    wb = _lib.empty(npairs, _lib.U32)
    wi = _lib.empty(npairs, _lib.U32)
    nw = np.zeros(1, dtype=np.uint64)
    _lib.call("geek_majority_vote", _lib.ptr(pair_bin.contiguous()), _lib.ptr(pair_id.contiguous()), npairs,
              _lib.ptr(bins.bin_size.contiguous()), bins.count, int(delta), _lib.ptr(wb), _lib.ptr(wi),
              _lib.hptr(nw), _lib.stream())
    k = int(nw[0])
    if k == 0:
        return GroupSet.empty(), torch.zeros(0, dtype=torch.int64, device=pair_bin.device)
    wb, wi = wb[:k].to(torch.int64), wi[:k]
    ub, cnt = torch.unique_consecutive(wb, return_counts=True)
    off = torch.zeros(ub.numel() + 1, dtype=torch.int64, device=wb.device)
    torch.cumsum(cnt, 0, out=off[1:])
    return GroupSet(wi.contiguous(), off), ub


def fused_votes_codes(bins: Bins, bt: BucketTable, bucket_sizes: torch.Tensor, delta: int):
    """Emission with the majority decided per id row (geek_emit_winners_codes),
    then winners grouped by bin.  None if an id reaches too many bins."""
    if bins.pair_bucket.numel() == 0:
        return GroupSet.empty(), torch.zeros(0, dtype=torch.int64, device=bins.pair_bin.device), 0
    nb = bt.m * bt.stride
    order = torch.argsort(bins.pair_bucket, stable=True)
    pbk = bins.pair_bucket[order]
    pbn = bins.pair_bin[order].to(torch.int32).contiguous()
    # an id's count in a bin is at most the number of distinct tables among the
    # bin's buckets (one bucket per table per id): bins with 2 * that <= |bin|
    # cannot be won by anyone, so their memberships are not emitted at all
    key = pbn.to(torch.int64) * bt.m + pbk // bt.stride
    dt = torch.bincount(torch.unique(key) // bt.m, minlength=bins.count)
    keep = (2 * dt > bins.bin_size.to(torch.int64))[pbn.to(torch.int64)]
    pbk, pbn = pbk[keep], pbn[keep].contiguous()
    cnt = torch.bincount(pbk, minlength=nb)
    bb_off = torch.zeros(nb + 1, dtype=torch.int64, device=pbk.device)
    torch.cumsum(cnt, 0, out=bb_off[1:])
    bb_off = bb_off.to(torch.int32).contiguous()
    cap = max(1, int(bucket_sizes[bins.pair_bucket].sum().item()))
    wb = _lib.empty(cap, _lib.U32)
    wi = _lib.empty(cap, _lib.U32)
    count = np.zeros(1, dtype=np.uint64)
    try:
        _lib.call("geek_emit_winners_codes", _lib.ptr(bt.codes), bt.n, bt.m, bt.stride, _lib.ptr(bb_off),
                  _lib.ptr(pbn), _lib.ptr(bins.bin_size.contiguous()), _lib.ptr(wb), _lib.ptr(wi), cap,
                  _lib.hptr(count), _lib.stream())
    except EngineError:
        return None
    nw = int(count[0])
    if nw == 0:
        return GroupSet.empty(), torch.zeros(0, dtype=torch.int64, device=wb.device), 0
    ob = _lib.empty(nw, _lib.U32)
    oi = _lib.empty(nw, _lib.U32)
    nk = np.zeros(1, dtype=np.uint64)
    _lib.call("geek_group_winners", _lib.ptr(wb), _lib.ptr(wi), nw, bins.count, bt.n, int(delta), _lib.ptr(ob),
              _lib.ptr(oi), _lib.hptr(nk), _lib.stream())
    k = int(nk[0])
    if k == 0:
        return GroupSet.empty(), torch.zeros(0, dtype=torch.int64, device=wb.device), nw
    ub, c = torch.unique_consecutive(ob[:k].to(torch.int64), return_counts=True)
    off = torch.zeros(ub.numel() + 1, dtype=torch.int64, device=wb.device)
    torch.cumsum(c, 0, out=off[1:])
    return GroupSet(oi[:k].contiguous(), off), ub, nw


def _concat_bins(parts) -> Bins:
    """Bins of consecutive SILK tables -> one Bins (bin ids offset, table-major kept)."""
    if len(parts) == 1:
        return parts[0]
    offs, base = [], 0
    for b in parts:
        offs.append(base)
        base += b.count
    return Bins(torch.cat([b.pair_bucket for b in parts]),
                torch.cat([b.pair_bin + o for b, o in zip(parts, offs)]),
                torch.cat([b.bin_size for b in parts]), torch.cat([b.bin_table for b in parts]),
                torch.cat([b.bin_sig for b in parts]))


def _bins_per_table(buckets: BucketTable, scheme: SignatureScheme, K: int, L: int, universe: int, owner, delta):
    """Signature buckets (member CSR): SILK signatures and the group-by one
    SILK table at a time, so neither the [L*K, buckets] signatures nor the
    L * buckets group-by rows exist at once (Criteo-like inputs reach ~10^8
    buckets per table).  Same bins, same table-major order."""
    flat, off = buckets.member_csr()
    nb = len(buckets)
    sizes = off[1:] - off[:-1]
    parts = []
    for st in range(L):
        sig = bucket_signatures_csr(flat, off, nb, scheme.functions(st))  # [K, nb]
        b = find_bins(sig, K, 1, universe, owner, tables=[0], prune=(sizes, delta))
        del sig
        b.bin_table = torch.full_like(b.bin_table, st)
        parts.append(b)
    return _concat_bins(parts), (flat, off)


def _group_all(rows: torch.Tensor, bits: np.ndarray):
    """Group-by of device rows [nr, w] u32 in lexicographic order ->
    (perm int64 sorted positions, gid int64 per sorted position, count)."""
    nr = int(rows.shape[0])
    perm = _lib.empty(nr, _lib.U32)
    gid = _lib.empty(nr, _lib.U32)
    ng = np.zeros(1, dtype=np.uint64)
    _lib.call("geek_group_rows", _lib.ptr(rows), nr, int(rows.shape[1]), _lib.hptr(bits), _lib.ptr(perm),
              _lib.ptr(gid), _lib.hptr(ng), _lib.stream())
    return perm.to(torch.int64), gid.to(torch.int64), int(ng[0])


def _bins_per_table_singletons(buckets: BucketTable, scheme: SignatureScheme, K: int, L: int, universe: int,
                               owner, delta: int):
    """_bins_per_table for delta >= 2 without group-by rows for singleton
    buckets (most signature buckets of a Criteo-like input hold one id).

    A singleton bucket {m} has signature (pi_1(m), .., pi_K(m)); pi_1 is a
    bijection, so it shares a bin key (owner o, sigma) with a bucket B only if
    m = pi_1^-1(sigma_1) -- B's pi_1-minimum, a member of B -- and
    pi_j(m) = sigma_j for every j.  A bin of singletons alone holds one id c
    times: at most c // (c // 2 + 1) <= 1 < delta winners, pruned.  So the
    group-by runs over the buckets of >= 2 ids only, each group's candidate
    singletons (m, o) are counted from one sorted key list, and the bins,
    their bucket lists (ascending bucket position, as the stable group-by
    emits them), the pruning rule and the table-major (owner, signature)
    order are those of _bins_per_table."""
    flat, off = buckets.member_csr()
    nb = len(buckets)
    dev = flat.device
    sizes = off[1:] - off[:-1]
    single = sizes == 1
    nidx = torch.nonzero(~single, as_tuple=True)[0]
    sidx = torch.nonzero(single, as_tuple=True)[0]
    G = 1 if owner is None else int(owner.max().item()) + 1 if owner.numel() else 1
    own = owner.to(torch.int64) if owner is not None else torch.zeros(nb, dtype=torch.int64, device=dev)
    skey = flat[off[:-1][sidx]].to(torch.int64) * G + own[sidx]
    skey, sord = torch.sort(skey, stable=True)  # equal keys keep ascending bucket position
    spos = sidx[sord]
    fN, oN = csr_gather(flat, off, nidx)
    szN = sizes[nidx]
    ownN = own[nidx].to(torch.int32)
    obits = max(1, int(G - 1).bit_length())
    bits = np.array(([obits] if owner is not None else []) + [max(1, int(universe - 1).bit_length())] * K,
                    dtype=np.int32)
    parts = []
    for st in range(L):
        funcs = scheme.functions(st)
        empty = Bins(torch.zeros(0, dtype=torch.int64, device=dev), torch.zeros(0, dtype=torch.int64, device=dev),
                     torch.zeros(0, dtype=torch.int32, device=dev), torch.zeros(0, dtype=torch.int64, device=dev),
                     torch.zeros((0, K), dtype=torch.int32, device=dev))
        if nidx.numel() == 0:
            parts.append(empty)
            continue
        sig = bucket_signatures_csr(fN, oN, int(nidx.numel()), funcs)  # [K, |N|]
        cols = ([ownN] if owner is not None else []) + [sig[j] for j in range(K)]
        rows = torch.stack(cols, dim=1).contiguous()
        del sig
        perm, gid, ng = _group_all(rows, bits)
        first = torch.ones(perm.numel(), dtype=torch.bool, device=dev)
        first[1:] = gid[1:] != gid[:-1]
        heads = perm[first]                                   # one N row per group, group order
        hsig = rows[heads][:, -K:].contiguous()               # [ng, K] int32 (u32 bits)
        hown = ownN[heads].to(torch.int64)
        cntN = torch.bincount(gid, minlength=ng)
        totN = torch.zeros(ng, dtype=torch.int64, device=dev).index_add_(0, gid, szN[perm])
        # candidate singleton id of each group and its count
        batch = PermBatch(funcs)
        s0 = hsig[:, 0].contiguous()
        m = _lib.empty(ng, _lib.U32)
        st_, n_, tab_ = PermBatch(funcs[:1]).args()
        _lib.call("geek_perm_inverse", st_, n_, tab_, _lib.ptr(s0), ng, _lib.ptr(m), _lib.stream())
        fw = _lib.empty(max(1, ng * K), _lib.U32)
        st_, n_, tab_ = batch.args()
        _lib.call("geek_perm_forward", st_, n_, tab_, _lib.ptr(m), ng, _lib.ptr(fw), _lib.stream())
        match = (fw[: ng * K].view(K, ng) == hsig.t()).all(dim=0)
        ckey = (m.to(torch.int64) & 0xFFFFFFFF) * G + hown
        lo = torch.searchsorted(skey, ckey, side="left")
        hi = torch.searchsorted(skey, ckey, side="right")
        cS = torch.where(match, hi - lo, torch.zeros_like(lo))
        bsize = cntN + cS
        need = bsize // 2 + 1
        keep = (bsize >= 2) & ((totN + cS) // need >= delta)
        kept = int(keep.sum().item())
        if kept == 0:
            parts.append(empty)
            continue
        newid = torch.cumsum(keep.to(torch.int64), 0) - 1
        selN = keep[gid]
        pbN = nidx[perm[selN]]
        pnN = newid[gid[selN]]
        kg = torch.nonzero(keep & (cS > 0), as_tuple=True)[0]
        if kg.numel():
            cnt = cS[kg]
            tot = int(cnt.sum().item())
            start = torch.repeat_interleave(lo[kg], cnt, output_size=tot)
            ooff = torch.zeros(kg.numel() + 1, dtype=torch.int64, device=dev)
            torch.cumsum(cnt, 0, out=ooff[1:])
            local = torch.arange(tot, device=dev, dtype=torch.int64) - torch.repeat_interleave(
                ooff[:-1], cnt, output_size=tot)
            pbS = spos[start + local]
            pnS = torch.repeat_interleave(newid[kg], cnt, output_size=tot)
            pb = torch.cat([pbN, pbS])
            pn = torch.cat([pnN, pnS])
            order = torch.argsort(pn * nb + pb)
            pb, pn = pb[order], pn[order]
        else:
            pb, pn = pbN, pnN
        parts.append(Bins(pb, pn, bsize[keep].to(torch.int32), torch.full((kept,), st, dtype=torch.int64,
                                                                             device=dev), hsig[keep]))
    return _concat_bins(parts), (flat, off)


_SPLIT_ROWS = 1 << 28  # group-by rows above which signature-bucket bins are formed table by table
_SINGLETON_BINS = True  # ... and singleton buckets join bins by lookup instead of group-by rows


def silk_votes(buckets, params: SeedingParams, universe: int, owner=None, info=None):
    """Every surviving vote of every SILK table (collect_votes / local_votes)
    -> (GroupSet, Bins, winning bin ids)."""
    scheme = params.scheme(universe)
    if (isinstance(buckets, BucketTable) and not (buckets.even and buckets.n == scheme.universe)
            and len(buckets) * params.num_tables > _SPLIT_ROWS):
        form = _bins_per_table_singletons if _SINGLETON_BINS and params.min_group_size >= 2 else _bins_per_table
        bins, csr = form(buckets, scheme, params.num_hashes, params.num_tables, universe, owner,
                         params.min_group_size)
        if info is not None:
            info["silk_bins_path"] = form.__name__
    else:
        sig, nb, csr = silk_signatures(buckets, scheme, info)
        bins = find_bins(sig, params.num_hashes, params.num_tables, universe, owner)
        del sig
        if isinstance(buckets, BucketTable) and not buckets.even:
            bins = _prune_bins(bins, buckets.bucket_sizes(), params.min_group_size)
    if isinstance(buckets, BucketTable):
        sizes = buckets.bucket_sizes()
        if info is not None:
            info["silk_buckets"] = len(buckets)
    else:
        sizes = _lib.to_dev(np.array([b.members.size for b in buckets], dtype=np.int64))
    if csr is None:
        fused = fused_votes_codes(bins, buckets, sizes, params.min_group_size)
        if fused is not None:
            groups, won, nw = fused
            if info is not None:
                info["bins"] = bins.count
                info["vote_winners"] = nw
                info["raw_groups"] = groups.count
            return groups, bins, won
    groups, won, npairs = _batched_votes(bins, buckets, csr, sizes, params.min_group_size)
    if info is not None:
        info["bins"] = bins.count
        info["vote_pairs"] = npairs
        info["raw_groups"] = groups.count
    return groups, bins, won


_PAIR_BATCH = 1 << 28  # (bin, id) pairs materialised at once


def _batched_votes(bins: Bins, buckets, csr, sizes, delta):
    """membership_pairs + vote over contiguous bin-id ranges holding at most
    _PAIR_BATCH pairs each (bins are independent; the concatenation keeps the
    bin-id order of the single pass), so giant buckets -- e.g. low-cardinality
    categorical attributes -- do not need all pairs in memory at once."""
    B = bins.count
    pb_sizes = sizes[bins.pair_bucket] if bins.pair_bucket.numel() else sizes[:0]
    total = int(pb_sizes.sum().item()) if pb_sizes.numel() else 0
    if total <= _PAIR_BATCH or B <= 1:
        pbin, pid = membership_pairs(bins, buckets, csr, sizes)
        g, w = vote(pbin, pid, bins, delta)
        return g, w, int(pbin.numel())
    per_bin = torch.zeros(B, dtype=torch.int64, device=pb_sizes.device).index_add_(0, bins.pair_bin, pb_sizes)
    cum = torch.cumsum(per_bin, 0).cpu().numpy()
    cuts, b0 = [0], 0
    while b0 < B:
        before = cum[b0 - 1] if b0 else 0
        b1 = int(np.searchsorted(cum, before + _PAIR_BATCH, side="right"))
        b1 = min(B, max(b1, b0 + 1))
        cuts.append(b1)
        b0 = b1
    parts, wons, npairs = [], [], 0
    pbn = bins.pair_bin
    ordered = bool((pbn[1:] >= pbn[:-1]).all().item())  # find_bins emits pairs in bin order
    if ordered:
        bounds = torch.searchsorted(pbn, torch.tensor(cuts, dtype=pbn.dtype, device=pbn.device)).cpu().numpy()
    for q, (b0, b1) in enumerate(zip(cuts[:-1], cuts[1:])):
        if ordered:
            m = slice(int(bounds[q]), int(bounds[q + 1]))
        else:
            m = (pbn >= b0) & (pbn < b1)
        sub = Bins(bins.pair_bucket[m], pbn[m] - b0, bins.bin_size[b0:b1], bins.bin_table[b0:b1],
                   bins.bin_sig[b0:b1])
        pbin, pid = membership_pairs(sub, buckets, csr, sizes)
        npairs += int(pbin.numel())
        g, w = vote(pbin, pid, sub, delta)
        del pbin, pid
        if g.count:
            parts.append(g)
            wons.append(w + b0)
    if not parts:
        return GroupSet.empty(), torch.zeros(0, dtype=torch.int64, device=pb_sizes.device), npairs
    flat = torch.cat([g.flat[: int(g.off[-1].item())] for g in parts])
    offs, base = [torch.zeros(1, dtype=torch.int64, device=flat.device)], 0
    for g in parts:
        offs.append(g.off[1:] + base)
        base += int(g.off[-1].item())
    return GroupSet(flat.contiguous(), torch.cat(offs)), torch.cat(wons), npairs


# ---------------------------------------------------------------------------
# dedup

def dedup_device(groups: GroupSet, params: SeedingParams, universe: int) -> GroupSet:
    """dedup_groups on the device (seeding.py:117-134) -> canonical order."""
    if groups.count > 1:
        scheme = params.dedup_scheme(universe)
        K = params.num_hashes
        bits = np.full(K, max(1, int(universe - 1).bit_length()), dtype=np.int32)
        for tb in range(params.dedup_tables):
            cnt = groups.count
            sig = set_signatures_device(scheme.functions(tb), groups.flat, groups.off, cnt)
            perm = _lib.empty(cnt, _lib.U32)
            gid = _lib.empty(cnt, _lib.U32)
            ng = np.zeros(1, dtype=np.uint64)
            _lib.call("geek_group_rows", _lib.ptr(sig.contiguous()), cnt, K, _lib.hptr(bits), _lib.ptr(perm),
                      _lib.ptr(gid), _lib.hptr(ng), _lib.stream())
            keep = _lib.empty(cnt, torch.uint8)
            _lib.call("geek_pick_representatives", _lib.ptr(groups.flat), _lib.ptr(groups.off), _lib.ptr(perm),
                      _lib.ptr(gid), cnt, _lib.ptr(keep), _lib.stream())
            groups = groups.select(torch.nonzero(keep, as_tuple=True)[0])
    return canonical_order(groups)


def canonical_order(groups: GroupSet) -> GroupSet:
    """Sort groups by member tuple, proper prefix first (data.py:200-202)."""
    cnt = groups.count
    if cnt <= 1:
        return groups
    order = _lib.empty(cnt, _lib.U32)
    _lib.call("geek_sort_groups", _lib.ptr(groups.flat), _lib.ptr(groups.off), cnt, _lib.ptr(order),
              _lib.stream())
    return groups.select(order.to(torch.int64))


# ---------------------------------------------------------------------------
# reference API

def bin_buckets(buckets, params: SeedingParams, table: int, universe: int) -> list:
    """seeding.py:93-104 -> list[Bin] in signature order."""
    if not buckets or len(buckets) == 0:
        return []
    scheme = params.scheme(universe)
    sig, nb, csr = silk_signatures(buckets, scheme)
    bins = find_bins(sig, params.num_hashes, params.num_tables, universe, None, tables=[table])
    pbk = bins.pair_bucket.cpu().numpy()
    pbn = bins.pair_bin.cpu().numpy()
    bsig = bins.bin_sig.cpu().numpy().view(np.uint32).astype(np.int64)
    out = []
    for b in range(bins.count):
        idx = tuple(int(i) for i in np.sort(pbk[pbn == b]))
        out.append(Bin(signature=tuple(int(v) for v in bsig[b]), bucket_indices=idx))
    return out


def majority_vote(bin_: Bin, buckets) -> SeedGroup | None:
    """seeding.py:107-114 (strict majority over the bin's buckets)."""
    parts = [buckets[i].members for i in bin_.bucket_indices]
    flat, off, sizes = csr_from_sets(parts)
    ids = flat[: int(sizes.sum())]
    pbin = torch.zeros_like(ids)
    bins = Bins(None, None, _lib.to_dev(np.array([len(parts)], dtype=np.int32)), np.zeros(1, np.int64), None)
    groups, _ = vote(pbin, ids, bins, 1)
    if groups.count == 0:
        return None
    return SeedGroup(groups.to_host()[0])


def collect_votes(buckets, params: SeedingParams, universe: int, trace=None) -> list:
    """seeding.py:154-165: every surviving vote, table-major, bins in signature order."""
    groups, bins, won = silk_votes(buckets, params, universe)
    out = groups.to_seed_groups()
    if trace is not None and out:
        pbk = bins.pair_bucket.cpu().numpy()
        pbn = bins.pair_bin.cpu().numpy()
        btab = bins.bin_table.cpu().numpy()
        for g, b in zip(out, won.cpu().numpy().tolist()):
            idx = np.sort(pbk[pbn == b])
            trace.append((int(btab[b]), tuple(buckets[int(i)].bucket_id for i in idx), g))
    return out


def find_seed_groups(buckets, params: SeedingParams, universe: int, trace=None) -> list:
    """seeding.py:137-151: bin + vote + delta, then dedup."""
    if buckets is None or len(buckets) == 0:
        raise InvalidInput("seeding needs at least one bucket")
    if trace is not None:
        raw = collect_votes(buckets, params, universe, trace)
        return dedup_device(GroupSet.from_host(raw), params, universe).to_seed_groups()
    groups, _, _ = silk_votes(buckets, params, universe)
    return dedup_device(groups, params, universe).to_seed_groups()


def dedup_groups(groups, params: SeedingParams, universe: int) -> list:
    """seeding.py:117-134."""
    gs = [g if isinstance(g, SeedGroup) else SeedGroup(g) for g in groups]
    if not gs:
        return []
    for g in gs:
        if g.members.max() >= universe:
            raise InvalidInput("element outside hash universe")
    return dedup_device(GroupSet.from_host(gs), params, universe).to_seed_groups()


def seeds_to_centers(groups, data) -> list:
    """seeding.py:168-197: exact centroid / attribute mode / majority membership."""
    from .numeric import dense_centers, mode_centers, sparse_centers

    gs = groups if isinstance(groups, GroupSet) else GroupSet.from_host(groups)
    if gs.count == 0:
        return []
    sizes = gs.sizes().cpu().numpy()
    if isinstance(data, DenseData):
        C = dense_centers(data.device_vectors(), gs).cpu().numpy()
        return [CentralVector("centroid", C[i], int(sizes[i])) for i in range(gs.count)]
    if isinstance(data, CategoricalData):
        M = mode_centers(data.device_codes(), data.code_space, gs).cpu().numpy()
        return [CentralVector("mode", M[i], int(sizes[i])) for i in range(gs.count)]
    if isinstance(data, SparseData):
        M = sparse_centers(data, gs).cpu().numpy()
        return [CentralVector("mode", M[i], int(sizes[i])) for i in range(gs.count)]
    raise InvalidInput("unsupported dataset type for center computation")
