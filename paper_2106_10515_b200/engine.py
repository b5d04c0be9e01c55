"""Partitioned-worker engine on one process per GPU (mirrors lshclust.engine,
engine.py:1-537).

Semantics are those of the reference's g logical workers (WorkerConfig):
contiguous id shards (engine.py:109-115), table j owned by worker j % g
(engine.py:199-238), bins formed only among one owner's tables
(engine.py:242-283), seed groups merged and deduplicated on every worker
(engine.py:285-295), exact centers reduced from per-shard sums
(engine.py:481-516), local assignment (engine.py:327-346).  The results
depend on g, never on the number of physical GPUs G (G must divide g).

Physical mapping (B200, NCCL over NVLink): each rank projects its own shard;
an all-to-all moves every table's keys to the rank owning it (j % G); the
owner rank-splits, scans and votes its tables over all n ids; seed groups
are all-gathered and deduplicated identically on every rank; exact digit
sums are all-reduced; radii (max) and sizes (sum) are all-reduced.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .assignment import (AssignStats, assign_cat_device, assign_l2_device, assign_sparse_device, pairwise_sum,
                         radii_sizes)
from .data import CategoricalData, CentralVector, Clustering, DenseData, MixedData, SeedGroup, SparseData
from .errors import EngineError, InvalidInput
from .hashing import DophReducer, derive_seed
from .numeric import (center_stats_bytes, digit_count, exponent_range, label_mode_centers, label_mode_counts,
                      label_sparse_counts, label_sums, mode_centers, mode_counts, partial_sums, round_means,
                      sparse_counts)
from .seeding import SeedingParams, dedup_device, silk_votes
from .tables import BucketTable, GroupSet
from .transform import (HomoTransformParams, MinhashTransformParams, categorical_token_csr, directions_device,
                        discretize_numeric, even_partition_sizes, group_signature_tables, project_keys,
                        projection_tolerance, rank_split_codes, signature_bucket_codes, signature_rows,
                        split_boundary_stats)

__all__ = ["EngineError", "WorkerConfig", "PipelineConfig", "PipelineResult", "split_data", "run_pipeline"]


@dataclass(frozen=True)
class WorkerConfig:
    """Logical worker count g, seeding memory budget, transport (engine.py:49-69).

    `transport` "in-process" (the reference's only kind) and "nccl" are
    accepted; with a torch.distributed process group of G ranks the engine
    always runs over it."""

    num_workers: int
    memory_budget: int = 1 << 30
    transport: str = "in-process"

    def __post_init__(self):
        if self.num_workers < 1:
            raise InvalidInput("need at least one worker")
        if self.memory_budget <= 0:
            raise InvalidInput("memory budget must be positive")
        if self.transport not in ("in-process", "nccl"):
            raise InvalidInput(f"unknown transport {self.transport!r}")


def split_data(n: int, g: int) -> list:
    """engine.py:109-115."""
    if g > n:
        raise InvalidInput(f"cannot split {n} objects across {g} workers")
    b = np.concatenate(([0], np.cumsum(even_partition_sizes(n, g))))
    return [(int(b[i]), int(b[i + 1])) for i in range(g)]


@dataclass
class PipelineConfig:
    metric: str
    transform_kind: str
    workers: WorkerConfig
    homo: HomoTransformParams = None
    minhash: MinhashTransformParams = None
    seeding: SeedingParams = None
    passes: int = 0
    fallback_seed: int = 0

    def table_count(self) -> int:
        return self.homo.num_tables if self.transform_kind == "dense" else self.minhash.num_tables


class PipelineResult:
    """Results stay on the device; the reference-typed fields materialise lazily."""

    def __init__(self, centers, groups: GroupSet, labels, best, radii, sizes, objective, timings, transport_bytes,
                 warnings, info, gather_labels=None):
        self._centers = centers
        self._groups = groups
        self.labels_device = labels
        self.best_device = best
        self.radii_device = radii
        self.sizes_device = sizes
        self.objective = objective
        self.timings = timings
        self.transport_bytes = transport_bytes
        self.warnings = warnings
        self.info = info
        self._gather_labels = gather_labels
        self._clustering = None
        self._seed_groups = None

    @property
    def k_star(self) -> int:
        return int((self.sizes_device > 0).sum().item())

    @property
    def seed_groups(self) -> list:
        if self._seed_groups is None:
            self._seed_groups = self._groups.to_seed_groups()
        return self._seed_groups

    @property
    def clustering(self) -> Clustering:
        if self._clustering is None:
            lab = self._gather_labels() if self._gather_labels else self.labels_device
            self._clustering = Clustering(centers=self._centers(), assignment=lab.cpu().numpy(),
                                          radii=self.radii_device.cpu().numpy(), objective=self.objective,
                                          sizes=self.sizes_device.cpu().numpy())
        return self._clustering


# ---------------------------------------------------------------------------

class _Comm:
    """torch.distributed plumbing with byte accounting per message kind."""

    def __init__(self):
        self.on = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
        self.G = dist.get_world_size() if self.on else 1
        self.rank = dist.get_rank() if self.on else 0
        self.bytes = {}

    def count(self, kind, nbytes):
        if self.on:
            self.bytes[kind] = self.bytes.get(kind, 0) + int(nbytes)

    def all_reduce(self, t, op, kind):
        if self.on:
            self.count(kind, t.numel() * t.element_size())
            dist.all_reduce(t, op=op)
        return t

    def all_gather_var(self, t: torch.Tensor, kind) -> torch.Tensor:
        """Concatenate 1-D tensors of varying length in rank order."""
        if not self.on:
            return t
        n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        ns = [torch.zeros_like(n) for _ in range(self.G)]
        dist.all_gather(ns, n)
        sizes = [int(x.item()) for x in ns]
        mx = max(sizes) if sizes else 0
        buf = torch.zeros(max(1, mx), dtype=t.dtype, device=t.device)
        buf[: t.numel()] = t
        outs = [torch.empty_like(buf) for _ in range(self.G)]
        self.count(kind, t.numel() * t.element_size() * (self.G - 1))
        dist.all_gather(outs, buf)
        return torch.cat([o[:s] for o, s in zip(outs, sizes)])


class _Timer:
    def __init__(self):
        self.t = {}
        self._ev = []

    def stage(self, name):
        timer = self

        class _S:
            def __enter__(self_):
                self_.a = torch.cuda.Event(enable_timing=True)
                self_.b = torch.cuda.Event(enable_timing=True)
                self_.a.record()

            def __exit__(self_, *exc):
                self_.b.record()
                timer._ev.append((name, self_.a, self_.b))

        return _S()

    def finish(self):
        torch.cuda.synchronize()
        for name, a, b in self._ev:
            self.t[name] = self.t.get(name, 0.0) + a.elapsed_time(b) / 1000.0
        self._ev = []
        return self.t


_SYMM = {}
_SYMM_DECISION = {}
_FUSED_COUNTS = bool(os.environ.get('GEEK_FUSED_COUNTS'))


def _symm_ready(comm: _Comm, rows: int, cols: int, device) -> bool:
    """Decide TOGETHER whether the peer-mapped key buffers can be used.

    Every rank checks locally (symmetric-memory module, all ranks on this
    node, GEEK_NO_ROUTED unset) and the flags are MIN-reduced; only if all
    ranks agree does the (collective) rendezvous run, and its outcome is
    MIN-reduced again.  So either every rank takes the routed projection or
    every rank takes the all_to_all path -- no rank can fall back alone after
    a barrier.  The decision is cached per shape, identically on every rank."""
    key = (comm.G, rows, cols, device.index)
    if key in _SYMM_DECISION:
        return _SYMM_DECISION[key]
    ok = not os.environ.get("GEEK_NO_ROUTED")
    try:
        import torch.distributed._symmetric_memory  # noqa: F401
        ok = ok and int(os.environ.get("LOCAL_WORLD_SIZE", comm.G)) == comm.G
    except Exception:
        ok = False
    flag = torch.tensor([int(ok)], dtype=torch.int32, device=device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    ok = bool(flag.item())
    if ok:
        try:
            _symm_keys(comm, rows, cols, device)
        except Exception:
            ok = False
        flag.fill_(int(ok))
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        ok = bool(flag.item())
    _SYMM_DECISION[key] = ok
    return ok


def _symm_keys(comm: _Comm, rows: int, cols: int, device):
    """Symmetric-memory int64 [rows, cols] buffer mapped on every rank (cached
    per shape; one live at a time)."""
    key = (comm.G, rows, cols, device.index)
    ent = _SYMM.get(key)
    if ent is None:
        import torch.distributed._symmetric_memory as symm
        group = dist.group.WORLD
        try:
            symm.enable_symm_mem_for_group(group.group_name)
        except Exception:  # already enabled / not needed on this torch
            pass
        _SYMM.clear()
        buf = symm.empty((rows, cols), dtype=torch.int64, device=device)
        handle = symm.rendezvous(buf, group)
        ent = (buf, handle)
        _SYMM[key] = ent
    return ent


def _routable(X: torch.Tensor, m: int, G: int) -> bool:
    return (X.is_cuda and X.dtype == torch.float32 and X.shape[1] % 4 == 0 and 4 <= X.shape[1] <= 128
            and 1 <= m <= 48 and G <= 8)


def project_routed(X_local: torch.Tensor, A: np.ndarray, n: int, row_lo: int, comm: _Comm,
                   exprange: torch.Tensor) -> torch.Tensor:
    """Projection with the bucket synchronisation fused in (engine.py:199-238):
    every rank stores the key of table j for its rows straight into owner
    j % G's symmetric buffer over NVLink (geek_project_keys_routed), so no
    all-to-all follows.  Returns this rank's [m_own, n] keys."""
    m, G = A.shape[0], comm.G
    n_local, d = X_local.shape
    buf, handle = _symm_keys(comm, -(-m // G), n, X_local.device)
    ptrs = np.array([int(p) for p in handle.buffer_ptrs], dtype=np.uint64)
    Ad = directions_device(A)
    handle.barrier()  # every owner is done with the previous job's keys
    _lib.call("geek_project_keys_routed", _lib.ptr(X_local), _lib.dtype_code(X_local), n_local, d, _lib.ptr(Ad),
              m, _lib.hptr(ptrs), G, n, row_lo, _lib.ptr(exprange), None, 0, None, _lib.stream())
    handle.barrier()  # all keys of this rank's tables have landed
    comm.count("BucketShard", n_local * m * 8 * (G - 1) // G)
    own = len([j for j in range(m) if j % G == comm.rank])
    return buf[:own]


def project_counted(X_local: torch.Tensor, A: np.ndarray, n: int, row_lo: int, comm: _Comm,
                    exprange: torch.Tensor, own):
    """Projection with the rank split's fine-bin histogram fused in.  The
    coarse cell histogram comes from the split's own sample rows (0, stride,
    2*stride, ... of the job: each rank projects the sample rows it holds,
    the histograms are summed), so every rank derives the same fine-bin
    layout (geek_fine_layout); the projection then counts every key into its
    fine bin as it stores it (G > 1: into the owner's symmetric buffer), the
    counts are summed over ranks, and the owners split their tables with
    geek_rank_split_counted -- no second pass over the keys for the histogram.
    Returns (keys_own [m_own, n], (hist_own, fcnt_own))."""
    m, G = A.shape[0], comm.G
    n_local, d = X_local.shape
    dev = X_local.device
    cb, stride = np.zeros(1, dtype=np.int32), np.zeros(1, dtype=np.uint64)
    _lib.call("geek_split_plan", n, _lib.hptr(cb), _lib.hptr(stride))
    cb, stride = int(cb[0]), int(stride[0])
    nc = 1 << cb
    first = -(-row_lo // stride) * stride
    idx = torch.arange(first, row_lo + n_local, stride, device=dev) - row_lo
    hist = torch.zeros(m * nc, dtype=torch.int32, device=dev)
    if idx.numel():
        ks = project_keys(X_local.index_select(0, idx).contiguous(), A)
        _lib.call("geek_coarse_hist", _lib.ptr(ks), ks.shape[1], m, cb, _lib.ptr(hist), _lib.stream())
        del ks
    comm.all_reduce(hist, dist.ReduceOp.SUM, "BucketShard")
    cinfo = _lib.empty(m * nc * 2, torch.int32)
    toff = _lib.empty(m + 1, torch.int32)
    nfb = np.zeros(1, dtype=np.uint64)
    _lib.call("geek_fine_layout", _lib.ptr(hist), m, n, _lib.ptr(cinfo), _lib.ptr(toff), _lib.hptr(nfb),
              _lib.stream())
    fcnt = torch.zeros(max(1, int(nfb[0])), dtype=torch.int32, device=dev)
    Ad = directions_device(A)
    if G > 1:
        buf, handle = _symm_keys(comm, -(-m // G), n, dev)
        ptrs = np.array([int(p) for p in handle.buffer_ptrs], dtype=np.uint64)
        handle.barrier()  # every owner is done with the previous job's keys
        _lib.call("geek_project_keys_routed", _lib.ptr(X_local), 0, n_local, d, _lib.ptr(Ad), m, _lib.hptr(ptrs),
                  G, n, row_lo, _lib.ptr(exprange), _lib.ptr(cinfo), cb, _lib.ptr(fcnt), _lib.stream())
        handle.barrier()  # all keys of this rank's tables have landed
        comm.count("BucketShard", n_local * m * 8 * (G - 1) // G)
        keys_own = buf[:len(own)]
        comm.all_reduce(fcnt, dist.ReduceOp.SUM, "BucketShard")
    else:
        keys = _lib.empty(max(1, m * n), torch.int64)
        ptrs = np.array([keys.data_ptr()], dtype=np.uint64)
        _lib.call("geek_project_keys_routed", _lib.ptr(X_local), 0, n_local, d, _lib.ptr(Ad), m, _lib.hptr(ptrs),
                  1, n, 0, _lib.ptr(exprange), _lib.ptr(cinfo), cb, _lib.ptr(fcnt), _lib.stream())
        keys_own = keys[: m * n].view(m, n)
    if len(own) == m:
        return keys_own, (hist, fcnt)
    toff_h = toff.cpu().numpy().astype(np.int64)
    hist_own = hist.view(m, nc)[torch.tensor(own, dtype=torch.int64, device=dev)].contiguous()
    fcnt_own = torch.cat([fcnt[toff_h[j]:toff_h[j + 1]] for j in own]) if own else fcnt[:0]
    return keys_own, (hist_own, fcnt_own.contiguous())


def rank_split_counted(keys: torch.Tensor, t: int, hist: torch.Tensor, fcnt: torch.Tensor, stats=None):
    m, n = keys.shape
    codes = _lib.empty(max(1, n * m), _lib.U32)
    st = np.zeros(4, dtype=np.uint64)
    _lib.call("geek_rank_split_counted", _lib.ptr(keys), n, m, t, _lib.ptr(hist), _lib.ptr(fcnt), _lib.ptr(codes),
              _lib.hptr(st), _lib.stream())
    if stats is not None:
        stats.update(fine_bins=int(st[0]), straddling=int(st[1]), max_straddle_bin=int(st[2]),
                     sorted_fallback=int(st[3]))
    return codes[: n * m].view(n, m)


_XBUF = {}
_COPY_STREAM = []


def _stream_host_rows(X_host: torch.Tensor, A: np.ndarray, n: int, row_lo: int, comm: _Comm,
                      exprange: torch.Tensor, own, chunks: int = 8):
    """Host rows (pinned for overlap) -> this GPU, projected chunk by chunk as
    they land: the host-to-device copy of chunk c+1 runs on a copy stream
    while chunk c is projected (keys stored locally, or straight into the
    owners' symmetric buffers when G > 1).  Returns (X_device, keys_own or
    None when the shape takes the unfused path)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    m, G = A.shape[0], comm.G
    n_local, d = X_host.shape
    key = (tuple(X_host.shape), X_host.dtype, dev.index)
    X_dev = _XBUF.get(key)
    if X_dev is None:
        _XBUF.clear()
        X_dev = torch.empty(X_host.shape, dtype=X_host.dtype, device=dev)
        _XBUF[key] = X_dev
    fused = (X_host.dtype == torch.float32 and d % 4 == 0 and 4 <= d <= 128 and 1 <= m <= 48 and G <= 8
             and (G == 1 or _symm_ready(comm, -(-m // G), n, dev)))
    main = torch.cuda.current_stream()
    if not fused:
        X_dev.copy_(X_host, non_blocking=True)
        return X_dev, None
    if not _COPY_STREAM:
        _COPY_STREAM.append(torch.cuda.Stream())
    cs = _COPY_STREAM[0]
    cs.wait_stream(main)  # the previous job's kernels are done with X_dev
    step = -(-(-(-n_local // chunks)) // 128) * 128
    spans = [(a, min(n_local, a + step)) for a in range(0, n_local, step)]
    events = []
    with torch.cuda.stream(cs):
        for a, b in spans:
            X_dev[a:b].copy_(X_host[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
            events.append(ev)
    Ad = directions_device(A)
    if G > 1:
        buf, handle = _symm_keys(comm, -(-m // G), n, dev)
        ptrs = np.array([int(p) for p in handle.buffer_ptrs], dtype=np.uint64)
        handle.barrier()  # every owner is done with the previous job's keys
    else:
        keys = _lib.empty(max(1, m * n), torch.int64)
        ptrs = np.array([keys.data_ptr()], dtype=np.uint64)
    for (a, b), ev in zip(spans, events):
        main.wait_event(ev)
        _lib.call("geek_project_keys_routed", _lib.ptr(X_dev[a:b]), 0, b - a, d, _lib.ptr(Ad), m, _lib.hptr(ptrs),
                  G, n, row_lo + a, _lib.ptr(exprange), None, 0, None, _lib.stream())
    if G > 1:
        handle.barrier()  # all keys of this rank's tables have landed
        comm.count("BucketShard", n_local * m * 8 * (G - 1) // G)
        return X_dev, buf[:len(own)]
    return X_dev, keys[: m * n].view(m, n)


def route_tables(keys: torch.Tensor, n: int, comm: _Comm) -> torch.Tensor:
    """Bucket synchronisation (engine.py:199-238): every rank holds keys
    [m, n_local] of its contiguous shard; table j goes to rank j % G, which
    receives [m_own, n] with the shards concatenated in id order."""
    if not comm.on:
        return keys
    m, G, rank = keys.shape[0], comm.G, comm.rank
    spans = split_data(n, G)
    mine = [[j for j in range(m) if j % G == q] for q in range(G)]
    own = mine[rank]
    send = torch.cat([keys[mine[q]].reshape(-1) for q in range(G)])
    recv_sizes = [len(own) * (hi - lo) for lo, hi in spans]
    recv = torch.empty(sum(recv_sizes), dtype=keys.dtype, device=keys.device)
    dist.all_to_all_single(recv, send, recv_sizes, [len(mine[q]) * keys.shape[1] for q in range(G)])
    comm.count("BucketShard", (send.numel() - len(own) * keys.shape[1]) * keys.element_size())
    parts = torch.split(recv, recv_sizes)
    return torch.cat([pt.view(len(own), hi - lo) for pt, (lo, hi) in zip(parts, spans)], dim=1).contiguous()


def _pw_leaf(vals) -> float:
    """numpy's pairwise_sum on <= 128 doubles (loops_utils.h: 8 accumulators)."""
    n = len(vals)
    if n < 8:
        res = 0.0
        for v in vals:
            res += v
        return res
    r = list(vals[:8])
    i = 8
    while i < n - n % 8:
        for j in range(8):
            r[j] += vals[i + j]
        i += 8
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < n:
        res += vals[i]
        i += 1
    return res


def sharded_pairwise_sum(best: torch.Tensor, n: int, row_lo: int, comm: _Comm) -> float:
    """numpy's pairwise sum of the n-element array whose rows [row_lo, row_lo +
    len(best)) this rank holds, without gathering it: every rank sums the
    maximal subtrees of numpy's recursion (n2 = n/2 rounded down to a multiple
    of 8) that lie inside its rows on the device, ships those values plus the
    elements of leaf blocks that cross a shard boundary, and the top of the
    tree is evaluated identically on every rank."""
    lo, hi = row_lo, row_lo + best.numel()
    nodes, elems = [], []

    def walk(a, m):
        if a >= hi or a + m <= lo or m == 0:
            return
        if lo <= a and a + m <= hi:
            nodes.append((a, m))
            return
        if m <= 128:  # a leaf block crossing a shard boundary: ship its elements
            elems.append((max(a, lo), min(a + m, hi)))
            return
        m2 = m // 2
        m2 -= m2 % 8
        walk(a, m2)
        walk(a + m2, m - m2)

    walk(0, n)
    vals = [pairwise_sum(best[a - lo:a - lo + m]) for a, m in nodes]
    node_t = torch.tensor([[a, m] for a, m in nodes], dtype=torch.int64).reshape(-1, 2)
    node_v = torch.cat(vals) if vals else torch.zeros(0, dtype=torch.float64, device=best.device)
    el_idx = [i for a, b in elems for i in range(a, b)]
    el_v = best[torch.tensor([i - lo for i in el_idx], dtype=torch.int64, device=best.device)] if el_idx else \
        torch.zeros(0, dtype=torch.float64, device=best.device)
    # ship (start, len, value) of the nodes and (index, value) of the elements
    packed = torch.cat([node_t.to(best.device).view(torch.float64).reshape(-1), node_v,
                        torch.tensor(el_idx, dtype=torch.int64, device=best.device).view(torch.float64), el_v])
    header = torch.tensor([len(nodes), len(el_idx)], dtype=torch.int64, device=best.device).view(torch.float64)
    allv = comm.all_gather_var(torch.cat([header, packed]), "Assignments").cpu()
    known, points = {}, {}
    pos = 0
    while pos < allv.numel():
        nn, ne = allv[pos:pos + 2].view(torch.int64).tolist()
        pos += 2
        nt = allv[pos:pos + 2 * nn].view(torch.int64).view(-1, 2).tolist()
        pos += 2 * nn
        nv = allv[pos:pos + nn].tolist()
        pos += nn
        ei = allv[pos:pos + ne].view(torch.int64).tolist()
        pos += ne
        ev = allv[pos:pos + ne].tolist()
        pos += ne
        for (a, m), v in zip(nt, nv):
            known[(a, m)] = v
        points.update(zip(ei, ev))

    def evaluate(a, m):
        if (a, m) in known:
            return known[(a, m)]
        if m <= 128:
            return _pw_leaf([points[i] for i in range(a, a + m)])
        m2 = m // 2
        m2 -= m2 % 8
        return evaluate(a, m2) + evaluate(a + m2, m - m2)

    return evaluate(0, n)


def _merge_groups(comm: _Comm, local: GroupSet) -> GroupSet:
    if not comm.on:
        return local
    sizes = comm.all_gather_var(local.sizes(), "SeedGroups")
    flat = comm.all_gather_var(local.flat[: int(local.off[-1].item())], "SeedGroups")
    off = torch.zeros(sizes.numel() + 1, dtype=torch.int64, device=sizes.device)
    torch.cumsum(sizes, 0, out=off[1:])
    return GroupSet(flat.contiguous() if flat.numel() else _lib.zeros(1, torch.int32), off)


def _fallback_groups(n, g, seed, warnings):
    warnings.append("seeding produced no groups; falling back to one random seed per worker")
    rng = np.random.default_rng(seed)
    picks = sorted(int(rng.integers(lo, hi)) for lo, hi in split_data(n, g))
    return GroupSet.from_host([np.array([p]) for p in picks])


class _Logical:
    """Transport accounting of the reference's g in-process workers
    (engine.py:79-104 Transport, serialize.py message bodies) when the g
    logical workers share one process: the bytes each message kind would
    carry, so `transport_bytes` reads as the reference's at G = 1."""

    def __init__(self, n: int, g: int, m: int):
        self.n, self.g, self.m = n, g, m
        self.spans = split_data(n, g)
        self.bytes = {}
        self._dev = None

    def add(self, kind, nbytes):
        if self.g > 1:
            self.bytes[kind] = self.bytes.get(kind, 0) + int(nbytes)

    def fragments(self, per_row: int, head: int):
        """BucketShard (engine.py:198-207): worker w sends table j to owner
        j % g != w; pack_fragment = 17 bytes + pack_array(body)."""
        for w, (lo, hi) in enumerate(self.spans):
            own = len(range(w, self.m, self.g))
            self.add("BucketShard", (self.m - own) * (17 + head + per_row * (hi - lo)))

    def seed_groups(self, groups: GroupSet):
        """SeedGroups (engine.py:285-287): every worker broadcasts its local
        groups (8 + per group pack_array(int64 members) = 18 + 8 len)."""
        total = int(groups.off[-1].item()) if groups.count else 0
        self.add("SeedGroups", (self.g - 1) * (8 * self.g + 18 * groups.count + 8 * total))

    def center_stats(self, k: int, per_group_fixed: int, value_bytes: int = 0):
        """LocalCenters (engine.py:486-490): every worker broadcasts 8 + per
        group (qB + body) bytes; value_bytes = the exact sums' pack_bigints
        bytes summed over workers (dense) or 0 (fixed-size count arrays)."""
        self.add("LocalCenters", (self.g - 1) * (self.g * (8 + per_group_fixed * k) + value_bytes))

    def device_counter(self):
        if self._dev is None:
            self._dev = _lib.zeros(1, torch.int64)
        return self._dev

    def flush_device(self, kind):
        if self._dev is not None and self.g > 1:
            self.add(kind, (self.g - 1) * int(self._dev.item()))
            self._dev.zero_()


def _check_budget(config: PipelineConfig, n: int):
    """engine.py:359-366 (_chunk_tables): a table's member lists take 8 n
    bytes; a budget below one table is an error of worker 0's seeding stage
    (worker 0 always owns table 0).  Larger budgets only change the
    reference's load chunking, never the result (engine.py:244-248)."""
    budget = config.workers.memory_budget
    if 8 * n > budget:
        raise EngineError(f"stage seeding, worker 0: memory budget {budget} below single table of {8 * n} bytes")


def _worker_digits(X_local, groups, emin, nd, logical, nonfinite, labels=None, k=None, keep=None):
    """Exact digit sums as the reference's workers form them (one partial per
    logical worker, engine.py:299-311 / 481-516), summed; each worker's
    pack_bigints bytes are accumulated for the LocalCenters accounting."""
    if logical is None or logical.g == 1:
        if labels is None:
            return partial_sums(X_local, groups, emin, nd, 0, nonfinite=nonfinite)
        return label_sums(X_local, labels, k, emin, nd)
    ctr = logical.device_counter()
    total = None
    for lo, hi in logical.spans:
        if labels is None:
            part = partial_sums(X_local[lo:hi], groups, emin, nd, lo, nonfinite=nonfinite)
        else:
            part = label_sums(X_local[lo:hi], labels[lo:hi], k, emin, nd)
        center_stats_bytes(part if keep is None else part[keep].contiguous(), emin, ctr)
        total = part if total is None else total.add_(part)
    return total


def _dense_pipeline(X_local: torch.Tensor, n: int, row_lo: int, config: PipelineConfig, comm: _Comm,
                    diagnostics: bool = False):
    g = config.workers.num_workers
    p: HomoTransformParams = config.homo
    sp: SeedingParams = config.seeding
    m, t, G, rank = p.num_tables, p.buckets_per_table, comm.G, comm.rank
    d = X_local.shape[1]
    if t > n:
        raise EngineError(f"stage setup: cannot split {n} objects into {t} buckets")
    if g % G:
        raise EngineError(f"stage setup: {G} GPUs must divide the {g} logical workers")
    info, warnings = {}, []
    tm = _Timer()
    A = p.direction_matrix(d)
    own = [j for j in range(m) if j % G == rank]
    logical = None if comm.on else _Logical(n, g, m)
    if logical:
        logical.fragments(8, 18)  # float64 projection fragments (pack_array 1-D f8)
    keys_own, counted = None, None
    with tm.stage("transform"):
        exprange = torch.tensor([1 << 30, -(1 << 30)], dtype=torch.int32,
                                device=torch.device("cuda", torch.cuda.current_device()))
        if not X_local.is_cuda:  # host rows: copied in chunks, each projected as it lands
            X_local, keys_own = _stream_host_rows(X_local, A, n, row_lo, comm, exprange, own)
        if (keys_own is None and _routable(X_local, m, G) and (comm.on or _FUSED_COUNTS)
                and (not comm.on or _symm_ready(comm, -(-m // G), n, X_local.device))):
            if _FUSED_COUNTS:  # measured slower on B200 (the counts stall the DMMA warps); kept opt-in
                keys_own, counted = project_counted(X_local, A, n, row_lo, comm, exprange, own)
            else:
                keys_own = project_routed(X_local, A, n, row_lo, comm, exprange)
        if keys_own is None:
            keys = project_keys(X_local, A, exprange)  # [m, n_local]; exponent window fused
    with tm.stage("sync_buckets"):
        if keys_own is None:
            keys_own = route_tables(keys, n, comm)
            del keys
        stats = {}
        if not own:
            codes = None
        elif counted is not None:
            codes = rank_split_counted(keys_own, t, counted[0], counted[1], stats)
        else:
            codes = rank_split_codes(keys_own.contiguous(), t, stats)
        info["rank_split"] = stats
    if diagnostics:  # boundary exceptions of the split (north_star tie tolerance)
        with tm.stage("diagnostics"):
            xe = exprange[1:2].to(torch.int64)
            if comm.on:  # not a reference message kind: kept out of transport_bytes
                dist.all_reduce(xe, op=dist.ReduceOp.MAX)
            if own:
                tol = projection_tolerance(A[own], int(xe.item()))
                info["split_boundary"] = split_boundary_stats(keys_own, codes, t, tol, tables=own)
    del keys_own, counted
    _check_budget(config, n)
    with tm.stage("seeding"):
        if own:
            bt = BucketTable(codes, n, [t] * len(own), "rank", even=True)
            owner = _lib.to_dev((np.repeat(np.array(own), t) % g).astype(np.int32))
            local, _, _ = silk_votes(bt, sp, n, owner, info)
        else:
            local = GroupSet.empty()
        merged = _merge_groups(comm, local)
        if logical:
            logical.seed_groups(merged)
        groups = dedup_device(merged, sp, n)
        if groups.count == 0:
            groups = _fallback_groups(n, g, config.fallback_seed, warnings)
    nonfinite = _lib.zeros(1, torch.int32)
    with tm.stage("centers"):
        r = torch.stack([-exprange[0], exprange[1]]).to(torch.int64)
        comm.all_reduce(r, dist.ReduceOp.MAX, "LocalCenters")
        emin, emax = -int(r[0].item()), int(r[1].item())
        nd = digit_count(emin, emax)
        if logical:
            digits = _worker_digits(X_local, groups, emin, nd, logical, nonfinite)
            logical.center_stats(groups.count, 25)
            logical.flush_device("LocalCenters")
        else:
            digits = partial_sums(X_local, groups, emin, nd, row_lo, nonfinite=nonfinite)
        comm.all_reduce(digits, dist.ReduceOp.SUM, "LocalCenters")
        C = round_means(digits, groups.sizes(), emin, nd)
    with tm.stage("assign"):
        astats = AssignStats()
        labels, best = assign_l2_device(X_local, C, astats)
        info["centers"] = int(groups.count)
    weights = groups.sizes()

    def reduce_assignment(labels, best, k):
        radii, sizes = radii_sizes(labels, best, k)
        comm.all_reduce(radii.view(torch.int64), dist.ReduceOp.MAX, "Assignments")
        comm.all_reduce(sizes, dist.ReduceOp.SUM, "Assignments")
        if comm.on:
            obj = torch.tensor([sharded_pairwise_sum(best, n, row_lo, comm)], dtype=torch.float64)
        else:
            obj = pairwise_sum(best)
        return radii, sizes, obj

    with tm.stage("assign"):
        radii, sizes, obj = reduce_assignment(labels, best, groups.count)
    for _ in range(config.passes):  # _refine_distributed (engine.py:519-537)
        with tm.stage("centers"):
            keep = torch.nonzero(sizes > 0).flatten()  # empty clusters are dropped
            if logical:
                digits = _worker_digits(X_local, None, emin, nd, logical, None, labels=labels, k=C.shape[0],
                                        keep=keep)
                logical.center_stats(keep.numel(), 25)
                logical.flush_device("LocalCenters")
            else:
                digits = label_sums(X_local, labels, C.shape[0], emin, nd)
            comm.all_reduce(digits, dist.ReduceOp.SUM, "LocalCenters")
            weights = sizes[keep].contiguous()
            C = round_means(digits[keep].contiguous(), weights, emin, nd)
        with tm.stage("assign"):
            labels, best = assign_l2_device(X_local, C)
            radii, sizes, obj = reduce_assignment(labels, best, C.shape[0])
    timings = tm.finish()
    info.update(astats.read())  # device counters + screen events of the first assignment
    if comm.on:
        dist.all_reduce(nonfinite, op=dist.ReduceOp.MAX)
    if int(nonfinite.item()):  # numeric.py:24-25 (exact_column_sums)
        raise InvalidInput("non-finite value in exact sum")
    sizes_h = weights.cpu().numpy()

    def centers():
        Ch = C.cpu().numpy()
        return [CentralVector("centroid", Ch[i], int(sizes_h[i])) for i in range(Ch.shape[0])]

    gather = (lambda: comm.all_gather_var(labels, "Assignments")) if comm.on else None
    return PipelineResult(centers, groups, labels, best, radii, sizes, float(obj.item()), timings,
                          dict(comm.bytes) if comm.on else dict(logical.bytes), warnings, info, gather)


def route_signature_rows(sig: torch.Tensor, n: int, K: int, comm: _Comm) -> torch.Tensor:
    """Bucket synchronisation for signature tables (engine.py:186-207, 227-238):
    rank r holds the [n_local, m*K] signatures of its contiguous rows; table j
    goes to rank j % G, which receives [m_own, n, K] with the shards in id order."""
    n_local, mK = sig.shape
    m, G, rank = mK // K, comm.G, comm.rank
    spans = split_data(n, G)
    mine = [[j for j in range(m) if j % G == q] for q in range(G)]
    own = mine[rank]
    r3 = sig.view(n_local, m, K)
    send = torch.cat([r3[:, mine[q], :].permute(1, 0, 2).reshape(-1) for q in range(G)])
    send_sizes = [len(mine[q]) * n_local * K for q in range(G)]
    recv_sizes = [len(own) * (hi - lo) * K for lo, hi in spans]
    recv = torch.empty(sum(recv_sizes), dtype=sig.dtype, device=sig.device)
    dist.all_to_all_single(recv, send, recv_sizes, send_sizes)
    comm.count("BucketShard", (send.numel() - len(own) * n_local * K) * sig.element_size())
    parts = torch.split(recv, recv_sizes)
    return torch.cat([pt.view(len(own), hi - lo, K) for pt, (lo, hi) in zip(parts, spans)], dim=1).contiguous()


def _dist_modes(keys: list, k: int, cs: int, comm: _Comm) -> torch.Tensor:
    """Per-attribute modes over a code space too large for dense counts, with the
    rows spread over ranks: keys[c] holds group * cs + code of this rank's rows;
    (key, count) runs are routed to the rank owning the group (group % G), summed
    there, each owned group keeps its most frequent code (the smallest among
    equal counts, seeding.py:180-185), and a MIN all-reduce assembles [k, d]."""
    G = comm.G
    dev = keys[0].device if keys else torch.device("cuda", torch.cuda.current_device())
    out = torch.empty((k, len(keys)), dtype=torch.int32, device=dev)
    for c, key in enumerate(keys):
        uk, cnt = torch.unique(key, sorted=True, return_counts=True)
        owner = (uk // cs) % G
        order = torch.sort(owner, stable=True).indices
        uk, cnt = uk[order].contiguous(), cnt[order].contiguous()
        send_n = torch.bincount(owner, minlength=G)
        recv_n = torch.empty_like(send_n)
        dist.all_to_all_single(recv_n, send_n)
        ss, rs = send_n.tolist(), recv_n.tolist()
        rk = torch.empty(sum(rs), dtype=uk.dtype, device=dev)
        rc = torch.empty(sum(rs), dtype=cnt.dtype, device=dev)
        dist.all_to_all_single(rk, uk, rs, ss)
        dist.all_to_all_single(rc, cnt, rs, ss)
        comm.count("LocalCenters", (uk.numel() + cnt.numel()) * 8)
        best = torch.full((k,), cs, dtype=torch.int64, device=dev)
        if rk.numel():
            u2, inv = torch.unique(rk, sorted=True, return_inverse=True)
            c2 = torch.zeros(u2.numel(), dtype=rc.dtype, device=dev).scatter_add_(0, inv, rc)
            g = u2 // cs
            top = torch.zeros(k, dtype=c2.dtype, device=dev).scatter_reduce(0, g, c2, "amax", include_self=False)
            win = c2 == top[g]
            best = best.scatter_reduce(0, g[win], (u2 - g * cs)[win], "amin", include_self=True)
        dist.all_reduce(best, op=dist.ReduceOp.MIN)
        out[:, c] = best.to(torch.int32)
    return out


def _signature_pipeline_sharded(data, config: PipelineConfig, comm: _Comm):
    """mixed / sparse data over G ranks (engine.py:173-238 signature fragments,
    :379-392 dataset-wide preprocessing).  Every rank holds the full input (the
    reference's run_pipeline contract); the dataset-wide step (numeric
    discretisation) runs identically on every rank, then each rank hashes its
    contiguous rows (DOPH is per set), the signature rows of table j go to rank
    j % G, which groups them into buckets and votes; seed groups are
    all-gathered and deduplicated identically; mode / membership counts are
    summed over ranks (exact); assignment is local; radii MAX, sizes SUM, the
    objective is numpy's pairwise sum over all ranks' rows."""
    g = config.workers.num_workers
    mp: MinhashTransformParams = config.minhash
    sp: SeedingParams = config.seeding
    G, rank = comm.G, comm.rank
    if g % G:
        raise EngineError(f"stage setup: {G} GPUs must divide the {g} logical workers")
    info, warnings = {}, []
    tm = _Timer()
    with tm.stage("prepare"):
        if config.transform_kind == "mixed":
            if isinstance(data, (MixedData, DenseData)):
                data = discretize_numeric(data, mp.bins_per_attribute)
            if not isinstance(data, CategoricalData):
                raise EngineError("stage setup: mixed transform expects mixed or categorical data")
            n = data.n
            if g > n:
                raise EngineError(f"stage setup: cannot split {n} objects across {g} workers")
            lo, hi = split_data(n, G)[rank]
            cat = CategoricalData.from_device(data.device_codes()[lo:hi], code_space=data.code_space)
            flat, off = categorical_token_csr(cat)
            universe = data.dim * data.code_space
        else:
            if not isinstance(data, SparseData):
                raise EngineError("stage setup: sparse transform expects sparse data")
            n = data.n
            if g > n:
                raise EngineError(f"stage setup: cannot split {n} objects across {g} workers")
            lo, hi = split_data(n, G)[rank]
            full_flat, full_off = data.csr()
            off_l = (full_off[lo:hi + 1] - full_off[lo]).contiguous()
            flat_l = full_flat[int(full_off[lo].item()):int(full_off[hi].item())].contiguous()
            universe = data.universe
            if mp.target_dims <= data.universe:
                red = DophReducer(derive_seed(mp.seed, 0xD0), data.universe, mp.target_dims)
                flat_l, off_l = red.reduce_device(flat_l, off_l, hi - lo)
                universe = mp.target_dims
            cat = SparseData.from_csr(flat_l.to(torch.int64) & 0xFFFFFFFF, off_l, universe)
            flat, off = cat.csr()
    n_local = hi - lo
    own = [j for j in range(mp.num_tables) if j % G == rank]
    _check_budget(config, n)
    with tm.stage("transform"):
        sig = signature_rows(mp.scheme(universe), flat, off, n_local)
    with tm.stage("sync_buckets"):
        sig_own = route_signature_rows(sig, n, mp.num_hashes, comm)  # [m_own, n, K]
        del sig
        if own:
            sig_own = sig_own.permute(1, 0, 2).reshape(n, len(own) * mp.num_hashes).contiguous()
            codes, tsizes = group_signature_tables(sig_own, mp.num_hashes, universe)
        del sig_own
    with tm.stage("seeding"):
        if own:
            bt = BucketTable(codes, n, tsizes, "sig", even=False)
            owner = _lib.to_dev(np.concatenate([np.full(ts, j % g, dtype=np.int32) for j, ts in zip(own, tsizes)]))
            local, _, _ = silk_votes(bt, sp, n, owner, info)
        else:
            local = GroupSet.empty()
        merged = _merge_groups(comm, local)
        groups = dedup_device(merged, sp, n)
        if groups.count == 0:
            groups = _fallback_groups(n, g, config.fallback_seed, warnings)
    categorical = isinstance(cat, CategoricalData)
    cs = cat.code_space if categorical else 0

    def modes_of(keys_fn, k, counts_fn):
        if k * cat.dim * cs <= (1 << 31):
            cnt = counts_fn()
            comm.all_reduce(cnt, dist.ReduceOp.SUM, "LocalCenters")
            return torch.argmax(cnt, dim=2).to(torch.int32)
        return _dist_modes(keys_fn(), k, cs, comm)

    with tm.stage("centers"):
        if categorical:
            codes_l = cat.device_codes()

            def group_keys():
                sizes = groups.sizes()
                gidx = torch.repeat_interleave(torch.arange(groups.count, device=sizes.device), sizes)
                ids = groups.flat[: int(groups.off[-1].item())].to(torch.int64) & 0xFFFFFFFF
                sel = (ids >= lo) & (ids < hi)
                gi, li = gidx[sel], ids[sel] - lo
                return [gi * cs + codes_l[li, c].to(torch.int64) for c in range(cat.dim)]

            M = modes_of(group_keys, groups.count, lambda: mode_counts(codes_l, cs, groups, lo))
        else:
            cnt = sparse_counts(cat, groups, lo, (flat, off))
            comm.all_reduce(cnt, dist.ReduceOp.SUM, "LocalCenters")
            M = (2 * cnt > groups.sizes()[:, None]).to(torch.int32)

    def assign_reduce(M):
        if categorical:
            labels, best = assign_cat_device(codes_l, M)
        else:
            labels, best = assign_sparse_device(flat, off, n_local, universe, M)
        radii, sizes = radii_sizes(labels, best, M.shape[0])
        comm.all_reduce(radii.view(torch.int64), dist.ReduceOp.MAX, "Assignments")
        comm.all_reduce(sizes, dist.ReduceOp.SUM, "Assignments")
        obj = sharded_pairwise_sum(best, n, lo, comm)
        return labels, best, radii, sizes, obj

    with tm.stage("assign"):
        labels, best, radii, sizes, obj = assign_reduce(M)
    weights = groups.sizes()
    for _ in range(config.passes):  # _refine_distributed (engine.py:519-537)
        with tm.stage("centers"):
            keep = torch.nonzero(sizes > 0).flatten()
            weights = sizes[keep].contiguous()
            k = M.shape[0]
            if categorical:
                def label_keys():
                    pos = torch.full((k,), -1, dtype=torch.int64, device=keep.device)
                    pos[keep] = torch.arange(keep.numel(), device=keep.device)
                    lp = pos[labels]
                    return [lp * cs + codes_l[:, c].to(torch.int64) for c in range(cat.dim)]

                if k * cat.dim * cs <= (1 << 31):
                    cnt = label_mode_counts(codes_l, cs, labels, k)
                    comm.all_reduce(cnt, dist.ReduceOp.SUM, "LocalCenters")
                    M = torch.argmax(cnt[keep], dim=2).to(torch.int32)
                else:
                    M = _dist_modes(label_keys(), keep.numel(), cs, comm)
            else:
                cnt = label_sparse_counts(flat, off, n_local, universe, labels, k)
                comm.all_reduce(cnt, dist.ReduceOp.SUM, "LocalCenters")
                M = (2 * cnt[keep] > weights[:, None]).to(torch.int32)
        with tm.stage("assign"):
            labels, best, radii, sizes, obj = assign_reduce(M)
    timings = tm.finish()
    sizes_h = weights.cpu().numpy()

    def centers():
        Mh = M.cpu().numpy()
        return [CentralVector("mode", Mh[i], int(sizes_h[i])) for i in range(Mh.shape[0])]

    gather = lambda: comm.all_gather_var(labels, "Assignments")  # noqa: E731
    return PipelineResult(centers, groups, labels, best, radii, sizes, obj, timings, dict(comm.bytes), warnings,
                          info, gather)


def _signature_pipeline(data, config: PipelineConfig, comm: _Comm):
    """mixed / sparse data on one device (logical g emulated)."""
    if comm.on:
        return _signature_pipeline_sharded(data, config, comm)
    g = config.workers.num_workers
    mp: MinhashTransformParams = config.minhash
    sp: SeedingParams = config.seeding
    info, warnings = {}, []
    tm = _Timer()
    with tm.stage("prepare"):
        if config.transform_kind == "mixed":
            if isinstance(data, (MixedData, DenseData)):
                data = discretize_numeric(data, mp.bins_per_attribute)
            if not isinstance(data, CategoricalData):
                raise EngineError("stage setup: mixed transform expects mixed or categorical data")
            flat, off = categorical_token_csr(data)
            universe = data.dim * data.code_space
        else:
            if not isinstance(data, SparseData):
                raise EngineError("stage setup: sparse transform expects sparse data")
            if mp.target_dims <= data.universe:
                red = DophReducer(derive_seed(mp.seed, 0xD0), data.universe, mp.target_dims)
                flat, off = red.reduce_device(*data.csr(), data.n)
                data = SparseData.from_csr(flat.to(torch.int64) & 0xFFFFFFFF, off, mp.target_dims)
            flat, off = data.csr()
            universe = data.universe
    n = data.n
    if g > n:
        raise EngineError(f"stage setup: cannot split {n} objects across {g} workers")
    logical = _Logical(n, g, mp.num_tables)
    logical.fragments(8 * mp.num_hashes, 26)  # signature fragments (pack_array 2-D u8)
    with tm.stage("transform"):
        codes, tsizes = signature_bucket_codes(mp.scheme(universe), flat, off, n)
        bt = BucketTable(codes, n, tsizes, "sig", even=False)
    _check_budget(config, n)
    with tm.stage("seeding"):
        owner = _lib.to_dev(np.concatenate([np.full(ts, j % g, dtype=np.int32) for j, ts in enumerate(tsizes)]))
        local, _, _ = silk_votes(bt, sp, n, owner, info)
        logical.seed_groups(local)
        groups = dedup_device(local, sp, n)
        if groups.count == 0:
            groups = _fallback_groups(n, g, config.fallback_seed, warnings)
    # LocalCenters bodies: per group qB + pack_array of the count table
    # (categorical [dim, code_space] int64, sparse [universe] int64)
    stat_fixed = (9 + 26 + 8 * data.dim * data.code_space if isinstance(data, CategoricalData)
                  else 9 + 18 + 8 * data.universe)
    with tm.stage("centers"):
        logical.center_stats(groups.count, stat_fixed)
        if isinstance(data, CategoricalData):
            M = mode_centers(data.device_codes(), data.code_space, groups)
        else:
            cnt = sparse_counts(data, groups)
            M = (2 * cnt > groups.sizes()[:, None]).to(torch.int32)
    with tm.stage("assign"):
        if isinstance(data, CategoricalData):
            labels, best = assign_cat_device(data.device_codes(), M)
        else:
            labels, best = assign_sparse_device(flat, off, n, data.universe, M)
        radii, sizes = radii_sizes(labels, best, groups.count)
        obj = pairwise_sum(best)
    weights = groups.sizes()
    for _ in range(config.passes):  # _refine_distributed (engine.py:519-537) on one device
        with tm.stage("centers"):
            keep = torch.nonzero(sizes > 0).flatten()
            logical.center_stats(keep.numel(), stat_fixed)
            weights = sizes[keep].contiguous()
            if isinstance(data, CategoricalData):
                M = label_mode_centers(data.device_codes(), data.code_space, labels, M.shape[0], keep)
            else:
                cnt = label_sparse_counts(flat, off, n, data.universe, labels, M.shape[0])[keep]
                M = (2 * cnt > weights[:, None]).to(torch.int32)
        with tm.stage("assign"):
            if isinstance(data, CategoricalData):
                labels, best = assign_cat_device(data.device_codes(), M)
            else:
                labels, best = assign_sparse_device(flat, off, n, data.universe, M)
            radii, sizes = radii_sizes(labels, best, M.shape[0])
            obj = pairwise_sum(best)
    timings = tm.finish()
    sizes_h = weights.cpu().numpy()

    def centers():
        Mh = M.cpu().numpy()
        return [CentralVector("mode", Mh[i], int(sizes_h[i])) for i in range(Mh.shape[0])]

    return PipelineResult(centers, groups, labels, best, radii, sizes, float(obj.item()), timings,
                          dict(logical.bytes), warnings, info)


def run_pipeline(data, config: PipelineConfig, *, diagnostics: bool = False) -> PipelineResult:
    """transform -> bucket sync -> seeding -> centers -> assignment (engine.py:395-472).

    Under an initialised torch.distributed group of G ranks every rank calls
    this with the full dataset (or use run_pipeline_shard with its own rows)."""
    if config.passes < 0:
        raise EngineError("stage setup: passes must be >= 0")
    comm = _Comm()
    if config.transform_kind == "dense":
        if not isinstance(data, DenseData):
            raise EngineError("stage setup: dense transform expects dense data")
        n = data.n
        if config.workers.num_workers > n:
            raise EngineError(f"stage setup: cannot split {n} objects across {config.workers.num_workers} workers")
        lo, hi = split_data(n, comm.G)[comm.rank] if comm.on else (0, n)
        X = data.device_vectors()[lo:hi].contiguous() if comm.on else data.device_vectors()
        return _dense_pipeline(X, n, lo, config, comm, diagnostics)
    if config.transform_kind in ("mixed", "sparse"):
        return _signature_pipeline(data, config, comm)
    raise EngineError(f"stage setup: unknown transform kind {config.transform_kind!r}")


def run_pipeline_shard(X_local: torch.Tensor, n: int, config: PipelineConfig, *,
                       diagnostics: bool = False) -> PipelineResult:
    """Dense pipeline where each rank holds its contiguous shard (rows
    split_data(n, G)[rank]), on its GPU or in (pinned) host memory -- host
    rows are streamed to the GPU in chunks that are projected as they land."""
    comm = _Comm()
    lo, hi = split_data(n, comm.G)[comm.rank]
    if X_local.shape[0] != hi - lo:
        raise EngineError(f"stage setup: rank {comm.rank} holds {X_local.shape[0]} rows, expected {hi - lo}")
    return _dense_pipeline(X_local, n, lo, config, comm, diagnostics)
