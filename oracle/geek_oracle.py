"""CPU oracle for the GEEK hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy / Python-int restatement of the reference
algorithm (``lshclust``, /root/reference/pkg/src/lshclust) for the path
bucketize -> SILK seeding -> one-pass assignment.  It exists so that the
CUDA product path can be checked bit-for-bit on the same inputs.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it; the product package never does.

Parity pin: every function below is checked against golden vectors that
``tests/golden/make_golden.py`` dumped from the reference itself (see
``tests/test_oracle_golden.py``).  Citations are ``file:line`` relative to
/root/reference/pkg/src/lshclust.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

M64 = (1 << 64) - 1
P61 = (1 << 61) - 1
RANK_TABLE_MAX = 4096  # hashing.py:25
DEDUP_TAG = 0xDED0  # seeding.py:38
DOPH_TAG = 0xD0  # transform.py:195, engine.py:390


# --------------------------------------------------------------------------
# seeds (hashing.py:28-41)

def mix64(z: int) -> int:
    """splitmix64 finaliser on a Python int (hashing.py:28-33)."""
    z = (z + 0x9E3779B97F4A7C15) & M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def sub_seed(master: int, *path: int) -> int:
    """derive_seed (hashing.py:36-41)."""
    z = mix64(master & M64)
    for p in path:
        z = mix64(z ^ mix64((p + 0x632BE59BD9B4E019) & M64))
    return z


# --------------------------------------------------------------------------
# MinHash permutation pi over [0, u)  (hashing.py:51-140)

def perm_params(seed: int, u: int):
    """(w, mask, c1, c2, a1, s1, s2) of the cycle-walking mix (hashing.py:97-113)."""
    w = max(1, (u - 1).bit_length())
    mask = (1 << w) - 1
    return (
        w,
        mask,
        (sub_seed(seed, 1) | 1) & mask,
        (sub_seed(seed, 2) | 1) & mask,
        sub_seed(seed, 3) & mask,
        max(1, w // 2),
        max(1, w // 3),
    )


def rank_table(seed: int, u: int) -> np.ndarray:
    """pi for u <= 4096: rank of a 64-bit mix of x + a1 (hashing.py:80-95)."""
    a1 = np.uint64(sub_seed(seed, 3))
    c1 = np.uint64(sub_seed(seed, 1) | 1)
    c2 = np.uint64(sub_seed(seed, 2) | 1)
    with np.errstate(over="ignore"):
        z = np.arange(u, dtype=np.uint64) + a1
        z = (z ^ (z >> np.uint64(30))) * c1
        z = (z ^ (z >> np.uint64(27))) * c2
        z = z ^ (z >> np.uint64(31))
    out = np.empty(u, dtype=np.uint64)
    out[np.argsort(z, kind="stable")] = np.arange(u, dtype=np.uint64)
    return out


def _mix_round(x, mask, c1, c2, a1, s1, s2):
    x = (x + a1) & mask
    x = x ^ (x >> s1)
    x = (x * c1) & mask
    x = x ^ (x >> s2)
    x = (x * c2) & mask
    return x ^ (x >> s1)


def permute(seed: int, u: int, elems) -> np.ndarray:
    """pi(elems) as uint64 (hashing.py:126-140); elements must be in [0, u)."""
    e = np.asarray(elems, dtype=np.int64)
    if e.size and (e.min() < 0 or e.max() >= u):
        raise ValueError("element outside hash universe")
    if u <= RANK_TABLE_MAX:
        return rank_table(seed, u)[e]
    _, mask, c1, c2, a1, s1, s2 = perm_params(seed, u)
    p = [np.uint64(v) for v in (mask, c1, c2, a1, s1, s2)]
    with np.errstate(over="ignore"):
        x = _mix_round(e.astype(np.uint64), *p)
        bad = x >= np.uint64(u)
        while bad.any():
            x[bad] = _mix_round(x[bad], *p)
            bad = x >= np.uint64(u)
    return x


def table_function_seeds(seed: int, table: int, K: int, pinned=None):
    """SignatureScheme.function_seeds (hashing.py:247-254)."""
    if pinned is not None:
        return tuple(int(s) for s in pinned[table])
    return tuple(sub_seed(seed, table, j) for j in range(K))


def set_signatures(fseeds, u: int, sets) -> np.ndarray:
    """(len(sets), K) min-pi matrix (hashing.py:265-282)."""
    sets = [np.asarray(s, dtype=np.int64) for s in sets]
    if not sets:
        return np.empty((0, len(fseeds)), dtype=np.uint64)
    sizes = np.array([s.size for s in sets])
    if (sizes == 0).any():
        raise ValueError("empty set")
    flat = np.concatenate(sets)
    heads = np.concatenate(([0], np.cumsum(sizes)[:-1]))
    out = np.empty((len(sets), len(fseeds)), dtype=np.uint64)
    for j, s in enumerate(fseeds):
        out[:, j] = np.minimum.reduceat(permute(s, u, flat), heads)
    return out


# --------------------------------------------------------------------------
# dense bucketize (hashing.py:208-211, transform.py:95-128)

def direction(seed: int, table: int, d: int) -> np.ndarray:
    return np.random.default_rng([seed & M64, table]).standard_normal(d)


def directions(seed: int, m: int, d: int) -> np.ndarray:
    return np.stack([direction(seed, j, d) for j in range(m)])


def split_sizes(n: int, parts: int) -> np.ndarray:
    q, r = divmod(n, parts)
    s = np.full(parts, q, dtype=np.int64)
    s[:r] += 1
    return s


def rank_split(values: np.ndarray, parts: int):
    """ids grouped by even rank split, ties by id (transform.py:103-109)."""
    order = np.lexsort((np.arange(values.shape[0]), values))
    return np.split(order, np.cumsum(split_sizes(values.shape[0], parts))[:-1])


def slot_codes(values: np.ndarray, parts: int) -> np.ndarray:
    """Per id, the slot index of its rank-split bucket (int64)."""
    codes = np.empty(values.shape[0], dtype=np.int64)
    for s, ids in enumerate(rank_split(values, parts)):
        codes[ids] = s
    return codes


def boundary_counts(values: np.ndarray, parts: int, rels=(1e-12, 1e-6)) -> list:
    """Ids whose projection lies within rel * |boundary| of a rank-split
    boundary midpoint (the north_star tie window around transform.py:103-109's
    split): per boundary s the midpoint of the last key of bucket s and the
    first key of bucket s+1 in the lexsort order; each id is measured against
    the two boundaries around its key (tests/golden/make_benchlaw_golden.py
    dumps the reference's own counts the same way)."""
    n = values.shape[0]
    order = np.lexsort((np.arange(n), values))
    vs = values[order]
    bounds = np.cumsum(split_sizes(n, parts))[:-1]
    if bounds.size == 0:
        return [0 for _ in rels]
    mid = vs[bounds - 1] + 0.5 * (vs[bounds] - vs[bounds - 1])
    pos = np.searchsorted(mid, values)
    lo_mid = mid[np.clip(pos - 1, 0, parts - 2)]
    hi_mid = mid[np.clip(pos, 0, parts - 2)]
    dist = np.minimum(np.abs(values - lo_mid), np.abs(values - hi_mid))
    scale = np.maximum(np.abs(lo_mid), np.abs(hi_mid))
    return [int((dist <= r * scale).sum()) for r in rels]


def homo_buckets(X: np.ndarray, m: int, t: int, seed: int = 0, dirs=None):
    """transform_homo (transform.py:112-128) -> list of (table, slot, members)."""
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    if t > n:
        raise ValueError("t > n")
    A = directions(seed, m, d) if dirs is None else np.asarray(dirs, dtype=np.float64)
    out = []
    for j in range(m):
        for s, ids in enumerate(rank_split(X @ A[j], t)):
            out.append((j, s, np.sort(ids)))
    return out


# --------------------------------------------------------------------------
# SILK (seeding.py:83-197)

def _groups_by_rows(sig: np.ndarray):
    """Indices grouped by identical signature rows, groups in sorted-row
    order, members ascending (seeding.py:83-90)."""
    _, inv = np.unique(sig, axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    order = np.argsort(inv, kind="stable")
    return np.split(order, np.cumsum(np.bincount(inv))[:-1])


def bins_for_table(member_sets, K, L, seed, st, universe, pinned=None):
    """bin_buckets (seeding.py:93-104): [(signature, positions)] with >= 2 positions."""
    if not member_sets:
        return []
    fs = table_function_seeds(seed, st, K, pinned)
    sig = set_signatures(fs, universe, member_sets)
    return [(tuple(sig[g[0]].tolist()), g) for g in _groups_by_rows(sig) if g.size > 1]


def majority(member_sets, positions):
    """majority_vote (seeding.py:107-114); None when nobody wins."""
    ids, cnt = np.unique(np.concatenate([member_sets[i] for i in positions]), return_counts=True)
    win = ids[2 * cnt > len(positions)]
    return win if win.size else None


def votes(member_sets, K, L, delta, seed, universe, pinned=None, trace_ids=None, trace=None):
    """collect_votes (seeding.py:154-165) -> list of sorted id arrays."""
    out = []
    for st in range(L):
        for _, pos in bins_for_table(member_sets, K, L, seed, st, universe, pinned):
            w = majority(member_sets, pos)
            if w is not None and w.size >= delta:
                out.append(w)
                if trace is not None:
                    trace.append((st, tuple(trace_ids[i] for i in pos), w))
    return out


def dedup(groups, K, seed, universe, dedup_tables=1, pinned=None):
    """dedup_groups (seeding.py:117-134) -> groups sorted by member tuple."""
    keep = [np.asarray(g, dtype=np.int64) for g in groups]
    if len(keep) > 1:
        dseed = sub_seed(seed, DEDUP_TAG)
        for tb in range(dedup_tables):
            fs = table_function_seeds(dseed, tb, K, pinned)
            sig = set_signatures(fs, universe, keep)
            nxt = []
            for idx in _groups_by_rows(sig):
                nxt.append(min((keep[i] for i in idx), key=lambda a: (-a.size, tuple(a.tolist()))))
            keep = nxt
    return sorted(keep, key=lambda a: tuple(a.tolist()))


def seed_groups(member_sets, K, L, delta, seed, universe, dedup_tables=1,
                pinned=None, dedup_pinned=None):
    """find_seed_groups (seeding.py:137-151)."""
    raw = votes(member_sets, K, L, delta, seed, universe, pinned)
    return dedup(raw, K, seed, universe, dedup_tables, dedup_pinned)


# --------------------------------------------------------------------------
# exact centroids (numeric.py:19-51)

def exact_sums(rows: np.ndarray) -> list:
    """Per-column exact sums as Python ints at scale 2^-1074."""
    rows = np.asarray(rows, dtype=np.float64)
    out = []
    for col in rows.T:
        tot = 0
        for v in col.tolist():
            if v != 0.0:
                num, den = v.as_integer_ratio()  # den is a power of two
                tot += (num << 1074) // den
        out.append(tot)
    return out


def mean_from_sums(sums, count: int) -> np.ndarray:
    den = count << 1074
    return np.array([float(Fraction(s, den)) for s in sums], dtype=np.float64)


def exact_mean(rows: np.ndarray) -> np.ndarray:
    rows = np.asarray(rows, dtype=np.float64)
    return mean_from_sums(exact_sums(rows), rows.shape[0])


def exact_mean_fast(rows: np.ndarray) -> np.ndarray:
    """Same value as exact_mean, via math.fsum (exactly rounded sum) is NOT
    enough for a correctly rounded mean, so this uses Fraction on the exact
    sum as well -- just vectorised per column with Python ints."""
    return exact_mean(rows)


# --------------------------------------------------------------------------
# assignment (assignment.py:44-107); numpy pairwise f64 order

def l2_distances(X: np.ndarray, C: np.ndarray) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    k, d = C.shape
    out = np.empty((X.shape[0], k))
    step = max(1, min(X.shape[0], (32 << 20) // max(1, 8 * k * d)))
    for lo in range(0, X.shape[0], step):
        diff = X[lo:lo + step, None, :] - C[None, :, :]
        out[lo:lo + step] = np.sqrt((diff * diff).sum(axis=2))
    return out


def assign_l2(X: np.ndarray, C: np.ndarray, chunk: int = 8192):
    """-> (labels int64, best f64, radii f64, objective)."""
    n = X.shape[0]
    lab = np.empty(n, dtype=np.int64)
    best = np.empty(n)
    for lo in range(0, n, chunk):
        dm = l2_distances(X[lo:lo + chunk], C)
        a = np.argmin(dm, axis=1)
        lab[lo:lo + chunk] = a
        best[lo:lo + chunk] = dm[np.arange(a.size), a]
    radii = np.zeros(C.shape[0])
    np.maximum.at(radii, lab, best)
    return lab, best, radii, float(best.sum())


def cat_distances(codes: np.ndarray, modes: np.ndarray) -> np.ndarray:
    """1 - m/(2d - m) (assignment.py:63-67)."""
    d = codes.shape[1]
    mt = (codes[:, None, :] == modes[None, :, :]).sum(axis=2)
    return 1.0 - mt / (2 * d - mt)


def sparse_distances(sets, universe: int, modes: np.ndarray) -> np.ndarray:
    """Binary Jaccard via a dense product (assignment.py:68-78)."""
    sizes_c = modes.sum(axis=1).astype(np.float64)
    Xb = np.zeros((len(sets), universe))
    for r, s in enumerate(sets):
        Xb[r, s] = 1.0
    inter = Xb @ modes.T.astype(np.float64)
    union = Xb.sum(axis=1)[:, None] + sizes_c[None, :] - inter
    with np.errstate(invalid="ignore"):
        return 1.0 - np.where(union > 0, inter / union, 1.0)


def assign_generic(dist_fn, n: int, k: int, chunk: int = 8192):
    lab = np.empty(n, dtype=np.int64)
    best = np.empty(n)
    for lo in range(0, n, chunk):
        dm = dist_fn(lo, min(lo + chunk, n))
        a = np.argmin(dm, axis=1)
        lab[lo:lo + a.size] = a
        best[lo:lo + a.size] = dm[np.arange(a.size), a]
    radii = np.zeros(k)
    np.maximum.at(radii, lab, best)
    return lab, best, radii, float(best.sum())


def mode_of(codes_sub: np.ndarray, code_space: int) -> np.ndarray:
    """Per-attribute mode, ties to the smaller code (seeding.py:180-185)."""
    return np.array([np.argmax(np.bincount(codes_sub[:, c], minlength=code_space))
                     for c in range(codes_sub.shape[1])], dtype=np.int32)


def sparse_mode(sets_sub, universe: int) -> np.ndarray:
    cnt = np.zeros(universe, dtype=np.int64)
    for s in sets_sub:
        cnt[s] += 1
    return (2 * cnt > len(sets_sub)).astype(np.int32)


# --------------------------------------------------------------------------
# sparse / mixed bucketize (hashing.py:285-332, transform.py:131-199)

def doph_reduce(sets, seed: int, D: int, r: int):
    """DophReducer.reduce for every set (hashing.py:312-329)."""
    width = -(-D // r)
    out = []
    for s in sets:
        p = permute(seed, D, s).astype(np.int64)
        b = p // width
        rel = p - b * width
        o = np.argsort(b, kind="stable")
        b, rel = b[o], rel[o]
        ub, st = np.unique(b, return_index=True)
        mins = np.minimum.reduceat(rel, st)
        out.append(np.unique((ub + (mins % P61)) % r))
    return out


def doph_sketch(s, seed: int, D: int, r: int) -> np.ndarray:
    width = -(-D // r)
    p = permute(seed, D, s).astype(np.int64)
    b = p // width
    rel = p - b * width
    out = np.full(r, -1, dtype=np.int64)
    for bb, rr in zip(b.tolist(), rel.tolist()):
        if out[bb] < 0 or rr < out[bb]:
            out[bb] = rr
    carry = -1
    for j in range(2 * r - 1, -1, -1):
        jj = j % r
        if out[jj] >= 0:
            carry = out[jj]
        elif carry >= 0:
            out[jj] = carry
    return out


def discretize(numeric: np.ndarray, bins: int) -> np.ndarray:
    numeric = np.asarray(numeric, dtype=np.float64)
    out = np.empty(numeric.shape, dtype=np.int32)
    for c in range(numeric.shape[1]):
        out[:, c] = slot_codes(numeric[:, c], bins)
    return out


def tokens_of(codes: np.ndarray, code_space: int):
    base = np.arange(codes.shape[1], dtype=np.int64) * code_space
    return [base + row for row in codes.astype(np.int64)]


def signature_buckets(sets, K, L, seed, universe, pinned=None):
    """_signature_buckets (transform.py:158-169) -> [(table, slot, ids)]."""
    out = []
    for tb in range(L):
        sig = set_signatures(table_function_seeds(seed, tb, K, pinned), universe, sets)
        for s, ids in enumerate(_groups_by_rows(sig)):
            out.append((tb, s, np.sort(ids)))
    return out


# --------------------------------------------------------------------------
# engine semantics for dense data at g logical workers (engine.py:109-472)

def shard_bounds(n: int, g: int):
    b = np.concatenate(([0], np.cumsum(split_sizes(n, g))))
    return [(int(b[i]), int(b[i + 1])) for i in range(g)]


def local_votes(tables_buckets, K, L, delta, seed, n, pinned=None):
    """Worker.local_votes (engine.py:242-283) for one worker's buckets."""
    flat = [b for b in tables_buckets]
    sets = [b[2] for b in flat]
    if not sets:
        return []
    sigs = [set_signatures(table_function_seeds(seed, st, K, pinned), n, sets) for st in range(L)]
    out = []
    for st in range(L):
        by = {}
        for i in range(len(sets)):
            by.setdefault(tuple(sigs[st][i].tolist()), []).append(i)
        for key in sorted(by):
            pos = by[key]
            if len(pos) < 2:
                continue
            w = majority(sets, pos)
            if w is not None and w.size >= delta:
                out.append(w)
    return out


def pipeline_dense(X, m, t, tseed, K, L, delta, sseed, g=1, dedup_tables=1,
                   dirs=None, pinned=None, dedup_pinned=None, fallback_seed=0, passes=0):
    """run_pipeline for transform_kind='dense', metric='euclidean'.

    Returns dict(groups, centers, labels, best, radii, objective, warnings).
    """
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    shards = shard_bounds(n, g)
    buckets = homo_buckets(X, m, t, tseed, dirs)  # identical to the synced tables (engine.py:216-225)
    merged = []
    for w in range(g):
        mine = [b for b in buckets if b[0] % g == w]
        merged.extend(local_votes(mine, K, L, delta, sseed, n, pinned))
    merged.sort(key=lambda a: tuple(a.tolist()))
    groups = dedup(merged, K, sseed, n, dedup_tables, dedup_pinned)
    warnings = []
    if not groups:
        warnings.append("fallback")
        rng = np.random.default_rng(fallback_seed)
        picks = sorted(int(rng.integers(lo, hi)) for lo, hi in shards)
        groups = [np.array([p], dtype=np.int64) for p in picks]
    centers = np.stack([exact_mean(X[gm]) for gm in groups])
    lab, best, radii, obj = assign_l2(X, centers)
    out = dict(groups=groups, centers=centers, labels=lab, best=best,
               radii=radii, objective=obj, warnings=warnings)
    if passes:  # _refine_distributed (engine.py:519-537); exact sums make it g-independent
        out.update(refine_dense(X, lab, centers.shape[0], passes))
    return out


# --------------------------------------------------------------------------
# refinement passes (assignment.py:110-170, engine.py:519-537)

def centers_from_labels(X: np.ndarray, labels: np.ndarray, k: int):
    """Exact centroids of the non-empty clusters in label order
    (assignment.py:110-127); -> (centers [k', d], sizes [k'])."""
    X = np.asarray(X, dtype=np.float64)
    rows = [np.flatnonzero(labels == j) for j in range(k)]
    rows = [r for r in rows if r.size]
    return np.stack([exact_mean(X[r]) for r in rows]), np.array([r.size for r in rows], dtype=np.int64)


def refine_dense(X: np.ndarray, labels: np.ndarray, k: int, passes: int):
    """refine(data, clustering, 'euclidean', passes) (assignment.py:157-170):
    -> dict(centers, sizes, labels, best, radii, objective) of the last pass."""
    out = None
    for _ in range(passes):
        C, sizes = centers_from_labels(X, labels, k)
        labels, best, radii, obj = assign_l2(X, C)
        k = C.shape[0]
        out = dict(centers=C, sizes=sizes, labels=labels, best=best, radii=radii, objective=obj)
    return out


def modes_from_labels(codes: np.ndarray, code_space: int, labels: np.ndarray, k: int) -> np.ndarray:
    """Categorical modes of the non-empty clusters (assignment.py:122-126)."""
    return np.stack([mode_of(codes[labels == j], code_space) for j in range(k) if (labels == j).any()])


def sparse_modes_from_labels(sets, universe: int, labels: np.ndarray, k: int) -> np.ndarray:
    """Sparse strict-majority modes of the non-empty clusters (assignment.py:127-131)."""
    return np.stack([sparse_mode([sets[i] for i in np.flatnonzero(labels == j)], universe)
                     for j in range(k) if (labels == j).any()])


# --------------------------------------------------------------------------
# comparison methods (baselines.py:34-136), dense Euclidean

def seed_random_idx(n: int, k: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).choice(n, size=k, replace=False)


def kmeanspp_idx(X: np.ndarray, k: int, seed: int) -> list:
    """baselines.py:52-80 with the Euclidean weights best**2."""
    rng = np.random.default_rng(seed)
    n = X.shape[0]
    chosen = [int(rng.integers(n))]
    best = None
    while len(chosen) < k:
        d_new = l2_distances(X, X[chosen[-1]][None, :])[:, 0]
        best = d_new if best is None else np.minimum(best, d_new)
        w = best ** 2
        w[chosen] = 0.0
        total = w.sum()
        if total <= 0.0:
            chosen.append(int(rng.choice(np.setdiff1d(np.arange(n), np.array(chosen)))))
        else:
            chosen.append(int(rng.choice(n, p=w / total)))
    return chosen


def lloyd_dense(X: np.ndarray, k: int, seed: int, max_iters: int = 100, tol: float = 1e-6):
    """baselines.py:83-114 -> dict(centers, labels, radii, objective)."""
    X = np.asarray(X, dtype=np.float64)
    C = X[seed_random_idx(X.shape[0], k, seed)]
    lab, best, radii, obj = assign_l2(X, C)
    for _ in range(max_iters):
        newC, _ = centers_from_labels(X, lab, C.shape[0])
        alive = np.bincount(lab, minlength=C.shape[0]) > 0
        moved = max((float(np.linalg.norm(a - b)) for a, b in zip(C[alive], newC)), default=0.0)
        C = newC
        lab, best, radii, obj = assign_l2(X, C)
        if moved < tol:
            break
    return dict(centers=C, labels=lab, radii=radii, objective=obj)


# --------------------------------------------------------------------------
# vector files (io.py:21-48)

def read_vecs(raw: bytes, bvecs: bool):
    """Parse .fvecs / .bvecs bytes -> float64 [n][d], or the reference's
    FormatError message as a string (io.py:21-48)."""
    raw = np.frombuffer(raw, dtype=np.uint8)
    if raw.size == 0:
        return np.empty((0, 0))
    if raw.size < 4:
        return "truncated record at byte 0"
    d = int(raw[:4].view("<i4")[0])
    if d <= 0:
        return "non-positive dimension at byte 0"
    dt = np.dtype("<u1") if bvecs else np.dtype("<f4")
    record = 4 + d * dt.itemsize
    if raw.size % record:
        return f"truncated record at byte {(raw.size // record) * record}"
    table = raw.reshape(-1, record)
    dims = table[:, :4].copy().view("<i4").ravel()
    if (dims != d).any():
        return f"inconsistent dimension at byte {int(np.flatnonzero(dims != d)[0]) * record}"
    return table[:, 4:].copy().view(dt).astype(np.float64)


# --------------------------------------------------------------------------
# synthetic data (synth.py:39-104), used to make parity inputs

def spread_means(k, dim, separation, rng):
    if k == 1:
        return np.zeros((1, dim))
    idx = np.arange(k)
    rad = np.sqrt(idx + 0.5)
    ang = idx * (np.pi * (3.0 - np.sqrt(5.0)))
    plane = np.stack([rad * np.cos(ang), rad * np.sin(ang)], axis=1)
    plane += 0.05 * rng.standard_normal(plane.shape)
    basis = np.linalg.qr(rng.standard_normal((dim, min(2, dim))))[0]
    means = plane[:, : basis.shape[1]] @ basis.T
    dmin = np.inf
    for lo in range(0, k, 256):
        blk = np.sqrt(((means[lo:lo + 256, None, :] - means[None, :, :]) ** 2).sum(-1))
        for r in range(blk.shape[0]):
            blk[r, lo + r] = np.inf
        dmin = min(dmin, blk.min())
    return means * (separation / dmin)


def gaussian_mixture(n, dim, clusters, separation=10.0, seed=0):
    rng = np.random.default_rng(seed)
    labels = np.sort(rng.integers(0, clusters, n))
    labels[:clusters] = np.arange(clusters)
    labels = np.sort(labels)
    means = spread_means(clusters, dim, separation, rng)
    return means[labels] + rng.standard_normal((n, dim)), labels
