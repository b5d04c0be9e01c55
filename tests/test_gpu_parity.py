"""GPU parity: the CUDA path (through libgeek's C ABI) against the CPU oracle
and the golden vectors dumped from the reference.  Integer outputs (pi
values, signatures, bucket codes, seed groups, labels) and the float64
centers / radii / objectives must be bit-identical."""

import hashlib

import numpy as np
import pytest
import torch

from oracle import geek_oracle as O
from tests.golden_io import baselines_meta, csr, groups as golden_groups, meta, npz, refine_meta

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2106_10515_b200")


def keys(gs):
    return [tuple(np.asarray(g.members if hasattr(g, "members") else g).tolist()) for g in gs]


WORKED = [(0, 0, [0, 1, 3]), (0, 1, [2, 4, 5]), (1, 0, [0, 1, 3, 4]), (1, 1, [5]),
          (2, 0, [0, 1, 3, 5]), (2, 1, [2, 4]), (3, 0, [0, 1, 3, 5]), (3, 1, [4, 5])]
WORKED_POINTS = np.array([[0.0, 0.0, 0.0, 0.0], [0.1, 0.1, 0.1, 0.1], [10.0, 0.2, 10.0, 0.3],
                          [0.2, 0.3, 0.2, 0.4], [10.1, 0.4, 10.1, 0.5], [12.0, 0.5, 12.0, 0.2]])


def worked_buckets():
    return [G.Bucket(t, s, np.array(m)) for t, s, m in WORKED]


def worked_params():
    return G.SeedingParams(2, 2, min_group_size=1, seed=0, dedup_tables=1, table_seeds=((6, 7), (15, 20)),
                           dedup_seeds=((0, 1001),))


# ---- MinHash ----------------------------------------------------------------

def test_permutation_golden():
    arr = npz("pi")
    for seed, u, key in meta()["pi_cases"]:
        if u >= (1 << 32):
            continue
        got = G.MinHashFunction(seed, u).permute(arr[key + "_x"])
        assert np.array_equal(got, arr[key + "_y"]), key


def test_permutation_bijective_and_inverse_scan_agree():
    for u in (6, 4096, 4097, 100_003):
        f = G.MinHashFunction(7, u)
        p = f.permute(np.arange(u))
        assert np.array_equal(np.sort(p), np.arange(u))


def test_signatures_golden():
    arr = npz("sigs")
    for K, L, u, seed in [(3, 4, 700, 13), (2, 3, 5000, 1), (3, 2, 100_000, 2)]:
        p = f"{K}_{L}_{u}_{seed}"
        sets = csr(arr[p + "_flat"], arr[p + "_off"])
        sch = G.SignatureScheme(K, L, u, seed=seed)
        for tb in range(L):
            assert np.array_equal(sch.signatures_for_sets(tb, sets), arr[f"{p}_{tb}"])


@pytest.mark.parametrize("u,lo,hi", [(50_000, 20, 300), (5_000_000, 1, 90), (3000, 30, 200)])
def test_set_minhash_large_sets_vs_oracle(u, lo, hi, monkeypatch):
    """Set signatures of large sets (cycle-walking permutations over universes
    above the rank-table limit, and rank tables below it) through the default
    kernels and the per-element kernel (GEEK_MINHASH_GENERIC=1) equal the
    oracle's min-pi over every function; ragged sizes incl. singletons,
    duplicate ids."""
    rng = np.random.default_rng(u + lo)
    sets = [rng.integers(0, u, rng.integers(lo, hi)) for _ in range(700)]
    sch = G.SignatureScheme(3, 20, u, seed=9)
    funcs = sch.all_functions()
    fseeds = [f.seed for f in funcs]
    want = O.set_signatures(fseeds, u, sets)
    from paper_2106_10515_b200.hashing import csr_from_sets, set_signatures_device
    flat, off, _ = csr_from_sets(sets)
    got = set_signatures_device(funcs, flat, off, len(sets)).cpu().numpy().view(np.uint32).astype(np.uint64)
    assert np.array_equal(got, want)
    monkeypatch.setenv("GEEK_MINHASH_GENERIC", "1")
    got2 = set_signatures_device(funcs, flat, off, len(sets)).cpu().numpy().view(np.uint32).astype(np.uint64)
    assert np.array_equal(got2, want)


def test_minhash_known_answers():
    assert G.MinHashFunction.identity(10)({3, 5, 7}) == 3
    assert G.MinHashFunction(42, 100)(np.arange(100)) == 0
    with pytest.raises(G.InvalidInput):
        G.MinHashFunction(1, 8)([8])


def test_doph_golden():
    arr = npz("doph")
    red = G.DophReducer(G.hashing.derive_seed(3, 0xD0), 3_000_000, 400)
    got = red.reduce_dataset(csr(arr["flat"], arr["off"]))
    want = csr(arr["red_flat"], arr["red_off"])
    assert all(np.array_equal(a, b) for a, b in zip(got, want))
    assert G.DophReducer(5, 12, 4).sketch(np.array([0, 5])).tolist() == [0, 0, 2, 2]


# ---- bucketize ----------------------------------------------------------------

def test_worked_points_transform():
    p = G.HomoTransformParams(4, 2, directions=np.eye(4))
    got = {(b.table, b.slot): b.members.tolist() for b in G.transform_homo(G.DenseData(WORKED_POINTS), p)}
    assert got == {(0, 0): [0, 1, 3], (0, 1): [2, 4, 5], (1, 0): [0, 1, 2], (1, 1): [3, 4, 5],
                   (2, 0): [0, 1, 3], (2, 1): [2, 4, 5], (3, 0): [0, 1, 5], (3, 1): [2, 3, 4]}


def test_rank_split_edge_cases():
    # uneven split, first bucket takes the extra id (test_transform.py:52-57)
    X = np.arange(7, dtype=float).reshape(7, 1)
    bt = G.transform_homo(G.DenseData(X), G.HomoTransformParams(1, 2, directions=np.ones((1, 1))))
    assert bt[0].members.tolist() == [0, 1, 2, 3]
    # ties by id, -0.0 == +0.0
    for vals in ([7.0] * 4, [0.0, -0.0, 0.0, -0.0], [1.0, -0.0, 0.0, -1.0, 0.0, 2.0]):
        v = np.array(vals).reshape(-1, 1)
        bt = G.transform_homo(G.DenseData(v), G.HomoTransformParams(1, 2, directions=np.ones((1, 1))))
        assert np.array_equal(bt.codes_host()[0], O.slot_codes(v[:, 0], 2))
    # t == n gives singletons
    bt = G.transform_homo(G.DenseData(np.arange(5.0).reshape(5, 1)), G.HomoTransformParams(2, 5, seed=3))
    assert all(b.members.size == 1 for b in bt)
    with pytest.raises(G.InvalidInput):
        G.transform_homo(G.DenseData(np.zeros((3, 2))), G.HomoTransformParams(1, 4))


@pytest.mark.parametrize("path", ["grouped", "per-bin", "coarse-groups"])
@pytest.mark.parametrize("n,t,dup", [(20_000, 3, True), (50_000, 997, False), (30_000, 30_000, False),
                                     (123_457, 1000, False)])
def test_rank_split_random_vs_oracle(n, t, dup, path, monkeypatch):
    """(path: the grouped split -- SMEM group counts, fine counts only in
    straddling groups, group codes -- the per-bin split of round 1, and coarse
    2^7 code groups over 2^3 counting groups)"""
    if path == "per-bin":
        monkeypatch.setenv("GEEK_SPLIT_GROUPS", "0")
    elif path == "coarse-groups":
        monkeypatch.setenv("GEEK_SPLIT_GROUPS", "7")
        monkeypatch.setenv("GEEK_SPLIT_CSHIFT", "3")
    rng = np.random.default_rng(n + t)
    X = rng.standard_normal((n, 5)).astype(np.float32)
    if dup:  # giant tie classes exercise the sorted fallback
        X[: n // 2] = X[0]
        X[n // 2:, 0] = 0.0
    from paper_2106_10515_b200 import transform as T

    A = O.directions(11, 3, 5)
    assert np.array_equal(A, G.HomoTransformParams(3, t, seed=11).direction_matrix(5))
    Xd = torch.from_numpy(X).cuda()
    keys = T.project_keys(Xd, A)
    codes = T.rank_split_codes(keys, t)
    tol = T.projection_tolerance(A, int(np.frexp(np.abs(X).max())[1]))
    st = T.split_boundary_stats(keys, codes, t, tol)
    want = np.stack([O.slot_codes(X.astype(np.float64) @ A[j], t) for j in range(3)])
    got = codes.cpu().numpy().T
    # the float64 projection order differs from BLAS, so a code may differ only
    # for an id the boundary pass reports as ambiguous (within the order bound)
    bad = set(zip(*np.nonzero(got != want)))
    amb = set(map(tuple, st["ambiguous_ids"].tolist()))
    assert st["listed_complete"] and bad <= amb, (len(bad), st["ambiguous"])
    assert st["ambiguous"] == len(amb)
    if not dup:  # window counts against the oracle's (searchsorted on the exact lexsort)
        V = X.astype(np.float64) @ A.T
        want_rel = np.sum([O.boundary_counts(V[:, j], t) for j in range(3)], axis=0)
        assert [st["within_rel"]["1e-12"], st["within_rel"]["1e-06"]] == want_rel.tolist()


@pytest.mark.parametrize("name", ["c06", "small"])
def test_codes_golden(name):
    m = meta()["pipelines"][name]
    arr = npz("pipelines")
    _, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    bt = G.transform_homo(G.DenseData(X), G.HomoTransformParams(m["m"], m["t"], seed=m["tseed"]))
    assert np.array_equal(bt.codes_host(), arr[name + "_codes"])


@pytest.mark.parametrize("proj", ["dmma", "tcgen05"])
def test_cfg1_codes_golden_sha(proj, monkeypatch):
    """(proj: K1 on kind::i8 tcgen05 digits, the default, or on DMMA, GEEK_TCPROJ=0)"""
    if proj == "dmma":
        monkeypatch.setenv("GEEK_TCPROJ", "0")
    m = meta()["pipelines"]["cfg1"]
    _, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    assert hashlib.sha256(X.tobytes()).hexdigest() == m["data_sha"]
    bt = G.transform_homo(G.DenseData(X), G.HomoTransformParams(m["m"], m["t"], seed=m["tseed"]))
    codes = bt.codes_host().astype(np.int32)
    assert hashlib.sha256(np.ascontiguousarray(codes).tobytes()).hexdigest() == m["codes_sha"]


# ---- SILK ---------------------------------------------------------------------

def test_worked_example_seeding():
    b, p = worked_buckets(), worked_params()
    bins = G.bin_buckets(b, p, 0, universe=6)
    got = {tuple(b[i].bucket_id for i in x.bucket_indices) for x in bins}
    assert got == {((0, 0), (1, 0), (2, 0), (3, 0)), ((0, 1), (2, 1), (3, 1))}
    assert keys(G.find_seed_groups(b, p, universe=6)) == [(0, 1, 3), (2, 4), (2, 4, 5), (5,)]
    trace = []
    G.find_seed_groups(b, p, universe=6, trace=trace)
    by_id = {x.bucket_id: x for x in b}
    assert trace
    for _, ids, grp in trace:
        for mem in grp.members:
            assert 2 * sum(mem in by_id[i].members for i in ids) > len(ids)
    raw = G.seeding.collect_votes(b, p, 6)
    assert sorted(keys(raw)) == sorted([(0, 1, 3), (0, 1, 3), (2, 4), (2, 4, 5), (5,)])
    merged = [G.SeedGroup(x) for x in ([0, 1, 3], [0, 1, 3], [2, 4], [2, 4], [5])]
    assert keys(G.dedup_groups(merged, p, 6)) == [(0, 1, 3), (2, 4), (5,)]


def test_majority_vote_rules():
    b = [G.Bucket(i, 0, np.array(m)) for i, m in enumerate([[1, 2], [1, 2], [1, 3], [1, 3]])]
    assert G.majority_vote(G.Bin((0,), (0, 1, 2, 3)), b).members.tolist() == [1]
    b = [G.Bucket(i, 0, np.array(m)) for i, m in enumerate([[1, 2], [1, 2], [1, 2], [1, 3]])]
    assert G.majority_vote(G.Bin((0,), (0, 1, 2, 3)), b).members.tolist() == [1, 2]


def test_invscan_equals_member_scan():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((40_000, 8)).astype(np.float32)
    bt = G.transform_homo(G.DenseData(X), G.HomoTransformParams(6, 300, seed=2))
    sch = G.SignatureScheme(3, 4, 40_000, seed=9)
    funcs = sch.all_functions()
    fast = G.seeding.bucket_signatures_codes(bt, funcs)
    flat, off = bt.member_csr()
    slow = G.seeding.bucket_signatures_csr(flat, off, len(bt), funcs)
    assert torch.equal(fast, slow)
    members = [b.members for b in bt]
    want = O.set_signatures(sch.function_seeds(1), 40_000, members)
    got = slow[3:6].t().cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want)


def test_dedup_random_vs_oracle():
    rng = np.random.default_rng(1)
    for seed in range(5):
        gs = [np.unique(rng.integers(0, 16, rng.integers(1, 7))) for _ in range(12)]
        gs += gs[:3]
        p = G.SeedingParams(2, 3, seed=seed)
        got = G.dedup_groups([G.SeedGroup(g) for g in gs], p, 16)
        assert keys(got) == keys(O.dedup(gs, 2, seed, 16))


# ---- centers + assign -----------------------------------------------------------

def test_exact_centroid_vs_oracle():
    rng = np.random.default_rng(7)
    for dtype in (np.float64, np.float32):
        X = (rng.standard_normal((500, 9)) * np.exp(rng.uniform(-20, 20, (500, 9)))).astype(dtype)
        X[3, 2] = 0.0
        X[4, 4] = -X[5, 4]
        got = G.numeric.exact_centroid(X)
        assert np.array_equal(got, O.exact_mean(X.astype(np.float64)))
    assert G.numeric.exact_centroid(np.array([[0.1], [0.2], [0.3]]))[0] == 0.2


def test_assign_c08_golden():
    arr = npz("pipelines")
    rng = np.random.default_rng(80)
    X = rng.standard_normal((10_000, 16))
    cents = [G.CentralVector("centroid", rng.standard_normal(16)) for _ in range(200)]
    got = G.assign(G.DenseData(X), cents, "euclidean")
    assert np.array_equal(got.assignment, arr["c08_labels"])
    assert np.array_equal(got.radii, arr["c08_radii"])
    assert got.objective == meta()["c08_objective"]
    codes = rng.integers(0, 8, (10_000, 9)).astype(np.int32)
    modes = [G.CentralVector("mode", rng.integers(0, 8, 9).astype(np.int32)) for _ in range(200)]
    got = G.assign(G.CategoricalData(codes, code_space=8), modes, "jaccard")
    assert np.array_equal(got.assignment, arr["c08cat_labels"])
    assert np.array_equal(got.radii, arr["c08cat_radii"])


@pytest.mark.parametrize("d", [3, 8, 100, 128, 129, 300, 960])
def test_assign_pairwise_order_vs_oracle(d):
    rng = np.random.default_rng(d)
    X = rng.standard_normal((700, d))
    C = rng.standard_normal((13, d))
    C[5] = C[2]  # exact duplicate center: ties go to the lower index
    got = G.assign(G.DenseData(X), [G.CentralVector("centroid", c) for c in C], "euclidean")
    lab, best, radii, obj = O.assign_l2(X, C)
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj


@pytest.mark.parametrize("d,k,n", [(960, 150, 1001), (257, 129, 7), (1536, 3, 5), (960, 8, 3333), (300, 16, 999),
                                   (129, 1, 77), (640, 5, 100_003)])
def test_assign_wide_rows_vs_oracle(d, k, n):
    """d > 128 without a screen: the transposed-center kernel (one thread per
    center, points in SMEM), float32 rows, duplicate centers, ragged n and k
    beyond one 128-center pass."""
    rng = np.random.default_rng(d + k)
    C = rng.standard_normal((k, d)) * 2
    X = (C[rng.integers(0, k, n)] + rng.standard_normal((n, d))).astype(np.float32)
    C[k - 1] = C[0]
    X[0] = C[0].astype(np.float32)
    got = G.assign(G.DenseData(X), [G.CentralVector("centroid", c) for c in C], "euclidean")
    lab, best, radii, obj = O.assign_l2(X.astype(np.float64), C)
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj


@pytest.mark.parametrize("wide", ["66", "65", "64"])
@pytest.mark.parametrize("case", ["gist", "offset", "overflow", "shuffled"])
def test_assign_wide_screens_vs_oracle(case, wide, monkeypatch):
    """d > 128 screens: the FP16x3 GEMM over K = 3d of rows centered at their
    tile's origin center (default, mode 66) or at the center mean (65), and the
    float64 DGEMM (GEEK_WIDE=64), then the exact classifier / recheck; near
    ties (duplicate and near-duplicate centers), a large common offset,
    shuffled rows (poor tile origins), and an f16 overflow (points far
    outside the centers' scale: mode 0, every point scanned exactly)."""
    monkeypatch.setenv("GEEK_WIDE", wide)
    rng = np.random.default_rng(7)
    d, k, n = (960, 150, 6000) if case == "gist" else (300, 64, 4000)
    C = rng.random((k, d)) * 0.2 if case == "gist" else rng.standard_normal((k, d)) * 2 + (50.0 if case == "offset" else 0.0)
    C[k - 1] = C[0]
    C[5] = C[4] + 1e-7
    lab0 = np.sort(rng.integers(0, k, n)) if case != "shuffled" else rng.integers(0, k, n)
    X = (C[lab0] + rng.standard_normal((n, d)) * (0.02 if case == "gist" else 1.0)).astype(np.float32)
    X[0] = C[0].astype(np.float32)
    if case == "overflow":
        X[::97] *= 1e4
    got = G.assign(G.DenseData(X), [G.CentralVector("centroid", c) for c in C], "euclidean")
    lab, best, radii, obj = O.assign_l2(X.astype(np.float64), C)
    st = G.assignment.last_assign_stats()
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj
    want_mode = 64 if wide == "64" else (0 if case == "overflow" else int(wide))
    assert st["screen_mode"] == want_mode
    if want_mode == 66 and case != "shuffled":
        assert st["assign_rechecked"] < 0.2 * n


@pytest.mark.parametrize("d,k,offset", [(128, 37, 0.0), (128, 300, 300.0), (16, 5, 0.0), (200, 64, 50.0)])
def test_assign_screened_f32_vs_oracle(d, k, offset):
    """float32 data takes the float32 screen + exact recheck path."""
    rng = np.random.default_rng(d * 1000 + k)
    C = rng.standard_normal((k, d)) * 3 + offset
    lab0 = rng.integers(0, k, 20_000)
    X = (C[lab0] + rng.standard_normal((20_000, d))).astype(np.float32)
    C[k // 2] = C[1]                     # duplicate centers: exact tie -> lower index
    X[:50] = ((C[2] + C[3]) / 2).astype(np.float32)  # equidistant points
    got = G.assign(G.DenseData(X), [G.CentralVector("centroid", c) for c in C], "euclidean")
    lab, best, radii, obj = O.assign_l2(X.astype(np.float64), C)
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj
    assert G.assignment.last_assign_stats()["assign_rechecked"] >= 50


def test_tcgen05_screen_selftest():
    """The tcgen05 screens agree with float64 far inside the classifier's bounds."""
    import ctypes

    out = (ctypes.c_double * 2)()
    L = G._lib.load_library()
    assert L.geek_tc_selftest(128, 256, 3, out) == 0
    assert out[0] < 1e-5  # TF32x3 bound used by the classifier: ~9e-5 * |x'||c'| at d = 128
    assert out[1] == 0
    assert L.geek_tc_selftest(128, 256, 1, out) == 0
    assert out[0] < 5e-4  # 1x TF32 bound: ~2.0e-3 * |x'||c'| at d = 128
    assert L.geek_tc_selftest(128, 256, 16, out) == 0
    assert out[0] < 1e-5  # FP16x3 (scaled operands): same significand as TF32x3
    assert out[1] == 0
    assert L.geek_tc_selftest(128, 256, 17, out) == 0
    assert out[0] < 5e-4  # tile-local FP16: one f16 product, error ~2^-10 |x''||c'| <= 2^-10 (|x'| + |c'|)|c'|


@pytest.mark.parametrize("mode", ["1", "3", "16", "17"])
def test_assign_screen_modes_vs_oracle(mode, monkeypatch):
    monkeypatch.setenv("GEEK_SCREEN", mode)
    rng = np.random.default_rng(11)
    C = rng.standard_normal((150, 128)) * 4 + 200.0
    C[7] = C[3] + 1e-9
    X = (C[rng.integers(0, 150, 30_000)] + rng.standard_normal((30_000, 128))).astype(np.float32)
    got = G.assign(G.DenseData(X), [G.CentralVector("centroid", c) for c in C], "euclidean")
    lab, best, radii, obj = O.assign_l2(X.astype(np.float64), C)
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj


@pytest.mark.parametrize("d,mode", [(100, "16"), (24, "16"), (9, "16"), (104, "17"), (24, "17")])
def test_fp16_screen_ragged_dims_and_tiny_coordinates(d, mode, monkeypatch):
    """FP16x3 / tile-local FP16 at dims that are not a multiple of the 16-dim
    K slice, with coordinates spanning ~9 orders of magnitude (scaled parts
    underflow to f16 subnormals: the bound's absolute term covers them)."""
    monkeypatch.setenv("GEEK_SCREEN", mode)
    rng = np.random.default_rng(100 + d)
    C = rng.standard_normal((90, d)) * 500.0
    C[:, : d // 3] *= 1e-6
    C[11] = C[5] + 1e-7
    X = (C[rng.integers(0, 90, 8_000)] + rng.standard_normal((8_000, d)) * 20.0).astype(np.float32)
    X[:, : d // 3] = (rng.standard_normal((8_000, d // 3)) * 1e-4).astype(np.float32)
    got = G.assign(G.DenseData(X), [G.CentralVector("centroid", c) for c in C], "euclidean")
    lab, best, radii, obj = O.assign_l2(X.astype(np.float64), C)
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj


@pytest.mark.parametrize("mode", ["16", "17"])
def test_fp16_screen_range_fallback(mode, monkeypatch):
    """A point far outside the centers' range overflows the scaled f16 operand:
    the screen is redone in TF32x3 and the labels stay exact."""
    monkeypatch.setenv("GEEK_SCREEN", mode)
    rng = np.random.default_rng(12)
    C = rng.standard_normal((40, 64)) * 3
    X = (C[rng.integers(0, 40, 5_000)] + rng.standard_normal((5_000, 64)) * 0.5).astype(np.float32)
    X[17, 5] = 3.0e6
    X[18] = 0.0
    got = G.assign(G.DenseData(X), [G.CentralVector("centroid", c) for c in C], "euclidean")
    lab, best, radii, obj = O.assign_l2(X.astype(np.float64), C)
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj


@pytest.mark.parametrize("bound", ["1", "0", "noskip"])
@pytest.mark.parametrize("order", ["clustered", "shuffled", "far"])
def test_fp16x3_start_bound_orders(order, bound, monkeypatch):
    """The default FP16x3 screen with its lists starting at a bound from each
    point tile's origin center and the center tiles out of reach skipped (and
    without skipping, and without bounds, GEEK_SCREEN_BOUND=0): exact labels
    for cluster-ordered ids, shuffled ids (poor origins: more insertions) and
    points far from every center (the bound sits far above the best)."""
    monkeypatch.setenv("GEEK_SCREEN_BOUND", "1" if bound == "noskip" else bound)
    if bound == "noskip":  # origin bounds without center-tile skipping
        monkeypatch.setenv("GEEK_SCREEN_SKIP", "0")
    rng = np.random.default_rng(23)
    k, d, n = 700, 96, 50_000
    C = np.cumsum(rng.standard_normal((k, d)) * 2.0, axis=0) + 100.0
    C[9] = C[8] + 1e-6
    C[400] = C[401]  # exact duplicate centers: ties to the lower index
    lab0 = np.sort(rng.integers(0, k, n))
    X = (C[lab0] + rng.standard_normal((n, d))).astype(np.float32)
    if order == "shuffled":
        X = X[rng.permutation(n)]
    if order == "far":
        X[::7] += 300.0
    got = G.assign(G.DenseData(X), [G.CentralVector("centroid", c) for c in C], "euclidean")
    lab, best, radii, obj = O.assign_l2(X.astype(np.float64), C)
    st = G.assignment.last_assign_stats()
    assert st["screen_mode"] == 16
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj


@pytest.mark.parametrize("order", ["clustered", "shuffled"])
def test_tile_local_screen_orders(order, monkeypatch):
    """The tile-local screen (GEEK_SCREEN=17): exact labels whatever the id order; on
    cluster-ordered ids (the reference generator's order) each tile's origin
    sits next to its points, so almost nothing beyond the near-duplicate
    centers reaches the recheck."""
    monkeypatch.setenv("GEEK_SCREEN", "17")
    rng = np.random.default_rng(21)
    k, d, n = 400, 128, 60_000
    C = np.cumsum(rng.standard_normal((k, d)) * 2.0, axis=0) + 100.0  # a long chain: large |x'|
    C[9] = C[8] + 1e-6  # near-duplicate centers: always rechecked
    lab0 = np.sort(rng.integers(0, k, n))
    X = (C[lab0] + rng.standard_normal((n, d))).astype(np.float32)
    if order == "shuffled":
        X = X[rng.permutation(n)]
    got = G.assign(G.DenseData(X), [G.CentralVector("centroid", c) for c in C], "euclidean")
    lab, best, radii, obj = O.assign_l2(X.astype(np.float64), C)
    st = G.assignment.last_assign_stats()
    assert st["screen_mode"] == 17
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj
    if order == "clustered":
        assert st["assign_rechecked"] < 0.02 * n + 2 * (lab0 == 8).sum() + 2 * (lab0 == 9).sum()


def test_assign_abi_workspace_stats_events():
    """The C-ABI contract of geek_assign_l2: caller workspace (size query;
    too small -> GEEK_ERANGE), device-side statistics, caller events around
    the screen, no host synchronisation needed to launch it."""
    from paper_2106_10515_b200 import _lib
    from paper_2106_10515_b200.assignment import AssignStats

    rng = np.random.default_rng(3)
    k, d, n = 300, 128, 50_000
    C = rng.standard_normal((k, d)) * 3
    X = (C[np.sort(rng.integers(0, k, n))] + rng.standard_normal((n, d))).astype(np.float32)
    Xd, Cd = torch.from_numpy(X).cuda(), torch.from_numpy(C).cuda()
    L = _lib.load_library()
    wsb = int(L.geek_assign_l2_workspace_size(n, d, k))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    lab = torch.empty(n, dtype=torch.int64, device="cuda")
    best = torch.empty(n, dtype=torch.float64, device="cuda")
    st = AssignStats()
    _lib.call("geek_assign_l2", _lib.ptr(Xd), 0, n, d, _lib.ptr(Cd), k, _lib.ptr(lab), _lib.ptr(best),
              _lib.ptr(st.dev), _lib.C.c_void_p(st.ev0.cuda_event), _lib.C.c_void_p(st.ev1.cuda_event),
              _lib.ptr(ws), wsb, _lib.stream())
    info = st.read()
    want_lab, want_best, _, _ = O.assign_l2(X.astype(np.float64), C)
    assert np.array_equal(lab.cpu().numpy(), want_lab)
    assert np.array_equal(best.cpu().numpy(), want_best)
    assert info["screen_mode"] == 16 and info["screen_ms"] > 0 and info["assign_rechecked"] >= info["assign_full_scans"]
    # center tiles out of every row's reach are skipped (cluster-ordered rows, 2 center tiles)
    total = -(-n // 128) * -(-k // 192)
    assert 0 < info["screen_tiles"] < total
    small = torch.empty(1 << 16, dtype=torch.uint8, device="cuda")
    with pytest.raises(G.EngineError, match="workspace"):
        _lib.call("geek_assign_l2", _lib.ptr(Xd), 0, n, d, _lib.ptr(Cd), k, _lib.ptr(lab), _lib.ptr(best), None, None,
                  None, _lib.ptr(small), small.numel(), _lib.stream())


def test_tie_to_lowest_index():
    c = G.assign(G.DenseData(np.array([[0.0]])),
                 [G.CentralVector("centroid", [v]) for v in (1.0, 2.0, 3.0, -1.0)], "euclidean")
    assert c.assignment[0] == 0


def test_pairwise_sum_long_vectors():
    rng = np.random.default_rng(5)
    for n in (1, 7, 8, 129, 1000, 100_003, 262_147):
        v = rng.random(n)
        got = G.assignment.pairwise_sum(torch.from_numpy(v).cuda()).item()
        assert got == v.sum(), n


# ---- end-to-end pipelines ----------------------------------------------------------

def dense_config(m, g):
    return G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(g),
                            homo=G.HomoTransformParams(m["m"], m["t"], seed=m["tseed"]),
                            seeding=G.SeedingParams(m["K"], m["L"], min_group_size=m["delta"], seed=m["sseed"]))


@pytest.mark.parametrize("name", ["c06", "small", "cfg1"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_dense_pipeline_golden(name, dtype):
    m = meta()["pipelines"][name]
    arr = npz("pipelines")
    _, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    if dtype == np.float32:
        X = X.astype(np.float32)
    for g in m["runs"]:
        out = G.run_pipeline(G.DenseData(X), dense_config(m, int(g)))
        if dtype == np.float32:  # different data: check against the oracle on the f32 values
            if name == "cfg1":
                continue
            ref = O.pipeline_dense(X.astype(np.float64), m["m"], m["t"], m["tseed"], m["K"], m["L"], m["delta"],
                                   m["sseed"], g=int(g))
            assert keys(out.seed_groups) == keys(ref["groups"])
            assert np.array_equal(out.clustering.assignment, ref["labels"])
            assert np.array_equal(out.clustering.radii, ref["radii"])
            continue
        want = golden_groups(arr, f"{name}_g{g}")
        assert keys(out.seed_groups) == keys(want), (name, g)
        Cg = np.stack([c.values for c in out.clustering.centers])
        assert np.array_equal(Cg, arr[f"{name}_g{g}_centers"])
        assert np.array_equal(out.clustering.assignment, arr[f"{name}_g{g}_labels"])
        assert np.array_equal(out.clustering.radii, arr[f"{name}_g{g}_radii"])
        assert out.clustering.objective == m["runs"][g]["objective"]
        assert out.k_star == m["runs"][g]["k_star"]


def test_worked_pipeline():
    cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(1),
                           homo=G.HomoTransformParams(4, 2, directions=np.eye(4)),
                           seeding=G.SeedingParams(2, 2, min_group_size=1, seed=0, table_seeds=((52, 3), (15, 63)),
                                                   dedup_seeds=((0, 1001),)))
    out = G.run_pipeline(G.DenseData(WORKED_POINTS), cfg)
    assert keys(out.seed_groups) == [(0, 1, 3), (2, 4), (2, 4, 5), (5,)]
    assert out.k_star == 3 and len(out.clustering.empty_clusters) == 1


def test_fallback_warns():
    rng = np.random.default_rng(9)
    cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(2),
                           homo=G.HomoTransformParams(4, 32, seed=1),
                           seeding=G.SeedingParams(3, 4, min_group_size=50, seed=2))
    X = rng.standard_normal((64, 4))
    out = G.run_pipeline(G.DenseData(X), cfg)
    ref = O.pipeline_dense(X, 4, 32, 1, 3, 4, 50, 2, g=2)
    assert out.warnings and ref["warnings"]
    assert keys(out.seed_groups) == keys(ref["groups"])


@pytest.mark.parametrize("g", [1, 2])
def test_sparse_pipeline_golden(g):
    m = meta()["sparse"]
    arr = npz("pipelines")
    sets = csr(arr["sp_flat"], arr["sp_off"])
    data = G.SparseData(sets, 20_000)
    mp = G.MinhashTransformParams(3, 6, seed=4, target_dims=400)
    bt, red = G.transform_sparse(data, mp)
    assert np.array_equal(bt.codes_host(), arr["sp_codes"])
    cfg = G.PipelineConfig(metric="jaccard", transform_kind="sparse", workers=G.WorkerConfig(g), minhash=mp,
                           seeding=G.SeedingParams(3, 6, min_group_size=3, seed=5))
    out = G.run_pipeline(data, cfg)
    assert keys(out.seed_groups) == keys(golden_groups(arr, f"sp_g{g}"))
    assert np.array_equal(np.stack([c.values for c in out.clustering.centers]), arr[f"sp_g{g}_centers"])
    assert np.array_equal(out.clustering.assignment, arr[f"sp_g{g}_labels"])
    assert np.array_equal(out.clustering.radii, arr[f"sp_g{g}_radii"])
    assert out.clustering.objective == m["runs"][str(g)]["objective"]


@pytest.mark.parametrize("g", [1, 2])
def test_mixed_pipeline_golden(g):
    m = meta()["mixed"]
    arr = npz("pipelines")
    data = G.MixedData(arr["mx_num"], arr["mx_cat"])
    mp = G.MinhashTransformParams(3, 6, seed=7, bins_per_attribute=16)
    bt, unified = G.transform_hetero(data, mp)
    assert np.array_equal(unified.codes, arr["mx_unified"])
    assert np.array_equal(bt.codes_host(), arr["mx_codes"])
    cfg = G.PipelineConfig(metric="jaccard", transform_kind="mixed", workers=G.WorkerConfig(g), minhash=mp,
                           seeding=G.SeedingParams(3, 6, min_group_size=3, seed=9))
    out = G.run_pipeline(data, cfg)
    assert keys(out.seed_groups) == keys(golden_groups(arr, f"mx_g{g}"))
    assert np.array_equal(np.stack([c.values for c in out.clustering.centers]), arr[f"mx_g{g}_centers"])
    assert np.array_equal(out.clustering.assignment, arr[f"mx_g{g}_labels"])
    assert np.array_equal(out.clustering.radii, arr[f"mx_g{g}_radii"])
    assert out.clustering.objective == m["runs"][str(g)]["objective"]


@pytest.mark.parametrize("singletons", [True, False])
@pytest.mark.parametrize("kind", ["sparse", "mixed"])
def test_signature_bins_table_by_table(kind, singletons, monkeypatch):
    """Large signature-bucket sets form their SILK bins one table at a time
    (memory), singleton buckets by lookup; forced here on the golden sparse /
    mixed pipelines: same output."""
    monkeypatch.setattr(G.seeding, "_SPLIT_ROWS", 0)
    monkeypatch.setattr(G.seeding, "_SINGLETON_BINS", singletons)
    arr = npz("pipelines")
    if kind == "sparse":
        m = meta()["sparse"]
        data = G.SparseData(csr(arr["sp_flat"], arr["sp_off"]), 20_000)
        cfg = G.PipelineConfig(metric="jaccard", transform_kind="sparse", workers=G.WorkerConfig(2),
                               minhash=G.MinhashTransformParams(3, 6, seed=4, target_dims=400),
                               seeding=G.SeedingParams(3, 6, min_group_size=3, seed=5))
        pre = "sp_g2"
    else:
        m = meta()["mixed"]
        data = G.MixedData(arr["mx_num"], arr["mx_cat"])
        cfg = G.PipelineConfig(metric="jaccard", transform_kind="mixed", workers=G.WorkerConfig(2),
                               minhash=G.MinhashTransformParams(3, 6, seed=7, bins_per_attribute=16),
                               seeding=G.SeedingParams(3, 6, min_group_size=3, seed=9))
        pre = "mx_g2"
    out = G.run_pipeline(data, cfg)
    assert keys(out.seed_groups) == keys(golden_groups(arr, pre))
    assert np.array_equal(out.clustering.assignment, arr[pre + "_labels"])
    assert out.clustering.objective == m["runs"]["2"]["objective"]


@pytest.mark.parametrize("K,G_,delta", [(1, 3, 2), (2, 1, 2), (1, 1, 3), (3, 8, 2)])
def test_singleton_bins_equal_group_by(K, G_, delta):
    """Bins with singleton buckets joined by pi_1^-1 lookup equal the full
    group-by + exact pruning, bucket lists and order included; small
    universes and K = 1 make singletons join larger buckets often."""
    from paper_2106_10515_b200.tables import BucketTable
    rng = np.random.default_rng(K * 100 + G_ * 10 + delta)
    n, m = 3000, 12
    tsizes = [int(x) for x in rng.integers(1200, 2600, m)]
    codes = np.stack([rng.integers(0, t, n) for t in tsizes], axis=1)
    for j, t in enumerate(tsizes):  # every slot non-empty
        codes[rng.permutation(n)[:t], j] = np.arange(t)
    bt = BucketTable(torch.from_numpy(codes.astype(np.int32)).cuda(), n, tsizes, "sig", False)
    owner = torch.from_numpy(np.concatenate([np.full(t, j % G_) for j, t in enumerate(tsizes)]).astype(np.int32)).cuda()
    sp = G.SeedingParams(K, 5, min_group_size=delta, seed=11)
    scheme = sp.scheme(n)
    a, _ = G.seeding._bins_per_table(bt, scheme, K, 5, n, owner, delta)
    b, _ = G.seeding._bins_per_table_singletons(bt, scheme, K, 5, n, owner, delta)
    sizes = bt.bucket_sizes()
    assert int((sizes == 1).sum()) > 1000
    assert a.count > 0 and a.count == b.count
    for f in ("pair_bucket", "pair_bin", "bin_size", "bin_table", "bin_sig"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    # some kept bins do mix singletons with larger buckets
    assert bool((sizes[b.pair_bucket] == 1).any())


def _key_values(k):
    """float64 values of f64_key's order-preserving uint64 keys (common.cuh)."""
    u = k.astype(np.uint64)
    neg = (u & np.uint64(1 << 63)) == 0
    b = np.where(neg, ~u, u & np.uint64((1 << 63) - 1))
    return b.view(np.float64)


def _exact_dot_err(X, A, V, rows):
    """|V - exact X @ A.T| for the sampled rows, with exact rational sums."""
    from fractions import Fraction
    out = np.zeros((len(rows), A.shape[0]))
    for r, i in enumerate(rows):
        xs = [Fraction(float(v)) for v in X[i]]
        for j in range(A.shape[0]):
            ex = sum(x * Fraction(float(a)) for x, a in zip(xs, A[j]))
            out[r, j] = abs(float(Fraction(float(V[j, i])) - ex)) if np.isfinite(V[j, i]) else 0.0
    return out


@pytest.mark.parametrize("n,d,m,case", [(1000, 128, 40, "gauss"), (777, 4, 3, "gauss"), (3001, 36, 20, "tiny"),
                                        (2048, 100, 8, "wide"), (513, 64, 48, "gauss"), (300, 128, 1, "special"),
                                        (5000, 128, 48, "gauss")])
def test_tc_projection_keys(n, d, m, case, monkeypatch):
    """K1 on kind::i8 tcgen05 MMAs (tc_project.cu, the default): every key within the
    float64 order bound (gamma_d 2^xmax |a|_1) of the exact dot product --
    checked with rational arithmetic on sampled rows -- so within
    projection_tolerance of numpy's BLAS keys and of the DMMA kernel's; the
    exponent window equals the DMMA pass's.  Cases: Gaussian rows, rows with
    elements 2^16..2^30 below their maximum (the remainder path), rows
    spanning many binades, and special rows (zeros, subnormal, huge, inf)."""
    from paper_2106_10515_b200 import transform as T
    rng = np.random.default_rng(n * 7 + d)
    X = rng.standard_normal((n, d)).astype(np.float32)
    if case == "tiny":
        mask = rng.random((n, d)) < 0.05
        X[mask] *= np.float32(2.0) ** -rng.integers(16, 30, mask.sum()).astype(np.float32)
    elif case == "wide":
        X *= (np.float32(2.0) ** rng.integers(-20, 20, (n, 1))).astype(np.float32)
        X[:, ::7] *= np.float32(1e-6)
    elif case == "special":
        X[0] = 0
        X[1] = np.float32(1e-42)
        X[2, 5] = np.float32(2.0 ** 60)
        X[3, 7] = np.inf
        X[4] *= np.float32(2.0 ** -100)
    A = O.directions(5, m, d)
    Xd = torch.from_numpy(X).cuda()

    def run():
        er = torch.tensor([2 ** 30, -2 ** 30], dtype=torch.int32, device="cuda")
        k = T.project_keys(Xd, A, er).cpu().numpy()
        return _key_values(k), er.cpu().numpy()

    V, er = run()  # K1 on tcgen05 (the default)
    monkeypatch.setenv("GEEK_TCPROJ", "0")
    Vd, erd = run()  # K1 on DMMA
    assert np.array_equal(er, erd)
    fin = np.isfinite(X).all(1)
    xmax = int(np.frexp(np.abs(X[fin]).max())[1])
    tol = T.projection_tolerance(A, xmax)[:, None]
    with np.errstate(invalid="ignore", over="ignore"):
        ref = (X[fin].astype(np.float64) @ A.T).T
    assert (np.abs(V[:, fin] - ref) <= tol).all()
    assert (np.abs(V[:, fin] - Vd[:, fin]) <= tol).all()
    assert np.array_equal(np.isnan(V[:, ~fin]), np.isnan(Vd[:, ~fin]))
    rows = [i for i in np.linspace(0, n - 1, 12).astype(int) if fin[i]]
    err = _exact_dot_err(X, A, V, rows)
    assert (err <= tol.T / 2).all(), (err / (tol.T / 2)).max()


@pytest.mark.parametrize("owners", [2, 3, 8])
def test_routed_projection_layout(owners):
    """geek_project_keys_routed (the fused bucket synchronisation) writes the
    same keys as geek_project_keys, table j of rows [lo, hi) at owner j % G,
    row (j / G), columns lo..hi of an ntot-row array -- checked on one GPU
    with ordinary device buffers standing in for the owners' peer mappings."""
    from paper_2106_10515_b200 import _lib
    from paper_2106_10515_b200.transform import project_keys
    rng = np.random.default_rng(owners)
    ntot, lo, hi, d, m = 5003, 1201, 4090, 32, 21
    X = rng.standard_normal((ntot, d)).astype(np.float32)
    A = rng.standard_normal((m, d))
    ref = project_keys(_lib.to_dev(X), A).cpu().numpy()
    bufs = [torch.full((-(-m // owners), ntot), -1, dtype=torch.int64, device="cuda") for _ in range(owners)]
    ptrs = np.array([b.data_ptr() for b in bufs], dtype=np.uint64)
    er = torch.tensor([1 << 30, -(1 << 30)], dtype=torch.int32, device="cuda")
    Xs = _lib.to_dev(X[lo:hi])
    _lib.call("geek_project_keys_routed", _lib.ptr(Xs), 0, hi - lo, d, _lib.ptr(_lib.to_dev(A)), m, _lib.hptr(ptrs),
              owners, ntot, lo, _lib.ptr(er), None, 0, None, _lib.stream())
    torch.cuda.synchronize()
    for j in range(m):
        got = bufs[j % owners][j // owners].cpu().numpy()
        assert np.array_equal(got[lo:hi], ref[j, lo:hi]), j
        assert (got[:lo] == -1).all() and (got[hi:] == -1).all(), j
    O_lo, O_hi = [], []  # exp_window of every nonzero value (project.cu)
    for v in X[lo:hi].ravel():
        if v != 0:
            e = (int(np.float32(v).view(np.uint32)) >> 23) & 0xFF
            O_lo.append(e - 150 if e else -172)
            O_hi.append(e - 126 if e else -148)
    want = np.array([min(O_lo), max(O_hi)], dtype=np.int32)
    assert np.array_equal(er.cpu().numpy(), want)


@pytest.mark.parametrize("n,t", [(50_000, 997), (120_000, 3), (7_000, 7_000)])
def test_counted_split_equals_split(n, t):
    """Fine-bin counts fused into the projection (geek_project_keys_routed with
    a layout from geek_fine_layout) + geek_rank_split_counted give the same
    bucket codes as the two-pass geek_rank_split on the same keys."""
    from paper_2106_10515_b200 import _lib
    from paper_2106_10515_b200.engine import _Comm, project_counted
    from paper_2106_10515_b200.transform import rank_split_codes
    rng = np.random.default_rng(n)
    d, m = 64, 9
    X = _lib.to_dev(rng.standard_normal((n, d)).astype(np.float32))
    X[: n // 10] = X[0]  # a block of identical points: ties broken by id
    A = rng.standard_normal((m, d))
    er = torch.tensor([1 << 30, -(1 << 30)], dtype=torch.int32, device="cuda")
    keys, (hist, fcnt) = project_counted(X, A, n, 0, _Comm(), er, list(range(m)))
    st = {}
    from paper_2106_10515_b200.engine import rank_split_counted
    got = rank_split_counted(keys, t, hist, fcnt, st).cpu().numpy()
    want = rank_split_codes(keys.contiguous(), t).cpu().numpy()
    assert np.array_equal(got, want)
    assert int(fcnt.sum().item()) == n * m


def test_host_rows_streamed_equal_device_rows():
    """run_pipeline_shard on pinned host rows (chunked H2D, each chunk projected
    as it lands) gives the same result as on device rows."""
    m = meta()["pipelines"]["cfg1"]
    _, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    X = X.astype(np.float32)
    cfg = dense_config(m, 1)
    dev = G.run_pipeline_shard(torch.from_numpy(X).cuda(), n, cfg)
    host = G.run_pipeline_shard(torch.from_numpy(X).pin_memory(), n, cfg)
    assert keys(dev.seed_groups) == keys(host.seed_groups)
    assert np.array_equal(dev.clustering.assignment, host.clustering.assignment)
    assert np.array_equal(dev.clustering.radii, host.clustering.radii)
    assert dev.clustering.objective == host.clustering.objective


# ---- refinement passes (assignment.py:157-170, engine.py:519-537) ----------

def _check_refined(cl, arr, rm, name):
    assert np.array_equal(np.stack([c.values for c in cl.centers]), arr[f"{name}_centers"]), name
    assert np.array_equal(np.array([c.weight for c in cl.centers]), arr[f"{name}_weights"]), name
    assert np.array_equal(cl.assignment, arr[f"{name}_labels"]), name
    assert np.array_equal(cl.radii, arr[f"{name}_radii"]), name
    assert cl.objective == rm[name]["objective"], name
    assert cl.k_star == rm[name]["k_star"], name


def test_refine_c08_golden():
    """geek_label_sums / geek_label_mode_counts + assignment against the
    reference's refine() outputs, bit for bit."""
    arr, rm = npz("refine"), refine_meta()
    rng = np.random.default_rng(80)
    dense = G.DenseData(rng.standard_normal((10_000, 16)))
    cents = [G.CentralVector("centroid", rng.standard_normal(16)) for _ in range(200)]
    c0 = G.assign(dense, cents, "euclidean")
    assert G.refine(dense, c0, "euclidean", 0) is c0
    for p in (1, 2):
        _check_refined(G.refine(dense, c0, "euclidean", p), arr, rm, f"c08_p{p}")
    codes = rng.integers(0, 8, (10_000, 9)).astype(np.int32)
    modes = [G.CentralVector("mode", rng.integers(0, 8, 9).astype(np.int32)) for _ in range(200)]
    cat = G.CategoricalData(codes, code_space=8)
    c0 = G.assign(cat, modes, "jaccard")
    _check_refined(G.refine(cat, c0, "jaccard", 2), arr, rm, "c08cat_p2")


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_refine_label_sums_ragged(dtype):
    """Label-keyed exact sums equal the member-list sums (geek_exact_sums) on
    shuffled labels, a float32 input, coordinates over many binades, d not a
    multiple of 32 and an empty cluster."""
    from paper_2106_10515_b200 import _lib, numeric
    from paper_2106_10515_b200.tables import GroupSet
    rng = np.random.default_rng(5)
    n, d, k = 4099, 45, 37
    X = (rng.standard_normal((n, d)) * np.exp2(rng.integers(-30, 30, (n, d)))).astype(dtype)
    X[rng.random((n, d)) < 0.05] = 0.0
    lab = rng.integers(0, k, n)
    lab[lab == 7] = 8  # cluster 7 empty
    Xd = _lib.to_dev(X)
    emin, emax = numeric.exponent_range(Xd)
    nd = numeric.digit_count(emin, emax)
    labd = _lib.to_dev(lab.astype(np.int64))
    got = numeric.label_sums(Xd, labd, k, emin, nd)  # short runs: label-sorted row order
    want = numeric.partial_sums(Xd, GroupSet.from_host([np.flatnonzero(lab == j) for j in range(k)]), emin, nd)
    storage = numeric.label_sums(Xd, labd, k, emin, nd, order=torch.arange(n, device=labd.device))
    C0 = numeric.round_means(storage, torch.bincount(labd, minlength=k), emin, nd).cpu().numpy()
    C1 = numeric.round_means(got, torch.bincount(_lib.to_dev(lab), minlength=k), emin, nd).cpu().numpy()
    C2 = numeric.round_means(want, torch.bincount(_lib.to_dev(lab), minlength=k), emin, nd).cpu().numpy()
    assert np.array_equal(C1, C2) and np.array_equal(C0, C2)
    for j in (0, 13, 36):
        assert np.array_equal(C1[j], O.exact_mean(X[lab == j].astype(np.float64)))


@pytest.mark.parametrize("g", [1, 2])
def test_refine_pipeline_golden(g):
    m = meta()["pipelines"]["small"]
    arr, rm = npz("refine"), refine_meta()
    _, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    cfg = dense_config(m, g)
    cfg.passes = 2
    for x in (X, X.astype(np.float32)):
        out = G.run_pipeline(G.DenseData(x), cfg)
        if x.dtype == np.float32:  # different data: the oracle on the f32 values
            ref = O.pipeline_dense(x.astype(np.float64), m["m"], m["t"], m["tseed"], m["K"], m["L"], m["delta"],
                                   m["sseed"], g=g, passes=2)
            assert np.array_equal(out.clustering.assignment, ref["labels"])
            assert np.array_equal(np.stack([c.values for c in out.clustering.centers]), ref["centers"])
            assert out.clustering.objective == ref["objective"]
        else:
            _check_refined(out.clustering, arr, rm, f"small_p2_g{g}")


def test_refine_pipeline_c06_sparse_mixed_golden():
    arr, rm = npz("refine"), refine_meta()
    m = meta()["pipelines"]["c06"]
    _, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    cfg = dense_config(m, 1)
    cfg.passes = 3
    _check_refined(G.run_pipeline(G.DenseData(X), cfg).clustering, arr, rm, "c06_p3_g1")
    parr = npz("pipelines")
    data = G.SparseData(csr(parr["sp_flat"], parr["sp_off"]), 20_000)
    cfg = G.PipelineConfig(metric="jaccard", transform_kind="sparse", workers=G.WorkerConfig(1),
                           minhash=G.MinhashTransformParams(3, 6, seed=4, target_dims=400),
                           seeding=G.SeedingParams(3, 6, min_group_size=3, seed=5), passes=2)
    _check_refined(G.run_pipeline(data, cfg).clustering, arr, rm, "sp_p2_g1")
    data = G.MixedData(parr["mx_num"], parr["mx_cat"])
    cfg = G.PipelineConfig(metric="jaccard", transform_kind="mixed", workers=G.WorkerConfig(1),
                           minhash=G.MinhashTransformParams(3, 6, seed=7, bins_per_attribute=16),
                           seeding=G.SeedingParams(3, 6, min_group_size=3, seed=9), passes=2)
    _check_refined(G.run_pipeline(data, cfg).clustering, arr, rm, "mx_p2_g1")


# ---- vector-file ingestion (io.py:21-62) ------------------------------------

@pytest.mark.parametrize("ext", ["fvecs", "bvecs"])
def test_read_vecs_golden_and_errors(ext, tmp_path):
    from paper_2106_10515_b200.io import FormatError, read_fvecs
    from tests.golden_io import GOLDEN
    import os
    got = read_fvecs(os.path.join(GOLDEN, f"io_small.{ext}"))
    assert got.vectors.is_cuda and got.vectors.dtype == torch.float32
    assert np.array_equal(got.host_f64(), npz("io")[ext])
    # many chunks (a few records each), errors past the first chunk
    rng = np.random.default_rng(3)
    n, d = 1001, 13
    elem, dt = (1, "<u1") if ext == "bvecs" else (4, "<f4")
    body = (rng.integers(0, 256, (n, d)) if ext == "bvecs" else rng.standard_normal((n, d))).astype(dt)
    rec = np.empty((n, 4 + d * elem), np.uint8)
    rec[:, :4] = np.frombuffer(np.int32(d).tobytes(), np.uint8)
    rec[:, 4:] = body.view(np.uint8).reshape(n, -1)
    cases = {"ok": rec.tobytes(), "trunc": rec.tobytes()[:-3], "short": b"\x01\x00",
             "nonpos": np.int32(-2).tobytes() + rec.tobytes()[4:], "empty": b""}
    bad = rec.copy()
    bad[777, :4] = np.frombuffer(np.int32(d + 1).tobytes(), np.uint8)
    bad[901, :4] = 0
    cases["inconsistent"] = bad.tobytes()
    for name, raw in cases.items():
        p = tmp_path / f"{name}.{ext}"
        p.write_bytes(raw)
        want = O.read_vecs(raw, ext == "bvecs")
        if isinstance(want, str):
            with pytest.raises(FormatError, match=want):
                read_fvecs(p, chunk_bytes=40 * (4 + d * elem))
        else:
            out = read_fvecs(p, chunk_bytes=40 * (4 + d * elem))
            assert out.n == want.shape[0]
            if want.size:
                assert np.array_equal(out.host_f64(), want)


# ---- comparison methods (baselines.py:34-136) -------------------------------

def test_baselines_golden():
    from paper_2106_10515_b200 import baselines as B
    arr, bm = npz("baselines"), baselines_meta()
    X, _ = O.gaussian_mixture(2000, 16, 10, 6.0, 5)
    dense = G.DenseData(X)
    rng = np.random.default_rng(12)
    cat = G.CategoricalData(rng.integers(0, 5, (1500, 7)).astype(np.int32), code_space=5)
    sp = G.SparseData(csr(arr["sp_flat"], arr["sp_off"]), bm["sp_universe"])

    def vals(cs):
        return np.stack([c.values for c in cs])

    assert np.array_equal(vals(B.seed_random(dense, 12, 3)), arr["rand_dense"])
    assert np.array_equal(vals(B.seed_kmeanspp(dense, 12, 4)), arr["pp_dense"])
    assert np.array_equal(vals(B.seed_kmeanspp(cat, 9, 5, metric="jaccard")), arr["pp_cat"])
    assert np.array_equal(vals(B.seed_kmeanspp(sp, 7, 6, metric="jaccard")), arr["pp_sparse"])
    for name, cl in (("lloyd", B.lloyd(dense, 12, 7)), ("lloyd_2it", B.lloyd(dense, 12, 7, max_iters=2)),
                     ("kmodes_cat", B.kmodes(cat, 9, 8)), ("kmodes_sparse", B.kmodes(sp, 7, 9))):
        assert np.array_equal(vals(cl.centers), arr[f"{name}_centers"]), name
        assert np.array_equal(cl.assignment, arr[f"{name}_labels"]), name
        assert np.array_equal(cl.radii, arr[f"{name}_radii"]), name
        assert cl.objective == bm[name]["objective"], name
    with pytest.raises(G.InvalidInput):
        B.seed_random(dense, 2001, 0)
    with pytest.raises(G.InvalidInput):
        B.kmodes(dense, 3, 0)


# ---- LSHC v1 artifacts (serialize.py:129-198) --------------------------------

def test_artifacts_byte_identical():
    """dump_buckets of a device BucketTable (geek_pack_buckets), seed groups
    and clustering of the 'small' case equal the reference's files byte for
    byte (sha256 in tests/golden/artifacts.json)."""
    import hashlib
    import json
    import os
    from tests.golden_io import GOLDEN
    from paper_2106_10515_b200 import serialize as S
    want = json.load(open(os.path.join(GOLDEN, "artifacts.json")))
    m = meta()["pipelines"]["small"]
    _, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    bt = G.transform_homo(G.DenseData(X), G.HomoTransformParams(8, 30, seed=1))
    raw = S.dump_buckets(bt)
    assert hashlib.sha256(raw).hexdigest() == want["small_buckets"]["sha256"]
    assert raw == S.dump_buckets(list(bt))  # device packing == host packing
    back = S.load_buckets(raw)
    assert [(b.table, b.slot) for b in back] == [(b.table, b.slot) for b in bt]
    out = G.run_pipeline(G.DenseData(X), dense_config(m, 2))
    assert hashlib.sha256(S.dump_seed_groups(out.seed_groups)).hexdigest() == want["small_groups"]["sha256"]
    assert hashlib.sha256(S.dump_clustering(out.clustering)).hexdigest() == want["small_clustering"]["sha256"]


@pytest.mark.parametrize("u,k", [(20, 7), (400, 300), (1000, 33), (2000, 9)])
def test_assign_sparse_bitsets_vs_oracle(u, k):
    """Jaccard assignment of sparse sets: bitset kernel (u <= 1024) and the
    dense-mode kernel above it, against the oracle's float64 formula; empty
    and duplicate modes, exact-tie similarities."""
    rng = np.random.default_rng(u + k)
    sets = [np.unique(rng.integers(0, u, rng.integers(1, min(u, 60)))) for _ in range(3001)]
    M = (rng.random((k, u)) < 0.08).astype(np.int32)
    M[0] = 0
    M[k - 1] = M[1]
    data = G.SparseData(sets, u)
    got = G.assign(data, [G.CentralVector("mode", m) for m in M], "jaccard")
    lab, best, radii, obj = O.assign_generic(lambda a, b: O.sparse_distances(sets[a:b], u, M), len(sets), k)
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj


@pytest.mark.parametrize("d,k,n", [(1, 3, 500), (7, 1, 300), (13, 300, 1031), (39, 513, 2000),
                                   (41, 257, 777), (64, 70, 900), (65, 40, 300)])
def test_assign_categorical_vs_oracle(d, k, n):
    """Categorical assignment: the register-tiled kernel (d <= 64: ragged d,
    center chunks of 256, partial point tiles) and the per-thread kernel
    (d > 64) against the oracle's 1 - m / (2d - m) argmin; duplicate modes and
    many exact ties (small code space) pin the first-index rule."""
    rng = np.random.default_rng(d * 1000 + k)
    codes = rng.integers(0, 3, (n, d)).astype(np.int32)
    codes[:, ::3] = rng.integers(0, 40, (n, (d + 2) // 3))
    M = rng.integers(0, 3, (k, d)).astype(np.int32)
    M[k - 1] = M[0]
    M[k // 2] = codes[0]
    data = G.CategoricalData(codes, 64)
    got = G.assign(data, [G.CentralVector("mode", m) for m in M], "jaccard")
    lab, best, radii, obj = O.assign_generic(lambda a, b: O.cat_distances(codes[a:b], M), n, k)
    assert np.array_equal(got.assignment, lab)
    assert np.array_equal(got.radii, radii)
    assert got.objective == obj


def test_sparse_mode_centers_match_dense_counts():
    """Large-code-space modes (sort + run-length, no [k, d, code_space] table)
    equal the dense-count argmax, ties to the smallest code."""
    from paper_2106_10515_b200 import _lib, numeric
    from paper_2106_10515_b200.tables import GroupSet
    rng = np.random.default_rng(9)
    codes = rng.integers(0, 6, (5000, 7)).astype(np.int32)
    groups = GroupSet.from_host([np.sort(rng.choice(5000, rng.integers(1, 40), replace=False)) for _ in range(300)])
    cd = _lib.to_dev(codes, torch.int32)
    dense = torch.argmax(numeric.mode_counts(cd, 6, groups), dim=2).to(torch.int32)
    sparse = numeric.sparse_mode_centers(cd, 6, groups.flat, groups.off)
    assert torch.equal(dense, sparse)


def test_batched_votes_match_single_pass(monkeypatch):
    """Votes over bin-id batches (bounded pair memory) give the same seed
    groups and results as one pass (sparse and mixed golden pipelines)."""
    from paper_2106_10515_b200 import seeding
    monkeypatch.setattr(seeding, "_PAIR_BATCH", 64)
    arr = npz("pipelines")
    data = G.SparseData(csr(arr["sp_flat"], arr["sp_off"]), 20_000)
    cfg = G.PipelineConfig(metric="jaccard", transform_kind="sparse", workers=G.WorkerConfig(2),
                           minhash=G.MinhashTransformParams(3, 6, seed=4, target_dims=400),
                           seeding=G.SeedingParams(3, 6, min_group_size=3, seed=5))
    out = G.run_pipeline(data, cfg)
    assert keys(out.seed_groups) == keys(golden_groups(arr, "sp_g2"))
    assert np.array_equal(out.clustering.assignment, arr["sp_g2_labels"])
    data = G.MixedData(arr["mx_num"], arr["mx_cat"])
    cfg = G.PipelineConfig(metric="jaccard", transform_kind="mixed", workers=G.WorkerConfig(1),
                           minhash=G.MinhashTransformParams(3, 6, seed=7, bins_per_attribute=16),
                           seeding=G.SeedingParams(3, 6, min_group_size=3, seed=9))
    out = G.run_pipeline(data, cfg)
    assert keys(out.seed_groups) == keys(golden_groups(arr, "mx_g1"))
    assert np.array_equal(out.clustering.assignment, arr["mx_g1_labels"])


def test_label_mode_centers_sort_path(monkeypatch):
    """Refinement modes for code spaces too large for dense counts (sort
    path) equal the dense label-keyed counts."""
    from paper_2106_10515_b200 import _lib, numeric
    rng = np.random.default_rng(4)
    codes = _lib.to_dev(rng.integers(0, 5, (4000, 6)).astype(np.int32), torch.int32)
    labels = _lib.to_dev(rng.integers(0, 40, 4000).astype(np.int64))
    labels[labels == 7] = 8
    keep = torch.nonzero(torch.bincount(labels, minlength=40) > 0).flatten()
    dense = numeric.label_mode_centers(codes, 5, labels, 40, keep)
    monkeypatch.setattr(numeric, "_DENSE_MODE_LIMIT", 0)
    assert torch.equal(numeric.label_mode_centers(codes, 5, labels, 40, keep), dense)
