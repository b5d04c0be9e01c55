"""Pin the CPU oracle (oracle/geek_oracle.py) against golden vectors dumped
from the reference itself (tests/golden/make_golden.py) and against the
reference's own known-answer tests (pkg/tests/conftest.py, test_*.py)."""

import numpy as np
import pytest

from oracle import geek_oracle as O
from tests.golden_io import baselines_meta, csr, groups, meta, npz, refine_meta

WORKED = [  # pkg/tests/conftest.py:23-41
    (0, 0, [0, 1, 3]), (0, 1, [2, 4, 5]), (1, 0, [0, 1, 3, 4]), (1, 1, [5]),
    (2, 0, [0, 1, 3, 5]), (2, 1, [2, 4]), (3, 0, [0, 1, 3, 5]), (3, 1, [4, 5]),
]
WORKED_SEEDS = dict(pinned=((6, 7), (15, 20)), dedup_pinned=((0, 1001),))  # conftest.py:44-54
WORKED_POINTS = np.array([  # conftest.py:61-70
    [0.0, 0.0, 0.0, 0.0], [0.1, 0.1, 0.1, 0.1], [10.0, 0.2, 10.0, 0.3],
    [0.2, 0.3, 0.2, 0.4], [10.1, 0.4, 10.1, 0.5], [12.0, 0.5, 12.0, 0.2]])


def keys(gs):
    return [tuple(np.asarray(g).tolist()) for g in gs]


def test_seeds_golden():
    m = meta()["seeds"]
    for master, path, want in m["derive"]:
        assert O.sub_seed(master, *path) == want
    for z, want in m["splitmix"]:
        assert O.mix64(z) == want


def test_permutation_golden():
    arr = npz("pi")
    for seed, u, key in meta()["pi_cases"]:
        x, y = arr[key + "_x"], arr[key + "_y"]
        assert np.array_equal(O.permute(seed, u, x), y), key


def test_signatures_golden():
    arr = npz("sigs")
    for K, L, u, seed in [(3, 4, 700, 13), (2, 3, 5000, 1), (3, 2, 100_000, 2)]:
        p = f"{K}_{L}_{u}_{seed}"
        sets = csr(arr[p + "_flat"], arr[p + "_off"])
        for tb in range(L):
            got = O.set_signatures(O.table_function_seeds(seed, tb, K), u, sets)
            assert np.array_equal(got, arr[f"{p}_{tb}"])


def test_directions_golden():
    arr = npz("dirs")
    for key in arr.files:
        s, j, d = (int(v) for v in key.split("_"))
        assert np.array_equal(O.direction(s, j, d), arr[key])


def test_doph_golden():
    assert O.doph_sketch(np.array([0, 5]), 5, 12, 4).tolist() == meta()["doph_sketch_5_12_4"]
    arr = npz("doph")
    sets = csr(arr["flat"], arr["off"])
    got = O.doph_reduce(sets, O.sub_seed(3, 0xD0), 3_000_000, 400)
    want = csr(arr["red_flat"], arr["red_off"])
    assert all(np.array_equal(a, b) for a, b in zip(got, want))


def test_worked_example_known_answers():
    sets = [np.array(m) for _, _, m in WORKED]
    # bins of table 0 (test_seeding.py:44-51)
    bins = O.bins_for_table(sets, 2, 2, 0, 0, 6, WORKED_SEEDS["pinned"])
    got = {tuple((WORKED[i][0], WORKED[i][1]) for i in pos) for _, pos in bins}
    assert got == {((0, 0), (1, 0), (2, 0), (3, 0)), ((0, 1), (2, 1), (3, 1))}
    # full seeding (test_seeding.py:101-103)
    g = O.seed_groups(sets, 2, 2, 1, 0, 6, 1, WORKED_SEEDS["pinned"], WORKED_SEEDS["dedup_pinned"])
    assert keys(g) == [(0, 1, 3), (2, 4), (2, 4, 5), (5,)]
    # local-vote variant (test_engine.py:144-168)
    w0 = O.local_votes([b for b in WORKED if b[0] % 2 == 0], 2, 2, 1, 0, 6, WORKED_SEEDS["pinned"])
    w1 = O.local_votes([b for b in WORKED if b[0] % 2 == 1], 2, 2, 1, 0, 6, WORKED_SEEDS["pinned"])
    assert sorted(keys(w0)) == [(0, 1, 3), (2, 4), (2, 4)]
    merged = sorted(w0 + w1, key=lambda a: tuple(a.tolist()))
    fin = O.dedup(merged, 2, 0, 6, 1, WORKED_SEEDS["dedup_pinned"])
    assert keys(fin) == [(0, 1, 3), (2, 4), (5,)]


def test_worked_points_transform_and_pipeline():
    bk = O.homo_buckets(WORKED_POINTS, 4, 2, dirs=np.eye(4))  # test_transform.py:41-49
    got = {(j, s): m.tolist() for j, s, m in bk}
    assert got == {(0, 0): [0, 1, 3], (0, 1): [2, 4, 5], (1, 0): [0, 1, 2], (1, 1): [3, 4, 5],
                   (2, 0): [0, 1, 3], (2, 1): [2, 4, 5], (3, 0): [0, 1, 5], (3, 1): [2, 3, 4]}
    out = O.pipeline_dense(WORKED_POINTS, 4, 2, 0, 2, 2, 1, 0, g=1, dirs=np.eye(4),
                           pinned=((52, 3), (15, 63)), dedup_pinned=((0, 1001),))
    assert keys(out["groups"]) == [(0, 1, 3), (2, 4), (2, 4, 5), (5,)]  # test_engine.py:282-309
    assert int((np.bincount(out["labels"], minlength=4) > 0).sum()) == 3


def test_uneven_split_and_ties():
    X = np.arange(7, dtype=float).reshape(7, 1)  # test_transform.py:52-57
    bk = O.homo_buckets(X, 1, 2, dirs=np.ones((1, 1)))
    assert bk[0][2].tolist() == [0, 1, 2, 3]
    assert O.slot_codes(np.array([7.0, 7.0, 7.0, 7.0]), 2).tolist() == [0, 0, 1, 1]
    assert O.slot_codes(np.array([0.0, -0.0, 0.0, -0.0]), 2).tolist() == [0, 0, 1, 1]


def test_exact_centroid_known_answers():
    assert O.exact_mean(np.array([[0.0, 0.0], [2.0, 2.0]])).tolist() == [1.0, 1.0]
    assert O.exact_mean(np.array([[1.0, 1.0], [1.0, 1.0], [4.0, 4.0], [4.0, 4.0]])).tolist() == [2.5, 2.5]
    rows = np.array([[0.1], [0.2], [0.3]])
    assert O.exact_mean(rows)[0] == 0.2  # correctly rounded (0.1+0.2+0.3)/3


def test_assign_c08_golden():
    arr = npz("pipelines")
    rng = np.random.default_rng(80)
    X = rng.standard_normal((10_000, 16))
    C = np.stack([rng.standard_normal(16) for _ in range(200)])
    lab, best, radii, obj = O.assign_l2(X, C)
    assert np.array_equal(lab, arr["c08_labels"])
    assert np.array_equal(radii, arr["c08_radii"])
    assert obj == meta()["c08_objective"]


@pytest.mark.parametrize("name", ["c06", "small"])
def test_dense_pipeline_golden(name):
    m = meta()["pipelines"][name]
    arr = npz("pipelines")
    kind, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    import hashlib
    assert hashlib.sha256(X.tobytes()).hexdigest() == m["data_sha"]
    codes = np.stack([O.slot_codes(X @ O.direction(m["tseed"], j, d), m["t"]) for j in range(m["m"])])
    assert np.array_equal(codes, arr[name + "_codes"])
    for g in m["runs"]:
        out = O.pipeline_dense(X, m["m"], m["t"], m["tseed"], m["K"], m["L"], m["delta"], m["sseed"], g=int(g))
        want = groups(arr, f"{name}_g{g}")
        assert keys(out["groups"]) == keys(want)
        assert np.array_equal(out["centers"], arr[f"{name}_g{g}_centers"])
        assert np.array_equal(out["labels"], arr[f"{name}_g{g}_labels"])
        assert np.array_equal(out["radii"], arr[f"{name}_g{g}_radii"])
        assert out["objective"] == m["runs"][g]["objective"]


@pytest.mark.slow
def test_cfg1_pipeline_golden_g8():
    m = meta()["pipelines"]["cfg1"]
    arr = npz("pipelines")
    kind, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    out = O.pipeline_dense(X, m["m"], m["t"], m["tseed"], m["K"], m["L"], m["delta"], m["sseed"], g=8)
    assert keys(out["groups"]) == keys(groups(arr, "cfg1_g8"))
    assert np.array_equal(out["labels"], arr["cfg1_g8_labels"])
    assert np.array_equal(out["radii"], arr["cfg1_g8_radii"])


def test_refine_c08_golden():
    """refine(..., passes) on the c08 inputs (assignment.py:157-170) against
    the reference's own outputs (tests/golden/make_refine_golden.py)."""
    arr, rm = npz("refine"), refine_meta()
    rng = np.random.default_rng(80)
    X = rng.standard_normal((10_000, 16))
    C = np.stack([rng.standard_normal(16) for _ in range(200)])
    lab, _, _, _ = O.assign_l2(X, C)
    for p in (1, 2):
        out = O.refine_dense(X, lab, 200, p)
        assert np.array_equal(out["centers"], arr[f"c08_p{p}_centers"])
        assert np.array_equal(out["sizes"], arr[f"c08_p{p}_weights"])
        assert np.array_equal(out["labels"], arr[f"c08_p{p}_labels"])
        assert np.array_equal(out["radii"], arr[f"c08_p{p}_radii"])
        assert out["objective"] == rm[f"c08_p{p}"]["objective"]
    codes = rng.integers(0, 8, (10_000, 9)).astype(np.int32)
    modes = np.stack([rng.integers(0, 8, 9).astype(np.int32) for _ in range(200)])
    lab, *_ = O.assign_generic(lambda a, b: O.cat_distances(codes[a:b], modes), 10_000, 200)
    for _ in range(2):
        modes = O.modes_from_labels(codes, 8, lab, modes.shape[0])
        lab, _, radii, obj = O.assign_generic(lambda a, b: O.cat_distances(codes[a:b], modes), 10_000,
                                              modes.shape[0])
    assert np.array_equal(modes, arr["c08cat_p2_centers"])
    assert np.array_equal(lab, arr["c08cat_p2_labels"])
    assert np.array_equal(radii, arr["c08cat_p2_radii"])
    assert obj == rm["c08cat_p2"]["objective"]


def test_refine_pipeline_golden():
    """run_pipeline(passes=2) (engine.py:464-465, :519-537) at g = 1 and 2."""
    m = meta()["pipelines"]["small"]
    arr, rm = npz("refine"), refine_meta()
    _, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    for g in (1, 2):
        out = O.pipeline_dense(X, m["m"], m["t"], m["tseed"], m["K"], m["L"], m["delta"], m["sseed"], g=g, passes=2)
        assert np.array_equal(out["centers"], arr[f"small_p2_g{g}_centers"])
        assert np.array_equal(out["labels"], arr[f"small_p2_g{g}_labels"])
        assert np.array_equal(out["radii"], arr[f"small_p2_g{g}_radii"])
        assert out["objective"] == rm[f"small_p2_g{g}"]["objective"]


@pytest.mark.parametrize("ext", ["fvecs", "bvecs"])
def test_vector_files_golden(ext, tmp_path):
    """Oracle reader against the reference's read_fvecs output; the package's
    (host-side) writer is byte-identical to the reference's write_fvecs."""
    import os
    from tests.golden_io import GOLDEN
    arr = npz("io")
    path = os.path.join(GOLDEN, f"io_small.{ext}")
    raw = open(path, "rb").read()
    assert np.array_equal(O.read_vecs(raw, ext == "bvecs"), arr[ext])
    from paper_2106_10515_b200.io import write_fvecs
    from paper_2106_10515_b200.data import DenseData
    out = tmp_path / f"w.{ext}"
    write_fvecs(out, DenseData(arr["src"]))
    assert out.read_bytes() == raw


def test_baselines_dense_golden():
    """k-means++ picks and Lloyd (baselines.py:52-114) against the reference's outputs."""
    arr, bm = npz("baselines"), baselines_meta()
    X, _ = O.gaussian_mixture(2000, 16, 10, 6.0, 5)
    assert np.array_equal(X[O.seed_random_idx(2000, 12, 3)], arr["rand_dense"])
    assert np.array_equal(X[O.kmeanspp_idx(X, 12, 4)], arr["pp_dense"])
    for name, it in (("lloyd", 100), ("lloyd_2it", 2)):
        out = O.lloyd_dense(X, 12, 7, max_iters=it)
        assert np.array_equal(out["centers"], arr[f"{name}_centers"])
        assert np.array_equal(out["labels"], arr[f"{name}_labels"])
        assert np.array_equal(out["radii"], arr[f"{name}_radii"])
        assert out["objective"] == bm[name]["objective"]


def test_artifacts_reference_files_roundtrip():
    """LSHC v1 files written by the reference load with the package's readers
    and re-dump byte-identically (host-side packing; serialize.py:129-198)."""
    import os
    from tests.golden_io import GOLDEN
    from paper_2106_10515_b200 import serialize as S
    raw = {n: open(os.path.join(GOLDEN, f"art_{n}.lshc"), "rb").read() for n in ("buckets", "groups", "clustering")}
    bk = S.load_buckets(raw["buckets"])
    assert [(b.table, b.slot, b.members.tolist()) for b in bk] == [(t, s_, m) for t, s_, m in WORKED]
    assert S.dump_buckets(bk) == raw["buckets"]
    assert S.dump_seed_groups(S.load_seed_groups(raw["groups"])) == raw["groups"]
    cl = S.load_clustering(raw["clustering"])
    assert S.dump_clustering(cl) == raw["clustering"]
    with pytest.raises(S.FormatError, match="bad magic"):
        S.load_buckets(b"XXXX" + raw["buckets"][4:])
    with pytest.raises(S.FormatError, match="expected 1"):
        S.load_buckets(raw["groups"])
    with pytest.raises(S.FormatError, match="truncated"):
        S.load_buckets(raw["buckets"][:-5])
