"""CPU-only checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/geek.h declares, the package imports, host
logic (seed derivation, splits, parameter validation) matches the oracle, and
compute calls fail loudly without a GPU (there is no CPU fallback)."""

import os
import re

import numpy as np
import pytest
import torch

from oracle import geek_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "geek.h")).read()
    return sorted(set(re.findall(r"\b(geek_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2106_10515_b200 import _lib

    L = _lib.load_library()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_lib._SIGS)  # every entry point is bound with a signature
    assert L.geek_version() == 1


def test_package_api_surface_matches_reference_names():
    import paper_2106_10515_b200 as G

    ref_names = ["Bucket", "Bin", "CategoricalData", "CentralVector", "Clustering", "DenseData", "InvalidInput",
                 "MixedData", "SeedGroup", "SparseData", "dist_euclidean", "dist_jaccard", "categorical_tokens",
                 "DophReducer", "MinHashFunction", "ProjectionFunction", "SignatureScheme", "HomoTransformParams",
                 "MinhashTransformParams", "discretize_numeric", "transform_hetero", "transform_homo",
                 "transform_sparse", "SeedingParams", "bin_buckets", "dedup_groups", "find_seed_groups",
                 "majority_vote", "seeds_to_centers", "assign", "refine"]  # lshclust/__init__.py:31-69
    for n in ref_names:
        assert hasattr(G, n), n
    for n in ("PipelineConfig", "WorkerConfig", "run_pipeline", "split_data", "EngineError"):
        assert hasattr(G, n)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_compute_without_gpu_fails_loudly():
    import paper_2106_10515_b200 as G

    with pytest.raises(G.EngineError):
        G.transform_homo(G.DenseData(np.zeros((4, 2))), G.HomoTransformParams(1, 2))
    with pytest.raises(G.EngineError):
        G.MinHashFunction(1, 10_000)([1, 2, 3])


def test_host_seed_derivation_matches_oracle():
    from paper_2106_10515_b200.hashing import MinHashFunction, derive_seed, splitmix64, _mulinv

    for z in (0, 1, 2**63, 2**64 - 1):
        assert splitmix64(z) == O.mix64(z)
    for m, p in [(0, ()), (5, (1, 2)), (2**64 - 1, (0xDED0,))]:
        assert derive_seed(m, *p) == O.sub_seed(m, *p)
    for u in (5000, 100_000, 10**8, 3 * 10**9):
        f = MinHashFunction(17, u)
        w, mask, c1, c2, a1, s1, s2 = f.params
        assert (w, mask, c1, c2, a1, s1, s2) == O.perm_params(17, u)
        assert (c1 * _mulinv(c1, w)) & mask == 1 and (c2 * _mulinv(c2, w)) & mask == 1
    tab = MinHashFunction(3, 100).table
    assert np.array_equal(tab, O.rank_table(3, 100))


def test_split_and_validation():
    import paper_2106_10515_b200 as G

    assert G.split_data(10, 2) == [(0, 5), (5, 10)]
    assert [hi - lo for lo, hi in G.split_data(7, 3)] == [3, 2, 2]
    with pytest.raises(G.InvalidInput):
        G.split_data(2, 3)
    with pytest.raises(G.InvalidInput):
        G.HomoTransformParams(1, 1)
    with pytest.raises(G.InvalidInput):
        G.SeedingParams(0, 1)
    with pytest.raises(G.InvalidInput):
        G.WorkerConfig(0)
    assert G.transform.even_partition_sizes(7, 2).tolist() == [4, 3]
    with pytest.raises(G.InvalidInput):
        G.Bucket(0, 0, np.array([], dtype=np.int64))
    c = G.Clustering(centers=[1, 2], assignment=np.array([0, 0]), radii=np.zeros(2), objective=0.0)
    assert c.k_star == 1 and c.empty_clusters.tolist() == [1]


def test_digit_count_bounds():
    from paper_2106_10515_b200.numeric import digit_count

    assert digit_count(-40, 10) >= 3
    # float32 full exponent range still fits the widest digit choice
    assert digit_count(-149 - 24, 128) <= 40
