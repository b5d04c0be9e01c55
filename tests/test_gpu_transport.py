"""Reference-facing engine bookkeeping on one GPU: the transport accounting of
the g logical workers (engine.py:79-104, serialize.py message bodies; the
reference's own tests read it, test_engine.py:348-356, acceptance c07) and
the memory-budget error (engine.py:359-366), against
tests/golden/transport.json dumped from the reference."""

import json
import os

import numpy as np
import pytest

from oracle import geek_oracle as O
from tests.golden_io import GOLDEN, csr, npz

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2106_10515_b200")


def _golden():
    with open(os.path.join(GOLDEN, "transport.json")) as f:
        return json.load(f)


DENSE = {"c06": ((2000, 16, 10, 20.0, 0), 48, 10, 48, 3, 5), "small": ((3000, 8, 6, 12.0, 4), 8, 30, 8, 3, 3)}


@pytest.mark.parametrize("name", ["c06", "small"])
@pytest.mark.parametrize("g,passes", [(1, 0), (2, 0), (4, 0), (8, 0), (2, 2), (8, 1)])
def test_dense_transport_bytes(name, g, passes):
    (n, d, C, sep, seed), m, t, L, K, delta = DENSE[name]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(g),
                           homo=G.HomoTransformParams(m, t, seed=1),
                           seeding=G.SeedingParams(K, L, min_group_size=delta, seed=2), passes=passes)
    out = G.run_pipeline(G.DenseData(X), cfg)
    assert out.transport_bytes == _golden()[f"{name}_g{g}_p{passes}"]


@pytest.mark.parametrize("g,passes", [(1, 0), (2, 0), (2, 1)])
def test_sparse_transport_bytes(g, passes):
    arr = npz("pipelines")
    data = G.SparseData(csr(arr["sp_flat"], arr["sp_off"]), 20_000)
    cfg = G.PipelineConfig(metric="jaccard", transform_kind="sparse", workers=G.WorkerConfig(g),
                           minhash=G.MinhashTransformParams(3, 6, seed=4, target_dims=400),
                           seeding=G.SeedingParams(3, 6, min_group_size=3, seed=5), passes=passes)
    assert G.run_pipeline(data, cfg).transport_bytes == _golden()[f"sparse_g{g}_p{passes}"]


@pytest.mark.parametrize("passes", [0, 1])
def test_mixed_transport_bytes(passes):
    arr = npz("pipelines")
    cfg = G.PipelineConfig(metric="jaccard", transform_kind="mixed", workers=G.WorkerConfig(2),
                           minhash=G.MinhashTransformParams(3, 6, seed=7, bins_per_attribute=16),
                           seeding=G.SeedingParams(3, 6, min_group_size=3, seed=9), passes=passes)
    out = G.run_pipeline(G.MixedData(arr["mx_num"], arr["mx_cat"]), cfg)
    assert out.transport_bytes == _golden()[f"mixed_g2_p{passes}"]


def test_memory_budget_below_one_table():
    X, _ = O.gaussian_mixture(3000, 8, 6, 12.0, 4)
    cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(2, memory_budget=1000),
                           homo=G.HomoTransformParams(8, 30, seed=1),
                           seeding=G.SeedingParams(3, 8, min_group_size=3, seed=2))
    with pytest.raises(G.EngineError) as exc:
        G.run_pipeline(G.DenseData(X), cfg)
    assert str(exc.value) == _golden()["budget_error"]


def test_nonfinite_exact_sum_raises():
    X, _ = O.gaussian_mixture(3000, 8, 6, 12.0, 4)
    X[55, 3] = np.inf  # a seed-group member: the reference raises ValueError in exact_column_sums
    # (numeric.py:24-25); checked against lshclust on this input when the golden was made
    cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(1),
                           homo=G.HomoTransformParams(8, 30, seed=1),
                           seeding=G.SeedingParams(3, 8, min_group_size=1, seed=2))
    with pytest.raises(ValueError):
        G.run_pipeline(G.DenseData(X), cfg)
