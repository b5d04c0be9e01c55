"""Dump golden vectors for refinement passes from the REAL reference
(lshclust.assignment.refine, assignment.py:157-170, and run_pipeline with
passes > 0, engine.py:464-465 / :519-537) into tests/golden/refine.npz +
refine.json.  Build container only (imports /root/reference/pkg/src):

    python tests/golden/make_refine_golden.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from lshclust import assignment, seeding, transform, data as D  # noqa: E402
from lshclust.engine import PipelineConfig, WorkerConfig, run_pipeline  # noqa: E402
from lshclust.synth import SyntheticSpec, gen_synthetic  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def put(arrays, meta, name, cl, extra=None):
    arrays[f"{name}_centers"] = np.stack([c.values for c in cl.centers])
    arrays[f"{name}_weights"] = np.array([c.weight for c in cl.centers], dtype=np.int64)
    arrays[f"{name}_labels"] = cl.assignment.astype(np.int32)
    arrays[f"{name}_radii"] = cl.radii
    meta[name] = dict(objective=cl.objective, k_star=cl.k_star, **(extra or {}))


def main():
    arrays, meta = {}, {}
    # standalone refine on the c08 inputs (test_acceptance.py:305-360)
    rng = np.random.default_rng(80)
    dense = D.DenseData(rng.standard_normal((10_000, 16)))
    cents = [D.CentralVector("centroid", rng.standard_normal(16)) for _ in range(200)]
    c0 = assignment.assign(dense, cents, "euclidean")
    for p in (1, 2):
        put(arrays, meta, f"c08_p{p}", assignment.refine(dense, c0, "euclidean", p))
    codes = rng.integers(0, 8, (10_000, 9)).astype(np.int32)
    modes = [D.CentralVector("mode", rng.integers(0, 8, 9).astype(np.int32)) for _ in range(200)]
    cat = D.CategoricalData(codes, code_space=8)
    c0 = assignment.assign(cat, modes, "jaccard")
    put(arrays, meta, "c08cat_p2", assignment.refine(cat, c0, "jaccard", 2))

    # pipelines with passes (same inputs as make_golden.py's cases)
    res = gen_synthetic(SyntheticSpec("gaussian-mixture", 3000, 8, 6, 12.0, 4))
    for g in (1, 2):
        cfg = PipelineConfig(metric="euclidean", transform_kind="dense", workers=WorkerConfig(g),
                             homo=transform.HomoTransformParams(8, 30, seed=1),
                             seeding=seeding.SeedingParams(3, 8, min_group_size=3, seed=2), passes=2)
        put(arrays, meta, f"small_p2_g{g}", run_pipeline(res.data, cfg).clustering)
    res = gen_synthetic(SyntheticSpec("gaussian-mixture", 2000, 16, 10, 20.0, 0))
    cfg = PipelineConfig(metric="euclidean", transform_kind="dense", workers=WorkerConfig(1),
                         homo=transform.HomoTransformParams(48, 10, seed=1),
                         seeding=seeding.SeedingParams(3, 48, min_group_size=5, seed=2), passes=3)
    put(arrays, meta, "c06_p3_g1", run_pipeline(res.data, cfg).clustering)

    res = gen_synthetic(SyntheticSpec("sparse-overlap", 1500, 20_000, 15, 10.0, 3))
    cfg = PipelineConfig(metric="jaccard", transform_kind="sparse", workers=WorkerConfig(1),
                         minhash=transform.MinhashTransformParams(3, 6, seed=4, target_dims=400),
                         seeding=seeding.SeedingParams(3, 6, min_group_size=3, seed=5), passes=2)
    put(arrays, meta, "sp_p2_g1", run_pipeline(res.data, cfg).clustering)

    rng = np.random.default_rng(11)
    nm = 1200
    lab = np.sort(rng.integers(0, 8, nm))
    num = rng.lognormal(mean=lab[:, None] * 0.5, sigma=0.3, size=(nm, 3))
    catm = (lab[:, None] * 3 + rng.integers(0, 2, (nm, 4))).astype(np.int32)
    cfg = PipelineConfig(metric="jaccard", transform_kind="mixed", workers=WorkerConfig(1),
                         minhash=transform.MinhashTransformParams(3, 6, seed=7, bins_per_attribute=16),
                         seeding=seeding.SeedingParams(3, 6, min_group_size=3, seed=9), passes=2)
    put(arrays, meta, "mx_p2_g1", run_pipeline(D.MixedData(num, catm), cfg).clustering)

    np.savez_compressed(os.path.join(OUT, "refine.npz"), **arrays)
    with open(os.path.join(OUT, "refine.json"), "w") as f:
        json.dump(meta, f, indent=1, default=lambda o: int(o) if isinstance(o, np.integer) else float(o))
    for k, v in meta.items():
        print(k, v)


if __name__ == "__main__":
    main()
