"""Dump the REAL reference's transport accounting (PipelineResult.transport_bytes,
engine.py:79-104 + serialize.py message bodies) and its memory-budget error
for the small golden pipelines.  Build container only:

    python tests/golden/make_transport_golden.py  ->  tests/golden/transport.json
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from lshclust import data as D, seeding, transform  # noqa: E402
from lshclust.engine import EngineError, PipelineConfig, WorkerConfig, run_pipeline  # noqa: E402
from lshclust.synth import SyntheticSpec, gen_synthetic  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    out = {}
    dense = {"c06": (SyntheticSpec("gaussian-mixture", 2000, 16, 10, 20.0, 0), 48, 10, 48, 3, 5),
             "small": (SyntheticSpec("gaussian-mixture", 3000, 8, 6, 12.0, 4), 8, 30, 8, 3, 3)}
    for name, (spec, m, t, L, K, delta) in dense.items():
        X = gen_synthetic(spec).data
        for g, passes in [(1, 0), (2, 0), (4, 0), (8, 0), (2, 2), (8, 1)]:
            cfg = PipelineConfig(metric="euclidean", transform_kind="dense", workers=WorkerConfig(g),
                                 homo=transform.HomoTransformParams(m, t, seed=1),
                                 seeding=seeding.SeedingParams(K, L, min_group_size=delta, seed=2), passes=passes)
            res = run_pipeline(X, cfg)
            out[f"{name}_g{g}_p{passes}"] = dict(res.transport_bytes)
    res = gen_synthetic(SyntheticSpec("sparse-overlap", 1500, 20_000, 15, 10.0, 3))
    mp = transform.MinhashTransformParams(3, 6, seed=4, target_dims=400)
    for g, passes in [(1, 0), (2, 0), (2, 1)]:
        cfg = PipelineConfig(metric="jaccard", transform_kind="sparse", workers=WorkerConfig(g), minhash=mp,
                             seeding=seeding.SeedingParams(3, 6, min_group_size=3, seed=5), passes=passes)
        out[f"sparse_g{g}_p{passes}"] = dict(run_pipeline(res.data, cfg).transport_bytes)
    rng = np.random.default_rng(11)
    nm = 1200
    lab = np.sort(rng.integers(0, 8, nm))
    num = rng.lognormal(mean=lab[:, None] * 0.5, sigma=0.3, size=(nm, 3))
    cat = (lab[:, None] * 3 + rng.integers(0, 2, (nm, 4))).astype(np.int32)
    mp2 = transform.MinhashTransformParams(3, 6, seed=7, bins_per_attribute=16)
    for g, passes in [(2, 0), (2, 1)]:
        cfg = PipelineConfig(metric="jaccard", transform_kind="mixed", workers=WorkerConfig(g), minhash=mp2,
                             seeding=seeding.SeedingParams(3, 6, min_group_size=3, seed=9), passes=passes)
        out[f"mixed_g{g}_p{passes}"] = dict(run_pipeline(D.MixedData(num, cat), cfg).transport_bytes)
    # memory budget below one table (engine.py:359-366)
    X = gen_synthetic(dense["small"][0]).data
    cfg = PipelineConfig(metric="euclidean", transform_kind="dense", workers=WorkerConfig(2, memory_budget=1000),
                         homo=transform.HomoTransformParams(8, 30, seed=1),
                         seeding=seeding.SeedingParams(3, 8, min_group_size=3, seed=2))
    try:
        run_pipeline(X, cfg)
        out["budget_error"] = None
    except EngineError as e:
        out["budget_error"] = str(e)
    with open(os.path.join(OUT, "transport.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
