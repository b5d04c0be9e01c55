"""LSHC v1 artifacts written by the REAL reference (lshclust.serialize,
serialize.py:129-198): the worked example in full (tests/golden/art_*.lshc)
and sha256 / length of the 'small' dense case's bucket, seed-group and
clustering files (tests/golden/artifacts.json).  Build container only:

    python tests/golden/make_artifact_golden.py
"""

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from lshclust import serialize, seeding, transform  # noqa: E402
from lshclust.data import Bucket, DenseData  # noqa: E402
from lshclust.engine import PipelineConfig, WorkerConfig, run_pipeline  # noqa: E402
from lshclust.synth import SyntheticSpec, gen_synthetic  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
WORKED = [(0, 0, [0, 1, 3]), (0, 1, [2, 4, 5]), (1, 0, [0, 1, 3, 4]), (1, 1, [5]),
          (2, 0, [0, 1, 3, 5]), (2, 1, [2, 4]), (3, 0, [0, 1, 3, 5]), (3, 1, [4, 5])]
POINTS = np.array([[0.0, 0.0, 0.0, 0.0], [0.1, 0.1, 0.1, 0.1], [10.0, 0.2, 10.0, 0.3],
                   [0.2, 0.3, 0.2, 0.4], [10.1, 0.4, 10.1, 0.5], [12.0, 0.5, 12.0, 0.2]])


def sha(b):
    return dict(sha256=hashlib.sha256(b).hexdigest(), bytes=len(b))


def main():
    meta = {}
    bk = [Bucket(t, s, np.array(m)) for t, s, m in WORKED]
    cfg = PipelineConfig(metric="euclidean", transform_kind="dense", workers=WorkerConfig(1),
                         homo=transform.HomoTransformParams(4, 2, seed=1),
                         seeding=seeding.SeedingParams(2, 4, min_group_size=2, seed=2))
    out = run_pipeline(DenseData(POINTS), cfg)
    files = {"art_buckets.lshc": serialize.dump_buckets(bk),
             "art_groups.lshc": serialize.dump_seed_groups(out.seed_groups),
             "art_clustering.lshc": serialize.dump_clustering(out.clustering)}
    for name, b in files.items():
        with open(os.path.join(OUT, name), "wb") as f:
            f.write(b)
    res = gen_synthetic(SyntheticSpec("gaussian-mixture", 3000, 8, 6, 12.0, 4))
    hp = transform.HomoTransformParams(8, 30, seed=1)
    meta["small_buckets"] = sha(serialize.dump_buckets(transform.transform_homo(res.data, hp)))
    cfg = PipelineConfig(metric="euclidean", transform_kind="dense", workers=WorkerConfig(2), homo=hp,
                         seeding=seeding.SeedingParams(3, 8, min_group_size=3, seed=2))
    out = run_pipeline(res.data, cfg)
    meta["small_groups"] = sha(serialize.dump_seed_groups(out.seed_groups))
    meta["small_clustering"] = sha(serialize.dump_clustering(out.clustering))
    with open(os.path.join(OUT, "artifacts.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(meta)


if __name__ == "__main__":
    main()
