"""Golden outputs of the reference's comparison methods (lshclust.baselines,
baselines.py:34-136) for tests/golden/baselines.npz + baselines.json.  Build
container only:

    python tests/golden/make_baselines_golden.py
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from lshclust import baselines as B  # noqa: E402
from lshclust import data as D  # noqa: E402
from lshclust.synth import SyntheticSpec, gen_synthetic  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    arrays, meta = {}, {}
    dense = gen_synthetic(SyntheticSpec("gaussian-mixture", 2000, 16, 10, 6.0, 5)).data
    rng = np.random.default_rng(12)
    cat = D.CategoricalData(rng.integers(0, 5, (1500, 7)).astype(np.int32), code_space=5)
    sp = gen_synthetic(SyntheticSpec("sparse-overlap", 600, 300, 6, 10.0, 2)).data

    arrays["sp_flat"] = np.concatenate(sp.sets)
    arrays["sp_off"] = np.concatenate(([0], np.cumsum([s.size for s in sp.sets])))
    meta["sp_universe"] = sp.universe

    def centers(name, cs):
        arrays[name] = np.stack([c.values for c in cs])

    centers("rand_dense", B.seed_random(dense, 12, 3))
    centers("pp_dense", B.seed_kmeanspp(dense, 12, 4))
    centers("pp_cat", B.seed_kmeanspp(cat, 9, 5, metric="jaccard"))
    centers("pp_sparse", B.seed_kmeanspp(sp, 7, 6, metric="jaccard"))
    for name, cl in (("lloyd", B.lloyd(dense, 12, 7)), ("lloyd_2it", B.lloyd(dense, 12, 7, max_iters=2)),
                     ("kmodes_cat", B.kmodes(cat, 9, 8)), ("kmodes_sparse", B.kmodes(sp, 7, 9))):
        centers(f"{name}_centers", cl.centers)
        arrays[f"{name}_labels"] = cl.assignment.astype(np.int32)
        arrays[f"{name}_radii"] = cl.radii
        meta[name] = dict(objective=cl.objective, k_star=cl.k_star)
    np.savez_compressed(os.path.join(OUT, "baselines.npz"), **arrays)
    with open(os.path.join(OUT, "baselines.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(meta)


if __name__ == "__main__":
    main()
