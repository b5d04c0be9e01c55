"""Parameter exploration on the GPU: k* and seeding statistics of the dense
pipeline for a few (n, C, t, K, L) settings of the SIFT-like law."""

import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2106_10515_b200 as G  # noqa: E402
from paper_2106_10515_b200.synth import gaussian_mixture_device  # noqa: E402


def run(n, C, t, K, L, m=40, delta=10, g=8, sep=10.0):
    X = gaussian_mixture_device(n, 128, C, sep, 0)
    cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(g),
                           homo=G.HomoTransformParams(m, t, seed=1),
                           seeding=G.SeedingParams(K, L, min_group_size=delta, seed=2))
    t0 = time.time()
    out = G.run_pipeline_shard(X, n, cfg)
    torch.cuda.synchronize()
    el = time.time() - t0
    rec = dict(n=n, C=C, t=t, K=K, L=L, m=m, k_star=out.k_star, groups=out._groups.count,
               warnings=len(out.warnings), sec=round(el, 3), info=out.info,
               stages={k: round(v, 4) for k, v in out.timings.items()})
    print(json.dumps(rec), flush=True)
    del X, out
    torch.cuda.empty_cache()


if __name__ == "__main__":
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
    for C, t, K in itertools.product([1000], [1000, 3000, 10000], [2, 3]):
        run(n, C, t * n // 10_000_000, K, 20)
