"""One pipeline step at a reduced size for ncu captures (single GPU).

    python tools/profile_step.py [n]      # default n = 10M (bench law, t = n/1e5)
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2106_10515_b200 as G  # noqa: E402
from paper_2106_10515_b200 import _lib  # noqa: E402

if os.environ.get("PROBE_DEBUG"):  # the -DGEEK_DEBUG_KNOBS build (tools/build_debug.py)
    _lib.load_library(os.path.join(os.path.dirname(_lib.LIB_PATH), "libgeek_dbg.so"))
from paper_2106_10515_b200.synth import gaussian_mixture_device  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
X = gaussian_mixture_device(n, 128, 1000, 10.0, 0)
cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(8),
                       homo=G.HomoTransformParams(40, max(2, n // 100_000), seed=1),
                       seeding=G.SeedingParams(2, 20, min_group_size=10, seed=2))
for _ in range(2):
    out = G.run_pipeline_shard(X, n, cfg)
torch.cuda.synchronize()
print(f"n={n} k*={out.k_star} groups={out._groups.count} info={out.info}")
