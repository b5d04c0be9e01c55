"""GIST-like configuration (BASELINE configs[2]): synthetic 10M x 960 float32 (argv[1] = n,
argv[2] = points per bucket, default 1000),
1000 planted clusters, m = 40, t = n/1000, L = 20, K = 2, delta = 10, g = 8;
one warm and one timed run of the pipeline with per-stage times and the
libgeek call times, and an exact float64 spot check of 20K sampled labels /
best distances against a numpy evaluation of the reference's distance."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2106_10515_b200 as G
from paper_2106_10515_b200 import _lib
from paper_2106_10515_b200.synth import gaussian_mixture_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
d = 960
t0 = time.time()
X = gaussian_mixture_device(n, d, 1000, 10.0, 0)
torch.cuda.synchronize()
gen_s = time.time() - t0
cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(8),
                       homo=G.HomoTransformParams(40, max(1, n // int(sys.argv[2]) if len(sys.argv) > 2 else n // 1000), seed=1),
                       seeding=G.SeedingParams(2, 20, min_group_size=10, seed=2))
out = G.run_pipeline_shard(X, n, cfg)
tm = _lib.CallTimer()
_lib.set_call_timer(tm)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
out = G.run_pipeline_shard(X, n, cfg)
b.record()
torch.cuda.synchronize()
_lib.set_call_timer(None)
ms = a.elapsed_time(b)
k = len(out.sizes_device)
rng = np.random.default_rng(0)
idx = np.sort(rng.choice(n, 20_000, replace=False))
xs = X[torch.from_numpy(idx).cuda()].double().cpu().numpy()
C = torch.stack([torch.from_numpy(c.values) for c in out.clustering.centers]).numpy()
lab = out.labels_device[torch.from_numpy(idx).cuda()].cpu().numpy()
best = out.best_device[torch.from_numpy(idx).cuda()].cpu().numpy()
bad = 0
for lo in range(0, idx.size, 256):
    dm = np.sqrt(((xs[lo:lo + 256, None, :] - C[None, :, :]) ** 2).sum(axis=2))
    a_ = np.argmin(dm, axis=1)
    bad += int((a_ != lab[lo:lo + 256]).sum() + (dm[np.arange(a_.size), a_] != best[lo:lo + 256]).sum())
print(json.dumps(dict(n=n, d=d, gen_s=gen_s, ms=ms, points_per_s=n / ms * 1e3, k=k, k_star=out.k_star,
                      stages_s=out.timings, info=out.info,
                      calls_ms={kk: round(v[0], 2) for kk, v in tm.ms_by_name().items()},
                      spot_check=dict(samples=int(idx.size), mismatches=bad)), indent=1))
