"""Criteo-like heterogeneous configuration (BASELINE configs[4]): N rows of 13
numeric (lognormal per cluster) + 26 categorical attributes (cardinalities
3 ... 1e6, a preferred code per cluster with p = 0.8, else a skewed draw),
1000 clusters, run_pipeline(transform_kind="mixed"): numeric columns rank-
discretised into 1024 codes, K = 3, L = 20 (transform and SILK), delta = 10,
g = 8.  One warm and one timed run; exact spot check of 2,000 sampled labels
/ distances against numpy's categorical Jaccard on the unified codes.

    python tools/mixed_probe.py N
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2106_10515_b200 as G
from paper_2106_10515_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
C = 1000
dev = torch.device("cuda", 0)
t0 = time.time()
gen = torch.Generator(device=dev)
gen.manual_seed(0)
lab = torch.sort(torch.randint(0, C, (n,), generator=gen, device=dev))[0]
mu = torch.rand((C, 13), generator=gen, device=dev, dtype=torch.float64) * 4
num = torch.exp(mu[lab] + 0.5 * torch.randn((n, 13), generator=gen, device=dev, dtype=torch.float64))
cards = torch.tensor(np.geomspace(3, 1e6, 26).astype(np.int64), device=dev)
pref = (torch.rand((C, 26), generator=gen, device=dev) * cards).to(torch.int64)
skew = (torch.rand((n, 26), generator=gen, device=dev) ** 3 * cards).to(torch.int64)
cat = torch.where(torch.rand((n, 26), generator=gen, device=dev) < 0.8, pref[lab], skew).to(torch.int32)
data = G.MixedData(num.cpu().numpy(), cat.cpu().numpy())
gen_s = time.time() - t0
cfg = G.PipelineConfig(metric="jaccard", transform_kind="mixed", workers=G.WorkerConfig(8),
                       minhash=G.MinhashTransformParams(3, 20, seed=7, bins_per_attribute=1024),
                       seeding=G.SeedingParams(3, 20, min_group_size=10, seed=9))
out = G.run_pipeline(data, cfg)
tm = _lib.CallTimer()
_lib.set_call_timer(tm)
torch.cuda.synchronize()
w0 = time.time()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
out = G.run_pipeline(data, cfg)
b.record()
torch.cuda.synchronize()
wall = time.time() - w0
_lib.set_call_timer(None)
ms = a.elapsed_time(b)
uni = G.discretize_numeric(data, 1024).codes
M = np.stack([c.values for c in out.clustering.centers])
rng = np.random.default_rng(1)
idx = np.sort(rng.choice(n, 2000, replace=False))
mt = (uni[idx][:, None, :] == M[None, :, :]).sum(2)
dist = 1.0 - mt / (2 * 39 - mt)
a_ = np.argmin(dist, 1)
labs = out.labels_device.cpu().numpy()[idx]
best = out.best_device.cpu().numpy()[idx]
bad = int((a_ != labs).sum() + (dist[np.arange(idx.size), a_] != best).sum())
print(json.dumps(dict(n=n, gen_s=gen_s, ms=ms, wall_s=wall, rows_per_s=n / ms * 1e3, k_star=out.k_star,
                      stages_s=out.timings, calls_ms={k: round(v[0], 2) for k, v in tm.ms_by_name().items()},
                      spot_check=dict(samples=int(idx.size), mismatches=bad)), indent=1))
