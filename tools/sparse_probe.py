"""URL-like sparse configuration (BASELINE configs[3]): N sets over a 3M-id
universe drawn on the device with the reference's sparse-overlap law
(synth.py:65-83: C clusters, base sets of universe//(4C) ids, each member keeps
a base id with p = 0.95 and adds base_size*0.05 random ids; cluster-sorted
labels), then run_pipeline(transform_kind="sparse") with DOPH to 400 dims,
K = 3, L = 20 (transform and SILK), delta = 10, g = 8 -- one warm, one timed
run, per-stage and per-call times, and an exact spot check of 2,000 sampled
labels / distances against numpy's Jaccard on the reduced sets.

    python tools/sparse_probe.py N [C]
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
C = int(sys.argv[2]) if len(sys.argv) > 2 else 6466
U = 3_000_000
dev = torch.device("cuda", 0)
t0 = time.time()
g = torch.Generator(device=dev)
g.manual_seed(0)
base_size = max(U // (C * 4), 8)
extras = max(1, int(base_size * 0.05))
bases = torch.sort(torch.stack([torch.randperm(U, generator=g, device=dev)[:base_size] for _ in range(C)]), 1)[0]
labels = torch.sort(torch.randint(0, C, (n,), generator=g, device=dev))[0]
flats, sizes = [], []
for lo in range(0, n, 1 << 21):
    hi = min(n, lo + (1 << 21))
    rows = bases[labels[lo:hi]]
    keep = torch.rand(rows.shape, generator=g, device=dev) < 0.95
    keep[:, 0] |= ~keep.any(1)
    rows = torch.where(keep, rows, torch.full_like(rows, U))
    ex = torch.randint(0, U, (hi - lo, extras), generator=g, device=dev)
    allv = torch.sort(torch.cat([rows, ex], 1), 1)[0]
    ok = allv < U
    ok[:, 1:] &= allv[:, 1:] != allv[:, :-1]
    flats.append(allv[ok])
    sizes.append(ok.sum(1))
flat = torch.cat(flats)
off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
torch.cumsum(torch.cat(sizes), 0, out=off[1:])
data = G.SparseData.from_csr(flat, off, U)
torch.cuda.synchronize()
gen_s = time.time() - t0
cfg = G.PipelineConfig(metric="jaccard", transform_kind="sparse", workers=G.WorkerConfig(8),
                       minhash=G.MinhashTransformParams(3, 20, seed=4, target_dims=400),
                       seeding=G.SeedingParams(3, 20, min_group_size=10, seed=5))
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
# spot check: exact Jaccard of sampled reduced sets against the modes
from paper_2106_10515_b200.hashing import DophReducer, derive_seed
red = DophReducer(derive_seed(4, 0xD0), U, 400)
rf, ro = red.reduce_device(*data.csr(), n)
rf, ro = rf.cpu().numpy().view(np.uint32), ro.cpu().numpy()
M = np.stack([c.values for c in out.clustering.centers]).astype(np.float64)
rng = np.random.default_rng(1)
idx = np.sort(rng.choice(n, 2000, replace=False))
Xb = np.zeros((idx.size, 400))
for r, i in enumerate(idx):
    Xb[r, rf[ro[i]:ro[i + 1]]] = 1.0
inter = Xb @ M.T
union = Xb.sum(1)[:, None] + M.sum(1)[None, :] - inter
dist = 1.0 - np.where(union > 0, inter / np.where(union > 0, union, 1), 1.0)
lab = out.labels_device.cpu().numpy()[idx]
best = out.best_device.cpu().numpy()[idx]
a_ = np.argmin(dist, 1)
bad = int((a_ != lab).sum() + (dist[np.arange(idx.size), a_] != best).sum())
print(json.dumps(dict(n=n, clusters=C, nnz=int(flat.numel()), gen_s=gen_s, ms=ms, wall_s=wall,
                      points_per_s=n / ms * 1e3, k_star=out.k_star, stages_s=out.timings,
                      calls_ms={k: round(v[0], 2) for k, v in tm.ms_by_name().items()},
                      info={k: v for k, v in out.info.items() if isinstance(v, (int, float, str))},
                      spot_check=dict(samples=int(idx.size), mismatches=bad)), indent=1, default=str))
