"""Refinement pass at bench scale (100M x 128 f32, bench parameters): time the
one-pass pipeline with passes = 0 and 1 and the label-keyed exact sums
(geek_label_sums) on the pipeline's labels and on shuffled labels, each as
achieved HBM GB/s over the algorithmic bytes (X read + labels read)."""
import json
import sys

import torch

import paper_2106_10515_b200 as G
from paper_2106_10515_b200 import _lib, numeric
from paper_2106_10515_b200.synth import gaussian_mixture_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
d, m, K, L, delta = 128, 40, 2, 20, 10
X = gaussian_mixture_device(n, d, 1000, 10.0, 0)
res = {}
for passes in (0, 1):
    cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(8),
                           homo=G.HomoTransformParams(m, n // 100_000, seed=1),
                           seeding=G.SeedingParams(K, L, min_group_size=delta, seed=2), passes=passes)
    out = G.run_pipeline_shard(X, n, cfg)  # warm
    t = _lib.CallTimer()
    _lib.set_call_timer(t)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = G.run_pipeline_shard(X, n, cfg)
    b.record()
    torch.cuda.synchronize()
    _lib.set_call_timer(None)
    calls = {k: round(v[0], 3) for k, v in t.ms_by_name().items()}
    res[f"passes{passes}"] = dict(ms=a.elapsed_time(b), k_star=out.k_star, objective=out.objective, calls_ms=calls)

emin, emax = numeric.exponent_range(X)
nd = numeric.digit_count(emin, emax)
lab = out.labels_device
k = int(lab.max().item()) + 1
alg = n * d * 4 + n * 8
for name, L_ in (("pipeline_labels", lab), ("shuffled_labels", lab[torch.randperm(n, device=lab.device)])):
    numeric.label_sums(X, L_, k, emin, nd)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        numeric.label_sums(X, L_, k, emin, nd)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    res[name] = dict(ms=ms, GBps=alg / ms / 1e6, nd=nd)
print(json.dumps(res, indent=1))
