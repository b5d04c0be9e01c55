"""Host synchronisations in one bench-law pipeline step (n = 1e7 by default):
counts of cudaStreamSynchronize / device-to-host copies / .item() from the
torch profiler, grouped by the Python frame that issued them.
usage: python tools/sync_count.py [n]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2106_10515_b200 as G  # noqa: E402
from paper_2106_10515_b200.synth import gaussian_mixture_device  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
X = gaussian_mixture_device(n, 128, 1000, 10.0, 0)
cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(8),
                       homo=G.HomoTransformParams(40, max(2, n // 100_000), seed=1),
                       seeding=G.SeedingParams(2, 20, min_group_size=10, seed=2))
G.run_pipeline_shard(X, n, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True) as prof:
    G.run_pipeline_shard(X, n, cfg)
    torch.cuda.synchronize()
cnt = collections.Counter()
where = collections.Counter()
for e in prof.events():
    if e.name in ("cudaStreamSynchronize", "cudaDeviceSynchronize", "cudaMemcpyAsync", "aten::item",
                  "aten::_local_scalar_dense", "cudaEventSynchronize"):
        cnt[e.name] += 1
        st = [f for f in (e.stack or []) if "paper_2106_10515_b200" in f]
        if st and e.name in ("cudaStreamSynchronize", "cudaMemcpyAsync", "aten::item"):
            where[(e.name, st[0])] += 1
print(dict(cnt))
for (name, frame), c in where.most_common(40):
    print(f"{c:5d} {name:22s} {frame}")
