"""torch.profiler breakdown of one Criteo-like mixed pipeline (tools/mixed_probe.py's data law):
the top CUDA and CPU operators of the step.  python tools/mixed_profile.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile, record_function  # noqa: E402

import paper_2106_10515_b200 as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
C = 1000
dev = torch.device("cuda", 0)
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
cfg = G.PipelineConfig(metric="jaccard", transform_kind="mixed", workers=G.WorkerConfig(8),
                       minhash=G.MinhashTransformParams(3, 20, seed=7, bins_per_attribute=1024),
                       seeding=G.SeedingParams(3, 20, min_group_size=10, seed=9))
G.run_pipeline(data, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True, with_stack=True) as prof:
    with record_function("pipeline"):
        out = G.run_pipeline(data, cfg)
        torch.cuda.synchronize()
print(out.timings, out.info)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=30))
print(prof.key_averages(group_by_input_shape=True).table(sort_by="cpu_time_total", row_limit=15))
print(prof.key_averages(group_by_stack_n=6).table(sort_by="cpu_time_total", row_limit=12))
