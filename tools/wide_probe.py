"""Wide-row (d > 128) assignment screens on GIST-like data: per-kernel CUDA
times (torch.profiler) and the screen's recheck counts for GEEK_WIDE=65
(FP16x3 GEMM, default) and 64 (float64 DGEMM).
usage: python tools/wide_probe.py [n] [k] [d]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2106_10515_b200.assignment import AssignStats, assign_l2_device  # noqa: E402
from paper_2106_10515_b200.synth import gaussian_mixture_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 753
d = int(sys.argv[3]) if len(sys.argv) > 3 else 960
X = gaussian_mixture_device(n, d, 1000, 10.0, 0)
g = torch.Generator(device="cuda").manual_seed(1)
C = X[torch.randint(0, n, (k,), device="cuda", generator=g)].double()
C += torch.randn(C.shape, device="cuda", dtype=torch.float64, generator=g) * 0.3
for mode in ("66", "65", "64"):
    os.environ["GEEK_WIDE"] = mode
    st = AssignStats()
    assign_l2_device(X, C, st)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        st = AssignStats()
        lab, best = assign_l2_device(X, C, st)
        torch.cuda.synchronize()
    print(f"GEEK_WIDE={mode}", st.read())
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
