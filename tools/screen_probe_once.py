"""One FP16x3 screen launch on the 20M-point probe data of tools/screen_probe.py (cluster-ordered
ids), for ncu captures: python tools/screen_probe_once.py [n] [k] [d]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2106_10515_b200.assignment import assign_l2_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 963
d = int(sys.argv[3]) if len(sys.argv) > 3 else 128
g = torch.Generator(device="cuda").manual_seed(0)
C = torch.randn(k, d, device="cuda", dtype=torch.float64, generator=g) * 10
lab = torch.sort(torch.randint(0, k, (n,), device="cuda", generator=g)).values
X = (C[lab] + torch.randn(n, d, device="cuda", dtype=torch.float64, generator=g)).float()
del lab
assign_l2_device(X, C)
torch.cuda.synchronize()
