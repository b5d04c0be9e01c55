"""H2D bandwidth from pinned host memory: one copy vs chunked copies over 1-4 streams."""
import time

import torch

n_bytes = int(51.2e9)
Xh = torch.empty(n_bytes // 4, dtype=torch.float32, pin_memory=True)
Xh.fill_(1.0)
Xd = torch.empty_like(Xh, device="cuda")
torch.cuda.synchronize()


def run(streams, chunks):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    n = Xh.numel()
    step = (n + chunks - 1) // chunks
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for c in range(chunks):
        lo, hi = c * step, min(n, (c + 1) * step)
        with torch.cuda.stream(ss[c % streams]):
            Xd[lo:hi].copy_(Xh[lo:hi], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"streams={streams} chunks={chunks}: {n_bytes / dt / 1e9:.1f} GB/s", flush=True)


for s, c in [(1, 1), (1, 16), (2, 16), (4, 16), (2, 2)]:
    run(s, c)
