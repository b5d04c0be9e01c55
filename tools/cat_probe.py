"""Time geek_assign_categorical (tiled vs per-thread kernel) on random codes.

usage: python tools/cat_probe.py N D K [NAIVE_N]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2106_10515_b200.assignment import assign_cat_device  # noqa: E402


def timed(codes, M):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lab, best = assign_cat_device(codes, M)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), lab, best


def main():
    n, d, k = (int(a) for a in sys.argv[1:4])
    nn = int(sys.argv[4]) if len(sys.argv) > 4 else min(n, 2_000_000)
    g = torch.Generator(device="cuda").manual_seed(1)
    codes = torch.randint(0, 6, (n, d), generator=g, device="cuda", dtype=torch.int32)
    M = torch.randint(0, 6, (k, d), generator=g, device="cuda", dtype=torch.int32)
    timed(codes[:1000], M)
    ms, lab, best = timed(codes, M)
    out = {"n": n, "d": d, "k": k, "tiled_ms": ms,
           "pairs_per_s": n * k / ms * 1e3, "attr_cmp_per_s": n * k * d / ms * 1e3}
    os.environ["GEEK_CAT_NAIVE"] = "1"
    ms2, lab2, best2 = timed(codes[:nn], M)
    del os.environ["GEEK_CAT_NAIVE"]
    out.update(naive_n=nn, naive_ms=ms2, naive_scaled_ms=ms2 * n / nn,
               equal=bool(torch.equal(lab[:nn], lab2) and torch.equal(best[:nn], best2)))
    print(json.dumps(out))


if __name__ == "__main__":
    t = time.time()
    main()
    print("wall", time.time() - t, file=sys.stderr)
