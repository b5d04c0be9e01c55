"""Time the tensor-core assignment screen (CUDA events around its launches)
at the bench size.  The GEEK_SCREEN_PROF knobs (0 normal, 1 no epilogue
math, 2 no MMAs, 3 no A writes, ...) and GEEK_SCREEN_DBG only act in a
library built with -DGEEK_DEBUG_KNOBS (they skip work, so the product
build ignores them).  Usage: python tools/screen_probe.py [n] [k] [d]."""
import os
import subprocess
import sys

if os.environ.get("_PROBE_CHILD"):
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2106_10515_b200 import _lib as L
    if os.environ.get("PROBE_DEBUG"):  # the -DGEEK_DEBUG_KNOBS build (tools/build_debug.py)
        L.load_library(os.path.join(os.path.dirname(L.LIB_PATH), "libgeek_dbg.so"))
    from paper_2106_10515_b200.assignment import AssignStats
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 963
    d = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    g = torch.Generator(device="cuda").manual_seed(0)
    C = torch.randn(k, d, device="cuda", dtype=torch.float64, generator=g) * 10
    X = torch.empty(n, d, device="cuda", dtype=torch.float32)
    for i in range(0, n, 10_000_000):
        j = min(n, i + 10_000_000)
        lab = torch.randint(0, k, (j - i,), device="cuda", generator=g)
        if os.environ.get("PROBE_SORTED"):  # cluster-ordered ids, as the reference generator's
            lab = torch.sort(lab).values
        X[i:j] = (C[lab] + torch.randn(j - i, d, device="cuda", dtype=torch.float64, generator=g)).float()
    labels = torch.empty(n, dtype=torch.int64, device="cuda")
    best = torch.empty(n, dtype=torch.float64, device="cuda")
    ms = []
    for it in range(4):
        st = AssignStats()
        L.call("geek_assign_l2", L.ptr(X), 0, n, d, L.ptr(C), k, L.ptr(labels), L.ptr(best), L.ptr(st.dev),
               L.C.c_void_p(st.ev0.cuda_event), L.C.c_void_p(st.ev1.cuda_event), None, 0, L.stream())
        torch.cuda.synchronize()
        ms.append(st.read()["screen_ms"])
    print(f"mode={os.environ.get('GEEK_SCREEN_PROF','0')} screen={os.environ.get('GEEK_SCREEN','16')} "
          f"sleep={os.environ.get('GEEK_SCREEN_SLEEP','0')} "
          f"screen_ms={min(ms[1:]):.2f} all={['%.2f' % v for v in ms]}", flush=True)
else:
    for scr in os.environ.get("PROBE_SCREENS", os.environ.get("GEEK_SCREEN", "16")).split(","):
        for mode in os.environ.get("PROBE_MODES", "0,1,2,3").split(","):
            env = dict(os.environ, _PROBE_CHILD="1", GEEK_SCREEN_PROF=mode, GEEK_SCREEN=scr)
            subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, check=False)
