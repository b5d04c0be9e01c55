"""Probe the tcgen05 screen's canonical-layout strides and error on the GPU."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2106_10515_b200 import _lib  # noqa: E402

L = _lib.load_library()
torch.cuda.init()
for nprod in (1, 3):
    for lbo, sbo in [(128, 256), (256, 128)]:
        out = (C.c_double * 2)()
        st = L.geek_tc_selftest(lbo, sbo, nprod, out)
        torch.cuda.synchronize()
        print(f"nprod={nprod} lbo={lbo} sbo={sbo} status={st} worst_rel={out[0]:.3e} bad_top1={out[1]:.0f}",
              flush=True)
