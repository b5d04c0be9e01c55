"""Build paper_2106_10515_b200/libgeek_dbg.so: the product sources with
-DGEEK_DEBUG_KNOBS (the GEEK_SCREEN_PROF / _DBG / _SLEEP / _PUSHCUT
profiling knobs, which skip or instrument work).  Probes load it with
`_lib.load_library(DEBUG_LIB)`; the product never does."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10515_b200 import _build  # noqa: E402

DEBUG_LIB = os.path.join(os.path.dirname(_build.LIB), "libgeek_dbg.so")


def main():
    out = os.path.join(_build.BUILD, "dbg")
    os.makedirs(out, exist_ok=True)
    cc = _build.nvcc()
    objs = []
    procs = []
    for src in _build.sources():
        obj = os.path.join(out, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen([cc, *_build.NVCC_FLAGS, "-DGEEK_DEBUG_KNOBS", "-c", src, "-o", obj]))
    if any(p.wait() for p in procs):
        raise SystemExit("nvcc failed")
    subprocess.run([cc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "--cudart", "static", *objs,
                    "-o", DEBUG_LIB], check=True)
    print(DEBUG_LIB)


if __name__ == "__main__":
    main()
