"""Golden vector files written and read back by the REAL reference
(lshclust.io.write_fvecs / read_fvecs, io.py:21-62).  Build container only:

    python tests/golden/make_io_golden.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from lshclust import io as rio  # noqa: E402
from lshclust.data import DenseData  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(21)
    X = rng.standard_normal((37, 11)) * 100.0
    arrays = {"src": X}
    for ext in ("fvecs", "bvecs"):
        path = os.path.join(OUT, f"io_small.{ext}")
        rio.write_fvecs(path, DenseData(X))
        arrays[ext] = rio.read_fvecs(path).vectors
    np.savez_compressed(os.path.join(OUT, "io.npz"), **arrays)


if __name__ == "__main__":
    main()
