"""Loader for the committed golden fixtures (tests/golden/*)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def meta():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def npz(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def groups(arr, prefix):
    flat, off = arr[prefix + "_gflat"], arr[prefix + "_goff"]
    return [flat[off[i]:off[i + 1]] for i in range(len(off) - 1)]


def csr(flat, off):
    return [flat[off[i]:off[i + 1]] for i in range(len(off) - 1)]


def refine_meta():
    with open(os.path.join(GOLDEN, "refine.json")) as f:
        return json.load(f)


def baselines_meta():
    with open(os.path.join(GOLDEN, "baselines.json")) as f:
        return json.load(f)
