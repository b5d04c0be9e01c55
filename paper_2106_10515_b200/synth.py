"""Synthetic inputs with the reference generator's law (synth.py:1-139).

`gen_synthetic` reproduces the reference's generator for all three kinds
(same numpy stream, so `gen` output files are byte-identical) -- host work
sized for parity fixtures and the CLI; `gaussian_mixture_device` draws the
gaussian-mixture law at benchmark scale directly into HBM: cluster means from
the host spiral (`spread_means`), labels uniform then sorted (so ids are
cluster-contiguous, as in the reference), x = mean + N(0, 1) from torch's
Philox generator, float32.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .data import CategoricalData, DenseData, SparseData
from .errors import InvalidInput

KINDS = ("gaussian-mixture", "categorical-patterns", "sparse-overlap")


@dataclass(frozen=True)
class SyntheticSpec:
    """synth.py:17-30"""

    kind: str
    n: int
    dim: int
    clusters: int
    separation: float = 10.0
    seed: int = 0

    def __post_init__(self):
        if self.kind not in KINDS:
            raise InvalidInput(f"unknown synthetic kind {self.kind!r}")
        if self.n < self.clusters or self.clusters < 1:
            raise InvalidInput("need n >= clusters >= 1")


@dataclass(frozen=True)
class SyntheticResult:
    data: object
    labels: np.ndarray
    true_radii: np.ndarray


def gen_synthetic(spec: SyntheticSpec) -> SyntheticResult:
    """synth.py:39-83: labels uniform then sorted (every cluster populated),
    then the kind's law, drawn from one default_rng(seed) stream."""
    rng = np.random.default_rng(spec.seed)
    labels = np.sort(rng.integers(0, spec.clusters, spec.n))
    labels[: spec.clusters] = np.arange(spec.clusters)
    labels = np.sort(labels)
    k = spec.clusters
    if spec.kind == "gaussian-mixture":
        means = spread_means(k, spec.dim, spec.separation, rng)
        points = means[labels] + rng.standard_normal((spec.n, spec.dim))
        radii = np.zeros(k)
        for j in range(k):
            radii[j] = np.sqrt(((points[labels == j] - means[j]) ** 2).sum(-1)).max()
        return SyntheticResult(DenseData(points), labels, radii)
    if spec.kind == "categorical-patterns":
        code_space = max(k * 2, 8)
        patterns = rng.integers(0, code_space, (k, spec.dim))
        codes = patterns[labels].copy()
        flips = rng.random((spec.n, spec.dim)) < (1.0 / max(spec.separation, 1.1))
        codes[flips] = rng.integers(0, code_space, int(flips.sum()))
        radii = np.zeros(k)
        for j in range(k):
            match = (codes[labels == j] == patterns[j]).sum(-1)
            radii[j] = (1.0 - match / (2 * spec.dim - match)).max()
        return SyntheticResult(CategoricalData(codes.astype(np.int32), code_space), labels, radii)
    universe = max(spec.dim, 16)
    base_size = max(universe // (k * 4), 8)
    bases = [np.sort(rng.choice(universe, base_size, replace=False)) for _ in range(k)]
    sets = []
    for lab in labels:
        base = bases[lab]
        mask = rng.random(base.size) < 0.95
        kept = base[mask] if mask.any() else base[:1]
        extras = rng.choice(universe, max(1, int(base_size * 0.05)), replace=False)
        sets.append(np.union1d(kept, extras))
    radii = np.zeros(k)
    for i, lab in enumerate(labels):
        inter = np.intersect1d(sets[i], bases[lab], assume_unique=True).size
        radii[lab] = max(radii[lab], 1.0 - inter / (sets[i].size + bases[lab].size - inter))
    return SyntheticResult(SparseData(sets, universe), labels, radii)


def spread_means(k: int, dim: int, separation: float, rng) -> np.ndarray:
    """Means on a jittered planar spiral, min pairwise distance = separation
    (synth.py:86-104); the min distance is evaluated in row blocks (same
    arithmetic per pair) so large k does not need a k*k*dim temporary."""
    if k == 1:
        return np.zeros((1, dim))
    idx = np.arange(k)
    rad = np.sqrt(idx + 0.5)
    ang = idx * (np.pi * (3.0 - np.sqrt(5.0)))
    plane = np.stack([rad * np.cos(ang), rad * np.sin(ang)], axis=1)
    plane += 0.05 * rng.standard_normal(plane.shape)
    basis = np.linalg.qr(rng.standard_normal((dim, min(2, dim))))[0]
    means = plane[:, : basis.shape[1]] @ basis.T
    dmin = np.inf
    step = max(1, (1 << 26) // max(1, k * dim))
    for lo in range(0, k, step):
        blk = np.sqrt(((means[lo:lo + step, None, :] - means[None, :, :]) ** 2).sum(-1))
        blk[np.arange(blk.shape[0]), lo + np.arange(blk.shape[0])] = np.inf
        dmin = min(dmin, float(blk.min()))
    return means * (separation / dmin)


def gaussian_mixture_host(n: int, dim: int, clusters: int, separation: float = 10.0, seed: int = 0):
    rng = np.random.default_rng(seed)
    labels = np.sort(rng.integers(0, clusters, n))
    labels[:clusters] = np.arange(clusters)
    labels = np.sort(labels)
    means = spread_means(clusters, dim, separation, rng)
    return means[labels] + rng.standard_normal((n, dim)), labels


def gaussian_mixture_device(n: int, dim: int, clusters: int, separation: float = 10.0, seed: int = 0,
                            row_lo: int = 0, rows: int = None, device=None, chunk: int = 1 << 22):
    """Rows [row_lo, row_lo + rows) of an n-point mixture as float32 on the GPU.

    Cluster sizes come from one seeded multinomial draw (identical on every
    rank), so shards of the same n/seed concatenate to the same dataset."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    rows = n - row_lo if rows is None else rows
    rng = np.random.default_rng(seed)
    sizes = rng.multinomial(n - clusters, np.full(clusters, 1.0 / clusters)) + 1
    means = torch.from_numpy(spread_means(clusters, dim, separation, rng).astype(np.float32)).to(device)
    bounds = np.concatenate(([0], np.cumsum(sizes)))
    X = torch.empty((rows, dim), dtype=torch.float32, device=device)
    gen = torch.Generator(device=device)
    ub = torch.from_numpy(bounds[1:]).to(device)
    # noise is drawn per global chunk so every sharding yields the same rows
    for c in range(row_lo // chunk, (row_lo + rows + chunk - 1) // chunk):
        g0, g1 = c * chunk, min(n, (c + 1) * chunk)
        a, b = max(g0, row_lo), min(g1, row_lo + rows)
        if a >= b:
            continue
        gen.manual_seed((seed * 1_000_003 + c) & ((1 << 63) - 1))
        noise = torch.randn((g1 - g0, dim), generator=gen, device=device, dtype=torch.float32)
        ids = torch.arange(a, b, device=device, dtype=torch.int64)
        lab = torch.searchsorted(ub, ids, right=True)
        X[a - row_lo:b - row_lo] = noise[a - g0:b - g0] + means[lab]
        del noise
    return X
