"""Synthetic inputs with the reference generator's law (synth.py:39-104).

`gaussian_mixture_host` reproduces gen_synthetic("gaussian-mixture") exactly
(same numpy stream) for parity-sized inputs; `gaussian_mixture_device`
draws the same law at benchmark scale directly into HBM: cluster means from
the host spiral (`spread_means`), labels uniform then sorted (so ids are
cluster-contiguous, as in the reference), x = mean + N(0, 1) from torch's
Philox generator, float32.
"""

from __future__ import annotations

import numpy as np
import torch


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
