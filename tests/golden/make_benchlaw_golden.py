"""Golden outputs of the REAL reference (lshclust.run_pipeline) on a reduced-n
instance of the benchmark's law.

bench.py runs 100M x 128 float32 points drawn from the reference generator's
gaussian-mixture law with C = 1000 planted clusters, t = n / C buckets per
table (one planted cluster's worth of points per bucket), m = 40, L = 20,
K = 2, delta = 10, g = 8 logical workers.  The same law at n = 1M is C = 1000,
t = 1000 (buckets of 1000 = one cluster): k* ~ 1000 seed groups, the regime
the benchmark measures.  Data: `gen_synthetic` itself (synth.py:39-51), cast
to float32 as the benchmark holds it (DenseData coerces it back to float64,
data.py:49, exactly).

Run in the build container only (imports /root/reference/pkg/src):

    python tests/golden/make_benchlaw_golden.py [n]

Writes tests/golden/benchlaw.npz + benchlaw.json.  Besides the pipeline
outputs it records, per table, the sha256 of the reference bucket codes and
the reference's own near-boundary statistics: how many ids' float64
projections lie within 1e-12 / 1e-6 (relative) of a rank-split boundary
(transform.py:103-109, engine.py:216-225), and the ids within 1e-9 with their
reference codes -- the only ids whose code may legitimately differ under a
different float64 summation order.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from lshclust import seeding, transform  # noqa: E402
from lshclust.engine import PipelineConfig, WorkerConfig, run_pipeline, split_data  # noqa: E402
from lshclust.synth import SyntheticSpec, gen_synthetic  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    C = 1000
    d, m, L, K, delta, g, tseed, sseed = 128, 40, 20, 2, 10, 8, 1, 2
    t = n // (n // C)  # buckets of one planted cluster's worth of points (= C)
    t0 = time.time()
    res = gen_synthetic(SyntheticSpec("gaussian-mixture", n, d, C, 10.0, 0))
    X32 = res.data.vectors.astype(np.float32)
    from lshclust.data import DenseData
    data = DenseData(X32)
    print(f"data {time.time() - t0:.1f}s", flush=True)

    homo = transform.HomoTransformParams(m, t, seed=tseed)
    # reference projections exactly as the engine forms them (engine.py:178-181:
    # per worker shard, then concatenated in worker order, engine.py:218-220)
    codes_sha, near_ids, near_codes, near_tab = [], [], [], []
    cnt12, cnt6, cnt9 = [], [], []
    sizes = transform.even_partition_sizes(n, t)
    bounds = np.cumsum(sizes)[:-1]
    shards = split_data(n, g)
    for table in range(m):
        a = homo.projection(table, d).direction
        v = np.concatenate([data.vectors[lo:hi] @ a for lo, hi in shards])
        order = np.lexsort((np.arange(n), v))
        codes = np.empty(n, np.int32)
        codes[order] = np.repeat(np.arange(t, dtype=np.int32), sizes)
        codes_sha.append(sha(codes))
        vs = v[order]
        mid = vs[bounds - 1] + 0.5 * (vs[bounds] - vs[bounds - 1])  # t-1 boundary midpoints
        # distance of every id's key to its nearest boundary midpoint
        pos = np.searchsorted(mid, v)
        lo_mid = mid[np.clip(pos - 1, 0, t - 2)]
        hi_mid = mid[np.clip(pos, 0, t - 2)]
        dist = np.minimum(np.abs(v - lo_mid), np.abs(v - hi_mid))
        scale = np.maximum(np.abs(lo_mid), np.abs(hi_mid))
        rel = dist / np.where(scale > 0, scale, 1.0)
        cnt12.append(int((rel <= 1e-12).sum()))
        cnt6.append(int((rel <= 1e-6).sum()))
        sel = np.nonzero(rel <= 1e-9)[0]
        cnt9.append(int(sel.size))
        near_ids.append(sel.astype(np.int32))
        near_codes.append(codes[sel])
        near_tab.append(np.full(sel.size, table, np.int32))
    print(f"codes {time.time() - t0:.1f}s near(1e-12)={sum(cnt12)} near(1e-9)={sum(cnt9)} "
          f"near(1e-6)={sum(cnt6)}", flush=True)

    cfg = PipelineConfig(metric="euclidean", transform_kind="dense", workers=WorkerConfig(g), homo=homo,
                         seeding=seeding.SeedingParams(K, L, min_group_size=delta, seed=sseed))
    t1 = time.time()
    out = run_pipeline(data, cfg)
    el = time.time() - t1
    grp = out.seed_groups
    cl = out.clustering
    C_ = np.stack([c.values for c in cl.centers])
    arrays = dict(
        gflat=np.concatenate([x.members for x in grp]).astype(np.int32) if grp else np.zeros(0, np.int32),
        goff=np.concatenate(([0], np.cumsum([len(x) for x in grp]))).astype(np.int64),
        centers=C_, weights=np.array([c.weight for c in cl.centers], np.int64),
        labels=cl.assignment.astype(np.int32), radii=cl.radii,
        near_tab=np.concatenate(near_tab), near_ids=np.concatenate(near_ids),
        near_codes=np.concatenate(near_codes),
    )
    np.savez_compressed(os.path.join(OUT, "benchlaw.npz"), **arrays)
    meta = dict(n=n, d=d, clusters=C, separation=10.0, data_seed=0, m=m, t=t, L=L, K=K, delta=delta, g=g,
                tseed=tseed, sseed=sseed, data_sha=sha(X32), codes_sha=codes_sha,
                near_1e12=cnt12, near_1e9=cnt9, near_1e6=cnt6,
                k_star=int(out.k_star), ngroups=len(grp), objective=float(cl.objective),
                seconds=el, timings=out.timings, warnings=out.warnings,
                transport_bytes=dict(out.transport_bytes), cpu_count=os.cpu_count(),
                openblas_threads=os.environ.get("OPENBLAS_NUM_THREADS"))
    with open(os.path.join(OUT, "benchlaw.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"run_pipeline {el:.1f}s k*={out.k_star} groups={len(grp)} timings={out.timings}", flush=True)


if __name__ == "__main__":
    main()
