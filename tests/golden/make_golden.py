"""Dump golden vectors from the REAL reference (lshclust) into tests/golden/.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python tests/golden/make_golden.py

The outputs are small .npz / .json fixtures committed to the repo; the
oracle (oracle/geek_oracle.py) is pinned against them by
tests/test_oracle_golden.py and the CUDA path is checked against both.
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

from lshclust import hashing, transform, seeding, assignment, data as D  # noqa: E402
from lshclust.engine import PipelineConfig, WorkerConfig, run_pipeline  # noqa: E402
from lshclust.synth import SyntheticSpec, gen_synthetic  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def codes_from_buckets(buckets, n, ntables):
    codes = np.full((ntables, n), -1, dtype=np.int64)
    for b in buckets:
        codes[b.table, b.members] = b.slot
    return codes


def seeds_and_pi():
    rng = np.random.default_rng(123)
    seeds = {}
    cases = [(0, ()), (1, (0,)), (2, (3, 1)), (2**64 - 1, (7, 8, 9)), (12345, (0xDED0,)), (99, (0xD0,))]
    seeds["derive"] = [[m, list(p), hashing.derive_seed(m, *p)] for m, p in cases]
    seeds["splitmix"] = [[z, hashing.splitmix64(z)] for z in (0, 1, 2**63, 2**64 - 1, 0xDEADBEEF)]
    pis = {}
    for seed, u in [(7, 6), (42, 100), (3, 4096), (7, 4097), (11, 65536), (5, 100_000),
                    (9, 1_000_003), (13, 100_000_000), (17, 3_000_000), (19, 39 * 1_000_000),
                    (2**63 + 5, 1 << 20), (23, 2_000_000_000)]:
        f = hashing.MinHashFunction(seed, u)
        if u <= 4096:
            x = np.arange(u)
        else:
            x = np.unique(np.concatenate([[0, 1, u - 1, u - 2], rng.integers(0, u, 3000)]))
        pis[f"{seed}_{u}"] = dict(seed=seed, u=u, x=x.astype(np.int64), y=f.permute(x).astype(np.uint64))
    return seeds, pis


def main():
    t0 = time.time()
    meta = {}
    seeds, pis = seeds_and_pi()
    meta["seeds"] = seeds
    np.savez_compressed(os.path.join(OUT, "pi.npz"), **{
        f"{k}_{f}": v[f] for k, v in pis.items() for f in ("x", "y")
    })
    meta["pi_cases"] = [[v["seed"], v["u"], k] for k, v in pis.items()]

    # set signatures over random sets (SignatureScheme.signatures_for_sets)
    rng = np.random.default_rng(5)
    sig_cases = {}
    for (K, L, u, seed) in [(3, 4, 700, 13), (2, 3, 5000, 1), (3, 2, 100_000, 2)]:
        sch = hashing.SignatureScheme(K, L, u, seed=seed)
        sets = [np.unique(rng.integers(0, u, rng.integers(1, 40))) for _ in range(50)]
        flat = np.concatenate(sets)
        off = np.concatenate(([0], np.cumsum([s.size for s in sets])))
        for tb in range(L):
            sig_cases[f"{K}_{L}_{u}_{seed}_{tb}"] = np.asarray(sch.signatures_for_sets(tb, sets), dtype=np.uint64)
        sig_cases[f"{K}_{L}_{u}_{seed}_flat"] = flat
        sig_cases[f"{K}_{L}_{u}_{seed}_off"] = off
    np.savez_compressed(os.path.join(OUT, "sigs.npz"), **sig_cases)

    # projection directions (ProjectionFunction.from_seed)
    dirs = {f"{s}_{j}_{d}": hashing.ProjectionFunction.from_seed(s, j, d).direction
            for s, j, d in [(1, 0, 128), (1, 19, 128), (2**64 - 1, 3, 16), (7, 0, 960)]}
    np.savez_compressed(os.path.join(OUT, "dirs.npz"), **dirs)

    # DOPH
    red = hashing.DophReducer(5, 12, 4)
    meta["doph_sketch_5_12_4"] = red.sketch(np.array([0, 5])).tolist()
    red2 = hashing.DophReducer(hashing.derive_seed(3, 0xD0), 3_000_000, 400)
    dsets = [np.unique(rng.integers(0, 3_000_000, rng.integers(1, 200))) for _ in range(100)]
    np.savez_compressed(os.path.join(OUT, "doph.npz"),
                        flat=np.concatenate(dsets),
                        off=np.concatenate(([0], np.cumsum([s.size for s in dsets]))),
                        red_flat=np.concatenate([red2.reduce(s) for s in dsets]),
                        red_off=np.concatenate(([0], np.cumsum([red2.reduce(s).size for s in dsets]))))

    # dense pipelines ------------------------------------------------------
    pipes = {}

    def dense_case(name, spec, m, t, L, K, delta, gs, tseed=1, sseed=2):
        res = gen_synthetic(spec)
        X = res.data.vectors
        bk = transform.transform_homo(res.data, transform.HomoTransformParams(m, t, seed=tseed))
        codes = codes_from_buckets(bk, X.shape[0], m)
        entry = dict(spec=[spec.kind, spec.n, spec.dim, spec.clusters, spec.separation, spec.seed],
                     m=m, t=t, L=L, K=K, delta=delta, tseed=tseed, sseed=sseed,
                     data_sha=sha(X), codes_sha=sha(codes.astype(np.int32)), runs={})
        arrays = {}
        if X.shape[0] * m <= 200_000:
            arrays[f"{name}_codes"] = codes.astype(np.int32)
        for g in gs:
            cfg = PipelineConfig(metric="euclidean", transform_kind="dense",
                                 workers=WorkerConfig(g),
                                 homo=transform.HomoTransformParams(m, t, seed=tseed),
                                 seeding=seeding.SeedingParams(K, L, min_group_size=delta, seed=sseed))
            t1 = time.time()
            out = run_pipeline(res.data, cfg)
            el = time.time() - t1
            grp = out.seed_groups
            arrays[f"{name}_g{g}_gflat"] = np.concatenate([x.members for x in grp]) if grp else np.zeros(0, np.int64)
            arrays[f"{name}_g{g}_goff"] = np.concatenate(([0], np.cumsum([len(x) for x in grp])))
            C = np.stack([c.values for c in out.clustering.centers])
            arrays[f"{name}_g{g}_centers"] = C
            arrays[f"{name}_g{g}_labels"] = out.clustering.assignment.astype(np.int32)
            arrays[f"{name}_g{g}_radii"] = out.clustering.radii
            entry["runs"][str(g)] = dict(k_star=out.k_star, ngroups=len(grp), objective=out.clustering.objective,
                                        seconds=el, timings=out.timings, warnings=out.warnings)
            print(name, g, "k*", out.k_star, "groups", len(grp), f"{el:.1f}s", flush=True)
        pipes[name] = entry
        return arrays

    arrays = {}
    arrays.update(dense_case("c06", SyntheticSpec("gaussian-mixture", 2000, 16, 10, 20.0, 0),
                             48, 10, 48, 3, 5, (1, 2, 4)))
    arrays.update(dense_case("small", SyntheticSpec("gaussian-mixture", 3000, 8, 6, 12.0, 4),
                             8, 30, 8, 3, 3, (1, 2, 8)))
    arrays.update(dense_case("cfg1", SyntheticSpec("gaussian-mixture", 100_000, 128, 100, 10.0, 0),
                             20, 100, 20, 3, 10, (1, 8)))
    meta["pipelines"] = pipes

    # c08 assignment oracle (test_acceptance.py:305-347)
    rng = np.random.default_rng(80)
    dense = D.DenseData(rng.standard_normal((10_000, 16)))
    cents = [D.CentralVector("centroid", rng.standard_normal(16)) for _ in range(200)]
    got = assignment.assign(dense, cents, "euclidean")
    arrays["c08_labels"] = got.assignment.astype(np.int32)
    arrays["c08_radii"] = got.radii
    meta["c08_objective"] = got.objective
    codes = rng.integers(0, 8, (10_000, 9)).astype(np.int32)
    modes = [D.CentralVector("mode", rng.integers(0, 8, 9).astype(np.int32)) for _ in range(200)]
    got = assignment.assign(D.CategoricalData(codes, code_space=8), modes, "jaccard")
    arrays["c08cat_labels"] = got.assignment.astype(np.int32)
    arrays["c08cat_radii"] = got.radii

    # sparse pipeline ------------------------------------------------------
    res = gen_synthetic(SyntheticSpec("sparse-overlap", 1500, 20_000, 15, 10.0, 3))
    mp = transform.MinhashTransformParams(3, 6, seed=4, target_dims=400)
    bk, red = transform.transform_sparse(res.data, mp)
    arrays["sp_flat"] = np.concatenate(res.data.sets)
    arrays["sp_off"] = np.concatenate(([0], np.cumsum([s.size for s in res.data.sets])))
    arrays["sp_red_flat"] = np.concatenate(red.sets)
    arrays["sp_red_off"] = np.concatenate(([0], np.cumsum([s.size for s in red.sets])))
    arrays["sp_codes"] = codes_from_buckets(bk, res.data.n, 6).astype(np.int32)
    sp_runs = {}
    for g in (1, 2):
        cfg = PipelineConfig(metric="jaccard", transform_kind="sparse", workers=WorkerConfig(g),
                             minhash=mp, seeding=seeding.SeedingParams(3, 6, min_group_size=3, seed=5))
        out = run_pipeline(res.data, cfg)
        grp = out.seed_groups
        arrays[f"sp_g{g}_gflat"] = np.concatenate([x.members for x in grp]) if grp else np.zeros(0, np.int64)
        arrays[f"sp_g{g}_goff"] = np.concatenate(([0], np.cumsum([len(x) for x in grp])))
        arrays[f"sp_g{g}_centers"] = np.stack([c.values for c in out.clustering.centers])
        arrays[f"sp_g{g}_labels"] = out.clustering.assignment.astype(np.int32)
        arrays[f"sp_g{g}_radii"] = out.clustering.radii
        sp_runs[str(g)] = dict(k_star=out.k_star, objective=out.clustering.objective, warnings=out.warnings)
        print("sparse", g, out.k_star, len(grp), flush=True)
    meta["sparse"] = dict(spec=["sparse-overlap", 1500, 20_000, 15, 10.0, 3], K=3, L=6, tseed=4,
                          target_dims=400, sK=3, sL=6, delta=3, sseed=5, runs=sp_runs)

    # mixed pipeline -------------------------------------------------------
    rng = np.random.default_rng(11)
    nm = 1200
    lab = np.sort(rng.integers(0, 8, nm))
    num = rng.lognormal(mean=lab[:, None] * 0.5, sigma=0.3, size=(nm, 3))
    cat = (lab[:, None] * 3 + rng.integers(0, 2, (nm, 4))).astype(np.int32)
    mixed = D.MixedData(num, cat)
    mp2 = transform.MinhashTransformParams(3, 6, seed=7, bins_per_attribute=16)
    bk, unified = transform.transform_hetero(mixed, mp2)
    arrays["mx_num"] = num
    arrays["mx_cat"] = cat
    arrays["mx_unified"] = unified.codes
    arrays["mx_codes"] = codes_from_buckets(bk, nm, 6).astype(np.int32)
    mx_runs = {}
    for g in (1, 2):
        cfg = PipelineConfig(metric="jaccard", transform_kind="mixed", workers=WorkerConfig(g),
                             minhash=mp2, seeding=seeding.SeedingParams(3, 6, min_group_size=3, seed=9))
        out = run_pipeline(mixed, cfg)
        grp = out.seed_groups
        arrays[f"mx_g{g}_gflat"] = np.concatenate([x.members for x in grp]) if grp else np.zeros(0, np.int64)
        arrays[f"mx_g{g}_goff"] = np.concatenate(([0], np.cumsum([len(x) for x in grp])))
        arrays[f"mx_g{g}_centers"] = np.stack([c.values for c in out.clustering.centers])
        arrays[f"mx_g{g}_labels"] = out.clustering.assignment.astype(np.int32)
        arrays[f"mx_g{g}_radii"] = out.clustering.radii
        mx_runs[str(g)] = dict(k_star=out.k_star, objective=out.clustering.objective, warnings=out.warnings)
        print("mixed", g, out.k_star, len(grp), flush=True)
    meta["mixed"] = dict(n=nm, K=3, L=6, tseed=7, bins=16, sK=3, sL=6, delta=3, sseed=9, runs=mx_runs)

    np.savez_compressed(os.path.join(OUT, "pipelines.npz"), **arrays)
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, default=lambda o: int(o) if isinstance(o, np.integer) else float(o))
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
