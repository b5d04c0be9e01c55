"""Multi-GPU parity: run under torchrun with G ranks; the sharded NCCL engine
must reproduce the golden single-process reference outputs exactly.

    torchrun --standalone --local-addr 127.0.0.1 --nproc-per-node 2 tools/mgpu_check.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2106_10515_b200 as G  # noqa: E402
from oracle import geek_oracle as O  # noqa: E402
from tests.golden_io import groups as golden_groups, meta, npz, refine_meta  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    arr = npz("pipelines")
    ok = True
    for name in ("c06", "small", "cfg1"):
        m = meta()["pipelines"][name]
        _, n, d, C, sep, seed = m["spec"]
        X, _ = O.gaussian_mixture(n, d, C, sep, seed)
        for g in m["runs"]:
            if int(g) % world:
                continue
            cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(int(g)),
                                   homo=G.HomoTransformParams(m["m"], m["t"], seed=m["tseed"]),
                                   seeding=G.SeedingParams(m["K"], m["L"], min_group_size=m["delta"],
                                                           seed=m["sseed"]))
            out = G.run_pipeline(G.DenseData(X), cfg)
            got = [tuple(x.members.tolist()) for x in out.seed_groups]
            want = [tuple(x.tolist()) for x in golden_groups(arr, f"{name}_g{g}")]
            cl = out.clustering
            good = (got == want and np.array_equal(cl.assignment, arr[f"{name}_g{g}_labels"])
                    and np.array_equal(cl.radii, arr[f"{name}_g{g}_radii"])
                    and np.array_equal(np.stack([c.values for c in cl.centers]), arr[f"{name}_g{g}_centers"])
                    and cl.objective == m["runs"][g]["objective"])
            ok &= good
            if rank == 0:
                print(f"[G={world}] {name} g={g}: {'OK' if good else 'MISMATCH'} groups={len(got)} "
                      f"bytes={out.transport_bytes}", flush=True)
    # float32 rows take the routed projection (keys stored into the owners'
    # symmetric buffers); checked against the oracle on the float32 values
    for name in ("c06", "small"):
        m = meta()["pipelines"][name]
        _, n, d, C, sep, seed = m["spec"]
        X, _ = O.gaussian_mixture(n, d, C, sep, seed)
        X = X.astype(np.float32)
        for g in m["runs"]:
            if int(g) % world:
                continue
            cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(int(g)),
                                   homo=G.HomoTransformParams(m["m"], m["t"], seed=m["tseed"]),
                                   seeding=G.SeedingParams(m["K"], m["L"], min_group_size=m["delta"],
                                                           seed=m["sseed"]))
            out = G.run_pipeline(G.DenseData(X), cfg)
            ref = O.pipeline_dense(X.astype(np.float64), m["m"], m["t"], m["tseed"], m["K"], m["L"], m["delta"],
                                   m["sseed"], g=int(g))
            got = [tuple(x.members.tolist()) for x in out.seed_groups]
            want = [tuple(np.asarray(x.members if hasattr(x, "members") else x).tolist()) for x in ref["groups"]]
            good = (got == want and np.array_equal(out.clustering.assignment, ref["labels"])
                    and np.array_equal(out.clustering.radii, ref["radii"]))
            ok &= good
            if rank == 0:
                print(f"[G={world}] {name} f32 g={g}: {'OK' if good else 'MISMATCH'} groups={len(got)} "
                      f"bytes={out.transport_bytes} warnings={out.warnings if hasattr(out, 'warnings') else ''}",
                      flush=True)
    # refinement passes across ranks (engine.py:519-537): label-keyed digit
    # sums all-reduced, against the reference's run_pipeline(passes=2)
    rarr, rmeta = npz("refine"), refine_meta()
    m = meta()["pipelines"]["small"]
    _, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    for g in (1, 2):
        if g % world:
            continue
        for x in (X, X.astype(np.float32)):
            cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(g),
                                   homo=G.HomoTransformParams(m["m"], m["t"], seed=m["tseed"]),
                                   seeding=G.SeedingParams(m["K"], m["L"], min_group_size=m["delta"],
                                                           seed=m["sseed"]), passes=2)
            cl = G.run_pipeline(G.DenseData(x), cfg).clustering
            if x.dtype == np.float32:
                ref = O.pipeline_dense(x.astype(np.float64), m["m"], m["t"], m["tseed"], m["K"], m["L"],
                                       m["delta"], m["sseed"], g=g, passes=2)
                good = (np.array_equal(cl.assignment, ref["labels"]) and cl.objective == ref["objective"]
                        and np.array_equal(np.stack([c.values for c in cl.centers]), ref["centers"]))
            else:
                nm = f"small_p2_g{g}"
                good = (np.array_equal(cl.assignment, rarr[f"{nm}_labels"])
                        and np.array_equal(cl.radii, rarr[f"{nm}_radii"])
                        and np.array_equal(np.stack([c.values for c in cl.centers]), rarr[f"{nm}_centers"])
                        and cl.objective == rmeta[nm]["objective"])
            ok &= good
            if rank == 0:
                print(f"[G={world}] small passes=2 {x.dtype} g={g}: {'OK' if good else 'MISMATCH'}", flush=True)
    # sparse and mixed pipelines over the ranks (signature rows routed to the
    # table owners, counts summed): the reference's g = 2 goldens
    from tests.golden_io import csr as _csr
    if 2 % world == 0:
        sm = meta()["sparse"]
        data = G.SparseData(_csr(arr["sp_flat"], arr["sp_off"]), 20_000)
        cfg = G.PipelineConfig(metric="jaccard", transform_kind="sparse", workers=G.WorkerConfig(2),
                               minhash=G.MinhashTransformParams(3, 6, seed=4, target_dims=400),
                               seeding=G.SeedingParams(3, 6, min_group_size=3, seed=5))
        out = G.run_pipeline(data, cfg)
        cl = out.clustering
        good = ([tuple(x.members.tolist()) for x in out.seed_groups] ==
                [tuple(x.tolist()) for x in golden_groups(arr, "sp_g2")]
                and np.array_equal(np.stack([c.values for c in cl.centers]), arr["sp_g2_centers"])
                and np.array_equal(cl.assignment, arr["sp_g2_labels"]) and np.array_equal(cl.radii, arr["sp_g2_radii"])
                and cl.objective == sm["runs"]["2"]["objective"])
        ok &= good
        if rank == 0:
            print(f"[G={world}] sparse g=2: {'OK' if good else 'MISMATCH'} bytes={out.transport_bytes}", flush=True)
        mm = meta()["mixed"]
        cfg = G.PipelineConfig(metric="jaccard", transform_kind="mixed", workers=G.WorkerConfig(2),
                               minhash=G.MinhashTransformParams(3, 6, seed=7, bins_per_attribute=16),
                               seeding=G.SeedingParams(3, 6, min_group_size=3, seed=9))
        out = G.run_pipeline(G.MixedData(arr["mx_num"], arr["mx_cat"]), cfg)
        cl = out.clustering
        good = ([tuple(x.members.tolist()) for x in out.seed_groups] ==
                [tuple(x.tolist()) for x in golden_groups(arr, "mx_g2")]
                and np.array_equal(np.stack([c.values for c in cl.centers]), arr["mx_g2_centers"])
                and np.array_equal(cl.assignment, arr["mx_g2_labels"]) and np.array_equal(cl.radii, arr["mx_g2_radii"])
                and cl.objective == mm["runs"]["2"]["objective"])
        ok &= good
        if rank == 0:
            print(f"[G={world}] mixed g=2: {'OK' if good else 'MISMATCH'} bytes={out.transport_bytes}", flush=True)
    # the fused projection (keys stored into the owners' symmetric buffers over
    # NVLink) against projection + all_to_all of the same rows, and host rows
    # streamed through the API against device rows
    from paper_2106_10515_b200 import engine as E
    from paper_2106_10515_b200.transform import project_keys
    comm = E._Comm()
    rng = np.random.default_rng(5)
    for n, d, m in ((10_007, 128, 40), (3001, 32, 7)):
        Xf = rng.standard_normal((n, d)).astype(np.float32)
        A = rng.standard_normal((m, d))
        lo, hi = E.split_data(n, world)[rank]
        Xl = torch.from_numpy(Xf[lo:hi]).cuda()
        er = torch.tensor([1 << 30, -(1 << 30)], dtype=torch.int32, device="cuda")
        assert E._symm_ready(comm, -(-m // world), n, Xl.device)
        routed = E.project_routed(Xl, A, n, lo, comm, er).clone()
        a2a = E.route_tables(project_keys(Xl, A), n, comm)
        good = bool(torch.equal(routed, a2a))
        ok &= good
        if rank == 0:
            print(f"[G={world}] routed projection == all_to_all (n={n}, d={d}, m={m}): {'OK' if good else 'MISMATCH'}",
                  flush=True)
    m = meta()["pipelines"]["cfg1"]
    _, n, d, C, sep, seed = m["spec"]
    X, _ = O.gaussian_mixture(n, d, C, sep, seed)
    X = X.astype(np.float32)
    lo, hi = E.split_data(n, world)[rank]
    cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(8),
                           homo=G.HomoTransformParams(m["m"], m["t"], seed=m["tseed"]),
                           seeding=G.SeedingParams(m["K"], m["L"], min_group_size=m["delta"], seed=m["sseed"]))
    dev = G.run_pipeline_shard(torch.from_numpy(X[lo:hi]).cuda(), n, cfg)
    host = G.run_pipeline_shard(torch.from_numpy(X[lo:hi]).pin_memory(), n, cfg)
    good = (torch.equal(dev.labels_device, host.labels_device) and torch.equal(dev.radii_device, host.radii_device)
            and dev.objective == host.objective)
    ok &= good
    if rank == 0:
        print(f"[G={world}] host rows streamed == device rows (cfg1 f32): {'OK' if good else 'MISMATCH'}", flush=True)
    # the benchmark's law at 1M against the reference (tests/golden/benchlaw.*)
    import json as _json
    bpath = os.path.join(ROOT, "tests", "golden", "benchlaw.json")
    if os.path.exists(bpath):
        bm = _json.load(open(bpath))
        barr = np.load(os.path.join(ROOT, "tests", "golden", "benchlaw.npz"))
        Xb, _ = O.gaussian_mixture(bm["n"], bm["d"], bm["clusters"], bm["separation"], bm["data_seed"])
        Xb = Xb.astype(np.float32)
        lo, hi = E.split_data(bm["n"], world)[rank]
        cfg = G.PipelineConfig(metric="euclidean", transform_kind="dense", workers=G.WorkerConfig(bm["g"]),
                               homo=G.HomoTransformParams(bm["m"], bm["t"], seed=bm["tseed"]),
                               seeding=G.SeedingParams(bm["K"], bm["L"], min_group_size=bm["delta"],
                                                       seed=bm["sseed"]))
        out = G.run_pipeline_shard(torch.from_numpy(Xb[lo:hi]).cuda(), bm["n"], cfg)
        grp = out.seed_groups
        cl = out.clustering
        good = (np.array_equal(np.concatenate([x.members for x in grp]).astype(np.int32), barr["gflat"])
                and np.array_equal(np.stack([c.values for c in cl.centers]), barr["centers"])
                and np.array_equal(cl.assignment, barr["labels"]) and np.array_equal(cl.radii, barr["radii"])
                and cl.objective == bm["objective"])
        ok &= good
        if rank == 0:
            print(f"[G={world}] bench law 1M vs reference: {'OK' if good else 'MISMATCH'} groups={len(grp)} "
                  f"bytes={out.transport_bytes}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
