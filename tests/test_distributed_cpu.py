"""Multi-process plumbing of the engine on CPU (gloo, world_size 2 and 4): table
routing to owners (engine.py:199-238) for projection keys and signature rows,
the sharded per-attribute mode reduction, seed-group all-gather (engine.py:285-295),
the float64 radii MAX reduction over bit patterns, the variable-size gather and
the sharded numpy-order pairwise sum of the objective.
The kernels themselves need a GPU; these tests cover the host-side exchange
logic that the NCCL runs use unchanged."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2106_10515_b200.engine import _Comm, _merge_groups, route_tables, split_data
        from paper_2106_10515_b200.tables import GroupSet

        comm = _Comm()
        assert comm.on and comm.G == world and comm.rank == rank
        full = torch.arange(m * n, dtype=torch.int64).view(m, n) * 7 + 3
        lo, hi = split_data(n, world)[rank]
        own = route_tables(full[:, lo:hi].contiguous(), n, comm)
        want = full[[j for j in range(m) if j % world == rank]]
        ok_route = bool(torch.equal(own, want))
        # seed groups: rank r contributes r+1 groups
        groups = [np.arange(rank * 10 + g, rank * 10 + g + 3) for g in range(rank + 1)]
        sizes = np.array([g.size for g in groups])
        off = np.concatenate(([0], np.cumsum(sizes)))
        gs = GroupSet(torch.from_numpy(np.concatenate(groups).astype(np.int32)), torch.from_numpy(off))
        merged = _merge_groups(comm, gs)
        got = [merged.flat[merged.off[i]:merged.off[i + 1]].tolist() for i in range(merged.count)]
        exp = [list(range(r * 10 + g, r * 10 + g + 3)) for r in range(world) for g in range(r + 1)]
        ok_merge = got == exp
        # radii: MAX over non-negative float64 bit patterns
        radii = torch.tensor([0.5, 2.0 + rank, 1e-300 * (rank + 1), 0.0], dtype=torch.float64)
        comm.all_reduce(radii.view(torch.int64), dist.ReduceOp.MAX, "Assignments")
        ok_radii = radii.tolist() == [0.5, 2.0 + world - 1, 1e-300 * world, 0.0]
        v = comm.all_gather_var(torch.arange(rank + 2, dtype=torch.float64), "Assignments")
        ok_gather = v.tolist() == [float(x) for r in range(world) for x in range(r + 2)]
        # objective: numpy's pairwise sum of the sharded best distances, exact
        import paper_2106_10515_b200.engine as E
        E.pairwise_sum = lambda t: torch.tensor([float(np.add.reduce(t.numpy()))], dtype=torch.float64)
        ok_pw = True
        for npts in (5, 130, 1000, 20_011):
            vals = np.random.default_rng(npts).standard_normal(npts) * 10.0 ** np.random.default_rng(1).integers(
                -8, 8, npts)
            plo, phi = split_data(npts, world)[rank]
            got_pw = E.sharded_pairwise_sum(torch.from_numpy(vals[plo:phi].copy()), npts, plo, comm)
            ok_pw &= got_pw == float(np.add.reduce(vals))
        # signature rows routed to table owners, and the sharded mode reduction
        from paper_2106_10515_b200.engine import _dist_modes, route_signature_rows
        K = 3
        sig_full = (torch.arange(n * m * K, dtype=torch.int32).view(n, m * K) * 13) % 1009
        got_sig = route_signature_rows(sig_full[lo:hi].contiguous(), n, K, comm)
        own_t = [j for j in range(m) if j % world == rank]
        want_sig = sig_full.view(n, m, K)[:, own_t, :].permute(1, 0, 2)
        ok_route &= bool(torch.equal(got_sig, want_sig))
        rng = np.random.default_rng(7)
        kk, cs, dd = 6, 50, 2
        grp = rng.integers(0, kk, n)
        cod = rng.integers(0, cs, (n, dd))
        keys = [torch.from_numpy(grp[lo:hi] * cs + cod[lo:hi, c]).to(torch.int64) for c in range(dd)]
        modes = _dist_modes(keys, kk, cs, comm).numpy()
        for gi in range(kk):
            for c in range(dd):
                vals = cod[grp == gi, c]
                want = np.argmax(np.bincount(vals, minlength=cs)) if vals.size else cs
                ok_merge &= int(modes[gi, c]) == int(want)
        q.put((rank, ok_route, ok_merge, ok_radii, ok_gather and ok_pw, dict(comm.bytes)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,m", [(2, 103, 5), (2, 40, 8), (4, 103, 5), (4, 1001, 9)])
def test_engine_exchanges_gloo(world, n, m):
    """world 2 and 4, n not divisible by the world size, m not a multiple of it"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_route, ok_merge, ok_radii, ok_gather, nbytes in res:
        assert ok_route, rank
        assert ok_merge, rank
        assert ok_radii, rank
        assert ok_gather, rank
        assert nbytes.get("BucketShard", 0) > 0 and nbytes.get("SeedGroups", 0) > 0
