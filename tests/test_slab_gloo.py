"""World-size-2 (and 3) gloo test of the z-slab protocol on CPU (no GPU).

The library's NCCL transport (NcclComm in hf_lib.cu) exchanges, per rank, the first/last OWNED
node plane with the lower/upper neighbour into the neighbour's ghost plane, and sums per-rank
partial dot products over OWNED nodes.  This test drives the same protocol with
torch.distributed (gloo) on CPU using the library's own partition (hf_slab_plan), and checks
that (1) each rank's local planes (owned + one ghost per interior side) reproduce the global
operator apply on its owned planes (oracle row evaluator), and (2) the allreduced owned-only dots
equal the global dot (no double counting of ghost planes).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    import paper_1905_07622_b200 as hf
    import oracle
    import synth
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = synth.Grid((7, 6, 13), (0.3, 0.25, 0.2))
        nx1, ny1, nz1 = g.nn
        plane = nx1 * ny1
        k, c = synth.random_fields(g, seed=3)
        u = synth.random_vector(g.n_nodes, seed=4)
        lo, hi = hf.hf_slab_plan(nz1, rank, world)
        z0 = lo - (1 if rank > 0 else 0)
        z1 = hi + (1 if rank < world - 1 else 0)
        # local vector: owned planes from the global field, ghosts left at garbage (NaN)
        loc = np.full((z1 - z0) * plane, np.nan)
        loc[(lo - z0) * plane:(hi - z0) * plane] = u[lo * plane:hi * plane]
        t = torch.from_numpy(loc)
        # ghost exchange exactly as NcclComm::exchange: send first/last owned plane, receive ghosts
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(t[(lo - z0) * plane:(lo - z0 + 1) * plane].clone(), rank - 1))
            lo_ghost = torch.empty(plane, dtype=torch.float64)
            reqs.append(dist.irecv(lo_ghost, rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(t[(hi - z0 - 1) * plane:(hi - z0) * plane].clone(), rank + 1))
            hi_ghost = torch.empty(plane, dtype=torch.float64)
            reqs.append(dist.irecv(hi_ghost, rank + 1))
        for r in reqs:
            r.wait()
        if rank > 0:
            t[0:plane] = lo_ghost
        if rank < world - 1:
            t[(z1 - z0 - 1) * plane:] = hi_ghost
        loc = t.numpy()
        assert np.isfinite(loc).all(), "ghost plane not filled"
        # the owned rows of the global apply only depend on local planes: evaluate them from a
        # global vector holding ONLY this rank's local data (zeros elsewhere)
        only_local = np.zeros(g.n_nodes)
        only_local[z0 * plane:z1 * plane] = loc
        o = oracle.Oracle(g, k, c, assemble=False)
        rows = np.arange(lo * plane, hi * plane)
        y_loc = o.apply_rows(0.3, 1.0, only_local, rows)
        y_ref = o.apply_rows(0.3, 1.0, u, rows)
        err = float(np.abs(y_loc - y_ref).max() / np.abs(y_ref).max())
        # owned-only dot, summed across ranks
        d = torch.tensor([float(np.dot(loc[(lo - z0) * plane:(hi - z0) * plane],
                                       loc[(lo - z0) * plane:(hi - z0) * plane]))], dtype=torch.float64)
        dist.all_reduce(d)
        q.put((rank, lo, hi, z0, z1, err, float(d.item()), float(np.dot(u, u))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in procs]
    [p.join(timeout=120) for p in procs]
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = sorted(q.get() for _ in range(world))
    # the partition covers all planes contiguously
    assert res[0][1] == 0 and res[-1][2] == 14
    for a, b in zip(res, res[1:]):
        assert a[2] == b[1]
    for rank, lo, hi, z0, z1, err, dot, dot_ref in res:
        assert err <= 1e-14, (rank, err)
        assert abs(dot - dot_ref) <= 1e-12 * dot_ref
