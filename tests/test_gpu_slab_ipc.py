"""z-slabs over peer memory between PROCESSES (transport 2, the bench's N > 1 path): two ranks,
one process each, mailboxes mapped with CUDA IPC, blobs all-gathered with torch.distributed
(gloo).  On this one-GPU box both processes share the B200 (time-sliced), which exercises the
IPC handshake, the in-kernel publish / wait protocol and the ghost-plane stores exactly as on
two GPUs.  Checked against the single-context run and the oracle (P:247-262 split, Alg. 1).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q, grid_args, nsteps):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import torch
        import torch.distributed as dist
        import paper_1905_07622_b200 as hf
        import synth
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        dev = torch.device("cuda:0")
        g = synth.Grid(*grid_args)
        k, c = synth.random_fields(g, seed=91)
        ctx = hf.hf_create_slab(g, rank, world, None, transport=hf.TRANSPORT_PEER_IPC, device=0)

        def all_gather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out
        hf.hf_peer_setup(ctx, all_gather)
        lo, hi, lp, z0 = ctx.slab
        plane = (g.ne[0] + 1) * (g.ne[1] + 1)
        hf.hf_set_coefficients(ctx, torch.tensor(k, device=dev), torch.tensor(c, device=dev))
        F = torch.empty(ctx.n_nodes, dtype=torch.float64, device=dev)
        hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
        u0 = synth.random_vector(g.n_nodes, 92) * 0.01
        u = torch.tensor(u0[z0 * plane:(z0 + lp) * plane], device=dev)
        st = hf.hf_simulate(ctx, 0.5, 0.05, nsteps, F, u)
        x = torch.zeros_like(u)
        b = torch.tensor(synth.random_vector(g.n_nodes, 93)[z0 * plane:(z0 + lp) * plane], device=dev)
        info = hf.hf_cg(ctx, 0.05, 1.0, b, x)
        torch.cuda.synchronize()
        q.put((rank, lo, hi, z0, u.cpu().numpy(), x.cpu().numpy(), st["total_iters"], info["iters"], None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, None, None, None, None, None, None, None, traceback.format_exc()))


def test_slab_two_processes_peer_ipc():
    import torch.multiprocessing as mp
    import oracle
    import synth
    import paper_1905_07622_b200 as hf
    grid_args = ((10, 9, 13), (0.3, 0.25, 0.2))
    nsteps = 4
    g = synth.Grid(*grid_args)
    k, c = synth.random_fields(g, seed=91)
    world = 2
    ctxq = mp.get_context("spawn")
    q = ctxq.Queue()
    port = _free_port()
    procs = [ctxq.Process(target=_rank_main, args=(r, world, port, q, grid_args, nsteps)) for r in range(world)]
    [p.start() for p in procs]
    res = [q.get(timeout=600) for _ in range(world)]
    [p.join(timeout=60) for p in procs]
    for r in res:
        assert r[-1] is None, r[-1]
    plane = (g.ne[0] + 1) * (g.ne[1] + 1)
    full = np.empty(g.n_nodes)
    xfull = np.empty(g.n_nodes)
    for rank, lo, hi, z0, u, x, its, cgits, _ in res:
        full[lo * plane:hi * plane] = u[(lo - z0) * plane:(hi - z0) * plane]
        xfull[lo * plane:hi * plane] = x[(lo - z0) * plane:(hi - z0) * plane]
    o = oracle.Oracle(g, k, c)
    u0 = synth.random_vector(g.n_nodes, 92) * 0.01
    uo, st, it, _ = o.simulate(0.5, 0.05, nsteps, o.face_load(synth.FACE_ZM, 1.0), u0)
    assert np.linalg.norm(full - uo) <= 1e-10 * np.linalg.norm(uo)
    xo, sto, _, _ = o.pcg(0.05, 1.0, synth.random_vector(g.n_nodes, 93), np.zeros(g.n_nodes))
    assert np.linalg.norm(xfull - xo) <= 1e-10 * np.linalg.norm(xo)
    # both ranks took the same loop decisions (bitwise-identical sums)
    assert res[0][6] == res[1][6] and res[0][7] == res[1][7]
    assert hf.HF_PEER_BLOB_BYTES == 256
