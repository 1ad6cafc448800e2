"""Corrosion inversion with the Metropolis-Hastings chains spread over processes, each with its
own GPU forward model (NEXT row f2).  (File name sorts first: the two spawned ranks
start while the test process is still small, before the full-size tests grow its host memory.)  Two ranks share the one B200 of the test box
(gloo for the final gather): the gathered chains must equal single-process runs of the same
chain groups (per-chain random streams, forward batches of the same size)."""
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

from paper_1905_07622_b200 import inverse as inv  # noqa: E402

CHAINS, NS, BURN, STEP, SEED, TRUTH = 4, 12, 6, 0.5, 5, 3.175


def _setup():
    g = synth.c5_grid(20)
    fwd = inv.CorrosionForward(g, nsteps=20, rtol=1e-8)
    cam = inv.camera_for(g, px=16, py=16, span=12.0)
    data = cam.observe(fwd.fronts([TRUTH])[0], np.random.default_rng(3))
    return fwd, cam, data


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import traceback
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        fwd, cam, data = _setup()
        res = inv.invert_distributed(fwd, cam, data, chains=CHAINS, n_samples=NS, burn_in=BURN, step=STEP, seed=SEED)
        if rank == 0:
            q.put(("ok", res.samples, res.forward_calls))
    except Exception:                      # report instead of leaving the parent waiting
        q.put(("error", f"rank {rank}: " + traceback.format_exc(), None))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_chains_over_two_processes_equal_single_process_groups():
    import gc
    import queue
    gc.collect()                           # earlier tests' contexts and cached blocks
    torch.cuda.empty_cache()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    msg = None
    for _ in range(600):
        try:
            msg = q.get(timeout=1)
            break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert msg is not None, [p.exitcode for p in procs]
    assert msg[0] == "ok", msg[1]
    _, samples, calls = msg
    fwd, cam, data = _setup()

    def ll(th):
        return np.array([cam.loglik(data, f) for f in fwd.fronts(th)])

    for r in range(2):
        ids = inv.chain_range(CHAINS, r, 2)
        ref = inv.metropolis_hastings(ll, np.full(len(ids), 0.5 * fwd.thickness), 0.0, fwd.thickness, NS, BURN, STEP,
                                      None, inv.chain_generators(SEED, ids))
        assert np.array_equal(samples[:, list(ids)], ref.samples)
    assert calls >= CHAINS * (NS + BURN)
