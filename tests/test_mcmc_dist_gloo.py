"""Metropolis-Hastings with the chains split over processes (NEXT row f2: the chains
fill the GPUs of a node).  World size 1, 2 and 3 over gloo on CPU with an analytic likelihood:
the gathered chains must equal a single-process run of the same chains (per-chain random
streams), and the posterior must be the target."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1905_07622_b200 import inverse as inv

MU, SD = 4.2, 0.7
CHAINS, N, BURN, STEP, SEED = 7, 400, 50, 0.5, 11


def loglik(th):
    return -0.5 * ((np.asarray(th) - MU) / SD) ** 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = inv.mh_distributed(loglik, CHAINS, 6.35, 0.0, 12.7, N, BURN, STEP, SEED)
        if rank == 0:
            q.put((res.samples, res.loglik, res.accept_rate, res.forward_calls))
    finally:
        dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_chain_range_partition():
    for chains in (1, 5, 8, 13):
        for world in (1, 2, 3, 8):
            got = [c for r in range(world) for c in inv.chain_range(chains, r, world)]
            assert got == list(range(chains))


def test_per_chain_streams_do_not_depend_on_the_batch():
    # chains 0..6 in one batch == chains 0..2 and 3..6 in two batches
    full = inv.metropolis_hastings(loglik, [6.35] * CHAINS, 0.0, 12.7, N, BURN, STEP, None,
                                   inv.chain_generators(SEED, range(CHAINS)))
    a = inv.metropolis_hastings(loglik, [6.35] * 3, 0.0, 12.7, N, BURN, STEP, None, inv.chain_generators(SEED, range(3)))
    b = inv.metropolis_hastings(loglik, [6.35] * 4, 0.0, 12.7, N, BURN, STEP, None,
                                inv.chain_generators(SEED, range(3, 7)))
    assert np.array_equal(full.samples, np.concatenate([a.samples, b.samples], axis=1))


@pytest.mark.parametrize("world", [1, 2, 3])
def test_distributed_chains_equal_single_process(world):
    samples, ll, rate, calls = _run(world)
    ref = inv.metropolis_hastings(loglik, [6.35] * CHAINS, 0.0, 12.7, N, BURN, STEP, None,
                                  inv.chain_generators(SEED, range(CHAINS)))
    assert np.array_equal(samples, ref.samples)
    assert np.array_equal(ll, ref.loglik)
    assert abs(rate - ref.accept_rate) < 1e-12
    s = samples.ravel()
    assert abs(s.mean() - MU) < 0.1 and abs(s.std() - SD) < 0.1
