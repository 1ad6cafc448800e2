"""Corrosion inversion through invert_distributed on the GPU (NEXT row f2): the
chains of one process's share, each with its own random stream, through the GPU forward model
must equal metropolis_hastings run directly on the same chains.  The multi-process logic (world
sizes 1-3, bitwise against one process) is tests/test_mcmc_dist_gloo.py; here the group has one
rank so that no two processes drive conditional-node graphs on the test box's single GPU at the
same time."""
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1905_07622_b200 import inverse as inv  # noqa: E402

CHAINS, NS, BURN, STEP, SEED, TRUTH = 4, 12, 6, 0.5, 5, 3.175


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_invert_distributed_one_rank_equals_direct_chains():
    import torch.distributed as dist
    g = synth.c5_grid(20)
    fwd = inv.CorrosionForward(g, nsteps=20, rtol=1e-8)
    cam = inv.camera_for(g, px=16, py=16, span=12.0)
    data = cam.observe(fwd.fronts([TRUTH])[0], np.random.default_rng(3))
    store = dist.TCPStore("127.0.0.1", _free_port(), 1, True)
    dist.init_process_group("gloo", store=store, rank=0, world_size=1)
    try:
        res = inv.invert_distributed(fwd, cam, data, chains=CHAINS, n_samples=NS, burn_in=BURN, step=STEP, seed=SEED)
    finally:
        dist.destroy_process_group()

    def ll(th):
        return np.array([cam.loglik(data, f) for f in fwd.fronts(th)])

    ref = inv.metropolis_hastings(ll, np.full(CHAINS, 0.5 * fwd.thickness), 0.0, fwd.thickness, NS, BURN, STEP,
                                  None, inv.chain_generators(SEED, range(CHAINS)))
    assert np.array_equal(res.samples, ref.samples)
    assert res.forward_calls >= CHAINS * (NS + BURN)
    assert abs(res.samples.mean() - TRUTH) < 1.5
