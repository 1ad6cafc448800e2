"""Corrosion-depth inversion by Metropolis-Hastings on the GPU forward model (NEXT row f2).

PAPER.md §5.4: a parabolic corrosion region of apex depth theta grows from the rear
face of a steel plate (Fig. 6; reading R13); a 10 W Gaussian laser heats the front
face for T_F = 10 s (reading R12); a thermal camera records the front-face temperature:
the FEM field interpolated to a finer pixel grid, averaged over each pixel, contaminated with
N(0, 0.1^2) noise and rounded to 0.1 degC.  The posterior p(theta | D) with a uniform
prior on [0, thickness] is sampled by Metropolis-Hastings, 200 burn-in
samples then the chain.

GPU part: every forward simulation is hf_simulate_batched (the B200 hot path, one system per
proposal; chains advance in lock-step so one batched call evaluates all their proposals).
Host part (this file): camera model, quantised-Gaussian likelihood, proposal/accept logic.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np


# ---------------------------------------------------------------------------------------------
# camera model

@dataclass
class Camera:
    """Pixel grid over the rectangle [x0,x1] x [y0,y1] of the front face; each pixel is the
    mean of sub x sub bilinear samples of the nodal field (interpolate to a finer grid, then
    average over the pixel area); noise sigma (0.1 degC) and rounding quantum (0.1 degC)."""
    nodes_x: np.ndarray          # node coordinates along x of the face
    nodes_y: np.ndarray
    x0: float
    x1: float
    y0: float
    y1: float
    px: int = 32
    py: int = 32
    sub: int = 4
    sigma: float = 0.1
    quantum: float = 0.1

    def __post_init__(self):
        sx = self.x0 + (np.arange(self.px * self.sub) + 0.5) * (self.x1 - self.x0) / (self.px * self.sub)
        sy = self.y0 + (np.arange(self.py * self.sub) + 0.5) * (self.y1 - self.y0) / (self.py * self.sub)
        self._ix, self._wx = self._bilin(self.nodes_x, sx)
        self._iy, self._wy = self._bilin(self.nodes_y, sy)

    @staticmethod
    def _bilin(nodes, s):
        i = np.clip(np.searchsorted(nodes, s) - 1, 0, len(nodes) - 2)
        w = (s - nodes[i]) / (nodes[i + 1] - nodes[i])
        return i, w

    def render(self, front: np.ndarray) -> np.ndarray:
        """front: (ny1, nx1) nodal temperatures of the face -> (py, px) pixel temperatures."""
        f = np.asarray(front, dtype=np.float64)
        iy, wy, ix, wx = self._iy, self._wy, self._ix, self._wx
        # bilinear interpolation on the sub-sample grid
        a = f[np.ix_(iy, ix)] * (1 - wy)[:, None] * (1 - wx)[None, :]
        a += f[np.ix_(iy, ix + 1)] * (1 - wy)[:, None] * wx[None, :]
        a += f[np.ix_(iy + 1, ix)] * wy[:, None] * (1 - wx)[None, :]
        a += f[np.ix_(iy + 1, ix + 1)] * wy[:, None] * wx[None, :]
        # average over each pixel's sub x sub samples
        return a.reshape(self.py, self.sub, self.px, self.sub).mean(axis=(1, 3))

    def observe(self, front: np.ndarray, rng: np.random.Generator) -> np.ndarray:
        """Camera data: render + N(0, sigma^2) + rounding to the quantum."""
        t = self.render(front) + self.sigma * rng.standard_normal((self.py, self.px))
        return np.round(t / self.quantum) * self.quantum

    def loglik(self, data: np.ndarray, front: np.ndarray) -> float:
        """log p(D | field): each pixel's datum is the rounded noisy temperature, so
        p(D_p) = Phi((D_p + q/2 - T_p)/s) - Phi((D_p - q/2 - T_p)/s)."""
        from scipy.special import log_ndtr
        t = self.render(front)
        q, s = self.quantum, self.sigma
        hi = (data + 0.5 * q - t) / s
        lo = (data - 0.5 * q - t) / s
        # log(Phi(hi) - Phi(lo)) computed on the tail side that keeps precision
        flip = lo > 0
        h2 = np.where(flip, -lo, hi)
        l2 = np.where(flip, -hi, lo)
        lh, ll = log_ndtr(h2), log_ndtr(l2)
        return float(np.sum(lh + np.log1p(-np.exp(np.minimum(ll - lh, -1e-300)))))


# ---------------------------------------------------------------------------------------------
# Metropolis-Hastings, chains in lock-step

@dataclass
class MHResult:
    samples: np.ndarray          # (n_samples, chains) after burn-in
    accept_rate: float
    loglik: np.ndarray           # (n_samples, chains)
    forward_calls: int


def chain_generators(seed: int, chain_ids: Sequence[int]) -> list:
    """One random stream per chain (numpy SeedSequence of (seed, chain id)): a chain draws the
    same proposals and acceptance variates whichever process or batch it runs in."""
    return [np.random.default_rng([int(seed), int(c)]) for c in chain_ids]


def metropolis_hastings(loglik_batch: Callable[[np.ndarray], np.ndarray], theta0: Sequence[float],
                        lo: float, hi: float, n_samples: int, burn_in: int, step: float,
                        rng: Optional[np.random.Generator], chain_rngs: Optional[Sequence] = None) -> MHResult:
    """theta_{i+1} = theta_hat with probability min(1, p(D|theta_hat)/p(D|theta_i)), else theta_i
    (P:363-364); uniform prior on [lo, hi]: proposals outside are rejected (their
    likelihood is never used).  loglik_batch evaluates a vector of candidate thetas (one batched
    GPU call) of a FIXED size, one per chain: an outside proposal is evaluated at its clipped
    value and discarded, so every forward batch has the same shape (the same stack grouping and
    reduction order) whatever the number of proposals inside the prior.
    Random numbers: one generator for all chains (rng), or one per chain (chain_rngs, see
    chain_generators) so that chains can be split over processes without changing them."""
    theta = np.asarray(theta0, dtype=np.float64).copy()
    chains = theta.size
    if chain_rngs is not None and len(chain_rngs) != chains:
        raise ValueError("chain_rngs: one generator per chain")

    def normals():
        if chain_rngs is None:
            return rng.standard_normal(chains)
        return np.array([g.standard_normal() for g in chain_rngs])

    def uniforms():
        if chain_rngs is None:
            return rng.uniform(size=chains)
        return np.array([g.uniform() for g in chain_rngs])

    ll = loglik_batch(theta)
    calls = chains
    out, outll = [], []
    acc = 0
    total = 0
    for it in range(burn_in + n_samples):
        prop = theta + step * normals()
        inside = (prop >= lo) & (prop <= hi)
        llp = np.full(chains, -np.inf)
        if inside.any():
            llp = np.where(inside, loglik_batch(np.clip(prop, lo, hi)), -np.inf)
            calls += chains
        logu = np.log(uniforms())
        take = inside & (logu < llp - ll)
        theta = np.where(take, prop, theta)
        ll = np.where(take, llp, ll)
        if it >= burn_in:
            out.append(theta.copy())
            outll.append(ll.copy())
            acc += int(take.sum())
            total += chains
    return MHResult(np.array(out), acc / max(total, 1), np.array(outll), calls)


# ---------------------------------------------------------------------------------------------
# the GPU forward model of the corrosion problem

# P:271 materials (rho C, k), verbatim (reading R11); 10 W in the same (g, mm, s) units (R12)
STEEL = (3.724e6, 4.9e8)
OXIDE = (1.65e6, 4.0e6)
BEAM_POWER = 10.0 * 1e9
FACE_ZM = 4


def corrosion_fields(grid, depth: float, half_height: float, z_rear: float, materials=(STEEL, OXIDE)):
    """Per-element (k, c) of a plate with the parabolic corrosion of apex depth `depth` grown
    from the rear face (Fig. 6, reading R13): an element is oxide iff its centroid
    has |y| <= H and (z_rear - z) <= depth (1 - (y/H)^2); constant along x."""
    nx, ny, nz = grid.ne
    yc = grid.origin[1] + (np.arange(ny) + 0.5) * grid.h[1]
    zc = grid.origin[2] + (np.arange(nz) + 0.5) * grid.h[2]
    inside = (np.abs(yc)[None, :] <= half_height) & \
             ((z_rear - zc)[:, None] <= depth * (1.0 - (yc / half_height) ** 2)[None, :])
    ids = np.broadcast_to(inside[:, :, None], (nz, ny, nx)).astype(np.uint8).ravel()
    cs = np.array([m[0] for m in materials])
    ks = np.array([m[1] for m in materials])
    return ks[ids], cs[ids]


class CorrosionForward:
    """theta (mm) -> front-face temperature field at T_F, for a batch of thetas per call."""

    def __init__(self, grid, nsteps: int = 300, t_final: float = 10.0, beam=None, thickness: float = 12.7,
                 half_height: float = 15.0, device: int = 0, rtol: float = 1e-8,
                 materials=None, k_factor: Optional[np.ndarray] = None):
        import torch
        from . import hf_create, hf_face_load, hf_set_coefficients
        self.torch = torch
        self.grid = grid
        self.nsteps = nsteps
        self.dt = t_final / nsteps
        self.thickness = thickness
        self.H = half_height
        self.rtol = rtol
        self.materials = materials or (STEEL, OXIDE)
        self.k_factor = k_factor
        self.dev = torch.device("cuda", device)
        self.ctx = hf_create(grid, device)
        k0, c0 = corrosion_fields(grid, 0.0, half_height, grid.origin[2] + thickness, self.materials)
        hf_set_coefficients(self.ctx, torch.tensor(k0, device=self.dev), torch.tensor(c0, device=self.dev))
        self.F = torch.empty(grid.n_nodes, dtype=torch.float64, device=self.dev)
        beam = beam or (BEAM_POWER, 2.0, 0.0, 0.0)
        hf_face_load(self.ctx, FACE_ZM, 0.0, beam, self.F)
        self.calls = 0

    def fields(self, thetas: np.ndarray):
        k, c = [], []
        for th in thetas:
            kk, cc = corrosion_fields(self.grid, float(th), self.H, self.grid.origin[2] + self.thickness,
                                      self.materials)
            if self.k_factor is not None:
                kk = kk * self.k_factor
            k.append(kk)
            c.append(cc)
        return np.stack(k), np.stack(c)

    def fronts(self, thetas: Sequence[float]) -> np.ndarray:
        from . import hf_simulate_batched
        torch = self.torch
        thetas = np.atleast_1d(np.asarray(thetas, dtype=np.float64))
        B = thetas.size
        k, c = self.fields(thetas)
        g = self.grid
        ub = torch.zeros(B * g.n_nodes, dtype=torch.float64, device=self.dev)
        plane = (g.ne[0] + 1) * (g.ne[1] + 1)
        front = torch.empty(B * plane, dtype=torch.float64, device=self.dev)
        hf_simulate_batched(self.ctx, B, torch.tensor(k.ravel(), device=self.dev),
                            torch.tensor(c.ravel(), device=self.dev), 0.5, self.dt, self.nsteps, self.F, ub, 0,
                            front, rtol=self.rtol)
        self.calls += B
        return front.cpu().numpy().reshape(B, g.ne[1] + 1, g.ne[0] + 1)


def camera_for(grid, px: int = 32, py: int = 32, span: float = 8.0, **kw) -> Camera:
    """Camera looking at the central span x span mm of the front face."""
    nx = grid.origin[0] + np.arange(grid.ne[0] + 1) * grid.h[0]
    ny = grid.origin[1] + np.arange(grid.ne[1] + 1) * grid.h[1]
    cx = grid.origin[0] + 0.5 * grid.ne[0] * grid.h[0]
    cy = grid.origin[1] + 0.5 * grid.ne[1] * grid.h[1]
    return Camera(nx, ny, cx - span / 2, cx + span / 2, cy - span / 2, cy + span / 2, px=px, py=py, **kw)


def invert(forward: CorrosionForward, camera: Camera, data: np.ndarray, chains: int = 4, n_samples: int = 200,
           burn_in: int = 50, step: float = 0.3, seed: int = 0) -> MHResult:
    """Posterior samples of the corrosion depth given camera data."""
    rng = np.random.default_rng(seed)

    def ll(thetas):
        fr = forward.fronts(thetas)
        return np.array([camera.loglik(data, f) for f in fr])

    theta0 = np.full(chains, 0.5 * forward.thickness)      # "middle of the prior"
    return metropolis_hastings(ll, theta0, 0.0, forward.thickness, n_samples, burn_in, step, rng)


def chain_range(chains: int, rank: int, world: int) -> range:
    """The chains of one process: contiguous, sizes differing by at most one."""
    return range(rank * chains // world, (rank + 1) * chains // world)


def mh_distributed(loglik_batch: Callable[[np.ndarray], np.ndarray], chains: int, theta0: float, lo: float,
                   hi: float, n_samples: int, burn_in: int, step: float, seed: int, group=None) -> MHResult:
    """Metropolis-Hastings with the chains split over the processes of a torch.distributed group
    (one GPU per process, each with its own forward model): the chains are independent, so the
    only communication is the final gather of the samples (all_gather_object, any backend).
    Every chain uses its own random stream (chain_generators), so the gathered result equals a
    single-process run of the same chains batched the same way."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = chain_range(chains, rank, world)
    res = None
    if len(mine):
        res = metropolis_hastings(loglik_batch, np.full(len(mine), float(theta0)), lo, hi, n_samples, burn_in,
                                  step, None, chain_generators(seed, mine))
    part = None if res is None else (list(mine), res.samples, res.loglik, res.accept_rate, res.forward_calls)
    parts = [None] * world
    dist.all_gather_object(parts, part, group=group)
    samples = np.zeros((n_samples, chains))
    loglik = np.zeros((n_samples, chains))
    acc, calls = 0.0, 0
    for pr in parts:
        if pr is None:
            continue
        ids, smp, ll, rate, nc = pr
        samples[:, ids] = smp
        loglik[:, ids] = ll
        acc += rate * len(ids) * n_samples
        calls += nc
    return MHResult(samples, acc / max(chains * n_samples, 1), loglik, calls)


def invert_distributed(forward: CorrosionForward, camera: Camera, data: np.ndarray, chains: int = 8,
                       n_samples: int = 200, burn_in: int = 50, step: float = 0.3, seed: int = 0,
                       group=None) -> MHResult:
    """invert() with the chains spread over the ranks of a process group, one GPU each (the
    rank's forward model lives on its own device): P:362-376 with the chains/ensemble filling
    the GPUs of one node."""
    def ll(thetas):
        fr = forward.fronts(thetas)
        return np.array([camera.loglik(data, f) for f in fr])

    return mh_distributed(ll, chains, 0.5 * forward.thickness, 0.0, forward.thickness, n_samples, burn_in, step,
                          seed, group)
