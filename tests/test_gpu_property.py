"""Randomised parity sweep (hypothesis): grid shapes that land anywhere relative to the 31-column
x tiles, the 15/31-row y tiles and the z chunks, anisotropic spacings, every element variant and
both precisions, against the oracle's assembled operator.  Bars: max-abs error <= 1e-12 of the
output scale in fp64 (rounding order only), rel-L2 <= 1e-5 in fp32."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_07622_b200 as hf  # noqa: E402

DEV = torch.device("cuda:0")


def T(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


grids = st.tuples(st.integers(1, 70), st.integers(1, 40), st.integers(1, 12),
                  st.floats(0.05, 2.0), st.floats(0.05, 2.0), st.floats(0.05, 2.0))


@settings(max_examples=24, deadline=None, derandomize=True)
@given(grid=grids, variant=st.sampled_from(["q1", "tets", "tetv"]), prec=st.sampled_from([64, 32]),
       seed=st.integers(0, 1000))
def test_random_grids_apply_and_diag(grid, variant, prec, seed):
    nx, ny, nz, hx, hy, hz = grid
    g = synth.Grid((nx, ny, nz), (hx, hy, hz), (0.3, -0.2, 1.0))
    rng = np.random.default_rng(seed)
    elem = 0 if variant == "q1" else 1
    vertex = variant == "tetv"
    n = g.n_nodes if vertex else g.n_elems
    k = rng.uniform(1.0, 120.0, n)
    c = rng.uniform(0.5, 2.0, n)
    o = oracle.Oracle(g, k, c, elem=elem, vertex=vertex)
    ctx = hf.hf_create(g, 0)
    if prec == 32:
        hf.hf_set_precision(ctx, 32)
    if elem:
        hf.hf_set_element(ctx, 1)
    if vertex:
        hf.hf_set_vertex_coefficients(ctx, T(k), T(c))
    else:
        hf.hf_set_coefficients(ctx, T(k), T(c))
    u = rng.standard_normal(g.n_nodes)
    aK, aM = float(rng.uniform(0.0, 0.1)), 1.0
    y = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_apply(ctx, aK, aM, T(u), y)
    yo = o.spmv(aK, aM, u)
    yg = y.cpu().numpy()
    if prec == 64:
        assert np.abs(yg - yo).max() <= 1e-12 * np.abs(yo).max(), (grid, variant)
    else:
        assert np.linalg.norm(yg - yo) <= 1e-5 * np.linalg.norm(yo), (grid, variant)
    d = torch.empty_like(y)
    hf.hf_diag(ctx, aK, aM, d)
    do = o.diag(aK, aM)
    assert np.abs(d.cpu().numpy() - do).max() <= (1e-13 if prec == 64 else 1e-6) * np.abs(do).max()
