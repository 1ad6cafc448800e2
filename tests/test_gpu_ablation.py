"""NEXT row f4: the paper's earlier interpretations of the assembly operator (Implementation 1,
two-pass flexible DbD with stored element matrices; Implementation 2, single-pass
FG DbD) rebuilt on sm_100a.  Each computes the same apply as the production stencil
(Eq. (1)), so each is checked element by element against the CPU oracle's assembled
SpMV with the apply bar (max-abs error <= 1e-12 of the output scale)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_07622_b200 as hf  # noqa: E402

DEV = torch.device("cuda:0")

GRIDS = {
    "1x1x1": synth.Grid((1, 1, 1), (1.0, 1.0, 1.0)),
    "c1": synth.Grid((8, 8, 8), (0.125, 0.125, 0.125)),
    # x rows longer than one Impl-2 CTA (128 nodes) with a ragged tail; odd nx1 (padded pitch)
    "ragged": synth.Grid((140, 9, 7), (0.3, 0.2, 0.7), (-1.0, 2.0, 0.5)),
    "tall": synth.Grid((5, 3, 60), (0.1, 0.4, 0.05)),
}


def T(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def N(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def maxerr(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("elem", [0, 1])
@pytest.mark.parametrize("gname", list(GRIDS))
def test_ablation_impls_match_oracle(gname, elem):
    g = GRIDS[gname]
    k, c = synth.random_fields(g, seed=61)
    o = oracle.Oracle(g, k, c, elem=elem)
    ctx = hf.hf_create(g, 0)
    hf.hf_set_element(ctx, elem)
    hf.hf_set_coefficients(ctx, T(k), T(c))
    u = synth.random_vector(g.n_nodes, seed=62)
    b = synth.random_vector(g.n_nodes, seed=63)
    ud, bd = T(u), T(b)
    y = torch.empty_like(ud)
    for aK, aM in [(1.0, 0.0), (0.0, 1.0), (0.005, 1.0), (-0.005, 1.0)]:
        yo = o.spmv(aK, aM, u)
        hf.hf_ablation_prepare(ctx, aK, aM)
        for impl in (1, 2, 3):
            y.fill_(float("nan"))
            hf.hf_apply_impl(ctx, impl, aK, aM, 1.0, ud, None, y)
            assert maxerr(N(y), yo) <= 1e-12, (gname, elem, impl, aK, aM)
        # the fused y = c A u + b of the second pass / FGDbDMVM_C
        for impl in (1, 2):
            hf.hf_apply_impl(ctx, impl, aK, aM, -1.0, ud, bd, y)
            assert maxerr(N(y), b - yo) <= 1e-12, (gname, elem, impl)


def test_ablation_host_buffers_and_state_errors():
    g = GRIDS["ragged"]
    k, c = synth.random_fields(g, seed=64)
    o = oracle.Oracle(g, k, c)
    ctx = hf.hf_create(g, 0)
    hf.hf_set_coefficients(ctx, k, c)
    u = synth.random_vector(g.n_nodes, seed=65)
    # Implementation 1 needs its preprocessing for the same (aK, aM)
    with pytest.raises(hf.HfError) as e:
        hf.hf_apply_impl(ctx, 1, 0.01, 1.0, 1.0, u, None, np.empty_like(u))
    assert e.value.status == hf.HF_E_STATE
    hf.hf_ablation_prepare(ctx, 0.01, 1.0)
    with pytest.raises(hf.HfError) as e:
        hf.hf_apply_impl(ctx, 1, 0.02, 1.0, 1.0, u, None, np.empty_like(u))
    assert e.value.status == hf.HF_E_STATE
    for impl in (1, 2):
        yh = np.empty_like(u)
        hf.hf_apply_impl(ctx, impl, 0.01, 1.0, 1.0, u, None, yh)      # host buffers, staged
        assert maxerr(yh, o.spmv(0.01, 1.0, u)) <= 1e-12
    # new coefficients invalidate the stored element matrices
    hf.hf_set_coefficients(ctx, k * 2.0, c)
    with pytest.raises(hf.HfError) as e:
        hf.hf_apply_impl(ctx, 1, 0.01, 1.0, 1.0, u, None, np.empty_like(u))
    assert e.value.status == hf.HF_E_STATE
    with pytest.raises(hf.HfError) as e:
        hf.hf_apply_impl(ctx, 4, 0.01, 1.0, 1.0, u, None, np.empty_like(u))
    assert e.value.status == hf.HF_E_ARG
    # fp32 contexts have no ablation kernels
    ctx32 = hf.hf_create(g, 0)
    hf.hf_set_precision(ctx32, 32)
    hf.hf_set_coefficients(ctx32, k, c)
    with pytest.raises(hf.HfError) as e:
        hf.hf_apply_impl(ctx32, 2, 0.01, 1.0, 1.0, u, None, np.empty_like(u))
    assert e.value.status == hf.HF_E_STATE


def test_ablation_c3_full():
    """BASELINE configs[2] (C3, 1M DoF, inclusion field) in full: all three interpretations
    against the oracle's assembled SpMV, in the launch configuration tools/ablation.py times."""
    p = synth.c3(nsteps=1)
    o, _ = oracle.problem_oracle(p)
    ctx = hf.hf_create(p.grid, 0)
    hf.hf_set_coefficients(ctx, T(p.k), T(p.c))
    u = synth.random_vector(p.grid.n_nodes, 66)
    aK = p.theta * p.dt
    yo = o.spmv(aK, 1.0, u)
    hf.hf_ablation_prepare(ctx, aK, 1.0)
    y = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    outs = []
    for impl in (1, 2, 3):
        hf.hf_apply_impl(ctx, impl, aK, 1.0, 1.0, T(u), None, y)
        outs.append(N(y))
        assert maxerr(outs[-1], yo) <= 1e-12, impl
