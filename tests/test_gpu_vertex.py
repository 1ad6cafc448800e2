"""Vertex materials averaged over each element (hf_set_vertex_coefficients) against
the oracle's vertex mode: Q1 voxels take the mean of their 8 corners; the paper's 6 tets per voxel
each take the mean of their 4 vertices (kernel variant EL_TETV)."""
import threading

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


def on_own_stream(fn, r):
    """Run a slab rank's thread on its own stream: ranks sharing the GPU wait for each other
    inside kernels, so they must never share (or implicitly synchronise with) a stream."""
    with torch.cuda.stream(torch.cuda.Stream(device=DEV)):
        fn(r)


def T(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def N(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def maxerr(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


GRIDS = {
    "c1": synth.Grid((8, 8, 8), (0.125, 0.125, 0.125)),
    "ragged": synth.Grid((70, 40, 13), (0.3, 0.2, 0.7), (-1.0, 2.0, 0.5)),
    "seams": synth.Grid((33, 65, 9), (0.2, 0.2, 0.2)),
}


def vertex_fields(g, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(1.0, 120.0, g.n_nodes), rng.uniform(0.5, 2.0, g.n_nodes)


def vctx(g, kn, cn, elem, prec=64):
    ctx = hf.hf_create(g, 0)
    if prec != 64:
        hf.hf_set_precision(ctx, prec)
    if elem:
        hf.hf_set_element(ctx, elem)
    hf.hf_set_vertex_coefficients(ctx, T(kn), T(cn))
    return ctx


@pytest.mark.parametrize("elem", [0, 1])
@pytest.mark.parametrize("gname", list(GRIDS))
def test_vertex_apply_and_diag(gname, elem):
    g = GRIDS[gname]
    kn, cn = vertex_fields(g, 51)
    o = oracle.Oracle(g, kn, cn, elem=elem, vertex=True)
    ctx = vctx(g, kn, cn, elem)
    u = synth.random_vector(g.n_nodes, 52)
    y = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    for aK, aM in [(1.0, 0.0), (0.0, 1.0), (0.005, 1.0)]:
        hf.hf_apply(ctx, aK, aM, T(u), y)
        assert maxerr(N(y), o.spmv(aK, aM, u)) <= 1e-12, (gname, elem, aK, aM)
    d = torch.empty_like(y)
    hf.hf_diag(ctx, 0.005, 1.0, d)
    assert maxerr(N(d), o.diag(0.005, 1.0)) <= 1e-13


@pytest.mark.parametrize("driver", [0, 1])
def test_vertex_tets_simulate_matches_oracle(driver):
    """The paper's Table 2 discretisation: laminate materials by vertex (steel for z <= 5 mm,
    P:271), averaged per tet, CN steps."""
    g = synth.Grid((12, 12, 10), (2.5, 2.5, 1.0), (-15.0, -15.0, 0.0))
    z = np.repeat(np.arange(g.ne[2] + 1) * g.h[2], (g.ne[0] + 1) * (g.ne[1] + 1))
    steel = z <= 5.0
    kn = np.where(steel, synth.STEEL[1], synth.OXIDE[1])
    cn = np.where(steel, synth.STEEL[0], synth.OXIDE[0])
    ctx = vctx(g, kn, cn, 1)
    hf.hf_set_driver(ctx, driver)
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
    u = T(np.zeros(g.n_nodes))
    hf.hf_simulate(ctx, 0.5, 0.01, 6, F, u, rtol=1e-12)
    o = oracle.Oracle(g, kn, cn, elem=1, vertex=True)
    uo, st, _, _ = o.simulate(0.5, 0.01, 6, o.face_load(synth.FACE_ZM, 1.0), np.zeros(g.n_nodes), tol=1e-12)
    assert st == 0 and rel(N(u), uo) <= 1e-10


def test_vertex_tets_fp32_and_switch_back():
    g = GRIDS["ragged"]
    kn, cn = vertex_fields(g, 53)
    o = oracle.Oracle(g, kn, cn, elem=1, vertex=True)
    ctx = vctx(g, kn, cn, 1, prec=32)
    u = synth.random_vector(g.n_nodes, 54)
    y = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_apply(ctx, 0.005, 1.0, T(u), y)
    assert rel(N(y), o.spmv(0.005, 1.0, u)) <= 1e-5
    # per-element coefficients again: the dense per-voxel tet operator
    ctx = vctx(g, kn, cn, 1)
    k, c = synth.random_fields(g, seed=55)
    hf.hf_set_coefficients(ctx, T(k), T(c))
    hf.hf_apply(ctx, 0.005, 1.0, T(u), y)
    assert maxerr(N(y), oracle.Oracle(g, k, c, elem=1).spmv(0.005, 1.0, u)) <= 1e-12
    with pytest.raises(hf.HfError):              # batched runs take per-element fields only
        ctx2 = vctx(g, kn, cn, 1)
        hf.hf_simulate_batched(ctx2, 1, T(k), None, 0.5, 0.01, 1, None, T(np.zeros(g.n_nodes)))


def test_vertex_tets_on_slabs_local_transport():
    """z-slabs carry the per-node pairs of their ghost planes: 2 slabs equal the oracle."""
    g = synth.Grid((10, 9, 13), (0.3, 0.3, 0.2))
    kn, cn = vertex_fields(g, 56)
    o = oracle.Oracle(g, kn, cn, elem=1, vertex=True)
    u0 = synth.random_vector(g.n_nodes, 57) * 0.01
    uo, _, _, _ = o.simulate(0.5, 0.05, 4, o.face_load(synth.FACE_ZM, 1.0), u0)
    nranks = 2
    grp = hf.hf_local_group_create(nranks)
    plane = (g.ne[0] + 1) * (g.ne[1] + 1)
    out, errs, ctxs = [None] * nranks, [], [None] * nranks

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            ctx = hf.hf_create_slab(g, r, nranks, grp, transport=1, device=0)
            ctxs[r] = ctx
            hf.hf_set_element(ctx, 1)
            lo, hi, lp, z0 = ctx.slab
            hf.hf_set_vertex_coefficients(ctx, T(kn), T(cn))
            F = torch.empty(ctx.n_nodes, dtype=torch.float64, device=DEV)
            hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
            u = T(u0[z0 * plane:(z0 + lp) * plane])
            hf.hf_simulate(ctx, 0.5, 0.05, 4, F, u)
            out[r] = (lo, hi, z0, N(u))
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=on_own_stream, args=(rank_main, r)) for r in range(nranks)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not errs, errs
    full = np.empty(g.n_nodes)
    for lo, hi, z0, u in out:
        full[lo * plane:hi * plane] = u[(lo - z0) * plane:(hi - z0) * plane]
    assert rel(full, uo) <= 1e-10
    del ctxs
    hf.hf_local_group_destroy(grp)
