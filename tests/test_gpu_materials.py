"""Materials by id (hf_set_material_ids): the paper's few-materials-by-region description (P:271,
P:345-357) streamed as one uint8 id per element (stencil variant EL_Q1P).  The operator must be
bit-identical to the per-element pair path (hf_set_coefficients with k_e = k_mat[id_e]) and
match the oracle with the apply / solution bars."""
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

GRIDS = {
    "1x1x1": synth.Grid((1, 1, 1), (1.0, 1.0, 1.0)),
    "c1": synth.Grid((8, 8, 8), (0.125, 0.125, 0.125)),
    "ragged": synth.Grid((70, 40, 13), (0.3, 0.2, 0.7), (-1.0, 2.0, 0.5)),
    "seams": synth.Grid((33, 65, 9), (0.2, 0.2, 0.2)),
    "wide": synth.Grid((150, 17, 5), (0.1, 0.1, 0.1)),
}


def T(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def N(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def maxerr(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def materials(n, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(1.0, 122.5, n), rng.uniform(0.5, 2.0, n)


def ctx_pair(g, ids, km, cm, tile_r=None):
    a, b = hf.hf_create(g, 0), hf.hf_create(g, 0)
    if tile_r is not None:
        hf.hf_set_tuning(a, "tile_r", tile_r)
        hf.hf_set_tuning(b, "tile_r", tile_r)
    hf.hf_set_material_ids(a, ids, km, cm)
    hf.hf_set_coefficients(b, T(km[ids]), T(cm[ids]))
    return a, b


@pytest.mark.parametrize("tile_r", [2, 4])
@pytest.mark.parametrize("gname", list(GRIDS))
def test_ids_apply_bitwise_and_oracle(gname, tile_r):
    g = GRIDS[gname]
    nmat = 5
    km, cm = materials(nmat, 81)
    ids = np.random.default_rng(82).integers(0, nmat, g.n_elems).astype(np.uint8)
    a, b = ctx_pair(g, ids, km, cm, tile_r)
    o = oracle.Oracle(g, km[ids], cm[ids])
    u = T(synth.random_vector(g.n_nodes, 83))
    bv = T(synth.random_vector(g.n_nodes, 84))
    ya, yb = torch.empty_like(u), torch.empty_like(u)
    for aK, aM in [(1.0, 0.0), (0.0, 1.0), (0.005, 1.0), (-0.005, 1.0)]:
        hf.hf_apply(a, aK, aM, u, ya)
        hf.hf_apply(b, aK, aM, u, yb)
        assert np.array_equal(N(ya), N(yb)), (gname, aK, aM)
        assert maxerr(N(ya), o.spmv(aK, aM, N(u))) <= 1e-12
    hf.hf_apply_axpby(a, 0.01, 1.0, -1.0, u, bv, ya)
    hf.hf_apply_axpby(b, 0.01, 1.0, -1.0, u, bv, yb)
    assert np.array_equal(N(ya), N(yb))


@pytest.mark.parametrize("driver", [0, 1])
def test_ids_simulate_bitwise_and_oracle(driver):
    """C1-style transient with Dirichlet faces on a ragged grid: identical to the pair path."""
    g = GRIDS["ragged"]
    km, cm = np.array([4.9e8, 4.0e6, 1e7]) * 1e-6, np.array([3.724e6, 1.65e6, 2e6]) * 1e-6
    ids = np.random.default_rng(85).integers(0, 3, g.n_elems).astype(np.uint8)
    a, b = ctx_pair(g, ids, km, cm)
    outs = []
    for ctx in (a, b):
        hf.hf_set_driver(ctx, driver)
        hf.hf_set_dirichlet_faces(ctx, (1 << synth.FACE_XM) | (1 << synth.FACE_YP), [0.5, 0, 0, -0.25, 0, 0])
        F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
        hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
        u = T(np.zeros(g.n_nodes))
        st = hf.hf_simulate(ctx, 0.5, 0.05, 6, F, u)
        outs.append((N(u), st["total_iters"]))
    assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]
    o = oracle.Oracle(g, km[ids], cm[ids])
    o.set_dirichlet((1 << synth.FACE_XM) | (1 << synth.FACE_YP), (0.5, 0, 0, -0.25, 0, 0))
    uo, _, _, _ = o.simulate(0.5, 0.05, 6, o.face_load(synth.FACE_ZM, 1.0), np.zeros(g.n_nodes))
    assert rel(outs[0][0], uo) <= 1e-10


def test_ids_state_switches_and_errors():
    g = GRIDS["c1"]
    km, cm = materials(2, 86)
    ids = np.random.default_rng(87).integers(0, 2, g.n_elems).astype(np.uint8)
    ctx = hf.hf_create(g, 0)
    with pytest.raises(hf.HfError) as e:
        hf.hf_set_material_ids(ctx, ids, km[:1], cm[:1])          # id 1 >= 1 material
    assert e.value.status == hf.HF_E_INDEX
    with pytest.raises(hf.HfError) as e:
        hf.hf_set_material_ids(ctx, ids, np.ones(64), np.ones(64))
    assert e.value.status == hf.HF_E_ARG
    hf.hf_set_material_ids(ctx, torch.tensor(ids, device=DEV), km, cm)     # device ids
    u = synth.random_vector(g.n_nodes, 88)
    y = np.empty_like(u)
    # tets on an id context read the pair layout filled from the table
    hf.hf_set_element(ctx, 1)
    hf.hf_apply(ctx, 0.3, 1.0, u, y)
    assert maxerr(y, oracle.Oracle(g, km[ids], cm[ids], elem=1).spmv(0.3, 1.0, u)) <= 1e-12
    hf.hf_set_element(ctx, 0)
    hf.hf_apply(ctx, 0.3, 1.0, u, y)
    assert maxerr(y, oracle.Oracle(g, km[ids], cm[ids]).spmv(0.3, 1.0, u)) <= 1e-12
    # back to per-element pairs
    k2, c2 = synth.random_fields(g, seed=89)
    hf.hf_set_coefficients(ctx, k2, c2)
    hf.hf_apply(ctx, 0.3, 1.0, u, y)
    assert maxerr(y, oracle.Oracle(g, k2, c2).spmv(0.3, 1.0, u)) <= 1e-12
    # diagonal from the id path equals the pair path's
    hf.hf_set_material_ids(ctx, ids, km, cm)
    d = np.empty_like(u)
    hf.hf_diag(ctx, 0.02, 1.0, d)
    assert maxerr(d, oracle.Oracle(g, km[ids], cm[ids]).diag(0.02, 1.0)) <= 1e-13


def test_ids_slabs_match_single():
    g = synth.Grid((20, 14, 23), (0.2, 0.2, 0.2))
    km, cm = materials(3, 90)
    ids = np.random.default_rng(91).integers(0, 3, g.n_elems).astype(np.uint8)
    u0 = synth.random_vector(g.n_nodes, 92) * 0.01
    ctx1 = hf.hf_create(g, 0)
    hf.hf_set_material_ids(ctx1, ids, km, cm)
    F1 = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx1, synth.FACE_ZM, 1.0, None, F1)
    u1 = T(u0)
    hf.hf_simulate(ctx1, 0.5, 0.02, 4, F1, u1)
    ref = N(u1)
    nranks = 2
    grp = hf.hf_local_group_create(nranks)
    plane = (g.ne[0] + 1) * (g.ne[1] + 1)
    out, errs, ctxs = [None] * nranks, [], [None] * nranks

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            ctx = hf.hf_create_slab(g, r, nranks, grp, transport=1, device=0)
            ctxs[r] = ctx
            lo, hi, lp, z0 = ctx.slab
            hf.hf_set_material_ids(ctx, ids, km, cm)
            F = torch.empty(ctx.n_nodes, dtype=torch.float64, device=DEV)
            hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
            u = T(u0[z0 * plane:(z0 + lp) * plane])
            hf.hf_simulate(ctx, 0.5, 0.02, 4, F, u)
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
    assert rel(full, ref) <= 1e-12
    del ctxs
    hf.hf_local_group_destroy(grp)


def test_ids_c3_two_steps():
    """BASELINE configs[2] (C3) through material ids, in the bench's launch configuration: the
    same solution as the pair path (bit for bit) and the oracle (<= 1e-10)."""
    p = synth.c3(nsteps=2)
    ids = p.extra["ids"]
    mats = p.extra["materials"]
    km = np.array([m[1] for m in mats])
    cm = np.array([m[0] for m in mats])
    assert np.array_equal(km[ids], p.k) and np.array_equal(cm[ids], p.c)
    a, b = ctx_pair(p.grid, ids, km, cm)
    res = []
    for ctx in (a, b):
        F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
        hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
        u = T(p.u0)
        hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol)
        res.append(N(u))
    assert np.array_equal(res[0], res[1])
    o, Fo = oracle.problem_oracle(p)
    uo, _, _, _ = o.simulate(p.theta, p.dt, p.nsteps, Fo, p.u0, tol=p.rtol)
    assert rel(res[0], uo) <= 1e-10


@pytest.mark.slow
def test_ids_c4_apply_sampled_rows():
    """The 512^3 apply through material ids in the launch configuration bench.py times
    (apply_512_ids: two materials, 20 % oxide, R = 4 tiles) on sampled rows, boundary classes
    and tile seams included, against the oracle's per-row evaluation."""
    g = synth.c4_grid()
    rng = np.random.default_rng(97)
    ids = (rng.random(g.n_elems) < 0.2).astype(np.uint8)
    km = np.array([synth.STEEL[1], synth.OXIDE[1]])
    cm = np.array([synth.STEEL[0], synth.OXIDE[0]])
    u = synth.random_vector(g.n_nodes, 98)
    ctx = hf.hf_create(g, 0)
    hf.hf_set_material_ids(ctx, ids, km, cm)
    y = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_apply(ctx, 0.005, 1.0, T(u), y)
    yg = N(y)
    del ctx
    torch.cuda.empty_cache()
    o = oracle.Oracle(g, km[ids], cm[ids], assemble=False)
    nx, ny, nz = g.nn
    rows = rng.integers(0, g.n_nodes, 4096)
    extra = [i + nx * (j + ny * kk) for (i, j, kk) in
             [(0, 0, 0), (nx - 1, ny - 1, nz - 1), (30, 30, 7), (31, 31, 8), (32, 62, 9), (61, 93, 500),
              (nx - 1, 0, 3), (0, ny - 1, nz - 1)]]
    rows = np.concatenate([rows, np.array(extra)])
    yo = o.apply_rows(0.005, 1.0, u, rows)
    assert maxerr(yg[rows], yo) <= 1e-12
