"""Host logic of the corrosion inversion (NEXT row f2): camera model, quantised
Gaussian likelihood, Metropolis-Hastings.  CPU tests use analytic forward models; the GPU test
runs a small inversion through hf_simulate_batched."""
import numpy as np
import pytest

import synth
from paper_1905_07622_b200 import inverse as inv


def _cam(n=21, span=8.0, **kw):
    g = synth.c5_grid(n)
    return g, inv.camera_for(g, px=16, py=12, span=span, **kw)


def test_camera_render_reproduces_bilinear_fields():
    g, cam = _cam()
    x, y, _ = g.node_coords()
    X, Y = x[0], y[0]                                   # face z = 0, shape (ny1, nx1)
    assert np.allclose(cam.render(np.full(X.shape, 3.25)), 3.25)
    lin = 1.0 + 0.5 * X - 0.25 * Y                      # bilinear fields are interpolated exactly;
    pix = cam.render(lin)                               # pixel average = value at pixel centre
    px = cam.x0 + (np.arange(cam.px) + 0.5) * (cam.x1 - cam.x0) / cam.px
    py = cam.y0 + (np.arange(cam.py) + 0.5) * (cam.y1 - cam.y0) / cam.py
    assert np.allclose(pix, 1.0 + 0.5 * px[None, :] - 0.25 * py[:, None], atol=1e-12)


def test_observe_quantised_and_loglik_peaks_at_truth():
    g, cam = _cam()
    x, y, _ = g.node_coords()
    field = 20.0 * np.exp(-(x[0] ** 2 + y[0] ** 2) / 8.0)
    rng = np.random.default_rng(0)
    data = cam.observe(field, rng)
    assert np.allclose(np.round(data / 0.1) * 0.1, data)
    ll = [cam.loglik(data, a * field) for a in (0.98, 0.99, 1.0, 1.01, 1.02)]
    assert int(np.argmax(ll)) == 2
    # a datum far in the tail still gives a finite log-probability
    assert np.isfinite(cam.loglik(data, field + 5.0))


def test_loglik_matches_quadrature_of_the_gaussian_over_the_rounding_cell():
    """log p(D|T) = sum_p log int_{D_p - q/2}^{D_p + q/2} N(t; T_p, sigma^2) dt,
    checked pixel by pixel against numerical quadrature, incl. a datum 4 sigma in the tail."""
    from scipy.integrate import quad
    g, cam = _cam()
    cam1 = inv.Camera(cam.nodes_x, cam.nodes_y, cam.x0, cam.x1, cam.y0, cam.y1, px=1, py=1, sub=2)
    front = np.full((g.ne[1] + 1, g.ne[0] + 1), 0.0)
    for T, D in ((20.0, 20.0), (20.0, 20.1), (20.03, 19.9), (20.0, 20.4), (20.0, 19.6)):
        front[:] = T
        dens = lambda t: np.exp(-0.5 * ((t - T) / 0.1) ** 2) / (0.1 * np.sqrt(2 * np.pi))
        ref = np.log(quad(dens, D - 0.05, D + 0.05, epsabs=0, epsrel=1e-12)[0])
        assert abs(cam1.loglik(np.array([[D]]), front) - ref) < 1e-9 * max(1.0, abs(ref))


def test_metropolis_hastings_recovers_gaussian_posterior():
    rng = np.random.default_rng(1)
    mu, sd = 3.175, 0.2

    def ll(th):
        return -0.5 * ((th - mu) / sd) ** 2

    res = inv.metropolis_hastings(ll, [6.35] * 8, 0.0, 12.7, 2500, 200, 0.4, rng)
    s = res.samples.ravel()
    assert abs(s.mean() - mu) < 0.02 and abs(s.std() - sd) < 0.02
    assert 0.2 < res.accept_rate < 0.9
    assert s.min() >= 0.0 and s.max() <= 12.7


def test_mh_uniform_prior_truncation():
    rng = np.random.default_rng(2)
    res = inv.metropolis_hastings(lambda th: np.zeros_like(th), [0.1] * 4, 0.0, 1.0, 4000, 100, 0.3, rng)
    s = res.samples.ravel()
    assert s.min() >= 0.0 and s.max() <= 1.0
    assert abs(s.mean() - 0.5) < 0.03               # flat likelihood -> uniform posterior


def test_corrosion_fields_match_generator():
    g = synth.c5_grid(24)
    for d in (0.0, 3.175, 7.0, 12.7):
        k, c = inv.corrosion_fields(g, d, 15.0, 12.7)
        k2, c2 = synth.ids_to_fields(synth.corrosion_ids(g, d, 15.0, 12.7))
        assert np.array_equal(k, k2) and np.array_equal(c, c2)


@pytest.mark.gpu
def test_inversion_recovers_depth_small_plate():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    g = synth.c5_grid(24)
    fwd = inv.CorrosionForward(g, nsteps=40, rtol=1e-8)
    cam = inv.camera_for(g, px=24, py=24, span=12.0)
    truth = 3.175
    data = cam.observe(fwd.fronts([truth])[0], np.random.default_rng(3))
    res = inv.invert(fwd, cam, data, chains=4, n_samples=60, burn_in=30, step=0.4, seed=4)
    est = res.samples.mean()
    assert abs(est - truth) < 0.5, (est, res.samples.std())
    assert fwd.calls > 100
