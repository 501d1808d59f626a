"""Near-field pair forms: the Gram form (leaf-centred
|t|^2 + |s|^2 - 2 t.s) for smooth kernels on tiles within the bound, the
difference form elsewhere. Every case is checked against the unmodified
reference FKT (oracle/_ref) at the 1e-10 gate and asserts which forms ran, so
the Gram-only, difference-only and mixed launches are all exercised."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cloud(fkt, x):
    return fkt.PointCloud.from_array(np.ascontiguousarray(x))


def _check(fkt, ref, x, name, prm, p, theta, leaf, y, diag=None):
    kw = {} if diag is None else {"diagonal": diag}
    pl = fkt.plan(_cloud(fkt, x), fkt.makeKernel(name, prm), fkt.FktOptions(p=p, theta=theta, leafCapacity=leaf, **kw))
    rp = ref.RefPlan(x, name, prm, p=p, theta=theta, leaf=leaf, diagonal=diag)
    err = fkt.relativeError(pl.multiply(y), rp.multiply(y))
    assert err <= 1e-10, (name, err)
    return pl.near_forms(), err


@pytest.mark.parametrize("name,prm,d", [("matern32", {"sigma": 1.3, "rho": 0.2}, 3), ("cauchy", {"sigma": 0.7}, 2),
                                        ("rational-quadratic", {"sigma": 0.5}, 3), ("gaussian", {}, 5),
                                        ("cauchy", {"sigma": 1.0}, 5)])
def test_gram_tiles_match_reference(fkt, ref, name, prm, d):
    rng = np.random.default_rng(3)
    x = rng.random((20000, d))
    (g, t), _ = _check(fkt, ref, x, name, prm, 6 if d < 5 else 4, 0.5, 256, rng.standard_normal(20000))
    assert t > 0 and g == t  # unit cube in canonical scale: every tile in Gram form


def test_difference_form_when_the_bound_fails(fkt, ref):
    # rho = 0.002 scales a unit cube to ~866 canonical units: every leaf is
    # outside the Gram bound, so the difference-form launch runs alone
    rng = np.random.default_rng(4)
    x = rng.random((12000, 3))
    (g, t), _ = _check(fkt, ref, x, "matern32", {"sigma": 1.0, "rho": 0.002}, 4, 0.5, 128, rng.standard_normal(12000))
    assert t > 0 and g == 0


def test_mixed_forms_in_one_plan(fkt, ref):
    # a dense cluster (small leaves, Gram) plus a sparse halo 1000x wider
    # (large leaves, difference form) under a Gaussian of unit length scale
    rng = np.random.default_rng(5)
    x = np.vstack([0.01 * rng.standard_normal((15000, 3)), 40.0 * rng.standard_normal((3000, 3))])
    y = rng.standard_normal(x.shape[0])
    (g, t), _ = _check(fkt, ref, x, "gaussian", {}, 4, 0.5, 128, y)
    assert 0 < g < t
    (g2, t2), _ = _check(fkt, ref, x, "matern32", {"sigma": 1.0, "rho": 1.0}, 4, 0.5, 128, y)
    assert 0 < g2 < t2


def test_gram_duplicates_and_coincident_sources(fkt, ref):
    # duplicates: Gram q rounds around 0 (the bias keeps it >= 0; Gaussian and
    # Matern take K(0) to ~1e-16)
    rng = np.random.default_rng(6)
    x = np.repeat(rng.random((3000, 3)), 4, axis=0)
    y = rng.standard_normal(x.shape[0])
    for name, prm in (("gaussian", {}), ("matern32", {"sigma": 1.0, "rho": 0.4}), ("cauchy", {"sigma": 2.0})):
        (g, t), err = _check(fkt, ref, x, name, prm, 4, 0.6, 64, y)
        assert g == t and err <= 1e-11


@pytest.mark.parametrize("name,prm,d", [("gaussian", {}, 3), ("matern32", {"sigma": 1.0, "rho": 0.4}, 3),
                                        ("cauchy", {"sigma": 0.5}, 2), ("rational-quadratic", {}, 5),
                                        ("gaussian", {}, 5)])
def test_gram_single_leaf_equals_dense(fkt, ref, name, prm, d):
    # one leaf: the FKT is the near field alone, so this pins the Gram form's
    # accuracy against dense (reference test_transform.cpp:38-50), duplicates
    # included
    rng = np.random.default_rng(9)
    x = np.repeat(rng.random((250, d)), 2, axis=0)
    y = rng.standard_normal(500)
    pl = fkt.plan(_cloud(fkt, x), fkt.makeKernel(name, prm), fkt.FktOptions(p=4, theta=0.5, leafCapacity=512))
    g, t = pl.near_forms()
    assert g == t == 2
    # the reference's own case (cauchy, sigma 1) holds 1e-13 (test_gpu_reference_suite);
    # longer canonical scales raise the Gram rounding bound B (here B ~ 70)
    # the exp kernels' near field uses a 1024-entry table with a degree-2 remainder
    # (|e^f - p(f)| <= 6.5e-12 relative per pair, fastmath.cuh): 1e-11 here, 1e-10 on z
    assert fkt.relativeError(pl.multiply(y), ref.dense(x, name, prm, y)) <= 1e-11


def test_select_kernels_keep_difference_form(fkt, ref):
    rng = np.random.default_rng(7)
    x = rng.random((8000, 3))
    y = rng.standard_normal(8000)
    (g, _), _ = _check(fkt, ref, x, "matern32", {"sigma": 1.0, "rho": 0.3}, 4, 0.5, 128, y, diag=0.5)
    assert g == 0  # explicit r == 0 select
    (g, _), _ = _check(fkt, ref, x, "inverse-r", {}, 4, 0.5, 128, y)
    assert g == 0  # singular kernel
