"""Golden fixtures (tests/golden/, written by tests/golden/make_golden.py).

CPU: the oracle against the reference's known answers (reference_kats.json)
and against its own committed fp64 trajectories (a regression pin).
GPU: the CUDA path against the committed trajectories at the north-star
parity bar (σ² per iteration within 1e-5 relative, final points within 1e-4
of the scene's bounding-box diagonal), without running the oracle.
"""
import importlib.util
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SIGMA_RTOL = 1e-5
POINT_FRAC = 1e-4


def _maker():
    spec = importlib.util.spec_from_file_location("make_golden",
                                                  os.path.join(GOLDEN, "make_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _fixture(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return json.loads(str(z["spec"])), z["sigma2_trace"], z["transformed"]


TRAJ = sorted(_maker().TRAJECTORIES)


@pytest.fixture(scope="module")
def fc():
    import paper_2006_06281_b200 as f
    return f


@pytest.fixture(scope="module")
def ctx(fc):
    c = fc.Context(0)
    yield c
    c.close()


def test_reference_kats(orc):
    kats = {k["name"]: k for k in json.load(open(os.path.join(GOLDEN, "reference_kats.json")))}
    k = kats["posterior_scalar_with_outlier"]["inputs"]
    p, _ = orc.posterior(np.array(k["x"]), np.array(k["y"]), k["omega"], k["sigma2"])
    assert p[0, 0] == pytest.approx(kats["posterior_scalar_with_outlier"]["value"], rel=1e-12)
    k = kats["posterior_equidistant"]["inputs"]
    p, _ = orc.posterior(np.array(k["x"]), np.array(k["y"]), k["omega"], k["sigma2"])
    assert np.allclose(p[:, 0], kats["posterior_equidistant"]["value"], rtol=1.19e-5)
    c, _ = orc.enforce_row_constraint(np.array(kats["row_constraint"]["inputs"]["p"]))
    assert np.allclose(c, kats["row_constraint"]["value"], rtol=1.19e-5, atol=0)
    k = kats["solve_fast_scalar"]["inputs"]
    w = orc.solve_fast(np.array(k["u"]), np.array(k["lam"]), k["lambda_reg"], k["sigma2"],
                       np.array(k["residual"]))
    assert w[0, 0] == pytest.approx(kats["solve_fast_scalar"]["value"], rel=1e-12)
    k = kats["gram_scalar"]["inputs"]
    assert orc.build_gram(np.array(k["x"]), k["beta"])[0, 1] == pytest.approx(
        kats["gram_scalar"]["value"], rel=1e-14)
    k = kats["eigen_duplicates"]["inputs"]
    _, lam, _ = orc.eigendecompose(orc.build_gram(np.array(k["x"]), k["beta"]), 2)
    assert np.allclose(lam, kats["eigen_duplicates"]["value"], atol=1e-12, rtol=0)
    k = kats["init_sigma2_scalar"]["inputs"]
    assert orc.init_sigma2(np.array(k["x"]), np.array(k["y"])) == pytest.approx(
        kats["init_sigma2_scalar"]["value"], rel=1e-14)


@pytest.mark.parametrize("name", TRAJ)
def test_oracle_reproduces_fixture(orc, name):
    spec, trace, pts = _fixture(name)
    x, y = _maker().trajectory_inputs(spec)
    r = orc.register(x, y, omega=spec["omega"], beta=spec["beta"], lambda_reg=spec["lambda_reg"],
                     iterations=spec["iterations"], variant=spec["variant"],
                     rank_fraction=spec["rank_fraction"])
    assert np.allclose(r.sigma2_trace, trace, rtol=1e-12, atol=0)
    assert np.allclose(r.transformed, pts, rtol=0, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name", TRAJ)
def test_cuda_path_matches_fixture(ctx, fc, name):
    spec, trace, pts = _fixture(name)
    x, y = _maker().trajectory_inputs(spec)
    cfg = fc.RegistrationConfig(omega=spec["omega"], beta=spec["beta"],
                                lambda_reg=spec["lambda_reg"], iterations=spec["iterations"],
                                variant=spec["variant"], rank_fraction=spec["rank_fraction"])
    got = ctx.register(x, y, cfg)
    rel = np.abs(got.sigma2_trace / trace - 1).max()
    diag = np.linalg.norm(y.max(0) - y.min(0))
    frac = np.abs(got.transformed - pts).max() / diag
    print(f"{name}: σ² rel {rel:.3g}, points {frac:.3g} of the bbox diagonal")
    assert len(got.sigma2_trace) == len(trace)
    assert rel <= SIGMA_RTOL, rel
    assert frac <= POINT_FRAC, frac
