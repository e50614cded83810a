"""Pin the CPU oracle against the reference's own known-answer tests.

Each test restates one doctest case from /root/reference/proj/tests (cited)
with the same inputs (test_util.hpp generators restated in the oracle with
std::mt19937_64) and the same tolerances.  No GPU needed.
"""
import math

import numpy as np
import pytest


def approx(v, rel=1e-5):
    # doctest::Approx default epsilon is float-epsilon*100 ≈ 1.19e-5
    return pytest.approx(v, rel=rel)


# ------------------------------------------------ test_correspondence.cpp


def test_single_component_takes_all_mass(orc):  # test_correspondence.cpp:10-16
    x = np.array([[0.0, 0.0]])
    y = orc.make_cloud(5, 2, 1)
    p, _ = orc.posterior(x, y, 0.0, 0.5)
    assert np.all(np.abs(p[0] - 1.0) <= 1e-14)


def test_equidistant_symmetry(orc):  # test_correspondence.cpp:18-24
    x = np.array([[-1.0, 0.0], [1.0, 0.0]])
    y = np.array([[0.0, 0.3]])
    p, _ = orc.posterior(x, y, 0.0, 0.25)
    assert p[0, 0] == approx(0.5) and p[1, 0] == approx(0.5)


def test_scalar_with_outlier(orc):  # test_correspondence.cpp:26-35
    p, _ = orc.posterior(np.array([[0.0]]), np.array([[1.0]]), 0.5, 1.0)
    e = math.exp(-0.5)
    assert p[0, 0] == pytest.approx(e / (e + math.sqrt(2 * math.pi)), rel=1e-12)
    assert p[0, 0] == pytest.approx(0.1948, rel=1e-3)


def test_posterior_parameter_handling(orc):  # test_correspondence.cpp:37-45
    x = orc.make_cloud(3, 2, 2)
    y = orc.make_cloud(4, 2, 3)
    for omega in (1.0, -0.1):
        with pytest.raises(orc.OracleError) as ei:
            orc.posterior(x, y, omega, 1.0)
        assert ei.value.kind == "ParameterError"
    _, clamped = orc.posterior(x, y, 0.5, 1e-30)
    assert clamped


def test_posterior_column_sums(orc):  # test_correspondence.cpp:47-60
    x = orc.make_cloud(8, 3, 4)
    y = orc.make_cloud(6, 3, 5)
    p0, _ = orc.posterior(x, y, 0.0, 0.3)
    assert np.allclose(p0.sum(0), 1.0, rtol=1e-10, atol=0)
    p, _ = orc.posterior(x, y, 0.7, 0.3)
    assert np.all(p.sum(0) <= 1 + 1e-10)
    assert p.min() >= 0 and p.max() <= 1


def test_posterior_unshifted_formula(orc):  # test_correspondence.cpp:62-83
    x = orc.make_cloud(5, 2, 6)
    y = orc.make_cloud(7, 2, 7)
    omega, s2 = 0.3, 0.4
    p, _ = orc.posterior(x, y, omega, s2)
    cc = (2 * math.pi * s2) ** 1.0 * (omega / (1 - omega)) * (5 / 7)
    for j in range(7):
        k = np.exp(-((y[j] - x) ** 2).sum(1) / (2 * s2))
        naive = k / (cc + k.sum())
        assert np.allclose(p[:, j], naive, rtol=1e-12, atol=0)


def test_row_constraint(orc):  # test_correspondence.cpp:85-106
    raw = np.array([[0.2, 0.2], [0.0, 0.5]])
    c, deg = orc.enforce_row_constraint(raw)
    assert c[0, 0] == approx(0.5) and c[0, 1] == approx(0.5)
    assert c[1, 0] == 0.0 and c[1, 1] == approx(1.0)
    assert deg == []
    again, _ = orc.enforce_row_constraint(c)
    assert np.abs(again - c).max() == 0.0
    fixed, deg = orc.enforce_row_constraint(np.zeros((1, 4)))
    assert deg == [0]
    assert np.all(fixed == 0.25)


def test_estimated_targets(orc):  # test_correspondence.cpp:108-139
    y = np.array([[0.0, 0.0], [2.0, 0.0]])
    assert np.abs(orc.estimated_targets(np.eye(2), y) - y).max() == 0.0
    assert orc.estimated_targets(np.full((1, 2), 0.5), y)[0, 0] == approx(1.0)
    y2 = np.array([[0.0, 0.0], [4.0, 0.0]])
    assert orc.estimated_targets(np.array([[0.25, 0.75]]), y2)[0, 0] == approx(3.0)
    ybig = orc.make_cloud(9, 3, 8)
    rc = orc.random_row_constrained(12, 9, 9)
    t = orc.estimated_targets(rc, ybig)
    assert np.all(t.min(0) >= ybig.min(0) - 1e-12)
    assert np.all(t.max(0) <= ybig.max(0) + 1e-12)
    with pytest.raises(orc.OracleError):
        orc.estimated_targets(np.eye(2), orc.make_cloud(5, 2, 1))


# ------------------------------------------------------ test_solvers.cpp


def make_instance(orc, m, n, d, seed):  # test_solvers.cpp:15-24
    x = orc.make_cloud(m, d, seed)
    y = orc.make_cloud(n, d, seed + 1)
    phi = orc.build_gram(x, 2.0)
    u, lam, raw = orc.eigendecompose(phi, m)
    p = orc.random_row_constrained(m, n, seed + 2)
    return dict(x=x, y=y, phi=phi, u=u, lam=lam, p=p, lreg=10.0, s2=0.3)


def test_solve_fast_zero_and_scalar(orc):  # test_solvers.cpp:35-49
    inst = make_instance(orc, 6, 6, 2, 20)
    w = orc.solve_fast(inst["u"], inst["lam"], 10.0, 0.3, np.zeros((6, 2)))
    assert np.abs(w).max() == 0.0
    w = orc.solve_fast(np.ones((1, 1)), np.ones(1), 2.0, 0.25, np.array([[0.8]]))
    assert w[0, 0] == pytest.approx(0.8 / 1.5, rel=1e-14)


def test_solve_fast_matches_dense(orc):  # test_solvers.cpp:51-68
    inst = make_instance(orc, 100, 80, 3, 21)
    r = inst["p"] @ inst["y"] - inst["x"]
    w = orc.solve_fast(inst["u"], inst["lam"], inst["lreg"], inst["s2"], r)
    a = inst["phi"] + inst["lreg"] * inst["s2"] * np.eye(100)
    dense = np.linalg.solve(a, r)
    assert np.linalg.norm(w - dense) <= 1e-8 * np.linalg.norm(dense)
    assert np.linalg.norm(a @ w - r) <= 1e-8 * np.linalg.norm(r)
    w35 = orc.solve_fast(inst["u"], inst["lam"], inst["lreg"], inst["s2"], 3.5 * r)
    assert np.linalg.norm(w35 - 3.5 * w) <= 1e-10 * np.linalg.norm(w35)


def test_lowrank_at_full_rank(orc):  # test_solvers.cpp:70-79
    inst = make_instance(orc, 40, 30, 2, 22)
    r = inst["p"] @ inst["y"] - inst["x"]
    full = orc.solve_fast(inst["u"], inst["lam"], inst["lreg"], inst["s2"], r)
    lr = orc.solve_fast_lowrank(inst["u"], inst["lam"], inst["lreg"], inst["s2"], r)
    assert np.abs(full - lr).max() <= 1e-12


def test_lowrank_truncated_galerkin(orc):  # test_solvers.cpp:81-102
    inst = make_instance(orc, 100, 100, 3, 23)
    u, lam, _ = orc.eigendecompose(inst["phi"], 10)
    r = inst["p"] @ inst["y"] - inst["x"]
    lr = orc.solve_fast_lowrank(u, lam, inst["lreg"], inst["s2"], r)
    a = u @ np.diag(lam) @ u.T + inst["lreg"] * inst["s2"] * np.eye(100)
    z = np.linalg.solve(u.T @ a @ u, u.T @ r)
    dense = u @ z
    assert np.linalg.norm(lr - dense) <= 1e-8 * np.linalg.norm(dense)
    assert np.linalg.norm(lr - u @ (u.T @ lr)) <= 1e-10 * np.linalg.norm(lr)
    assert np.linalg.norm(u.T @ (a @ lr - r)) <= 1e-8 * np.linalg.norm(r)


@pytest.mark.parametrize("seed", [30, 31, 32])
def test_cpd_baseline_equals_fast(orc, seed):  # test_solvers.cpp:104-113
    inst = make_instance(orc, 100, 90, 3, seed)
    r = inst["p"] @ inst["y"] - inst["x"]
    fast = orc.solve_fast(inst["u"], inst["lam"], inst["lreg"], inst["s2"], r)
    cpd = orc.solve_cpd_baseline(inst["phi"], inst["p"], inst["lreg"], inst["s2"], inst["y"],
                                 inst["x"])
    assert np.linalg.norm(fast - cpd) <= 1e-8 * np.linalg.norm(fast)


def test_apply_transform_variants(orc):  # test_solvers.cpp:151-190
    inst = make_instance(orc, 30, 30, 3, 35)
    x, phi, u, lam = inst["x"], inst["phi"], inst["u"], inst["lam"]
    assert np.abs(orc.apply_transform(x, phi, np.zeros((30, 3))) - x).max() == 0.0
    x1 = np.array([[0.1, 0.2]])
    t1 = orc.apply_transform(x1, orc.build_gram(x1, 2.0), np.array([[0.3, -0.4]]))
    assert t1[0, 0] == approx(0.4) and t1[0, 1] == approx(-0.2)
    w = orc.make_cloud(30, 3, 36) * 0.1
    t = orc.apply_transform(x, phi, w)
    for i in range(30):
        acc = x[i] + (w * np.exp(-((x[i] - x) ** 2).sum(1) / 8.0)[:, None]).sum(0)
        assert np.abs(t[i] - acc).max() <= 1e-10
    assert np.abs(orc.apply_transform_lowrank(x, u, lam, w) - t).max() <= 1e-10
    ut, lt, _ = orc.eigendecompose(phi, 5)
    recon = ut @ np.diag(lt) @ ut.T
    assert np.abs(orc.apply_transform_lowrank(x, ut, lt, w) - (x + recon @ w)).max() <= 1e-10


def test_update_sigma2(orc):  # test_solvers.cpp:192-223
    y = orc.make_cloud(10, 2, 40)
    assert orc.update_sigma2(y, np.eye(10), y) == 1e-10
    assert orc.update_sigma2(np.array([[2.0]]), np.ones((1, 1)), np.array([[0.0]])) == \
        pytest.approx(4.0, rel=1e-14)
    yb = orc.make_cloud(30, 3, 41)
    xb = orc.make_cloud(20, 3, 42)
    p = orc.random_row_constrained(20, 30, 43)
    trace = orc.update_sigma2(yb, p, xb)
    dbl = sum(p[i, j] * ((yb[j] - xb[i]) ** 2).sum() for i in range(20) for j in range(30))
    assert trace == pytest.approx(dbl / 60.0, rel=1e-10)
    with pytest.raises(orc.OracleError) as ei:
        orc.update_sigma2(yb, p, xb, row_constrained=False)
    assert ei.value.kind == "ParameterError"


# ------------------------------------------------------- test_kernel.cpp


def test_gram_scalars(orc):  # test_kernel.cpp:11-26
    assert orc.build_gram(np.array([[0.3, -0.7]]), 2.0)[0, 0] == 1.0
    assert orc.build_gram(np.array([[1.0, 1.0], [1.0, 1.0]]), 2.0).min() == approx(1.0)
    line = np.array([[0.0], [2.0]])
    assert orc.build_gram(line, 2.0)[0, 1] == approx(math.exp(-0.5))
    for beta in (0.0, -1.0):
        with pytest.raises(orc.OracleError):
            orc.build_gram(line, beta)


def test_gram_invariants(orc):  # test_kernel.cpp:28-38
    phi = orc.build_gram(orc.make_cloud(60, 3, 11), 2.0)
    assert np.abs(phi - phi.T).max() == 0.0
    assert np.diag(phi).min() == 1.0 and phi.min() > 0 and phi.max() <= 1.0
    _, lam, _ = orc.eigendecompose(phi, 60)
    assert lam.min() >= -1e-8 * 60


def test_eig_near_identity_and_duplicates(orc):  # test_kernel.cpp:40-59
    phi = orc.build_gram(np.array([[0.0], [1e5], [2e5], [3e5]]), 2.0)
    u, lam, _ = orc.eigendecompose(phi, 4)
    assert np.allclose(lam, 1.0, rtol=1e-12)
    assert np.abs(u.T @ u - np.eye(4)).max() <= 1e-8
    _, lam, _ = orc.eigendecompose(orc.build_gram(np.ones((2, 2)), 2.0), 2)
    assert lam[0] == approx(2.0) and lam[1] == pytest.approx(0.0, abs=1e-12)


def test_full_rank_reconstruction(orc):  # test_kernel.cpp:61-75
    phi = orc.build_gram(orc.make_cloud(50, 3, 3), 2.0)
    u, lam, _ = orc.eigendecompose(phi, 50)
    assert np.abs(u.T @ u - np.eye(50)).max() <= 1e-8
    assert np.linalg.norm(u @ np.diag(lam) @ u.T - phi) <= 1e-6 * np.linalg.norm(phi)
    assert np.all(np.diff(lam) <= 0)
    for r in (0, 51):
        with pytest.raises(orc.OracleError):
            orc.eigendecompose(phi, r)


# -------------------------------------------------- test_registration.cpp


def test_init_sigma2(orc):  # test_registration.cpp:13-27
    s = np.array([[3.0, 4.0]])
    assert orc.init_sigma2(s, s) == 0.0
    assert orc.init_sigma2(np.array([[0.0]]), np.array([[2.0]])) == pytest.approx(4.0, rel=1e-14)
    a = orc.make_cloud(10, 3, 50)
    b = orc.make_cloud(15, 3, 51)
    base = orc.init_sigma2(a, b)
    sh = np.array([5.0, -2.0, 1.0])
    assert orc.init_sigma2(a + sh, b + sh) == pytest.approx(base, rel=1e-10)


def test_self_registration(orc):  # test_registration.cpp:29-42
    x = orc.make_torus(120, 52)
    res = orc.register(x, x, iterations=50)
    assert len(res.sigma2_trace) == 50
    rmse = math.sqrt(((res.transformed - x) ** 2).sum(1).mean())
    assert rmse <= 1e-3
    assert np.all(np.diff(res.sigma2_trace) <= 1e-12)


def test_zero_iterations(orc):  # test_registration.cpp:44-53
    x = orc.make_cloud(20, 2, 53)
    y = orc.make_cloud(25, 2, 54)
    res = orc.register(x, y, iterations=0)
    assert np.abs(res.transformed - x).max() <= 1e-12
    assert np.abs(res.coefficients).max() == 0.0
    assert len(res.sigma2_trace) == 0


def test_timing_identities(orc):  # test_registration.cpp:55-70
    x = orc.make_cloud(60, 3, 55)
    y = orc.make_cloud(60, 3, 56)
    for v in ("fast", "fast_lowrank"):
        t = orc.register(x, y, iterations=5, variant=v).timing
        assert t["t_f"] == t["t_eig"] + t["t_iter"]
        assert t["t_total"] == t["t_c"] + t["t_f"] + t["t_o"]


def test_bitwise_determinism(orc):  # test_registration.cpp:72-83
    x = orc.make_torus(80, 57)
    y = orc.make_torus(90, 58)
    a = orc.register(x, y, iterations=15)
    b = orc.register(x, y, iterations=15)
    assert np.array_equal(a.sigma2_trace, b.sigma2_trace)
    assert np.array_equal(a.transformed, b.transformed)


def test_degenerate_sizes(orc):  # test_registration.cpp:85-97
    x = np.array([[0.2, 0.1]])
    y = np.array([[0, 0], [1, 0], [0, 1.0]])
    for v in ("fast", "fast_lowrank"):
        res = orc.register(x, y, iterations=3, variant=v)
        assert res.transformed.shape == (1, 2) and len(res.sigma2_trace) == 3


def test_register_validation(orc):  # test_registration.cpp:99-106
    x = orc.make_cloud(5, 2, 59)
    with pytest.raises(orc.OracleError) as ei:
        orc.register(x, orc.make_cloud(5, 3, 60))
    assert ei.value.kind == "DimensionError"
    with pytest.raises(orc.OracleError) as ei:
        orc.register(x, x, iterations=-1)
    assert ei.value.kind == "ParameterError"


# -------------------------------------------------------- test_pointset.cpp


def test_normalize_pair(orc):  # test_pointset.cpp:77-88, :90-96, :98-113
    xo, yo, c, s, deg = orc.normalize_pair(np.array([[0, 0], [4, 0.0]]), np.array([[2, 0.0]]))
    assert c[0] == approx(2.0) and c[1] == approx(0.0) and s == approx(2.0) and not deg
    assert xo[0, 0] == approx(-1.0) and xo[1, 0] == approx(1.0) and yo[0, 0] == approx(0.0)
    z = np.zeros((1, 2))
    xo, _, _, s, deg = orc.normalize_pair(z, z)
    assert s == 1.0 and deg and np.abs(xo).max() == 0.0
    for seed in (1, 2, 3):
        x = orc.make_cloud(40, 3, seed) * 37 + 5
        y = orc.make_cloud(60, 3, seed + 100) * 37 + 5
        xo, yo, c, s, _ = orc.normalize_pair(x, y)
        assert np.abs(xo).max() <= 1 + 1e-15 and np.abs(yo).max() <= 1 + 1e-15
        assert np.abs(xo * s + c - x).max() <= 1e-12 * np.abs(x).max()


# ------------------------------------------------------------ acceptance.cpp


def acc_instance(orc, m, d, seed):  # acceptance.cpp:40-50
    x = orc.make_cloud(m, d, seed)
    y = orc.make_cloud(m + m // 5, d, seed + 1)
    phi = orc.build_gram(x, 2.0)
    u, lam, _ = orc.eigendecompose(phi, m)
    p = orc.random_row_constrained(m, y.shape[0], seed + 2)
    return x, y, phi, u, lam, p, 10.0, 0.05 + 0.01 * (seed % 30)


def test_acceptance_criterion_1(orc):  # acceptance.cpp:53-77 (first 12 of 50 instances)
    worst = 0.0
    for seed in range(12):
        x, y, phi, u, lam, p, lreg, s2 = acc_instance(orc, [50, 100, 200][seed % 3],
                                                      [2, 3][seed % 2], 1000 + seed * 7)
        r = p @ y - x
        fast = orc.solve_fast(u, lam, lreg, s2, r)
        cpd = orc.solve_cpd_baseline(phi, p, lreg, s2, y, x)
        worst = max(worst, np.linalg.norm(fast - cpd) / np.linalg.norm(fast))
    assert worst <= 1e-8


def test_acceptance_criterion_3(orc):  # acceptance.cpp:118-141
    worst = 0.0
    for seed in range(50):
        m = 20 + (seed % 5) * 10
        n, d = m + 10, (3 if seed % 2 else 2)
        y = orc.make_cloud(n, d, 3000 + seed)
        xt = orc.make_cloud(m, d, 4000 + seed)
        p = orc.random_row_constrained(m, n, 5000 + seed)
        trace = orc.update_sigma2(y, p, xt)
        d2 = ((y[None, :, :] - xt[:, None, :]) ** 2).sum(-1)
        dbl = (p * d2).sum() / (d * m)
        worst = max(worst, abs(trace - dbl) / dbl)
    assert worst <= 1e-10


def test_acceptance_criterion_8(orc):  # acceptance.cpp:263-316 (module invariants)
    x = orc.make_cloud(30, 3, 14)
    y = orc.make_cloud(40, 3, 15)
    p, _ = orc.posterior(x, y, 0.7, 0.2)
    p, _ = orc.enforce_row_constraint(p)
    assert np.abs(p.sum(1) - 1).max() <= 1e-10
    t = orc.estimated_targets(p, y)
    assert np.all(t.min(0) >= y.min(0) - 1e-12) and np.all(t.max(0) <= y.max(0) + 1e-12)
    pp, _ = orc.enforce_row_constraint(p)
    assert np.abs(pp - p).max() <= 1e-15
    phi = orc.build_gram(x, 2.0)
    u, lam, _ = orc.eigendecompose(phi, 30)
    assert lam.min() >= -1e-8 * 30
    r = p @ y - x
    w = orc.solve_fast(u, lam, 10.0, 0.3, r)
    a = phi + 3.0 * np.eye(30)
    assert np.linalg.norm(a @ w - r) <= 1e-8 * np.linalg.norm(r)
    r1 = orc.register(x, y, iterations=10)
    r2 = orc.register(x, y, iterations=10)
    assert np.array_equal(r1.sigma2_trace, r2.sigma2_trace)


# ------------------------------------- streaming restatement == dense oracle


@pytest.mark.parametrize("omega,s2", [(0.0, 0.3), (0.2, 1e-3), (0.7, 2e-5), (0.0, 1e-6)])
def test_stream_estep_matches_dense(orc, omega, s2):
    """The non-materialising algebra the GPU uses
    equals posterior → enforce_row_constraint → estimated_targets."""
    xt = orc.make_cloud(300, 3, 70) * 0.5
    y = orc.make_cloud(360, 3, 71) * 0.5
    p, _ = orc.posterior(xt, y, omega, s2)
    raw_rows = p.sum(1)
    pc, deg = orc.enforce_row_constraint(p)
    pty = orc.estimated_targets(pc, y)
    es = orc.estep_stream(xt, y, omega, s2)
    assert sorted(np.nonzero(es.degenerate)[0].tolist()) == deg
    assert np.abs(es.ptilde_y - pty).max() <= 1e-12
    ok = raw_rows > 1e-290
    assert np.allclose(es.p1[ok], raw_rows[ok], rtol=1e-9, atol=0)
    d2 = ((y[None, :, :] - xt[:, None, :]) ** 2).sum(-1)
    var = (pc * d2).sum(1)
    assert np.allclose(es.var, var, rtol=1e-9, atol=1e-300)
    assert np.allclose(es.pt1, p.sum(0), rtol=1e-10, atol=1e-300)


def test_spectral_cache_round_trip(orc, tmp_path):  # test_kernel.cpp:98-110
    x = orc.make_cloud(20, 3, 5)
    u, lam, _ = orc.eigendecompose(orc.build_gram(x, 2.0), 7)
    path = str(tmp_path / "fcpd_cache.bin")
    orc.save_spectral_cache(path, u, lam, 2.0)
    back, blam, beta = orc.load_spectral_cache(path)
    assert beta == 2.0 and back.shape == (20, 7)
    assert np.abs(back - u).max() == 0.0 and np.abs(blam - lam).max() == 0.0
    raw = open(path, "rb").read()
    assert raw[:4] == b"FCPD" and len(raw) == 4 + 4 + 8 + 8 + 8 + 8 * (20 * 7 + 7)
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(orc.OracleError) as ei:
        orc.load_spectral_cache(str(bad))
    assert ei.value.kind == "ParseError"


@pytest.mark.parametrize("variant,omega", [("fast", 0.0), ("fast_lowrank", 0.3)])
def test_streaming_register_equals_dense(orc, variant, omega):
    """The streaming restatement used as the oracle for configs 2–4 (no M×N
    matrix, per-row σ²) equals the dense faithful restatement."""
    x = orc.make_torus(150, 3)
    y = orc.make_torus(170, 4) * 1.05
    xn, _, _, _, _ = orc.normalize_pair(x, y)
    phi = orc.build_gram(xn, 2.0)
    k = 150 if variant == "fast" else 30
    u, lam, raw = orc.eigendecompose(phi, k)
    ref = orc.register(x, y, omega=omega, beta=2.0, lambda_reg=3.0, iterations=20, variant=variant,
                       rank_fraction=k / 150)
    st = orc.register_stream(x, y, u, lam, raw if variant == "fast" else lam, omega=omega,
                             lambda_reg=3.0, iterations=20)
    assert np.abs(st.sigma2_trace / ref.sigma2_trace - 1).max() <= 1e-11
    assert np.abs(st.transformed - ref.transformed).max() <= 1e-11
