"""The fp64 device L2 entry points (l2api.cu, through the C ABI) against the
fp64 oracle on the same inputs: update_sigma2 (solvers.hpp:160-176),
estimated_targets / enforce_row_constraint (correspondence.hpp:83-105),
apply_transform[_lowrank] and solve_fast[_lowrank] (solvers.hpp:61-155),
eigendecompose of a given Φ (kernel.hpp:49-72), normalize_pair
(pointset.hpp:124-148)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2006_06281_b200 as f
    c = f.Context(0)
    yield c
    c.close()


def test_l2_entry_points_match_oracle(ctx, orc):
    import paper_2006_06281_b200 as f
    x = orc.make_cloud(120, 3, 3)
    y = orc.make_cloud(150, 3, 4)
    p = orc.random_row_constrained(120, 150, 5)
    # P·Y and the σ² trace form
    assert np.abs(ctx.estimated_targets(p, y) - orc.estimated_targets(p, y)).max() <= 1e-13
    s2 = ctx.update_sigma2(y, p, x)
    assert s2 == pytest.approx(orc.update_sigma2(y, p, x), rel=1e-12)
    with pytest.raises(f.ParameterError):
        ctx.update_sigma2(y, p, x, row_constrained=False)
    # row constraint with a zero row (uniform fallback)
    raw = p.copy()
    raw[7] = 0.0
    got, deg = ctx.enforce_row_constraint(raw)
    ref, rdeg = orc.enforce_row_constraint(raw)
    assert deg == [7] and np.abs(got - ref).max() <= 1e-15
    # basis, solve, transforms
    phi = orc.build_gram(x, 2.0)
    u, lam, raw_lam = ctx.eigendecompose(phi, 120)
    ru, rlam, rraw = orc.eigendecompose(phi, 120)
    assert np.abs(raw_lam - rraw).max() <= 1e-12 * rraw[0]
    r = orc.estimated_targets(p, y) - x
    w = ctx.solve_fast(u, lam, 10.0, 0.3, r)
    wr = orc.solve_fast(ru, rlam, 10.0, 0.3, r)
    assert np.abs(w - wr).max() <= 1e-8 * np.abs(wr).max()
    t = ctx.apply_transform(x, phi, w)
    assert np.abs(t - orc.apply_transform(x, phi, w)).max() <= 1e-12
    tl = ctx.apply_transform_lowrank(x, u[:, :20], lam[:20], w)
    assert np.abs(tl - orc.apply_transform_lowrank(x, u[:, :20], lam[:20], w)).max() <= 1e-10
    err = ctx.lowrank_reconstruction_error(u[:, :20], lam[:20], phi)
    assert err == pytest.approx(np.sqrt((rraw[20:] ** 2).sum()), rel=1e-6)
    # normalize_pair
    xo, yo, c, sc, dg = ctx.normalize_pair(x * 3 + 1, y * 3 + 1)
    rx, ry, rc, rsc, rdg = orc.normalize_pair(x * 3 + 1, y * 3 + 1)
    assert np.abs(xo - rx).max() == 0.0 and np.abs(yo - ry).max() == 0.0
    assert sc == rsc and dg == rdg
