"""The scene-sharded multi-GPU data plane run as a loopback
group: G virtual ranks on one B200, each with its own scene shard, model
row shard, basis shard and graph nodes, the collectives (reduce-scatter of
the row sums, all-reduce of z and the flagged count, all-gather of x̃ with
the σ² partials, and the conditional fallback exchange) as device kernels.
No rank waits on another: each phase is enqueued for every rank between
collectives on one stream.  Against the single-GPU path (same algorithm,
different fp32 segment boundaries) and the oracle
(registration.hpp:117-161, correspondence.hpp:68-98)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fc():
    import paper_2006_06281_b200 as f
    return f


def bbox_diag(y):
    return float(np.linalg.norm(y.max(0) - y.min(0)))


@pytest.mark.parametrize("world,variant,name,m,cull", [
    (2, "fast", "c1", 2500, "0"), (4, "fast", "c1", 2500, "0"),
    (2, "fast_lowrank", "c2", 12000, "1"), (4, "fast_lowrank", "c2", 12000, "1"),
    (3, "fast_lowrank", "c3", 6000, "1")])
def test_loopback_matches_single_gpu(fc, orc, monkeypatch, world, variant, name, m, cull):
    from paper_2006_06281_b200 import datagen
    monkeypatch.setenv("FCPD_CULL", cull)
    monkeypatch.setenv("FCPD_MSTEP_FUSED", "0")  # the sharded M-step streams the basis
    x, y, w = datagen.generate(name, m=m)
    cfg = datagen.config_for(w, iterations=30)
    cfg.variant = variant
    cfg.rank_fraction = 0.02 if variant == "fast_lowrank" else 1.0
    with fc.Context(0) as one:
        ref = one.register(x, y, cfg)
    with fc.Context.loopback(0, world) as grp:
        assert grp.world == (0, world)
        got = grp.register(x, y, cfg)
        again = grp.register(x, y, cfg)
        k_per_it = grp.kernels_per_iteration
    rel = np.abs(got.sigma2_trace / ref.sigma2_trace - 1).max()
    pts = np.abs(got.transformed - ref.transformed).max() / bbox_diag(y)
    print(f"world {world} {name} {variant}: σ² rel {rel:.3g}  points {pts:.3g}  "
          f"kernels/iteration {k_per_it}")
    # same algorithm, different fp32 segment boundaries per shard
    assert rel <= 1e-6, rel
    assert pts <= 1e-7, pts
    assert np.array_equal(got.sigma2_trace, again.sigma2_trace)  # bitwise reproducible
    assert got.sigma2_initial == pytest.approx(ref.sigma2_initial, rel=1e-12)


@pytest.mark.parametrize("world", [2, 4])
def test_loopback_sharded_topk_basis(fc, monkeypatch, tmp_path, world):
    """The group's top-K setup with row-sharded Φ·V products (each rank its
    M/G rows, an all-gather; kernel.hpp:49-72): every output row is summed
    in the same order as on one GPU, so the basis is the single-GPU one up
    to the last bits of the group's normalisation statistics, and the
    registration matches as in the test above."""
    from paper_2006_06281_b200 import datagen
    monkeypatch.setenv("FCPD_TOPK_MIN_M", "1000")  # force the top-K path at M = 6000
    monkeypatch.setenv("FCPD_MSTEP_FUSED", "0")
    x, y, w = datagen.generate("c2", m=6000)
    cfg = datagen.config_for(w, iterations=20)
    cfg.rank_fraction = 0.02
    with fc.Context(0) as one:
        ref = one.register(x, y, cfg)
        one.save_spectral_cache(str(tmp_path / "one.bin"))
    with fc.Context.loopback(0, world) as grp:
        got = grp.register(x, y, cfg)
        grp.save_spectral_cache(str(tmp_path / "grp.bin"))
    assert got.timing.t_eig > 0.0 and not got.basis_reused
    def read(path):  # kernel.hpp:85-144 layout
        raw = path.read_bytes()
        m, k = np.frombuffer(raw[8:24], dtype=np.uint64)
        u = np.frombuffer(raw[32:32 + 8 * m * k], dtype=np.float64).reshape(m, k)
        lam = np.frombuffer(raw[32 + 8 * m * k:32 + 8 * m * k + 8 * k], dtype=np.float64)
        return u, lam
    ua, la = read(tmp_path / "one.bin")
    ub, lb = read(tmp_path / "grp.bin")
    assert ua.shape == ub.shape
    assert np.abs(la - lb).max() <= 1e-12 * la[0]
    z = np.random.default_rng(5).standard_normal((ua.shape[0], 4))
    pa, pb = ua @ (la[:, None] * (ua.T @ z)), ub @ (lb[:, None] * (ub.T @ z))
    assert np.abs(pa - pb).max() <= 1e-9 * np.abs(pa).max()
    rel = np.abs(got.sigma2_trace / ref.sigma2_trace - 1).max()
    pts = np.abs(got.transformed - ref.transformed).max() / bbox_diag(y)
    print(f"world {world} sharded top-K: σ² rel {rel:.3g} points {pts:.3g} "
          f"t_eig group {got.timing.t_eig:.3f} s single {ref.timing.t_eig:.3f} s")
    assert rel <= 1e-6 and pts <= 1e-7


def test_loopback_fallback_rows_match(fc, orc):
    """Model points far from every scene point (their fp32 row mass
    underflows): the group-wide flagged count turns on the conditional
    fallback exchange; the rows must match the single-GPU exact fallback and
    the dense oracle."""
    x = orc.make_torus(300, 81)
    far = np.full((12, 3), 4.0) + orc.make_cloud(12, 3, 82) * 0.05
    xm = np.vstack([x, far])
    y = orc.make_torus(330, 83) * 1.03
    cfg = fc.RegistrationConfig(omega=0.0, beta=2.0, lambda_reg=3.0, iterations=40)
    with fc.Context(0) as one:
        ref = one.register(xm, y, cfg)
    with fc.Context.loopback(0, 3) as grp:
        got = grp.register(xm, y, cfg)
    orc_ref = orc.register(xm, y, omega=0.0, beta=2.0, lambda_reg=3.0, iterations=40)
    rel = np.abs(got.sigma2_trace / ref.sigma2_trace - 1).max()
    rel_o = np.abs(got.sigma2_trace / orc_ref.sigma2_trace - 1).max()
    pts = np.abs(got.transformed - orc_ref.transformed).max() / bbox_diag(y)
    print(f"σ² vs single {rel:.3g}, vs oracle {rel_o:.3g}; points {pts:.3g}; "
          f"final σ² {got.sigma2_trace[-1]:.3g}")
    assert rel <= 1e-6 and rel_o <= 1e-5 and pts <= 1e-4


def test_loopback_matches_oracle(fc, orc):
    x = orc.make_torus(400, 91)
    y = orc.make_torus(440, 92) * np.array([1.1, 0.9, 1.0]) + 0.05
    cfg = fc.RegistrationConfig(omega=0.3, iterations=40, variant="fast_lowrank",
                                rank_fraction=0.2)
    with fc.Context.loopback(0, 4) as grp:
        got = grp.register(x, y, cfg)
    ref = orc.register(x, y, omega=0.3, iterations=40, variant="fast_lowrank",
                       rank_fraction=0.2)
    rel = np.abs(got.sigma2_trace / ref.sigma2_trace - 1).max()
    assert rel <= 1e-5, rel
    assert np.abs(got.transformed - ref.transformed).max() <= 1e-4 * bbox_diag(y)
