"""Seeded synthetic stand-ins for the BASELINE.json workloads (C0–C4).

The paper's datasets (TOSCA wolf, Stanford bunny) are not available; the
configs in BASELINE.json define synthetic generators instead.  Ambiguities are
pinned as SURVEY.md Appendix B recommends:

* "normalised to zero mean and unit variance" — per set: subtract the
  centroid, divide by the isotropic RMS sqrt(Σ var_axis / D).  The
  reference's own ``normalize_pair`` (joint centroid, max-abs scale) still
  runs inside ``register_pointsets``.
* GRBF warps use the reference's convention exp(−‖x−c‖²/(2w²))
  (degradations.hpp:126) with the stated width w.
* outliers are uniform in the scene's bounding box padded 5 % per side
  (add_outliers, degradations.hpp:51-55), appended, then the scene is
  permuted.
* C3's warp parameters are C0's (50 centres, N(0, 0.1²), width 0.5); C4
  uses C2's generator and C2's ω/β/λ, 100 iterations.
* RNG: numpy PCG64, seed 0 per config, streams split with SeedSequence.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    m: int
    n: int
    omega: float
    beta: float
    lambda_reg: float
    iterations: int
    variant: str
    rank_fraction: float
    description: str


WORKLOADS = {
    "c0": Workload("c0", 2000, 2000, 0.0, 2.0, 3.0, 50, "fast", 1.0,
                   "full-rank, cube + 50-centre GRBF warp, M=N=2000"),
    "c1": Workload("c1", 20000, 24000, 0.2, 2.0, 3.0, 100, "fast", 1.0,
                   "full-rank, cube + GRBF warp + 20% outliers, M=20000 N=24000"),
    "c2": Workload("c2", 50000, 50000, 0.1, 1.0, 2.0, 100, "fast_lowrank", 200 / 50000,
                   "low-rank K=200, bumpy sphere + GRBF warp, M=N=50000"),
    "c3": Workload("c3", 100000, 150000, 0.3, 2.0, 3.0, 100, "fast_lowrank", 500 / 100000,
                   "low-rank K=500, cube + warped resample + 50k outliers"),
    "c4": Workload("c4", 200000, 200000, 0.1, 1.0, 2.0, 100, "fast_lowrank", 300 / 200000,
                   "low-rank K=300, bumpy sphere, M=N=200000"),
}


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, stream])))


def grbf_warp(pts: np.ndarray, centres: np.ndarray, coeff: np.ndarray, width: float,
              chunk: int = 65536) -> np.ndarray:
    out = np.empty_like(pts)
    inv = 1.0 / (2.0 * width * width)
    for s in range(0, len(pts), chunk):
        p = pts[s:s + chunk]
        d2 = ((p[:, None, :] - centres[None, :, :]) ** 2).sum(-1)
        out[s:s + chunk] = p + np.exp(-d2 * inv) @ coeff
    return out


def standardise(p: np.ndarray) -> np.ndarray:
    c = p - p.mean(0)
    return c / np.sqrt((c ** 2).mean(0).sum() / p.shape[1])


def add_outliers(y: np.ndarray, count: int, rng: np.random.Generator) -> np.ndarray:
    lo, hi = y.min(0), y.max(0)
    pad = (hi - lo) * 0.05
    lo, hi = lo - pad, hi + pad
    extra = lo + rng.random((count, y.shape[1])) * (hi - lo)
    return np.vstack([y, extra])


def bumpy_sphere(m: int, rng: np.random.Generator) -> np.ndarray:
    v = rng.standard_normal((m, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    theta = np.arccos(np.clip(v[:, 2], -1, 1))
    phi = np.arctan2(v[:, 1], v[:, 0])
    r = 1.0 + 0.1 * np.sin(5 * theta) * np.cos(3 * phi)
    return v * r[:, None]


def generate(name: str, seed: int = 0, m: int | None = None, n_scale: float | None = None):
    """Return (X, Y, Workload) as (M,3)/(N,3) float64 arrays.

    ``m`` overrides the model size (tests use reduced sizes of the same
    generator); the scene keeps the config's N/M ratio.
    """
    w = WORKLOADS[name]
    mm = w.m if m is None else int(m)
    ratio = w.n / w.m
    if name in ("c0", "c1"):
        r = _rng(seed, 1)
        x = r.uniform(-1.0, 1.0, (mm, 3))
        centres = r.uniform(-1.0, 1.0, (50, 3))
        coeff = r.normal(0.0, 0.1, (50, 3))
        y = grbf_warp(x, centres, coeff, 0.5) + r.normal(0.0, 0.01, (mm, 3))
        y = y[r.permutation(mm)]
        x, y = standardise(x), standardise(y)
        if name == "c1":
            y = add_outliers(y, int(round(mm * (ratio - 1.0))), r)
            y = y[r.permutation(len(y))]
    elif name in ("c2", "c4"):
        r = _rng(seed, 2 if name == "c2" else 4)
        x = bumpy_sphere(mm, r)
        centres = x[r.integers(0, mm, 100)]
        coeff = r.normal(0.0, 0.05, (100, 3))
        y = grbf_warp(x, centres, coeff, 0.3) + r.normal(0.0, 0.005, (mm, 3))
        y = y[r.permutation(mm)]
    elif name == "c3":
        r = _rng(seed, 3)
        x = r.uniform(0.0, 1.0, (mm, 3))
        res = r.uniform(0.0, 1.0, (mm, 3))
        centres = r.uniform(0.0, 1.0, (50, 3))
        coeff = r.normal(0.0, 0.1, (50, 3))
        y = grbf_warp(res, centres, coeff, 0.5)
        y = add_outliers(y, int(round(mm * (ratio - 1.0))), r)
        y = y[r.permutation(len(y))]
    else:
        raise KeyError(name)
    return np.ascontiguousarray(x), np.ascontiguousarray(y), w


def config_for(w: Workload, iterations: int | None = None):
    from . import RegistrationConfig
    return RegistrationConfig(omega=w.omega, beta=w.beta, lambda_reg=w.lambda_reg,
                              iterations=w.iterations if iterations is None else iterations,
                              variant=w.variant, rank_fraction=w.rank_fraction)
