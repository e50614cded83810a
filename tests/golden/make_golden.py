"""Write the committed golden fixtures of tests/golden/ (test infrastructure).

The reference cannot be built or imported here (Eigen3 and its vendored
test framework are absent), so there are no reference-produced
output files.  The fixtures are therefore of two kinds:

* ``reference_kats.json`` — the known answers the reference's own tests
  hold for this path (scalars and tolerances, each with its test file:line).
  ``tests/test_golden.py`` checks the oracle against them.
* ``*.npz`` — fp64 registration trajectories of the CPU oracle
  (oracle/fcpd_oracle.cpp, itself pinned by those KATs) on seeded inputs:
  σ² per iteration and the final transformed points.  The GPU tests compare
  the CUDA path against these files without running the oracle, and the CPU
  suite checks that the oracle still reproduces them bit for bit.

Regenerate (deterministic): python tests/golden/make_golden.py
"""
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

# Inputs of each trajectory fixture: (name, generator, registration arguments).
# Generators are the oracle's restatements of test_util.hpp (mt19937_64) or
# the seeded BASELINE generator (paper_2006_06281_b200/datagen.py).
TRAJECTORIES = {
    "torus_fast_w0.2": dict(gen="torus", m=400, n=430, seed_x=11, seed_y=12, scale=1.05,
                            shift=0.03, omega=0.2, beta=2.0, lambda_reg=3.0, iterations=30,
                            variant="fast", rank_fraction=1.0),
    "torus_lowrank_w0.5": dict(gen="torus", m=300, n=300, seed_x=21, seed_y=22, scale=0.97,
                               shift=-0.02, omega=0.5, beta=1.5, lambda_reg=2.0, iterations=30,
                               variant="fast_lowrank", rank_fraction=0.2),
    "c0_50it": dict(gen="c0", omega=0.0, beta=2.0, lambda_reg=3.0, iterations=50,
                    variant="fast", rank_fraction=1.0),
}

# Known answers held by the reference's tests (proj/tests/*.cpp).
REFERENCE_KATS = [
    {"name": "posterior_scalar_with_outlier", "site": "test_correspondence.cpp:26-35",
     "inputs": {"x": [[0.0]], "y": [[1.0]], "omega": 0.5, "sigma2": 1.0},
     "value": math.exp(-0.5) / (math.exp(-0.5) + math.sqrt(2 * math.pi)), "rtol": 1e-12},
    {"name": "posterior_equidistant", "site": "test_correspondence.cpp:18-24",
     "inputs": {"x": [[-1.0, 0.0], [1.0, 0.0]], "y": [[0.0, 0.3]], "omega": 0.0,
                "sigma2": 0.25},
     "value": [0.5, 0.5], "rtol": 1.19e-5},
    {"name": "row_constraint", "site": "test_correspondence.cpp:85-106",
     "inputs": {"p": [[0.2, 0.2], [0.0, 0.5]]}, "value": [[0.5, 0.5], [0.0, 1.0]],
     "rtol": 1.19e-5},
    {"name": "solve_fast_scalar", "site": "test_solvers.cpp:35-49",
     "inputs": {"u": [[1.0]], "lam": [1.0], "lambda_reg": 2.0, "sigma2": 0.25,
                "residual": [[0.8]]},
     "value": 0.8 / 1.5, "rtol": 1e-12},
    {"name": "gram_scalar", "site": "test_kernel.cpp:11-26",
     "inputs": {"x": [[0.0], [2.0]], "beta": 2.0}, "value": math.exp(-4.0 / 8.0),
     "rtol": 1e-14},
    {"name": "eigen_duplicates", "site": "test_kernel.cpp:40-59",
     "inputs": {"x": [[1.0, 1.0], [1.0, 1.0]], "beta": 2.0}, "value": [2.0, 0.0],
     "atol": 1e-12},
    {"name": "init_sigma2_scalar", "site": "test_registration.cpp:13-27",
     "inputs": {"x": [[0.0]], "y": [[2.0]]}, "value": 4.0, "rtol": 1e-14},
]


def trajectory_inputs(spec):
    from oracle import oracle as orc
    if spec["gen"] == "torus":
        x = orc.make_torus(spec["m"], spec["seed_x"])
        y = orc.make_torus(spec["n"], spec["seed_y"]) * spec["scale"] + spec["shift"]
        return x, y
    from paper_2006_06281_b200 import datagen
    x, y, _ = datagen.generate(spec["gen"])
    return x, y


def main():
    from oracle import oracle as orc
    with open(os.path.join(HERE, "reference_kats.json"), "w") as f:
        json.dump(REFERENCE_KATS, f, indent=1)
    for name, spec in TRAJECTORIES.items():
        x, y = trajectory_inputs(spec)
        r = orc.register(x, y, omega=spec["omega"], beta=spec["beta"],
                         lambda_reg=spec["lambda_reg"], iterations=spec["iterations"],
                         variant=spec["variant"], rank_fraction=spec["rank_fraction"])
        np.savez_compressed(os.path.join(HERE, name + ".npz"), sigma2_trace=r.sigma2_trace,
                            transformed=r.transformed, spec=json.dumps(spec))
        print(name, "σ² final", r.sigma2_trace[-1])


if __name__ == "__main__":
    main()
