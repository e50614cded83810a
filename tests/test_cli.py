"""Point-file I/O, the run report and the `fcpd register` CLI (SURVEY §8f
rank 3; reference: pointset.hpp:45-119, registration.hpp:178-204,
tools/fcpd.cpp:56-83, tests/test_pointset.cpp, tests/test_cli.cpp)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2006_06281_b200")
LIBDIR = os.path.join(PKG, "lib")
CLI = os.path.join(PKG, "bin", "fcpd")


def build():
    subprocess.run(["make", "-s", "-j8", "-C", PKG], check=True)
    return CLI


def _run_host_cpp(tmp_path, name):
    build()
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    exe = str(tmp_path / name)
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I",
                    os.path.join(ROOT, "include"), src, "-L", LIBDIR, "-lfcpd_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=60)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL:" not in r.stdout


def test_pointio_and_report_match_reference_tests(tmp_path):
    """tests/test_pointset.cpp restated against the drop-in header (host only)."""
    _run_host_cpp(tmp_path, "test_pointio")


def test_bench_harness_helpers(tmp_path):
    """tests/test_metrics.cpp host cases: rmse, subsample, random_affine,
    make_bench_pair and the byte-stable bench CSV (host only)."""
    _run_host_cpp(tmp_path, "test_metrics")


def test_cli_usage_and_errors(tmp_path):
    exe = build()
    r = subprocess.run([exe, "--help"], capture_output=True, text=True)
    assert r.returncode == 0 and "register MODEL SCENE" in r.stdout
    r = subprocess.run([exe, "degrade", "x"], capture_output=True, text=True)
    assert r.returncode == 2
    r = subprocess.run([exe, "bench", "--sizes", "40"], capture_output=True, text=True)
    assert r.returncode != 0 and "--synthetic" in r.stderr
    r = subprocess.run([exe, "bench", "--synthetic", "--sizes", "40", "--frobnicate"],
                       capture_output=True, text=True)
    assert r.returncode != 0 and "unknown option" in r.stderr
    # a missing scene file is reported by name before any device work
    model = tmp_path / "model_only.txt"
    np.savetxt(model, np.random.default_rng(201).uniform(-1, 1, (10, 2)))
    r = subprocess.run([exe, "register", str(model), str(tmp_path / "no_such_scene.txt")],
                       capture_output=True, text=True)
    assert r.returncode != 0 and "no_such_scene.txt" in r.stderr
    r = subprocess.run([exe, "register", str(model), str(model), "--variant", "bogus"],
                       capture_output=True, text=True)
    assert r.returncode != 0 and "unknown solver variant" in r.stderr


def test_cli_plot_from_bench_csv(tmp_path):
    """tests/test_cli.cpp:118-126: `plot` renders a bench CSV as a
    deterministic SVG and rejects a file that is not a bench CSV (host only)."""
    exe = build()
    csv = tmp_path / "bench.csv"
    rows = ["M,N,variant,t_c,t_eig,t_iter,t_f,t_o,t_total,rmse,iterations"]
    for m, v, ti in [(40, "fast", 0.01), (60, "fast", 0.02), (40, "fast_lowrank", 0.012),
                     (60, "fast_lowrank", 0.03), (40, "cpd", 0.0)]:
        err = -1.0 if v == "cpd" else 1e-4
        rows.append(f"{m},{m},{v},0.001000,0.002000,{ti:.6f},{0.002 + ti:.6f},0.000100,"
                    f"{0.0031 + ti:.6f},{err},2")
    csv.write_text("\n".join(rows) + "\n")
    outs = []
    for k in range(2):
        svg = tmp_path / f"plot{k}.svg"
        r = subprocess.run([exe, "plot", str(csv), "--out", str(svg)], capture_output=True,
                           text=True, timeout=60)
        assert r.returncode == 0, r.stderr
        outs.append(svg.read_text())
    assert outs[0] == outs[1] and outs[0].count('<path d="M ') == 2
    bad = tmp_path / "bad.csv"
    bad.write_text("1 2 3\n")
    r = subprocess.run([exe, "plot", str(bad)], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0


@pytest.mark.gpu
def test_cli_register_on_gpu(tmp_path, orc):
    """tests/test_cli.cpp:39-63: register an identical torus pair, 20
    iterations; the report's final σ² does not exceed the initial one and the
    output equals the library call with the same configuration."""
    import paper_2006_06281_b200 as fc

    exe = build()
    cloud = orc.make_torus(80, 200)
    pts = tmp_path / "cloud.txt"
    np.savetxt(pts, cloud, fmt="%.17g")
    out, rep, svg = tmp_path / "reg_out.txt", tmp_path / "reg_report.txt", tmp_path / "reg.svg"
    r = subprocess.run([exe, "register", str(pts), str(pts), "--iters", "20", "--out", str(out),
                        "--report", str(rep), "--svg", str(svg)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert out.exists() and svg.exists()
    kv = dict(line.split("=", 1) for line in rep.read_text().splitlines())
    initial, final = float(kv["sigma2_initial"]), float(kv["sigma2[19]"])
    assert 0.0 <= final <= initial
    assert kv["variant"] == "fast" and kv["iterations"] == "20"
    got = np.loadtxt(out)
    ref = fc.register_pointsets(cloud, cloud, fc.RegistrationConfig(iterations=20))
    assert np.abs(got - ref.transformed).max() <= 1e-12


@pytest.mark.gpu
def test_cli_bench_on_gpu(tmp_path):
    """tests/test_cli.cpp:108-116 and test_metrics.cpp:66-82: a synthetic
    sweep over two sizes × two variants writes four CSV records in the
    reference schema; every cell converges (rmse ≥ 0, small), the timing
    identities hold in the file and the dense `cpd` variant, which the device
    path does not provide, is recorded as a failed cell rather than aborting."""
    exe = build()
    csv = tmp_path / "bench.csv"
    svg = tmp_path / "bench.svg"
    r = subprocess.run([exe, "bench", "--synthetic", "--sizes", "40,60", "--variants",
                        "fast,fast-lowrank,cpd", "--iters", "30", "--csv", str(csv),
                        "--svg", str(svg)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert svg.read_text().count('<path d="M ') == 2  # cpd cells failed: no path
    lines = csv.read_text().splitlines()
    assert lines[0] == "M,N,variant,t_c,t_eig,t_iter,t_f,t_o,t_total,rmse,iterations"
    rows = [ln.split(",") for ln in lines[1:]]
    assert len(rows) == 6
    assert [int(x[0]) for x in rows] == [40, 40, 40, 60, 60, 60]
    for x in rows:
        tc, te, ti, tf, to, tt, err = (float(v) for v in x[3:10])
        assert abs(tf - (te + ti)) <= 1e-9 and abs(tt - (tc + tf + to)) <= 1e-9
        assert int(x[10]) == 30
        if x[2] == "cpd":
            assert err == -1.0
        else:
            assert 0.0 <= err < 0.2, x
