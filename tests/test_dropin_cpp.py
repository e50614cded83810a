"""The C++ drop-in header (include/fastcpd/fastcpd.hpp) compiles against the
reference-style test program and, on a B200, passes the reference's
registration tests (proj/tests/test_registration.cpp restated)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")
LIBDIR = os.path.join(ROOT, "paper_2006_06281_b200", "lib")


def build_dropin():
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2006_06281_b200")],
                   check=True)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    SRC, "-L", LIBDIR, "-lfcpd_b200", f"-Wl,-rpath,{LIBDIR}", "-o", OUT],
                   check=True)
    return OUT


def test_dropin_header_compiles_and_links():
    assert os.path.exists(build_dropin())


@pytest.mark.gpu
def test_dropin_reference_tests_pass_on_gpu():
    exe = build_dropin()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
