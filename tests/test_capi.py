"""CPU-only checks of the C ABI boundary: the library loads without a GPU
and exports every symbol include/fcpd_capi.h declares; host-side helpers
mirror the reference (solvers.hpp:20-54)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fcpd_capi.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FCPD_API\s+[\w\s\*]+?\b(fcpd_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def built():
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2006_06281_b200")],
                   check=True)
    import paper_2006_06281_b200 as f
    return f


def test_header_declares_boundary():
    syms = declared_symbols()
    for s in ("fcpd_register", "fcpd_estep", "fcpd_build_basis", "fcpd_solve_fast_lowrank",
              "fcpd_session_begin", "fcpd_last_error", "fcpd_create", "fcpd_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(built):
    lib = ctypes.CDLL(built.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", built.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (fcpd_\w+)", out))
    assert exported == set(declared_symbols())


def test_library_is_sm100a(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_config_defaults_match_reference(built):
    # registration.hpp:30-40
    c = built._Config()
    built.lib().fcpd_config_default(ctypes.byref(c))
    assert (c.omega, c.beta, c.lambda_reg, c.iterations, c.variant, c.rank_fraction,
            c.normalize, c.early_stop) == (0.7, 2.0, 10.0, 100, 2, 0.1, 1, 0)
    py = built.RegistrationConfig()
    assert (py.omega, py.beta, py.lambda_reg, py.iterations, py.variant) == \
        (0.7, 2.0, 10.0, 100, "fast")


def test_variant_and_rank_helpers(built):
    assert built.variant_from_string("fast-lowrank") == "fast_lowrank"
    with pytest.raises(built.ParameterError):
        built.variant_from_string("nope")
    assert built.lowrank_rank(0.004, 50000) == 200
    assert built.lowrank_rank(0.0015, 200000) == 300
    assert built.lowrank_rank(1e-9, 10) == 1
    with pytest.raises(built.ParameterError):
        built.lowrank_rank(0.0, 10)


def test_no_gpu_fails_loudly(built):
    """Without a GPU the product raises instead of silently computing on CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(built.Error):
        built.Context(0)
