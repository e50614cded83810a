"""ctypes wrapper for the CPU parity oracle (``oracle/fcpd_oracle.cpp``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and the CPU legs of ``bench.py``.  The product never imports this module.

Point sets are ``(count, dim)`` float64 arrays; they are passed to C in
column-major (Fortran) order, matching ``Eigen::MatrixXd`` in the reference
(``proj/include/fastcpd/pointset.hpp:19-27``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libfcpd_oracle.so")

_P = C.POINTER(C.c_double)
_I64 = C.c_int64


class OracleError(RuntimeError):
    """Raised with the reference's error category (errors.hpp:8-34)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = {1: "ParameterError", 2: "DimensionError", 3: "NumericError",
                     4: "IoError", 5: "ParseError"}.get(code, "Error")


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_get_threads.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(_P) if a is not None else None


def _col(a, dim=None) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1 if dim is None else dim)
    return np.asfortranarray(a)


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def set_threads(n: int):
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return lib().orc_get_threads()


# ---------------------------------------------------------------- functions


def normalize_pair(x, y):
    x, y = _col(x), _col(y)
    if x.shape[1] != y.shape[1]:
        raise OracleError(2, "normalize_pair: dimension mismatch")
    m, d = x.shape
    n = y.shape[0]
    xo = np.zeros((m, d), order="F")
    yo = np.zeros((n, d), order="F")
    center = np.zeros(d)
    scale = C.c_double()
    deg = C.c_int()
    _check(lib().orc_normalize_pair(_ptr(x), _I64(m), _ptr(y), _I64(n), d, _ptr(xo),
                                    _ptr(yo), _ptr(center), C.byref(scale), C.byref(deg)))
    return xo, yo, center, scale.value, bool(deg.value)


def init_sigma2(x, y) -> float:
    x, y = _col(x), _col(y)
    if x.shape[1] != y.shape[1]:
        raise OracleError(2, "init_sigma2: dimension mismatch")
    out = C.c_double()
    _check(lib().orc_init_sigma2(_ptr(x), _I64(x.shape[0]), _ptr(y), _I64(y.shape[0]),
                                 x.shape[1], C.byref(out)))
    return out.value


def build_gram(x, beta: float) -> np.ndarray:
    x = _col(x)
    m, d = x.shape
    phi = np.zeros((m, m), order="F")
    _check(lib().orc_build_gram(_ptr(x), _I64(m), d, C.c_double(beta), _ptr(phi)))
    return phi


def eigendecompose(phi, rank: int):
    phi = np.asfortranarray(phi, dtype=np.float64)
    m = phi.shape[0]
    if rank < 1 or rank > m:
        raise OracleError(1, "eigendecompose: rank out of [1, M]")
    u = np.zeros((m, rank), order="F")
    lam = np.zeros(rank)
    raw = np.zeros(rank)
    _check(lib().orc_eigendecompose(_ptr(phi), _I64(m), _I64(rank), _ptr(u), _ptr(lam),
                                    _ptr(raw)))
    return u, lam, raw


def posterior(xt, y, omega: float, sigma2: float):
    xt, y = _col(xt), _col(y)
    if xt.shape[1] != y.shape[1]:
        raise OracleError(2, "posterior: dimension mismatch")
    m, d = xt.shape
    n = y.shape[0]
    p = np.zeros((m, n), order="F")
    clamped = C.c_int()
    _check(lib().orc_posterior(_ptr(xt), _I64(m), _ptr(y), _I64(n), d, C.c_double(omega),
                               C.c_double(sigma2), _ptr(p), C.byref(clamped)))
    return p, bool(clamped.value)


def enforce_row_constraint(p):
    p = np.array(p, dtype=np.float64, order="F", copy=True)
    m, n = p.shape
    rows = np.zeros(m, dtype=np.int64)
    nd = C.c_int64()
    _check(lib().orc_enforce_row_constraint(_ptr(p), _I64(m), _I64(n),
                                            rows.ctypes.data_as(C.POINTER(C.c_int64)),
                                            C.byref(nd)))
    return p, rows[: nd.value].tolist()


def estimated_targets(p, y):
    p = np.asfortranarray(p, dtype=np.float64)
    y = _col(y)
    m, n = p.shape
    out = np.zeros((m, y.shape[1]), order="F")
    _check(lib().orc_estimated_targets(_ptr(p), _I64(m), _I64(n), _ptr(y), _I64(y.shape[0]),
                                       y.shape[1], _ptr(out)))
    return out


def solve_fast_lowrank(u, lam, lambda_reg, sigma2, residual):
    u = np.asfortranarray(u, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    r = _col(residual)
    m, k = u.shape
    w = np.zeros(r.shape, order="F")
    _check(lib().orc_solve_fast_lowrank(_ptr(u), _ptr(lam), _I64(m), _I64(k),
                                        C.c_double(lambda_reg), C.c_double(sigma2), _ptr(r),
                                        _I64(r.shape[0]), r.shape[1], _ptr(w)))
    return w


def solve_fast(u, lam, lambda_reg, sigma2, residual):
    u = np.asarray(u)
    if u.shape[0] != u.shape[1]:
        raise OracleError(1, "solve_fast expects the full spectral basis")
    return solve_fast_lowrank(u, lam, lambda_reg, sigma2, residual)


def apply_transform(x, phi, w):
    x, w = _col(x), _col(w)
    phi = np.asfortranarray(phi, dtype=np.float64)
    out = np.zeros(x.shape, order="F")
    _check(lib().orc_apply_transform(_ptr(x), _I64(x.shape[0]), x.shape[1], _ptr(phi),
                                     _ptr(w), _ptr(out)))
    return out


def apply_transform_lowrank(x, u, lam, w):
    x, w = _col(x), _col(w)
    u = np.asfortranarray(u, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    out = np.zeros(x.shape, order="F")
    _check(lib().orc_apply_transform_lowrank(_ptr(x), _I64(x.shape[0]), x.shape[1], _ptr(u),
                                             _ptr(lam), _I64(u.shape[1]), _ptr(w), _ptr(out)))
    return out


def update_sigma2(y, p, xt, row_constrained=True) -> float:
    y, xt = _col(y), _col(xt)
    p = np.asfortranarray(p, dtype=np.float64)
    out = C.c_double()
    _check(lib().orc_update_sigma2(_ptr(y), _I64(y.shape[0]), _ptr(p), _I64(p.shape[0]),
                                   _ptr(xt), xt.shape[1], int(bool(row_constrained)),
                                   C.byref(out)))
    return out.value


def solve_cpd_baseline(phi, p, lambda_reg, sigma2, y, x):
    phi = np.asfortranarray(phi, dtype=np.float64)
    p = np.asfortranarray(p, dtype=np.float64)
    y, x = _col(y), _col(x)
    w = np.zeros(x.shape, order="F")
    _check(lib().orc_solve_cpd_baseline(_ptr(phi), _I64(phi.shape[0]), _ptr(p),
                                        _I64(p.shape[1]), C.c_double(lambda_reg),
                                        C.c_double(sigma2), _ptr(y), _ptr(x), x.shape[1],
                                        _ptr(w)))
    return w


@dataclass
class EStep:
    ptilde_y: np.ndarray
    p1: np.ndarray
    var: np.ndarray
    degenerate: np.ndarray
    pt1: np.ndarray
    clamped: bool


def estep_stream(xt, y, omega, sigma2) -> EStep:
    xt, y = _col(xt), _col(y)
    m, d = xt.shape
    n = y.shape[0]
    pty = np.zeros((m, d), order="F")
    p1 = np.zeros(m)
    var = np.zeros(m)
    deg = np.zeros(m, dtype=np.int32)
    pt1 = np.zeros(n)
    cl = C.c_int()
    _check(lib().orc_estep_stream(_ptr(xt), _I64(m), _ptr(y), _I64(n), d, C.c_double(omega),
                                  C.c_double(sigma2), _ptr(pty), _ptr(p1), _ptr(var),
                                  deg.ctypes.data_as(C.POINTER(C.c_int32)), _ptr(pt1),
                                  C.byref(cl)))
    return EStep(pty, p1, var, deg.astype(bool), pt1, bool(cl.value))


@dataclass
class Result:
    transformed: np.ndarray
    coefficients: np.ndarray
    sigma2_trace: np.ndarray
    sigma2_initial: float
    timing: dict = field(default_factory=dict)
    degenerate_rows: int = 0
    sigma2_clamps: int = 0


VARIANTS = {"cpd": 0, "cpd_lowrank": 1, "fast": 2, "fast_lowrank": 3}


def register(x, y, *, omega=0.7, beta=2.0, lambda_reg=10.0, iterations=100,
             variant="fast", rank_fraction=0.1, normalize=True, early_stop=False,
             basis=None) -> Result:
    """registration.hpp:79-175 restated (fast / fast_lowrank)."""
    x, y = _col(x), _col(y)
    if x.shape[1] != y.shape[1]:
        raise OracleError(2, "register: model and scene dimension mismatch")
    m, d = x.shape
    n = y.shape[0]
    out_x = np.zeros((m, d), order="F")
    out_w = np.zeros((m, d), order="F")
    trace = np.zeros(max(iterations, 1))
    it = C.c_int()
    s0 = C.c_double()
    timing = np.zeros(7)
    diag = np.zeros(2, dtype=np.int64)
    bu = bl = None
    brank = 0
    if basis is not None:
        bu = np.asfortranarray(basis[0], dtype=np.float64)
        bl = np.ascontiguousarray(basis[1], dtype=np.float64)
        brank = bu.shape[1]
    _check(lib().orc_register(_ptr(x), _I64(m), _ptr(y), _I64(n), d, C.c_double(omega),
                              C.c_double(beta), C.c_double(lambda_reg), int(iterations),
                              VARIANTS[variant], C.c_double(rank_fraction), int(normalize),
                              int(early_stop), _ptr(bu), _ptr(bl), _I64(brank), _ptr(out_x),
                              _ptr(out_w), _ptr(trace), C.byref(it), C.byref(s0),
                              _ptr(timing), diag.ctypes.data_as(C.POINTER(C.c_int64))))
    keys = ["t_c", "t_eig", "t_iter", "t_f", "t_o", "t_total", "t_loop"]
    return Result(np.ascontiguousarray(out_x), np.ascontiguousarray(out_w),
                  trace[: it.value].copy(), s0.value, dict(zip(keys, timing.tolist())),
                  int(diag[0]), int(diag[1]))


# ------------------------------------------- reference test fixtures (test_util.hpp)


def make_cloud(m: int, d: int, seed: int) -> np.ndarray:
    out = np.zeros((m, d), order="F")
    lib().orc_make_cloud(_I64(m), d, C.c_uint64(seed), _ptr(out))
    return np.ascontiguousarray(out)


def make_torus(m: int, seed: int) -> np.ndarray:
    out = np.zeros((m, 3), order="F")
    lib().orc_make_torus(_I64(m), C.c_uint64(seed), _ptr(out))
    return np.ascontiguousarray(out)


def random_row_constrained(m: int, n: int, seed: int) -> np.ndarray:
    p = np.zeros((m, n), order="F")
    lib().orc_random_row_constrained(_I64(m), _I64(n), C.c_uint64(seed), _ptr(p))
    return p


# ------------------------------------------- spectral cache + streaming register


def save_spectral_cache(path: str, u, lam, beta: float):
    """kernel.hpp:92-110."""
    u = np.asfortranarray(u, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    _check(lib().orc_save_spectral_cache(path.encode(), _ptr(u), _ptr(lam), _I64(u.shape[0]),
                                         _I64(u.shape[1]), C.c_double(beta)))


def load_spectral_cache(path: str):
    """kernel.hpp:112-144 → (u (M×K), lambda (K), beta)."""
    m, k, beta = C.c_int64(), C.c_int64(), C.c_double()
    _check(lib().orc_load_spectral_cache(path.encode(), C.byref(m), C.byref(k), C.byref(beta),
                                         None, None))
    u = np.zeros((m.value, k.value), order="F")
    lam = np.zeros(k.value)
    _check(lib().orc_load_spectral_cache(path.encode(), C.byref(m), C.byref(k), C.byref(beta),
                                         _ptr(u), _ptr(lam)))
    return u, lam, beta.value


def register_stream(x, y, u, lam, lam_num=None, *, omega, lambda_reg, iterations,
                    normalize=True, xt_start=None, sigma2_start=None) -> Result:
    """Streaming-E-step restatement of register_pointsets with a given basis
    (configs 2–4: no M×N matrix).  ``xt_start``/``sigma2_start`` resume the
    EM from a given state (x̃ in the loop's frame, σ²): a window of late
    iterations is then checked without replaying the whole run."""
    x, y = _col(x), _col(y)
    u = np.asfortranarray(u, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    lam_num = lam if lam_num is None else np.ascontiguousarray(lam_num, dtype=np.float64)
    m, d = x.shape
    xs = None if xt_start is None else _col(xt_start)
    out_x = np.zeros((m, d), order="F")
    trace = np.zeros(max(iterations, 1))
    it = C.c_int()
    s0 = C.c_double()
    _check(lib().orc_register_stream(_ptr(x), _I64(m), _ptr(y), _I64(y.shape[0]), d,
                                     C.c_double(omega), C.c_double(lambda_reg), int(iterations),
                                     int(normalize), _ptr(u), _ptr(lam), _ptr(lam_num),
                                     _I64(u.shape[1]), _ptr(xs),
                                     C.c_double(sigma2_start or 0.0), _ptr(out_x), _ptr(trace),
                                     C.byref(it), C.byref(s0)))
    return Result(np.ascontiguousarray(out_x), np.zeros_like(out_x), trace[: it.value].copy(),
                  s0.value)


# ------------------------------------------- top-K basis without forming Φ


def gram_rows(x, beta: float, rows) -> np.ndarray:
    """Rows ``rows`` of Φ (kernel.hpp:31-47) as a len(rows) × M array."""
    x = _col(x)
    m, d = x.shape
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((len(rows), m), order="F")
    _check(lib().orc_gram_rows(_ptr(x), _I64(m), d, C.c_double(beta),
                               rows.ctypes.data_as(C.POINTER(C.c_int64)), _I64(len(rows)),
                               _ptr(out)))
    return out


def gram_apply(x, beta: float, v, rows=None, block: int = 2048) -> np.ndarray:
    """Φ[rows]·V in fp64 without forming Φ (row blocks of Φ from the C
    restatement, times V through BLAS)."""
    m = np.asarray(x).shape[0]
    rows = np.arange(m) if rows is None else np.asarray(rows, dtype=np.int64)
    v = np.asarray(v, dtype=np.float64)
    out = np.empty((len(rows), v.shape[1]))
    for s in range(0, len(rows), block):
        out[s:s + block] = gram_rows(x, beta, rows[s:s + block]) @ v
    return out


def topk_basis(x, beta: float, rank: int, *, power_iters: int = 4, oversample=None,
               seed: int = 1234):
    """Top-``rank`` eigenpairs of Φ (kernel.hpp:49-72 semantics: descending,
    λ < 1e-12·λmax clamped to 0) by randomized block subspace iteration in
    fp64 — an implementation independent of the device's (different start,
    numpy QR / eigh, CPU Φ·V).  Returns (U, λ clamped, λ raw, residuals),
    residuals[i] = ‖Φu_i − λ_i u_i‖ / λ_1."""
    m = np.asarray(x).shape[0]
    p = max(16, rank // 5) if oversample is None else oversample
    b = min(m, rank + p)
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(gram_apply(x, beta, rng.standard_normal((m, b))))
    for _ in range(power_iters):
        q, _ = np.linalg.qr(gram_apply(x, beta, q))
    z = gram_apply(x, beta, q)
    bm = q.T @ z
    theta, s = np.linalg.eigh(0.5 * (bm + bm.T))
    order = np.argsort(theta)[::-1][:rank]
    theta, s = theta[order], s[:, order]
    u = q @ s
    res = np.linalg.norm(z @ s - u * theta, axis=0) / max(theta[0], 1e-300)
    lam_raw = theta.copy()
    lam = theta.copy()
    lam[lam < 1e-12 * max(lam[0], 0.0)] = 0.0  # kernel.hpp:68-70
    return np.asfortranarray(u), lam, lam_raw, res


def eigen_residuals(x, beta: float, u, lam, rows) -> np.ndarray:
    """max over the sampled model rows of |(Φu_i)_r − λ_i u_ir| / λ_1 per
    eigenpair: an independent fp64 check of a device basis at full size."""
    u = np.asarray(u, dtype=np.float64)
    rows = np.asarray(rows, dtype=np.int64)
    pu = gram_apply(x, beta, u, rows=rows)
    return np.abs(pu - u[rows] * np.asarray(lam)[None, :]).max(axis=0) / max(lam[0], 1e-300)
