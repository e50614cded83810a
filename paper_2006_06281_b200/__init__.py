"""B200-native Fast Coherent Point Drift (arXiv 2006.06281).

Python mirror of the reference's registration API
(/root/reference/proj/include/fastcpd/registration.hpp:21-175) over the C ABI
of ``lib/libfcpd_b200.so`` (declared in ``include/fcpd_capi.h``).  Every call
runs on the GPU; there is no CPU fallback — importing this package on a
machine without the built library raises, and calling into it without a GPU
returns the CUDA error as :class:`Error`.

Point sets are ``(count, dim)`` float64 arrays (one point per row, as
``PointSet::pts``); they cross the ABI column-major, i.e. exactly the memory
layout of ``Eigen::MatrixXd``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "Error", "ParseError", "DimensionError", "ParameterError", "NumericError", "IoError",
    "RegistrationConfig", "RegistrationResult", "TimingBreakdown", "Context",
    "register_pointsets", "variant_from_string", "lowrank_rank", "LIB_PATH",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# FCPD_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("FCPD_LIB") or os.path.join(HERE, "lib", "libfcpd_b200.so")


# ------------------------------------------------------------- errors.hpp:8-34
class Error(RuntimeError):
    pass


class ParseError(Error):
    pass


class DimensionError(Error):
    pass


class ParameterError(Error):
    pass


class NumericError(Error):
    pass


class IoError(Error):
    pass


class CudaError(Error):
    pass


_CODES = {1: ParameterError, 2: DimensionError, 3: NumericError, 4: IoError, 5: ParseError,
          10: CudaError, 11: CudaError, 12: CudaError}

VARIANTS = {"cpd": 0, "cpd_lowrank": 1, "fast": 2, "fast_lowrank": 3}


def variant_from_string(s: str) -> str:  # solvers.hpp:20-36
    alias = {"cpd-lowrank": "cpd_lowrank", "fast-lowrank": "fast_lowrank"}
    s = alias.get(s, s)
    if s not in VARIANTS:
        raise ParameterError("unknown solver variant: " + s)
    return s


def lowrank_rank(rank_fraction: float, m: int) -> int:  # solvers.hpp:46-54
    if rank_fraction <= 0.0 or rank_fraction > 1.0:
        raise ParameterError("rank_fraction must lie in (0, 1]")
    return max(1, min(_llround(rank_fraction * m), m))


def cull_units_total(m: int, n: int) -> tuple[int, int]:
    """Work-list entries of one unculled E-step iteration, the unit of
    ``tiles_evaluated``: (256-point scene blocks × 32-point model sub-tiles,
    256-point model blocks × 32-point scene sub-tiles)."""
    return (-(-n // 256) * -(-m // 32), -(-m // 256) * -(-n // 32))


def _llround(v: float) -> int:
    return int(np.floor(v + 0.5)) if v >= 0 else -int(np.floor(-v + 0.5))


# ------------------------------------------------------------------ C structs
class _Config(C.Structure):
    _fields_ = [("omega", C.c_double), ("beta", C.c_double), ("lambda_reg", C.c_double),
                ("iterations", C.c_int32), ("variant", C.c_int32),
                ("rank_fraction", C.c_double), ("seed", C.c_uint64),
                ("normalize", C.c_int32), ("early_stop", C.c_int32), ("pad0", C.c_int32),
                ("spectral_tau", C.c_double)]


class _Timing(C.Structure):
    _fields_ = [(k, C.c_double) for k in
                ("t_c", "t_eig", "t_iter", "t_f", "t_o", "t_total", "t_setup")]


class _Result(C.Structure):
    _fields_ = [("transformed", C.POINTER(C.c_double)),
                ("coefficients", C.POINTER(C.c_double)),
                ("sigma2_trace", C.POINTER(C.c_double)),
                ("correspondence", C.POINTER(C.c_double)),
                ("degenerate_mask", C.POINTER(C.c_int32)),
                ("iterations_run", C.c_int32), ("basis_reused", C.c_int32),
                ("sigma2_initial", C.c_double), ("degenerate_rows", C.c_int64),
                ("sigma2_clamps", C.c_int64), ("timing", _Timing),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("tiles_evaluated", C.c_int64 * 2),
                ("spectral_rank", C.c_int64),
                ("mstep_fused", C.c_int32), ("reserved0", C.c_int32),
                ("pairs_by_form", C.c_int64 * 4)]


_lib = None


def lib():
    """Load the CUDA engine; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, I64, I32, D = C.POINTER(C.c_double), C.c_int64, C.c_int32, C.c_double
        PI32, PI64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
        vp = C.c_void_p
        sig = {
            "fcpd_config_default": (None, [C.POINTER(_Config)]),
            "fcpd_create": (C.c_int, [C.POINTER(vp), C.c_int]),
            "fcpd_destroy": (None, [vp]),
            "fcpd_last_error": (C.c_char_p, [vp]),
            "fcpd_version": (C.c_char_p, []),
            "fcpd_register": (C.c_int, [vp, P, I64, P, I64, I32, C.POINTER(_Config),
                                        C.POINTER(_Result)]),
            "fcpd_session_begin": (C.c_int, [vp, P, I64, P, I64, I32, C.POINTER(_Config)]),
            "fcpd_session_run": (C.c_int, [vp, I32]),
            "fcpd_session_sync": (C.c_int, [vp]),
            "fcpd_session_read": (C.c_int, [vp, C.POINTER(_Result)]),
            "fcpd_session_profile": (C.c_int, [vp, I32, P]),
            "fcpd_stream": (vp, [vp]),
            "fcpd_kernels_per_iteration": (I32, [vp]),
            "fcpd_estep": (C.c_int, [vp, P, I64, P, I64, I32, D, D, P, P, P, PI32, P, PI32]),
            "fcpd_posterior_dense": (C.c_int, [vp, P, I64, P, I64, I32, D, D, I32, P, PI32,
                                               PI64, PI64]),
            "fcpd_build_basis": (C.c_int, [vp, P, I64, I32, D, I64, P, P, P]),
            "fcpd_build_gram": (C.c_int, [vp, P, I64, I32, D, P]),
            "fcpd_build_basis_topk": (C.c_int, [vp, P, I64, I32, D, I64, I32, P, P, P]),
            "fcpd_save_spectral_cache": (C.c_int, [vp, C.c_char_p]),
            "fcpd_load_spectral_cache": (C.c_int, [vp, C.c_char_p, P, I64, P, I64, I32,
                                                   C.POINTER(_Config)]),
            "fcpd_nccl_unique_id": (C.c_int, [C.c_char_p]),
            "fcpd_create_dist": (C.c_int, [C.POINTER(vp), C.c_int, C.c_int, C.c_int,
                                           C.c_char_p]),
            "fcpd_world": (C.c_int, [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
            "fcpd_create_loopback": (C.c_int, [C.POINTER(vp), C.c_int, C.c_int]),
            "fcpd_solve_fast_lowrank": (C.c_int, [vp, P, P, I64, I64, D, D, P, I64, I32, P]),
            "fcpd_apply_transform_lowrank": (C.c_int, [vp, P, I64, I32, P, I64, P, I64, P, I64,
                                                       I32, P]),
            "fcpd_apply_transform": (C.c_int, [vp, P, I64, I32, P, I64, P, I64, I32, P]),
            "fcpd_estimated_targets": (C.c_int, [vp, P, I64, I64, P, I64, I32, P]),
            "fcpd_enforce_row_constraint": (C.c_int, [vp, P, I64, I64, PI32]),
            "fcpd_update_sigma2": (C.c_int, [vp, P, I64, P, I64, I64, P, I64, I32, I32, P]),
            "fcpd_eigendecompose": (C.c_int, [vp, P, I64, I64, P, P, P]),
            "fcpd_lowrank_reconstruction_error": (C.c_int, [vp, P, I64, P, I64, P, I64, P]),
            "fcpd_normalize_pair": (C.c_int, [vp, P, I64, I32, P, I64, I32, P, P, P, P, PI32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _pi32(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


def _colmajor(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a)


# ----------------------------------------------------- registration.hpp types
@dataclass
class RegistrationConfig:  # registration.hpp:30-40
    omega: float = 0.7
    beta: float = 2.0
    lambda_reg: float = 10.0
    iterations: int = 100
    variant: str = "fast"
    rank_fraction: float = 0.1
    seed: int = 0
    normalize: bool = True
    early_stop: bool = False
    # extension: skip eigenpairs whose spectral filter is below tau in the
    # per-iteration basis streams (0 = stream all K)
    spectral_tau: float = 1e-10

    def _c(self) -> _Config:
        return _Config(self.omega, self.beta, self.lambda_reg, int(self.iterations),
                       VARIANTS[variant_from_string(self.variant)], self.rank_fraction,
                       int(self.seed), int(bool(self.normalize)), int(bool(self.early_stop)), 0,
                       float(self.spectral_tau))


@dataclass
class TimingBreakdown:  # registration.hpp:21-28 (+ t_setup)
    t_c: float = 0.0
    t_eig: float = 0.0
    t_iter: float = 0.0
    t_f: float = 0.0
    t_o: float = 0.0
    t_total: float = 0.0
    t_setup: float = 0.0


@dataclass
class RegistrationResult:  # registration.hpp:48-56
    transformed: np.ndarray
    coefficients: np.ndarray
    sigma2_trace: np.ndarray
    sigma2_initial: float
    timing: TimingBreakdown
    degenerate_rows: int = 0
    sigma2_clamps: int = 0
    correspondence: Optional[np.ndarray] = None
    degenerate_mask: Optional[np.ndarray] = None
    basis_reused: bool = False
    baseline_solver: str = "dense LDLT factorization"
    h2d_bytes: int = 0
    d2h_bytes: int = 0


# ------------------------------------------------------------------ context
def nccl_unique_id() -> bytes:
    """128-byte NCCL id for fcpd_create_dist (rank 0 makes it, all ranks share it)."""
    buf = C.create_string_buffer(128)
    if lib().fcpd_nccl_unique_id(buf) != 0:
        raise CudaError("ncclGetUniqueId failed")
    return buf.raw


class Context:
    """One CUDA device: stream, cuSOLVER handle, cached basis, graphs.

    ``Context.distributed(device, rank, world, uid)`` joins a multi-GPU
    group (one process per GPU): register/session calls then take the full
    model and this rank's scene shard (see include/fcpd_capi.h)."""

    def __init__(self, device: int = 0, *, _dist=None, _loopback=None):
        self._h = C.c_void_p()
        if _loopback is not None:
            rc = lib().fcpd_create_loopback(C.byref(self._h), int(device), int(_loopback))
            if rc != 0:
                raise _CODES.get(rc, Error)(f"fcpd_create_loopback failed (code {rc})")
        elif _dist is None:
            self._check(lib().fcpd_create(C.byref(self._h), int(device)))
        else:
            rank, world, uid = _dist
            rc = lib().fcpd_create_dist(C.byref(self._h), int(device), int(rank), int(world),
                                        bytes(uid))
            if rc != 0:
                raise _CODES.get(rc, Error)(f"fcpd_create_dist failed (code {rc})")

    @classmethod
    def distributed(cls, device: int, rank: int, world: int, uid: bytes) -> "Context":
        return cls(device, _dist=(rank, world, uid))

    @classmethod
    def loopback(cls, device: int, world: int) -> "Context":
        """`world` virtual ranks of the scene-sharded path on one device
        (collectives as device kernels); register/session take the FULL
        scene, split into contiguous shards."""
        return cls(device, _loopback=world)

    @property
    def world(self):
        r, w = C.c_int32(), C.c_int32()
        lib().fcpd_world(self._h, C.byref(r), C.byref(w))
        return r.value, w.value

    def close(self):
        if self._h:
            lib().fcpd_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc: int):
        if rc != 0:
            msg = lib().fcpd_last_error(self._h) if self._h else b"fcpd_create failed"
            raise _CODES.get(rc, Error)((msg or b"").decode())

    # -- register_pointsets (registration.hpp:79-175)
    def register(self, x, y, cfg: RegistrationConfig = None, *,
                 want_correspondence: bool = False) -> RegistrationResult:
        cfg = cfg or RegistrationConfig()
        x, y = _colmajor(x), _colmajor(y)
        if x.shape[1] != y.shape[1]:
            raise DimensionError("register: model and scene dimension mismatch")
        m, d = x.shape
        n = y.shape[0]
        out_x = np.zeros((m, d), order="F")
        out_w = np.zeros((m, d), order="F")
        trace = np.zeros(max(int(cfg.iterations), 1))
        corr = np.zeros((m, n), order="F") if want_correspondence else None
        mask = np.zeros(m, dtype=np.int32)
        res = _Result(_p(out_x), _p(out_w), _p(trace), _p(corr), _pi32(mask))
        c = cfg._c()
        self._check(lib().fcpd_register(self._h, _p(x), m, _p(y), n, d, C.byref(c),
                                        C.byref(res)))
        t = res.timing
        # (M, D) results as filled by the C ABI (column-major, like the input
        # it was given); a C-order copy would cost a transpose per call
        return RegistrationResult(
            out_x, out_w,
            trace[: res.iterations_run].copy(), res.sigma2_initial,
            TimingBreakdown(t.t_c, t.t_eig, t.t_iter, t.t_f, t.t_o, t.t_total, t.t_setup),
            int(res.degenerate_rows), int(res.sigma2_clamps), corr, mask.astype(bool),
            bool(res.basis_reused), h2d_bytes=int(res.h2d_bytes), d2h_bytes=int(res.d2h_bytes))

    # -- device-resident session (bench / serving)
    def session_begin(self, x, y, cfg: RegistrationConfig):
        x, y = _colmajor(x), _colmajor(y)
        if x.shape[1] != y.shape[1]:
            raise DimensionError("register: model and scene dimension mismatch")
        self._sess = (x.shape[0], x.shape[1], cfg)
        c = cfg._c()
        self._check(lib().fcpd_session_begin(self._h, _p(x), x.shape[0], _p(y), y.shape[0],
                                             x.shape[1], C.byref(c)))

    def session_run(self, iterations: int):
        self._check(lib().fcpd_session_run(self._h, int(iterations)))

    def session_sync(self):
        self._check(lib().fcpd_session_sync(self._h))

    PHASES = ("estep_pass1", "estep_pass2", "qt_r_stream", "zreduce_filter", "q_g_stream",
              "transform_sigma2")

    def session_profile(self, iterations: int) -> dict:
        """Mean ms per kernel group over `iterations` eager iterations (CUDA
        events on the context stream)."""
        ms = np.zeros(6)
        self._check(lib().fcpd_session_profile(self._h, int(iterations), _p(ms)))
        return dict(zip(self.PHASES, ms.tolist()))

    def session_read(self, with_points=True) -> dict:
        m, d, cfg = self._sess
        out_x = np.zeros((m, d), order="F") if with_points else None
        trace = np.zeros(max(int(cfg.iterations), 1))
        res = _Result(_p(out_x), None, _p(trace), None, None)
        self._check(lib().fcpd_session_read(self._h, C.byref(res)))
        return dict(transformed=None if out_x is None else np.ascontiguousarray(out_x),
                    sigma2_trace=trace[: res.iterations_run].copy(),
                    iterations_run=res.iterations_run, degenerate_rows=res.degenerate_rows,
                    tiles_evaluated=(int(res.tiles_evaluated[0]), int(res.tiles_evaluated[1])),
                    pairs_by_form=tuple(int(v) for v in res.pairs_by_form),
                    spectral_rank=int(res.spectral_rank),
                    mstep_fused=bool(res.mstep_fused),
                    # device-stamped phase sums over the run (s): E-step, and
                    # the M-step from the z pass to the transform
                    t_c=float(res.timing.t_c), t_iter=float(res.timing.t_iter))

    @property
    def stream_ptr(self) -> int:
        return lib().fcpd_stream(self._h) or 0

    @property
    def kernels_per_iteration(self) -> int:
        return int(lib().fcpd_kernels_per_iteration(self._h))

    # -- L2 entry points (correspondence.hpp, kernel.hpp, solvers.hpp)
    def estep(self, xt, y, omega: float, sigma2: float) -> dict:
        xt, y = _colmajor(xt), _colmajor(y)
        if xt.shape[1] != y.shape[1]:
            raise DimensionError("posterior: dimension mismatch")
        m, d = xt.shape
        n = y.shape[0]
        pty = np.zeros((m, d), order="F")
        p1, var, pt1 = np.zeros(m), np.zeros(m), np.zeros(n)
        deg = np.zeros(m, dtype=np.int32)
        cl = C.c_int32()
        self._check(lib().fcpd_estep(self._h, _p(xt), m, _p(y), n, d, omega, sigma2, _p(pty),
                                     _p(p1), _p(var), _pi32(deg), _p(pt1), C.byref(cl)))
        return dict(ptilde_y=np.ascontiguousarray(pty), p1=p1, var=var,
                    degenerate=deg.astype(bool), pt1=pt1, clamped=bool(cl.value))

    def posterior(self, xt, y, omega: float, sigma2: float, row_constrain: bool = False):
        xt, y = _colmajor(xt), _colmajor(y)
        if xt.shape[1] != y.shape[1]:
            raise DimensionError("posterior: dimension mismatch")
        m, d = xt.shape
        n = y.shape[0]
        p = np.zeros((m, n), order="F")
        cl = C.c_int32()
        rows = np.zeros(m, dtype=np.int64)
        nd = C.c_int64()
        self._check(lib().fcpd_posterior_dense(
            self._h, _p(xt), m, _p(y), n, d, omega, sigma2, int(row_constrain), _p(p),
            C.byref(cl), rows.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(nd)))
        return p, bool(cl.value), rows[: nd.value].tolist()

    def build_gram(self, x, beta: float) -> np.ndarray:
        x = _colmajor(x)
        m, d = x.shape
        phi = np.zeros((m, m), order="F")
        self._check(lib().fcpd_build_gram(self._h, _p(x), m, d, beta, _p(phi)))
        return phi

    def build_basis(self, x, beta: float, rank: int):
        x = _colmajor(x)
        m, d = x.shape
        u = np.zeros((m, rank), order="F")
        lam, raw = np.zeros(rank), np.zeros(rank)
        self._check(lib().fcpd_build_basis(self._h, _p(x), m, d, beta, int(rank), _p(u),
                                           _p(lam), _p(raw)))
        return u, lam, raw

    def save_spectral_cache(self, path: str):
        """Write the context's current basis in the reference format (kernel.hpp:92-110)."""
        self._check(lib().fcpd_save_spectral_cache(self._h, os.fsencode(path)))

    def load_spectral_cache(self, path: str, x, y, cfg: RegistrationConfig):
        """Install a cached basis for register(x, y, cfg) (kernel.hpp:112-144)."""
        x, y = _colmajor(x), _colmajor(y)
        c = cfg._c()
        self._check(lib().fcpd_load_spectral_cache(self._h, os.fsencode(path), _p(x), x.shape[0],
                                                   _p(y), y.shape[0], x.shape[1], C.byref(c)))

    def build_basis_topk(self, x, beta: float, rank: int, iterations: int = 0):
        """Top-K eigenpairs of Φ without forming it (configs 2–4 setup)."""
        x = _colmajor(x)
        m, d = x.shape
        u = np.zeros((m, rank), order="F")
        lam, raw = np.zeros(rank), np.zeros(rank)
        self._check(lib().fcpd_build_basis_topk(self._h, _p(x), m, d, beta, int(rank),
                                                int(iterations), _p(u), _p(lam), _p(raw)))
        return u, lam, raw

    # fp64 device restatements of the reference's L2 functions (l2api.cu)
    def solve_fast_lowrank(self, u, lam, lambda_reg: float, sigma2: float, residual):
        """solvers.hpp:61-73 — W = U diag(1/(λ+λσ²)) Uᵀ R."""
        u = np.asfortranarray(u, dtype=np.float64)
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        r = _colmajor(residual)
        m, k = u.shape
        w = np.zeros(r.shape, order="F")
        self._check(lib().fcpd_solve_fast_lowrank(self._h, _p(u), _p(lam), m, k, lambda_reg,
                                                  sigma2, _p(r), r.shape[0], r.shape[1], _p(w)))
        return np.ascontiguousarray(w)

    def solve_fast(self, u, lam, lambda_reg: float, sigma2: float, residual):
        """solvers.hpp:75-80 (full basis)."""
        u = np.asarray(u)
        if u.shape[0] != u.shape[1]:
            raise ParameterError("solve_fast expects the full spectral basis")
        return self.solve_fast_lowrank(u, lam, lambda_reg, sigma2, residual)

    def apply_transform_lowrank(self, x, u, lam, w):
        """solvers.hpp:147-155 — X + U Λ Uᵀ W."""
        x, w = _colmajor(x), _colmajor(w)
        u = np.asfortranarray(u, dtype=np.float64)
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        m, d = x.shape
        out = np.zeros((m, d), order="F")
        self._check(lib().fcpd_apply_transform_lowrank(self._h, _p(x), m, d, _p(u), u.shape[0],
                                                       _p(lam), u.shape[1], _p(w), w.shape[0],
                                                       w.shape[1], _p(out)))
        return np.ascontiguousarray(out)

    def apply_transform(self, x, phi, w):
        """solvers.hpp:138-144 — X + Φ W."""
        x, w = _colmajor(x), _colmajor(w)
        phi = np.asfortranarray(phi, dtype=np.float64)
        m, d = x.shape
        out = np.zeros((m, d), order="F")
        self._check(lib().fcpd_apply_transform(self._h, _p(x), m, d, _p(phi), phi.shape[0],
                                               _p(w), w.shape[0], w.shape[1], _p(out)))
        return np.ascontiguousarray(out)

    def estimated_targets(self, p, y):
        """correspondence.hpp:101-105 — P·Y."""
        p = np.asfortranarray(p, dtype=np.float64)
        y = _colmajor(y)
        out = np.zeros((p.shape[0], y.shape[1]), order="F")
        self._check(lib().fcpd_estimated_targets(self._h, _p(p), p.shape[0], p.shape[1], _p(y),
                                                 y.shape[0], y.shape[1], _p(out)))
        return np.ascontiguousarray(out)

    def enforce_row_constraint(self, p):
        """correspondence.hpp:83-98 — (P̃, degenerate row indices)."""
        q = np.array(p, dtype=np.float64, order="F", copy=True)
        deg = np.zeros(q.shape[0], dtype=np.int32)
        self._check(lib().fcpd_enforce_row_constraint(self._h, _p(q), q.shape[0], q.shape[1],
                                                      _pi32(deg)))
        return q, np.nonzero(deg)[0].tolist()

    def update_sigma2(self, y, p, xt, row_constrained: bool = True) -> float:
        """solvers.hpp:160-176 (trace form)."""
        y, xt = _colmajor(y), _colmajor(xt)
        p = np.asfortranarray(p, dtype=np.float64)
        out = C.c_double()
        self._check(lib().fcpd_update_sigma2(self._h, _p(y), y.shape[0], _p(p), p.shape[0],
                                             p.shape[1], _p(xt), xt.shape[0], xt.shape[1],
                                             int(bool(row_constrained)), C.byref(out)))
        return out.value

    def eigendecompose(self, phi, rank: int):
        """kernel.hpp:49-72 of a given Φ — (U, λ clamped, λ raw)."""
        phi = np.asfortranarray(phi, dtype=np.float64)
        m = phi.shape[0]
        u = np.zeros((m, rank), order="F")
        lam, raw = np.zeros(rank), np.zeros(rank)
        self._check(lib().fcpd_eigendecompose(self._h, _p(phi), m, int(rank), _p(u), _p(lam),
                                              _p(raw)))
        return u, lam, raw

    def lowrank_reconstruction_error(self, u, lam, phi) -> float:
        """kernel.hpp:76-83 — ‖Φ − U Λ Uᵀ‖_F."""
        phi = np.asfortranarray(phi, dtype=np.float64)
        u = np.asfortranarray(u, dtype=np.float64)
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        out = C.c_double()
        self._check(lib().fcpd_lowrank_reconstruction_error(
            self._h, _p(phi), phi.shape[0], _p(u), u.shape[0], _p(lam), u.shape[1],
            C.byref(out)))
        return out.value

    def normalize_pair(self, x, y):
        """pointset.hpp:124-148 — (x', y', center, scale, degenerate)."""
        x, y = _colmajor(x), _colmajor(y)
        xo, yo = np.zeros(x.shape, order="F"), np.zeros(y.shape, order="F")
        c = np.zeros(max(x.shape[1], 1))
        sc = C.c_double()
        deg = C.c_int32()
        self._check(lib().fcpd_normalize_pair(self._h, _p(x), x.shape[0], x.shape[1], _p(y),
                                              y.shape[0], y.shape[1], _p(xo), _p(yo), _p(c),
                                              C.byref(sc), C.byref(deg)))
        return (np.ascontiguousarray(xo), np.ascontiguousarray(yo), c[: x.shape[1]], sc.value,
                bool(deg.value))


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def register_pointsets(x, y, cfg: RegistrationConfig = None, **kw) -> RegistrationResult:
    """registration.hpp:79-175 on the B200 (module-level convenience)."""
    return default_context().register(x, y, cfg, **kw)
