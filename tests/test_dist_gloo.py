"""World-size-2 and -4 CPU tests of the multi-GPU decomposition.

The device path (engine.cu enqueue_iteration_group + csrc/dist.cu) splits
one EM iteration into per-rank work and, in the common case, THREE
collectives:

  pass 1        column-local over the rank's scene shard (no communication)
  pass 2        per-row partial sums (S0, Σw·y, Σw·d²) over local columns
                → reduce-scatter to the row-shard owners
  own rows      finalised; rows whose global mass is too small for the fp32
                fast path are flagged and get a zero residual for now
  M-step        z_r = Q_rᵀ R_r → all-reduce, carrying the flagged-row count
  fallback      only if the count is nonzero (a conditional graph node):
                all-gather of the flags, all-reduce MAX of the flagged rows'
                max log-posterior, reduce-scatter of the shifted sums, the
                flagged rows' z correction → all-reduce
  x̃             V_r = Q_r (f⊙z), x̃ own rows, σ² partial of the own rows;
                all-gather of x̃ with the σ² partials riding along; every
                rank sums the partials in rank order
  normalize     global centroid / max-abs / scene moments (host all-reduce)

This test runs exactly that decomposition in fp64 numpy on gloo ranks and
checks it against the unsharded oracle restatement of register_pointsets.
(gloo has no reduce-scatter: all-reduce + taking the own rows is the same
reduction.)  `flag_below` forces the flagged path for rows whose mass is
below it, so the fallback exchange is exercised.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(a, op=dist.ReduceOp.SUM):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_reduce(t, op=op)
    return t.numpy()


def sharded_register(x, y_shard, rank, world, omega, beta, lam_reg, iters, u, lam_raw, lam_c,
                     full_rank, flag_below=0.0):
    m, d = x.shape
    n_loc = y_shard.shape[0]
    # normalize_pair with global statistics (pointset.hpp:124-148)
    red = _allreduce(np.concatenate([[n_loc], y_shard.sum(0)]))
    n = int(red[0])
    center = (x.sum(0) + red[1:]) / (m + n)
    sc = max(np.abs(x - center).max(), np.abs(y_shard - center).max())
    sc = float(_allreduce(np.array([sc]), dist.ReduceOp.MAX)[0])
    sc = sc if sc > 0 else 1.0
    X = (x - center) / sc
    Y = (y_shard - center) / sc
    mom = _allreduce(np.concatenate([Y.sum(0), [(Y ** 2).sum()]]))
    ymean, ysq = mom[:3] / n, mom[3] / n
    # init_sigma2 (registration.hpp:59-69)
    s2 = max((m * mom[3] + n * (X ** 2).sum() - 2 * X.sum(0) @ mom[:3]) / (d * m * n), 0.0)
    # row shard
    mr = (m + world - 1) // world
    m0, m1 = rank * mr, min(m, rank * mr + mr)
    U = u[m0:m1]
    k = U.shape[1]
    lam_num = lam_raw if full_rank else lam_c
    xt = X.copy()
    trace = []
    fallbacks = 0
    for _ in range(iters):
        s2e = max(s2, 1e-10)
        d2 = ((Y[None, :, :] - xt[:, None, :]) ** 2).sum(-1)  # M × n_loc
        e = -d2 / (2 * s2e)
        shift = e.max(0)
        if omega > 0:
            log_c = 0.5 * d * math.log(2 * math.pi * s2e) + math.log(omega / (1 - omega)) \
                + math.log(m / n)
            shift = np.maximum(shift, log_c)
        E = np.exp(e - shift)
        den = E.sum(0) + (np.exp(log_c - shift) if omega > 0 else 0.0)
        P = E / den                                          # pass 1: column-local
        logP = e - shift - np.log(den)
        part = np.column_stack([P.sum(1), P @ Y, (P * d2).sum(1)])  # pass 2 partials
        S = _allreduce(part)[m0:m1]                          # collective 1: "reduce-scatter"
        flag = S[:, 0] < flag_below                          # mass too small: fallback
        xo = xt[m0:m1]

        def finalize(S, rows):
            deg = S[:, 0] < 1e-300
            pty = np.where(deg[:, None], ymean, S[:, 1:4] / np.where(deg, 1, S[:, 0])[:, None])
            xr = xo[rows]
            var = np.where(deg, ysq - 2 * xr @ ymean + (xr ** 2).sum(1),
                           S[:, 4] / np.where(deg, 1, S[:, 0]))
            return pty, var

        pty, var = finalize(S, slice(None))
        R = pty - X[m0:m1]
        R[flag] = 0.0                                        # filled by the fallback
        zc = np.concatenate([(U.T @ R).ravel(), [flag.sum()]])
        zc = _allreduce(zc)                                  # collective 2: z + flagged count
        z = zc[:-1].reshape(k, 3)
        if zc[-1] > 0:                                       # the conditional fallback
            fallbacks += 1
            mask = np.zeros(world * mr)
            mask[m0:m0 + (m1 - m0)] = flag
            mask = _allreduce(mask)[:m] > 0                  # "all-gather" of the flags
            lmax = np.where(mask, (logP.max(1) if n_loc else -np.inf), -np.inf)
            lmax = _allreduce(lmax, dist.ReduceOp.MAX)       # max log P over all columns
            W = np.exp(logP - np.where(mask, lmax, 0.0)[:, None]) * mask[:, None]
            fs = np.column_stack([W.sum(1), W @ Y, (W * d2).sum(1)])
            fs = _allreduce(fs)[m0:m1]                       # "reduce-scatter" shifted sums
            fpty, fvar = finalize(fs, slice(None))
            pty[flag], var[flag] = fpty[flag], fvar[flag]
            R[flag] = pty[flag] - X[m0:m1][flag]
            Rc = np.where(flag[:, None], R, 0.0)
            z = z + _allreduce(U.T @ Rc)                     # z correction
        diag = lam_c + lam_reg * s2
        assert diag.min() > 0
        g = z * (lam_num / diag)[:, None]
        xn = X[m0:m1] + U @ g
        dlt = xn - xo
        term = (var - 2 * (dlt * (pty - xo)).sum(1) + (dlt ** 2).sum(1)).sum()
        # collective 3: all-gather x̃ with the σ² partial riding along
        own = torch.zeros(mr + 1, 3, dtype=torch.float64)
        own[: m1 - m0] = torch.from_numpy(xn)
        own[mr, 0] = term
        gathered = [torch.zeros(mr + 1, 3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, own)
        val = sum(float(gv[mr, 0]) for gv in gathered) / (d * m)   # rank order
        nxt = max(val, 1e-10)
        trace.append(nxt)
        s2 = nxt
        xt = torch.cat([gv[:mr] for gv in gathered]).numpy()[:m]
    return np.array(trace), xt * sc + center, fallbacks


def _worker(rank, world, port, q, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc
    x = orc.make_torus(case["m"], 11)
    y = orc.make_torus(case["n"], 12) * np.array([1.1, 0.95, 1.0]) + 0.03
    xn, yn, _, _, _ = orc.normalize_pair(x, y)
    phi = orc.build_gram(xn, case["beta"])
    k = case["m"] if case["full"] else case["k"]
    u, lam_c, lam_raw = orc.eigendecompose(phi, k)
    n = y.shape[0]
    y_shard = y[rank * n // world:(rank + 1) * n // world]
    trace, pts, fb = sharded_register(x, y_shard, rank, world, case["omega"], case["beta"],
                                      case["lam"], case["iters"], u, lam_raw, lam_c, case["full"],
                                      case.get("flag_below", 0.0))
    q.put((rank, trace, pts, fb))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, dict(m=120, n=150, omega=0.0, beta=2.0, lam=3.0, iters=12, full=True, k=120)),
    (2, dict(m=121, n=149, omega=0.3, beta=2.0, lam=3.0, iters=12, full=False, k=20)),
    (4, dict(m=122, n=151, omega=0.1, beta=2.0, lam=3.0, iters=10, full=False, k=24)),
    # rows with mass below one point take the fallback exchange
    (2, dict(m=120, n=150, omega=0.2, beta=2.0, lam=3.0, iters=10, full=True, k=120,
             flag_below=1.0)),
])
def test_sharded_em_matches_oracle(orc, world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, case)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = orc.make_torus(case["m"], 11)
    y = orc.make_torus(case["n"], 12) * np.array([1.1, 0.95, 1.0]) + 0.03
    ref = orc.register(x, y, omega=case["omega"], beta=case["beta"], lambda_reg=case["lam"],
                       iterations=case["iters"],
                       variant="fast" if case["full"] else "fast_lowrank",
                       rank_fraction=case["k"] / case["m"])
    for _, trace, pts, fb in res:
        assert np.allclose(trace, ref.sigma2_trace, rtol=1e-10, atol=0)
        assert np.abs(pts - ref.transformed).max() <= 1e-10
        assert (fb > 0) == (case.get("flag_below", 0.0) > 0)
    # every rank ends with the same full result
    for r in res[1:]:
        assert np.array_equal(res[0][2], r[2])


# ---------------------------------------------------------------------------
# The group's top-K setup (engine.cu group_topk_basis, topk.cu
# gram_matmul_sharded): every Φ·V product is row-sharded — rank r forms rows
# [r·M_b, (r+1)·M_b) — and all-gathered; the b×b / M×b algebra and the
# adaptive stop (every top-K Ritz residual ≤ 1e-11·θ₁, max-reduced over the
# ranks) are replicated.  kernel.hpp:49-72.

def topk_adaptive(x, beta, rank, product, max_steps=4, tol=1e-11, seed=7, agree=None):
    """The device's adaptive randomized subspace iteration in fp64 numpy;
    `product(V)` returns Φ·V; `agree(worst)` makes the stop decision common."""
    m = x.shape[0]
    b = min(m, rank + max(16, rank // 5))
    v, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((m, b)))
    products = 0
    for step in range(max_steps + 1):
        w = product(v)
        products += 1
        if step < 1 and step < max_steps:
            v, _ = np.linalg.qr(w)
            continue
        t = v.T @ w
        theta, s = np.linalg.eigh(0.5 * (t + t.T))
        s_top, th = s[:, -rank:], theta[-rank:]
        u = v @ s_top
        if step >= max_steps:
            break
        res = np.linalg.norm(w @ s_top - u * th, axis=0).max()
        worst = agree(res) if agree else res
        if worst <= tol * abs(theta[-1]):
            break
        v, _ = np.linalg.qr(w)
    return u[:, ::-1], th[::-1], products


def _topk_worker(rank, world, port, q, m, k):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc
    x = orc.normalize_pair(orc.make_torus(m, 21), orc.make_torus(m, 22))[0]
    rows = -(-m // world)  # block rows per rank

    def product(v):
        mine = np.arange(rank * rows, min((rank + 1) * rows, m))
        blk = np.zeros((rows, v.shape[1]))
        blk[:len(mine)] = orc.gram_apply(x, 2.0, v, rows=mine)
        out = [torch.zeros(rows, v.shape[1], dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(blk))
        return torch.cat(out).numpy()[:m]

    def agree(worst):
        return float(_allreduce(np.array([worst]), op=dist.ReduceOp.MAX)[0])

    u, lam, products = topk_adaptive(x, 2.0, k, product, agree=agree)
    q.put((rank, u, lam, products))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_topk_setup_matches_unsharded(orc, world):
    m, k = 900, 40
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_topk_worker, args=(r, world, port, q, m, k)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = orc.normalize_pair(orc.make_torus(m, 21), orc.make_torus(m, 22))[0]
    u1, lam1, p1 = topk_adaptive(x, 2.0, k, lambda v: orc.gram_apply(x, 2.0, v))
    for _, u, lam, products in res:
        # row-sharded products are the unsharded rows: the same basis, bit for bit
        assert products == p1
        assert np.array_equal(lam, lam1) and np.array_equal(u, u1)
    # and it is the top-K eigenbasis of Φ (LAPACK on the dense Gram matrix)
    phi = orc.build_gram(x, 2.0)
    _, _, raw = orc.eigendecompose(phi, k)
    assert np.abs(lam1 - raw).max() <= 1e-10 * raw[0]
