"""World-size-2 CPU test of the multi-GPU decomposition.

The device path (csrc/dist.cu + engine.cu enqueue_iteration_dist) splits one
EM iteration into per-rank work and collectives:

  pass 1        column-local over the rank's scene shard (no communication)
  pass 2        per-row partial sums (S0, Σw·y, Σw·d²) over local columns
                → reduce-scatter to the row-shard owners
  M-step        z_r = Q_rᵀ R_r → all-reduce; V_r = Q_r (f⊙z) on own rows
  σ²            per-row terms on own rows → all-reduce
  x̃             all-gather
  normalize     global centroid / max-abs / scene moments via all-reduce

This test runs exactly that decomposition in fp64 numpy on 2 gloo ranks and
checks it against the unsharded oracle restatement of register_pointsets.
(gloo has no reduce-scatter: all-reduce + taking the own rows is the same
reduction.)
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
                     full_rank):
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
    lam_num = lam_raw if full_rank else lam_c
    xt = X.copy()
    trace = []
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
        part = np.column_stack([P.sum(1), P @ Y, (P * d2).sum(1)])  # pass 2 partials
        S = _allreduce(part)[m0:m1]                          # "reduce-scatter"
        deg = S[:, 0] < 1e-300
        pty = np.where(deg[:, None], ymean, S[:, 1:4] / np.where(deg, 1, S[:, 0])[:, None])
        xo = xt[m0:m1]
        var = np.where(deg, ysq - 2 * xo @ ymean + (xo ** 2).sum(1),
                       S[:, 4] / np.where(deg, 1, S[:, 0]))
        R = pty - X[m0:m1]
        z = _allreduce(U.T @ R)                              # all-reduce K×3
        diag = lam_c + lam_reg * s2
        assert diag.min() > 0
        g = z * (lam_num / diag)[:, None]
        xn = X[m0:m1] + U @ g
        dlt = xn - xo
        term = (var - 2 * (dlt * (pty - xo)).sum(1) + (dlt ** 2).sum(1)).sum()
        val = float(_allreduce(np.array([term]))[0]) / (d * m)
        nxt = max(val, 1e-10)
        trace.append(nxt)
        s2 = nxt
        gathered = [torch.zeros(mr, 3, dtype=torch.float64) for _ in range(world)]
        own = torch.zeros(mr, 3, dtype=torch.float64)
        own[: m1 - m0] = torch.from_numpy(xn)
        dist.all_gather(gathered, own)                       # all-gather x̃
        xt = torch.cat(gathered).numpy()[:m]
    return np.array(trace), xt * sc + center


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
    trace, pts = sharded_register(x, y_shard, rank, world, case["omega"], case["beta"],
                                  case["lam"], case["iters"], u, lam_raw, lam_c, case["full"])
    q.put((rank, trace, pts))
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    dict(m=120, n=150, omega=0.0, beta=2.0, lam=3.0, iters=12, full=True, k=120),
    dict(m=121, n=149, omega=0.3, beta=2.0, lam=3.0, iters=12, full=False, k=20),
])
def test_two_rank_sharded_em_matches_oracle(orc, case):
    world = 2
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
    for _, trace, pts in res:
        assert np.allclose(trace, ref.sigma2_trace, rtol=1e-10, atol=0)
        assert np.abs(pts - ref.transformed).max() <= 1e-10
    # every rank ends with the same full result
    assert np.array_equal(res[0][2], res[1][2])
