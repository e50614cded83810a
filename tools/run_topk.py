"""Time the top-K eigensolver alone on a workload's normalised model (setup
profiling helper: python tools/run_topk.py c2)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2006_06281_b200 as fc  # noqa: E402
from paper_2006_06281_b200 import datagen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
x, y, w = datagen.generate(name)
with fc.Context(0) as ctx:
    xn = ctx.normalize_pair(x, y)[0]
    k = int(round(w.rank_fraction * w.m))
    t = time.perf_counter()
    u, lam, raw = ctx.build_basis_topk(xn, w.beta, k)
    print(f"{name}: M={w.m} K={k} topk {time.perf_counter() - t:.3f} s, lam1 {raw[0]:.6e}, "
          f"resolved {(lam > 0).sum()}")
