"""Per-iteration trace of a bench workload: σ², device time and the fraction
of tile pairs each E-step pass evaluated (culling).  Diagnostic only.

  python tools/cull_trace.py c2 [iterations]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_06281_b200 as fcpd  # noqa: E402
from paper_2006_06281_b200 import datagen  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
    x, y, w = datagen.generate(wl)
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else w.iterations
    ctx = fcpd.Context(0)
    cfg = datagen.config_for(w, iterations=iters)
    ctx.session_begin(x, y, cfg)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", 0))
    flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")
    tiles_total = fcpd.cull_units_total(x.shape[0], y.shape[0])
    prev = ctx.session_read(with_points=False)["tiles_evaluated"]
    rows = []
    for i in range(iters):
        with torch.cuda.stream(stream):
            flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.session_run(1)
        e1.record(stream)
        e1.synchronize()
        st = ctx.session_read(with_points=False)
        t = st["tiles_evaluated"]
        rows.append({"it": i, "ms": e0.elapsed_time(e1), "sigma2": float(st["sigma2_trace"][-1]),
                     "f1": (t[0] - prev[0]) / tiles_total[0] or 1.0,
                     "f2": (t[1] - prev[1]) / tiles_total[1] or 1.0,
                     "keff": st["spectral_rank"]})
        prev = t
    tot = sum(r["ms"] for r in rows)
    print(json.dumps({"workload": wl, "iterations": iters, "total_ms": tot,
                      "it_per_s": iters / tot * 1e3, "trace": rows}))
    ctx.close()


if __name__ == "__main__":
    main()
