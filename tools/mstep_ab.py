"""Fused vs streaming M-step on one workload, for an ncu launch list.
Diagnostic only:  python tools/mstep_ab.py c1 [iterations]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2006_06281_b200 as fcpd  # noqa: E402
from paper_2006_06281_b200 import datagen  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
x, y, w = datagen.generate(wl)
ctx = fcpd.Context(0)
for fused in ("0", "1"):
    os.environ["FCPD_MSTEP_FUSED"] = fused
    ctx.session_begin(x, y, datagen.config_for(w, iterations=iters))
    ctx.session_run(iters)
    ctx.session_sync()
    print(wl, "fused" if fused == "1" else "stream", ctx.session_read(with_points=False)["sigma2_trace"][-1])
ctx.close()
