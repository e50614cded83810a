"""Where does a register_pointsets call spend its host time? (diagnostic)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06281_b200 as fcpd  # noqa: E402
from paper_2006_06281_b200 import datagen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
x, y, w = datagen.generate(name)
cfg = datagen.config_for(w)
ctx = fcpd.Context(0)
t0 = time.perf_counter()
r = ctx.register(x, y, cfg)
print(f"first register {time.perf_counter() - t0:.3f}s setup={r.timing.t_setup:.3f}s")
for _ in range(3):
    t0 = time.perf_counter()
    ctx.session_begin(x, y, cfg)
    t1 = time.perf_counter()
    ctx.session_run(cfg.iterations)
    ctx.session_sync()
    t2 = time.perf_counter()
    ctx.session_read()
    t3 = time.perf_counter()
    r = ctx.register(x, y, cfg)
    t4 = time.perf_counter()
    print(f"begin {1e3*(t1-t0):.1f} ms  run+sync {1e3*(t2-t1):.1f} ms  read {1e3*(t3-t2):.1f} ms"
          f"  register {1e3*(t4-t3):.1f} ms  (t_c {1e3*r.timing.t_c:.1f} t_iter "
          f"{1e3*r.timing.t_iter:.1f} t_o {1e3*r.timing.t_o:.1f} reused {r.basis_reused})")
