"""Per-iteration device phase split (E-step, M-step to V, transform + σ²)
from the engine timestamps, fused vs streaming M-step, C1.  Diagnostic."""
import os, sys
sys.path.insert(0, '/root/repo')
import paper_2006_06281_b200 as fcpd
from paper_2006_06281_b200 import datagen
x, y, w = datagen.generate(sys.argv[1] if len(sys.argv) > 1 else 'c1')
ctx = fcpd.Context(0)
for fused in ('1', '0'):
    os.environ['FCPD_MSTEP_FUSED'] = fused
    cfg = datagen.config_for(w, iterations=100)
    r = ctx.register(x, y, cfg)
    r = ctx.register(x, y, cfg)
    t = r.timing
    print(w.name if hasattr(w, 'name') else '', 'fused' if fused == '1' else 'stream', {k: round(getattr(t, k) * 1e4, 2) for k in ('t_c', 't_iter', 't_o')}, '(us per iteration)')
